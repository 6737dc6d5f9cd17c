OUT=gpurun_out/${TAG:-r02l}; mkdir -p $OUT
TDG_LIB_PATH=abtest/lib_${PV}.so TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -rs --deselect tests/test_gpu_dist_two_rank.py::test_two_ranks_one_gpu_match_single_rank > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash tools/ab_libs.sh $OUT detect ${VARS}
TDG_LIB_PATH=abtest/lib_${PV}.so python tools/sweep.py "" "wave_pairs=10,ring=3" "wave_pairs=12,ring=3" "wave_pairs=16,ring=2" "wave_pairs=16,ring=3" "wave_pairs=6,ring=4" "wave_pairs=8,ring=3" > $OUT/sweep.txt 2>&1
nvidia-smi > $OUT/smi_end.txt 2>&1
