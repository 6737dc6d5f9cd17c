OUT=gpurun_out/${TAG:-r02h}; mkdir -p $OUT
./tools/microbench/lds_pattern > $OUT/lds_pattern.txt 2>&1
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum --csv ./tools/microbench/lds_pattern > $OUT/lds_pattern_ncu.csv 2>&1
TDG_LIB_PATH=abtest/lib_W.so TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -rs --deselect tests/test_gpu_dist_two_rank.py::test_two_ranks_one_gpu_match_single_rank > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash tools/ab_libs.sh $OUT detect S W
nvidia-smi > $OUT/smi_end.txt 2>&1
