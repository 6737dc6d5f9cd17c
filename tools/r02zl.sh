OUT=gpurun_out/${TAG:-r02zl}; mkdir -p $OUT
TDG_LIB_PATH=abtest/lib_NA.so timeout 300 python tools/sweep.py "" > $OUT/quick.txt 2>&1; echo "quick rc=$?" >> $OUT/quick.txt
TDG_LIB_PATH=abtest/lib_NA.so TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash tools/ab_libs.sh $OUT detect NB NA
nvidia-smi > $OUT/smi_end.txt 2>&1
