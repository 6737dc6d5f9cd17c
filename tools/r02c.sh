OUT=gpurun_out/${TAG:-r02c}; mkdir -p $OUT
TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash tools/ab_libs.sh $OUT detect ${VARS:-A N}
