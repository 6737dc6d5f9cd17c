OUT=gpurun_out/${TAG:-r02x}; mkdir -p $OUT
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "search_shape or beyond_the_menu or batch_xcorr or tracking_batch" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "end_to_end_desk_fractional or tracking_batch" > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 60 nvidia-smi > $OUT/smi_after.txt 2>&1
