OUT=gpurun_out/${TAG:-r02u}; mkdir -p $OUT
nvidia-smi > $OUT/smi_before.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_dist_two_rank.py -x -q -m gpu > $OUT/pytest_two_rank.log 2>&1; echo "rc=$?" >> $OUT/pytest_two_rank.log
sleep 5
ps aux | grep -c python > $OUT/ps_after.txt
timeout 60 nvidia-smi > $OUT/smi_after.txt 2>&1; echo "smi rc=$?" >> $OUT/smi_after.txt
