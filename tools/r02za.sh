OUT=gpurun_out/${TAG:-r02za}; mkdir -p $OUT
TDG_LIB_PATH=abtest/lib_K.so TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for i in 1 2; do for v in F K; do
TDG_LIB_PATH=abtest/lib_$v.so python bench.py --workload tracking 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['batches']; print('$v ' + ' '.join('B%s %.1fus %.0f/s' % (k, v['p50_ms']*1e3, v['tasks_per_s']) for k, v in b.items()))" >> $OUT/track_ab.txt
done; done
nvidia-smi > $OUT/smi_end.txt 2>&1
