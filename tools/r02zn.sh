OUT=gpurun_out/${TAG:-r02zn}; mkdir -p $OUT
for i in 1 2 3; do for v in H S2; do
TDG_LIB_PATH=abtest/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']; print('$v value %.0f stats %.3f demod %.3f corr %.3f' % (d['value'], k['stats'], k['demod'], k['corr']))" >> $OUT/ab.txt
done; done
TDG_LIB_PATH=abtest/lib_S2.so TDG_PARITY_OUT=$OUT timeout 900 python -m pytest tests -x -q -m gpu -k "statistics or search_shape or cfg2 or tracking or golden or end_to_end" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
nvidia-smi > $OUT/smi_end.txt 2>&1
