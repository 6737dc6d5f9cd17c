#!/bin/bash
# A/B timing of builds of libtagdsp_gpu.so on one box, alternated so that all
# see the same thermal / power-cap state.  Copy the builds to abtest/lib_<V>.so
# (git-ignored; they travel with gpurun), then e.g.
#   gpurun -- 'bash tools/ab_libs.sh gpurun_out/ab detect A B'
#   modes: detect (tools/sweep.py: correlation + statistics, spectra cached),
#          step   (bench.py device + e2e lines), track (bench.py tracking)
OUT=${1:-gpurun_out/ab}; MODE=${2:-detect}; shift 2; VARIANTS=${@:-A B}
mkdir -p "$OUT"
python tools/sweep.py "" "" "" "" > /dev/null 2>&1   # warm the GPU
for i in 1 2 3; do
  for v in $VARIANTS; do
    case $MODE in
    detect) TDG_LIB_PATH=abtest/lib_$v.so python tools/sweep.py "" ${SPECS:-"" ""} | tail -n +2 | sed "s/^/$v /" >> "$OUT/ab.txt" ;;
    step) TDG_LIB_PATH=abtest/lib_$v.so python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v value %.0f e2e %.0f' % (d['value'], d['e2e']['value']))" >> "$OUT/ab.txt" ;;
    track) TDG_LIB_PATH=abtest/lib_$v.so python bench.py --workload tracking 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['batches']; print('$v ' + ' '.join('B%s %.1fus %.0f/s' % (k, v['p50_ms']*1e3, v['tasks_per_s']) for k, v in b.items()))" >> "$OUT/ab.txt" ;;
    esac
  done
done
