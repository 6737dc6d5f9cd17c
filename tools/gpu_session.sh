#!/bin/bash
# One gpurun session: GPU parity tests, smoke, bench, launch list, ncu capture
# of the two correlation passes.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_session.sh [tag] [what...]   what: tests smoke bench launches ncu
set -x
TAG=${1:-run}; shift
WHAT=${@:-tests smoke bench launches ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
for w in $WHAT; do
case $w in
tests)
  TDG_PARITY_OUT=$OUT timeout 1500 python -m pytest tests -x -q -m gpu -rs --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
smoke)
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log ;;
bench)
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err ;;
benchfast)
  timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --profile-from-start off --csv \
      --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/launches_bench.log 2>&1 ;;
ncu)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_corr_pass --profile-from-start off -c 2 \
      -o $OUT/corr python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/ncuA.log 2>&1
  true ;;
track)
  timeout 600 python bench.py --workload tracking > $OUT/track.json 2> $OUT/track.err; echo "track rc=$?" >> $OUT/track.err ;;
roster)
  timeout 600 python bench.py --workload roster --no-cpu-baseline > $OUT/roster.json 2> $OUT/roster.err; echo "roster rc=$?" >> $OUT/roster.err ;;
streams)
  timeout 600 python bench.py --workload streams --no-cpu-baseline > $OUT/streams.json 2> $OUT/streams.err; echo "streams rc=$?" >> $OUT/streams.err ;;
reference)
  timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/ref.err ;;
full)
  timeout 900 ncu --set full --warp-sampling-interval 0 --warp-sampling-max-passes 20 --warp-sampling-buffer-size 268435456 --clock-control none --import-source on -k regex:k_corr_pass --profile-from-start off -s 4 -c 2 \
      -o $OUT/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/ncu_full.log 2>&1
  true ;;
smi)
  nvidia-smi > $OUT/smi_end.txt 2>&1 ;;
sweep)
  timeout 600 python tools/sweep.py $SWEEP > $OUT/sweep.log 2>&1 ;;
esac
done
ls -la $OUT
