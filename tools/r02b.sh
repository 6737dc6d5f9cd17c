set -x
OUT=gpurun_out/r02b; mkdir -p $OUT
./tools/microbench/pipes > $OUT/pipes.txt 2>&1
bash tools/ab_libs.sh $OUT detect A P T PT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_corr_pass --profile-from-start off -c 2 \
      -o $OUT/corr python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/ncuA.log 2>&1
true
