OUT=gpurun_out/${TAG:-r02w}; mkdir -p $OUT
for rep in 1 2; do
TDG_LIB_PATH=abtest/lib_G.so python tools/sweep.py "" "sweep_pairs=4,d_keep=1" "sweep_pairs=4,d_keep=0" "sweep_pairs=6,d_keep=1" "sweep_pairs=8,d_keep=1" "sweep_pairs=2,d_keep=1" >> $OUT/sweep.txt 2>&1
done
for sp in 2 4; do
TDG_LIB_PATH=abtest/lib_G.so TDG_BENCH_OPTIONS="sweep_pairs=$sp" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --profile-from-start off --csv --log-file $OUT/launches_sp$sp.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/launches_sp$sp.log 2>&1
done
nvidia-smi > $OUT/smi_end.txt 2>&1
