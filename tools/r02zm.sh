OUT=gpurun_out/${TAG:-r02zm}; mkdir -p $OUT
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k_demod|k_stats" --profile-from-start off -c 2 -o $OUT/ds python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/ncu.log 2>&1
nvidia-smi > $OUT/smi_end.txt 2>&1
