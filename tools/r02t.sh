OUT=gpurun_out/${TAG:-r02t}; mkdir -p $OUT
TDG_LIB_PATH=abtest/lib_${PV}.so timeout 600 ncu --set full --warp-sampling-interval 0 --warp-sampling-max-passes 20 --warp-sampling-buffer-size 268435456 --clock-control none --import-source on -k regex:k_corr_pass --profile-from-start off -s 4 -c 1 -o $OUT/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > $OUT/ncu.log 2>&1
nvidia-smi > $OUT/smi_end.txt 2>&1
