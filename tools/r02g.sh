OUT=gpurun_out/${TAG:-r02g}; mkdir -p $OUT
./tools/microbench/mix > $OUT/mix.txt 2>&1
python tools/sweep.py "" "cta_cap_a=0,cta_cap_b=1,n_streams=6" "cta_cap_a=0,cta_cap_b=1,n_streams=8" "cta_cap_a=2,cta_cap_b=1,n_streams=8" "cta_cap_a=1,cta_cap_b=1,n_streams=8" "cta_cap_a=2,cta_cap_b=2,n_streams=8" "cta_cap_a=0,cta_cap_b=2,n_streams=8,wave_pairs=4,ring=6" "cta_cap_a=0,cta_cap_b=2,n_streams=6,wave_pairs=8,ring=3" > $OUT/sweep.txt 2>&1
nvidia-smi > $OUT/smi_end.txt 2>&1
