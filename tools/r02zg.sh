OUT=gpurun_out/${TAG:-r02zg}; mkdir -p $OUT
B="wave_pairs=8,ring=3"
python tools/sweep.py "$B" "wave_pairs=8,ring=2" "$B" "wave_pairs=8,ring=2" "$B" "wave_pairs=6,ring=3" "$B" "wave_pairs=6,ring=4" "$B" "wave_pairs=10,ring=2" "$B" > $OUT/sweep.txt 2>&1
nvidia-smi > $OUT/smi_end.txt 2>&1
