OUT=gpurun_out/${TAG:-r02e}; mkdir -p $OUT
SPECS="cta_cap_b=3 cta_cap_b=0" bash tools/ab_libs.sh $OUT detect N M41 M42 M51
nvidia-smi > $OUT/smi_end.txt 2>&1
