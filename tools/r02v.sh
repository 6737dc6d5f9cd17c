OUT=gpurun_out/${TAG:-r02v}; mkdir -p $OUT
TDG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench2.json 2> $OUT/bench2.err; echo "rc=$?" >> $OUT/bench2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/ref2.json 2> $OUT/ref2.err; echo "rc=$?" >> $OUT/ref2.err
timeout 60 nvidia-smi > $OUT/smi_after.txt 2>&1
