#!/bin/bash
# 4 GPUs: C2 bench at N = 4 with the windowed per-rank world build
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29851 bench.py --gpus 4 > $O/w4_bench_c2_n4.json 2> $O/w4_bench_c2_n4.err
cat $O/w4_bench_c2_n4.json
