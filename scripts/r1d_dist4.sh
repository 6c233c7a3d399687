#!/bin/bash
# C2 at 2 and 4 GPUs (one process per GPU), cluster of 16 vs 8 CTAs; multi-GPU parity tests
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -x -q > $O/d4_dist_tests.txt 2>&1
for n in 2 4; do
  $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n --no-cpu-baseline > $O/bench_c2_n$n.json 2> $O/bench_c2_n$n.err
  CHROMA_CLUSTER_SIZE=8 $TR --nproc-per-node $n --master-port 2954$n bench.py --gpus $n --no-cpu-baseline --no-e2e > $O/bench_c2_n${n}_cl8.json 2> $O/bench_c2_n${n}_cl8.err
done
CHROMA_CLUSTER_SIZE=8 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2_n1_cl8.json 2> $O/bench_c2_n1_cl8.err
tail -2 $O/d4_dist_tests.txt
for f in $O/bench_c2_n*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'])"; done
