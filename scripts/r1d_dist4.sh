#!/bin/bash
# 4 GPUs: multi-process parity tests, C2 and C3 at N = 2 and 4 (one process per GPU)
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -x -q > $O/d4_dist_tests.txt 2>&1
for n in 2 4; do
  $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n --no-cpu-baseline > $O/bench_c2_n$n.json 2> $O/bench_c2_n$n.err
  $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --workload c3 --no-e2e > $O/bench_c3_n$n.json 2> $O/bench_c3_n$n.err
done
tail -2 $O/d4_dist_tests.txt
for f in $O/bench_c2_n2.json $O/bench_c2_n4.json $O/bench_c3_n2.json $O/bench_c3_n4.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['config'].get('rounds'), d['config'].get('colors'))"; done
