#!/bin/bash
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/d4_all_tests.txt 2>&1
for n in 2 4; do
  $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n > $O/bench_c2_n$n.json 2> $O/bench_c2_n$n.err
  $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --workload c3 --no-e2e > $O/bench_c3_n$n.json 2> $O/bench_c3_n$n.err
done
python bench.py > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err
python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
tail -2 $O/d4_all_tests.txt
