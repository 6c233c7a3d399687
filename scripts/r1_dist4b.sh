#!/bin/bash
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
TRACE0=1 $TR --nproc-per-node 4 --master-port 29511 scripts/probe_dist.py > $O/d4_trace.txt 2>&1
$TR --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --workload c3 --no-e2e > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err
$TR --nproc-per-node 2 --master-port 29516 bench.py --gpus 2 --workload c3 --no-e2e > $O/bench_c3_n2.json 2> $O/bench_c3_n2.err
python bench.py --workload c3 --no-e2e --no-cpu-baseline > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q > $O/d4_tests.txt 2>&1
tail -2 $O/d4_tests.txt
