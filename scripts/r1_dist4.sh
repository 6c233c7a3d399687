#!/bin/bash
# 4-GPU pass: free-mode R-MAT s24 probes (hubs first vs not), distributed free tests, C3 bench at N=4
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$TR --nproc-per-node 4 --master-port 29511 scripts/probe_dist.py > $O/d4_hubs.txt 2>&1
CHROMA_NO_HUBS=1 $TR --nproc-per-node 4 --master-port 29512 scripts/probe_dist.py > $O/d4_nohubs.txt 2>&1
$TR --nproc-per-node 2 --master-port 29513 scripts/probe_dist.py > $O/d2_hubs.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_free_gpu.py -x -q > $O/d4_tests.txt 2>&1
$TR --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --workload c3 > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err
$TR --nproc-per-node 4 --master-port 29515 bench.py --gpus 4 > $O/bench_c2_n4.json 2> $O/bench_c2_n4.err
tail -2 $O/d4_tests.txt
