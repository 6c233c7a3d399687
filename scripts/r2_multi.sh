#!/usr/bin/env bash
# Round-2 multi-GPU pass (gpurun --gpus 4): C3 / C2 / C5 bench lines at N = 2 and 4 over
# torchrun + NCCL, then the multi-GPU test suites.  Usage: bash scripts/r2_multi.sh [prefix]
set -u
P=${1:-r2h}
for n in 2 4; do
  for wl in c3 c2; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --workload $wl --steps 10 --warmup 3 \
      > gpurun_out/${P}_bench_${wl}_n$n.json 2> gpurun_out/${P}_bench_${wl}_n$n.err
  done
done
timeout 1500 python -m pytest tests/test_multidev_gpu.py tests/test_dist_gpu.py -m gpu -x -q > gpurun_out/${P}_multigpu_tests.txt 2>&1
tail -3 gpurun_out/${P}_multigpu_tests.txt
