#!/bin/bash
# per-phase host-synchronised timings of round 0 (CHROMA_ROUND_TRACE) at N = 2, 4 (C2)
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "at_scale or cluster_runs or run_distributed_matches" > $O/pytest_rt.log 2>&1; tail -1 $O/pytest_rt.log
for n in 2 4; do
  CHROMA_ROUND_TRACE=1 $TR --nproc-per-node $n --master-port 2962$n bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/rt_c2_n$n.json 2> $O/rt_c2_n$n.err
done
CHROMA_ROUND_TRACE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/rt_c2_n1.json 2> $O/rt_c2_n1.err
for n in 1 2 4; do echo "N=$n"; grep "round0" $O/rt_c2_n$n.err | tail -16; done
for n in 1 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $n --master-port 2972$n bench.py --gpus $n --no-cpu-baseline --no-e2e > $O/b_c2_n$n.json 2>/dev/null; python -c "import json; d=json.load(open(\"$O/b_c2_n$n.json\")); print($n, d[\"ms_per_step\"], d[\"roofline\"][\"kernel_ms\"])"; done
