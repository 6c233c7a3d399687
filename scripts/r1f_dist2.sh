#!/bin/bash
# 2 GPUs: windowed column upload in the per-rank world build — dist tests, C2 bench at N = 2
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -x -q > $O/w2_pytest.log 2>&1; echo "pytest rc=$?" >> $O/w2_pytest.log
timeout 600 $TR --nproc-per-node 2 --master-port 29822 bench.py --gpus 2 > $O/w2_bench_c2_n2.json 2> $O/w2_bench_c2_n2.err
tail -2 $O/w2_pytest.log
python -c "import json; d=json.load(open('$O/w2_bench_c2_n2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e'], d['clocks'])"
