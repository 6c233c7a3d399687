#!/bin/bash
# 2 GPUs: multi-process NCCL/NVLink tests, C2 bench at N = 2, C3 at N = 2
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -x -q > $O/d2_pytest.log 2>&1; echo "pytest rc=$?" >> $O/d2_pytest.log
timeout 600 $TR --nproc-per-node 2 --master-port 29822 bench.py --gpus 2 > $O/d2_bench_c2_n2.json 2> $O/d2_bench_c2_n2.err
timeout 600 $TR --nproc-per-node 2 --master-port 29823 bench.py --gpus 2 --workload c3 --no-e2e > $O/d2_bench_c3_n2.json 2> $O/d2_bench_c3_n2.err
timeout 300 $TR --nproc-per-node 2 --master-port 29824 bench.py --gpus 2 --impl reference > $O/d2_bench_ref_n2.json 2> $O/d2_bench_ref_n2.err
tail -2 $O/d2_pytest.log
for f in $O/d2_bench_c2_n2.json $O/d2_bench_c3_n2.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e']['value'] if d.get('e2e') else None, d['config'].get('rounds'), d['config'].get('colors'), d['clocks'])"; done
cat $O/d2_bench_ref_n2.json
