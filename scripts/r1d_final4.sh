#!/bin/bash
# 4 GPUs: full GPU suite (incl. multi-process NCCL/NVLink tests), smoke, bench N = 1, 2, 4 (C2) and C3 at N = 1, 4
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/f4_pytest.log 2>&1; echo "pytest rc=$?" >> $O/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/f4_smoke.log 2>&1; echo "smoke rc=$?" >> $O/f4_smoke.log
timeout 600 python bench.py > $O/f4_bench_c2_n1.json 2> $O/f4_bench_c2_n1.err
for n in 2 4; do
  timeout 600 $TR --nproc-per-node $n --master-port 2982$n bench.py --gpus $n > $O/f4_bench_c2_n$n.json 2> $O/f4_bench_c2_n$n.err
done
timeout 600 python bench.py --workload c3 --no-cpu-baseline > $O/f4_bench_c3_n1.json 2> $O/f4_bench_c3_n1.err
timeout 600 $TR --nproc-per-node 4 --master-port 29834 bench.py --gpus 4 --workload c3 --no-e2e > $O/f4_bench_c3_n4.json 2> $O/f4_bench_c3_n4.err
timeout 300 python bench.py --impl reference > $O/f4_bench_ref.json 2> $O/f4_bench_ref.err
tail -2 $O/f4_pytest.log; tail -2 $O/f4_smoke.log
for f in $O/f4_bench_c2_n1.json $O/f4_bench_c2_n2.json $O/f4_bench_c2_n4.json $O/f4_bench_c3_n1.json $O/f4_bench_c3_n4.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e']['value'] if d.get('e2e') else None, d['config'].get('rounds'), d['config'].get('colors'))"; done
cat $O/f4_bench_ref.json
