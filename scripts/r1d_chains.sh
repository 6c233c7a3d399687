#!/bin/bash
# chain-mode (runs on one level) check: new + at-scale parity, levels trace, C2 bench
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster_runs or at_scale or c1_full or large_meshes" > $O/pytest_chains.log 2>&1; echo "pytest rc=$?" >> $O/pytest_chains.log
CHROMA_LEVEL_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c2_chains_trace.json 2> $O/bench_c2_chains_trace.err
timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_chains.json 2> $O/bench_c2_chains.err
CHROMA_NO_CHAINS=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2_nochains.json 2> $O/bench_c2_nochains.err
tail -3 $O/pytest_chains.log; grep -E "levels|cluster" $O/bench_c2_chains_trace.err | head; cat $O/bench_c2_chains.json $O/bench_c2_nochains.json
