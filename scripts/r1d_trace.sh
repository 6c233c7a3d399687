#!/bin/bash
O=gpurun_out
CHROMA_LEVEL_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c2_trace.json 2> $O/bench_c2_trace.err
grep -E "levels|cluster" $O/bench_c2_trace.err | head -4
