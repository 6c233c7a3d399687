#!/usr/bin/env bash
# Round-2 measurement pass on one B200: every BASELINE workload's bench line.
set -u
for wl in c3 c2 c1 c4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.err
done
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
