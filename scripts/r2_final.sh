#!/usr/bin/env bash
# Round-2 final measurement pass on one B200 (outputs in gpurun_out/, copied to profiles/):
# every BASELINE workload's bench line, the C3 reference arm, and the C3 launch list +
# one --set full capture of k_gs_chunked (scripts/profile.sh).
set -u
for wl in c3 c2 c1 c4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/r2f_bench_$wl.json 2> gpurun_out/r2f_bench_$wl.err
done
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_c5.json 2> gpurun_out/r2f_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2f_bench_c3_reference.json 2> gpurun_out/r2f_bench_c3_reference.err
timeout 1500 bash scripts/profile.sh c3 k_gs_chunked
ls -la gpurun_out/r2f_* gpurun_out/prof_c3*
