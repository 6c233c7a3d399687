#!/usr/bin/env bash
# Round-2 (late) measurement pass: the default bench line (C3), the C3 launch list and one
# --set full capture of k_gs_chunked (scripts/profile.sh), and one of the checker kernel.
set -u
timeout 900 python bench.py > gpurun_out/r2g_bench_c3.json 2> gpurun_out/r2g_bench_c3.err
timeout 1500 bash scripts/profile.sh c3 k_gs_chunked
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_d1 -c 1 \
    -o gpurun_out/r2g_k_count_d1_c3 python scripts/probe.py verify --graph c3 --reps 1 > gpurun_out/r2g_verify_ncu.log 2>&1
ls -la gpurun_out/r2g_* gpurun_out/prof_c3*
