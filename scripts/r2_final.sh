#!/usr/bin/env bash
# Round-2 final measurement pass on one B200 (outputs in gpurun_out/, copied to profiles/):
# every BASELINE workload's bench line, the C3 reference arm, the GPU test suite, and the
# C3 launch list + one --set full capture of k_gs_chunked (scripts/profile.sh), and one
# of the net-centric PD2 pick kernel.   Usage: bash scripts/r2_final.sh [prefix]
set -u
P=${1:-r2h}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_gpu_tests.txt 2>&1
for wl in c3 c2 c1 c4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/${P}_bench_$wl.json 2> gpurun_out/${P}_bench_$wl.err
done
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${P}_bench_c3_reference.json 2> gpurun_out/${P}_bench_c3_reference.err
timeout 1500 bash scripts/profile.sh c3 k_gs_chunked
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pick_waves -c 1 \
    -o gpurun_out/${P}_k_pick_waves_c5 python scripts/probe.py run --graph c5 --algo free --reps 1 > gpurun_out/${P}_c5_ncu.log 2>&1
ls -la gpurun_out/${P}_* gpurun_out/prof_c3*
