for b in 1 2 3; do echo "bps=$b"; CHROMA_GS_BPS=$b python scripts/probe_gs.py sched 2>&1 | grep "C2" | cut -c1-150; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_c2_n1_levels.json; cut -c1-400 gpurun_out/r1_c2_n1_levels.json
