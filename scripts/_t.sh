python scripts/probe_gs.py sched 2>&1 | cut -c1-150
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | cut -c1-330
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
