#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "at_scale or cluster_runs or c1_full" > $O/pytest_e2e.log 2>&1; tail -1 $O/pytest_e2e.log
for gm in 8 16; do echo "grid x$gm"; CHROMA_LEVEL_GRID=$gm CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py 2>&1 | grep -E "build [0-9]|h2d" | tail -2; done
