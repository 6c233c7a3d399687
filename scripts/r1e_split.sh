#!/bin/bash
# 1 GPU: C2 e2e phase split (world build phases, round trace, level loop) and level-step grid sweep
O=gpurun_out
CHROMA_BUILD_TIMING=1 CHROMA_ROUND_TRACE=1 CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py > $O/s_e2e.log 2>&1
for gm in 2 4 8; do echo "grid x$gm"; CHROMA_LEVEL_GRID=$gm CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py 2>&1 | grep -E "level loop|levels\] build|h2d" | tail -3; done > $O/s_grid.log 2>&1
tail -40 $O/s_e2e.log; cat $O/s_grid.log
