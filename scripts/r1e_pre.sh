#!/bin/bash
# 1 GPU: level step with the first frontier entry loaded beside the level size
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "at_scale or cluster_runs or c1_full or level" > $O/q_pytest.log 2>&1; echo "pytest rc=$?" >> $O/q_pytest.log
for k in 1 2; do CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py 2>&1 | grep -E "level loop|levels\] build|h2d" | tail -3; done > $O/q_e2e.log 2>&1
CHROMA_LEVEL_TRACE=1 timeout 300 python tests/c1_probe.py 2>&1 | grep -E "levels\]|^run|^8b" > $O/q_c1.log 2>&1
tail -2 $O/q_pytest.log; cat $O/q_e2e.log $O/q_c1.log
