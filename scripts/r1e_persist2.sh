#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "at_scale or cluster_runs or c1_full or level" > $O/p2_pytest.log 2>&1; echo "pytest rc=$?" >> $O/p2_pytest.log
for ps in 1 0; do echo "persist=$ps"; CHROMA_LEVEL_PERSIST=$ps CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py 2>&1 | grep -E "levels|h2d|level" | tail -3; done > $O/p2_e2e.log 2>&1
for ps in 1 0; do echo "persist=$ps"; CHROMA_LEVEL_PERSIST=$ps CHROMA_LEVEL_TRACE=1 timeout 300 python tests/c1_probe.py 2>&1 | grep -E "levels\]|^run|^8b" ; done > $O/p2_c1.log 2>&1
tail -2 $O/p2_pytest.log; cat $O/p2_e2e.log $O/p2_c1.log
