python scripts/probe_gs.py rounds 2>&1 | head -28
python scripts/probe_gs.py free 2>&1 | grep -v "gs P8"
