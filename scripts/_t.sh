for pa in 0 1; do echo "poll_all=$pa"; CHROMA_GS_POLL_ALL=$pa python scripts/probe_gs.py sched 2>&1 | cut -c1-150 | grep -v "R-MAT s20 gs P8"; done
