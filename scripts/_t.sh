for sc in 0 1 2 3; do echo "schedule=$sc"; CHROMA_LEVEL_TRACE=1 CHROMA_GS_SCHEDULE=$sc python scripts/probe_gs.py sched 2>&1 | grep -v "^\[levels\] [0-9]* levels" | cut -c1-160; done
