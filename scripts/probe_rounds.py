"""Probe: per-round phase times of deterministic and free C3 over P virtual ranks."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R
scale = int(sys.argv[1]); Ps = [int(x) for x in sys.argv[2].split(",")]
g = G.gen_rmat(scale, device="cuda")
for P in Ps:
    w = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
    for algo in ("gauss-seidel", "free"):
        cfg = R.AlgorithmConfig(mode=R.Mode.D1, deterministic=algo == "gauss-seidel", algorithm=None if algo == "gauss-seidel" else algo)
        for it in range(2):
            c, reps = R.run_distributed(w, cfg)
        tc = sum(r.time_color_s for r in reps) * 1e3; tm = sum(r.time_comm_s for r in reps) * 1e3; td = sum(r.time_detect_s for r in reps) * 1e3
        print(f"P={P} {algo}: rounds {len(reps)} color {tc:.1f} comm {tm:.1f} detect {td:.1f} ms; bytes {sum(r.bytes_sent for r in reps)}", flush=True)
        for r in reps:
            print(f"   r{r.round_index}: conflicts {r.conflicts} recol {sum(r.recolored_per_rank)} color {r.time_color_s*1e3:.2f} comm {r.time_comm_s*1e3:.2f} detect {r.time_detect_s*1e3:.2f}", flush=True)
    del w
