"""Probe: C3-like R-MAT at P ranks, every algorithm (Jacobi VB default, Jacobi EB,
Gauss-Seidel, free): device time per run_distributed, rounds, colours."""
import sys, os
import ctypes as C
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, localcolor as L, _lib
scale = int(sys.argv[1]); P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = G.gen_rmat(scale, device="cuda")
w = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
tb = (C.c_double * 5)()
cfgs = {"jacobi (default)": R.AlgorithmConfig(),
        "jacobi EB": R.AlgorithmConfig(kernel=L.KernelChoice(max_degree_threshold=1)),
        "gauss-seidel": R.AlgorithmConfig(deterministic=True),
        "free": R.AlgorithmConfig(algorithm="free")}
for name, cfg in cfgs.items():
    for it in range(3):
        c, reps = R.run_distributed(w, cfg)
    _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
    print(f"s{scale} P={P} {name}: rounds {len(reps)} dev {tb[0]*1e3:.2f} ms colours {int(np.max(c))}", flush=True)
