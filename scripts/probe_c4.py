"""Probe: C4 (7-pt 200^3, D2) deterministic / Jacobi / free at P virtual ranks: cold and
steady device times per run_distributed."""
import sys, os
import ctypes as C
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, _lib
L = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = G.gen_hex_mesh_device(L, L, L, "cuda")
tb = (C.c_double * 5)()
for P in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")]:
    w = RT.build_local_graphs(g, PT.partition_block(g, P), 2)
    for name, cfg in (("gauss-seidel", R.AlgorithmConfig(mode=R.Mode.D2, deterministic=True)),
                      ("jacobi", R.AlgorithmConfig(mode=R.Mode.D2)),
                      ("free", R.AlgorithmConfig(mode=R.Mode.D2, algorithm="free"))):
        ts = []
        for it in range(3):
            c, reps = R.run_distributed(w, cfg)
            _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
            ts.append(tb[0] * 1e3)
        print(f"C4 L={L} P={P} {name}: rounds {len(reps)} cold {ts[0]:.2f} ms, steady {ts[-1]:.2f} ms, colours {int(np.max(c))}", flush=True)
    del w
