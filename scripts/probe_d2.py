"""Probe: D2 / PD2 free and deterministic timings (C4, C5) at P = 1, 8 (virtual ranks)."""
import hashlib, sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, verify as V, _lib
import ctypes as C
tb = (C.c_double * 5)()
which = sys.argv[1:] or ["c5", "c4"]
for name in which:
    if name == "c5":
        g = G.gen_random_bipartite(1 << 22, 32, 3, device="cuda").graph; mode = "pd2"
    elif name == "c5s":
        g = G.gen_random_bipartite(1 << 20, 32, 3, device="cuda").graph; mode = "pd2"
    else:
        g = G.gen_hex_mesh_device(200, 200, 200, "cuda"); mode = "d2"
    mask = None
    if mode == "pd2":
        mask = np.zeros(g.num_vertices, np.uint8); mask[: g.num_vertices // 2] = 1
    for P in (1, 8):
        w = RT.build_local_graphs(g, PT.partition_block(g, P), 2)
        out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
        for algo in ("free", "gauss-seidel"):
            if algo == "gauss-seidel" and (name == "c5"):
                continue
            cfg = R.AlgorithmConfig(mode=R.Mode(mode), deterministic=algo == "gauss-seidel",
                                    algorithm=None if algo == "gauss-seidel" else algo)
            ts = []
            for it in range(3):
                c, reps = R.run_distributed(w, cfg, out=out)
                _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
                ts.append(tb[0] * 1e3)
            ch = out.cpu().numpy()
            print(f"{name} P={P} {algo}: rounds {len(reps)} colors {len(np.unique(ch))} ms {[round(x, 2) for x in ts]} "
                  f"viol {V.count_violations(g, ch, 'd2' if mode == 'd2' else 'pd2', mask)} "
                  f"sha {hashlib.sha256(ch.astype('<i4').tobytes()).hexdigest()[:16]}", flush=True)
        del w
