"""Probe: device R-MAT generation + deterministic / free D1 on C3 at P = 1, 8 (virtual ranks)."""
import hashlib, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, verify as V, _lib
import ctypes as C

def sha(a, dt): return hashlib.sha256(np.ascontiguousarray(a).astype(dt).tobytes()).hexdigest()[:16]
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
Ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")]
for sc in (10, 14):
    gd = G.gen_rmat(sc, device="cuda"); gh = G.gen_rmat(sc)
    print("gen match", sc, np.array_equal(gd.row_offsets, gh.row_offsets) and np.array_equal(gd.col_indices, gh.col_indices), flush=True)
torch.cuda.synchronize(); t = time.time()
g = G.gen_rmat(scale, device="cuda"); torch.cuda.synchronize()
print(f"gen s{scale} {time.time()-t:.2f}s nnz {len(g.col_indices)} csr sha {sha(g.col_indices,'<i8')} {sha(g.row_offsets,'<i8')}", flush=True)
tb = (C.c_double * 5)()
for P in Ps:
    pm = PT.partition_block(g, P)
    t = time.time(); w = RT.build_local_graphs(g, pm, 1); torch.cuda.synchronize(); print(f"P={P} build {time.time()-t:.2f}s", flush=True)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    for algo in ("gauss-seidel", "free"):
        cfg = R.AlgorithmConfig(mode=R.Mode.D1, deterministic=algo == "gauss-seidel", algorithm=None if algo == "gauss-seidel" else algo)
        ts = []
        for it in range(4):
            t = time.time(); c, reps = R.run_distributed(w, cfg, out=out); torch.cuda.synchronize(); el = time.time() - t
            _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
            ts.append((el, tb[0], tb[1]))
        ch = out.cpu().numpy()
        print(f"P={P} {algo}: rounds {len(reps)} colors {ch.max()} sha {sha(ch,'<i4')} conflicts {[r.conflicts for r in reps][:8]}", flush=True)
        for x in ts: print(f"   wall {x[0]*1e3:.2f} ms dev {x[1]*1e3:.2f} ms kern {x[2]*1e3:.2f} ms", flush=True)
        print("   violations", V.count_violations(g, ch, "d1"), flush=True)
    del w
