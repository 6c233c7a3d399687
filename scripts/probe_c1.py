"""Dev probe: C1 (grid 1000^2, D1, P=1, deterministic) and C4-like meshes -- device time
of run_distributed and of the colouring kernel, colours and sha256 of the C1 result."""
import ctypes as C, hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, verify as V, _lib

for name, g, mode, gl in [("C1 grid 1000^2 D1", G.gen_hex_mesh(1000, 1000, 1), "d1", 1),
                          ("27-pt 128^3 D1-2GL P=1", G.gen_stencil27(128, device="cuda:0"), "d1-2gl", 2),
                          ("7-pt 200^3 D2 P=1", G.gen_hex_mesh(200, 200, 200), "d2", 2)]:
    w = RT.build_local_graphs(g, PT.partition_block(g, 1), gl)
    cfg = R.AlgorithmConfig(mode=R.Mode(mode), deterministic=True)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda:0")
    tb = (C.c_double * 5)()
    ts = []
    for it in range(4):
        _, reps = R.run_distributed(w, cfg, out=out)
        _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
        ts.append((tb[0], tb[1]))
    col = out.cpu().numpy()
    h = hashlib.sha256(col.astype("<i4").tobytes()).hexdigest()[:16]
    print(f"{name}: run {min(t[0] for t in ts)*1e3:.3f} ms, colour kernel {min(t[1] for t in ts)*1e3:.3f} ms, "
          f"rounds {len(reps)}, colours {V.color_stats(col)[0]}, sha256 {h}", flush=True)
