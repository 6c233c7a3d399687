"""Dev: e2e step time with run_distributed's host colours in pageable vs pinned memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R
g = G.gen_stencil27(128, device="cuda")
off = torch.from_numpy(g.row_offsets).pin_memory(); col = torch.from_numpy(g.col_indices).pin_memory()
hg = G.Graph(g.num_vertices, off.numpy(), col.numpy())
pm = PT.partition_block(hg, 1)
cfg = R.AlgorithmConfig(mode=R.Mode.D1_2GL, deterministic=True)
pinned = R._host_colors
for variant in ("pageable", "pinned", "pageable", "pinned"):
    R._host_colors = pinned if variant == "pinned" else (lambda n: np.zeros(n, dtype=np.int32))
    ts = []
    out = None
    for it in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        w = RT.build_local_graphs(hg, pm, 2); torch.cuda.synchronize(); t1 = time.perf_counter()
        out, rep = R.run_distributed(w, cfg); t2 = time.perf_counter()
        del w
        ts.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
    print(variant, " ".join(f"{a:.1f}+{b:.1f}" for a, b in ts), flush=True)
