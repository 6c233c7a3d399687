"""Dev: where the e2e step (host CSR -> build -> run -> host colours) spends its time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R
g = G.gen_stencil27(128, device="cuda")
off = torch.from_numpy(g.row_offsets).pin_memory(); col = torch.from_numpy(g.col_indices).pin_memory()
hg = G.Graph(g.num_vertices, off.numpy(), col.numpy())
pm = PT.partition_block(hg, 1)
cfg = R.AlgorithmConfig(mode=R.Mode.D1_2GL, deterministic=True)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = col.cuda(non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    del d
    w = RT.build_local_graphs(hg, pm, 2); torch.cuda.synchronize(); t2 = time.perf_counter()
    c, rep = R.run_distributed(w, cfg); t3 = time.perf_counter()
    del w; t4 = time.perf_counter()
    print(f"h2d(col only) {1e3*(t1-t0):.1f} ms  build {1e3*(t2-t1):.1f} ms  run {1e3*(t3-t2):.1f} ms  free {1e3*(t4-t3):.1f} ms", flush=True)
