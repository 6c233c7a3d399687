"""Probe: world build + run end to end for C3 from host int64 CSR, pinned and pageable
(CHROMA_BUILD_TIMING=1 adds the builder's phase times)."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R
g = G.gen_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24, device="cuda")
print("host cores", os.cpu_count(), len(os.sched_getaffinity(0)), flush=True)
off = np.ascontiguousarray(g.row_offsets)
col = np.ascontiguousarray(g.col_indices)
for kind in ("pinned", "pageable"):
    if kind == "pinned":
        hg = G.Graph(g.num_vertices, torch.from_numpy(off).pin_memory().numpy(), torch.from_numpy(col).pin_memory().numpy())
    else:
        hg = G.Graph(g.num_vertices, off.copy(), col.copy())
    pm = PT.partition_block(hg, 1)
    for it in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        w = RT.build_local_graphs(hg, pm, 1)
        torch.cuda.synchronize(); tb = time.perf_counter() - t
        c, _ = R.run_distributed(w, R.AlgorithmConfig(deterministic=True))
        torch.cuda.synchronize(); tt = time.perf_counter() - t
        print(f"{kind}: build {tb*1e3:.1f} ms, build+run+D2H {tt*1e3:.1f} ms", flush=True)
        del w
