"""Dev: critical path of the GS kernel from per-vertex commit timestamps
(CHROMA_GS_TRACE=<file>): per-hop latency, intra- vs cross-chunk hops."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

shape = sys.argv[1]
path = f"gpurun_out/vtrace_{shape}.bin"
os.environ["CHROMA_GS_TRACE"] = path
from paper_2107_00075_b200 import graph as G, localcolor as L  # noqa: E402

g = {"c2": lambda: G.gen_stencil27(128, device="cuda"), "c1": lambda: G.gen_hex_mesh(1000, 1000, 1),
     "rmat": lambda: G.gen_rmat(18, 16, 1, device="cuda"), "d2": lambda: G.gen_hex_mesh(100, 100, 100)}[shape]()
for _ in range(2):
    L.serial_greedy(g)
vt = np.fromfile(path + ".v" if os.path.exists(path + ".v") else path, dtype=np.uint64).astype(np.int64)[: g.num_vertices]
T = (vt - vt.min()) / 1e3
off, col = g.row_offsets, g.col_indices
src = np.repeat(np.arange(g.num_vertices), np.diff(off))
lower = col < src
order = np.lexsort((T[col[lower]], src[lower]))
s2, c2 = src[lower][order], col[lower][order]
last = np.r_[s2[1:] != s2[:-1], True]
arg = np.full(g.num_vertices, -1)
arg[s2[last]] = c2[last]
v = int(np.argmax(T))
hops = []
while arg[v] >= 0:
    u = int(arg[v])
    hops.append((T[v] - T[u], u // 32 == v // 32, T[v]))
    v = u
h = np.array(hops)
intra, cross = h[h[:, 1] == 1, 0], h[h[:, 1] == 0, 0]
print(f"{shape}: T {T.max():.0f} us; critical path {len(h)} hops: intra {len(intra)} "
      f"(sum {intra.sum():.0f} us, median {np.median(intra) if len(intra) else 0:.2f}), cross {len(cross)} "
      f"(sum {cross.sum():.0f} us, median {np.median(cross):.2f}, p90 {np.percentile(cross, 90):.2f})")
print("commit histogram over time (10 bins):", np.histogram(T, bins=10)[0].tolist())
