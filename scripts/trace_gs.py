"""Dev: per-chunk timeline of the GS kernel (CHROMA_GS_TRACE) on one shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
shape = sys.argv[1]
path = f"gpurun_out/trace_{shape}_{os.environ.get('CHROMA_GS_BPS','4')}.bin"
os.environ["CHROMA_GS_TRACE"] = path
from paper_2107_00075_b200 import graph as G, localcolor as L
g = {"c2": lambda: G.gen_stencil27(128, device="cuda"), "c1": lambda: G.gen_hex_mesh(1000, 1000, 1),
     "rmat": lambda: G.gen_rmat(18, 16, 1, device="cuda")}[shape]()
for _ in range(2):
    L.serial_greedy(g)
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
t0 = t[:, 0].min()
claim, a, done = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
print(shape, "chunks", len(t), "total us", done.max(), "sms", len(np.unique(t[:, 3])))
print("phaseA us: median", np.median(a - claim), "p99", np.percentile(a - claim, 99))
print("wait after A: median", np.median(done - a), "p99", np.percentile(done - a, 99))
for q in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
    k = int(q * (len(t) - 1))
    print(f"chunk {k:7d} claim {claim[k]:9.1f} A {a[k]:9.1f} done {done[k]:9.1f}")
# frontier speed: time when chunk k done, vs k
order = np.argsort(done)
print("done-time per 1000 chunks (us):", np.diff(np.maximum.accumulate(done)[::max(1, len(t)//20)]).round(1).tolist())
# ---- per-vertex hop analysis (identity worklist: serial_greedy)
vt = np.fromfile(path + ".v", dtype=np.uint64).astype(np.int64)[: g.num_vertices]
T = (vt - t0) / 1e3
off, col = g.row_offsets, g.col_indices
src = np.repeat(np.arange(g.num_vertices), np.diff(off))
lower = col < src
D = np.full(g.num_vertices, -1.0)
np.maximum.at(D, src[lower], T[col[lower]])
has = D >= 0
hop = T[has] - D[has]
# the dep achieving the max: same chunk or not
arg = np.full(g.num_vertices, -1)
order = np.lexsort((T[col[lower]], src[lower]))
s2, c2 = src[lower][order], col[lower][order]
last = np.r_[s2[1:] != s2[:-1], True]
arg[s2[last]] = c2[last]
v_idx = np.flatnonzero(has)
same = (arg[v_idx] // 32) == (v_idx // 32)
print("hop us (T(v) - max T(dep)): intra-chunk median %.2f p90 %.2f | cross-chunk median %.2f p90 %.2f" % (
    np.median(hop[same]), np.percentile(hop[same], 90), np.median(hop[~same]), np.percentile(hop[~same], 90)))
print("fraction cross", (~same).mean(), "T max", T.max())
# critical path: walk back from the last vertex via the latest dep
v = int(np.argmax(T)); path_intra = path_cross = 0; t_intra = t_cross = 0.0
while arg[v] >= 0:
    u = int(arg[v])
    if u // 32 == v // 32: path_intra += 1; t_intra += T[v] - T[u]
    else: path_cross += 1; t_cross += T[v] - T[u]
    v = u
print(f"critical path: {path_intra} intra hops ({t_intra:.0f} us), {path_cross} cross hops ({t_cross:.0f} us), start T {T[v]:.0f} us")
# critical-path hop details
ck = t  # per-chunk claim/A/done
claimT = (ck[:, 0] - t0) / 1e3; aT = (ck[:, 1] - t0) / 1e3
v = int(np.argmax(T)); rows = []
while arg[v] >= 0:
    u = int(arg[v]); rows.append((T[v] - T[u], v % 32, u % 32, v // 32 - u // 32, claimT[v // 32], aT[v // 32], T[u], T[v])); v = u
rows = np.array(rows)
cross = rows[rows[:, 3] != 0]
print("critical cross hops: n", len(cross), "latency pct 10/50/90/99:", np.percentile(cross[:, 0], [10, 50, 90, 99]).round(2).tolist())
big = cross[cross[:, 0] > 5]
print("slow (>5us) cross hops:", len(big), "sum us", big[:, 0].sum().round(0))
for r in big[:12]:
    print("  lat %.1f  v_lane %d dep_lane %d chunkdist %d  claim(v) %.1f A(v) %.1f T(dep) %.1f T(v) %.1f" % tuple(r))
print("time  claim_ptr  frontier  in_flight  waiting_after_A")
for tau in np.linspace(0, done.max(), 12)[1:-1]:
    cp = int((claim <= tau).sum()); unfinished = np.flatnonzero(done > tau)
    fr = int(unfinished.min()) if len(unfinished) else len(t)
    inflight = int(((claim <= tau) & (done > tau)).sum()); wa = int(((a <= tau) & (done > tau)).sum())
    print(f"{tau:8.0f} {cp:9d} {fr:9d} {inflight:9d} {wa:9d}")
