"""Check: Jacobi run_distributed (the reference's default mode) against the C oracle on
small graphs, and print sha256 of C3-like runs (compare with CHROMA_JACOBI_FULL=1)."""
import sys, os, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
import oracle
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R
bad = 0
cases = [("rmat%d" % s, G.gen_rmat(s)) for s in (8, 10, 12, 14)] + \
        [("gnp", G.gen_random_gnp(400, 0.05, 3)), ("myc", G.gen_mycielskian(9)), ("star", G.preprocess(3000, [(0, i) for i in range(1, 3000)] + [(i, i + 1) for i in range(1, 2999)]))]
for name, g in cases:
    for P in (1, 3):
        pm = PT.partition_block(g, P)
        w = RT.build_local_graphs(g, pm, 1)
        c, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode.D1))
        ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, 1)
        rc, rr = ow.run("d1", False, False)
        ok = np.array_equal(c, rc) and [r.conflicts for r in reps] == [r["conflicts"] for r in rr]
        bad += not ok
        print(name, "P", P, "ok", ok, flush=True)
print("BAD", bad, flush=True)
for s in (int(x) for x in sys.argv[1:]):
    g = G.gen_rmat(s, device="cuda")
    for P in (1, 4):
        w = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
        c, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode.D1))
        print(f"s{s} P={P} rounds {len(reps)} sha {hashlib.sha256(np.asarray(c, '<i4').tobytes()).hexdigest()[:16]}", flush=True)
