"""Check: serial_greedy and deterministic run_distributed against the C oracle on small
graphs (run with CHROMA_GS_CHUNKS=4 to exercise the multi-chunk path of gs_chunked.cu)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2107_00075_b200 import graph as G, localcolor as LC, partition as PT, runtime as RT, protocol as R
bad = 0
cases = [("rmat%d" % s, G.gen_rmat(s)) for s in (8, 10, 12, 14)] + \
        [("gnp", G.gen_random_gnp(400, 0.05, 3)), ("myc", G.gen_mycielskian(8)), ("bip", G.gen_random_bipartite(2000, 16, 3).graph)]
for name, g in cases:
    ref = oracle.serial_greedy(g.row_offsets, g.col_indices)
    got = LC.serial_greedy(g)
    ok = np.array_equal(ref, got)
    bad += not ok
    for P in (1, 3, 8):
        pm = PT.partition_block(g, P)
        w = RT.build_local_graphs(g, pm, 1)
        c, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode.D1, deterministic=True))
        ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, 1)
        rc, rr = ow.run("d1", False, True)
        ok2 = np.array_equal(c, rc) and [r.conflicts for r in reps] == [r["conflicts"] for r in rr]
        bad += not ok2
        print(name, "P", P, "serial", ok, "run", ok2, "colors", ref.max(), flush=True)
print("BAD", bad)
