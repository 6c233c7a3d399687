"""Dev probe: deterministic D1 through the cluster kernel vs the oracle on small meshes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R, runtime as RT

only = os.environ.get("ONLY")
for name, g in [("hex32", G.gen_hex_mesh(32, 32, 32)), ("hex64x64", G.gen_hex_mesh(64, 64, 1)),
                ("hex16", G.gen_hex_mesh(16, 16, 16)), ("st27_16", G.gen_stencil27(16))]:
    if only and name != only:
        continue
    pm = PT.partition_block(g, 1)
    w = RT.build_local_graphs(g, pm, 1)
    cfg = R.AlgorithmConfig(mode=R.Mode("d1"), deterministic=True)
    col, _ = R.run_distributed(w, cfg)
    ref, _ = oracle.World(g.row_offsets, g.col_indices, pm.owner, 1, 1).run("d1", False, True)
    bad = np.flatnonzero(np.asarray(col) != ref)
    print(name, "n", g.num_vertices, "mismatches", len(bad), bad[:10], np.asarray(col)[bad[:10]], ref[bad[:10]], flush=True)
    if len(bad):
        v = bad[0]
        nb = g.col_indices[g.row_offsets[v]:g.row_offsets[v + 1]]
        print("   v", v, "nbrs", nb, "gpu", np.asarray(col)[nb], "ref", ref[nb])
