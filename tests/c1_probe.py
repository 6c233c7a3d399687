import sys, faulthandler; faulthandler.enable()
sys.path.insert(0,'.')
import numpy as np
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, verify as V
import hashlib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
g = G.gen_hex_mesh(n, n, 1)
print("graph", g.num_vertices, flush=True)
world = RT.build_local_graphs(g, PT.partition_block(g, 1), 1)
print("world", flush=True)
colors, reports = R.run_distributed(world, R.AlgorithmConfig(mode=R.Mode.D1, deterministic=True))
print("run", len(reports), reports[0].time_color_s, flush=True)
print(hashlib.sha256(colors.astype('<i4').tobytes()).hexdigest(), flush=True)
print(V.color_stats(colors), flush=True)
print(len(V.verify_d1(g, colors)), flush=True)
