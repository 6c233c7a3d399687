"""Probe: one Jacobi (default config) run_distributed on R-MAT scale S at P ranks."""
import sys, os
import ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, _lib
scale = int(sys.argv[1]); P = int(sys.argv[2]) if len(sys.argv) > 2 else 1; runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = G.gen_rmat(scale, device="cuda")
w = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
tb = (C.c_double * 5)()
for it in range(runs):
    c, reps = R.run_distributed(w, R.AlgorithmConfig())
    _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
    print(f"s{scale} P={P} jacobi: rounds {len(reps)} dev {tb[0]*1e3:.2f} ms", flush=True)
