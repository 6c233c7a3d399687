"""Probe: deterministic D1 on R-MAT at P ranks (virtual), device times and colour sha.
CHROMA_GS_CHUNK_TRACE=1 prints the chunked kernel's phase times per call."""
import hashlib, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CHROMA_MULTI_GPU", "0")
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, _lib
import ctypes as C
scale = int(sys.argv[1]); P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = G.gen_rmat(scale, device="cuda")
w = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
cfg = R.AlgorithmConfig(mode=R.Mode.D1, deterministic=True)
tb = (C.c_double * 5)()
for it in range(3):
    c, reps = R.run_distributed(w, cfg, out=out)
    _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
    h = hashlib.sha256(out.cpu().numpy().astype('<i4').tobytes()).hexdigest()[:16]
    print(f"s{scale} P={P} rounds {len(reps)} dev {tb[0]*1e3:.2f} ms kern {tb[1]*1e3:.2f} ms sha {h}", flush=True)
