"""Probe: deterministic D1 / D1-2GL on the mesh configurations (C1 grid, C2 stencil) at P=1."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, _lib
import ctypes as C
tb = (C.c_double * 5)()
for name in sys.argv[1:] or ["c1", "c2"]:
    g = G.gen_hex_mesh_device(1000, 1000, 1, "cuda") if name == "c1" else G.gen_stencil27(128, device="cuda")
    mode = R.Mode.D1 if name == "c1" else R.Mode.D1_2GL
    w = RT.build_local_graphs(g, PT.partition_block(g, 1), R.ghost_layers_for(mode))
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    for it in range(4):
        R.run_distributed(w, R.AlgorithmConfig(mode=mode, deterministic=True), out=out)
        _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
        print(f"{name} call {it}: dev {tb[0]*1e3:.3f} ms kern {tb[1]*1e3:.3f} ms", flush=True)
