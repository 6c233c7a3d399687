"""Dev probe: free-running D1 on R-MAT over P virtual ranks on one GPU (rounds, time, colours, properness)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R, runtime as RT, verify as V

for spec in sys.argv[1:]:
    sc, P = map(int, spec.split("x"))
    g = G.gen_rmat(sc, 16, 1, device="cuda:0")
    pm = PT.partition_block(g, P)
    w = RT.build_local_graphs(g, pm, 1)
    cfg = R.AlgorithmConfig(mode=R.Mode("d1"), deterministic=False, algorithm="free")
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda:0")
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _, reps = R.run_distributed(w, cfg, out=out)
        torch.cuda.synchronize(); el = time.perf_counter() - t0
    col = out.cpu().numpy()
    nv = V.count_violations(g, col, "d1")
    print(f"s{sc} P={P}: rounds={len(reps)} wall={el*1e3:.1f} ms colors={V.color_stats(col)[0]} viol={nv} "
          f"uncoloured={(col == 0).sum()}", flush=True)
    for r in reps[:6]:
        print(f"  round {r.round_index} conflicts={r.conflicts} recolored={sum(r.recolored_per_rank)} "
              f"color={r.time_color_s*1e3:.2f} comm={r.time_comm_s*1e3:.2f} detect={r.time_detect_s*1e3:.2f}")
