"""Dev probe: per-round timings of run_distributed over NCCL (one rank per GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R, _lib
from paper_2107_00075_b200.dist import DistWorld

rank, N, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
if rank == 0 and os.environ.get("TRACE0"):
    os.environ["CHROMA_FREE_TRACE"] = "1"
    os.environ["CHROMA_ROUND_TRACE"] = "1"
torch.cuda.set_device(local)
_lib.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
sc = int(os.environ.get("SCALE", "24"))
alg = os.environ.get("ALG", "free")
g = G.gen_rmat(sc, 16, 1, device=f"cuda:{local}")
pm = PT.partition_block(g, N)
w = DistWorld(g, pm, 1)
cfg = R.AlgorithmConfig(mode=R.Mode("d1"), deterministic=alg == "gs", algorithm=None if alg == "gs" else alg,
                        recolor_degrees=bool(int(os.environ.get("RD", "0"))))
out = torch.empty(w.output_length(), dtype=torch.int32, device=f"cuda:{local}")
for it in range(3):
    dist.barrier()
    t0 = time.perf_counter()
    _, reps = R.run_distributed(w, cfg, out=out)
    el = time.perf_counter() - t0
if rank == 0:
    print(f"N={N} scale={sc} alg={alg} rd={cfg.recolor_degrees} rounds={len(reps)} wall={el*1e3:.1f} ms colors(rank0 max)={int(out.max())}")
    tc = sum(r.time_color_s for r in reps); tm = sum(r.time_comm_s for r in reps); td = sum(r.time_detect_s for r in reps)
    print(f"  sum color={tc*1e3:.2f} comm={tm*1e3:.2f} detect={td*1e3:.2f} ms")
    for r in reps:
        print(f"  round {r.round_index:3d} conflicts={r.conflicts:8d} recolored={sum(r.recolored_per_rank):8d} "
              f"color={r.time_color_s*1e3:7.3f} comm={r.time_comm_s*1e3:7.3f} detect={r.time_detect_s*1e3:7.3f} "
              f"bytes={r.bytes_sent}")
dist.destroy_process_group()
