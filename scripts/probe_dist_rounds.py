"""Probe (torchrun, one process per GPU): per-round phase times of C3 on rank 0
(deterministic and free), device-generated graph, DistWorld built once."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R, dist as D
rank = int(os.environ["RANK"]); ws = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
g = G.gen_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24, device="cuda")
w = D.DistWorld(g, PT.partition_block(g, ws), 1)
for algo in ("gauss-seidel", "free"):
    cfg = R.AlgorithmConfig(deterministic=algo == "gauss-seidel", algorithm=None if algo == "gauss-seidel" else algo)
    for it in range(3):
        c, reps = R.run_distributed(w, cfg)
    if rank == 0:
        tot = sum(r.time_color_s + r.time_comm_s + r.time_detect_s for r in reps) * 1e3
        print(f"P={ws} {algo}: rounds {len(reps)} total {tot:.2f} ms", flush=True)
        for r in reps:
            print(f"   r{r.round_index}: conflicts {r.conflicts} recol {sum(r.recolored_per_rank)} color {r.time_color_s*1e3:.2f} "
                  f"comm {r.time_comm_s*1e3:.2f} detect {r.time_detect_s*1e3:.2f}", flush=True)
dist.destroy_process_group()
