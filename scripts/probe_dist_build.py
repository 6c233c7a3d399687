"""Probe (torchrun, one process per GPU): where an end-to-end DistWorld step of C3 spends
its time -- world build from pageable NumPy, routing/connect, run_distributed."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R, dist as D, runtime as RT
rank = int(os.environ["RANK"]); ws = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
g = G.gen_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24, device="cuda")
pg = G.Graph(g.num_vertices, np.array(g.row_offsets, np.int64), np.array(g.col_indices, np.int64))
pm = PT.partition_block(pg, ws)
cfg = R.AlgorithmConfig(deterministic=True)
for it in range(4):
    dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
    h = RT.WorldHandle(pg, pm, 1, rank, rank + 1, rank)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del h
    dist.barrier(); torch.cuda.synchronize(); t2 = time.perf_counter()
    w = D.DistWorld(pg, pm, 1)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    c, reps = R.run_distributed(w, cfg)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    del w
    print(f"rank {rank} it {it}: handle {1e3*(t1-t0):.1f} ms; DistWorld {1e3*(t3-t2):.1f} ms; run {1e3*(t4-t3):.1f} ms", flush=True)
dist.destroy_process_group()
