import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_2107_00075_b200 import graph as G, partition as PT, protocol as R
from paper_2107_00075_b200.dist import DistWorld
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, P = dist.get_rank(), dist.get_world_size()
g = G.gen_random_gnp(400, 0.03, 7)
pm = PT.partition_block(g, P)
for mode, det in (("d1", True), ("d1", False), ("d2", True)):
    gl = R.ghost_layers_for(R.Mode(mode))
    w = DistWorld(g, pm, gl)
    lg = w.local_graph
    print(rank, "owned", lg.owned_count, "ghost", lg.ghost_count, "halo send", w.halo_send, "recv", w.halo_recv, flush=True)
    try:
        colors, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode(mode), deterministic=det, max_rounds=6))
        print(rank, mode, det, "ok", [r.conflicts for r in reps], flush=True)
    except R.NonConvergenceError as e:
        print(rank, mode, det, "NONCONV", [r.conflicts for r in e.reports], [r.bytes_sent for r in e.reports], flush=True)
    ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl)
    ref, rr = ow.run(mode, False, det)
    print(rank, mode, det, "oracle", [x["conflicts"] for x in rr], [x["bytes_sent"] for x in rr], flush=True)
dist.destroy_process_group()
