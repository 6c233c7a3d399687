"""torchrun entry: one rank per GPU (NCCL) runs run_distributed through
paper_2107_00075_b200.dist.DistWorld and checks its owned colours and every integer
RoundReport field against the C oracle's single-process run (same graph, partition,
P).  Launched by tests/test_dist_gpu.py; exits non-zero on any mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    import oracle
    from paper_2107_00075_b200 import graph as G
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    from paper_2107_00075_b200.dist import DistWorld

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, P = dist.get_rank(), dist.get_world_size()
    graphs = {"gnp": G.gen_random_gnp(400, 0.03, 7), "myciel": G.gen_mycielskian(7),
              "st27": G.gen_stencil27(20), "bip": G.gen_random_bipartite(300, 6, 2).graph,
              "rmat": G.gen_rmat(11, 16, 1)}
    bad = 0
    checked = 0
    for name, g in graphs.items():
        for part in ("block", "random"):
            pm = PT.partition_block(g, P) if part == "block" else PT.partition_random(g, P, 3)
            for mode in ("d1", "d1-2gl", "d2", "pd2"):
                for det in (True, False):
                    rd = (len(name) + len(part) + len(mode)) % 2 == 1  # same on every rank
                    gl = R.ghost_layers_for(R.Mode(mode))
                    w = DistWorld(g, pm, gl)
                    colors, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode(mode), recolor_degrees=rd,
                                                                          deterministic=det))
                    ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl)
                    ref, ref_reps = ow.run(mode, rd, det)
                    owned = w.local_graph.gids[: w.local_graph.owned_count]
                    ok = np.array_equal(colors, ref[owned])
                    ok &= [r.conflicts for r in reps] == [x["conflicts"] for x in ref_reps]
                    ok &= [r.bytes_sent for r in reps] == [x["bytes_sent"] for x in ref_reps]
                    ok &= [r.messages_sent for r in reps] == [x["messages_sent"] for x in ref_reps]
                    ok &= [list(r.recolored_per_rank) for r in reps] == [x["recolored_per_rank"] for x in ref_reps]
                    checked += 1
                    if not ok:
                        bad += 1
                        print(f"rank {rank} MISMATCH {name} {part} {mode} det={det} rd={rd} "
                              f"{[r.conflicts for r in reps]} vs {[x['conflicts'] for x in ref_reps]}", flush=True)
                    del w
    t = torch.tensor([bad], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist parity P={P}: {checked} runs per rank, mismatches (all ranks) = {int(t.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
