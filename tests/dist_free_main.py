"""torchrun entry: free-running mode over NCCL + NVLink peer memory, one rank per GPU.
Gathers the owned colours, checks properness with the oracle's verifier and the colour
count against the oracle's deterministic run.  Launched by tests/test_dist_gpu.py."""
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
    graphs = {"rmat14": G.gen_rmat(14, 16, 1), "rmat16": G.gen_rmat(16, 32, 7), "st27": G.gen_stencil27(20),
              "gnp": G.gen_random_gnp(2000, 0.01, 3), "bip": G.gen_random_bipartite(2000, 8, 2).graph}
    bad = 0
    checked = 0
    vmode = {"d1": "d1", "d1-2gl": "d1", "d2": "d2", "pd2": "pd2"}
    for name, g in graphs.items():
        for part in ("block", "random"):
            pm = PT.partition_block(g, P) if part == "block" else PT.partition_random(g, P, 5)
            for mode in ("d1", "d1-2gl", "d2", "pd2"):
                if name.startswith("rmat") and mode in ("d2", "pd2"):
                    continue
                gl = R.ghost_layers_for(R.Mode(mode))
                w = DistWorld(g, pm, gl)
                cfg = R.AlgorithmConfig(mode=R.Mode(mode), deterministic=False, algorithm="free")
                for rep in range(2):  # the world is reused: the second run starts from its state
                    colors, reps = R.run_distributed(w, cfg)
                    owned = np.asarray(w.local_graph.gids[: w.local_graph.owned_count])
                    parts = [None] * P
                    dist.all_gather_object(parts, (owned, np.asarray(colors)))
                    full = np.zeros(g.num_vertices, np.int32)
                    for o, c in parts:
                        full[o] = c
                    viol = len(oracle.verify(g.row_offsets, g.col_indices, full, vmode[mode]))
                    ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl)
                    ref, _ = ow.run(mode, False, True)
                    bound = 1.10 * ref.max() + 1 if mode in ("d1", "d1-2gl") else 1.5 * ref.max()
                    ok = viol == 0 and full.min() >= 1 and full.max() <= bound and reps[-1].conflicts == 0
                    checked += 1
                    if not ok:
                        bad += 1
                        if rank == 0:
                            print(f"FAIL {name} {part} {mode} rep={rep}: violations={viol} colors={full.max()} "
                                  f"oracle={ref.max()} rounds={len(reps)}", flush=True)
                del w
    t = torch.tensor([bad], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist free P={P}: {checked} runs, failures = {int(t.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
