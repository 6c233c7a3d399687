"""CPU, world_size 2 over gloo: the host logic of the one-rank-per-GPU path.

Each process builds the static halo routing with paper_2107_00075_b200.dist.build_routing
over torch.distributed (the code the GPU ranks run), then replays the GPU round-loop
formulation (Gauss-Seidel on owned worklist vertices only, exchange-every-ghost data
movement with changed-only accounting per peer, in-place detection, allreduce of
[conflicts, bytes, messages, recolored...]) with the C oracle's per-rank kernels.  The
result must equal the single-process reference semantics (oracle.World.run).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(kind):
    from paper_2107_00075_b200 import graph as G
    if kind == "gnp":
        return G.gen_random_gnp(300, 0.04, 5)
    if kind == "st27":
        return G.gen_stencil27(9)
    return G.gen_random_bipartite(200, 6, 2).graph


def _worker(rank, P, port, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200.dist import build_routing, torch_alltoallv
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    a2a = torch_alltoallv()
    try:
        for kind, mode, rd, part in cases:
            g = _graph(kind)
            pm = PT.partition_block(g, P) if part == "block" else PT.partition_random(g, P, 7)
            gl = 1 if mode == "d1" else 2
            ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl)
            R = ow.rank(rank)
            deg = ow.degrees()[rank]
            oc, nl = R["owned"], R["owned"] + R["ghost"]
            sc, sl, rc, rl = build_routing(R["gids"], oc, R["ghost_owner"], P, rank, a2a)
            # routing agrees with the reference's send_targets: what I send to p is what p expects
            sb = np.concatenate([[0], np.cumsum(sc)])
            rb = np.concatenate([[0], np.cumsum(rc)])
            mine = [R["gids"][sl[sb[p]: sb[p + 1]]] for p in range(P)]
            theirs = a2a([R["gids"][rl[rb[p]: rb[p + 1]]] for p in range(P)])
            for p in range(P):
                assert np.array_equal(mine[p], theirs[p])
            routed = np.unique(sl)
            last = {}
            colors = np.zeros(nl, np.int32)
            d2 = mode in ("d2", "pd2")
            reports = []
            for rnd in range(50):
                wl = np.arange(oc) if rnd == 0 else np.flatnonzero(colors[:oc] == 0)
                rec = np.zeros(P, np.int64)
                rec[rank] = len(wl)
                if len(wl):
                    oracle.speculative_color(R["row_offsets"], R["col_indices"], colors, wl, 2 if d2 else 1,
                                             mode == "pd2", True)
                changed = {}
                for v in routed.tolist():
                    c = int(colors[v])
                    changed[v] = rnd == 0 or last.get(v) != c
                    if changed[v]:
                        last[v] = c
                per_peer = [sum(changed[int(v)] for v in sl[sb[p]: sb[p + 1]]) for p in range(P)]
                got = a2a([colors[sl[sb[p]: sb[p + 1]]].astype(np.int64) for p in range(P)])
                for p in range(P):
                    colors[rl[rb[p]: rb[p + 1]]] = got[p]
                if d2:
                    k = oracle.detect_d2(R["row_offsets"], R["col_indices"], colors, R["gids"], deg,
                                         R["boundary_d2"], mode == "pd2", rd)
                else:
                    k = oracle.detect_d1(oc, R["row_offsets"], R["col_indices"], colors, R["gids"], deg, rd)
                vec = torch.tensor([k, 12 * sum(per_peer), sum(1 for x in per_peer if x)] + rec.tolist(),
                                   dtype=torch.int64)
                dist.all_reduce(vec)
                v = vec.tolist()
                reports.append({"conflicts": v[0], "bytes_sent": v[1], "messages_sent": v[2],
                                "recolored_per_rank": v[3:]})
                if v[0] == 0:
                    break
            ref_colors, ref_reports = ow.run(mode, rd, True)
            assert np.array_equal(colors[:oc], ref_colors[R["gids"][:oc]]), (kind, mode, rd, part)
            for a, b in zip(reports, ref_reports):
                assert a == {k: b[k] for k in a}, (kind, mode, rd, part)
            assert len(reports) == len(ref_reports)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_dist_protocol_world_size_2():
    cases = [(k, m, rd, part) for k in ("gnp", "st27", "bip") for m in ("d1", "d1-2gl", "d2", "pd2")
             for rd in (False, True) for part in ("block", "random")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"
