"""Developer probes behind the numbers in DESIGN.md (run on a GPU box; dev aids, not tests).

    python scripts/probe.py run   --graph c3 --P 1,2,4 --algo gs,free,jacobi [--trace]
        device time per run_distributed (CUDA events inside the library), rounds, colours,
        colour sha; --rounds prints every round's phases.  Graphs: c1 c2 c3 c4 c5 c5s, or
        rmat:S (R-MAT scale S).  --trace sets the library's phase traces
        (CHROMA_GS_CHUNK_TRACE, CHROMA_DETECT_TRACE, CHROMA_JACOBI_TRACE, CHROMA_LEVEL_TRACE).
    python scripts/probe.py e2e   --graph c3            build from pinned / pageable host arrays + run
    torchrun --nproc-per-node N scripts/probe.py dist --graph c3 [--e2e]
        one process per GPU: per-round phases on rank 0 (or DistWorld build + run end to end)

Virtual ranks (P > 1 on one GPU) unless run under torchrun.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ALGOS = {"gs": dict(deterministic=True), "free": dict(algorithm="free"), "jacobi": dict()}


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a)).astype("<i4").tobytes()).hexdigest()[:16]


def make_graph(name: str):
    from paper_2107_00075_b200 import graph as G
    from paper_2107_00075_b200 import protocol as R
    if name.startswith("rmat:"):
        return G.gen_rmat(int(name[5:]), device="cuda"), R.Mode.D1
    return {
        "c1": lambda: (G.gen_hex_mesh_device(1000, 1000, 1, "cuda"), R.Mode.D1),
        "c2": lambda: (G.gen_stencil27(128, device="cuda"), R.Mode.D1_2GL),
        "c3": lambda: (G.gen_rmat(24, device="cuda"), R.Mode.D1),
        "c4": lambda: (G.gen_hex_mesh_device(200, 200, 200, "cuda"), R.Mode.D2),
        "c5": lambda: (G.gen_random_bipartite(1 << 22, 32, 3, device="cuda").graph, R.Mode.PD2),
        "c5s": lambda: (G.gen_random_bipartite(1 << 20, 32, 3, device="cuda").graph, R.Mode.PD2),
    }[name]()


def cmd_run(args):
    os.environ.setdefault("CHROMA_MULTI_GPU", "0")
    if args.trace:
        for k in ("CHROMA_GS_CHUNK_TRACE", "CHROMA_DETECT_TRACE", "CHROMA_JACOBI_TRACE", "CHROMA_LEVEL_TRACE"):
            os.environ[k] = "1"
    import torch
    from paper_2107_00075_b200 import _lib
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    from paper_2107_00075_b200 import runtime as RT
    g, mode = make_graph(args.graph)
    tb = (C.c_double * 5)()
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    for P in (int(x) for x in args.P.split(",")):
        w = RT.build_local_graphs(g, PT.partition_block(g, P), R.ghost_layers_for(mode))
        for a in args.algo.split(","):
            cfg = R.AlgorithmConfig(mode=mode, **ALGOS[a])
            ts = []
            for _ in range(args.reps):
                _, reps = R.run_distributed(w, cfg, out=out)
                _lib.check(_lib.lib().chroma_world_last_timing(w.handle.h, tb))
                ts.append((tb[0] * 1e3, tb[1] * 1e3))
            c = out.cpu().numpy()
            print(f"{args.graph} P={P} {a}: rounds {len(reps)} cold {ts[0][0]:.2f} ms, steady {ts[-1][0]:.2f} ms "
                  f"(kernel {ts[-1][1]:.2f}), colours {int(c.max())}, sha {sha16(c)}", flush=True)
            if args.rounds:
                for r in reps:
                    print(f"   r{r.round_index}: conflicts {r.conflicts} recol {sum(r.recolored_per_rank)} "
                          f"color {r.time_color_s * 1e3:.2f} comm {r.time_comm_s * 1e3:.2f} "
                          f"detect {r.time_detect_s * 1e3:.2f}", flush=True)
        del w


def cmd_e2e(args):
    import torch
    from paper_2107_00075_b200 import graph as G
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    from paper_2107_00075_b200 import runtime as RT
    g, mode = make_graph(args.graph)
    print("host cores", len(os.sched_getaffinity(0)), flush=True)
    off, col = np.ascontiguousarray(g.row_offsets), np.ascontiguousarray(g.col_indices)
    for kind in ("pinned", "pageable"):
        if kind == "pinned":
            hg = G.Graph(g.num_vertices, torch.from_numpy(off).pin_memory().numpy(),
                         torch.from_numpy(col).pin_memory().numpy())
        else:
            hg = G.Graph(g.num_vertices, off.copy(), col.copy())
        pm = PT.partition_block(hg, 1)
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            w = RT.build_local_graphs(hg, pm, R.ghost_layers_for(mode))
            torch.cuda.synchronize()
            tb = time.perf_counter() - t
            R.run_distributed(w, R.AlgorithmConfig(mode=mode, deterministic=True))
            torch.cuda.synchronize()
            print(f"{kind}: build {tb * 1e3:.1f} ms, build+run+D2H {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
            del w


def cmd_dist(args):
    import torch
    import torch.distributed as dist
    from paper_2107_00075_b200 import dist as D
    from paper_2107_00075_b200 import graph as G
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    g, mode = make_graph(args.graph)
    gl = R.ghost_layers_for(mode)
    if args.e2e:  # DistWorld build from pageable arrays + run, per step
        pg = G.Graph(g.num_vertices, np.array(g.row_offsets, np.int64), np.array(g.col_indices, np.int64))
        pm = PT.partition_block(pg, ws)
        for it in range(args.reps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            w = D.DistWorld(pg, pm, gl)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            R.run_distributed(w, R.AlgorithmConfig(mode=mode, deterministic=True))
            torch.cuda.synchronize()
            print(f"rank {rank} it {it}: DistWorld {1e3 * (t1 - t0):.1f} ms; run {1e3 * (time.perf_counter() - t1):.1f} ms",
                  flush=True)
            del w
    else:
        w = D.DistWorld(g, PT.partition_block(g, ws), gl)
        for a in args.algo.split(","):
            cfg = R.AlgorithmConfig(mode=mode, **ALGOS[a])
            for _ in range(args.reps):
                _, reps = R.run_distributed(w, cfg)
            if rank == 0:
                tot = sum(r.time_color_s + r.time_comm_s + r.time_detect_s for r in reps) * 1e3
                print(f"P={ws} {a}: rounds {len(reps)} total {tot:.2f} ms", flush=True)
                for r in reps:
                    print(f"   r{r.round_index}: conflicts {r.conflicts} recol {sum(r.recolored_per_rank)} "
                          f"color {r.time_color_s * 1e3:.2f} comm {r.time_comm_s * 1e3:.2f} "
                          f"detect {r.time_detect_s * 1e3:.2f}", flush=True)
    dist.destroy_process_group()


def cmd_verify(args):
    """Count-only checker (verify_d1) on the device colours of a deterministic run:
    CUDA-event time per chroma_verify call and its violation count."""
    import torch
    from paper_2107_00075_b200 import _lib
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    from paper_2107_00075_b200 import runtime as RT
    g, mode = make_graph(args.graph)
    w = RT.build_local_graphs(g, PT.partition_block(g, 1), R.ghost_layers_for(mode))
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    R.run_distributed(w, R.AlgorithmConfig(mode=mode, deterministic=True), out=out)
    del w
    h = _lib.csr_of(g)
    vm = 0 if mode in (R.Mode.D1, R.Mode.D1_2GL) else (2 if mode is R.Mode.PD2 else 1)
    nv = C.c_int64(0)
    rows = np.zeros((1, 4), np.int64)
    for bad in (False, True):
        if bad:  # random colours 0..7: many violations; the listing path must count the same
            out = torch.randint(0, 8, (g.num_vertices,), dtype=torch.int32, device="cuda",
                                generator=torch.Generator("cuda").manual_seed(7))
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            _lib.check(_lib.lib().chroma_verify(h.h, C.c_void_p(out.data_ptr()), None, vm, C.byref(nv), None, 0, 1))
            ts.append((time.perf_counter() - t) * 1e3)
        cnt = nv.value
        _lib.check(_lib.lib().chroma_verify(h.h, C.c_void_p(out.data_ptr()), None, vm, C.byref(nv),
                                            _lib.ptr(rows), 1, 1))
        print(f"{args.graph} verify{'(random colours)' if bad else ''}: violations {cnt} (listing path {nv.value}), "
              f"ms {' '.join(f'{x:.3f}' for x in ts)}", flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("cmd", choices=["run", "e2e", "dist", "verify"])
    ap.add_argument("--graph", default="c3")
    ap.add_argument("--P", default="1")
    ap.add_argument("--algo", default="gs")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", action="store_true")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--e2e", action="store_true")
    args = ap.parse_args()
    {"run": cmd_run, "e2e": cmd_e2e, "dist": cmd_dist, "verify": cmd_verify}[args.cmd](args)


if __name__ == "__main__":
    main()
