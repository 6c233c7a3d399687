#!/usr/bin/env python
"""Benchmark: distributed speculate-and-iterate colouring on B200 (BASELINE.json metric).

Default workload (configs[1], "C2"): D1-2GL colouring of the 3-D 27-point stencil mesh
128^3 (2,097,152 vertices, 26,822,908 undirected edges), partition_block over P = N
ranks, one rank per GPU, deterministic mode (bit-exact with the reference).  One step =
one full run_distributed (every round: colour, halo exchange over NVLink, detection,
allreduce) on the device-resident world.

"--workload c3" runs configs[2], the north-star target: D1 colouring of the permuted
R-MAT scale-24 graph (edge factor 16), P = N, free-running mode by default.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path
    python bench.py --workload c3 [--scale 24] [...]            # R-MAT (north-star target)
    python bench.py --impl reference [...]                      # reference arm (CPU)
    torchrun --nproc-per-node N bench.py --gpus N ...           # N > 1

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

UNIT = "edges/s"


class Workload:
    """The benchmarked configuration (BASELINE.json configs[1] or configs[2])."""

    def __init__(self, args):
        self.name = args.workload
        if self.name == "c2":
            self.mode, self.gl, self.vmode = "d1-2gl", 2, "d1"
            self.metric = f"coloring edges/s (D1-2GL, 27-pt stencil {args.L}^3)"
            self.algorithm = args.algorithm or "gauss-seidel"
            self.desc = f"C2: D1-2GL 27-point stencil {args.L}^3"
            self.data = "synthetic (27-point stencil generated on device, id = x + L(y + L z))"
        else:
            self.mode, self.gl, self.vmode = "d1", 1, "d1"
            self.metric = f"coloring edges/s (D1, R-MAT scale-{args.scale} ef16)"
            self.algorithm = args.algorithm or "free"
            self.desc = f"C3: D1 R-MAT scale-{args.scale} edge factor 16 (permuted)"
            self.data = "synthetic (Graph500 R-MAT a=.57 b=c=.19, seeded label permutation, generated on device)"
        self.args = args

    def graph(self, device=None, scale=None):
        from paper_2107_00075_b200 import graph as G
        if self.name == "c2":
            return G.gen_stencil27(self.args.L, device=device)
        return G.gen_rmat(scale or self.args.scale, 16, 1, device=device)

    def sample_scale(self) -> int:
        """Bounded CPU sample for the C3 oracle timing (the full graph takes hours in Python)."""
        return min(self.args.scale, 18)


_JSON_FD = None


def quiet_stdout():
    """Route everything (Python prints, NCCL/C-level writes) to stderr so stdout
    carries exactly the one JSON line."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3"])
    ap.add_argument("--L", type=int, default=128, help="C2 stencil edge length (128 = BASELINE config)")
    ap.add_argument("--scale", type=int, default=24, help="C3 R-MAT scale (24 = BASELINE config)")
    ap.add_argument("--algorithm", default=None, choices=["gauss-seidel", "free", "jacobi"],
                    help="default: gauss-seidel (deterministic, bit-exact) for c2, free for c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def round0_bytes(n_owned: int, nnz_owned: int, touched: int) -> int:
    """Algorithmic bytes of one round-0 colouring launch: colour write,
    row pointers (int64 pair per row), int32 column indices, distinct colours read."""
    return 4 * n_owned + 8 * (n_owned + 1) + 4 * nnz_owned + 4 * touched


def cpu_baseline(wl: "Workload", P: int, budget_s: float = 30.0) -> dict:
    """The C oracle (port of the reference path) on the host, single thread."""
    import oracle
    from paper_2107_00075_b200 import partition as PT
    g = wl.graph(scale=wl.sample_scale() if wl.name == "c3" else None)
    pm = PT.partition_block(g, P)
    w = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, wl.gl)
    t0 = time.perf_counter()
    reps = 0
    while True:
        w.run(wl.mode, False, True)
        reps += 1
        el = time.perf_counter() - t0
        if el > budget_s / 3 or reps >= 3:
            break
    sec = el / reps
    m = len(g.col_indices) // 2
    what = (f"the full 27-pt {wl.args.L}^3 mesh" if wl.name == "c2"
            else f"R-MAT scale-{wl.sample_scale()} (bounded sample of the scale-{wl.args.scale} workload)")
    return {"value": m / sec, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle run_distributed ({wl.mode}, deterministic) on {what}, "
                      f"P={P}, {reps} rep(s), {sec:.3f} s/step, 1 of {os.cpu_count()} cores"}


def run_reference(args):
    """Reference arm: the CPU port of the reference path (oracle/), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2107_00075_b200 import partition as PT
    wl = Workload(args)
    P = args.gpus
    g = wl.graph(scale=wl.sample_scale() if wl.name == "c3" else None)
    pm = PT.partition_block(g, P)
    w = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, wl.gl)
    for _ in range(args.warmup):
        w.run(wl.mode, False, True)
    t = []
    colors = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        colors, reps = w.run(wl.mode, False, True)
        t.append(time.perf_counter() - t0)
    m = len(g.col_indices) // 2
    T = sum(t)
    val = m * args.steps / T
    ncol = int(len(np.unique(colors[colors > 0])))
    sample = ("full workload each step" if wl.name == "c2"
              else f"R-MAT scale-{wl.sample_scale()} each step (bounded sample of scale {args.scale})")
    line = {"metric": wl.metric, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"{wl.desc}, partition_block P={P}, deterministic (oracle)",
                       "n": g.num_vertices, "m": m, "rounds": len(reps), "colors": ncol},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": f"oracle/ C port of the reference path, {sample}, "
                                       f"1 of {os.cpu_count()} cores"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    args = parse()
    quiet_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2107_00075_b200 import launch_count
    from paper_2107_00075_b200 import partition as PT
    from paper_2107_00075_b200 import protocol as R
    from paper_2107_00075_b200 import runtime as RT
    from paper_2107_00075_b200 import verify as V
    from paper_2107_00075_b200 import _lib

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world_size
    if N != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={N}")
    torch.cuda.set_device(local)
    _lib.set_device(local)
    if N > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    def barrier():
        if N > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if N == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    wl = Workload(args)
    g = wl.graph(device=f"cuda:{local}")
    m = len(g.col_indices) // 2
    pm = PT.partition_block(g, N)
    cfg = R.AlgorithmConfig(mode=R.Mode(wl.mode), deterministic=wl.algorithm == "gauss-seidel",
                            algorithm=None if wl.algorithm == "gauss-seidel" else wl.algorithm)

    def make_world():
        if N == 1:
            return RT.build_local_graphs(g, pm, wl.gl)
        from paper_2107_00075_b200.dist import DistWorld
        return DistWorld(g, pm, wl.gl)

    world = make_world()
    lg = world.local_graphs[0] if N == 1 else world.local_graph
    # `value` keeps the result in HBM (device output); e2e below returns it to the host
    n_out = world.output_length() if hasattr(world, "output_length") else world.num_global_vertices
    out = torch.empty(n_out, dtype=torch.int32, device=f"cuda:{local}")
    for _ in range(args.warmup):
        R.run_distributed(world, cfg, out=out)

    import ctypes as C
    tbuf = (C.c_double * 5)()
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(local) if rank == 0 else None
    l0 = launch_count()
    per = []
    kern = []
    r0 = []
    rounds = 0
    colors = None
    for _ in range(args.steps):
        barrier()
        colors, reports = R.run_distributed(world, cfg, out=out)
        _lib.check(_lib.lib().chroma_world_last_timing(world.handle.h, tbuf))
        per.append(tbuf[0])
        kern.append(tbuf[1])
        r0.append(reports[0].time_color_s)
        rounds = len(reports)
    torch.cuda.synchronize()
    barrier()
    launches = launch_count() - l0
    clocks = clk.stop() if clk else None
    T = allmax(sum(per))
    TK = allmax(sum(kern))
    value = m * args.steps / T
    # ---- colour count and properness (global, after timing)
    colors = colors.cpu().numpy()
    if N == 1:
        gcol = colors
    else:
        own = torch.from_numpy(colors.astype(np.int32)).cuda()
        sizes = [None] * N
        dist.all_gather_object(sizes, int(own.numel()))
        bufs = [torch.empty(s, dtype=torch.int32, device=own.device) for s in sizes]
        dist.all_gather(bufs, own)
        gcol = torch.cat(bufs).cpu().numpy()  # partition_block: owned ranges are contiguous in gid order
    ncol, _ = V.color_stats(gcol) if rank == 0 else (None, None)
    nviol = V.count_violations(g, gcol, wl.vmode) if rank == 0 else None
    # ---- roofline of the dominant kernel (colouring, round 0 bytes)
    n_o = lg.owned_count
    nnz_o = int(lg.row_offsets[n_o]) if N > 1 else len(g.col_indices)
    touched = lg.num_local if N > 1 else g.num_vertices
    B = round0_bytes(n_o, nnz_o, touched)
    kernel_s = TK / args.steps
    if wl.algorithm == "free":
        # free mode: round 0's colour phase (heavy waves + light speculation) is the unit
        kernel_s = allmax(sum(r0)) / args.steps
    peak, peak_kind = peaks()
    achieved = B / kernel_s / 1e9
    traffic = None
    if N == 1 and wl.name == "c2" and args.L == 128 and wl.algorithm == "gauss-seidel":
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                traffic = json.load(fh)["colour_kernel_c2_p1"]["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        off_p = torch.from_numpy(np.ascontiguousarray(g.row_offsets, dtype=np.int64)).pin_memory()
        col_p = torch.from_numpy(np.ascontiguousarray(g.col_indices, dtype=np.int64)).pin_memory()
        own_p = torch.from_numpy(np.ascontiguousarray(pm.owner, dtype=np.int32)).pin_memory()
        from paper_2107_00075_b200.graph import Graph
        hg = Graph(g.num_vertices, off_p.numpy(), col_p.numpy())
        hpm = PT.PartitionMap(own_p.numpy(), N)
        et = []
        # W untimed warm-up calls (as for `value`): the first calls fill the device pool
        # and torch's pinned host cache that the returned colour arrays come from
        ew = max(1, args.warmup)
        for it in range(max(1, min(args.steps, 3)) + ew):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if N == 1:
                wv = RT.build_local_graphs(hg, hpm, wl.gl)
            else:
                from paper_2107_00075_b200.dist import DistWorld
                wv = DistWorld(hg, hpm, wl.gl)
            out, _ = R.run_distributed(wv, cfg)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            del wv
            if it >= ew:
                et.append(el)
        te = allmax(sum(et) / len(et))
        e2e = {"value": m / te, "unit": UNIT,
               "h2d_bytes_per_step": int(off_p.numel() * 8 + col_p.numel() * 8 + own_p.numel() * 4),
               "d2h_bytes_per_step": int(4 * (g.num_vertices if N == 1 else n_o)),
               "timing": "host perf_counter around build_local_graphs + run_distributed (synchronous API)"}
    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, N)
    if rank == 0:
        line = {"metric": wl.metric, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": wl.data,
                "config": {"workload": f"{wl.desc}, partition_block P={N}, {wl.algorithm}",
                           "n": g.num_vertices, "m": m, "ghost_layers": wl.gl, "rounds": rounds, "colors": ncol,
                           "violations": nviol, "parallelism": f"vertex-range x{N}",
                           "l2": f"inputs larger than L2 (int32 col {4 * len(g.col_indices) / 1e6:.0f} MB)"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "kernel": ("Gauss-Seidel colouring kernel (k_gs_cluster: level-synchronous, one "
                                        "16-CTA cluster, colours in DSMEM)" if wl.algorithm == "gauss-seidel"
                                        else "round-0 colour phase (hub waves + light/tiny passes)"),
                             "algorithmic_bytes_per_launch": B, "kernel_ms": kernel_s * 1e3,
                             "peak_kind": peak_kind},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        emit(line)
    if N > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
