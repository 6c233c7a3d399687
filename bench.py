#!/usr/bin/env python
"""Benchmark: distributed speculate-and-iterate colouring on B200 (BASELINE.json metric).

Default workload (configs[2], "C3", the largest single-GPU configuration and the
north-star target): D1 colouring of the permuted Graph500 R-MAT scale 24, edge factor
16 (16.8 M vertices, 260.4 M undirected edges), partition_block over P = N ranks (one
per GPU), deterministic mode -- the reference's Gauss-Seidel semantics, bit-exact with
the C oracle (the colour array's sha256 is printed beside the oracle's).  One step =
one full run_distributed on the device-resident world, colours left in HBM; nothing is
cached between steps (the chunked Gauss-Seidel kernel builds everything it needs per
call).  A "free" sub-record times the free-running mode on the same world, and a "jacobi"
sub-record the reference's default mode (Jacobi sweeps) with its sha against the oracle's.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path (C3)
    python bench.py --workload c1|c2|c4|c5 [...]                # other BASELINE configs
    python bench.py --impl reference [...]                      # reference arm (CPU)
    torchrun --nproc-per-node N bench.py --gpus N ...           # N > 1

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import hashlib
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
GOLDEN = os.path.join(ROOT, "tests", "golden", "scale.json")


class Workload:
    """One BASELINE.json configuration."""

    SPECS = {
        "c1": dict(mode="d1", gl=1, vmode="d1", key="c1_1000",
                   metric="coloring edges/s (D1, 2-D 5-point grid 1000x1000)",
                   desc="C1: D1 grid 1000x1000 (gen_hex_mesh(1000,1000,1))",
                   data="synthetic (reference gen_hex_mesh recipe, generated on device)"),
        "c2": dict(mode="d1-2gl", gl=2, vmode="d1", key="c2_128",
                   metric="coloring edges/s (D1-2GL, 27-pt stencil 128^3)",
                   desc="C2: D1-2GL 27-point stencil 128^3",
                   data="synthetic (27-point stencil generated on device, id = x + L(y + L z))"),
        "c3": dict(mode="d1", gl=1, vmode="d1", key="c3_s24",
                   metric="coloring edges/s (D1, R-MAT scale-24 ef16)",
                   desc="C3: D1 R-MAT scale-24 edge factor 16 (a=.57 b=c=.19, permuted labels)",
                   data="synthetic (counter-based Graph500 R-MAT generated on device; identical CSR to the "
                        "C oracle's generator, sha256 checked)"),
        "c4": dict(mode="d2", gl=2, vmode="d2", key="c4_200",
                   metric="coloring edges/s (D2, 7-pt mesh 200^3)",
                   desc="C4: D2 7-point mesh 200^3 (gen_hex_mesh(200,200,200))",
                   data="synthetic (reference gen_hex_mesh recipe, generated on device)"),
        "c5": dict(mode="pd2", gl=2, vmode="pd2", key="c5_2p22",
                   metric="coloring edges/s (PD2, random 4M x 4M, 32 nnz/row)",
                   desc="C5: PD2 random sparse 2^22 x 2^22, 32 nnz/row -> bipartite",
                   data="synthetic (counter-based random sparse pattern generated on device; identical CSR "
                        "to the C oracle's generator)"),
    }

    def __init__(self, args):
        self.name = args.workload
        self.__dict__.update(self.SPECS[self.name])
        self.args = args
        self.algorithm = args.algorithm or ("free" if self.name == "c5" else "gauss-seidel")

    def graph(self, device=None):
        """The workload's graph (host CSR arrays; built on `device` when given)."""
        from paper_2107_00075_b200 import graph as G
        if self.name == "c1":
            return G.gen_hex_mesh_device(1000, 1000, 1, device) if device else G.gen_hex_mesh(1000, 1000, 1)
        if self.name == "c2":
            return G.gen_stencil27(128, device=device)
        if self.name == "c3":
            return G.gen_rmat(self.args.scale, 16, 1, device=device)
        if self.name == "c4":
            return G.gen_hex_mesh_device(200, 200, 200, device) if device else G.gen_hex_mesh(200, 200, 200)
        return G.gen_random_bipartite(1 << 22, 32, 3, device=device).graph

    def oracle_graph(self, sample: bool = False):
        """The same CSR arrays from the oracle's own generator (reference arm: no GPU).
        sample: a bounded sample of the workload (C3 scale 20, C5 2^18 rows) for P > 1,
        where one oracle run of the full graph takes minutes (the reference's
        rounds grow with P)."""
        import oracle
        if self.name == "c3":
            return oracle.gen_rmat(min(self.args.scale, 20) if sample else self.args.scale)
        if self.name == "c5":
            return oracle.gen_bipartite(1 << (18 if sample else 22), 32, 3)
        g = self.graph()
        return g.row_offsets, g.col_indices

    def golden(self, P: int):
        """The oracle's full-scale values for this workload at P ranks (tests/golden/scale.json,
        written by oracle/gen_scale_golden.py), or None."""
        if not self.key or (self.name == "c3" and self.args.scale != 24):
            return None
        try:
            with open(GOLDEN) as fh:
                d = json.load(fh).get(self.key)
        except Exception:
            return None
        return dict(d, run=d.get(f"{self.mode}_p{P}")) if d else None


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
    ap.add_argument("--workload", default="c3", choices=sorted(Workload.SPECS))
    ap.add_argument("--scale", type=int, default=24, help="C3 R-MAT scale (24 = BASELINE config)")
    ap.add_argument("--algorithm", default=None, choices=["gauss-seidel", "free", "jacobi"],
                    help="default: gauss-seidel (deterministic, bit-exact); free for c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-free", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
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


def gather_rate():
    """Measured random-load rate of this GPU type (L2-resident int32 array, 16 loads in
    flight per thread): profiles/gather_roofline.json, written by scripts/gather_roofline.cu."""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_roofline.json")) as fh:
            return float(json.loads(fh.readline())["gather_i32_64MB"]["gathers_per_s"])
    except Exception:
        return None


def sha256_i32(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<i4").tobytes()).hexdigest()


def cpu_baseline(wl: "Workload", g, P: int) -> dict:
    """The C oracle (port of the reference path) on the host, one thread, on the same
    CSR arrays the GPU coloured: one full run_distributed (deterministic)."""
    import oracle
    from paper_2107_00075_b200 import partition as PT
    pm = PT.partition_block(g, P)
    w = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, wl.gl)
    t0 = time.perf_counter()
    w.run(wl.mode, False, True)
    sec = time.perf_counter() - t0
    m = len(g.col_indices) // 2
    return {"value": m / sec, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle run_distributed ({wl.mode}, deterministic) on the full {wl.desc} graph, P={P}, "
                      f"1 run, {sec:.2f} s; 1 of {os.cpu_count()} host cores"}


def run_reference(args):
    """Reference arm: the CPU port of the reference path (oracle/) on the same
    workload, rank 0 only; the graph comes from the oracle's own generator."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    wl = Workload(args)
    P = args.gpus
    t0 = time.perf_counter()
    sample = P > 1 and wl.name in ("c3", "c5")
    off, col = wl.oracle_graph(sample)
    n = len(off) - 1
    owner = np.empty(n, np.int32)
    for r in range(P):
        owner[r * n // P:(r + 1) * n // P] = r
    w = oracle.World(off, col, owner, P, wl.gl)
    setup = time.perf_counter() - t0
    for _ in range(args.warmup):
        w.run(wl.mode, False, True)
    t = []
    colors = reps = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        colors, reps = w.run(wl.mode, False, True)
        t.append(time.perf_counter() - t0)
    m = len(col) // 2
    T = sum(t)
    val = m * args.steps / T
    gold = None if sample else wl.golden(P)
    sha = sha256_i32(colors)
    what = (f"full workload each step" if not sample else
            f"bounded sample each step: {'R-MAT scale 20' if wl.name == 'c3' else 'PD2 2^18 rows'} at P={P}")
    line = {"metric": wl.metric, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (oracle generator, same CSR as the GPU arm)",
            "config": {"workload": (f"{wl.desc}, partition_block P={P}, gauss-seidel" if not sample else
                                    f"{wl.desc} (bounded sample), partition_block P={P}, gauss-seidel"),
                       "n": n, "m": m, "rounds": len(reps), "colors": int(len(np.unique(colors[colors > 0]))),
                       "colour_sha256": sha,
                       "golden_match": (gold or {}).get("run", {}).get("sha256") == sha if gold else None,
                       "setup_s": round(setup, 1)},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": f"oracle/ C port of the reference path, {what}, "
                                       f"1 of {os.cpu_count()} host cores (the reference is single-threaded, "
                                       f"chroma/runtime.py:125)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    args = parse()
    quiet_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    import ctypes as C
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

    def cfg_for(algorithm):
        return R.AlgorithmConfig(mode=R.Mode(wl.mode), deterministic=algorithm == "gauss-seidel",
                                 algorithm=None if algorithm == "gauss-seidel" else algorithm)

    def make_world(graph, partition):
        if N == 1:
            return RT.build_local_graphs(graph, partition, wl.gl)
        from paper_2107_00075_b200.dist import DistWorld
        return DistWorld(graph, partition, wl.gl)

    world = make_world(g, pm)
    lg = world.local_graphs[0] if N == 1 else world.local_graph
    cold_ms = None  # first call on a fresh world: includes any per-world schedule (C1/C2)
    n_out = world.output_length() if hasattr(world, "output_length") else world.num_global_vertices
    out = torch.empty(n_out, dtype=torch.int32, device=f"cuda:{local}")
    tbuf = (C.c_double * 5)()

    def timed_steps(cfg, K, W):
        """W untimed + K timed run_distributed calls; per-step device times (CUDA events
        on the world's stream inside the library: whole call, colouring kernel)."""
        nonlocal cold_ms
        for i in range(W):
            R.run_distributed(world, cfg, out=out)
            if i == 0 and cold_ms is None:
                _lib.check(_lib.lib().chroma_world_last_timing(world.handle.h, tbuf))
                cold_ms = tbuf[0] * 1e3
        barrier()
        torch.cuda.synchronize()
        l0 = launch_count()
        per, kern, reps = [], [], None
        for _ in range(K):
            barrier()
            _, reps = R.run_distributed(world, cfg, out=out)
            _lib.check(_lib.lib().chroma_world_last_timing(world.handle.h, tbuf))
            per.append(tbuf[0])
            kern.append(tbuf[1] if cfg.deterministic else reps[0].time_color_s)
        torch.cuda.synchronize()
        barrier()
        return per, kern, reps, launch_count() - l0

    # ---- the headline: deterministic (bit-exact) colouring
    cfg = cfg_for(wl.algorithm)
    clk = Clocks(local) if rank == 0 else None
    per, kern, reports, launches = timed_steps(cfg, args.steps, args.warmup)
    clocks = clk.stop() if clk else None
    T = allmax(sum(per))
    TK = allmax(sum(kern))
    value = m * args.steps / T

    def gather_colors():
        c = out.cpu().numpy()
        if N == 1:
            return c
        own = out.clone()
        sizes = [None] * N
        dist.all_gather_object(sizes, int(own.numel()))
        bufs = [torch.empty(s, dtype=torch.int32, device=own.device) for s in sizes]
        dist.all_gather(bufs, own)
        return torch.cat(bufs).cpu().numpy()  # partition_block: owned ranges are contiguous in gid order

    # per-phase device times and the halo (RoundReport fields, chroma/runtime.py:83-108)
    phases = {"color_ms": 1e3 * sum(r.time_color_s for r in reports),
              "comm_ms": 1e3 * sum(r.time_comm_s for r in reports),
              "detect_ms": 1e3 * sum(r.time_detect_s for r in reports)}
    pairs = sum(r.bytes_sent for r in reports) // 12  # reference accounting: 12 B per (gid, colour)
    halo = {"pairs_per_step": pairs, "bytes_sent_reference_accounting": 12 * pairs,
            "payload_bytes": 4 * pairs,  # int32 colour per ghost copy on the wire
            "nvlink_GBps": (4 * pairs / (phases["comm_ms"] * 1e-3) / 1e9) if N > 1 and phases["comm_ms"] > 0 else None,
            "nvlink_peak_GBps": "770 per direction (measured peer copy, B200_PROFILING.md)"}
    gcol = gather_colors()
    ncol = nviol = sha = None
    gold = wl.golden(N)
    if rank == 0:
        ncol, _ = V.color_stats(gcol)
        mask = None
        if wl.mode == "pd2":
            mask = np.zeros(g.num_vertices, np.uint8)
            mask[: g.num_vertices // 2] = 1
        nviol = V.count_violations(g, gcol, wl.vmode, mask)
        sha = sha256_i32(gcol)
    parity = None
    if rank == 0 and gold and cfg.deterministic:
        ref = (gold.get("run") or {})
        parity = {"oracle_sha256": ref.get("sha256"), "colour_sha256": sha,
                  "match": ref.get("sha256") == sha if ref.get("sha256") else None,
                  "oracle_rounds": ref.get("rounds"), "rounds": len(reports),
                  "oracle_colors": ref.get("colors"),
                  "csr_sha256_match": gold.get("col_sha256") == hashlib.sha256(
                      np.ascontiguousarray(g.col_indices).astype("<i8").tobytes()).hexdigest()}
    # ---- free-running mode on the same world (sub-record)
    free = None
    if not args.no_free and cfg.deterministic and wl.name in ("c3", "c4", "c5"):
        fcfg = cfg_for("free")
        fper, _, freps, _ = timed_steps(fcfg, args.steps, 1)
        Tf = allmax(sum(fper))
        fcol = gather_colors()
        if rank == 0:
            fn, _ = V.color_stats(fcol)
            ref_n = ((gold or {}).get("run") or {}).get("colors")
            free = {"value": m * args.steps / Tf, "ms_per_step": 1e3 * Tf / args.steps, "rounds": len(freps),
                    "phases_ms_rank0": {"color_ms": 1e3 * sum(r.time_color_s for r in freps),
                                        "comm_ms": 1e3 * sum(r.time_comm_s for r in freps),
                                        "detect_ms": 1e3 * sum(r.time_detect_s for r in freps)},
                    "colors": fn, "oracle_deterministic_colors": ref_n,
                    "within_5pct": (fn <= 1.05 * ref_n) if ref_n else None,
                    "violations": V.count_violations(g, fcol, wl.vmode)}
    # ---- the reference's default mode (Jacobi sweeps, deterministic=False) on the same world
    jac = None
    if not args.no_free and cfg.deterministic and wl.name == "c3":
        jcfg = R.AlgorithmConfig(mode=R.Mode(wl.mode))  # the reference's defaults
        jsteps = max(1, min(args.steps, 2))
        jper, _, jreps, _ = timed_steps(jcfg, jsteps, 1)
        Tj = allmax(sum(jper))
        jcol = gather_colors()
        if rank == 0:
            jsha = sha256_i32(jcol)
            jref = (gold or {}).get(f"{wl.mode}_p{N}_jacobi") or {}
            jac = {"value": m * jsteps / Tj, "ms_per_step": 1e3 * Tj / jsteps, "rounds": len(jreps),
                   "colors": V.color_stats(jcol)[0], "colour_sha256": jsha,
                   "oracle_sha256": jref.get("sha256"),
                   "match": (jref.get("sha256") == jsha) if jref.get("sha256") else None,
                   "oracle_run_s": jref.get("oracle_run_s")}
    # ---- the checker (verify_d1 count, k_count_d1) on the headline's device colours, C3 at N=1
    ver = None
    if rank == 0 and N == 1 and wl.name == "c3" and not args.no_free:
        R.run_distributed(world, cfg, out=out)
        h = _lib.csr_of(g)
        nv = C.c_int64(0)
        vt = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(_lib.lib().chroma_verify(h.h, C.c_void_p(out.data_ptr()), None, 0, C.byref(nv), None, 0,
                                                1), "verify")
            vt.append(time.perf_counter() - t0)
        tv = min(vt[1:])
        rate = gather_rate()
        ver = {"ms": 1e3 * tv, "violations": int(nv.value), "edges_per_s": m / tv,
               "timing": "host perf_counter around chroma_verify (device colours, count only), best of 3 after 1",
               "gather_floor_ms": 1e3 * m / rate if rate else None,
               "gather_frac": (m / rate) / tv if rate else None,
               "note": "one random colour load per edge (u > v), L1-wavefront bound (profiles/gather_roofline.json)"}
    # ---- roofline of the dominant kernel (the round-0 colouring)
    n_o = lg.owned_count
    nnz_o = int(lg.row_offsets[n_o]) if N > 1 else len(g.col_indices)
    touched = lg.num_local if N > 1 else g.num_vertices
    B = round0_bytes(n_o, nnz_o, touched)
    kernel_s = TK / args.steps
    peak, peak_kind = peaks()
    achieved = B / kernel_s / 1e9 if kernel_s > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"{wl.name}_{wl.algorithm}_p{N}", {}).get("dram_bytes_per_launch")
    except Exception:
        traffic = None
    kname = {"c3": "k_gs_chunked (chunked exact Gauss-Seidel: throughput first pass + latency-bound dataflow)",
             "c1": "k_gs_cluster (level-synchronous Gauss-Seidel on one cluster)",
             "c2": "k_gs_cluster (level-synchronous Gauss-Seidel on one cluster)",
             "c4": "gs_d1_kernel over the square G^2 (level-ordered Gauss-Seidel; algorithmic bytes counted on G)"}.get(wl.name, "round-0 colour phase")
    # second roofline: random neighbour-colour loads retire at ~1 per SM clock from L2
    # (one L1 wavefront each; scripts/gather_roofline.cu), so a colouring pass that loads
    # each lower neighbour's colour once has a floor of (lower entries) / (gather rate)
    gather_roof = None
    rate = gather_rate()
    if rate and wl.name == "c3":
        lower = m if N == 1 else nnz_o // 2
        gather_roof = {"gathers_per_launch": lower, "rate_per_s": rate,
                       "floor_ms": 1e3 * lower / rate, "frac": (lower / rate) / kernel_s if kernel_s > 0 else None,
                       "gathers": "one colour load per lower neighbour (round 0 reads rows up to the vertex)"
                                  + ("" if N == 1 else "; nnz_owned / 2 at N > 1")}
    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        from paper_2107_00075_b200.graph import Graph
        off_p = torch.from_numpy(np.ascontiguousarray(g.row_offsets, dtype=np.int64)).pin_memory()
        col_p = torch.from_numpy(np.ascontiguousarray(g.col_indices, dtype=np.int64)).pin_memory()
        hg = Graph(g.num_vertices, off_p.numpy(), col_p.numpy())
        hpm = PT.partition_block(hg, N)

        def e2e_steps(graph, partition, K, W):
            et = []
            for it in range(K + W):
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                wv = make_world(graph, partition)
                t1 = time.perf_counter()
                colors, _ = R.run_distributed(wv, cfg)
                torch.cuda.synchronize()
                el = time.perf_counter() - t0
                t2 = time.perf_counter()
                del wv, colors
                if os.environ.get("CHROMA_E2E_TRACE"):
                    print(f"[e2e] step {it}: build {1e3 * (t1 - t0):.1f} ms, run {1e3 * (el - (t1 - t0)):.1f} ms, "
                          f"release {1e3 * (time.perf_counter() - t2):.1f} ms", file=sys.stderr, flush=True)
                if it >= W:
                    et.append(el)
            return allmax(sum(et) / len(et))

        K = max(1, min(args.steps, 3))
        # the drop-in caller's input: plain (pageable) NumPy int64 arrays
        pg = Graph(g.num_vertices, np.array(g.row_offsets, np.int64), np.array(g.col_indices, np.int64))
        tp = e2e_steps(pg, PT.partition_block(pg, N), K, max(1, min(args.warmup, 3)))
        te = e2e_steps(hg, hpm, K, 1)
        e2e = {"value": m / tp, "unit": UNIT,
               "h2d_bytes_per_step": int(off_p.numel() * 8 + col_p.numel() * 8),
               "d2h_bytes_per_step": int(4 * n_out),
               "timing": "host perf_counter around build_local_graphs (int64 CSR from pageable NumPy arrays "
                         "to the device world) + run_distributed (colours back into host memory)",
               "pinned_value": m / te,
               "host_cores": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()}
        del pg
        del off_p, col_p
    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, g, N)
    if rank == 0:
        line = {"metric": wl.metric, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": wl.data,
                "config": {"workload": f"{wl.desc}, partition_block P={N}, {wl.algorithm}",
                           "n": g.num_vertices, "m": m, "ghost_layers": wl.gl, "rounds": len(reports),
                           "colors": ncol, "violations": nviol, "colour_sha256": sha,
                           "parallelism": f"vertex-range x{N}", "phases_ms_rank0": phases, "halo": halo,
                           "caching": "none: every step rebuilds the colouring state (no per-world schedule)"
                                      if wl.name == "c3" else "per-world round-0 schedule built in warm-up",
                           "cold_call_ms": cold_ms,
                           "l2": f"inputs larger than L2 (int32 col {4 * len(g.col_indices) / 1e6:.0f} MB)"},
                "parity": parity, "free": free, "jacobi": jac, "verify": ver,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak if achieved else None, "traffic": traffic,
                             "kernel": kname, "algorithmic_bytes_per_launch": B, "kernel_ms": kernel_s * 1e3,
                             "peak_kind": peak_kind, "gather": gather_roof},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        emit(line)
    if N > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
