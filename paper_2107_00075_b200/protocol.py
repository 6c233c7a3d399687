"""Distributed driver and cross-rank conflict resolution (drop-in for chroma.protocol).

``run_distributed`` executes the whole speculate-and-iterate loop of
chroma/protocol.py:263-334 inside libchroma_b200 (colour kernel, halo exchange,
conflict detection, count allreduce) with one 8*(3+P)-byte D2H per round for loop
control and RoundReport accounting.  Deterministic mode (Gauss-Seidel colouring +
exact replay of the in-place detection scan) and Jacobi mode are bit-exact with the
reference; the free-running mode (localcolor.set_free_running) trades that for
throughput and is checked by validity and colour count.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .localcolor import Kernel, KernelChoice, select_kernel, _algo
from .runtime import LocalGraph, RankWorld, RoundReport

__all__ = ["Mode", "AlgorithmConfig", "NonConvergenceError", "gid_rand", "gid_rand_array",
           "check_conflicts", "detect_conflicts_d1", "detect_conflicts_d2", "compute_global_degrees",
           "run_distributed", "ghost_layers_for"]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


class Mode(str, Enum):
    D1 = "d1"
    D1_2GL = "d1-2gl"
    D2 = "d2"
    PD2 = "pd2"


@dataclass
class AlgorithmConfig:
    """chroma/protocol.py:54-64.  ``algorithm`` (extension, default None) picks the
    GPU path for deterministic=False: None -> exact Jacobi, "free" -> free-running."""

    mode: Mode = Mode.D1
    recolor_degrees: bool = False
    kernel: KernelChoice = field(default_factory=KernelChoice)
    deterministic: bool = False
    max_rounds: int = 200
    algorithm: str | None = None

    def __post_init__(self) -> None:
        if self.max_rounds < 1:
            raise ValueError("max_rounds must be >= 1")
        if self.algorithm not in (None, "free", "jacobi", "gauss-seidel"):
            raise ValueError(f"unknown algorithm {self.algorithm!r}")

    def algo_code(self) -> int:
        if self.algorithm == "free":
            return _lib.ALGO_FREE
        if self.algorithm == "jacobi":
            return _lib.ALGO_JACOBI
        if self.algorithm == "gauss-seidel":
            return _lib.ALGO_GS
        return _algo(self.deterministic)


class NonConvergenceError(RuntimeError):
    def __init__(self, message: str, reports: list):
        super().__init__(message)
        self.reports = reports


def ghost_layers_for(mode: Mode) -> int:
    return 1 if Mode(mode) is Mode.D1 else 2


def gid_rand(gid: int) -> int:
    """splitmix64 finaliser of gid + 0x9E3779B97F4A7C15 (chroma/protocol.py:79-88)."""
    return int(_lib.lib().chroma_gid_rand(C.c_int64(int(gid)).value))


def gid_rand_array(gids: np.ndarray) -> np.ndarray:
    z = np.asarray(gids).astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def check_conflicts(v: int, u: int, colors: np.ndarray, gids: np.ndarray, degrees: np.ndarray,
                    recolor_degrees: bool) -> int:
    """Resolve one potential conflict in place (chroma/protocol.py:99-133)."""
    cv, cu = int(colors[v]), int(colors[u])
    if cv == 0 or cu == 0 or cv != cu:
        return 0
    c2 = np.array([cv, cu], dtype=np.int32)
    g2 = np.array([int(gids[v]), int(gids[u])], dtype=np.int64)
    d2 = np.array([int(degrees[v]), int(degrees[u])], dtype=np.int64) if degrees is not None \
        else np.zeros(2, np.int64)
    res = C.c_int(0)
    _lib.check(_lib.lib().chroma_check_conflicts(0, 1, _lib.ptr(c2), _lib.ptr(g2), _lib.ptr(d2),
                                                 int(bool(recolor_degrees)), C.byref(res)))
    colors[v], colors[u] = c2[0], c2[1]
    return int(res.value)


def _detect(lg, colors, degrees, dist: int, partial: bool, recolor_degrees: bool) -> int:
    buf = np.ascontiguousarray(colors, dtype=np.int32)
    if len(buf) != lg.num_local:
        raise ValueError("colors length does not match the local graph")
    cnt = C.c_int64(0)
    wh = getattr(lg, "_wh", None)
    if isinstance(lg, LocalGraph) and wh is not None:
        deg = None if degrees is None else _lib.i64(degrees)
        _lib.check(_lib.lib().chroma_world_detect(wh.h, lg.rank, _lib.ptr(buf),
                                                  _lib.ptr(deg) if deg is not None else None, dist,
                                                  int(partial), int(bool(recolor_degrees)), C.byref(cnt)),
                   "detect_conflicts")
    else:
        h = _lib.csr_of(lg)
        gids = _lib.i64(lg.gids)
        deg = _lib.i64(degrees) if degrees is not None else np.zeros(lg.num_local, np.int64)
        rows = (np.arange(lg.owned_count, lg.num_local, dtype=np.int64) if dist == 1
                else _lib.i64(lg.boundary_d2))
        _lib.check(_lib.lib().chroma_detect(h.h, _lib.ptr(buf), _lib.ptr(gids), _lib.ptr(deg),
                                            _lib.ptr(rows), rows.size, dist, int(partial),
                                            int(bool(recolor_degrees)), C.byref(cnt), 0),
                   "detect_conflicts")
    if buf is not colors:
        colors[...] = buf
    return int(cnt.value)


def detect_conflicts_d1(lg, colors: np.ndarray, degrees: np.ndarray, recolor_degrees: bool) -> int:
    """Ghost-row scan with in-place uncolouring (chroma/protocol.py:136-157), GPU-exact."""
    return _detect(lg, colors, degrees, 1, False, recolor_degrees)


def detect_conflicts_d2(lg, colors: np.ndarray, degrees: np.ndarray, do_partial: bool,
                        recolor_degrees: bool) -> int:
    """boundary_d2 two-hop scan (chroma/protocol.py:160-194), GPU-exact."""
    if lg.ghost_layers < 2:
        raise ValueError("distance-2 detection needs a second ghost layer")
    return _detect(lg, colors, degrees, 2, bool(do_partial), recolor_degrees)


def compute_global_degrees(world: RankWorld) -> list:
    """Global degree of every owned and ghost vertex per rank (chroma/protocol.py:197-218)."""
    out = []
    for lg in world.local_graphs:
        d = np.zeros(lg.num_local, dtype=np.int64)
        _lib.check(_lib.lib().chroma_world_global_degrees(lg._wh.h, lg.rank, _lib.ptr(d)))
        lg.global_degrees = d
        out.append(d)
    return out


def _reports_from(rep, rec, n, P) -> list:
    return [RoundReport(round_index=int(rep[i].round_index), conflicts=int(rep[i].conflicts),
                        recolored_per_rank=[int(x) for x in rec[i, :P]],
                        bytes_sent=int(rep[i].bytes_sent), messages_sent=int(rep[i].messages_sent),
                        time_color_s=float(rep[i].time_color_s), time_comm_s=float(rep[i].time_comm_s),
                        time_detect_s=float(rep[i].time_detect_s)) for i in range(n)]


def _host_colors(n):
    """The int32 result array, in page-locked memory from torch's caching host
    allocator: the device-to-host copy runs at DMA speed into pages that are already
    mapped (a fresh np.zeros array costs ~1 ms of page faults per 8 MB), and the block
    returns to the cache when the caller drops the array.  Every element is written
    by the device before the array is returned."""
    try:
        import torch
    except ImportError:  # the package needs only NumPy on the host side
        return np.zeros(n, dtype=np.int32)
    if n > 0 and torch.cuda.is_available():
        return torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
    return np.zeros(n, dtype=np.int32)


def run_distributed(world, cfg: AlgorithmConfig, out=None):
    """Speculate-and-iterate driver for all four modes (chroma/protocol.py:263-334).

    Returns (int32[num_global_vertices] colours, list[RoundReport]) for a RankWorld;
    for a dist.DistWorld (one rank per process) the colours are this rank's owned slice.
    ``out`` (extension): a contiguous int32 CUDA tensor of that length on the world's
    device; the colours are written there (no device-to-host copy) and it is returned.
    """
    mode = Mode(cfg.mode)
    needed = ghost_layers_for(mode)
    if world.ghost_layers < needed:
        raise ValueError(f"mode {mode.value} needs {needed} ghost layer(s), "
                         f"world was built with {world.ghost_layers}")
    world.reset_exchange_state()
    # Kernel.EDGE_BASED iff delta_max > threshold (chroma/protocol.py:281): the Jacobi
    # sweeps then run edge-parallel (same losers, F3)
    kernel = select_kernel(world.source_stats, cfg.kernel)
    algo = cfg.algo_code()
    if algo == _lib.ALGO_JACOBI and kernel.kind is Kernel.EDGE_BASED and mode in (Mode.D1, Mode.D1_2GL):
        algo = _lib.ALGO_JACOBI_EB
    P = world.num_ranks
    cap = cfg.max_rounds + 2
    rep = (_lib.RoundReportC * cap)()
    rec = np.zeros((cap, P), dtype=np.int64)
    nrep = C.c_int64(0)
    n_out = world.output_length() if hasattr(world, "output_length") else world.num_global_vertices
    if hasattr(world, "run") and hasattr(world, "devices"):  # MultiDeviceWorld
        colors, st, rep, rec, nr = world.run(_lib.MODE[mode.value], bool(cfg.recolor_degrees), algo,
                                             int(cfg.max_rounds))
        reports = _reports_from(rep, rec, nr, P)
        world.total_bytes = sum(r.bytes_sent for r in reports)
        world.total_messages = sum(r.messages_sent for r in reports)
        if st == _lib.ENONCONV:
            raise NonConvergenceError(f"no convergence after {cfg.max_rounds} rounds", reports)
        _lib.check(st, "run_distributed")
        if out is not None:
            import torch
            out.copy_(torch.from_numpy(colors))
            return out, reports
        return colors, reports
    if out is not None:
        if (not getattr(out, "is_cuda", False) or str(out.dtype) != "torch.int32" or not out.is_contiguous()
                or out.numel() != n_out):
            raise ValueError(f"out must be a contiguous int32 CUDA tensor of {n_out} elements")
        colors, optr, flags = out, C.c_void_p(out.data_ptr()), 1
    else:
        colors = _host_colors(n_out)
        optr, flags = _lib.ptr(colors), 0
    st = _lib.lib().chroma_run_distributed(world.handle.h, _lib.MODE[mode.value],
                                           int(bool(cfg.recolor_degrees)), algo,
                                           int(cfg.max_rounds), optr, rep, _lib.ptr(rec),
                                           cap, C.byref(nrep), flags)
    reports = _reports_from(rep, rec, nrep.value, P)
    world.total_bytes = sum(r.bytes_sent for r in reports)
    world.total_messages = sum(r.messages_sent for r in reports)
    if st == _lib.ENONCONV:
        raise NonConvergenceError(f"no convergence after {cfg.max_rounds} rounds", reports)
    _lib.check(st, "run_distributed")
    return colors, reports
