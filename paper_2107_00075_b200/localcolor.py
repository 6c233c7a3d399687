"""On-rank colouring kernels (drop-in for chroma.localcolor, chroma/localcolor.py).

``speculative_color`` / ``speculative_color_d2`` / ``serial_greedy`` run on the GPU
(libchroma_b200):
  deterministic=True  -> ordered-dataflow Gauss-Seidel first fit (bit-exact with the
                         reference's ascending-order loop, chroma/localcolor.py:161-165)
  deterministic=False -> the reference's synchronous Jacobi sweeps with the
                         larger-id-wins loser rule (chroma/localcolor.py:214-227,
                         292-303), also bit-exact.  ``set_free_running(True)`` switches
                         to the B200 free-running speculative kernel instead.
The VB / EB kernel choice selects the same losers in the reference (F3); on the GPU the
Jacobi sweep runs warp-per-vertex kernels for VB and edge-parallel (merge-path over the
pending rows' entries) kernels for EB -- same colours, different load balance.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum

import numpy as np

from . import _lib

__all__ = ["Kernel", "KernelChoice", "ForbiddenMask", "first_fit_color", "new_coloring",
           "serial_greedy", "select_kernel", "speculative_color", "speculative_color_d2",
           "two_hop_neighbors", "set_free_running"]

_MAX_INTERNAL_SWEEPS = 10_000
_FREE_RUNNING = False


def set_free_running(flag: bool) -> None:
    """deterministic=False -> B200 free-running kernel (True) or exact Jacobi (False)."""
    global _FREE_RUNNING
    _FREE_RUNNING = bool(flag)


def _algo(deterministic: bool) -> int:
    if deterministic:
        return _lib.ALGO_GS
    return _lib.ALGO_FREE if _FREE_RUNNING else _lib.ALGO_JACOBI


class Kernel(Enum):
    VERTEX_BASED = "vb"
    EDGE_BASED = "eb"
    NET_BASED_D2 = "nb-d2"


@dataclass(frozen=True)
class KernelChoice:
    kind: Kernel | None = None
    max_degree_threshold: int = 6000

    def __post_init__(self) -> None:
        if self.max_degree_threshold <= 0:
            raise ValueError("max_degree_threshold must be positive")


def select_kernel(st, cfg: KernelChoice | None = None) -> KernelChoice:
    """Edge-based iff delta_max > threshold (chroma/localcolor.py:55-61)."""
    cfg = cfg or KernelChoice()
    if cfg.kind is not None:
        return cfg
    return replace(cfg, kind=Kernel.EDGE_BASED if st.delta_max > cfg.max_degree_threshold
                   else Kernel.VERTEX_BASED)


class ForbiddenMask:
    """64-colour sliding window (chroma/localcolor.py:64-95)."""

    __slots__ = ("base", "bits")
    _FULL = (1 << 64) - 1

    def __init__(self, base: int = 1):
        self.base = base
        self.bits = 0

    def forbid(self, color: int) -> None:
        off = color - self.base
        if 0 <= off < 64:
            self.bits |= 1 << off

    @property
    def saturated(self) -> bool:
        return self.bits == self._FULL

    def advance(self) -> None:
        self.base += 64
        self.bits = 0

    def smallest_allowed(self):
        if self.saturated:
            return None
        free = ~self.bits & self._FULL
        return self.base + (free & -free).bit_length() - 1


def first_fit_color(forbidden) -> int:
    """Smallest positive colour absent from `forbidden` (zeros/negatives ignored)."""
    a = np.asarray(forbidden).ravel()
    a = a[a > 0]
    if a.size == 0:
        return 1
    present = np.zeros(a.size + 2, dtype=bool)
    small = a[a <= a.size + 1].astype(np.int64)
    present[small] = True
    present[0] = True
    return int(np.argmin(present))


def new_coloring(num_vertices: int) -> np.ndarray:
    return np.zeros(num_vertices, dtype=np.int32)


def two_hop_neighbors(g, v: int) -> np.ndarray:
    """Vertices reachable in exactly two hops through any middle, minus v (chroma/localcolor.py:136-144)."""
    off, idx = g.row_offsets, g.col_indices
    one = idx[off[v]: off[v + 1]]
    if one.size == 0:
        return one
    two = np.unique(np.concatenate([idx[off[u]: off[u + 1]] for u in one.tolist()]))
    return two[two != v]


def serial_greedy(g, order=None) -> np.ndarray:
    """First fit in the given order (default ascending) on the GPU (chroma/localcolor.py:120-133)."""
    n = g.num_vertices
    if order is not None:
        order = np.asarray(order, dtype=np.int64)
        if len(order) != n or not np.array_equal(np.sort(order), np.arange(n)):
            raise ValueError("order is not a permutation of the vertices")
    out = np.zeros(n, dtype=np.int32)
    if n == 0:
        return out
    h = _lib.csr_of(g)
    o = None if order is None else _lib.i64(order)
    _lib.check(_lib.lib().chroma_serial_greedy(h.h, _lib.ptr(o) if o is not None else None,
                                               _lib.ptr(out), 0), "serial_greedy")
    return out


def _world_of(lg):
    wh = getattr(lg, "_wh", None)
    return wh if isinstance(getattr(lg, "rank", None), int) and wh is not None else None


def _color(lg, colors, worklist, dist: int, partial: bool, deterministic: bool, edge_based: bool = False):
    wl = _lib.i64(worklist).ravel()
    if wl.size == 0:
        return colors
    nl = lg.num_vertices
    if len(colors) != nl:
        raise ValueError("colors length does not match the graph")
    buf = np.ascontiguousarray(colors, dtype=np.int32)
    wh = _world_of(lg)
    algo = _algo(deterministic)
    if algo == _lib.ALGO_JACOBI and edge_based and dist == 1:
        algo = _lib.ALGO_JACOBI_EB
    if wh is not None:
        _lib.check(_lib.lib().chroma_world_color(wh.h, lg.rank, _lib.ptr(buf), _lib.ptr(wl), wl.size,
                                                 dist, int(partial), algo), "speculative_color")
    else:
        h = _lib.csr_of(lg)
        _lib.check(_lib.lib().chroma_color(h.h, _lib.ptr(buf), _lib.ptr(wl), wl.size, dist,
                                           int(partial), algo, 0), "speculative_color")
    if buf is not colors:
        colors[...] = buf
    return colors


def speculative_color(lg, colors, worklist, kernel: KernelChoice | None = None,
                      deterministic: bool = False) -> np.ndarray:
    """Distance-1 colouring of `worklist` in place (chroma/localcolor.py:198-227).
    kernel.kind EDGE_BASED runs the edge-parallel Jacobi kernels (181-195)."""
    eb = kernel is not None and kernel.kind is Kernel.EDGE_BASED
    return _color(lg, colors, worklist, 1, False, deterministic, eb)


def speculative_color_d2(lg, colors, worklist, partial: bool = False,
                         deterministic: bool = False) -> np.ndarray:
    """Distance-2 (partial: two-hop only) colouring in place (chroma/localcolor.py:274-303)."""
    return _color(lg, colors, worklist, 2, bool(partial), deterministic)
