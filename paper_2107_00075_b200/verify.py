"""GPU properness checker (drop-in for chroma.verify, chroma/verify.py).

verify_d1 / verify_d2 / color_stats run as CUDA kernels over the undistributed
graph; violations are returned as the reference's Violation objects in the
reference's order (uncoloured, then d1 edges by (u, w), then two-hop paths by
(middle, i, j)).  chromatic_oracle is the reference's exact small-graph oracle,
kept on the host (exponential backtracking for <= a few dozen vertices).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib

__all__ = ["ViolationKind", "Violation", "verify_d1", "verify_d2", "chromatic_oracle", "color_stats",
           "GraphTooLarge", "count_violations"]


class ViolationKind(str, Enum):
    D1_EDGE = "d1-edge"
    D2_PATH = "d2-path"
    PD2_PATH = "pd2-path"
    UNCOLORED = "uncolored"


_KINDS = {0: ViolationKind.UNCOLORED, 1: ViolationKind.D1_EDGE, 2: ViolationKind.D2_PATH,
          3: ViolationKind.PD2_PATH}


@dataclass(frozen=True)
class Violation:
    kind: ViolationKind
    u: int
    w: int | None = None
    middle: int | None = None

    def __str__(self) -> str:
        if self.kind is ViolationKind.UNCOLORED:
            return f"vertex {self.u} is uncolored"
        if self.kind is ViolationKind.D1_EDGE:
            return f"edge ({self.u},{self.w}) shares a color"
        return f"path {self.u}-{self.middle}-{self.w} endpoints share a color"


class GraphTooLarge(ValueError):
    pass


def _run(g, colors, mode: int, mask, want_rows: bool):
    if len(colors) != g.num_vertices:
        raise ValueError(f"coloring has {len(colors)} entries for {g.num_vertices} vertices")
    c = _lib.i32(colors)
    m = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
    h = _lib.csr_of(g)
    nv = C.c_int64(0)
    _lib.check(_lib.lib().chroma_verify(h.h, _lib.ptr(c), _lib.ptr(m) if m is not None else None, mode,
                                        C.byref(nv), None, 0, 0), "verify")
    total = int(nv.value)
    if not want_rows or total == 0:
        return total, np.zeros((0, 4), np.int64)
    rows = np.zeros((total, 4), dtype=np.int64)
    _lib.check(_lib.lib().chroma_verify(h.h, _lib.ptr(c), _lib.ptr(m) if m is not None else None, mode,
                                        C.byref(nv), _lib.ptr(rows), total, 0), "verify")
    return total, rows


def _to_violations(rows: np.ndarray) -> list:
    out = []
    for k, u, w, m in rows.tolist():
        out.append(Violation(_KINDS[k], int(u), None if w < 0 else int(w), None if m < 0 else int(m)))
    return out


def verify_d1(g, colors: np.ndarray) -> list:
    """Empty iff a proper distance-1 colouring with no uncoloured vertex (chroma/verify.py:61-70)."""
    return _to_violations(_run(g, colors, 0, None, True)[1])


def verify_d2(g, colors: np.ndarray, partial: bool = False, endpoint_mask: np.ndarray | None = None) -> list:
    """Distance-2 checker; partial -> only two-path endpoints must differ (chroma/verify.py:73-104)."""
    return _to_violations(_run(g, colors, 2 if partial else 1, endpoint_mask, True)[1])


def count_violations(g, colors, mode: str = "d1", endpoint_mask=None) -> int:
    """Number of violations only (no listing) -- the fast path used by the bench."""
    return _run(g, colors, {"d1": 0, "d2": 1, "pd2": 2}[mode], endpoint_mask, False)[0]


def color_stats(colors: np.ndarray):
    """(number of distinct positive colours, {colour: count}) (chroma/verify.py:107-112)."""
    c = _lib.i32(colors).ravel()
    k, mx = C.c_int64(0), C.c_int64(0)
    _lib.check(_lib.lib().chroma_color_stats(_lib.ptr(c), c.size, _lib.default_device(), C.byref(k),
                                             C.byref(mx), None, 0, 0), "color_stats")
    hist = np.zeros(int(mx.value) + 1, dtype=np.int64)
    _lib.check(_lib.lib().chroma_color_stats(_lib.ptr(c), c.size, _lib.default_device(), C.byref(k),
                                             C.byref(mx), _lib.ptr(hist), hist.size, 0), "color_stats")
    return int(k.value), {int(i): int(v) for i, v in enumerate(hist.tolist()) if i > 0 and v > 0}


def chromatic_oracle(g, max_n: int = 12) -> int:
    """Exact chromatic number by iterative deepening (host; chroma/verify.py:115-177)."""
    n = g.num_vertices
    if n > max_n:
        raise GraphTooLarge(f"graph has {n} vertices, oracle limit is {max_n}")
    if n == 0:
        return 0
    if len(g.col_indices) == 0:
        return 1
    adj = [g.col_indices[g.row_offsets[v]: g.row_offsets[v + 1]].tolist() for v in range(n)]
    deg = [len(a) for a in adj]
    for k in range(2, n + 1):
        color = [0] * n
        banned = [0] * n     # bitmask of colours used by neighbours

        def choose():
            best, key = -1, (-1, -1)
            for v in range(n):
                if not color[v]:
                    kk = (bin(banned[v]).count("1"), deg[v])
                    if kk > key:
                        best, key = v, kk
            return best

        def place(v, used):
            if v < 0:
                return True
            for c in range(1, min(used + 1, k) + 1):
                bit = 1 << c
                if banned[v] & bit:
                    continue
                color[v] = c
                changed = [u for u in adj[v] if not banned[u] & bit]
                for u in changed:
                    banned[u] |= bit
                if place(choose(), max(used, c)):
                    return True
                color[v] = 0
                for u in changed:
                    banned[u] &= ~bit
            return False

        if place(choose(), 0):
            return k
    return n
