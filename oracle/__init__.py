"""ctypes front-end of the C oracle (oracle/chroma_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package.
The C file restates the reference `chroma` algorithms (see its header for the
file:line map); tests/test_oracle_golden.py pins it against the reference's own
outputs stored in tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "chroma_oracle.c")
SRCS = (SRC, os.path.join(HERE, "chroma_gen.c"))

MODES = {"d1": 0, "d1-2gl": 1, "d2": 2, "pd2": 3}


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or any(os.path.getmtime(LIB_PATH) < os.path.getmtime(x)
                                                     for x in SRCS):
        subprocess.check_call(["make", "-C", HERE, "-s"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int32
        L.orc_gid_rand.restype = C.c_uint64
        L.orc_gid_rand.argtypes = [i64]
        L.orc_check_conflicts.argtypes = [i64, i64, P, P, P, C.c_int]
        L.orc_first_fit.restype = i32
        L.orc_first_fit.argtypes = [P, i64]
        L.orc_speculative_color.argtypes = [i64, P, P, P, P, i64, C.c_int, C.c_int, C.c_int]
        L.orc_serial_greedy.argtypes = [i64, P, P, P, P]
        L.orc_detect_d1.restype = i64
        L.orc_detect_d1.argtypes = [i64, i64, P, P, P, P, P, C.c_int]
        L.orc_detect_d2.restype = i64
        L.orc_detect_d2.argtypes = [P, P, P, P, P, P, i64, C.c_int, C.c_int]
        L.orc_world_build.restype = P
        L.orc_world_build.argtypes = [i64, P, P, i32, P, C.c_int, C.POINTER(C.c_int)]
        L.orc_world_free.argtypes = [P]
        L.orc_world_rank_info.argtypes = [P, i32, P]
        L.orc_world_rank_arrays.argtypes = [P, i32, P, P, P, P, P, P]
        L.orc_global_degrees.argtypes = [P]
        L.orc_world_rank_degrees.argtypes = [P, i32, P]
        L.orc_reset_exchange.argtypes = [P]
        L.orc_exchange.argtypes = [P, P, C.c_int, P, P]
        L.orc_run_distributed.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P, i64, P]
        L.orc_gen_rmat.restype = i64
        L.orc_gen_rmat.argtypes = [C.c_int, i64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, P, P]
        L.orc_gen_bipartite.restype = i64
        L.orc_gen_bipartite.argtypes = [i64, i64, C.c_uint64, P, P]
        L.orc_verify.restype = i64
        L.orc_verify.argtypes = [i64, P, P, P, P, C.c_int, P, i64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def gid_rand(gid: int) -> int:
    return int(lib().orc_gid_rand(int(gid)))


def first_fit(vals) -> int:
    a = _i64(vals)
    return int(lib().orc_first_fit(_p(a), len(a)))


def serial_greedy(off, col, order=None) -> np.ndarray:
    off, col = _i64(off), _i64(col)
    n = len(off) - 1
    out = np.zeros(n, dtype=np.int32)
    o = None if order is None else _i64(order)
    lib().orc_serial_greedy(n, _p(off), _p(col), None if o is None else _p(o), _p(out))
    return out


def speculative_color(off, col, colors: np.ndarray, worklist, dist=1, partial=False,
                      deterministic=False) -> np.ndarray:
    off, col = _i64(off), _i64(col)
    wl = _i64(worklist)
    assert colors.dtype == np.int32 and colors.flags.c_contiguous
    st = lib().orc_speculative_color(len(off) - 1, _p(off), _p(col), _p(colors), _p(wl), len(wl),
                                     dist, int(partial), int(deterministic))
    if st == 1:
        raise ValueError("worklist out of range")
    if st == 4:
        raise RuntimeError("speculative loop failed to settle")
    return colors


def detect_d1(owned, off, col, colors, gids, deg, rd) -> int:
    off, col, gids, deg = _i64(off), _i64(col), _i64(gids), _i64(deg)
    r = lib().orc_detect_d1(owned, len(off) - 1, _p(off), _p(col), _p(colors), _p(gids), _p(deg),
                            int(rd))
    if r < 0:
        raise ValueError("conflict check on the same global vertex")
    return int(r)


def detect_d2(off, col, colors, gids, deg, b2, partial, rd) -> int:
    off, col, gids, deg, b2 = _i64(off), _i64(col), _i64(gids), _i64(deg), _i64(b2)
    r = lib().orc_detect_d2(_p(off), _p(col), _p(colors), _p(gids), _p(deg), _p(b2), len(b2),
                            int(partial), int(rd))
    if r < 0:
        raise ValueError("conflict check on the same global vertex")
    return int(r)


def verify(off, col, colors, mode: str, mask=None, cap: int = 1 << 20) -> np.ndarray:
    off, col = _i64(off), _i64(col)
    colors = _i32(colors)
    n = len(off) - 1
    m = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
    out = np.zeros((cap, 4), dtype=np.int64)
    k = lib().orc_verify(n, _p(off), _p(col), _p(colors), None if m is None else _p(m),
                         {"d1": 0, "d2": 1, "pd2": 2}[mode], _p(out), cap)
    return out[: min(k, cap)].copy()


class World:
    """All ranks of a reference-semantics world (chroma/runtime.py:111-139)."""

    def __init__(self, off, col, owner, num_ranks: int, ghost_layers: int):
        self.off, self.col = _i64(off), _i64(col)
        self.owner = _i32(owner)
        self.n = len(self.off) - 1
        self.P = int(num_ranks)
        st = C.c_int(0)
        self.h = lib().orc_world_build(self.n, _p(self.off), _p(self.col), self.P, _p(self.owner),
                                       int(ghost_layers), C.byref(st))
        if st.value:
            raise ValueError("invalid world arguments")
        self.ghost_layers = ghost_layers

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_world_free(h)
            self.h = None

    def info(self, r: int) -> dict:
        a = np.zeros(8, dtype=np.int64)
        lib().orc_world_rank_info(self.h, r, _p(a))
        keys = ("owned", "ghost", "l1", "e_local", "e_ghost", "nnz", "nb1", "nb2")
        return dict(zip(keys, (int(x) for x in a)))

    def rank(self, r: int) -> dict:
        i = self.info(r)
        nl = i["owned"] + i["ghost"]
        off = np.zeros(nl + 1, np.int64)
        col = np.zeros(i["nnz"], np.int64)
        gids = np.zeros(nl, np.int64)
        go = np.zeros(i["ghost"], np.int32)
        b1 = np.zeros(i["nb1"], np.int64)
        b2 = np.zeros(i["nb2"], np.int64)
        lib().orc_world_rank_arrays(self.h, r, _p(off), _p(col), _p(gids), _p(go), _p(b1), _p(b2))
        i.update(row_offsets=off, col_indices=col, gids=gids, ghost_owner=go, boundary_d1=b1,
                 boundary_d2=b2)
        return i

    def degrees(self) -> list:
        lib().orc_global_degrees(self.h)
        out = []
        for r in range(self.P):
            i = self.info(r)
            d = np.zeros(i["owned"] + i["ghost"], np.int64)
            lib().orc_world_rank_degrees(self.h, r, _p(d))
            out.append(d)
        return out

    def reset_exchange(self) -> None:
        lib().orc_reset_exchange(self.h)

    def exchange(self, colorings: list, changed_only: bool) -> tuple:
        for c in colorings:
            assert c.dtype == np.int32 and c.flags.c_contiguous
        ptrs = (C.c_void_p * self.P)(*[c.ctypes.data for c in colorings])
        b, m = C.c_int64(0), C.c_int64(0)
        lib().orc_exchange(self.h, ptrs, int(changed_only), C.byref(b), C.byref(m))
        return int(b.value), int(m.value)

    def run(self, mode: str, recolor_degrees=False, deterministic=True, max_rounds=200):
        """Returns (colors, reports) with reports = list of dicts of the integer fields."""
        cap = max_rounds + 2
        colors = np.zeros(self.n, np.int32)
        rep = np.zeros((cap, 4), np.int64)
        rec = np.zeros((cap, self.P), np.int64)
        nr = C.c_int64(0)
        st = lib().orc_run_distributed(self.h, MODES[mode], int(recolor_degrees), int(deterministic),
                                       int(max_rounds), _p(colors), _p(rep), _p(rec), cap,
                                       C.byref(nr))
        reports = [{"round": i, "conflicts": int(rep[i, 0]), "bytes_sent": int(rep[i, 1]),
                    "messages_sent": int(rep[i, 2]), "recolored_per_rank": rec[i].tolist()}
                   for i in range(nr.value)]
        if st == 1:
            raise ValueError("invalid run arguments")
        if st == 3:
            raise RuntimeError(f"NonConvergence after {max_rounds} rounds")
        if st == 4:
            raise RuntimeError("internal sweep tripwire")
        return colors, reports


def gen_rmat(scale: int, edge_factor: int = 16, seed: int = 1, thresholds=None, permute: bool = True):
    """(row_offsets, col_indices) of the counter-based R-MAT (oracle/chroma_gen.c)."""
    if thresholds is None:
        a, b, c = 0.57, 0.19, 0.19
        t = float(1 << 32)
        thresholds = (int(a * t), int((a + b) * t), int((a + b + c) * t))
    n = 1 << scale
    off = np.zeros(n + 1, dtype=np.int64)
    col = np.empty(2 * edge_factor * n, dtype=np.int64)
    nnz = lib().orc_gen_rmat(scale, edge_factor, seed, *thresholds, int(permute), _p(off), _p(col))
    return off, col[:nnz]


def gen_bipartite(rows: int, nnz_per_row: int = 32, seed: int = 3):
    """(row_offsets, col_indices) of the counter-based random bipartite PD2 input."""
    off = np.zeros(2 * rows + 1, dtype=np.int64)
    col = np.empty(max(2 * rows * nnz_per_row, 1), dtype=np.int64)
    nnz = lib().orc_gen_bipartite(rows, nnz_per_row, seed, _p(off), _p(col))
    return off, col[:nnz]
