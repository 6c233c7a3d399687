"""ctypes binding of libchroma_b200.so (include/chroma_b200.h).

The library is built in-tree by ``paper_2107_00075_b200._build`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared library is
missing or no CUDA device is visible, every colouring entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libchroma_b200.so")

OK, EVALUE, EPROTOCOL, ENONCONV, ERUNTIME, ECUDA = range(6)
DEVICE_PTRS = 1
MODE = {"d1": 0, "d1-2gl": 1, "d2": 2, "pd2": 3}
ALGO_GS, ALGO_FREE, ALGO_JACOBI, ALGO_JACOBI_EB = 0, 1, 2, 3


class RoundReportC(C.Structure):
    _fields_ = [("round_index", C.c_int64), ("conflicts", C.c_int64), ("bytes_sent", C.c_int64),
                ("messages_sent", C.c_int64), ("time_color_s", C.c_double),
                ("time_comm_s", C.c_double), ("time_detect_s", C.c_double)]


_lib = None


def lib():
    """Load the native library (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64, i32, u32, I = C.c_int64, C.c_int32, C.c_uint32, C.c_int
    PI64 = C.POINTER(C.c_int64)
    sig = {
        "chroma_last_error": (C.c_char_p, []),
        "chroma_version": (C.c_char_p, []),
        "chroma_device_count": (I, [C.POINTER(C.c_int)]),
        "chroma_gid_rand": (C.c_uint64, [i64]),
        "chroma_check_conflicts": (I, [i64, i64, P, P, P, I, C.POINTER(C.c_int)]),
        "chroma_csr_create": (I, [i64, P, P, I, u32, C.POINTER(P)]),
        "chroma_csr_destroy": (I, [P]),
        "chroma_serial_greedy": (I, [P, P, P, u32]),
        "chroma_color": (I, [P, P, P, i64, I, I, I, u32]),
        "chroma_detect": (I, [P, P, P, P, P, i64, I, I, I, PI64, u32]),
        "chroma_verify": (I, [P, P, P, I, PI64, P, i64, u32]),
        "chroma_color_stats": (I, [P, i64, I, PI64, PI64, P, i64, u32]),
        "chroma_world_create": (I, [i64, P, P, i32, P, i32, i32, i32, I, C.POINTER(P)]),
        "chroma_world_destroy": (I, [P]),
        "chroma_world_rank_info": (I, [P, i32, P]),
        "chroma_world_rank_arrays": (I, [P, i32, P, P, P, P, P, P]),
        "chroma_nccl_unique_id": (I, [P]),
        "chroma_comm_create": (I, [P, i32, i32, I, C.POINTER(P)]),
        "chroma_comm_destroy": (I, [P]),
        "chroma_comm_create_all": (I, [i32, P, P]),
        "chroma_world_connect": (I, [P, P, i32, i32, P, P, P, P]),
        "chroma_world_global_degrees": (I, [P, i32, P]),
        "chroma_world_reset_exchange": (I, [P]),
        "chroma_world_exchange": (I, [P, P, I, PI64, PI64]),
        "chroma_world_color": (I, [P, i32, P, P, i64, I, I, I]),
        "chroma_world_detect": (I, [P, i32, P, P, I, I, I, PI64]),
        "chroma_run_distributed": (I, [P, I, I, I, I, P, P, P, i64, PI64, u32]),
        "chroma_world_colors_device": (I, [P, i32, C.POINTER(P), PI64]),
        "chroma_world_last_timing": (I, [P, P]),
        "chroma_launch_count": (i64, []),
        "chroma_gen_rmat": (I, [i32, i64, C.c_uint64, u32, u32, u32, I, I, P, P, PI64]),
        "chroma_gen_random_bipartite": (I, [i64, i64, C.c_uint64, I, P, P, PI64]),
        "chroma_gen_box": (I, [i32, i64, i64, i64, I, P, P, PI64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTS = ("chroma_last_error", "chroma_version", "chroma_device_count", "chroma_gid_rand",
           "chroma_check_conflicts", "chroma_csr_create", "chroma_csr_destroy",
           "chroma_serial_greedy", "chroma_color", "chroma_detect", "chroma_verify",
           "chroma_color_stats", "chroma_world_create", "chroma_world_destroy",
           "chroma_world_rank_info", "chroma_world_rank_arrays", "chroma_nccl_unique_id",
           "chroma_comm_create", "chroma_comm_destroy",
           "chroma_world_connect", "chroma_world_global_degrees", "chroma_world_reset_exchange",
           "chroma_world_exchange", "chroma_world_color", "chroma_world_detect",
           "chroma_run_distributed", "chroma_world_colors_device", "chroma_world_last_timing",
           "chroma_launch_count", "chroma_gen_rmat", "chroma_gen_random_bipartite", "chroma_gen_box",
           "chroma_comm_create_all")


def error_for(status: int, msg: str) -> Exception:
    """The reference's exception class for a status code."""
    if status == EVALUE:
        return ValueError(msg)
    if status == EPROTOCOL:
        from .runtime import ProtocolError
        return ProtocolError(msg)
    if status == ERUNTIME:
        return RuntimeError(msg)
    return RuntimeError(f"CUDA failure ({status}): {msg}")


def check(status: int, what: str = "") -> None:
    """Map a status code to the reference's exception classes."""
    if status == OK:
        return
    msg = lib().chroma_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    raise error_for(status, msg)


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int64)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


_device = None


def default_device() -> int:
    """CUDA device used by handles created without an explicit device."""
    global _device
    if _device is None:
        env = os.environ.get("CHROMA_DEVICE")
        if env is not None:
            _device = int(env)
        else:
            try:
                import torch
                _device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except Exception:
                _device = 0
    return _device


def set_device(d: int) -> None:
    global _device
    _device = int(d)


class CsrHandle:
    """Device copy of a CSR graph (chroma_csr)."""

    def __init__(self, row_offsets, col_indices, device: int | None = None):
        off, col = i64(row_offsets), i64(col_indices)
        self.n = len(off) - 1
        self.device = default_device() if device is None else device
        h = C.c_void_p()
        check(lib().chroma_csr_create(self.n, ptr(off), ptr(col), self.device, 0, C.byref(h)),
              "chroma_csr_create")
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.chroma_csr_destroy(h)
            self.h = None


def csr_of(g) -> CsrHandle:
    """Cached device CSR for any graph-like object (row_offsets / col_indices)."""
    key = (id(g.row_offsets), id(g.col_indices), len(g.col_indices))
    cached = getattr(g, "_chroma_csr", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    h = CsrHandle(g.row_offsets, g.col_indices)
    try:
        object.__setattr__(g, "_chroma_csr", (key, h))
    except Exception:
        pass
    return h


def launch_count() -> int:
    return int(lib().chroma_launch_count())
