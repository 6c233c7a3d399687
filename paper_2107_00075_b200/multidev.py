"""One process, several GPUs: rank r of a partition on cuda:devices[r].

The reference keeps every rank in one process (chroma/runtime.py:111-139) and
run_distributed returns the global int32[n] (chroma/protocol.py:331-334).  On a box
with at least P GPUs, ``runtime.build_local_graphs(g, pm)`` returns this world
instead of P virtual ranks on one GPU: each rank's local graph is built on its own
device (the same device builder as one-rank-per-process ``dist.DistWorld``), the
static halo routing is agreed in-process, one NCCL communicator per rank comes from
ncclCommInitAll, and run_distributed drives every rank's round loop (pack -> NCCL
send/recv over NVLink -> unpack, detection, allreduce) from its own host thread --
the library calls release the GIL.  The caller's code does not change.

Selection: CHROMA_DEVICES="0,1,..." names the devices explicitly; otherwise all
visible devices are used when there are at least P of them and P > 1;
CHROMA_MULTI_GPU=0 keeps virtual ranks on one GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .dist import build_routing
from .runtime import LocalGraph, WorldHandle, device_stats

__all__ = ["MultiDeviceWorld", "devices_for"]


def devices_for(num_ranks: int):
    """The device list for a num_ranks-way world, or None for virtual ranks."""
    if num_ranks < 2 or os.environ.get("CHROMA_MULTI_GPU", "1") == "0":
        return None
    env = os.environ.get("CHROMA_DEVICES")
    if env:
        devs = [int(x) for x in env.split(",") if x.strip()]
        return devs[:num_ranks] if len(devs) >= num_ranks else None
    n = C.c_int(0)
    if _lib.lib().chroma_device_count(C.byref(n)) != _lib.OK:
        return None
    return list(range(num_ranks)) if n.value >= num_ranks else None


class _Comms:
    def __init__(self, devices):
        self.n = len(devices)
        arr = (C.c_int * self.n)(*devices)
        self.h = (C.c_void_p * self.n)()
        _lib.check(_lib.lib().chroma_comm_create_all(self.n, arr, self.h), "chroma_comm_create_all")

    def __del__(self):
        if _lib is not None and getattr(_lib, "_lib", None) is not None:
            for i in range(self.n):
                if self.h[i]:
                    _lib._lib.chroma_comm_destroy(self.h[i])


class MultiDeviceWorld:
    """All ranks of a partition in this process, rank r on devices[r] (RankWorld API)."""

    def __init__(self, g, pm, ghost_layers: int, devices):
        P = pm.num_ranks
        self.num_ranks = P
        self.ghost_layers = ghost_layers
        self.partition = pm
        self.num_global_vertices = g.num_vertices
        self.devices = list(devices)
        self.total_bytes = 0
        self.total_messages = 0
        self.workers = P
        # one host thread per rank, always the same one (per-thread library scratch is
        # also keyed by device, but a fixed thread keeps each rank's CUDA state local)
        self._pools = [ThreadPoolExecutor(max_workers=1) for _ in range(P)]
        # build every rank on its device, concurrently (each upload + build is one C call)
        self.handles = self.map_ranks(lambda r: WorldHandle(g, pm, ghost_layers, r, r + 1, self.devices[r]))
        self.handle = self.handles[0]
        self.source_stats = device_stats(self.handles[0])
        self.local_graphs = [LocalGraph(self.handles[r], r, ghost_layers) for r in range(P)]
        # static routing, agreed in-process (the alltoallv is a transpose of lists)
        lgs = self.local_graphs
        req = {}
        for r in range(P):
            build_routing_requests(lgs[r], P, r, req)
        self._routing = []
        for r in range(P):
            incoming = [req[p][r] for p in range(P)]
            self._routing.append(build_routing(lgs[r].gids, lgs[r].owned_count, lgs[r].ghost_owner, P, r,
                                               lambda _out, inc=incoming: inc))
        self._comms = _Comms(self.devices)

        def connect(r):
            sc, sl, rc, rl = (_lib.i64(x) for x in self._routing[r])
            st = _lib.lib().chroma_world_connect(self.handles[r].h, self._comms.h[r], P, r, _lib.ptr(sc),
                                                 _lib.ptr(sl), _lib.ptr(rc), _lib.ptr(rl))
            if st != _lib.OK:
                raise _lib.error_for(st, "chroma_world_connect: " +
                                     _lib.lib().chroma_last_error().decode(errors="replace"))

        self.map_ranks(connect)
        self._owned_gids = [lg.gids[: lg.owned_count].copy() for lg in lgs]
        self._graph = g
        self._vw = None

    def virtual_world(self):
        """A virtual-rank copy on devices[0] for the fine-grained exchange API
        (exchange_boundary_colors keeps its changed-only state there)."""
        if self._vw is None:
            from .runtime import _build_virtual
            self._vw = _build_virtual(self._graph, self.partition, self.ghost_layers, self.devices[0])
        return self._vw

    def map_ranks(self, fn):
        futs = [self._pools[r].submit(fn, r) for r in range(self.num_ranks)]
        return [f.result() for f in futs]

    def reset_exchange_state(self) -> None:
        self.total_bytes = 0
        self.total_messages = 0
        for h in self.handles:
            _lib.check(_lib.lib().chroma_world_reset_exchange(h.h))
        if self._vw is not None:
            self._vw.reset_exchange_state()

    def output_length(self) -> int:
        return self.num_global_vertices

    def run(self, mode: int, rd: bool, algo: int, max_rounds: int):
        """Every rank's chroma_run_distributed at once; returns (global colours, status,
        rank 0's report arrays)."""
        P = self.num_ranks
        cap = max_rounds + 2
        outs = [np.zeros(lg.owned_count, np.int32) for lg in self.local_graphs]
        reps = [(_lib.RoundReportC * cap)() for _ in range(P)]
        recs = [np.zeros((cap, P), np.int64) for _ in range(P)]
        nreps = [C.c_int64(0) for _ in range(P)]

        msgs = [""] * P

        def one(r):
            st = _lib.lib().chroma_run_distributed(self.handles[r].h, mode, int(rd), algo, int(max_rounds),
                                                   _lib.ptr(outs[r]), reps[r], _lib.ptr(recs[r]), cap,
                                                   C.byref(nreps[r]), 0)
            if st != _lib.OK:  # the message is thread-local in the library
                msgs[r] = _lib.lib().chroma_last_error().decode(errors="replace")
            return st

        sts = self.map_ranks(one)
        bad = [r for r in range(P) if sts[r] not in (_lib.OK, _lib.ENONCONV)]
        if bad:
            raise _lib.error_for(sts[bad[0]], f"run_distributed (rank {bad[0]}): {msgs[bad[0]]}")
        colors = np.zeros(self.num_global_vertices, np.int32)
        for r in range(P):
            colors[self._owned_gids[r]] = outs[r]
        st = next((x for x in sts if x not in (_lib.OK, _lib.ENONCONV)), None)
        if st is None:
            st = _lib.ENONCONV if _lib.ENONCONV in sts else _lib.OK
        return colors, st, reps[0], recs[0], nreps[0].value

    def last_timing(self):
        """Per-rank CUDA-event times of the last run (max over ranks is the step time)."""
        out = []
        for h in self.handles:
            t = (C.c_double * 5)()
            _lib.check(_lib.lib().chroma_world_last_timing(h.h, t))
            out.append(list(t))
        return out


def build_routing_requests(lg, P: int, r: int, req: dict) -> None:
    """Rank r's per-owner lists of ghost gids (what build_routing sends to each peer)."""
    gids = np.asarray(lg.gids, np.int64)
    go = np.asarray(lg.ghost_owner, np.int64)
    slots = np.argsort(go, kind="stable")
    counts = np.bincount(go, minlength=P)
    bounds = np.concatenate([[0], np.cumsum(counts)])
    asked = gids[lg.owned_count:][slots]
    req[r] = [asked[bounds[p]: bounds[p + 1]] for p in range(P)]
