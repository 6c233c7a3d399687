"""Device-resident ranks and the halo exchange (drop-in for chroma.runtime).

The reference simulates ranks as Python data in one process (chroma/runtime.py:1-9).
Here ``build_local_graphs`` builds every rank's local graph ON THE GPU
(libchroma_b200 ``chroma_world_create``) with the reference's exact local-id layout
(owned, layer-1, layer-2 ghosts each ascending by gid; rows sorted by local id;
chroma/runtime.py:149-268).  ``LocalGraph`` arrays are views fetched lazily from
the device, so the reference's attribute API keeps working.

One process can hold all ranks of a partition ("virtual ranks", halo exchange is a
device copy) or -- see ``paper_2107_00075_b200.dist`` -- exactly one rank per GPU
process, with the halo moving over NCCL / NVLink.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import GraphStats
from .partition import PartitionMap

__all__ = ["LocalGraph", "RankWorld", "RoundReport", "ProtocolError", "build_local_graphs",
           "exchange_boundary_colors", "allreduce_sum", "snapshot_ghost_colors",
           "restore_ghost_colors"]

BYTES_PER_PAIR = 12   # u64 gid + u32 colour per updated ghost copy (chroma/runtime.py:34)


class ProtocolError(RuntimeError):
    """A message referenced a gid unknown to the receiving rank (chroma/runtime.py:37-38)."""


class WorldHandle:
    """Owns one chroma_world."""

    def __init__(self, g, pm, ghost_layers: int, rank_lo: int, rank_hi: int, device: int | None = None):
        off = _lib.i64(g.row_offsets)
        col = _lib.i64(g.col_indices)
        # partition_block maps are regenerated on the device (no owner array upload)
        owner = None if getattr(pm, "_block", False) else _lib.i32(pm.owner)
        self.device = _lib.default_device() if device is None else device
        h = C.c_void_p()
        _lib.check(_lib.lib().chroma_world_create(int(g.num_vertices), _lib.ptr(off), _lib.ptr(col),
                                                  int(pm.num_ranks), _lib.ptr(owner) if owner is not None
                                                  else None, int(ghost_layers),
                                                  int(rank_lo), int(rank_hi), self.device, C.byref(h)),
                   "build_local_graphs")
        self.h = h
        self.rank_lo, self.rank_hi = rank_lo, rank_hi

    def info(self, r: int) -> dict:
        a = np.zeros(16, dtype=np.int64)
        _lib.check(_lib.lib().chroma_world_rank_info(self.h, r, _lib.ptr(a)))
        keys = ("owned", "ghost", "l1", "e_local", "e_ghost", "nnz", "nb1", "nb2", "delta_max",
                "n_global", "m_global", "ghost_layers", "lid_off")
        return {k: int(a[i]) for i, k in enumerate(keys)}

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None and getattr(_lib, "_lib", None) is not None:
            _lib._lib.chroma_world_destroy(h)
            self.h = None


class LocalGraph:
    """One rank's subgraph: owned vertices first, then ghosts (chroma/runtime.py:41-80).

    Array attributes (row_offsets, col_indices, gids, ghost_owner, boundary_d1,
    boundary_d2) are int64/int32 NumPy copies of the device data, fetched on first use.
    """

    _ARRAYS = ("row_offsets", "col_indices", "gids", "ghost_owner", "boundary_d1", "boundary_d2")

    def __init__(self, world_handle: WorldHandle, rank: int, ghost_layers: int):
        self._wh = world_handle
        self.rank = rank
        i = world_handle.info(rank)
        self.owned_count = i["owned"]
        self.ghost_count = i["ghost"]
        self.first_layer_ghost_count = i["l1"]
        self.num_local_edges = i["e_local"]
        self.num_ghost_edges = i["e_ghost"]
        self.ghost_layers = ghost_layers
        self._nnz, self._nb1, self._nb2 = i["nnz"], i["nb1"], i["nb2"]
        self._arrays: dict | None = None
        self._gid_to_lid: dict | None = None
        self.global_degrees: np.ndarray | None = None

    def _fetch(self, name: str) -> np.ndarray:
        """One LocalGraph array, copied from the device on first use."""
        if self._arrays is None:
            self._arrays = {}
        if name not in self._arrays:
            nl = self.num_local
            shapes = {"row_offsets": (nl + 1, np.int64), "col_indices": (self._nnz, np.int64),
                      "gids": (nl, np.int64), "ghost_owner": (self.ghost_count, np.int32),
                      "boundary_d1": (self._nb1, np.int64), "boundary_d2": (self._nb2, np.int64)}
            size, dt = shapes[name]
            arr = np.zeros(size, dt)
            ptrs = [_lib.ptr(arr) if k == name else None for k in self._ARRAYS]
            _lib.check(_lib.lib().chroma_world_rank_arrays(self._wh.h, self.rank, *ptrs))
            self._arrays[name] = arr
        return self._arrays[name]

    def __getattr__(self, name):
        if name in LocalGraph._ARRAYS:
            return self._fetch(name)
        raise AttributeError(name)

    @property
    def gid_to_lid(self) -> dict:
        if self._gid_to_lid is None:
            self._gid_to_lid = {int(g): i for i, g in enumerate(self.gids.tolist())}
        return self._gid_to_lid

    @property
    def num_local(self) -> int:
        return self.owned_count + self.ghost_count

    @property
    def num_vertices(self) -> int:
        return self.num_local

    def adj(self, v: int) -> np.ndarray:
        off = self.row_offsets
        return self.col_indices[off[v]: off[v + 1]]

    def is_ghost(self, lid: int) -> bool:
        return lid >= self.owned_count


@dataclass
class RoundReport:
    """Per-iteration accounting for one protocol round (chroma/runtime.py:83-108)."""

    round_index: int
    conflicts: int
    recolored_per_rank: list[int]
    bytes_sent: int
    messages_sent: int
    time_color_s: float = 0.0
    time_comm_s: float = 0.0
    time_detect_s: float = 0.0

    def to_dict(self, include_timings: bool = True) -> dict:
        d = {"round": self.round_index, "conflicts": self.conflicts,
             "recolored_per_rank": list(self.recolored_per_rank), "bytes_sent": self.bytes_sent,
             "messages_sent": self.messages_sent}
        if include_timings:
            d.update(time_color_ms=self.time_color_s * 1e3, time_comm_ms=self.time_comm_s * 1e3,
                     time_detect_ms=self.time_detect_s * 1e3)
        return d


@dataclass
class RankWorld:
    """All ranks' local graphs plus the routing between them (chroma/runtime.py:111-139)."""

    num_ranks: int
    ghost_layers: int
    local_graphs: list
    partition: PartitionMap
    num_global_vertices: int
    source_stats: GraphStats
    handle: WorldHandle | None = None
    last_sent: list = field(default_factory=list)
    workers: int = 1
    total_bytes: int = 0
    total_messages: int = 0
    _send_targets: list | None = None

    @property
    def send_targets(self) -> list:
        """send_targets[r][owned lid] -> ranks holding a ghost copy (chroma/runtime.py:249-256)."""
        if self._send_targets is None:
            st: list[dict] = [dict() for _ in range(self.num_ranks)]
            for r, lg in enumerate(self.local_graphs):
                for slot in range(lg.ghost_count):
                    gid = int(lg.gids[lg.owned_count + slot])
                    o = int(self.partition.owner[gid])
                    st[o].setdefault(self.local_graphs[o].gid_to_lid[gid], []).append(r)
            self._send_targets = st
        return self._send_targets

    def map_ranks(self, fn):
        return [fn(r) for r in range(self.num_ranks)]

    def reset_exchange_state(self) -> None:
        self.last_sent = [dict() for _ in range(self.num_ranks)]
        self.total_bytes = 0
        self.total_messages = 0
        if self.handle is not None:
            _lib.check(_lib.lib().chroma_world_reset_exchange(self.handle.h))


def device_stats(wh: WorldHandle) -> GraphStats:
    """GraphStats of the source graph (chroma/graph.py:380-385) from the device build."""
    i = wh.info(wh.rank_lo)
    n, m = i["n_global"], i["m_global"]
    return GraphStats(n, m, (2.0 * m / n) if n else 0.0, i["delta_max"] if n else 0)


def build_local_graphs(g, pm: PartitionMap, ghost_layers: int = 1) -> RankWorld:
    """Split g across pm's ranks with one or two ghost layers, on the GPU."""
    if ghost_layers not in (1, 2):
        raise ValueError("ghost_layers must be 1 or 2")
    if pm.num_ranks < 1:
        raise ValueError("num_ranks must be >= 1")
    if len(pm.owner) != g.num_vertices:
        raise ValueError("partition size does not match graph")
    # one process, several GPUs: rank r on its own device (multidev.py)
    from .multidev import MultiDeviceWorld, devices_for
    devs = devices_for(pm.num_ranks)
    if devs is not None:
        return MultiDeviceWorld(g, pm, ghost_layers, devs)
    return _build_virtual(g, pm, ghost_layers)


def _build_virtual(g, pm: PartitionMap, ghost_layers: int, device: int | None = None) -> RankWorld:
    """Every rank on one device ("virtual ranks"; the halo is a device copy)."""
    # owner range / empty-rank validation (PartitionMap.validate) runs on the device
    wh = WorldHandle(g, pm, ghost_layers, 0, pm.num_ranks, device)
    lgs = [LocalGraph(wh, r, ghost_layers) for r in range(pm.num_ranks)]
    world = RankWorld(num_ranks=pm.num_ranks, ghost_layers=ghost_layers, local_graphs=lgs,
                      partition=pm, num_global_vertices=g.num_vertices, source_stats=device_stats(wh),
                      handle=wh)
    world.reset_exchange_state()
    return world


def exchange_boundary_colors(world: RankWorld, colorings: list, changed_only: bool = False):
    """Owner -> every ghost copy, changed-only against the last broadcast
    (chroma/runtime.py:271-308).  Returns (bytes_sent, messages_sent)."""
    if hasattr(world, "virtual_world"):  # MultiDeviceWorld: the virtual copy keeps the state
        b, m = exchange_boundary_colors(world.virtual_world(), colorings, changed_only)
        world.total_bytes += b
        world.total_messages += m
        return b, m
    if world.handle is None:
        raise ValueError("world was not built by paper_2107_00075_b200.runtime.build_local_graphs")
    bufs = [np.ascontiguousarray(c, dtype=np.int32) for c in colorings]
    arr = (C.c_void_p * world.num_ranks)(*[b.ctypes.data for b in bufs])
    b, m = C.c_int64(0), C.c_int64(0)
    _lib.check(_lib.lib().chroma_world_exchange(world.handle.h, arr, int(bool(changed_only)),
                                                C.byref(b), C.byref(m)), "exchange_boundary_colors")
    for c, buf in zip(colorings, bufs):
        if buf is not c:
            c[...] = buf
    world.total_bytes += int(b.value)
    world.total_messages += int(m.value)
    return int(b.value), int(m.value)


def allreduce_sum(world, per_rank_values) -> int:
    values = list(per_rank_values)
    if len(values) != world.num_ranks:
        raise ValueError("allreduce requires a contribution from every rank")
    return int(sum(values))


def snapshot_ghost_colors(lg, colors: np.ndarray) -> np.ndarray:
    return colors[lg.owned_count:].copy()


def restore_ghost_colors(lg, colors: np.ndarray, saved: np.ndarray) -> None:
    if len(saved) != lg.ghost_count:
        raise ValueError("ghost snapshot length mismatch")
    colors[lg.owned_count:] = saved
