"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED reference.

Test infrastructure only.  This script imports the reference package `chroma`
read-only from /root/reference/pkg/src (it only exists in the dev container) and
records its outputs so that the oracle (oracle/chroma_oracle.c) and the CUDA path
can be pinned against them on machines where the reference is absent.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Outputs
  tests/golden/runs.json          run_distributed RunRecords (sha256 of the gathered
                                   int32 colour array, per-round integer report fields)
  tests/golden/arrays.npz         small input graphs / partitions and full outputs of the
                                   fine-grained entry points (build_local_graphs,
                                   speculative_color*, detect_conflicts_*, exchange, verify_*)
  tests/golden/unit.json          scalar known answers (gid_rand, check_conflicts, first_fit)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("CHROMA_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from chroma import graph as G  # noqa: E402
from chroma import localcolor as L  # noqa: E402
from chroma import partition as P  # noqa: E402
from chroma import protocol as R  # noqa: E402
from chroma import runtime as RT  # noqa: E402
from chroma import verify as V  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha(a: np.ndarray, dtype="<i4") -> str:
    return hashlib.sha256(np.ascontiguousarray(a.astype(dtype)).tobytes()).hexdigest()


# ---------------------------------------------------------------- inputs not in the reference
def stencil27(L_: int):
    """27-point stencil on an L^3 lattice, id = x + L(y + L z), through the reference preprocess."""
    ids = np.arange(L_ ** 3, dtype=np.int64).reshape(L_, L_, L_)  # [z, y, x]
    pieces = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if (dz, dy, dx) <= (0, 0, 0):
                    continue
                zs = slice(max(0, -dz), L_ - max(0, dz))
                ys = slice(max(0, -dy), L_ - max(0, dy))
                xs = slice(max(0, -dx), L_ - max(0, dx))
                a = ids[zs, ys, xs]
                b = ids[(slice(zs.start + dz, zs.stop + dz), slice(ys.start + dy, ys.stop + dy),
                         slice(xs.start + dx, xs.stop + dx))]
                pieces.append(np.column_stack([a.ravel(), b.ravel()]))
    return G.preprocess(L_ ** 3, np.concatenate(pieces))


def rmat_edges(scale: int, ef: int, seed: int):
    """Graph500 R-MAT (a,b,c,d)=(.57,.19,.19,.05) with a seeded label permutation."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = ef * n
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    for _ in range(scale):
        r = rng.random(m)
        bit_s = (r >= 0.57 + 0.19).astype(np.int64)          # c or d quadrant
        bit_d = (((r >= 0.57) & (r < 0.76)) | (r >= 0.95)).astype(np.int64)  # b or d
        src = (src << 1) | bit_s
        dst = (dst << 1) | bit_d
    perm = rng.permutation(n)
    return n, np.column_stack([perm[src], perm[dst]])


def random_bipartite(rows: int, nnz_row: int, seed: int):
    rng = np.random.default_rng(seed)
    src = np.repeat(np.arange(rows, dtype=np.int64), nnz_row)
    dst = rng.integers(0, rows, size=rows * nnz_row)
    d = G.preprocess_directed(rows, np.column_stack([src, dst]))
    return G.to_bipartite(d).graph


# ---------------------------------------------------------------- helpers
arrays: dict[str, np.ndarray] = {}


def put(key: str, a) -> None:
    a = np.array(a, copy=True)  # snapshot: callers keep mutating their arrays
    if a.dtype == np.int64 and (a.size == 0 or (a.min() >= -2**31 and a.max() < 2**31)):
        a = a.astype(np.int32)
    arrays[key] = a


def put_graph(name: str, g) -> None:
    put(f"graph/{name}/row_offsets", g.row_offsets)
    put(f"graph/{name}/col_indices", g.col_indices)


def run_record(g, pm, mode, rd, det, kernel=None):
    world = RT.build_local_graphs(g, pm, R.ghost_layers_for(mode))
    cfg = R.AlgorithmConfig(mode=mode, recolor_degrees=rd, deterministic=det,
                            kernel=kernel or L.KernelChoice())
    t = time.perf_counter()
    colors, reports = R.run_distributed(world, cfg)
    dt = time.perf_counter() - t
    ncol, _ = V.color_stats(colors)
    return colors, {
        "rounds": len(reports),
        "colors": ncol,
        "sha256": sha(colors),
        "conflicts": [r.conflicts for r in reports],
        "recolored_per_rank": [list(r.recolored_per_rank) for r in reports],
        "bytes_sent": [r.bytes_sent for r in reports],
        "messages_sent": [r.messages_sent for r in reports],
        "ref_seconds": round(dt, 4),
    }


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    runs = []
    M = R.Mode

    graphs = {
        "gnp400": G.gen_random_gnp(400, 0.03, 7),
        "myciel7": G.gen_mycielskian(7),
        "hex32": G.gen_hex_mesh(32, 32, 32),
        "hex64x64": G.gen_hex_mesh(64, 64, 1),
        "st27_30": stencil27(30),
        "bip10": random_bipartite(1 << 10, 8, 3),
        "rmat10": G.preprocess(*rmat_edges(10, 16, 1)),
        "gnp200": G.gen_random_gnp(200, 0.06, 11),
        "hex6x5x4": G.gen_hex_mesh(6, 5, 4),
    }
    for name, g in graphs.items():
        put(f"graph/{name}/sha_col", np.frombuffer(bytes.fromhex(sha(g.col_indices, "<i8")), np.uint8))
        if g.num_vertices <= 5000 or name in ("bip10", "rmat10"):
            put_graph(name, g)
    gsha = {name: {"n": g.num_vertices, "nnz": int(len(g.col_indices)),
                   "sha_col_i8": sha(g.col_indices, "<i8"),
                   "sha_off_i8": sha(g.row_offsets, "<i8")} for name, g in graphs.items()}

    def add(case, g, pm, mode, Pn, rd, det, part="block", kernel=None, keep=False):
        colors, rec = run_record(g, pm, mode, rd, det, kernel)
        rec.update({"graph": case, "mode": mode.value, "P": Pn, "rd": rd, "det": det,
                    "partition": part,
                    "kernel": None if kernel is None else
                    {"kind": None if kernel.kind is None else kernel.kind.value,
                     "threshold": kernel.max_degree_threshold}})
        rid = len(runs)
        rec["id"] = rid
        if keep:
            put(f"run/{rid}/colors", colors)
        runs.append(rec)
        print(f"[{rid}] {case} {mode.value} P={Pn} rd={rd} det={det} {part}: "
              f"rounds={rec['rounds']} colors={rec['colors']} {rec['ref_seconds']}s", flush=True)

    modes = [M.D1, M.D1_2GL, M.D2, M.PD2]
    # deterministic runs on block partitions
    for case in ("gnp400", "myciel7", "hex64x64", "bip10", "rmat10", "hex32"):
        g = graphs[case]
        for mode in modes:
            for Pn in (1, 2, 4, 8):
                for rd in ((False,) if Pn == 1 else (False, True)):
                    add(case, g, P.partition_block(g, Pn), mode, Pn, rd, True,
                        keep=g.num_vertices <= 5000)
    g = graphs["st27_30"]
    for mode in (M.D1, M.D1_2GL):
        for Pn in (1, 2, 4, 8):
            for rd in ((False,) if Pn == 1 else (False, True)):
                add("st27_30", g, P.partition_block(g, Pn), mode, Pn, rd, True)
    # adversarial random partitions (non-contiguous ownership)
    g = graphs["gnp200"]
    for seed in range(4):
        for Pn in (3, 4):
            pm = P.partition_random(g, Pn, seed)
            put(f"part/gnp200/{seed}/{Pn}", pm.owner)
            for mode in modes:
                for rd in (False, True):
                    add("gnp200", g, pm, mode, Pn, rd, True, part=f"random:{seed}", keep=True)
    # Jacobi mode (deterministic=False) -- the reference's other (also deterministic) mode
    for case in ("gnp400", "myciel7", "gnp200", "bip10"):
        g = graphs[case]
        for mode in modes:
            for Pn in (1, 2, 8):
                add(case, g, P.partition_block(g, Pn), mode, Pn, True, False, keep=True)
    g = graphs["gnp400"]
    add("gnp400", g, P.partition_block(g, 8), M.D1, 8, False, False,
        kernel=L.KernelChoice(max_degree_threshold=5), keep=True)
    add("gnp400", g, P.partition_block(g, 8), M.D1, 8, False, False,
        kernel=L.KernelChoice(kind=L.Kernel.VERTEX_BASED), keep=True)
    for mode in modes:
        add("hex6x5x4", graphs["hex6x5x4"], P.partition_block(graphs["hex6x5x4"], 3), mode, 3,
            True, False, keep=True)

    # ------------------------------------------------------------ fine-grained entry points
    rng = np.random.default_rng(2024)
    fine = []
    # build_local_graphs layouts
    for case, pm_kind, Pn, gl in (("gnp200", "random:1", 4, 1), ("gnp200", "random:1", 4, 2),
                                  ("hex6x5x4", "block", 3, 2), ("hex6x5x4", "block", 3, 1),
                                  ("gnp400", "block", 4, 2), ("myciel7", "random:5", 3, 2)):
        g = graphs[case]
        pm = P.partition_block(g, Pn) if pm_kind == "block" else \
            P.partition_random(g, Pn, int(pm_kind.split(":")[1]))
        world = RT.build_local_graphs(g, pm, gl)
        key = f"lg/{case}/{pm_kind}/{Pn}/{gl}"
        put(key + "/owner", pm.owner)
        meta = []
        for r, lg in enumerate(world.local_graphs):
            for fld in ("row_offsets", "col_indices", "gids", "ghost_owner", "boundary_d1",
                        "boundary_d2"):
                put(f"{key}/{r}/{fld}", getattr(lg, fld))
            meta.append([lg.owned_count, lg.ghost_count, lg.first_layer_ghost_count,
                         lg.num_local_edges, lg.num_ghost_edges])
        put(key + "/meta", np.array(meta, dtype=np.int64))
        deg = R.compute_global_degrees(world)
        for r in range(Pn):
            put(f"{key}/{r}/degrees", deg[r])
        # speculative colouring on rank 1 with arbitrary worklists and pre-set colours
        lg = world.local_graphs[1]
        for trial in range(3):
            colors0 = rng.integers(0, 6, size=lg.num_local).astype(np.int32)
            colors0[rng.random(lg.num_local) < 0.5] = 0
            wl = rng.choice(lg.num_local, size=max(1, lg.num_local // 2), replace=False)
            put(f"{key}/spec/{trial}/colors_in", colors0)
            put(f"{key}/spec/{trial}/worklist", wl)
            for det in (True, False):
                for kind in (L.Kernel.VERTEX_BASED, L.Kernel.EDGE_BASED):
                    c = colors0.copy()
                    L.speculative_color(lg, c, wl, L.KernelChoice(kind=kind), deterministic=det)
                    put(f"{key}/spec/{trial}/d1/{int(det)}/{kind.value}", c)
                for partial in (False, True):
                    c = colors0.copy()
                    L.speculative_color_d2(lg, c, wl, partial=partial, deterministic=det)
                    put(f"{key}/spec/{trial}/d2/{int(det)}/{int(partial)}", c)
        # conflict detection on random colourings
        for trial in range(3):
            cs = [rng.integers(0, 4, size=lgr.num_local).astype(np.int32)
                  for lgr in world.local_graphs]
            for r in range(Pn):
                put(f"{key}/det/{trial}/{r}/colors_in", cs[r])
                for rd in (False, True):
                    c = cs[r].copy()
                    n1 = R.detect_conflicts_d1(world.local_graphs[r], c, deg[r], rd)
                    put(f"{key}/det/{trial}/{r}/d1/{int(rd)}", c)
                    fine.append({"key": f"{key}/det/{trial}/{r}/d1/{int(rd)}", "count": n1})
                    if gl == 2:
                        for partial in (False, True):
                            c = cs[r].copy()
                            n2 = R.detect_conflicts_d2(world.local_graphs[r], c, deg[r], partial, rd)
                            put(f"{key}/det/{trial}/{r}/d2/{int(partial)}/{int(rd)}", c)
                            fine.append({"key": f"{key}/det/{trial}/{r}/d2/{int(partial)}/{int(rd)}",
                                         "count": n2})
        # exchange sequence: full, then changed_only twice
        world.reset_exchange_state()
        cs = [rng.integers(1, 5, size=lgr.num_local).astype(np.int32) for lgr in world.local_graphs]
        for r in range(Pn):
            put(f"{key}/xchg/{r}/in", cs[r])
        res = [list(RT.exchange_boundary_colors(world, cs, changed_only=False))]
        for r in range(Pn):
            put(f"{key}/xchg/{r}/after0", cs[r])
            lgr = world.local_graphs[r]
            sel = rng.random(lgr.owned_count) < 0.2
            cs[r][: lgr.owned_count][sel] = rng.integers(1, 5, size=int(sel.sum()))
            put(f"{key}/xchg/{r}/mod1", cs[r])
        res.append(list(RT.exchange_boundary_colors(world, cs, changed_only=True)))
        for r in range(Pn):
            put(f"{key}/xchg/{r}/after1", cs[r])
        res.append(list(RT.exchange_boundary_colors(world, cs, changed_only=True)))
        fine.append({"key": f"{key}/xchg", "results": res,
                     "total": [world.total_bytes, world.total_messages]})

    # verify on random colourings
    for case in ("gnp200", "myciel7", "hex6x5x4", "bip10"):
        g = graphs[case]
        for trial in range(2):
            c = rng.integers(0, 8, size=g.num_vertices).astype(np.int32)
            put(f"verify/{case}/{trial}/colors", c)
            mask = rng.random(g.num_vertices) < 0.6
            put(f"verify/{case}/{trial}/mask", mask.astype(np.uint8))
            for label, res in (("d1", V.verify_d1(g, c)),
                               ("d2", V.verify_d2(g, c)),
                               ("pd2", V.verify_d2(g, c, partial=True)),
                               ("pd2m", V.verify_d2(g, c, partial=True, endpoint_mask=mask)),
                               ("d2m", V.verify_d2(g, c, partial=False, endpoint_mask=mask))):
                kinds = {"uncolored": 0, "d1-edge": 1, "d2-path": 2, "pd2-path": 3}
                arr = np.array([[kinds[v.kind.value], v.u, -1 if v.w is None else v.w,
                                 -1 if v.middle is None else v.middle] for v in res],
                               dtype=np.int64).reshape(-1, 4)
                put(f"verify/{case}/{trial}/{label}", arr)
            n_c, hist = V.color_stats(c)
            fine.append({"key": f"verify/{case}/{trial}/stats", "num_colors": n_c,
                         "hist": {str(k): v for k, v in hist.items()}})
        order = rng.permutation(g.num_vertices)
        put(f"serial/{case}/order", order)
        put(f"serial/{case}/natural", L.serial_greedy(g))
        put(f"serial/{case}/ordered", L.serial_greedy(g, order))

    # ------------------------------------------------------------ scalar known answers
    gids = [0, 1, 2, 3, 17, 2**31 - 1, 2**31, 2**40 + 5, 123456789, 2**62 + 3]
    unit = {"gid_rand": {str(x): format(R.gid_rand(x), "016x") for x in gids}}
    checks = []
    for _ in range(2000):
        v, u = 0, 1
        gids_ = rng.integers(0, 1 << 40, size=2)
        if gids_[0] == gids_[1]:
            continue
        deg_ = rng.integers(1, 4, size=2)
        col = int(rng.integers(0, 3))
        cu = col if rng.random() < 0.8 else int(rng.integers(0, 3))
        for rdf in (False, True):
            c = np.array([col, cu], dtype=np.int32)
            k = R.check_conflicts(v, u, c, gids_, deg_, rdf)
            checks.append([int(gids_[0]), int(gids_[1]), int(deg_[0]), int(deg_[1]), col, cu,
                           int(rdf), k, int(c[0]), int(c[1])])
    unit["check_conflicts"] = checks
    ff = []
    for _ in range(300):
        k = int(rng.integers(0, 200))
        arr = rng.integers(-2, int(rng.integers(1, 300)), size=k)
        if rng.random() < 0.3:
            arr = np.concatenate([arr, np.arange(1, int(rng.integers(60, 200)))])
        ff.append([arr.tolist(), L.first_fit_color(arr)])
    unit["first_fit"] = ff
    unit["select_kernel"] = [[dm, th, L.select_kernel(G.GraphStats(10, 10, 1.0, dm),
                                                      L.KernelChoice(max_degree_threshold=th)).kind.value]
                             for dm, th in ((6000, 6000), (6001, 6000), (5, 5), (6, 5))]

    # full-scale C1 hash (configs[0])
    t = time.perf_counter()
    c1 = G.gen_hex_mesh(1000, 1000, 1)
    c1_colors, c1_rec = run_record(c1, P.partition_block(c1, 1), M.D1, False, True)
    unit["C1"] = {"sha256": c1_rec["sha256"], "rounds": c1_rec["rounds"], "colors": c1_rec["colors"],
                  "ref_run_seconds": c1_rec["ref_seconds"], "total_seconds": time.perf_counter() - t}
    print("C1", unit["C1"], flush=True)

    with open(os.path.join(OUT, "runs.json"), "w") as fh:
        json.dump({"graphs": gsha, "runs": runs, "fine": fine}, fh, indent=0)
    with open(os.path.join(OUT, "unit.json"), "w") as fh:
        json.dump(unit, fh)
    np.savez_compressed(os.path.join(OUT, "arrays.npz"), **arrays)
    print("wrote", len(runs), "runs,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
