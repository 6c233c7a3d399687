"""GPU parity: the CUDA path (through the reference-facing API -> C ABI) against the
reference's golden outputs (tests/golden, produced by oracle/gen_golden.py from the
unmodified reference) and against the C oracle on seeded random inputs.
Integer path: everything is compared bit-exactly."""
import numpy as np
import pytest

import oracle
from paper_2107_00075_b200 import graph as G
from paper_2107_00075_b200 import localcolor as L
from paper_2107_00075_b200 import partition as PT
from paper_2107_00075_b200 import protocol as R
from paper_2107_00075_b200 import runtime as RT
from paper_2107_00075_b200 import verify as V
from tests.common import golden_graph, golden_partition, sha

pytestmark = pytest.mark.gpu

_GRAPHS = {}


def _graph(name, arrays):
    if name not in _GRAPHS:
        _GRAPHS[name] = golden_graph(name, arrays)
    return _GRAPHS[name]


def _load_runs():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "runs.json")) as fh:
        return json.load(fh)["runs"]


RUNS = _load_runs()


@pytest.mark.parametrize("rec", RUNS, ids=[f"{r['id']}-{r['graph']}-{r['mode']}-P{r['P']}-rd{int(r['rd'])}-"
                                          f"{'gs' if r['det'] else 'jac'}" for r in RUNS])
def test_run_distributed_matches_reference(rec, golden_arrays):
    g = _graph(rec["graph"], golden_arrays)
    pm = golden_partition(rec, g, golden_arrays)
    mode = R.Mode(rec["mode"])
    world = RT.build_local_graphs(g, pm, R.ghost_layers_for(mode))
    kern = rec["kernel"]
    kc = L.KernelChoice() if kern is None else L.KernelChoice(
        kind=None if kern["kind"] is None else L.Kernel(kern["kind"]), max_degree_threshold=kern["threshold"])
    cfg = R.AlgorithmConfig(mode=mode, recolor_degrees=rec["rd"], deterministic=rec["det"], kernel=kc)
    colors, reports = R.run_distributed(world, cfg)
    assert sha(colors) == rec["sha256"]
    assert len(reports) == rec["rounds"]
    assert [r.conflicts for r in reports] == rec["conflicts"]
    assert [list(r.recolored_per_rank) for r in reports] == rec["recolored_per_rank"]
    assert [r.bytes_sent for r in reports] == rec["bytes_sent"]
    assert [r.messages_sent for r in reports] == rec["messages_sent"]
    if mode in (R.Mode.D1, R.Mode.D1_2GL):
        assert V.count_violations(g, colors, "d1") == 0
    elif mode is R.Mode.D2:
        assert V.count_violations(g, colors, "d2") == 0
    else:
        assert V.count_violations(g, colors, "pd2") == 0


def test_c1_full_scale_hash(golden_unit):
    """configs[0]: 1000x1000 grid, one partition, deterministic D1 == reference sha256."""
    g = G.gen_hex_mesh(1000, 1000, 1)
    world = RT.build_local_graphs(g, PT.partition_block(g, 1), 1)
    colors, reports = R.run_distributed(world, R.AlgorithmConfig(mode=R.Mode.D1, deterministic=True))
    assert sha(colors) == golden_unit["C1"]["sha256"]
    assert len(reports) == 1
    assert V.color_stats(colors)[0] == 2
    assert V.verify_d1(g, colors) == []


def _lg_cases(arrays):
    keys = sorted({k.rsplit("/", 1)[0] for k in arrays.files if k.startswith("lg/") and k.endswith("/meta")})
    return keys


def _world_for(key, arrays):
    _, case, pm_kind, Pn, gl = key.split("/")
    g = _graph(case, arrays)
    pm = PT.PartitionMap(arrays[key + "/owner"].astype(np.int32), int(Pn))
    return g, pm, RT.build_local_graphs(g, pm, int(gl))


def test_build_local_graphs_layout(golden_arrays):
    for key in _lg_cases(golden_arrays):
        g, pm, world = _world_for(key, golden_arrays)
        meta = golden_arrays[key + "/meta"]
        for r, lg in enumerate(world.local_graphs):
            assert [lg.owned_count, lg.ghost_count, lg.first_layer_ghost_count, lg.num_local_edges,
                    lg.num_ghost_edges] == meta[r].tolist(), key
            for fld in ("row_offsets", "col_indices", "gids", "ghost_owner", "boundary_d1", "boundary_d2"):
                assert np.array_equal(getattr(lg, fld), golden_arrays[f"{key}/{r}/{fld}"]), (key, r, fld)
        deg = R.compute_global_degrees(world)
        for r in range(pm.num_ranks):
            assert np.array_equal(deg[r], golden_arrays[f"{key}/{r}/degrees"]), (key, r)


def test_speculative_color_fine_grained(golden_arrays):
    for key in _lg_cases(golden_arrays):
        g, pm, world = _world_for(key, golden_arrays)
        lg = world.local_graphs[1]
        for trial in range(3):
            base = f"{key}/spec/{trial}"
            c0 = golden_arrays[base + "/colors_in"]
            wl = golden_arrays[base + "/worklist"].astype(np.int64)
            for det in (True, False):
                for kind in (L.Kernel.VERTEX_BASED, L.Kernel.EDGE_BASED):
                    c = c0.copy()
                    L.speculative_color(lg, c, wl, L.KernelChoice(kind=kind), deterministic=det)
                    assert np.array_equal(c, golden_arrays[f"{base}/d1/{int(det)}/{kind.value}"]), (base, det, kind)
                for partial in (False, True):
                    c = c0.copy()
                    L.speculative_color_d2(lg, c, wl, partial=partial, deterministic=det)
                    assert np.array_equal(c, golden_arrays[f"{base}/d2/{int(det)}/{int(partial)}"]), \
                        (base, det, partial)
            # the same through a plain (non-world) CSR object
            plain = G.Graph(lg.num_local, lg.row_offsets.copy(), lg.col_indices.copy())
            c = c0.copy()
            L.speculative_color(plain, c, wl, deterministic=True)
            assert np.array_equal(c, golden_arrays[f"{base}/d1/1/vb"])


def test_detect_conflicts_fine_grained(golden_runs, golden_arrays):
    counts = {f["key"]: f["count"] for f in golden_runs["fine"] if "count" in f}
    for key in _lg_cases(golden_arrays):
        g, pm, world = _world_for(key, golden_arrays)
        gl = int(key.split("/")[-1])
        deg = R.compute_global_degrees(world)
        for trial in range(3):
            for r in range(pm.num_ranks):
                base = f"{key}/det/{trial}/{r}"
                cin = golden_arrays[base + "/colors_in"]
                for rd in (False, True):
                    c = cin.copy()
                    n1 = R.detect_conflicts_d1(world.local_graphs[r], c, deg[r], rd)
                    assert n1 == counts[f"{base}/d1/{int(rd)}"]
                    assert np.array_equal(c, golden_arrays[f"{base}/d1/{int(rd)}"])
                    if gl == 2:
                        for partial in (False, True):
                            c = cin.copy()
                            n2 = R.detect_conflicts_d2(world.local_graphs[r], c, deg[r], partial, rd)
                            k2 = f"{base}/d2/{int(partial)}/{int(rd)}"
                            assert n2 == counts[k2], k2
                            assert np.array_equal(c, golden_arrays[k2]), k2


def test_exchange_fine_grained(golden_runs, golden_arrays):
    res = {f["key"]: f for f in golden_runs["fine"] if "results" in f}
    for key in _lg_cases(golden_arrays):
        g, pm, world = _world_for(key, golden_arrays)
        world.reset_exchange_state()
        cs = [golden_arrays[f"{key}/xchg/{r}/in"].copy() for r in range(pm.num_ranks)]
        out = [list(RT.exchange_boundary_colors(world, cs, changed_only=False))]
        for r in range(pm.num_ranks):
            assert np.array_equal(cs[r], golden_arrays[f"{key}/xchg/{r}/after0"])
            cs[r] = golden_arrays[f"{key}/xchg/{r}/mod1"].copy()
        out.append(list(RT.exchange_boundary_colors(world, cs, changed_only=True)))
        for r in range(pm.num_ranks):
            assert np.array_equal(cs[r], golden_arrays[f"{key}/xchg/{r}/after1"])
        out.append(list(RT.exchange_boundary_colors(world, cs, changed_only=True)))
        assert out == res[f"{key}/xchg"]["results"]
        assert [world.total_bytes, world.total_messages] == res[f"{key}/xchg"]["total"]


def test_verify_and_stats(golden_runs, golden_arrays):
    stats = {f["key"]: f for f in golden_runs["fine"] if "num_colors" in f}
    kinds = {V.ViolationKind.UNCOLORED: 0, V.ViolationKind.D1_EDGE: 1, V.ViolationKind.D2_PATH: 2,
             V.ViolationKind.PD2_PATH: 3}
    for case in ("gnp200", "myciel7", "hex6x5x4", "bip10"):
        g = _graph(case, golden_arrays)
        for trial in range(2):
            base = f"verify/{case}/{trial}"
            c = golden_arrays[base + "/colors"]
            mask = golden_arrays[base + "/mask"].astype(bool)
            got = {"d1": V.verify_d1(g, c), "d2": V.verify_d2(g, c), "pd2": V.verify_d2(g, c, partial=True),
                   "pd2m": V.verify_d2(g, c, partial=True, endpoint_mask=mask),
                   "d2m": V.verify_d2(g, c, partial=False, endpoint_mask=mask)}
            for label, viol in got.items():
                arr = np.array([[kinds[v.kind], v.u, -1 if v.w is None else v.w,
                                 -1 if v.middle is None else v.middle] for v in viol], dtype=np.int64).reshape(-1, 4)
                assert np.array_equal(arr, golden_arrays[f"{base}/{label}"].astype(np.int64)), (base, label)
            # the count-only checker (edge-tiled kernel) agrees with the golden listing
            assert V.count_violations(g, c, "d1") == len(got["d1"]), base
            n_c, hist = V.color_stats(c)
            assert n_c == stats[base + "/stats"]["num_colors"]
            assert {str(k): v for k, v in hist.items()} == stats[base + "/stats"]["hist"]
        assert np.array_equal(L.serial_greedy(g), golden_arrays[f"serial/{case}/natural"])
        order = golden_arrays[f"serial/{case}/order"].astype(np.int64)
        assert np.array_equal(L.serial_greedy(g, order), golden_arrays[f"serial/{case}/ordered"])


@pytest.mark.parametrize("case", ["rmat", "star", "isolated", "empty"])
def test_count_violations_matches_listing(case):
    """count_violations (edge tiles of 4096 entries, 16-bit colour copy) against the
    listing path: skewed rows, tiles spanning thousands of one-entry rows, isolated
    vertices, colours above 0xFFFE (saturated in the copy)."""
    rng = np.random.default_rng(5)
    if case == "rmat":
        g = G.gen_rmat(14, 16, 3)
    elif case == "star":  # vertex 0 joined to 1..6000: tiles over 6000 one-entry rows
        n = 9000
        g = G.preprocess(n, np.stack([np.zeros(6000, np.int64), np.arange(1, 6001)], 1))
    elif case == "isolated":
        g = G.preprocess(50000, rng.integers(0, 50000, size=(3000, 2)))
    else:
        g = G.Graph(10, np.zeros(11, np.int64), np.zeros(0, np.int64))
    for palette in (3, 7, 1 << 17):
        c = rng.integers(0, palette, size=g.num_vertices).astype(np.int32)
        if palette > 0xFFFF and g.num_vertices > 4:  # equal and unequal colours above 0xFFFE
            c[:4] = [0xFFFF, 0x1FFFF, 0xFFFF, 0x10000]
        assert V.count_violations(g, c, "d1") == len(V.verify_d1(g, c)), (case, palette)


# ------------------------------------------------------------------ seeded random vs the C oracle
def _random_graph(kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "gnp":
        return G.gen_random_gnp(int(rng.integers(50, 600)), float(rng.uniform(0.005, 0.08)), seed)
    if kind == "rmat":
        return G.gen_rmat(int(rng.integers(8, 12)), 8, seed)
    if kind == "bip":
        return G.gen_random_bipartite(int(rng.integers(64, 700)), int(rng.integers(2, 12)), seed).graph
    if kind == "hex":
        return G.gen_hex_mesh(*(int(x) for x in rng.integers(2, 14, size=3)))
    return G.gen_stencil27(int(rng.integers(4, 12)))


@pytest.mark.parametrize("seed", range(24))
def test_random_worlds_vs_oracle(seed):
    kind = ["gnp", "rmat", "bip", "hex", "st27"][seed % 5]
    g = _random_graph(kind, seed)
    rng = np.random.default_rng(1000 + seed)
    P = int(rng.choice([1, 2, 3, 4, 8]))
    pm = PT.partition_random(g, P, seed) if seed % 3 == 0 else PT.partition_block(g, P)
    for mode in ("d1", "d1-2gl", "d2", "pd2"):
        for det in (True, False):
            if not det and kind in ("hex", "st27") and g.num_vertices > 600:
                continue  # Jacobi is O(n * depth) on meshes
            rd = bool(rng.integers(0, 2))
            gl = R.ghost_layers_for(R.Mode(mode))
            world = RT.build_local_graphs(g, pm, gl)
            colors, reports = R.run_distributed(world, R.AlgorithmConfig(mode=R.Mode(mode), recolor_degrees=rd,
                                                                        deterministic=det))
            ow = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl)
            ref, ref_rep = ow.run(mode, rd, det)
            assert np.array_equal(colors, ref), (kind, mode, P, det, rd)
            assert [r.conflicts for r in reports] == [r["conflicts"] for r in ref_rep]
            assert [r.bytes_sent for r in reports] == [r["bytes_sent"] for r in ref_rep]
            assert [r.messages_sent for r in reports] == [r["messages_sent"] for r in ref_rep]


def test_many_colors_slow_path():
    """Colours beyond the 256-colour fast window (K300, star D2, dense gnp)."""
    n = 300
    iu, iv = np.triu_indices(n, 1)
    k = G.preprocess(n, np.column_stack([iu, iv]))
    c = L.serial_greedy(k)
    assert np.array_equal(c, np.arange(1, n + 1, dtype=np.int32))
    star = G.preprocess(401, np.column_stack([np.zeros(400, np.int64), np.arange(1, 401)]))
    for g in (k, star, G.gen_random_gnp(700, 0.6, 5)):
        for dist, partial in ((1, False), (2, False), (2, True)):
            for det in (True, False):
                cc = np.zeros(g.num_vertices, np.int32)
                wl = np.arange(g.num_vertices)
                fn = (lambda: L.speculative_color(g, cc, wl, deterministic=det)) if dist == 1 else \
                    (lambda: L.speculative_color_d2(g, cc, wl, partial=partial, deterministic=det))
                fn()
                ref = oracle.speculative_color(g.row_offsets, g.col_indices, np.zeros(g.num_vertices, np.int32),
                                               wl, dist, partial, det)
                assert np.array_equal(cc, ref), (g.num_vertices, dist, partial, det)


def test_gs_large_meshes_vs_oracle():
    """Size-independent check at larger sizes: GS D1 over a 27-pt 48^3 stencil and an
    R-MAT s14 equals the oracle's serial_greedy; D2 on a 7-pt 40^3 mesh equals the oracle."""
    for g in (G.gen_stencil27(48), G.gen_rmat(14, 16, 1)):
        c = L.serial_greedy(g)
        assert np.array_equal(c, oracle.serial_greedy(g.row_offsets, g.col_indices))
        assert V.count_violations(g, c, "d1") == 0
    g = G.gen_hex_mesh(40, 40, 40)
    cc = np.zeros(g.num_vertices, np.int32)
    L.speculative_color_d2(g, cc, np.arange(g.num_vertices), deterministic=True)
    ref = oracle.speculative_color(g.row_offsets, g.col_indices, np.zeros(g.num_vertices, np.int32),
                                   np.arange(g.num_vertices), 2, False, True)
    assert np.array_equal(cc, ref)
    assert V.count_violations(g, cc, "d2") == 0


def test_errors_match_reference():
    g = G.gen_random_gnp(50, 0.1, 1)
    with pytest.raises(ValueError):
        RT.build_local_graphs(g, PT.partition_block(g, 2), 3)
    w = RT.build_local_graphs(g, PT.partition_block(g, 2), 1)
    with pytest.raises(ValueError):
        R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode.D2))
    with pytest.raises(ValueError):
        R.detect_conflicts_d2(w.local_graphs[0], np.zeros(w.local_graphs[0].num_local, np.int32),
                              np.zeros(w.local_graphs[0].num_local, np.int64), False, False)
    with pytest.raises(ValueError):
        L.serial_greedy(g, np.zeros(50, np.int64))
    g = G.gen_random_gnp(400, 0.03, 7)
    w2 = RT.build_local_graphs(g, PT.partition_block(g, 8), 1)
    with pytest.raises(R.NonConvergenceError) as ei:
        R.run_distributed(w2, R.AlgorithmConfig(mode=R.Mode.D1, deterministic=True, max_rounds=1))
    assert len(ei.value.reports) == 2


@pytest.mark.parametrize("name,mode,P", [("rmat17", "d1", 8), ("st27_64", "d1-2gl", 8), ("st27_64", "d1-2gl", 1),
                                         ("grid400", "d1", 4), ("st27_128", "d1-2gl", 1), ("st27_128", "d1-2gl", 8)])
def test_run_distributed_at_scale_vs_oracle(name, mode, P):
    """Whole protocol at sizes that exercise the round-0 schedules (DAG levels, rank
    interleave) and the grid-wide event resolution (> 32k detection events): colours
    and every per-round report field equal the oracle's."""
    g = {"rmat17": lambda: G.gen_rmat(17, 16, 1), "st27_64": lambda: G.gen_stencil27(64),
         "grid400": lambda: G.gen_hex_mesh(400, 400, 1),
         "st27_128": lambda: G.gen_stencil27(128, device="cuda")}[name]()  # C2: DAG-level schedule
    pm = PT.partition_block(g, P)
    gl = R.ghost_layers_for(R.Mode(mode))
    w = RT.build_local_graphs(g, pm, gl)
    colors, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode(mode), deterministic=True))
    ref, ref_reps = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl).run(mode, False, True)
    assert np.array_equal(colors, ref)
    assert [r.conflicts for r in reps] == [x["conflicts"] for x in ref_reps]
    assert [r.bytes_sent for r in reps] == [x["bytes_sent"] for x in ref_reps]
    assert [list(r.recolored_per_rank) for r in reps] == [x["recolored_per_rank"] for x in ref_reps]


def _band_graph(n, p_chain, extra, span, seed):
    """Bounded-degree graph with irregular runs: v ~ v-1 with probability p_chain,
    plus `extra` random edges per vertex to v-k, k in [2, span]."""
    rng = np.random.default_rng(seed)
    v = np.arange(1, n)
    keep = rng.random(n - 1) < p_chain
    a = [v[keep]]
    b = [v[keep] - 1]
    for _ in range(extra):
        x = rng.integers(span, n, size=n // 2)
        a.append(x)
        b.append(x - rng.integers(2, span + 1, size=x.size))
    return G.preprocess(n, np.stack([np.concatenate(a), np.concatenate(b)], 1))


@pytest.mark.parametrize("kind,P", [("band", 1), ("band", 4), ("band_long", 1), ("st27_60", 8), ("st27_60", 1),
                                    ("grid1000x300", 1), ("hex40", 8)])
def test_cluster_runs_vs_oracle(kind, P):
    """Round 0 on the cluster kernel with runs of adjacent consecutive ids on one level
    (map-composition prefix scan; gs_levels.cu chain mode): irregular runs, runs cut at
    item and 1024-id block boundaries, multi-round protocols (odd slabs); colours and
    reports equal the oracle's."""
    g = {"band": lambda: _band_graph(300_000, 0.85, 2, 3000, 5),
         "band_long": lambda: _band_graph(400_000, 0.98, 1, 200_000, 6),
         "st27_60": lambda: G.gen_stencil27(60),
         "grid1000x300": lambda: G.gen_hex_mesh(1000, 300, 1),
         "hex40": lambda: G.gen_hex_mesh(40, 40, 40)}[kind]()
    assert int(np.diff(g.row_offsets).max()) <= 32
    pm = PT.partition_block(g, P)
    mode = "d1-2gl" if P > 1 else "d1"
    gl = R.ghost_layers_for(R.Mode(mode))
    w = RT.build_local_graphs(g, pm, gl)
    colors, reps = R.run_distributed(w, R.AlgorithmConfig(mode=R.Mode(mode), deterministic=True))
    ref, ref_reps = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, gl).run(mode, False, True)
    assert np.array_equal(colors, ref)
    assert [r.conflicts for r in reps] == [x["conflicts"] for x in ref_reps]
    assert [list(r.recolored_per_rank) for r in reps] == [x["recolored_per_rank"] for x in ref_reps]
    if P == 1:
        assert np.array_equal(colors, L.serial_greedy(g))


@pytest.mark.parametrize("P", [1, 4])
@pytest.mark.parametrize("kind", ["vb", "eb"])
def test_jacobi_vertex_and_edge_based_kernels_on_skewed_graph(P, kind):
    """KernelChoice is honoured: EDGE_BASED runs the edge-parallel Jacobi kernels
    (chroma/localcolor.py:181-195), VERTEX_BASED the warp-per-vertex ones; both give
    the reference's Jacobi colours exactly (F3), here on R-MAT s16 (hub rows)."""
    g = G.gen_rmat(16, 16, 1)
    pm = PT.partition_block(g, P)
    w = RT.build_local_graphs(g, pm, 1)
    cfg = R.AlgorithmConfig(mode=R.Mode.D1, kernel=L.KernelChoice(kind=L.Kernel(kind)))
    colors, reports = R.run_distributed(w, cfg)
    ref, ref_reports = oracle.World(g.row_offsets, g.col_indices, pm.owner, P, 1).run("d1", False, False)
    assert np.array_equal(colors, ref)
    assert [r.conflicts for r in reports] == [r["conflicts"] for r in ref_reports]


def test_select_kernel_picks_edge_based_above_threshold():
    """Auto choice (chroma/localcolor.py:55-61): EB iff delta_max > threshold; the result
    is unchanged either way."""
    g = G.gen_rmat(14, 16, 1)
    pm = PT.partition_block(g, 2)
    out = []
    for thr in (5, 10 ** 9):
        w = RT.build_local_graphs(g, pm, 1)
        assert L.select_kernel(w.source_stats, L.KernelChoice(max_degree_threshold=thr)).kind is \
            (L.Kernel.EDGE_BASED if thr == 5 else L.Kernel.VERTEX_BASED)
        out.append(R.run_distributed(w, R.AlgorithmConfig(kernel=L.KernelChoice(max_degree_threshold=thr)))[0])
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("gl", [1, 2])
@pytest.mark.parametrize("part", ["block", "random", "strided"])
def test_single_rank_world_matches_full_build(gl, part):
    """A world holding one rank (the one-process-per-GPU form; windowed column upload
    for contiguous ownership) has exactly the local graph the all-ranks build gives
    that rank -- block, random and strided ownership, ranks with and without ghosts."""
    g = G.gen_rmat(12, 8, 5)
    P = 4
    if part == "block":
        pm = PT.partition_block(g, P)
    elif part == "random":
        pm = PT.partition_random(g, P, 3)
    else:
        pm = PT.PartitionMap((np.arange(g.num_vertices) % P).astype(np.int32), P)
    full = RT.build_local_graphs(g, pm, gl)
    for r in range(P):
        wh = RT.WorldHandle(g, pm, gl, r, r + 1)
        lg = RT.LocalGraph(wh, r, gl)
        ref = full.local_graphs[r]
        for name in ("row_offsets", "col_indices", "gids", "ghost_owner", "boundary_d1", "boundary_d2"):
            assert np.array_equal(getattr(lg, name), getattr(ref, name)), (part, gl, r, name)
        assert (lg.owned_count, lg.ghost_count, lg.num_local_edges, lg.num_ghost_edges) == \
            (ref.owned_count, ref.ghost_count, ref.num_local_edges, ref.num_ghost_edges)


def test_world_create_rejects_out_of_range_columns():
    g = G.gen_hex_mesh(8, 8, 1)
    bad = G.Graph(g.num_vertices, g.row_offsets.copy(), g.col_indices.copy())
    bad.col_indices[5] = g.num_vertices + 7
    for P, lo, hi in ((1, 0, 1), (2, 0, 1)):
        with pytest.raises(ValueError):
            RT.WorldHandle(bad, PT.partition_block(bad, P), 1, lo, hi)
