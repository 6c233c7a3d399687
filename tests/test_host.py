"""CPU: host-side logic, the C ABI surface, and the no-fallback rule."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2107_00075_b200 import _lib
from paper_2107_00075_b200 import graph as G
from paper_2107_00075_b200 import localcolor as L
from paper_2107_00075_b200 import partition as PT
from paper_2107_00075_b200 import protocol as R
from paper_2107_00075_b200 import runtime as RT
from paper_2107_00075_b200 import verify as V

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_exports_every_declared_symbol():
    """libchroma_b200.so loads and exports every entry point of include/chroma_b200.h."""
    hdr = open(os.path.join(ROOT, "include", "chroma_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = sorted(set(re.findall(r"\b(chroma_[a-z0-9_]+)\s*\(", hdr)))
    assert len(declared) >= 20
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == set(declared)
    assert _lib.lib().chroma_version().startswith(b"chroma_b200")


def test_gid_rand_and_check_conflicts(golden_unit):
    for gid, h in golden_unit["gid_rand"].items():
        assert format(R.gid_rand(int(gid)), "016x") == h
    arr = np.array([int(x) for x in golden_unit["gid_rand"]], dtype=np.int64)
    assert [format(int(x), "016x") for x in R.gid_rand_array(arr)] == list(golden_unit["gid_rand"].values())
    for gv, gu, dv, du, cv, cu, rd, k, ov, ou in golden_unit["check_conflicts"]:
        c = np.array([cv, cu], np.int32)
        assert R.check_conflicts(0, 1, c, np.array([gv, gu]), np.array([dv, du]), bool(rd)) == k
        assert c.tolist() == [ov, ou]
    with pytest.raises(ValueError):
        R.check_conflicts(0, 1, np.array([2, 2], np.int32), np.array([5, 5]), np.array([1, 1]), False)


def test_first_fit_and_mask(golden_unit):
    for arr, want in golden_unit["first_fit"]:
        assert L.first_fit_color(arr) == want
    assert L.first_fit_color([]) == 1
    assert L.first_fit_color([1, 2]) == 3 and L.first_fit_color([0, 0, 2]) == 1
    m = L.ForbiddenMask()
    for c in range(1, 65):
        m.forbid(c)
    assert m.saturated and m.smallest_allowed() is None
    m.advance()
    assert m.smallest_allowed() == 65
    for dm, th, kind in golden_unit["select_kernel"]:
        assert L.select_kernel(G.GraphStats(10, 10, 1.0, dm), L.KernelChoice(max_degree_threshold=th)).kind.value == kind
    with pytest.raises(ValueError):
        L.KernelChoice(max_degree_threshold=0)


def test_graph_model():
    g = G.gen_hex_mesh(3, 3, 3)
    assert g.num_edges == 54
    g.validate()
    c5 = G.gen_mycielskian(3)
    assert c5.num_vertices == 5 and c5.num_edges == 5
    st = G.stats(G.preprocess(10, np.column_stack([np.zeros(9, np.int64), np.arange(1, 10)])))
    assert st.delta_max == 9 and abs(st.delta_avg - 1.8) < 1e-12
    assert G.stats(G.preprocess(0, np.empty((0, 2)))).num_vertices == 0
    bad = G.Graph(3, np.array([0, 1, 1, 1]), np.array([1]))
    with pytest.raises(ValueError):
        bad.validate()
    with pytest.raises(ValueError):
        G.gen_hex_mesh(0, 1, 1)
    with pytest.raises(ValueError):
        G.gen_mycielskian(13)
    with pytest.raises(ValueError):
        G.gen_random_gnp(5, 1.5, 0)
    d = G.preprocess_directed(4, np.array([[0, 1], [0, 1], [2, 2], [3, 0]]))
    assert d.num_edges == 2
    b = G.to_bipartite(d)
    assert b.graph.num_vertices == 8 and b.s_mask().sum() == 4
    b.graph.validate()
    s27 = G.gen_stencil27(5)
    s27.validate()
    assert s27.num_edges == 3 * 4 * 25 + 6 * 16 * 5 + 4 * 64


def test_file_formats(tmp_path):
    g = G.gen_random_gnp(60, 0.1, 3)
    p = str(tmp_path / "g.chrg")
    G.save_csr_cache(g, p)
    h = G.load_graph(p)
    assert np.array_equal(h.col_indices, g.col_indices) and np.array_equal(h.row_offsets, g.row_offsets)
    el = tmp_path / "e.txt"
    el.write_text("# comment\n10 20\n20 30\n\n30 10\n10 10\n")
    e = G.load_graph(str(el))
    assert e.num_vertices == 3 and e.num_edges == 3 and e.source_ids.tolist() == [10, 20, 30]
    mm = tmp_path / "m.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n% c\n3 3 2\n1 2\n3 1\n")
    m = G.load_graph(str(mm))
    assert m.num_vertices == 3 and m.num_edges == 2
    bad = tmp_path / "b.chrg"
    bad.write_bytes(b"CHRG" + b"\x02\x00\x00\x00")
    with pytest.raises(ValueError):
        G.load_csr_cache(str(bad))


def test_partitions(golden_arrays):
    g = G.gen_random_gnp(200, 0.06, 11)
    for seed in range(4):
        for P in (3, 4):
            assert np.array_equal(PT.partition_random(g, P, seed).owner, golden_arrays[f"part/gnp200/{seed}/{P}"])
    pm = PT.partition_block(G.gen_hex_mesh(16, 16, 16), 4)
    assert pm.counts().tolist() == [1024] * 4
    assert PT.block_bounds(4096, 4, 1) == (1024, 2048)
    pm3 = PT.partition_block(G.gen_hex_mesh(10, 1, 1), 3)
    assert pm3.owner.tolist() == [0, 0, 0, 1, 1, 1, 2, 2, 2, 2]
    e = PT.partition_edge_balanced(g, 4, 0)
    e.validate()
    assert PT.edge_cut(g, pm3 if False else e) >= 0 and PT.endpoint_imbalance(g, e) >= 1.0
    with pytest.raises(ValueError):
        PT.PartitionMap(np.array([0, 0, 0], np.int32), 2).validate()
    with pytest.raises(ValueError):
        PT.partition_block(g, 0)


def test_config_and_reports():
    with pytest.raises(ValueError):
        R.AlgorithmConfig(max_rounds=0)
    with pytest.raises(ValueError):
        R.AlgorithmConfig(algorithm="bogus")
    assert R.ghost_layers_for(R.Mode.D1) == 1 and R.ghost_layers_for(R.Mode.PD2) == 2
    assert R.AlgorithmConfig(deterministic=True).algo_code() == _lib.ALGO_GS
    assert R.AlgorithmConfig().algo_code() == _lib.ALGO_JACOBI
    assert R.AlgorithmConfig(algorithm="free").algo_code() == _lib.ALGO_FREE
    rr = RT.RoundReport(0, 3, [1, 2], 24, 2, 0.001, 0.002, 0.003)
    d = rr.to_dict()
    assert d["time_comm_ms"] == pytest.approx(2.0) and rr.to_dict(False).keys() == {
        "round", "conflicts", "recolored_per_rank", "bytes_sent", "messages_sent"}


def test_chromatic_oracle():
    assert V.chromatic_oracle(G.gen_mycielskian(3)) == 3
    assert V.chromatic_oracle(G.gen_mycielskian(4)) == 4
    k4 = G.preprocess(4, np.array([[i, j] for i in range(4) for j in range(i + 1, 4)]))
    assert V.chromatic_oracle(k4) == 4
    with pytest.raises(V.GraphTooLarge):
        V.chromatic_oracle(G.gen_hex_mesh(4, 4, 1))


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a CUDA device the colouring path fails loudly instead of computing on the CPU."""
    g = G.gen_random_gnp(30, 0.2, 1)
    with pytest.raises(RuntimeError):
        L.serial_greedy(g)
    with pytest.raises(RuntimeError):
        RT.build_local_graphs(g, PT.partition_block(g, 2), 1)
    with pytest.raises(RuntimeError):
        V.verify_d1(g, np.ones(30, np.int32))


def test_chroma_import_path_is_the_b200_backend():
    """`from chroma import protocol` (the reference's module paths) resolves to this
    package (drop-in: callers' imports do not change)."""
    import importlib
    import paper_2107_00075_b200 as pkg
    for m in ("graph", "partition", "runtime", "localcolor", "protocol", "verify"):
        shim = importlib.import_module(f"chroma.{m}")
        impl = getattr(pkg, m) if hasattr(pkg, m) else importlib.import_module(f"paper_2107_00075_b200.{m}")
        for name in getattr(impl, "__all__", []):
            assert getattr(shim, name) is getattr(impl, name), (m, name)
