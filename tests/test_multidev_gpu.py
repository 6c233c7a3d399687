"""One process driving several GPUs through the unchanged API (multidev.py):
build_local_graphs(g, pm) puts rank r on cuda:r when the box has >= P GPUs, and
run_distributed returns the global colours -- bit-exact with the reference's golden
RunRecords (tests/golden/runs.json) and the full-scale oracle values (scale.json)."""
import json
import os

import numpy as np
import pytest

from paper_2107_00075_b200 import graph as G
from paper_2107_00075_b200 import localcolor as L
from paper_2107_00075_b200 import partition as PT
from paper_2107_00075_b200 import protocol as R
from paper_2107_00075_b200 import runtime as RT
from paper_2107_00075_b200.multidev import MultiDeviceWorld
from tests.common import golden_graph, golden_partition, sha

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


NGPU = _ngpu()
with open(os.path.join(os.path.dirname(__file__), "golden", "runs.json")) as _fh:
    RUNS = [r for r in json.load(_fh)["runs"] if 2 <= r["P"] <= max(NGPU, 2) and r["P"] in (2, 4, 8)]


@pytest.fixture(autouse=True)
def _multi(monkeypatch):
    if NGPU < 2:
        pytest.skip("needs at least 2 GPUs")
    monkeypatch.setenv("CHROMA_MULTI_GPU", "1")


@pytest.mark.parametrize("rec", RUNS, ids=[f"{r['id']}-{r['graph']}-{r['mode']}-P{r['P']}" for r in RUNS])
def test_golden_runs_multi_gpu(rec, golden_arrays):
    if rec["P"] > NGPU:
        pytest.skip(f"needs {rec['P']} GPUs")
    g = golden_graph(rec["graph"], golden_arrays)
    pm = golden_partition(rec, g, golden_arrays)
    mode = R.Mode(rec["mode"])
    world = RT.build_local_graphs(g, pm, R.ghost_layers_for(mode))
    assert isinstance(world, MultiDeviceWorld)
    kern = rec["kernel"]
    kc = L.KernelChoice() if kern is None else L.KernelChoice(
        kind=None if kern["kind"] is None else L.Kernel(kern["kind"]), max_degree_threshold=kern["threshold"])
    cfg = R.AlgorithmConfig(mode=mode, recolor_degrees=rec["rd"], deterministic=rec["det"], kernel=kc)
    colors, reports = R.run_distributed(world, cfg)
    assert sha(colors) == rec["sha256"]
    assert [r.conflicts for r in reports] == rec["conflicts"]
    assert [list(r.recolored_per_rank) for r in reports] == rec["recolored_per_rank"]
    assert [r.bytes_sent for r in reports] == rec["bytes_sent"]
    assert [r.messages_sent for r in reports] == rec["messages_sent"]


@pytest.mark.parametrize("P", [2, 4])
def test_c2_full_scale_multi_gpu(P):
    if P > NGPU:
        pytest.skip(f"needs {P} GPUs")
    with open(os.path.join(os.path.dirname(__file__), "golden", "scale.json")) as fh:
        ref = json.load(fh)["c2_128"][f"d1-2gl_p{P}"]
    g = G.gen_stencil27(128, device="cuda")
    world = RT.build_local_graphs(g, PT.partition_block(g, P), 2)
    colors, reports = R.run_distributed(world, R.AlgorithmConfig(mode=R.Mode.D1_2GL, deterministic=True))
    assert sha(colors) == ref["sha256"]
    assert [r.conflicts for r in reports] == ref["conflicts"]


def test_free_mode_multi_gpu_proper():
    P = 2
    g = G.gen_rmat(16, 16, 1)
    world = RT.build_local_graphs(g, PT.partition_block(g, P), 1)
    colors, reports = R.run_distributed(world, R.AlgorithmConfig(mode=R.Mode.D1, algorithm="free"))
    import oracle
    assert colors.min() >= 1
    assert len(oracle.verify(g.row_offsets, g.col_indices, colors, "d1")) == 0
