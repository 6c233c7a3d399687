"""CLI on the GPU: colour, verify and bench end to end."""
import json
import os

import numpy as np
import pytest

from paper_2107_00075_b200 import cli

pytestmark = pytest.mark.gpu


def test_color_mesh_proper(tmp_path, capsys):
    out = tmp_path / "r.json"
    rc = cli.main(["color", "--gen", "mesh:16,16,16", "--mode", "d1", "--ranks", "4", "--deterministic",
                   "--out", str(out)])
    line = capsys.readouterr().out.strip().splitlines()[-1]
    assert rc == 0 and "proper=true" in line and "ranks=4" in line
    rec = json.loads(out.read_text())
    assert rec["total_colors"] <= 7 and rec["verification"] == "proper"  # delta_max + 1
    assert json.loads(json.dumps(rec)) == rec


def test_color_myciel_lower_bound(capsys):
    assert cli.main(["color", "--gen", "myciel:5", "--mode", "d1", "--ranks", "1", "--deterministic"]) == 0
    line = capsys.readouterr().out.strip().splitlines()[-1]
    assert int(line.split("colors=")[1].split()[0]) >= 5


def test_color_d2_and_verify_roundtrip(tmp_path, capsys):
    cfile = tmp_path / "c.txt"
    assert cli.main(["color", "--gen", "gnp:100,0.1,7", "--mode", "d2", "--ranks", "2",
                     "--colors-out", str(cfile)]) == 0
    gfile = tmp_path / "g.chrg"
    from paper_2107_00075_b200 import graph as G
    g = G.gen_random_gnp(100, 0.1, 7)
    G.save_csr_cache(g, str(gfile))  # the CHRG v1 cache keeps n (an edge list would infer it)
    src = np.repeat(np.arange(g.num_vertices), np.diff(g.row_offsets))
    keep = src < g.col_indices
    assert cli.main(["verify", "--graph", str(gfile), "--colors", str(cfile), "--mode", "d2"]) == 0
    bad = np.loadtxt(cfile, dtype=np.int64)
    u, w = int(src[keep][0]), int(g.col_indices[keep][0])
    bad[w] = bad[u]
    np.savetxt(cfile, bad, fmt="%d")
    assert cli.main(["verify", "--graph", str(gfile), "--colors", str(cfile), "--mode", "d1"]) == 1
    np.savetxt(cfile, bad[:-1], fmt="%d")
    assert cli.main(["verify", "--graph", str(gfile), "--colors", str(cfile), "--mode", "d1"]) == 2


def test_bench_csv(capsys):
    assert cli.main(["bench", "--gen", "mesh:8,8,8", "--mode", "d1-2gl", "--sweep", "ranks=1,2", "--repeat", "2",
                     "--deterministic"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "mode,ranks,seed,rounds,colors,recolored_total,bytes_sent,comm_ms,comp_ms,total_ms"
    assert len(rows) == 5
    assert all(r.split(",")[6] == "0" for r in rows[1:] if r.split(",")[1] == "1")  # ranks=1: no bytes


def test_config_error_exit_2():
    assert cli.main(["color", "--gen", "nosuch:1"]) == 2
