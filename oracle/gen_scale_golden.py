"""Full-scale golden values for the BASELINE configurations, from the C oracle.

TEST INFRASTRUCTURE: runs oracle/ (the pinned C restatement of the reference,
tests/test_oracle_golden.py) on the exact inputs of C1-C5 -- built by the oracle's
own counter-based generator (oracle/chroma_gen.c) for C3/C5 and by the reference's
gen_hex_mesh recipe for C1/C4 -- and writes tests/golden/scale.json: CSR hashes
(so the device generators can be checked against the same arrays), and for each
deterministic run the sha256 of the int32 colour array, rounds, colours and the
per-round conflict counts.  The Python reference itself would need hours to days at
these sizes; the C oracle is pinned to it on the Appendix A goldens.

    python oracle/gen_scale_golden.py [item ...]      # default: every missing item
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "scale.json")

import oracle  # noqa: E402


def sha(a, dt) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype(dt).tobytes()).hexdigest()


def block_owner(n: int, P: int) -> np.ndarray:
    """partition_block (chroma/partition.py:49-58): floor(r n / P) boundaries."""
    owner = np.empty(n, np.int32)
    for r in range(P):
        owner[r * n // P:(r + 1) * n // P] = r
    return owner


def run(off, col, P: int, mode: str, gl: int, deterministic: bool = True) -> dict:
    t = time.time()
    w = oracle.World(off, col, block_owner(len(off) - 1, P), P, gl)
    tb = time.time() - t
    t = time.time()
    c, reps = w.run(mode, False, deterministic)
    tr = time.time() - t
    del w
    return {"sha256": sha(c, "<i4"), "rounds": len(reps), "colors": int(len(np.unique(c[c > 0]))),
            "max_color": int(c.max()) if len(c) else 0, "conflicts": [r["conflicts"] for r in reps],
            "oracle_build_s": round(tb, 2), "oracle_run_s": round(tr, 2)}


def hex_mesh(nx, ny, nz):
    from paper_2107_00075_b200 import graph as G
    g = G.gen_hex_mesh(nx, ny, nz)
    return g.row_offsets, g.col_indices


def stencil27(L):
    from paper_2107_00075_b200 import graph as G
    g = G.gen_stencil27(L)
    return g.row_offsets, g.col_indices


ITEMS = {
    "c1_1000": (lambda: hex_mesh(1000, 1000, 1), [(1, "d1", 1)]),
    # name: (graph builder, [(P, mode, ghost layers[, "jacobi"])]); "jacobi": the
    # reference's default speculative mode (deterministic=False), key suffix _jacobi
    "c3_s24": (lambda: oracle.gen_rmat(24), [(1, "d1", 1), (8, "d1", 1), (1, "d1", 1, "jacobi"), (4, "d1", 1, "jacobi")]),
    "c5_2p20": (lambda: oracle.gen_bipartite(1 << 20, 32, 3), [(1, "pd2", 2), (8, "pd2", 2)]),
    "c4_200": (lambda: hex_mesh(200, 200, 200), [(8, "d2", 2), (1, "d2", 2)]),
    "c2_128": (lambda: stencil27(128), [(2, "d1-2gl", 2), (4, "d1-2gl", 2), (8, "d1-2gl", 2)]),
    "c5_2p22": (lambda: oracle.gen_bipartite(1 << 22, 32, 3), [(1, "pd2", 2), (8, "pd2", 2)]),
}


def main(names):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for name in names:
        build, runs = ITEMS[name]
        entry = data.get(name, {})
        t = time.time()
        off, col = build()
        entry["n"] = len(off) - 1
        entry["nnz"] = int(len(col))
        entry["col_sha256"] = sha(col, "<i8")
        entry["rowptr_sha256"] = sha(off, "<i8")
        print(f"{name}: graph n={entry['n']} nnz={entry['nnz']} in {time.time() - t:.1f}s", flush=True)
        for P, mode, gl, *alg in runs:
            key = f"{mode}_p{P}" + ("_jacobi" if alg else "")
            if key in entry:
                continue
            entry[key] = run(off, col, P, mode, gl, deterministic=not alg)
            print(f"  {key}: {entry[key]}", flush=True)
            data[name] = entry
            with open(OUT, "w") as fh:
                json.dump(data, fh, indent=1, sort_keys=True)
        data[name] = entry
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
        del off, col


if __name__ == "__main__":
    main(sys.argv[1:] or list(ITEMS))
