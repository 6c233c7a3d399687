"""Shared helpers: rebuild the golden input graphs on either side (CPU oracle or GPU)."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2107_00075_b200 import graph as G  # noqa: E402
from paper_2107_00075_b200 import partition as PT  # noqa: E402


def sha(a, dtype="<i4"):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dtype)).tobytes()).hexdigest()


def golden_graph(name, arrays):
    """The golden input graphs.  Deterministic generators are rebuilt here (and checked
    against the reference's CSR hash in test_inputs); random ones come from the fixture."""
    key = f"graph/{name}/row_offsets"
    if key in arrays:
        off = arrays[key].astype(np.int64)
        col = arrays[f"graph/{name}/col_indices"].astype(np.int64)
        return G.Graph(len(off) - 1, off, col)
    builders = {"hex32": lambda: G.gen_hex_mesh(32, 32, 32),
                "hex64x64": lambda: G.gen_hex_mesh(64, 64, 1),
                "st27_30": lambda: G.gen_stencil27(30)}
    return builders[name]()


def golden_partition(rec, g, arrays):
    part = rec["partition"]
    if part == "block":
        return PT.partition_block(g, rec["P"])
    seed = int(part.split(":")[1])
    return PT.PartitionMap(arrays[f"part/{rec['graph']}/{seed}/{rec['P']}"].astype(np.int32), rec["P"])
