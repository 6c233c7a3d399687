"""Command-line front end (declared by the reference as the console
script chroma.cli:main, pyproject.toml:16, but not shipped there).

    python -m paper_2107_00075_b200.cli color  --gen mesh:16,16,16 --mode d1 --ranks 4 [--out r.json]
    python -m paper_2107_00075_b200.cli verify --graph G --colors C --mode d1
    python -m paper_2107_00075_b200.cli bench  --gen gnp:400,0.03,7 --mode d1 --sweep ranks=1,2,4,8 --repeat 3

color  runs run_distributed end to end on the GPU, verifies the result with the GPU
       checker and prints "mode=<m> ranks=<r> rounds=<k> colors=<c> proper=<bool>";
       exit 1 on an improper result or non-convergence, 2 on an I/O or config error.
verify prints up to 20 violations and their count; exit 0 iff proper, 2 on a size
       mismatch.  Colour files hold one integer per line (line i = vertex i).
bench  prints CSV: mode,ranks,seed,rounds,colors,recolored_total,bytes_sent,comm_ms,
       comp_ms,total_ms -- one row per (ranks, repeat).
Generators: mesh:NX,NY,NZ  myciel:K  gnp:N,P[,SEED]  stencil27:L  rmat:SCALE[,EF]
bip:ROWS[,K] (PD2 input); --graph reads an edge list, Matrix Market or CHRG file.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

__all__ = ["main", "cmd_color", "cmd_verify", "cmd_bench"]


class ConfigError(Exception):
    pass


def _graph(args):
    from . import graph as G
    if args.graph:
        try:
            g = G.load_graph(args.graph, directed=args.mode == "pd2")
        except (OSError, ValueError) as e:
            raise ConfigError(f"cannot read {args.graph}: {e}")
        if isinstance(g, G.DirectedGraph):
            b = G.to_bipartite(g)
            return b.graph, b.s_mask()
        if isinstance(g, G.BipartiteGraph):
            return g.graph, g.s_mask()
        return g, None
    if not args.gen:
        raise ConfigError("one of --graph or --gen is required")
    kind, _, spec = args.gen.partition(":")
    try:
        vals = [x for x in spec.split(",") if x]
        if kind == "mesh":
            return G.gen_hex_mesh(*[int(x) for x in vals]), None
        if kind == "myciel":
            return G.gen_mycielskian(int(vals[0])), None
        if kind == "gnp":
            seed = int(vals[2]) if len(vals) > 2 else args.seed
            return G.gen_random_gnp(int(vals[0]), float(vals[1]), seed), None
        if kind == "stencil27":
            return G.gen_stencil27(int(vals[0])), None
        if kind == "rmat":
            return G.gen_rmat(int(vals[0]), int(vals[1]) if len(vals) > 1 else 16, args.seed), None
        if kind == "bip":
            b = G.gen_random_bipartite(int(vals[0]), int(vals[1]) if len(vals) > 1 else 32, args.seed)
            return b.graph, b.s_mask()
    except (IndexError, ValueError) as e:
        raise ConfigError(f"bad --gen {args.gen}: {e}")
    raise ConfigError(f"unknown generator {kind!r}")


def _partition(g, args, ranks):
    from . import partition as PT
    if args.partition == "block":
        return PT.partition_block(g, ranks)
    if args.partition == "edge":
        return PT.partition_edge_balanced(g, ranks)
    if args.partition == "random":
        return PT.partition_random(g, ranks, args.seed)
    raise ConfigError(f"unknown partition {args.partition!r}")


def _run_once(g, mask, args, ranks):
    from . import graph as G
    from . import localcolor as L
    from . import protocol as R
    from . import runtime as RT
    from . import verify as V
    mode = R.Mode(args.mode)
    pm = _partition(g, args, ranks)
    t0 = time.perf_counter()
    world = RT.build_local_graphs(g, pm, R.ghost_layers_for(mode))
    t_build = time.perf_counter() - t0
    cfg = R.AlgorithmConfig(mode=mode, recolor_degrees=args.recolor_degrees == "on",
                            deterministic=args.deterministic,
                            algorithm="free" if args.free else None,
                            kernel=L.KernelChoice(max_degree_threshold=args.eb_threshold))
    t0 = time.perf_counter()
    converged = True
    try:
        colors, reports = R.run_distributed(world, cfg)
    except R.NonConvergenceError as e:
        colors, reports, converged = None, e.reports, False
    t_run = time.perf_counter() - t0
    viol = None
    if colors is not None:
        vmode = {"d1": "d1", "d1-2gl": "d1", "d2": "d2", "pd2": "pd2"}[mode.value]
        viol = V.count_violations(g, colors, vmode, mask if vmode == "pd2" else None)
    st = G.stats(g)
    record = {
        "config": {"mode": mode.value, "ranks": ranks, "partition": args.partition, "seed": args.seed,
                   "recolor_degrees": args.recolor_degrees, "deterministic": args.deterministic,
                   "free": args.free, "eb_threshold": args.eb_threshold, "graph": args.graph or args.gen},
        "graph_stats": {"num_vertices": st.num_vertices, "num_edges": st.num_edges,
                        "avg_degree": st.delta_avg, "delta_max": st.delta_max},
        "mode": mode.value, "ranks": ranks, "seed": args.seed,
        "rounds": [r.to_dict() for r in reports],
        "total_colors": int(len(np.unique(colors[colors > 0]))) if colors is not None else None,
        "times_ms": {"build": 1e3 * t_build, "run": 1e3 * t_run,
                     "comm": 1e3 * sum(r.time_comm_s for r in reports),
                     "comp": 1e3 * sum(r.time_color_s + r.time_detect_s for r in reports)},
        "verification": ("proper" if viol == 0 else f"{viol} violations") if colors is not None
        else "not converged",
    }
    return record, colors, converged and viol == 0


def cmd_color(args) -> int:
    g, mask = _graph(args)
    record, colors, ok = _run_once(g, mask, args, args.ranks)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(record, fh, indent=1)
    if args.colors_out and colors is not None:
        np.savetxt(args.colors_out, colors, fmt="%d")
    print(f"mode={record['mode']} ranks={record['ranks']} rounds={len(record['rounds'])} "
          f"colors={record['total_colors']} proper={str(ok).lower()}")
    return 0 if ok else 1


def cmd_verify(args) -> int:
    from . import verify as V
    g, mask = _graph(args)
    try:
        colors = np.loadtxt(args.colors, dtype=np.int64, ndmin=1).astype(np.int32)
    except OSError as e:
        raise ConfigError(f"cannot read {args.colors}: {e}")
    if len(colors) != g.num_vertices:
        print(f"size mismatch: {len(colors)} colours for {g.num_vertices} vertices", file=sys.stderr)
        return 2
    if args.mode in ("d1", "d1-2gl"):
        viol = V.verify_d1(g, colors)
    else:
        viol = V.verify_d2(g, colors, partial=args.mode == "pd2", endpoint_mask=mask if args.mode == "pd2" else None)
    for v in viol[:20]:
        print(v)
    print(f"violations={len(viol)}")
    return 0 if not viol else 1


def cmd_bench(args) -> int:
    g, mask = _graph(args)
    key, _, vals = args.sweep.partition("=")
    if key != "ranks":
        raise ConfigError("--sweep takes ranks=R1,R2,...")
    ranks_list = [int(x) for x in vals.split(",") if x]
    print("mode,ranks,seed,rounds,colors,recolored_total,bytes_sent,comm_ms,comp_ms,total_ms")
    rc = 0
    for ranks in ranks_list:
        for _ in range(args.repeat):
            record, _, ok = _run_once(g, mask, args, ranks)
            rounds = record["rounds"]
            print(f"{record['mode']},{ranks},{args.seed},{len(rounds)},{record['total_colors']},"
                  f"{sum(sum(r['recolored_per_rank']) for r in rounds)},{sum(r['bytes_sent'] for r in rounds)},"
                  f"{record['times_ms']['comm']:.3f},{record['times_ms']['comp']:.3f},{record['times_ms']['run']:.3f}")
            rc |= 0 if ok else 1
    return rc


def _parser():
    ap = argparse.ArgumentParser(prog="chroma", description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("color", "verify", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--graph")
        p.add_argument("--gen")
        p.add_argument("--mode", default="d1", choices=["d1", "d1-2gl", "d2", "pd2"])
        p.add_argument("--seed", type=int, default=1)
        if name == "verify":
            p.add_argument("--colors", required=True)
            continue
        p.add_argument("--ranks", type=int, default=1)
        p.add_argument("--partition", default="block", choices=["block", "edge", "random"])
        p.add_argument("--recolor-degrees", default="off", choices=["on", "off"])
        p.add_argument("--deterministic", action="store_true")
        p.add_argument("--free", action="store_true", help="free-running GPU mode (extension)")
        p.add_argument("--eb-threshold", type=int, default=6000)
        if name == "color":
            p.add_argument("--out")
            p.add_argument("--colors-out")
        else:
            p.add_argument("--sweep", default="ranks=1,2,4,8")
            p.add_argument("--repeat", type=int, default=1)
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return {"color": cmd_color, "verify": cmd_verify, "bench": cmd_bench}[args.cmd](args)
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
