"""Dev probe: GS colouring kernel time on BASELINE-like shapes (+ oracle check)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import oracle
from paper_2107_00075_b200 import graph as G, partition as PT, runtime as RT, protocol as R, _lib

def run(name, g, mode, check=True, reps=3, P=1, algorithm=None):
    t0 = time.perf_counter()
    w = RT.build_local_graphs(g, PT.partition_block(g, P), R.ghost_layers_for(R.Mode(mode)))
    tb = time.perf_counter() - t0
    cfg = R.AlgorithmConfig(mode=R.Mode(mode), deterministic=algorithm is None, algorithm=algorithm)
    tb5 = (C.c_double * 5)()
    best = None
    for _ in range(reps):
        colors, reps_ = R.run_distributed(w, cfg)
        _lib.lib().chroma_world_last_timing(w.handle.h, tb5)
        t = list(tb5)
        best = t if best is None or t[0] < best[0] else best
    ok = ""
    if check:
        ow = oracle.World(g.row_offsets, g.col_indices, PT.partition_block(g, P).owner, P, R.ghost_layers_for(R.Mode(mode)))
        ref, _ = ow.run(mode, False, True)
        if algorithm == "free":
            vm = {"d1": "d1", "d1-2gl": "d1", "d2": "d2", "pd2": "pd2"}[mode]
            bad = len(oracle.verify(g.row_offsets, g.col_indices, colors, vm))
            ok = f"{'PROPER' if bad == 0 else f'BAD({bad})'} gs_colors={ref.max()} ratio={colors.max()/max(1,ref.max()):.3f}"
        else:
            ok = "EXACT" if np.array_equal(ref, colors) else "MISMATCH"
    print(f"{name:28s} {mode:6s} P={P} n={g.num_vertices:9d} m={len(g.col_indices)//2:10d} build={tb*1e3:8.1f}ms "
          f"total={best[0]*1e3:8.3f}ms kernel={best[1]*1e3:8.3f}ms detect={best[4]*1e3:7.3f}ms rounds={len(reps_)} "
          f"colors={colors.max()} {ok}", flush=True)

which = sys.argv[1:] or ["c1", "c2", "rmat18", "d2_100", "pd2_16", "c2p4"]
if "c1" in which: run("grid 1000^2", G.gen_hex_mesh(1000, 1000, 1), "d1")
if "c2" in which: run("27pt 128^3", G.gen_stencil27(128, device="cuda"), "d1-2gl")
if "c2p4" in which: run("27pt 128^3", G.gen_stencil27(128, device="cuda"), "d1-2gl", P=4)
if "rmat18" in which: run("rmat s18", G.gen_rmat(18, 16, 1, device="cuda"), "d1", check=True)
if "rmat20" in which: run("rmat s20", G.gen_rmat(20, 16, 1, device="cuda"), "d1", check=True)
if "d2_100" in which: run("7pt 100^3", G.gen_hex_mesh(100, 100, 100), "d2")
if "pd2_16" in which: run("pd2 2^16 rows", G.gen_random_bipartite(1 << 16, 32, 3, device="cuda").graph, "pd2")
if "pd2_18" in which: run("pd2 2^18 rows", G.gen_random_bipartite(1 << 18, 32, 3, device="cuda").graph, "pd2", check=False)
if "jac" in which:
    run("rmat s18 jacobi", G.gen_rmat(18, 16, 1, device="cuda"), "d1", check=False, algorithm="jacobi")
    run("rmat s20 jacobi", G.gen_rmat(20, 16, 1, device="cuda"), "d1", check=False, algorithm="jacobi")
    run("rmat s18 free", G.gen_rmat(18, 16, 1, device="cuda"), "d1", check=False, algorithm="free")
    run("27pt 32^3 jacobi", G.gen_stencil27(32, device="cuda"), "d1-2gl", check=False, algorithm="jacobi")
    run("rmat s18 jacobi P8", G.gen_rmat(18, 16, 1, device="cuda"), "d1", check=False, algorithm="jacobi", P=8)
    run("rmat s18 gs P8", G.gen_rmat(18, 16, 1, device="cuda"), "d1", check=False, P=8)
if "pd2s" in which:
    for sc in (16, 18, 20):
        run(f"pd2 2^{sc} rows", G.gen_random_bipartite(1 << sc, 32, 3, device="cuda").graph, "pd2", check=(sc <= 18))
if "d2s" in which:
    run("7pt 100^3 d2", G.gen_hex_mesh(100, 100, 100), "d2")
    run("7pt 200^3 d2", G.gen_hex_mesh(200, 200, 200), "d2", check=False)
if "free" in which:
    run("27pt 128^3 free", G.gen_stencil27(128, device="cuda"), "d1-2gl", algorithm="free")
    run("27pt 128^3 free P8", G.gen_stencil27(128, device="cuda"), "d1-2gl", algorithm="free", P=8)
    run("rmat s18 free", G.gen_rmat(18, 16, 1, device="cuda"), "d1", algorithm="free")
    run("rmat s20 free", G.gen_rmat(20, 16, 1, device="cuda"), "d1", algorithm="free")
    run("rmat s20 free P8", G.gen_rmat(20, 16, 1, device="cuda"), "d1", algorithm="free", P=8)
    run("rmat s20 gs P8", G.gen_rmat(20, 16, 1, device="cuda"), "d1", check=False, P=8)
    run("7pt 100^3 d2 free", G.gen_hex_mesh(100, 100, 100), "d2", algorithm="free")
    run("pd2 2^18 free", G.gen_random_bipartite(1 << 18, 32, 3, device="cuda").graph, "pd2", algorithm="free")
    run("pd2 2^20 free", G.gen_random_bipartite(1 << 20, 32, 3, device="cuda").graph, "pd2", algorithm="free", check=False)
    run("rmat s22 free P8", G.gen_rmat(22, 16, 1, device="cuda"), "d1", algorithm="free", P=8, check=False)
if "freetrace" in which:
    run("27pt 128^3 free", G.gen_stencil27(128, device="cuda"), "d1-2gl", algorithm="free", reps=1, check=False)
    run("rmat s20 free", G.gen_rmat(20, 16, 1, device="cuda"), "d1", algorithm="free", reps=1, check=False)
    run("pd2 2^18 free", G.gen_random_bipartite(1 << 18, 32, 3, device="cuda").graph, "pd2", algorithm="free", reps=1, check=False)
if "rounds" in which:
    g = G.gen_rmat(20, 16, 1, device="cuda")
    for alg in ("free", None):
        w = RT.build_local_graphs(g, PT.partition_block(g, 8), 1)
        cfg = R.AlgorithmConfig(mode=R.Mode("d1"), deterministic=alg is None, algorithm=alg)
        colors, reps_ = R.run_distributed(w, cfg)
        colors, reps_ = R.run_distributed(w, cfg)
        print("algorithm", alg)
        for r in reps_:
            print(f"  round {r.round_index:3d} conflicts={r.conflicts:7d} recolored={sum(r.recolored_per_rank):8d} "
                  f"color={r.time_color_s*1e3:7.3f}ms comm={r.time_comm_s*1e3:7.3f}ms detect={r.time_detect_s*1e3:7.3f}ms")
if "c3trace" in which:
    sc = int(os.environ.get("SCALE", "24"))
    g = G.gen_rmat(sc, 16, 1, device="cuda")
    print("max degree", int(np.diff(g.row_offsets).max()), "heavy>1024", int((np.diff(g.row_offsets) > 1024).sum()),
          ">4096", int((np.diff(g.row_offsets) > 4096).sum()), flush=True)
    run(f"rmat s{sc} free", g, "d1", algorithm="free", check=False, reps=2)
if "table" in which:
    run("C1 grid 1000^2 gs", G.gen_hex_mesh(1000, 1000, 1), "d1")
    run("C2 27pt 128^3 gs", G.gen_stencil27(128, device="cuda"), "d1-2gl")
    run("C2 27pt 128^3 gs P8", G.gen_stencil27(128, device="cuda"), "d1-2gl", P=8)
    run("R-MAT s20 gs", G.gen_rmat(20, 16, 1, device="cuda"), "d1")
    run("R-MAT s20 free", G.gen_rmat(20, 16, 1, device="cuda"), "d1", algorithm="free")
    run("C4 7pt 200^3 d2 gs", G.gen_hex_mesh(200, 200, 200), "d2", check=False)
    run("C4 7pt 200^3 d2 free", G.gen_hex_mesh(200, 200, 200), "d2", check=False, algorithm="free")
    run("C4 7pt 200^3 d2 gs P8", G.gen_hex_mesh(200, 200, 200), "d2", check=False, P=8)
    run("C5 pd2 2^20 gs", G.gen_random_bipartite(1 << 20, 32, 3, device="cuda").graph, "pd2", check=False)
    run("C5 pd2 2^20 free", G.gen_random_bipartite(1 << 20, 32, 3, device="cuda").graph, "pd2", check=False, algorithm="free")
    run("C5 pd2 2^22 free", G.gen_random_bipartite(1 << 22, 32, 3, device="cuda").graph, "pd2", check=False, algorithm="free")
    run("C5 pd2 2^22 free P8", G.gen_random_bipartite(1 << 22, 32, 3, device="cuda").graph, "pd2", check=False, algorithm="free", P=8)
if "d2free" in which:
    run("C4 7pt 200^3 d2 free", G.gen_hex_mesh(200, 200, 200), "d2", check=False, algorithm="free")
    run("C4 7pt 200^3 d2 free P8", G.gen_hex_mesh(200, 200, 200), "d2", check=False, algorithm="free", P=8)
    run("7pt 100^3 d2 free P8", G.gen_hex_mesh(100, 100, 100), "d2", algorithm="free", P=8)
    run("pd2 2^18 free P8", G.gen_random_bipartite(1 << 18, 32, 3, device="cuda").graph, "pd2", algorithm="free", P=8)
    run("C5 pd2 2^22 free P8", G.gen_random_bipartite(1 << 22, 32, 3, device="cuda").graph, "pd2", check=False, algorithm="free", P=8)
if "sched" in which:
    run("C1 grid 1000^2 gs", G.gen_hex_mesh(1000, 1000, 1), "d1", check=False)
    run("C2 27pt 128^3 gs", G.gen_stencil27(128, device="cuda"), "d1-2gl", check=False)
    run("C2 27pt 128^3 gs P8", G.gen_stencil27(128, device="cuda"), "d1-2gl", P=8, check=False)
    run("C2 27pt 128^3 gs P2", G.gen_stencil27(128, device="cuda"), "d1-2gl", P=2, check=False)
    run("R-MAT s20 gs", G.gen_rmat(20, 16, 1, device="cuda"), "d1", check=False)
    run("R-MAT s20 gs P8", G.gen_rmat(20, 16, 1, device="cuda"), "d1", check=False, P=8)
    run("C1 grid 1000^2 gs P8", G.gen_hex_mesh(1000, 1000, 1), "d1", check=False, P=8)
