/*
 * chroma_b200.h -- C-ABI of libchroma_b200.so, the B200-native backend of the
 * distributed speculate-and-iterate graph colouring of arXiv 2107.00075.
 *
 * Every entry point replaces one function of the reference package `chroma`
 * (/root/reference/pkg/src/chroma, cited as chroma/<module>.py:line).  The
 * reference is pure Python and has no FFI of its own; these are the bindings a
 * maintainer would add behind its Python signatures (see INTEGRATION.md for the
 * ctypes stubs).  Plain pointers and sizes only: int64 CSR exactly as
 * chroma.graph.Graph stores it (chroma/graph.py:40-64), int32 colours
 * (chroma/localcolor.py:115-117), int64 gids/degrees/worklists.
 *
 * Pointer arguments are HOST pointers unless the call's `flags` has
 * CHROMA_DEVICE_PTRS, in which case they are device pointers on the handle's
 * device.  All calls are synchronous with respect to the caller and return a
 * status code; chroma_last_error() gives a thread-local message.
 * Calls on one handle are not re-entrant.
 */
#ifndef CHROMA_B200_H
#define CHROMA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -- map 1:1 to the reference's exceptions */
#define CHROMA_OK 0
#define CHROMA_EVALUE 1       /* ValueError                                     */
#define CHROMA_EPROTOCOL 2    /* runtime.ProtocolError   (chroma/runtime.py:37) */
#define CHROMA_ENONCONV 3     /* protocol.NonConvergenceError (protocol.py:67) */
#define CHROMA_ERUNTIME 4     /* RuntimeError (sweep tripwire, localcolor.py:34)*/
#define CHROMA_ECUDA 5        /* CUDA / NCCL failure                            */

#define CHROMA_DEVICE_PTRS 1u

/* modes: chroma/protocol.py:47-51 */
#define CHROMA_MODE_D1 0
#define CHROMA_MODE_D1_2GL 1
#define CHROMA_MODE_D2 2
#define CHROMA_MODE_PD2 3

/* colouring algorithms selected by AlgorithmConfig.deterministic (+ extension) */
#define CHROMA_ALGO_GAUSS_SEIDEL 0   /* deterministic=True: ascending-lid first fit, bit-exact */
#define CHROMA_ALGO_FREE 1           /* deterministic=False: free-running speculative (B200)   */
#define CHROMA_ALGO_JACOBI 2         /* deterministic=False, jacobi_exact: reference sweeps   */
#define CHROMA_ALGO_JACOBI_EB 3      /* same sweeps, Kernel.EDGE_BASED (chroma/localcolor.py:181-195) */

typedef struct chroma_csr chroma_csr;      /* a device-resident CSR graph        */
typedef struct chroma_world chroma_world;  /* device-resident ranks + routing    */

typedef struct chroma_round_report {       /* chroma/runtime.py:83-108 */
  int64_t round_index;
  int64_t conflicts;
  int64_t bytes_sent;
  int64_t messages_sent;
  double time_color_s;
  double time_comm_s;
  double time_detect_s;
} chroma_round_report;

const char* chroma_last_error(void);
const char* chroma_version(void);
int chroma_device_count(int* count);

/* gid hash and the pairwise loser rule: chroma/protocol.py:79-88, 99-133 (host) */
uint64_t chroma_gid_rand(int64_t gid);
int chroma_check_conflicts(int64_t v, int64_t u, int32_t* colors, const int64_t* gids,
                           const int64_t* degrees, int recolor_degrees, int* result);

/* ---------------------------------------------------------------- CSR graphs */
/* Upload an undirected CSR graph (chroma/graph.py:40-64). */
int chroma_csr_create(int64_t n, const int64_t* row_offsets, const int64_t* col_indices,
                      int device, uint32_t flags, chroma_csr** out);
int chroma_csr_destroy(chroma_csr* g);

/* chroma/localcolor.py:120-133 serial_greedy(g, order=None) -> colors (int32[n]).
 * order may be NULL (ascending ids); otherwise a permutation (ValueError if not). */
int chroma_serial_greedy(chroma_csr* g, const int64_t* order, int32_t* colors_out, uint32_t flags);

/* chroma/localcolor.py:198-227 speculative_color (dist=1) and
 * chroma/localcolor.py:274-303 speculative_color_d2 (dist=2, partial).
 * colors (int32[n]) is updated in place; worklist holds int64 vertex ids. */
int chroma_color(chroma_csr* g, int32_t* colors, const int64_t* worklist, int64_t nwl, int dist,
                 int partial, int algo, uint32_t flags);

/* chroma/protocol.py:136-194 detect_conflicts_d1 (dist 1, rows = ghost local ids
 * owned_count..num_local-1) / detect_conflicts_d2 (dist 2, rows = boundary_d2) on an
 * arbitrary local CSR: colors updated in place, *count = conflicts found. */
int chroma_detect(chroma_csr* g, int32_t* colors, const int64_t* gids, const int64_t* degrees,
                  const int64_t* rows, int64_t nrows, int dist, int partial, int recolor_degrees,
                  int64_t* count, uint32_t flags);

/* chroma/verify.py:61-104.  mode 0 = verify_d1, 1 = verify_d2, 2 = verify_d2(partial).
 * endpoint_mask (uint8[n]) may be NULL.  Writes up to `cap` violation rows
 * (kind, u, w, middle) in the reference's order; *n_violations is the total.
 * kind: 0 uncoloured, 1 d1-edge, 2 d2-path, 3 pd2-path. */
int chroma_verify(chroma_csr* g, const int32_t* colors, const uint8_t* endpoint_mask, int mode,
                  int64_t* n_violations, int64_t* rows_out, int64_t cap, uint32_t flags);

/* chroma/verify.py:107-112: number of distinct positive colours; hist_out (int64,
 * length hist_cap, index = colour) is filled when non-NULL. */
int chroma_color_stats(const int32_t* colors, int64_t n, int device, int64_t* num_colors,
                       int64_t* max_color, int64_t* hist_out, int64_t hist_cap, uint32_t flags);

/* ---------------------------------------------------------------- worlds */
/* chroma/runtime.py:149-268 build_local_graphs(g, pm, ghost_layers): builds the
 * local graphs of ranks [rank_lo, rank_hi) of a `num_ranks`-way partition on
 * `device` with the reference's exact local-id layout (owned, layer-1, layer-2
 * ghosts, each ascending by gid; rows sorted by local id).  A single process may
 * hold all ranks ("virtual ranks", exchange is a device copy) or one rank per
 * process (then call chroma_world_connect). */
int chroma_world_create(int64_t n, const int64_t* row_offsets, const int64_t* col_indices,
                        int32_t num_ranks, const int32_t* owner, int32_t ghost_layers,
                        int32_t rank_lo, int32_t rank_hi, int device, chroma_world** out);
int chroma_world_destroy(chroma_world* w);

/* info[0..15]: owned, ghost, first_layer_ghost_count, num_local_edges,
 * num_ghost_edges, nnz, n_boundary_d1, n_boundary_d2, delta_max(global graph),
 * num_global_vertices, num_edges(global), ghost_layers, 0... */
int chroma_world_rank_info(chroma_world* w, int32_t rank, int64_t* info);
/* host copies of a rank's LocalGraph arrays (chroma/runtime.py:41-66), local ids */
int chroma_world_rank_arrays(chroma_world* w, int32_t rank, int64_t* row_offsets,
                             int64_t* col_indices, int64_t* gids, int32_t* ghost_owner,
                             int64_t* boundary_d1, int64_t* boundary_d2);

/* NCCL: 128-byte unique id from rank 0, then connect every process's world
 * (one rank per process) with its static halo routing (local ids): send_counts[p]
 * owned vertices to peer p listed in send_lids (peer-major, in the order the peer
 * expects), recv_counts[p] ghost slots from peer p listed in recv_lids.  This is the
 * precomputed form of chroma/runtime.py:249-256 send_targets. */
typedef struct chroma_comm chroma_comm;   /* an NCCL communicator (one per process) */
int chroma_nccl_unique_id(void* id_out_128);
int chroma_comm_create(const void* nccl_id_128, int32_t nranks, int32_t rank, int device,
                       chroma_comm** out);
/* One process driving ndev GPUs (rank i on devices[i]): ncclCommInitAll; out[i] is
 * rank i's communicator.  Each rank's world must then be connected and run from its
 * own host thread (the calls are collective). */
int chroma_comm_create_all(int32_t ndev, const int* devices, chroma_comm** out);
int chroma_comm_destroy(chroma_comm* c);
/* The world borrows `comm` (which must outlive it). */
int chroma_world_connect(chroma_world* w, chroma_comm* comm, int32_t nranks, int32_t rank,
                         const int64_t* send_counts, const int64_t* send_lids,
                         const int64_t* recv_counts, const int64_t* recv_lids);

/* chroma/protocol.py:197-218 compute_global_degrees: int64[num_local] of `rank`. */
int chroma_world_global_degrees(chroma_world* w, int32_t rank, int64_t* degrees_out);

/* chroma/runtime.py:136-139 reset_exchange_state */
int chroma_world_reset_exchange(chroma_world* w);
/* chroma/runtime.py:271-308 exchange_boundary_colors over all local ranks.
 * colorings[r] -> int32[num_local(r)] for r in [rank_lo, rank_hi). */
int chroma_world_exchange(chroma_world* w, int32_t** colorings, int changed_only,
                          int64_t* bytes_sent, int64_t* messages_sent);

/* chroma/localcolor.py:198-303 on a world rank's local graph (worklist: local ids). */
int chroma_world_color(chroma_world* w, int32_t rank, int32_t* colors, const int64_t* worklist,
                       int64_t nwl, int dist, int partial, int algo);
/* chroma/protocol.py:136-194 detect_conflicts_d1 / detect_conflicts_d2 on one rank.
 * degrees may be NULL (the world's global degrees are used). */
int chroma_world_detect(chroma_world* w, int32_t rank, int32_t* colors, const int64_t* degrees,
                        int dist, int partial, int recolor_degrees, int64_t* count);

/* chroma/protocol.py:263-334 run_distributed.  colors_out: int32[num_global] in
 * virtual mode (all ranks local); in connected mode int32[owned] of this rank.
 * reports: up to `cap` entries; recolored: cap x num_ranks int64.
 * Returns CHROMA_ENONCONV with the reports filled when max_rounds is exceeded. */
int chroma_run_distributed(chroma_world* w, int mode, int recolor_degrees, int algo,
                           int max_rounds, int32_t* colors_out, chroma_round_report* reports,
                           int64_t* recolored, int64_t cap, int64_t* n_reports, uint32_t flags);

/* Device pointer to the world's concatenated colour array and per-rank lid offset
 * (for zero-copy verification/bench). */
int chroma_world_colors_device(chroma_world* w, int32_t rank, int32_t** dev_ptr, int64_t* lid_offset);

/* CUDA-event times of the last chroma_run_distributed on this world, seconds:
 * out[0] whole call on the device stream, out[1] colouring kernel only (summed over
 * rounds), out[2] colour phase, out[3] exchange phase, out[4] detect phase. */
int chroma_world_last_timing(chroma_world* w, double* out5);

/* ---------------------------------------------------------------- generators */
/* Synthetic BASELINE inputs built on `device` straight into int64 CSR (device
 * pointers): sorted, simple, symmetric rows as chroma/graph.py:166-179 preprocess
 * leaves them.  Counter-based draws (mix64 = the gid_rand finaliser of
 * chroma/protocol.py:79-88) so that graph.py's NumPy path and the C oracle build the
 * identical graph; the exact recipe is in csrc/gen.cu and DESIGN.md.
 *   chroma_gen_rmat: Graph500 R-MAT, 2^scale vertices, edge_factor * 2^scale draws,
 *     level thresholds t_* = floor(p * 2^32) for a, a+b, a+b+c; labels permuted when
 *     `permute`.  col must hold 2 * edge_factor * 2^scale entries.
 *   chroma_gen_random_bipartite: rows x rows pattern with nnz_per_row uniform
 *     columns per row -> preprocess_directed -> to_bipartite (chroma/graph.py:182-188,
 *     388-399): 2*rows vertices.  col must hold 2 * rows * nnz_per_row entries.
 *   chroma_gen_box: kind 0 = gen_hex_mesh(nx, ny, nz) (chroma/graph.py:320-341),
 *     kind 1 = 27-point stencil; call with col NULL to learn *nnz_out first. */
int chroma_gen_rmat(int32_t scale, int64_t edge_factor, uint64_t seed, uint32_t t_a, uint32_t t_ab,
                    uint32_t t_abc, int permute, int device, int64_t* row_offsets, int64_t* col_indices,
                    int64_t* nnz_out);
int chroma_gen_random_bipartite(int64_t rows, int64_t nnz_per_row, uint64_t seed, int device,
                                int64_t* row_offsets, int64_t* col_indices, int64_t* nnz_out);
int chroma_gen_box(int32_t kind, int64_t nx, int64_t ny, int64_t nz, int device, int64_t* row_offsets,
                   int64_t* col_indices, int64_t* nnz_out);

/* Number of kernels this library launched on `w` (or globally if w is NULL). */
int64_t chroma_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
