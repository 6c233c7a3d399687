// Device-resident world: the local graphs of the ranks held by this process,
// concatenated into one block-diagonal CSR (each rank's local ids shifted by its
// lid offset), plus the halo routing and the protocol scratch.
#pragma once
#include <vector>

#include "kernels.cuh"

#ifdef CHROMA_WITH_NCCL
#include <nccl.h>
#endif

namespace chroma {

struct RankMeta {
  int rank = 0;
  i64 lid_off = 0, owned = 0, ghost = 0, l1 = 0;
  i64 nnz_off = 0, nnz = 0, e_local = 0, e_ghost = 0;
  i64 b1_off = 0, nb1 = 0, b2_off = 0, nb2 = 0, ghost_off = 0;
};

struct Csr {
  int device = 0;
  cudaStream_t stream = nullptr;
  i64 n = 0, nnz = 0;
  DBuf<i64> rowptr;
  DBuf<i32> col;
};

// Level-synchronous Gauss-Seidel plan for one thread-block cluster (gs_cluster.cu)
struct ClusterPlan {
  bool ok = false;
  int CL = 0, CAP = 0, DW = 0, logB = 10, logCL = 4, nthreads = 0;
  bool chains = false;  // the schedule puts runs (gs_levels.cu) on one level
  bool zero_nm = false;  // built assuming every non-member colour is 0 (slots dropped)
  i64 per = 0, nv = 0, L = 0;
  size_t smem = 0;
  DBuf<i32> v, blob, item_sz, cta_item;  // v: scratch of the plan build
  DBuf<i64> item_o;
};

// Colouring scratch shared by every entry point that colours a CSR.
struct ColorScratch {
  DBuf<i32> wl, val, old, prop, pend2;
  DBuf<i64> nwl, np2;
  DBuf<uint8_t> flags, in_round;
  DBuf<unsigned long long> ticket;
  DBuf<i32> fl[6];  // free-running light/heavy/tiny lists x 2
  // optional schedule for the next Gauss-Seidel launch (gs_levels.cu): a level
  // schedule (level_mode) or a rank-interleaved id order
  const i32* level_wl = nullptr;
  i64 level_n = 0;
  bool level_mode = true;
  const ClusterPlan* cplan = nullptr;  // level schedule on one cluster (gs_cluster.cu)
  // free mode: keep the speculative path even without heavy rows (hubs pre-coloured)
  bool keep_free = false;
  DBuf<i64> level_n_dev;
  DBuf<i64> fcnt;
  FreeWaveScratch fw;
  ChunkedScratch chunked;
  NetScratch net;
  EbScratch eb;
  JacobiIncScratch ji;
  bool upper_zero = false;  // gs_chunked: no neighbour above a member is coloured yet
};

// Global hub pre-colouring scratch (hubs.cu)
struct HubScratch {
  DBuf<uint8_t> flags;
  DBuf<u32> bits;                          // hub bitmap over local lids
  DBuf<i32> lhubs, unit_hub;
  DBuf<i64> nlh, lcnt, loff, lgid, nunits, ustart;  // this world's owned hubs
  DBuf<i32> lnbr;                          // their hub neighbours (gids)
  DBuf<i64> ggid, cntz, pad64;             // H order (all ranks)
  DBuf<i32> gnbr, pad32;
  DBuf<i64> rowptr;
  DBuf<i32> table;                         // gid -> H index (hub gids only)
  DBuf<i32> col, colors, list, ovf;
  DBuf<i64> novf;
  DBuf<unsigned long long> missing;
  FreeWaveScratch fw;
};

struct World {
  int device = 0;
  cudaStream_t stream = nullptr;
  i32 P = 1, rank_lo = 0, rank_hi = 1, gl = 1;
  i64 n_global = 0, m_global = 0, delta_max = 0;
  std::vector<RankMeta> ranks;
  i64 NL = 0, NNZ = 0, NGHOST = 0, NB1 = 0, NB2 = 0;
  Csr g;                       // concatenated local graphs
  DBuf<i64> gids;
  DBuf<i32> deg;               // global degree of every local vertex (loser rule)
  DBuf<i32> colors;
  DBuf<i32> ghost_owner;       // per ghost slot, concatenated
  DBuf<i32> ghosts;            // ghost lids (D1 detection rows)
  DBuf<i32> b1, b2;            // boundary lids
  DBuf<uint8_t> owned_flag;
  DBuf<i32> rank_of;           // local rank index of every lid (for per-rank counts)
  // halo routes whose endpoints are both local (virtual ranks)
  i64 nrouted = 0;
  DBuf<i32> routed, st_dst, st_pair, last_sent;
  DBuf<i64> st_off;
  DBuf<unsigned long long> pair_cnt;
  // halo routes to other processes (NCCL)
  bool connected = false;
  i32 my_rank = 0;
  std::vector<i64> send_cnt, recv_cnt, send_off, recv_off;
  DBuf<i32> send_lids, send_peer, recv_lids, sendbuf, recvbuf;
  i64 nsend = 0, nrecv = 0;
  i64 nrouted_remote = 0;
  DBuf<i32> routed_remote, last_sent_remote;
  DBuf<uint8_t> changed;       // per local lid
#ifdef CHROMA_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  // NVLink peer-memory halo (connected worlds, free-running fast path): this
  // rank's colours live in an IPC-shared cudaMalloc region [ctrl | colours | flags];
  // owners store changed colours straight into their peers' ghost slots and raise
  // the slot's changed flag there.
  bool p2p = false;
  void* ipc_base = nullptr;                 // own region (cudaMalloc)
  std::vector<void*> peer_base;             // opened peer regions (nullptr for self)
  unsigned long long* my_ctrl = nullptr;    // [1] barrier arrivals
  uint8_t* my_flag = nullptr;               // loser flag per lid (raised by any rank's detection)
  DBuf<i32*> peer_colors;                   // device arrays [P]
  DBuf<uint8_t*> peer_flag;
  DBuf<unsigned long long*> peer_ctrl;
  DBuf<i64> rs_off;                         // owned lid -> send entries (CSR)
  DBuf<i32> rs_peer, rs_rlid, rs_last;      // per send entry: peer, remote lid, last sent
  unsigned long long bar_epoch = 0;
  std::vector<unsigned long long> route_pair_static;  // routes per (src,dst) pair
  // virtual worlds: owned lid -> routed index (-1: not routed), built lazily
  DBuf<i32> route_idx;
  DBuf<uint8_t> gflag;                      // loser flag per lid (virtual worlds)
  DBuf<i32> kill_lid, kill_rank;            // per ghost lid: owner's lid / owner process (-1: here)
  DBuf<i32> next_wl;                        // owned losers of the last detection
  DBuf<unsigned long long> nghost_dev;      // NGHOST on the device (round-0 changed list)
  // protocol scratch
  ColorScratch cs;
  DetectScratch det;
  HubScratch hub;
  DBuf<unsigned long long> stats;  // [0] conflicts [1] bytes [2] msgs [3..3+P) recolored
  DBuf<i32> deg_override;
  // schedule of the full owned worklist (computed on first use, -1 = not yet)
  DBuf<i32> level_wl;
  i64 level_n = -1;
  bool level_mode = false;
  int level_sq = 0;  // the schedule is of G (0) or of the square of that kind (sq_kind)
  ClusterPlan cplan;
  // the square of the local graph (square.cu), built on the first
  // distance-2 run of a bounded-degree world: 0 not yet, 1 built, -1 not applicable
  int sq_state = 0;
  int sq_kind = 0;  // 1 square, 2 partial square (two-hop only), 3 partial square of the owned rows
  DBuf<i64> sq_rowptr;
  DBuf<i32> sq_col;
  i64 sq_delta = 0;
  // device-side timing of the last run_distributed (CUDA events on `stream`)
  double t_total = 0, t_color_kernel = 0, t_color = 0, t_comm = 0, t_detect = 0;

  bool all_local() const { return rank_lo == 0 && rank_hi == P; }
  const RankMeta& meta(int rank) const {
    CHROMA_REQUIRE(rank >= rank_lo && rank < rank_hi, CHROMA_EVALUE, "rank not held by this world");
    return ranks[rank - rank_lo];
  }
};

World* world_create(i64 n, const i64* off, const i64* col, i32 P, const i32* owner, i32 gl, i32 lo,
                    i32 hi, int device);
void world_destroy(World* w);
void world_reset_exchange(World& w);
void world_exchange_local(World& w, bool changed_only, bool write_all);

// halo_p2p.cu: worklist-driven exchange (free-running distance-1 path)
void halo_route_index(World& w);
void halo_exchange_local_list(World& w, const i32* wl, const i64* nwl_dev, i64 nwl_max);
void halo_exchange_p2p(World& w, const i32* wl, const i64* nwl_dev, i64 nwl_max);
void halo_init_p2p_last(World& w);
void halo_next_worklist(World& w, i32* out, i64* n_out);  // flagged owned losers, ascending
KillRoute halo_kill_route(World& w);
void halo_barrier(World& w);  // all ranks' peer stores visible (no-op without NVLink peers)
// detection's owned losers -> 0 in every ghost copy (owners are the only writers)
void halo_broadcast_losers(World& w, const i32* list, const i64* n_dev, i64 n_max);
void halo_setup_p2p(World& w, const std::vector<i32>& send_lids_abs, const std::vector<i32>& send_peer,
                    const std::vector<i32>& recv_lids_abs);
void halo_release_p2p(World& w);

// Level schedule of a sorted worklist (padded to chunks; false if the DAG is too
// deep and narrow to benefit).  gs_levels.cu.
// sizes_out: the (unpadded) size of every level; min_width_override > 0 replaces the
// minimum average level width (CHROMA_LEVEL_MIN_WIDTH, default 2048).  chains: a
// run of consecutive adjacent ids inside one 1024-id block shares one level (only
// the cluster kernel, which scans runs, may consume such a schedule).
bool build_level_order(const i64* rowptr, const i32* col, i64 nv, const i32* wl, i64 nwl, DBuf<i32>& out,
                       i64& nout, cudaStream_t s, std::vector<i64>* sizes_out = nullptr,
                       i64 min_width_override = -1, bool chains = false);

// Level-synchronous Gauss-Seidel on one thread-block cluster (gs_cluster.cu): the
// plan is built once from a level schedule (bounded degree <= 32, colours of every
// vertex fit the cluster's shared memory as bytes); false if not applicable.
bool square_for(World& w, int dist, bool partial, int algo, bool owned_worklist, const i64*& crow, const i32*& ccol,
                int& cdist, i64& cdelta);
i64 cluster_max_vertices();
bool build_cluster_plan(const i64* rowptr, const i32* col, i64 nv, i64 max_deg, const i32* level_wl,
                        i64 level_n, const std::vector<i64>& level_sizes, ClusterPlan& plan, cudaStream_t s,
                        bool chains = false, bool zero_nonmembers = false);
void launch_gs_cluster(const ClusterPlan& plan, i32* val, const i32* old, cudaStream_t s);

// Round-robin chunk order over the virtual ranks of a world (rank_counts = owned
// vertices per rank, contiguous in wl).  gs_levels.cu.
bool build_rank_interleave(const i32* wl, const std::vector<i64>& rank_counts, DBuf<i32>& out, i64& nout,
                           cudaStream_t s);

// Colour every hub (global degree > T) of all ranks exactly, identically on every
// rank, into the owned hubs and the ghost copies of hubs; returns the number of hubs.
// Collective over the processes of a connected world.  hubs.cu.
i64 hub_precolor(World& w, i32 T);

// Colour the worklist of a CSR (absolute vertex ids).  `wl_sorted_unique` skips the
// device sort/dedupe for protocol worklists that are produced in order.
void color_csr(const i64* rowptr, const i32* col, i64 nv, i32* colors, const i32* wl_dev,
               const i64* nwl_dev, i64 nwl_max, bool wl_sorted_unique, int dist, bool partial,
               int algo, bool colors_nonneg, ColorScratch& S, cudaStream_t s,
               cudaEvent_t ev_k0 = nullptr, cudaEvent_t ev_k1 = nullptr);

}  // namespace chroma
