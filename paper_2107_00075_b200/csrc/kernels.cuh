// Kernel launch interfaces shared by the host-side runtime (world/protocol/capi).
#pragma once
#include "common.cuh"

namespace chroma {

void count_launch(int k = 1);
void retain_pool_memory(int device);
i64 launch_count();

// ---------------------------------------------------------------- colouring
struct GsLaunch {
  const i64* rowptr = nullptr;
  const i32* col = nullptr;
  i32* val = nullptr;          // colours, worklist entries preset to PENDING
  const i32* old = nullptr;    // optional pre-call colours of worklist vertices
  const i32* wl = nullptr;     // optional sorted unique worklist
  i64 wl_base = 0;             // identity worklist base when wl == nullptr
  const i64* nwl_dev = nullptr;
  i64 nwl_max = 0;             // upper bound used to size the grid
  const i32* prio = nullptr;   // optional ordering key
  unsigned long long* ticket = nullptr;
  int dist = 1;
  bool partial = false;
  i64 nv = 0;                  // number of vertices (ids are < nv)
  bool level_mode = false;     // wl is a padded level schedule (gs_levels.cu), D1 only
};
void launch_gs(const GsLaunch& L, cudaStream_t s);
// Exact Gauss-Seidel (D1) by chunked fixed point (gs_chunked.cu); nwl = exact
// worklist length.  false: a colour above 1024 appeared, the worklist is back at
// PENDING and the caller takes launch_gs.
struct ChunkedScratch {
  DBuf<u32> pool, hub_bm;
  DBuf<i32> heavy, iota, flag, hub_cnt, hub_open;
  DBuf<int2> slice;
  DBuf<unsigned> hub_top;
  DBuf<unsigned> cnt;
  DBuf<u32> desc;
  DBuf<unsigned long long> pool_top;
  DBuf<unsigned long long> nhubs;
  // hub-row count of the last iota worklist (round 0 of a world): key and value
  const i64* hub_key = nullptr;
  const i32* hub_key_wl = nullptr;
  i64 hub_key_nv = -1, hub_key_base = -1, hub_key_n = -1, hub_rows = 0;
};
// upper_zero: every neighbour above a worklist member contributes colour 0 (round 0:
// nothing is coloured yet), so rows are read up to the vertex only.
bool launch_gs_chunked(const GsLaunch& L, i64 nwl, bool upper_zero, ChunkedScratch& S, cudaStream_t s);
bool launch_gs_d1(const GsLaunch& L, cudaStream_t s);  // false if not applicable

// Jacobi sweep pieces (chroma/localcolor.py:214-227, 292-303)
void launch_jacobi_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pending,
                           const i64* np_dev, i64 np_max, i32* prop, int dist, bool partial,
                           cudaStream_t s);
void launch_jacobi_losers(const i64* rowptr, const i32* col, i32* colors, const i32* pending,
                          const i64* np_dev, i64 np_max, const i32* prop, const uint8_t* in_round,
                          uint8_t* lose, int dist, bool partial, cudaStream_t s);

// Edge-based Jacobi sweep (Kernel.EDGE_BASED, distance 1): proposals into prop, the
// commit, and losers into lose, edge-parallel over the pending rows.
// the square G^2 (partial: two-hop only) over the rows with want[v] (square.cu);
// false if a row is too long or the rows exceed max_entries
bool build_square(const i64* rowptr, const i32* col, i64 nv, i64 delta, bool partial, i64 max_entries,
                  const uint8_t* want, DBuf<i64>& rowptr2, DBuf<i32>& col2, i64& maxdeg, cudaStream_t s);

// incremental Jacobi state (jacobi_inc.cu)
struct JacobiIncScratch {
  DBuf<uint8_t> pendf, hlose;
  DBuf<i32> hslot, hv, llen, nb, hprop;
  DBuf<i32> act[4];  // active slots: [2 * class + parity], class 0 warp, 1 CTA
  DBuf<u32> fb;
  DBuf<i64> loff, len64;
  DBuf<unsigned long long> cnt;  // [0] heavy slots, [1] overflow, [2 + 2 * class + parity] active counts
  i64 nheavy = 0;
  int par = 0;
  bool on = false;
};
bool jacobi_inc_init(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, i64 np, i64 nv,
                     JacobiIncScratch& S, cudaStream_t s);
void jacobi_inc_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, const i64* np_dev,
                        i64 np, i32* prop, JacobiIncScratch& S, cudaStream_t s);
void jacobi_inc_losers(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, const i64* np_dev,
                       i64 np, const uint8_t* in_round, uint8_t* lose, JacobiIncScratch& S, cudaStream_t s);
void jacobi_inc_update(const i32* colors, const i32* pend, const i64* np_dev, i64 np, const uint8_t* lose,
                       JacobiIncScratch& S, cudaStream_t s);
const unsigned* jacobi_inc_overflow_dev(const JacobiIncScratch& S);

struct EbScratch {
  DBuf<i64> len, eoff, np;
  DBuf<u32> mask;
  DBuf<unsigned long long> left;
};
void launch_jacobi_eb(const i64* rowptr, const i32* col, i32* colors, const i32* pending, i64 np, i32* prop,
                      const uint8_t* in_round, uint8_t* lose, EbScratch& S, cudaStream_t s);

// Free-running speculative colouring (deterministic=False, algorithm="free").
// Pending vertices are kept in light (warp per vertex), heavy (CTA per vertex) and
// tiny (8 lanes per vertex) lists, double-buffered by parity p; cnt[3p + {0,1,2}]
// are the light / heavy / tiny lengths.
struct FreeLists {
  i32* light[2];
  i32* heavy[2];
  i32* tiny[2];
  i64* cnt;  // [6]
};
void launch_free_split(const i32* wl, const i64* n_dev, i64 n_max, const i64* rowptr, i64 tiny_deg, i64 heavy_deg,
                       FreeLists& f, int p, cudaStream_t s);
// colour lists[p] (rank_cap > 0: snapshot rank-offset first fit, skipping up to
// rank_cap free colours), resolve, losers -> lists[p^1]; nmax = host upper bounds
// of the three lengths
void launch_free_iteration(const i64* rowptr, const i32* col, i32* colors, FreeLists& f, int p, const i64* nmax,
                           int rank_cap, int dist, bool partial, cudaStream_t s);
struct FreeWaveScratch {
  DBuf<u32> F, A;
  DBuf<int> ovf;
  DBuf<unsigned> bar;
  DBuf<u64> dbg;
  DBuf<u64> keys;
};
// Exact wave colouring of the heavy list (sorted in place); vertices whose colour
// would exceed the heavy mask are appended to light[*nlight].
void launch_free_heavy(const i64* rowptr, const i32* col, i32* colors, i32* heavy, i64 n, i32* light,
                       i64* nlight, int dist, bool partial, FreeWaveScratch& ws, cudaStream_t s);
void launch_free_split(const i32* wl, const i64* n_dev, i64 n_max, const i64* rowptr, i64 heavy_deg, FreeLists& f,
                       int p, cudaStream_t s);
// colour lists[p] (rank_cap > 0: snapshot rank-offset first fit, skipping up to
// rank_cap free colours), resolve, losers -> lists[p^1]
void launch_free_iteration(const i64* rowptr, const i32* col, i32* colors, FreeLists& f, int p, i64 nlight_max,
                           i64 nheavy_max, int rank_cap, int dist, bool partial, cudaStream_t s);

// Net-centric free-running D2/PD2 (color_net.cu): worklist colours must be 0 on entry.
// false: a colour above 256 was needed (worklist back at 0, caller falls back).
struct NetScratch {
  DBuf<unsigned long long> mask, cnt;
  DBuf<uint8_t> pend;
  DBuf<i32> wl[2];
};
bool launch_free_net(const i64* rowptr, const i32* col, i64 nv, i32* colors, const i32* wl, i64 nwl, bool partial,
                     NetScratch& S, cudaStream_t s);
i64 worklist_max_degree(const i32* wl, i64 n, const i64* rowptr, NetScratch& S, cudaStream_t s);

// ---------------------------------------------------------------- utilities
void launch_fill_i32(i32* p, i64 n, i32 v, cudaStream_t s);
void launch_iota_i32(i32* p, i64 n, i32 base, cudaStream_t s);
void launch_scatter_const(i32* val, const i32* idx, const i64* n_dev, i64 n_max, i32 v, cudaStream_t s);
void launch_scatter_from(i32* dst, const i32* src, const i32* idx, const i64* n_dev, i64 n_max,
                         cudaStream_t s);
void launch_scatter_idx_values(i32* dst, const i32* idx, const i32* values, const i64* n_dev,
                               i64 n_max, cudaStream_t s);
void launch_clamp_nonneg(i32* dst, const i32* src, i64 n, cudaStream_t s);
// ordered compaction of indices i in [0,n) with flag[i] != 0; count -> *n_out (device)
void select_flagged(const uint8_t* flags, i64 n, i32* out, i64* n_out, cudaStream_t s);
// same, emitting base + i
void select_flagged_base(const uint8_t* flags, i64 n, i32 base, i32* out, i64* n_out, cudaStream_t s);
void select_flagged_values(const i32* values, const uint8_t* flags, i64 n, i32* out, i64* n_out,
                           cudaStream_t s);
void exclusive_scan_i64(const i64* in, i64* out, i64 n, cudaStream_t s);
i64 unique_u64(const u64* in, i64 n, u64* out, cudaStream_t s);  // sorted input; returns count
// host -> device through the pinned staging ring (upload.cu); large arrays only
bool staged_upload_wanted(i64 bytes);
void upload_narrow_host(const i64* src, i64 k, i64 n, i32* out, cudaStream_t s, const char* what);
void upload_bytes_host(const void* src, i64 bytes, void* out, cudaStream_t s);
// DBuf::upload for large host arrays (staged when that pays)
template <typename T>
void upload_large(DBuf<T>& b, const T* h, i64 count, cudaStream_t s) {
  const i64 bytes = (i64)sizeof(T) * count;
  if (!staged_upload_wanted(bytes)) {
    b.upload(h, count, s);
    return;
  }
  b.alloc(count, s);
  upload_bytes_host(h, bytes, b.p, s);
}
void narrow_ids_checked(const i64* src, i64 k, i64 n, bool src_on_device, i32* out, cudaStream_t s,
                        const char* what);
void sort_i32(i32* keys, i64 n, cudaStream_t s);  // ascending, in place (non-negative keys)
void sort_u64(u64* keys, i64 n, cudaStream_t s);  // ascending, in place

// ---------------------------------------------------------------- detection
struct DetectArgs {
  const i64* rowptr;
  const i32* col;
  i32* colors;
  const i64* gids;
  const i32* deg;
  const i32* rows;    // detection rows: ghost lids (D1) / boundary_d2 lids (D2)
  i64 nrows;
  int dist;
  bool partial;
  bool recolor_degrees;
  bool sequential;    // exact replay of the reference's in-place scan (F5)
  bool incremental = false;  // scan only rows near vertices whose colour changed since
                             // the previous incremental call (S.prev)
  const uint8_t* owned_flag = nullptr;  // D1 free-running fast path: pairs with a ghost end
};
struct DetectScratch {
  DBuf<i64> cnt, off;
  DBuf<int2> ev;
  DBuf<uint8_t> fired;
  DBuf<i32> kill;
  DBuf<unsigned long long> kill64;  // grid resolve: (sweep tag << 32 | event) per vertex
  DBuf<unsigned long long> result;  // [0] conflicts
  DBuf<i64> total;
  // incremental mode: colours at the end of the previous detection, row marks
  DBuf<i32> prev, arows;
  DBuf<uint8_t> mark;
  DBuf<i64> narows;
  DBuf<i32> chl, chh;  // changed vertices, light / heavy rows (free-running D1)
  DBuf<u64> keys, ukeys;  // keyed event emission (sequential D1)
  DBuf<unsigned long long> nch;
  bool prev_valid = false;
};
// Free-running detection around explicit changed-vertex lists (device counts).
// Every pair with one owned end, one ghost end and equal non-zero colours
// uncolours its loser at the loser's owner -- locally, or through KillRoute for a
// ghost: the owner's lid in this process's colour array (virtual ranks, peer =
// -1) or in peer `owner_rank`'s NVLink-mapped array -- and raises the owner's
// loser flag.  Adds the number of vertices uncoloured to *conflicts.
struct FreeList {
  const i32* ids;
  const unsigned long long* n_dev;
  i64 cap;
};
struct KillRoute {
  const i32* owner_lid = nullptr;    // per lid: owner's lid of a ghost, -1 for owned
  const i32* owner_rank = nullptr;   // per lid: owner process rank (NVLink), -1 = this array
  i32* const* peer_colors = nullptr;
  uint8_t* const* peer_flag = nullptr;
  uint8_t* flags = nullptr;          // this process's loser flags (per lid)
};
void run_detect_free_lists(const DetectArgs& A, i64 nv, const FreeList* lists, int nlists, const KillRoute& kr,
                           DetectScratch& S, unsigned long long* conflicts, cudaStream_t s);
// Adds the number of conflicts to *conflicts_dev (device, unsigned long long).
void run_detect(const DetectArgs& a, i64 num_vertices, DetectScratch& S,
                unsigned long long* conflicts_dev, cudaStream_t s);

// ---------------------------------------------------------------- exchange (device copy)
void launch_exchange_local(const i32* routed, i64 nrouted, const i64* st_off, const i32* st_dst,
                           const i32* st_pair, i32* colors, i32* last_sent, bool changed_only,
                           bool write_all, unsigned long long* pair_cnt, i64 npairs, cudaStream_t s);
void launch_pair_stats(unsigned long long* pair_cnt, i64 npairs, unsigned long long* stats2,
                       cudaStream_t s);

// ---------------------------------------------------------------- verification
struct VerifyResult {
  i64 total;
};
i64 run_verify(const i64* rowptr, const i32* col, i64 n, const i32* colors, const uint8_t* mask,
               int mode, i64* rows_host, i64 cap, cudaStream_t s);
void run_color_stats(const i32* colors, i64 n, i64* num_colors, i64* max_color, i64* hist_host,
                     i64 hist_cap, cudaStream_t s);

}  // namespace chroma
