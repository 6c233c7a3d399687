// Exact Gauss-Seidel first fit (distance 1) for skewed graphs: chunked dataflow.
//
// Reference: chroma/localcolor.py:161-165 (_gauss_seidel over _forbidden_d1,
// 147-149) -- the worklist W is coloured in ascending local id, each vertex taking
// mex{ colours of its neighbours at that moment }: final colours of smaller
// worklist members, pre-call colours of larger ones, current colours of non-members.
//
// Round 1's id-ordered kernel waited on every smaller neighbour and stalled behind
// the hub rows (920 ms on C3, R-MAT scale 24).  Here W is cut into position chunks
// of B vertices, processed in order:
//   * first pass (throughput): every member v of the chunk scans the lower part of
//     its row once -- a lane for rows of <= 32 entries, 8 lanes up to 256, a warp
//     up to 4096, CTAs (32k-entry slices) beyond.  Neighbours outside the chunk and chunk members that are already
//     final form v's external colour set.  If no smaller chunk member is still open,
//     v is final at once: mex(external), ~90 % of the vertices.  Otherwise v stays
//     open and its external set is kept as a bitmap record (pool).
//   * dataflow (latency): each lane of the "resolver" threads walks its own slice
//     of chunk positions in ascending order and resolves the open vertex there (rows
//     of up to 4096 entries; a per-thread bitmap of 1024 colours in shared memory):
//     it walks the intra segment of the row (entries in [chunk start, v)), folds the
//     final colours into the external bitmap and spins on an entry that is still
//     open until its owner publishes it.  Open rows beyond 4096 entries (hubs) are
//     resolved by whole warps, each taking its share of the chunk's hubs in
//     ascending order.  A vertex only waits on smaller ids, whose resolvers only wait
//     on still smaller ids, so every wait ends; no resolver waits for another one
//     to finish unrelated work.
// Every vertex is evaluated once in the first pass and, if open, once more.
// Encoding inside the call: a member holds PENDING (-1) until final, then -(t + 2);
// non-members keep their colour (>= 0), so one load tells the cases apart.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace chroma {
namespace cg = cooperative_groups;
namespace {

constexpr int CF_THREADS = 1024;
constexpr int CF_WARPS = CF_THREADS / 32;
constexpr int CF_WORDS = 32;          // bitmap of colours 1..1024
constexpr i64 CF_TINY = 32;           // rows up to this length: one lane
constexpr i64 CF_HEAVY = 4096;        // rows longer than this: one CTA
constexpr int CF_HDR = 4;             // pool record: [k0, k1, nw, nopen | bitmap words | open lids]
constexpr int CF_OPEN = 128;          // open intra members listed per long row (more: walk the segment)
constexpr int CF_HUB_OPEN = 1024;     // ... per hub row
constexpr i64 CF_SLICE = 32768;       // a hub row is scanned by ceil(len / CF_SLICE) CTAs
constexpr u32 OPEN_WALK = 0xffffffffu;
constexpr unsigned FULLM = 0xffffffffu;
constexpr int CF_HUBW = 2;            // warps per CTA that resolve open hub rows

struct CfArgs {
  const i64* rowptr;
  const i32* col;
  i32* val;
  const i32* old;       // pre-call colours of members (nullptr: 0)
  const i32* wl;        // sorted unique worklist
  i64 nwl, chunk;
  bool upper_zero;      // every neighbour above a member contributes colour 0
  i32* big[3];          // first pass: warp rows / CTA row slices / group rows of the chunk
  int2* slice;          // per CTA item: (hub slot, slice index)
  // per hub row (slot): colour bitmap, [intra, nlt0, nltv, slices left, open count], open lids
  u32* hub_bm;
  int* hub_cnt;
  i32* hub_open;
  unsigned* hub_top;    // next free slot
  unsigned hub_cap;     // slots (more hubs than counted: overflow, the caller falls back)
  int hub_list;         // open members listed per hub row (<= CF_HUB_OPEN; more: walk)
  unsigned* cnt;        // [0..2] big counts (even chunks), [3..5] (odd chunks), [6] overflow
  i64 med;              // rows of CF_TINY < deg <= med: one 8-lane group (first pass)
  u32* pool;
  unsigned long long* pool_top;
  u32* desc;            // per vertex: pool offset of its record
  unsigned long long* trace;  // optional: (globaltimer, phase << 32 | count) per step
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// colour of neighbour u as seen by member v in the first pass; `open` for a smaller
// chunk member that is not final yet
__device__ __forceinline__ i32 colour_of(i32 x) { return x >= 0 ? x : -x - 2; }

__device__ __forceinline__ i32 nb_colour(const CfArgs& a, i32 u, i32 v, i32 s0, bool& open) {
  open = false;
  const i32 x = ld_relaxed_nb(a.val + u);
  if (x >= 0) return x;                      // non-member: current colour
  if (u > v) return a.old ? a.old[u] : 0;    // larger member: pre-call colour
  if (x == PENDING) {                        // smaller member of this chunk, open
    open = true;
    return 0;
  }
  return colour_of(x);                       // smaller member, final
}

__device__ __forceinline__ u32 pool_alloc(const CfArgs& a, int nw) {
  return (u32)atomicAdd(a.pool_top, (unsigned long long)(CF_HDR + nw));
}

__device__ __forceinline__ int words_for(i64 deg) {
  const i64 nw = (deg + 1) / 32 + 1;
  return nw > CF_WORDS ? CF_WORDS : (int)nw;
}

__device__ __forceinline__ void publish(const CfArgs& a, i32 v, i32 t) { st_relaxed(a.val + v, -(t + 2)); }

// ------------------------------------------------------------------ first pass
// a row of <= 32 entries by one lane (64-bit window: mex <= deg + 1 <= 33)
__device__ void first_lane(const CfArgs& a, i32 v, i32 s0) {
  const i64 rs = a.rowptr[v], re = a.rowptr[v + 1];
  unsigned long long m = 0;
  int intra = 0, nlt0 = 0, nltv = 0;
  bool above = false;
  for (i64 j = rs; j < re && !above; j += 8) {
    i32 us[8];
#pragma unroll
    for (int q = 0; q < 8; q++) us[q] = j + q < re ? a.col[j + q] : -1;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const i32 u = us[q];
      if (u < 0) continue;
      if (u > v && a.upper_zero) {
        above = true;
        continue;
      }
      bool open;
      const i32 c = nb_colour(a, u, v, s0, open);
      intra += open;
      nlt0 += u < s0;
      nltv += u < v;
      if (c >= 1 && c <= 64) m |= 1ull << (c - 1);
    }
  }
  const i32 t = __ffsll((long long)~m);
  if (intra == 0) {
    publish(a, v, t);
    return;
  }
  const u32 off = pool_alloc(a, 2);
  u32* r = a.pool + off;
  r[0] = (u32)nlt0;
  r[1] = (u32)nltv;
  r[2] = 2;
  r[3] = OPEN_WALK;  // a short row: the resolver walks its (<= 32-entry) segment
  r[4] = (u32)m;
  r[5] = (u32)(m >> 32);
  a.desc[v] = off;
}

struct RowScan {
  int intra, nlt0, nltv;
};
// a row scanned by `nthreads` cooperating threads (lanes gm of a warp, or a CTA when cta) into
// the shared bitmap bm; stops after the step that reached entries above v
__device__ void first_scan(const CfArgs& a, i32 v, i32 s0, int tid, int nthreads, bool cta, u32* bm,
                           RowScan& out, i32* olist, int* on, i64 rs = -1, i64 re = -1, unsigned gm = FULLM,
                           int cap = CF_OPEN) {
  if (rs < 0) {
    rs = a.rowptr[v];
    re = a.rowptr[v + 1];
  }
  int intra = 0, nlt0 = 0, nltv = 0;
  for (i64 j = rs; j < re; j += (i64)nthreads * 4) {
    i32 us[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const i64 jj = j + tid + (i64)q * nthreads;
      us[q] = jj < re ? a.col[jj] : -1;
    }
    bool above = false;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const i32 u = us[q];
      if (u < 0) continue;
      if (u > v && a.upper_zero) {
        above = true;
        continue;
      }
      bool open;
      const i32 c = nb_colour(a, u, v, s0, open);
      intra += open;
      nlt0 += u < s0;
      nltv += u < v;
      if (open) {  // list it (the resolver then waits on these entries only)
        const int k = atomicAdd(on, 1);
        if (k < cap) olist[k] = u;
      }
      if (c >= 1 && c <= CF_WORDS * 32) atomicOr(bm + ((c - 1) >> 5), 1u << ((c - 1) & 31));
    }
    const bool any = cta ? __syncthreads_or(above) : __any_sync(gm, above);
    if (any) break;
  }
  out = {intra, nlt0, nltv};
}

// first zero bit of bm[0..32) (colour, 1-based) by one warp; 0 if full
__device__ __forceinline__ i32 warp_mex(const u32* bm, int lane) {
  const u32 w = bm[lane];
  const unsigned nf = __ballot_sync(FULLM, w != FULLM);
  if (!nf) return 0;
  const int l = __ffs(nf) - 1;
  const u32 wl = __shfl_sync(FULLM, w, l);
  return l * 32 + __ffs(~wl);
}

// first zero bit of bm[0..32) by the G lanes gm of a warp (gl: lane in the group); 0 if full
template <int G>
__device__ __forceinline__ i32 group_mex(const u32* bm, int gl, unsigned gm) {
  constexpr int PER = 32 / G;
  int wi = 32;
#pragma unroll
  for (int k = PER - 1; k >= 0; k--)
    if (bm[gl * PER + k] != FULLM) wi = gl * PER + k;
  wi = (int)__reduce_min_sync(gm, (unsigned)wi);
  return wi == 32 ? 0 : wi * 32 + __ffs(~bm[wi]);
}

// finish a cooperative first pass (G lanes gm of a warp, led by lane `lead`)
template <int G>
__device__ void first_finish(const CfArgs& a, i32 v, const RowScan& r, const u32* bm, int gl, unsigned gm, int lead,
                             const i32* olist, int nopen, int cap = CF_OPEN) {
  const i32 t = group_mex<G>(bm, gl, gm);
  if (t == 0) {  // more than 1024 colours: publish anything (no waiter may hang), fall back
    if (gl == 0) {
      atomicOr(a.cnt + 6, 1u);
      publish(a, v, 1);
    }
    return;
  }
  if (r.intra == 0) {
    if (gl == 0) publish(a, v, t);
    return;
  }
  const int nw = words_for(a.rowptr[v + 1] - a.rowptr[v]);
  const bool listed = nopen <= cap;
  u32 off = 0;
  if (gl == 0) {
    off = pool_alloc(a, nw + (listed ? nopen : 0));
    u32* rec = a.pool + off;
    rec[0] = (u32)r.nlt0;
    rec[1] = (u32)r.nltv;
    rec[2] = (u32)nw;
    rec[3] = listed ? (u32)nopen : OPEN_WALK;
    a.desc[v] = off;
  }
  off = __shfl_sync(gm, off, lead);
  for (int w = gl; w < nw; w += G) a.pool[off + CF_HDR + w] = bm[w];
  if (listed)
    for (int k = gl; k < nopen; k += G) a.pool[off + CF_HDR + nw + k] = (u32)olist[k];
}

// ------------------------------------------------------------------ dataflow
__device__ __forceinline__ i32 wait_final(const CfArgs& a, i32 u) {
  i32 x = ld_relaxed(a.val + u);
  unsigned ns = 16;
  while (x == PENDING) {
    __nanosleep(ns);
    ns = ns < 128 ? ns * 2 : ns;
    x = ld_relaxed(a.val + u);
  }
  return x;
}

// open vertex v (row <= CF_HEAVY entries) resolved by one thread; lbm: this thread's
// 32-word column of the shared bitmap (stride CF_THREADS)
__device__ void resolve_lane(const CfArgs& a, i32 v, u32* lbm) {
  const u32* rec = a.pool + __ldcg(a.desc + v);
  const i64 rs = a.rowptr[v];
  const i64 k0 = rs + __ldcg(rec), k1 = rs + __ldcg(rec + 1);
  const int nw = (int)__ldcg(rec + 2);
  const u32 nopen = __ldcg(rec + 3);
#pragma unroll 4
  for (int w = 0; w < CF_WORDS; w++) lbm[w * CF_THREADS] = w < nw ? __ldcg(rec + CF_HDR + w) : 0u;
  const bool listed = nopen != OPEN_WALK && a.rowptr[v + 1] - rs > CF_TINY;
  if (a.trace && !listed && a.rowptr[v + 1] - rs > CF_TINY) {
    atomicAdd(a.trace + 8190, 1ull);
    atomicAdd(a.trace + 8191, (unsigned long long)(k1 - k0));
  }
  // listed members: 8 loads in flight, spin only on the ones still open
  for (u32 k = 0; listed && k < nopen; k += 8) {
    i32 us[8], xs[8];
#pragma unroll
    for (int q = 0; q < 8; q++) us[q] = k + q < nopen ? (i32)__ldcg(rec + CF_HDR + nw + k + q) : -1;
#pragma unroll
    for (int q = 0; q < 8; q++) xs[q] = us[q] >= 0 ? ld_relaxed(a.val + us[q]) : 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (us[q] < 0) continue;
      const i32 x = xs[q] == PENDING ? wait_final(a, us[q]) : xs[q];
      const i32 c = -x - 2;
      if (c >= 1 && c <= CF_WORDS * 32) lbm[((c - 1) >> 5) * CF_THREADS] |= 1u << ((c - 1) & 31);
    }
  }
  for (i64 j = listed ? k1 : k0; j < k1; j += 8) {
    i32 us[8], xs[8];
#pragma unroll
    for (int q = 0; q < 8; q++) us[q] = j + q < k1 ? a.col[j + q] : -1;
#pragma unroll
    for (int q = 0; q < 8; q++) xs[q] = us[q] >= 0 ? ld_relaxed(a.val + us[q]) : 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (us[q] < 0 || xs[q] >= 0) continue;  // non-members are in the external set
      const i32 x = xs[q] == PENDING ? wait_final(a, us[q]) : xs[q];
      const i32 c = -x - 2;
      if (c >= 1 && c <= CF_WORDS * 32) lbm[((c - 1) >> 5) * CF_THREADS] |= 1u << ((c - 1) & 31);
    }
  }
  i32 t = 0;
  for (int w = 0; w < CF_WORDS && !t; w++) {
    const u32 x = lbm[w * CF_THREADS];
    if (x != FULLM) t = w * 32 + __ffs(~x);
  }
  if (t == 0) {
    atomicOr(a.cnt + 6, 1u);
    t = 1;
  }
  publish(a, v, t);
}

// open long-row vertex v resolved by one warp
__device__ void resolve_warp(const CfArgs& a, i32 v, u32* bm, int lane) {
  const u32* rec = a.pool + __ldcg(a.desc + v);
  const i64 rs = a.rowptr[v];
  const i64 k0 = rs + __ldcg(rec), k1 = rs + __ldcg(rec + 1);
  const int nw = (int)__ldcg(rec + 2);
  const u32 nopen = __ldcg(rec + 3);
  bm[lane] = lane < nw ? __ldcg(rec + CF_HDR + lane) : 0u;
  __syncwarp();
  if (a.trace && lane == 0) {
    atomicAdd(a.trace + 8188, 1ull);
    if (nopen == OPEN_WALK) atomicAdd(a.trace + 8189, (unsigned long long)(k1 - k0));
  }
  if (nopen != OPEN_WALK) {
    // only the intra members that were open at the first pass can add colours
    for (u32 k = lane; k < nopen; k += 32 * 8) {
      i32 us[8], xs[8];
#pragma unroll
      for (int q = 0; q < 8; q++) us[q] = k + 32 * q < nopen ? (i32)__ldcg(rec + CF_HDR + nw + k + 32 * q) : -1;
#pragma unroll
      for (int q = 0; q < 8; q++) xs[q] = us[q] >= 0 ? ld_relaxed(a.val + us[q]) : 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (us[q] < 0) continue;
        const i32 x = xs[q] == PENDING ? wait_final(a, us[q]) : xs[q];
        const i32 c = -x - 2;
        if (c >= 1 && c <= CF_WORDS * 32) atomicOr(bm + ((c - 1) >> 5), 1u << ((c - 1) & 31));
      }
    }
    __syncwarp();
    const i32 t = warp_mex(bm, lane);
    if (lane == 0) {
      if (t == 0) atomicOr(a.cnt + 6, 1u);
      publish(a, v, t == 0 ? 1 : t);
    }
    __syncwarp();
    return;
  }
  for (i64 j = k0 + lane; j < k1; j += 32 * 8) {
    i32 us[8], xs[8];
#pragma unroll
    for (int q = 0; q < 8; q++) us[q] = j + 32 * q < k1 ? a.col[j + 32 * q] : -1;
#pragma unroll
    for (int q = 0; q < 8; q++) xs[q] = us[q] >= 0 ? ld_relaxed(a.val + us[q]) : 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (us[q] < 0 || xs[q] >= 0) continue;
      const i32 x = xs[q] == PENDING ? wait_final(a, us[q]) : xs[q];
      const i32 c = -x - 2;
      if (c >= 1 && c <= CF_WORDS * 32) atomicOr(bm + ((c - 1) >> 5), 1u << ((c - 1) & 31));
    }
  }
  __syncwarp();
  const i32 t = warp_mex(bm, lane);
  if (lane == 0) {
    if (t == 0) atomicOr(a.cnt + 6, 1u);
    publish(a, v, t == 0 ? 1 : t);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(CF_THREADS, 1) k_gs_chunked(CfArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ u32 lbm_all[];  // [CF_WORDS][CF_THREADS]: per-thread colour bitmaps
  __shared__ u32 wbm[CF_WARPS][CF_WORDS];
  __shared__ u32 cbm[CF_WORDS];
  __shared__ int cred[3][CF_WARPS];
  __shared__ i32 wlist[CF_WARPS][CF_OPEN];  // open intra members of a long row (first pass)
  __shared__ i32 clist[CF_HUB_OPEN];
  __shared__ int wlen[CF_WARPS], clen, glen[CF_WARPS * 4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u32* bm = wbm[wid];
  const i64 gw = (i64)blockIdx.x * CF_WARPS + wid, nwarps = (i64)gridDim.x * CF_WARPS;
  unsigned ntr = 0;
  auto tr = [&](unsigned phase, unsigned count) {
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && ntr < 4090) {
      a.trace[2 + 2 * ntr] = gtimer();
      a.trace[3 + 2 * ntr] = ((unsigned long long)phase << 32) | count;
      a.trace[0] = ++ntr;
    }
  };
  tr(0, 0);
  for (i64 a0 = 0; a0 < a.nwl; a0 += a.chunk) {
    // big-row counters alternate by chunk parity: the other pair is reset during
    // this chunk's dataflow, between barriers that order it after its last reader
    // (previous chunk) and before its next writer (next chunk)
    unsigned* const bc = a.cnt + (((a0 / a.chunk) & 1) ? 3 : 0);
    unsigned* const bc_next = a.cnt + (((a0 / a.chunk) & 1) ? 0 : 3);
    // first-pass (2) items are grabbed dynamically (rows differ widely in length):
    // [0] warp rows, [1] hub slices, [2] group rows (quads); same parity scheme
    unsigned* const gc = a.cnt + (((a0 / a.chunk) & 1) ? 11 : 8);
    unsigned* const gc_next = a.cnt + (((a0 / a.chunk) & 1) ? 8 : 11);
    const i64 a1 = a0 + a.chunk < a.nwl ? a0 + a.chunk : a.nwl;
    const i32 s0 = a.wl[a0];
    const i64 ngroups = (a1 - a0 + 31) / 32;
    // ---------------- first pass (1): lanes take short rows; longer rows are listed
    for (i64 g = gw; g < ngroups; g += nwarps) {
      const i64 p = a0 + g * 32 + lane;
      const i32 v = p < a1 ? a.wl[p] : -1;
      const i64 deg = v >= 0 ? a.rowptr[v + 1] - a.rowptr[v] : 0;
      if (v >= 0 && deg <= CF_TINY) first_lane(a, v, s0);
      {
        // warp rows (list 0) and group rows (list 2)
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const bool mine = v >= 0 && deg > CF_TINY && deg <= CF_HEAVY && (deg <= a.med) == (q == 1);
          const unsigned b = __ballot_sync(FULLM, mine);
          if (b) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(bc + 2 * q, (unsigned)__popc(b));
            base = __shfl_sync(FULLM, base, 0);
            if (mine) a.big[2 * q][base + __popc(b & ((1u << lane) - 1u))] = v;
          }
        }
      }
      if (v >= 0 && deg > CF_HEAVY) {  // a hub: one accumulator slot, one item per slice
        const int nsl = (int)((deg + CF_SLICE - 1) / CF_SLICE);
        const unsigned slot = atomicAdd(a.hub_top, 1u);
        if (slot >= a.hub_cap) {  // cannot happen with an exact count; never leave a waiter hanging
          atomicOr(a.cnt + 6, 1u);
          publish(a, v, 1);
          continue;
        }
        const unsigned base = atomicAdd(bc + 1, (unsigned)nsl);
        u32* hb = a.hub_bm + (i64)slot * CF_WORDS;
        for (int w = 0; w < CF_WORDS; w++) hb[w] = 0;
        int* hc = a.hub_cnt + (i64)slot * 8;
        hc[0] = hc[1] = hc[2] = 0;
        hc[3] = nsl;
        hc[4] = 0;
        for (int j = 0; j < nsl; j++) {
          a.big[1][base + j] = v;
          a.slice[base + j] = make_int2((int)slot, j);
        }
      }
    }
    grid.sync();
    tr(1, __ldcg(bc + 1));
    // ---------------- first pass (2): CTA rows, then warp rows
    {
      // lists and counts written by other SMs before the barrier: read at L2
      const unsigned nc = __ldcg(bc + 1), nwr = __ldcg(bc + 0);
      // hub rows: every slice by one CTA; partial results meet in the hub's slot and
      // the CTA that finishes the last slice finishes the row
      __shared__ int last;
      __shared__ unsigned item;
      for (;;) {
        if (threadIdx.x == 0) item = atomicAdd(gc + 1, 1u);
        __syncthreads();
        const unsigned h = item;
        if (h >= nc) break;
        const i32 vh = __ldcg(a.big[1] + h);
        const int2 it = __ldcg(a.slice + h);
        const i64 rs = a.rowptr[vh], re = a.rowptr[vh + 1];
        const i64 b0 = rs + (i64)it.y * CF_SLICE, b1 = b0 + CF_SLICE < re ? b0 + CF_SLICE : re;
        if (threadIdx.x < CF_WORDS) cbm[threadIdx.x] = 0;
        if (threadIdx.x == 0) clen = 0;
        __syncthreads();
        RowScan r;
        first_scan(a, vh, s0, threadIdx.x, CF_THREADS, true, cbm, r, clist, &clen, b0, b1, FULLM, a.hub_list);
        r.intra = __reduce_add_sync(FULLM, r.intra);
        r.nlt0 = __reduce_add_sync(FULLM, r.nlt0);
        r.nltv = __reduce_add_sync(FULLM, r.nltv);
        if (lane == 0) {
          cred[0][wid] = r.intra;
          cred[1][wid] = r.nlt0;
          cred[2][wid] = r.nltv;
        }
        __syncthreads();
        u32* hb = a.hub_bm + (i64)it.x * CF_WORDS;
        int* hc = a.hub_cnt + (i64)it.x * 8;
        i32* ho = a.hub_open + (i64)it.x * CF_HUB_OPEN;
        if (wid == 0) {
          RowScan t{cred[0][lane], cred[1][lane], cred[2][lane]};
          t.intra = __reduce_add_sync(FULLM, t.intra);
          t.nlt0 = __reduce_add_sync(FULLM, t.nlt0);
          t.nltv = __reduce_add_sync(FULLM, t.nltv);
          if (cbm[lane]) atomicOr(hb + lane, cbm[lane]);
          const int nl = clen < a.hub_list ? clen : a.hub_list;
          int base = 0;
          if (lane == 0) {
            atomicAdd(hc + 0, t.intra);
            atomicAdd(hc + 1, t.nlt0);
            atomicAdd(hc + 2, t.nltv);
            base = atomicAdd(hc + 4, clen);  // > CF_HUB_OPEN in total: the resolver walks the segment
          }
          base = __shfl_sync(FULLM, base, 0);
          for (int k = lane; k < nl && base + k < a.hub_list; k += 32) ho[base + k] = clist[k];
          __threadfence();
          __syncwarp();
          if (lane == 0) last = atomicSub(hc + 3, 1) == 1;
        }
        __syncthreads();
        if (last && wid == 0) {  // every slice is in: finish the row from the slot
          __threadfence();
          cbm[lane] = __ldcg(hb + lane);
          const int nopen = __ldcg(hc + 4);
          for (int k = lane; k < a.hub_list && k < nopen; k += 32) clist[k] = __ldcg(ho + k);
          __syncwarp();
          const RowScan t{__ldcg(hc + 0), __ldcg(hc + 1), __ldcg(hc + 2)};
          first_finish<32>(a, vh, t, cbm, lane, FULLM, 0, clist, nopen, a.hub_list);
        }
        __syncthreads();
      }
      for (;;) {
        unsigned h = 0;
        if (lane == 0) h = atomicAdd(gc + 0, 1u);
        h = __shfl_sync(FULLM, h, 0);
        if (h >= nwr) break;
        const i32 vl = __ldcg(a.big[0] + h);
        bm[lane] = 0;
        if (lane == 0) wlen[wid] = 0;
        __syncwarp();
        RowScan r;
        first_scan(a, vl, s0, lane, 32, false, bm, r, wlist[wid], &wlen[wid]);
        r.intra = __reduce_add_sync(FULLM, r.intra);
        r.nlt0 = __reduce_add_sync(FULLM, r.nlt0);
        r.nltv = __reduce_add_sync(FULLM, r.nltv);
        __syncwarp();
        first_finish<32>(a, vl, r, bm, lane, FULLM, 0, wlist[wid], wlen[wid]);
        __syncwarp();
      }
      // group rows: four per warp, 8 lanes each; bitmaps and open lists in the
      // resolvers' shared memory, which the first pass does not use
      {
        constexpr int G = 8, NG = 32 / G;
        const unsigned nmed = __ldcg(bc + 2);
        const int g = lane / G, gl = lane % G;
        const unsigned gm = ((1u << G) - 1u) << (g * G);
        const int slot = wid * NG + g;
        u32* gbm = lbm_all + slot * CF_WORDS;
        i32* glist = (i32*)lbm_all + CF_WARPS * NG * CF_WORDS + slot * CF_OPEN;
        for (;;) {
          unsigned h0 = 0;
          if (lane == 0) h0 = atomicAdd(gc + 2, (unsigned)NG);
          h0 = __shfl_sync(FULLM, h0, 0);
          if (h0 >= nmed) break;
          const i64 h = h0 + g;
          if (h < nmed) {
            const i32 vm = __ldcg(a.big[2] + h);
            for (int w = gl; w < CF_WORDS; w += G) gbm[w] = 0;
            if (gl == 0) glen[slot] = 0;
            __syncwarp(gm);
            RowScan r;
            first_scan(a, vm, s0, gl, G, false, gbm, r, glist, &glen[slot], -1, -1, gm);
            r.intra = __reduce_add_sync(gm, r.intra);
            r.nlt0 = __reduce_add_sync(gm, r.nlt0);
            r.nltv = __reduce_add_sync(gm, r.nltv);
            __syncwarp(gm);
            first_finish<G>(a, vm, r, gbm, gl, gm, g * G, glist, glen[slot]);
            __syncwarp(gm);
          }
        }
      }
    }
    grid.sync();
    tr(2, 0);
    // ---------------- dataflow over the open vertices
    if (blockIdx.x == 0 && threadIdx.x < 3) {
      bc_next[threadIdx.x] = 0;
      gc_next[threadIdx.x] = 0;
    }
    if (wid < CF_HUBW) {
      // hub warps: this warp's hubs of the chunk, ascending
      const unsigned nh = __ldcg(bc + 1);
      const i64 hw = (i64)blockIdx.x * CF_HUBW + wid, nhw = (i64)gridDim.x * CF_HUBW;
      i32 mine = INT32_MAX;  // lane k holds this warp's k-th hub
      int nm = 0;
      for (i64 h = hw; h < nh; h += nhw) {
        const i32 x = __ldcg(a.big[1] + h);
        if (lane == nm) mine = x;
        nm++;
      }
      if (nm > 32) {
        if (lane == 0) atomicOr(a.cnt + 6, 1u);  // cannot happen below 4,736 hubs per chunk
        nm = 32;
      }
      for (int k = 0; k < nm; k++) {
        const i32 h = __reduce_min_sync(FULLM, (unsigned)mine) ;
        if (mine == h) mine = INT32_MAX;
        if (ld_relaxed(a.val + h) == PENDING) resolve_warp(a, h, bm, lane);
      }
    } else {
      // every other thread walks its own positions, ascending
      const i64 tid = (i64)blockIdx.x * (CF_THREADS - 32 * CF_HUBW) + (threadIdx.x - 32 * CF_HUBW);
      const i64 nth = (i64)gridDim.x * (CF_THREADS - 32 * CF_HUBW);
      u32* lbm = lbm_all + threadIdx.x;
      for (i64 p = a0 + tid; p < a1; p += nth) {
        const i32 v = a.wl[p];
        if (ld_relaxed(a.val + v) != PENDING) continue;
        if (a.rowptr[v + 1] - a.rowptr[v] > CF_HEAVY) continue;  // a hub warp's
        resolve_lane(a, v, lbm);
      }
    }
    grid.sync();
    tr(3, 0);
  }
}

__global__ void k_count_hubs(const i32* wl, i64 n, const i64* rowptr, unsigned long long* out) {
  unsigned long long c = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    c += rowptr[v + 1] - rowptr[v] > CF_HEAVY;
  }
  c = __reduce_add_sync(FULLM, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_decode(const i32* wl, i64 n, i32* val) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    const i32 x = val[v];
    if (x <= -2) val[v] = -x - 2;
  }
}

}  // namespace

// Returns false (worklist entries back at PENDING) if a colour above 1024 appeared.
bool launch_gs_chunked(const GsLaunch& L, i64 nwl, bool upper_zero, ChunkedScratch& S, cudaStream_t s) {
  if (nwl <= 0) return true;
  const i64 nv = L.nv;
  const i32* wl = L.wl;
  if (!wl) {
    S.iota.reserve(nwl, s);
    launch_iota_i32(S.iota.p, nwl, (i32)L.wl_base, s);
    wl = S.iota.p;
  }
  static const i64 med = [] {
    const char* e = std::getenv("CHROMA_GS_MED");
    return e ? std::atoll(e) : (i64)256;
  }();
  static const i64 nchunks_env = [] {
    const char* e = std::getenv("CHROMA_GS_CHUNKS");
    return e ? std::atoll(e) : 0;
  }();
  const i64 nchunks = nchunks_env > 0 ? nchunks_env : 64;  // C3: 32 -> 12.00 ms, 64 -> 11.83, 128 -> 13.5
  i64 chunk = std::max<i64>((i64)1 << 15, (nwl + nchunks - 1) / nchunks);
  if (chunk > nwl) chunk = nwl;
  // hub rows (deg > CF_HEAVY) of the worklist, counted (cached for an iota worklist):
  // one accumulator slot and open list each; their slices (<= deg / CF_SLICE + 1 per
  // hub) are the chunk's CTA items
  i64 nnz_all = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nnz_all, L.rowptr + nv, sizeof(i64), cudaMemcpyDeviceToHost, s));
  // cacheable: an iota worklist, or the round-0 worklist of a world (every owned
  // vertex: the same set on every call of this scratch's world)
  const bool iota = L.wl == nullptr || upper_zero;
  i64 hubs = 0;
  if (iota && S.hub_key == L.rowptr && S.hub_key_nv == nv && S.hub_key_base == L.wl_base && S.hub_key_n == nwl &&
      S.hub_key_wl == L.wl) {
    hubs = S.hub_rows;
    CUDA_CHECK(cudaStreamSynchronize(s));
  } else {
    S.nhubs.reserve(1, s);
    S.nhubs.zero(s);
    k_count_hubs<<<grid_for(nwl, 256, num_sms() * 8), 256, 0, s>>>(wl, nwl, L.rowptr, S.nhubs.p);
    count_launch();
    unsigned long long h = 0;
    CUDA_CHECK(cudaMemcpyAsync(&h, S.nhubs.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    hubs = (i64)h;
    if (iota) {
      S.hub_key = L.rowptr;
      S.hub_key_nv = nv;
      S.hub_key_base = L.wl_base;
      S.hub_key_n = nwl;
      S.hub_key_wl = L.wl;
      S.hub_rows = hubs;
    }
  }
  const i64 hub_cap = hubs + 1;
  const i64 item_cap = chunk + nnz_all / CF_SLICE + 2;
  S.heavy.reserve(2 * chunk + item_cap, s);
  S.slice.reserve(item_cap, s);
  S.hub_bm.reserve(hub_cap * CF_WORDS, s);
  S.hub_cnt.reserve(hub_cap * 8, s);
  S.hub_open.reserve(hub_cap * CF_HUB_OPEN, s);
  S.hub_top.reserve(1, s);
  CUDA_CHECK(cudaMemsetAsync(S.hub_top.p, 0, sizeof(unsigned), s));
  S.cnt.reserve(16, s);
  S.cnt.zero(s);
  S.desc.reserve(nv, s);
  const i64 nnz = nnz_all;
  // bitmaps (<= deg/32 + 2 words), headers, and open lids (<= intra entries <= nnz)
  const i64 pool_words = nnz / 32 + (i64)(CF_HDR + 4) * nwl +
                         std::min<i64>(nnz, (i64)CF_OPEN * nwl + (i64)CF_HUB_OPEN * hubs) + 4096;
  S.pool.reserve(pool_words, s);
  S.pool_top.reserve(1, s);
  S.pool_top.zero(s);
  CfArgs a;
  a.rowptr = L.rowptr;
  a.col = L.col;
  a.val = L.val;
  a.old = L.old;
  a.wl = wl;
  a.nwl = nwl;
  a.chunk = chunk;
  a.upper_zero = upper_zero && L.old == nullptr;
  a.big[0] = S.heavy.p;
  a.big[1] = S.heavy.p + chunk;
  a.big[2] = S.heavy.p + chunk + item_cap;
  a.med = med;
  a.slice = S.slice.p;
  a.hub_bm = S.hub_bm.p;
  a.hub_cnt = S.hub_cnt.p;
  a.hub_open = S.hub_open.p;
  a.hub_top = S.hub_top.p;
  a.hub_cap = (unsigned)hub_cap;
  // measured (C3): long hub lists pay in later rounds (dense cores of recoloured hubs,
  // whose segments are long) and cost in round 0 (rows read up to the vertex only)
  static const int hub_list_env = [] {
    const char* e = std::getenv("CHROMA_GS_HUB_OPEN");
    return e ? std::max(1, std::min(CF_HUB_OPEN, std::atoi(e))) : 0;
  }();
  a.hub_list = hub_list_env ? hub_list_env : a.upper_zero ? CF_OPEN : CF_HUB_OPEN;
  a.cnt = S.cnt.p;
  a.pool = S.pool.p;
  a.pool_top = S.pool_top.p;
  a.desc = S.desc.p;
  const int grid = num_sms();
  void* args[] = {&a};
  // CHROMA_GS_CHUNK_TRACE (dev aid): per-phase device times of this call on stderr
  static const bool trace_on = std::getenv("CHROMA_GS_CHUNK_TRACE") != nullptr;
  DBuf<unsigned long long> tbuf;
  a.trace = nullptr;
  if (trace_on) {
    tbuf.alloc(8192, s);
    tbuf.zero(s);
    a.trace = tbuf.p;
  }
  const size_t dsmem = sizeof(u32) * CF_WORDS * CF_THREADS;
  static bool attr[64] = {};  // per device
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    CUDA_CHECK(cudaFuncSetAttribute((void*)k_gs_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  CUDA_CHECK(cudaLaunchCooperativeKernel((void*)k_gs_chunked, grid, CF_THREADS, args, dsmem, s));
  count_launch();
  if (trace_on) {
    std::vector<unsigned long long> h(8192);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), tbuf.p, sizeof(unsigned long long) * 8192, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    unsigned long long tp = h[2], ph_t[4] = {0, 0, 0, 0};
    for (unsigned long long i = 1; i < h[0]; i++) {
      ph_t[(unsigned)(h[3 + 2 * i] >> 32) & 3] += h[2 + 2 * i] - tp;
      tp = h[2 + 2 * i];
    }
    std::fprintf(stderr,
                 "[gs_chunked] nwl %lld chunk %lld: short rows %.1f us, long rows %.1f us, dataflow %.1f us; "
                 "lane walks %llu (%llu entries), open hubs %llu (walked %llu entries)\n",
                 (long long)nwl, (long long)chunk, ph_t[1] * 1e-3, ph_t[2] * 1e-3, ph_t[3] * 1e-3, h[8190], h[8191],
                 h[8188], h[8189]);
  }
  unsigned ovf = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ovf, S.cnt.p + 6, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (ovf) {
    launch_scatter_const(L.val, wl, L.nwl_dev, nwl, PENDING, s);
    return false;
  }
  k_decode<<<grid_for(nwl, 256, num_sms() * 8), 256, 0, s>>>(wl, nwl, L.val);
  count_launch();
  return true;
}

}  // namespace chroma
