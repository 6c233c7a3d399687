// Gauss-Seidel first fit, distance 1, ascending local-id order: the "lite" dataflow
// kernel used for deterministic D1/D1-2GL colouring and serial_greedy().
//
// Reference: chroma/localcolor.py:161-165 (_gauss_seidel over _forbidden_d1,
// 147-149) and 120-133 (serial_greedy).  With ids as keys and rows sorted by id
// (chroma/graph.py:40-56, chroma/runtime.py:201), the vertices v has to wait for
// are exactly the worklist members of the row prefix below v, so no neighbourhood
// pre-scan is needed when a chunk is claimed:
//   * claim: each lane binary-searches its row for the split points kfirst (first
//     vertex of the chunk) and v -> external prefix [rs,p0), in-chunk range [p0,p1);
//     in-chunk worklist members become a lane mask; the sentinel is the largest
//     external candidate (the entry just below kfirst);
//   * wait: a lane polls its sentinel (one load); when it is committed the lane reads
//     its whole row in batches of independent loads -- if an external worklist member
//     is still PENDING the largest such becomes the new sentinel, otherwise the same
//     pass has built the 256-colour forbidden mask of every settled neighbour
//     (later worklist members still hold their pre-call colour);
//   * commit: in lane order through the in-chunk mask (colours shared in smem),
//     first free bit, relaxed store of the colour -- the value is the ready flag.
// Claims are cheap, so a chunk claimed late on the critical path costs a few memory
// round trips instead of a full neighbourhood walk (the bound of color_gs.cu).
#include <cstdlib>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr int WORDS = 8;
constexpr int FAST = 32 * WORDS;
constexpr int WARPS = 4;
constexpr int BATCH = 8;                 // independent loads per lane per scan step
constexpr int PL = 16;                   // per-lane list of pending external dependencies
constexpr i64 HEAVY = 256;               // rows longer than this are scanned by the warp
constexpr unsigned NS_MAX = 256;
constexpr unsigned FULL = 0xffffffffu;

struct D1Args {
  const i64* rowptr;
  const i32* col;
  i32* val;
  const i32* old;
  const i32* wl;
  i64 wl_base;
  const i64* nwl;
  unsigned long long* ticket;
  bool level_mode;  // wl is a level schedule (gs_levels.cu): no in-chunk dependencies,
                    // -1 entries pad levels to whole chunks
  bool poll_all;    // poll the whole pending list instead of the sentinel
};

struct D1Smem {
  i32 v[32];
  i32 ccol[32];
  i32 plist[32][PL];
};

__device__ __forceinline__ int first_free(const u32 (&m)[WORDS]) {
#pragma unroll
  for (int w = 0; w < WORDS; w++)
    if (m[w] != FULL) return w * 32 + __ffs(~m[w]);
  return 0;
}

// first index in [lo, hi) with col[i] >= x (rows are sorted)
__device__ __forceinline__ i64 lower_bound(const i32* col, i64 lo, i64 hi, i32 x) {
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (col[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Scan entries [b, e) of a row: fold settled colours into m, count external PENDING
// entries (< kfirst) and remember the largest one.  Entries in [kfirst, kv) are
// in-chunk (handled through the lane mask) and skipped.
__device__ __forceinline__ void scan_row(const D1Args& a, i64 b, i64 e, int step, i32 kfirst, i32 kv,
                                         u32 (&m)[WORDS], int& pend, i32& sentinel, i32* list) {
  for (i64 i = b; i < e; i += (i64)BATCH * step) {
    i32 x[BATCH], c[BATCH];
#pragma unroll
    for (int k = 0; k < BATCH; k++) {
      const i64 j = i + (i64)k * step;
      x[k] = j < e ? a.col[j] : -1;
    }
#pragma unroll
    for (int k = 0; k < BATCH; k++) c[k] = x[k] >= 0 ? ld_relaxed(a.val + x[k]) : 0;
#pragma unroll
    for (int k = 0; k < BATCH; k++) {
      if (x[k] < 0) continue;
      i32 cc = c[k];
      if (cc == PENDING) {
        if (x[k] < kfirst) {
          if (list && pend < PL) list[pend] = x[k];
          pend++;
          sentinel = x[k] > sentinel ? x[k] : sentinel;
          continue;
        }
        if (x[k] < kv) continue;          // in-chunk predecessor: colour comes from smem
        cc = a.old ? a.old[x[k]] : 0;     // later worklist vertex: pre-call colour
      }
      if (cc > 0 && cc <= FAST) m[(cc - 1) >> 5] |= 1u << ((cc - 1) & 31);
    }
  }
}

__global__ void __launch_bounds__(WARPS * 32) gs_d1_kernel(D1Args a) {
  __shared__ D1Smem smem[WARPS];
  D1Smem& sm = smem[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const i64 nwl = *a.nwl;
  const i64 nchunks = (nwl + 31) >> 5;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    const i64 chunk = (i64)__shfl_sync(FULL, t, 0);
    if (chunk >= nchunks) break;
    const i64 idx = chunk * 32 + lane;
    i32 v = idx < nwl ? (a.wl ? a.wl[idx] : (i32)(a.wl_base + idx)) : -1;
    const bool act = v >= 0;
    if (!act) v = INT32_MAX;
    sm.v[lane] = v;
    // level schedule: every smaller neighbour is external (claimed in an earlier chunk)
    const i32 kfirst = a.level_mode ? v : __shfl_sync(FULL, v, 0);
    const i64 rs = act ? a.rowptr[v] : 0, re = act ? a.rowptr[v + 1] : 0;
    const bool heavy = act && re - rs > HEAVY;
    i64 p0 = rs, p1 = rs;
    u32 dep = 0;
    if (act && !heavy) {
      p0 = lower_bound(a.col, rs, re, kfirst);
      p1 = lower_bound(a.col, p0, re, v);
    }
    __syncwarp();
    // in-chunk predecessors: worklist members of [kfirst, v) are chunk lanes
    if (act && !heavy && !a.level_mode) {
      for (i64 i = p0; i < p1; i++) {
        const i32 u = a.col[i];
        int lo = 0;  // lane holding u (sm.v is ascending; inactive lanes hold INT32_MAX)
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1)
          if (sm.v[lo + s] <= u) lo += s;
        if (sm.v[lo] == u) dep |= 1u << lo;
      }
    }
    // heavy rows: the warp computes splits and the in-chunk mask cooperatively
    u32 hv = __ballot_sync(FULL, heavy && !a.level_mode);
    while (hv) {
      const int l = __ffs(hv) - 1;
      hv &= hv - 1;
      const i32 vl = sm.v[l];
      const i64 rsl = a.rowptr[vl], rel = a.rowptr[vl + 1];
      u32 dl = 0;
      for (i64 i = rsl + lane; i < rel; i += 32) {
        const i32 u = a.col[i];
        if (u >= kfirst && u < vl) {
          int lo = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1)
            if (sm.v[lo + s] <= u) lo += s;
          if (sm.v[lo] == u) dl |= 1u << lo;
        }
      }
      dl = __reduce_or_sync(FULL, dl);
      if (lane == l) dep = dl;
    }
    // state: 0 waiting on external, 1 mask built (waiting on in-chunk), 2 committed
    int state = act ? 0 : 2;
    i32 sentinel = -1;
    if (act && !heavy && p0 > rs) sentinel = a.col[p0 - 1];
    u32 m[WORDS];
#pragma unroll
    for (int w = 0; w < WORDS; w++) m[w] = 0;
    bool need = act;  // first pass: scan immediately (dependencies may be settled)
    int npend = 0;    // listed pending dependencies (> PL: overflow, rescan the row)
    u32 mlist[WORDS]; // colours folded by list re-checks since the last full scan
#pragma unroll
    for (int w = 0; w < WORDS; w++) mlist[w] = 0;
    unsigned ns = 32;
    for (;;) {
      // ---- scan rows whose sentinel resolved (or never had one)
      if (state == 0 && !heavy && need) {
        if (npend > 0 && npend <= PL) {
          // re-check only the listed dependencies: one batch of independent loads
          i32 xs[PL], cs[PL];
#pragma unroll
          for (int k = 0; k < PL; k++) {
            xs[k] = k < npend ? sm.plist[lane][k] : 0;
            cs[k] = k < npend ? ld_relaxed(a.val + xs[k]) : 0;
          }
          int w = 0;
          i32 sent = -1;
#pragma unroll
          for (int k = 0; k < PL; k++) {
            if (k < npend) {
              if (cs[k] == PENDING) {
                sm.plist[lane][w++] = xs[k];
                sent = xs[k] > sent ? xs[k] : sent;
              } else if (cs[k] > 0 && cs[k] <= FAST) {
                mlist[(cs[k] - 1) >> 5] |= 1u << ((cs[k] - 1) & 31);
              }
            }
          }
          npend = w;
          sentinel = sent;
          if (w == 0) {
            state = 1;
#pragma unroll
            for (int ww = 0; ww < WORDS; ww++) m[ww] |= mlist[ww];
          }
        } else {
#pragma unroll
          for (int w = 0; w < WORDS; w++) m[w] = 0;
          int pend = 0;
          i32 sent = -1;
          scan_row(a, rs, re, 1, kfirst, v, m, pend, sent, sm.plist[lane]);
          npend = pend;
#pragma unroll
          for (int w = 0; w < WORDS; w++) mlist[w] = 0;
          if (pend == 0) state = 1;
          else sentinel = sent;
        }
      }
      u32 hs = __ballot_sync(FULL, state == 0 && heavy && need);
      while (hs) {
        const int l = __ffs(hs) - 1;
        hs &= hs - 1;
        const i32 vl = sm.v[l];
        u32 mm[WORDS];
#pragma unroll
        for (int w = 0; w < WORDS; w++) mm[w] = 0;
        int pend = 0;
        i32 sent = -1;
        scan_row(a, a.rowptr[vl] + lane, a.rowptr[vl + 1], 32, a.level_mode ? vl : kfirst, vl, mm, pend, sent,
                 nullptr);
        pend = __reduce_add_sync(FULL, pend);
        sent = __reduce_max_sync(FULL, sent);
#pragma unroll
        for (int w = 0; w < WORDS; w++) mm[w] = __reduce_or_sync(FULL, mm[w]);
        if (lane == l) {
          if (pend == 0) {
            state = 1;
#pragma unroll
            for (int w = 0; w < WORDS; w++) m[w] = mm[w];
          } else {
            sentinel = sent;
          }
        }
      }
      // ---- commit in-chunk chains
      u32 done = __ballot_sync(FULL, state == 2);
      for (;;) {
        const bool ready = state == 1 && (dep & ~done) == 0;
        int r = 1;
        if (ready) {
          u32 mm[WORDS];
#pragma unroll
          for (int w = 0; w < WORDS; w++) mm[w] = m[w];
          for (u32 bits = dep; bits; bits &= bits - 1) {
            const i32 c = sm.ccol[__ffs(bits) - 1];
            if (c <= FAST) mm[(c - 1) >> 5] |= 1u << ((c - 1) & 31);
          }
          r = first_free(mm);
          if (r) {
            st_relaxed(a.val + v, r);
            sm.ccol[lane] = r;
            state = 2;
          }
        }
        u32 slow = __ballot_sync(FULL, ready && r == 0);
        while (slow) {  // > FAST colours: warp window walk over the row, all settled now
          const int l = __ffs(slow) - 1;
          slow &= slow - 1;
          const i32 vl = sm.v[l];
          const i64 rsl = a.rowptr[vl], rel = a.rowptr[vl + 1];
          i32 col_l = 0;
          for (i32 base = FAST + 1;; base += FAST) {
            u32 mm[WORDS];
#pragma unroll
            for (int w = 0; w < WORDS; w++) mm[w] = 0;
            for (i64 i = rsl + lane; i < rel; i += 32) {
              const i32 x = a.col[i];
              i32 c = ld_relaxed(a.val + x);
              if (c == PENDING) c = (x > vl && a.old) ? a.old[x] : 0;
              const i32 o = c - base;
              if (o >= 0 && o < FAST) mm[o >> 5] |= 1u << (o & 31);
            }
            int rr = 0;
#pragma unroll
            for (int w = 0; w < WORDS; w++) {
              const u32 mw = __reduce_or_sync(FULL, mm[w]);
              if (!rr && mw != FULL) rr = w * 32 + __ffs(~mw);
            }
            if (rr) {
              col_l = base + rr - 1;
              break;
            }
          }
          if (lane == l) {
            st_relaxed(a.val + v, col_l);
            sm.ccol[lane] = col_l;
            state = 2;
          }
        }
        __syncwarp();
        const u32 nd = __ballot_sync(FULL, state == 2);
        if (nd == done) break;
        done = nd;
      }
      if (done == FULL) break;
      // ---- poll sentinels (one load per waiting lane)
      need = false;
      if (state == 0) {
        // level schedule: re-check the whole (short) list each poll -- one batch of
        // loads -- rather than waiting on the sentinel first: deps of one level
        // commit in any order
        if (a.poll_all && !heavy && npend > 0 && npend <= PL) need = true;
        else need = sentinel < 0 || ld_relaxed(a.val + sentinel) != PENDING;
      }
      if (__any_sync(FULL, need)) {
        ns = 32;
      } else {
        __nanosleep(ns);
        ns = ns < NS_MAX ? ns * 2 : ns;
      }
    }
    __syncwarp();
  }
}

}  // namespace

bool launch_gs_d1(const GsLaunch& L, cudaStream_t s) {
  if (L.dist != 1 || L.prio != nullptr) return false;
  D1Args a;
  a.rowptr = L.rowptr;
  a.col = L.col;
  a.val = L.val;
  a.old = L.old;
  a.wl = L.wl;
  a.wl_base = L.wl_base;
  a.nwl = L.nwl_dev;
  a.ticket = L.ticket;
  a.level_mode = L.level_mode;
  a.poll_all = L.level_mode;
  CUDA_CHECK(cudaMemsetAsync(L.ticket, 0, sizeof(unsigned long long), s));
  const i64 nchunks = (L.nwl_max + 31) / 32;
  static const int bps_env = std::getenv("CHROMA_GS_BPS") ? std::atoi(std::getenv("CHROMA_GS_BPS")) : 0;
  // id order needs a wide claim window (the wavefront spans the id range); a level
  // schedule needs only a few levels in flight, and fewer pollers keep the
  // critical-path warps issuing
  const int bps = bps_env > 0 ? bps_env : (L.level_mode ? 2 : 16);
  int grid = (int)std::min<i64>((nchunks + WARPS - 1) / WARPS, (i64)num_sms() * bps);
  if (grid < 1) grid = 1;
  gs_d1_kernel<<<grid, WARPS * 32, 0, s>>>(a);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
  return true;
}

}  // namespace chroma
