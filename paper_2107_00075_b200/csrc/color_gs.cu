// Gauss-Seidel first-fit colouring as an ordered-dataflow persistent kernel.
//
// Reference semantics (deterministic=True): chroma/localcolor.py:161-165 colours
// the worklist in ascending local-id order, each vertex taking the smallest
// positive colour absent from its forbidden set (D1: N(v), chroma/localcolor.py:
// 147-149; D2: N(v) u N2(v), PD2: N2(v), chroma/localcolor.py:136-158), with
// every earlier commit visible.  The same result is produced here without a
// sequential loop: vertex v only has to wait for the worklist vertices with a
// smaller key inside its forbidden set (the DAG-depth critical path, F6).
//
// Execution model
//   * the sorted worklist is cut into 32-vertex chunks; warps of a persistent
//     grid take chunks from an atomic ticket in ascending order, so every chunk
//     a warp waits on has already been claimed by a running warp (deadlock-free);
//   * phase A walks the chunk's whole neighbourhood edge-parallel (D1: the 32
//     rows flattened by a warp prefix sum; D2: a second flattening level over
//     the middles' rows), coalesced on col[], folding committed colours into a
//     256-colour shared-memory bitmask per vertex.  Not-yet-committed earlier
//     vertices go to a per-warp dependency queue; same-chunk dependencies become
//     a 32-bit lane mask;
//   * phase B is a per-lane dataflow loop: a lane commits as soon as its own queue
//     entries resolved and its in-chunk predecessors committed (so a chunk that
//     straddles independent regions never serialises them), publishing with a
//     relaxed store -- the colour value itself is the ready flag (PENDING = -1);
//     idle polling backs off with __nanosleep;
//   * vertices whose first 256 colours are all forbidden take a warp-cooperative
//     rescan window by window (the reference's 64-colour window walk,
//     chroma/localcolor.py:64-112, generalised).
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace chroma {

namespace {

constexpr int WORDS = 8;                 // 8 x 32 bits = colours 1..256 in the fast path
constexpr int FAST_COLORS = 32 * WORDS;
constexpr int WARPS = 4;
constexpr i64 HEAVY = 64;                // forbidden sets larger than this are rescanned by the warp
constexpr unsigned NS_MAX = 512;         // idle polling back-off cap (ns)
constexpr int PL = 24;                   // per-lane list of pending earlier dependencies
constexpr unsigned FULL = 0xffffffffu;

struct WarpSmem {
  u32 mask[32][WORDS];
  u32 dep[32];                 // in-chunk predecessors (lane mask)
  i32 key[32];
  i32 v[32];
  i32 pcnt[32];                // earlier vertices still pending at the last scan
  unsigned long long sent[32]; // sentinel: max (key << 32 | vertex) among them
  i32 plist[32][PL];           // the pending ones (first PL; povf marks overflow)
  u32 povf[32];
  i32 ccol[32];
  i64 setsz[32];               // size of the forbidden-set walk (rescan cost)
  i64 excl[32];
  i64 rs[32];
  i64 excl2[32];
  i64 rs2[32];
  i32 own2[32];
};

struct GsArgs {
  const i64* rowptr;
  const i32* col;
  i32* val;           // colours; worklist entries hold PENDING until committed
  const i32* old;     // optional: colours of pending vertices before the call
  const i32* wl;      // optional: sorted unique worklist (else wl_base + i)
  i64 wl_base;
  const i64* nwl;     // device scalar: worklist length
  const i32* prio;    // optional ordering key (serial_greedy with an order)
  unsigned long long* ticket;
  unsigned long long* trace;  // optional per-chunk timestamps (CHROMA_GS_TRACE)
  unsigned long long* vtrace; // optional per-worklist-entry commit timestamps
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ i32 key_of(const GsArgs& a, i32 x) { return a.prio ? a.prio[x] : x; }
__device__ __forceinline__ unsigned long long pack(i32 k, i32 x) {
  return ((unsigned long long)(u32)k << 32) | (u32)x;
}

// largest j in [0,32) with arr[j] <= e (arr nondecreasing, arr[0] <= e)
template <typename T>
__device__ __forceinline__ int search32(const T* arr, T e) {
  int j = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1)
    if (arr[j + s] <= e) j += s;
  return j;
}

__device__ __forceinline__ void forbid(WarpSmem& sm, int j, i32 c) {
  if (c > 0 && c <= FAST_COLORS) atomicOr(&sm.mask[j][(c - 1) >> 5], 1u << ((c - 1) & 31));
}

// One forbidden-set candidate x of chunk lane j (phase A).
__device__ __forceinline__ void visit(const GsArgs& a, WarpSmem& sm, int j, i32 x, i32 kfirst,
                                      bool ident_lanes, i32 vfirst) {
  i32 c = a.val[x];  // a stale L1 copy can only read PENDING; resolved below
  if (c == PENDING) {
    const i32 kx = key_of(a, x);
    const i32 kv = sm.key[j];
    if (kx > kv) {
      // later in the order: it still holds its pre-call colour (it depends on v)
      c = a.old ? a.old[x] : 0;
    } else if (kx >= kfirst) {
      const int l = ident_lanes ? (x - vfirst) : search32<i32>(sm.key, kx);
      atomicOr(&sm.dep[j], 1u << l);
      return;
    } else {
      // possibly a stale PENDING: the list check in phase B resolves it
      const int k = atomicAdd(&sm.pcnt[j], 1);
      if (k < PL) sm.plist[j][k] = x;
      else sm.povf[j] = 1;
      atomicMax(&sm.sent[j], pack(kx, x));
      return;
    }
  }
  forbid(sm, j, c);
}

// Re-visit of a forbidden-set candidate once the lane's sentinel committed:
// committed colours are folded (idempotent), earlier pending ones counted.
__device__ __forceinline__ void revisit(const GsArgs& a, WarpSmem& sm, int j, i32 x, i32 kfirst, int& pend,
                                        unsigned long long& best) {
  const i32 c = ld_relaxed(a.val + x);
  if (c == PENDING) {
    const i32 kx = key_of(a, x);
    if (kx < kfirst) {
      pend++;
      const unsigned long long p = pack(kx, x);
      best = p > best ? p : best;
    }
  } else {
    forbid(sm, j, c);
  }
}

__device__ __forceinline__ int first_free(const u32 (&m)[WORDS]) {
#pragma unroll
  for (int w = 0; w < WORDS; w++)
    if (m[w] != FULL) return w * 32 + __ffs(~m[w]);
  return 0;
}

// Walk v's forbidden set: D1 N(v); D2 N(v) u N2(v); PD2 N2(v) -- split over `lanes`
// threads starting at `first` (1 = lane-serial, 32 = warp-cooperative).
template <int DIST, bool PARTIAL, typename F>
__device__ __forceinline__ void walk_set(const GsArgs& a, i32 v, int first, int lanes, F&& f) {
  const i64 rs = a.rowptr[v], re = a.rowptr[v + 1];
  if (DIST == 1) {
    for (i64 e = rs + first; e < re; e += lanes) f(a.col[e]);
  } else {
    for (i64 e = rs; e < re; e++) {
      const i32 u = a.col[e];
      if (!PARTIAL && first == 0) f(u);
      const i64 us = a.rowptr[u], ue = a.rowptr[u + 1];
      for (i64 g = us + first; g < ue; g += lanes) {
        const i32 x = a.col[g];
        if (x != v) f(x);
      }
    }
  }
}

// Warp-cooperative colour search above the fast window, once every dependency of v
// is committed.  Uniform across the warp.
template <int DIST, bool PARTIAL>
__device__ i32 slow_color(const GsArgs& a, i32 v, i32 kv, int lane) {
  for (i32 base = FAST_COLORS + 1;; base += FAST_COLORS) {
    u32 m[WORDS];
#pragma unroll
    for (int w = 0; w < WORDS; w++) m[w] = 0;
    walk_set<DIST, PARTIAL>(a, v, lane, 32, [&](i32 x) {
      i32 c = ld_relaxed(a.val + x);
      if (c == PENDING) c = (key_of(a, x) > kv && a.old) ? a.old[x] : 0;
      const i32 o = c - base;
      if (o >= 0 && o < FAST_COLORS) m[o >> 5] |= 1u << (o & 31);
    });
#pragma unroll
    for (int w = 0; w < WORDS; w++) m[w] = __reduce_or_sync(FULL, m[w]);
    const int r = first_free(m);
    if (r) return base + r - 1;
  }
}

template <int DIST, bool PARTIAL>
__global__ void __launch_bounds__(WARPS * 32)
gs_kernel(GsArgs a) {
  __shared__ WarpSmem smem[WARPS];
  const int lane = threadIdx.x & 31;
  WarpSmem& sm = smem[threadIdx.x >> 5];
  const i64 nwl = *a.nwl;
  const i64 nchunks = (nwl + 31) >> 5;
  const bool ident = (a.wl == nullptr) && (a.prio == nullptr);

  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    const i64 chunk = (i64)__shfl_sync(FULL, t, 0);
    if (chunk >= nchunks) break;
    unsigned long long t_claim = 0;
    if (a.trace && lane == 0) t_claim = gtimer();

    const i64 idx = chunk * 32 + lane;
    const bool act = idx < nwl;
    const i32 v = act ? (a.wl ? a.wl[idx] : (i32)(a.wl_base + idx)) : 0;
    const i32 kv = act ? key_of(a, v) : INT32_MAX;
    const i64 rs = act ? a.rowptr[v] : 0;
    const i64 d = act ? a.rowptr[v + 1] - rs : 0;
    i64 incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i64 tt = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += tt;
    }
    const i64 total = __shfl_sync(FULL, incl, 31);
    sm.excl[lane] = incl - d;
    sm.rs[lane] = rs;
    sm.key[lane] = kv;
    sm.v[lane] = v;
    sm.dep[lane] = 0;
    sm.pcnt[lane] = 0;
    sm.sent[lane] = 0;
    sm.povf[lane] = 0;
    sm.setsz[lane] = DIST == 1 ? d : 0;
#pragma unroll
    for (int w = 0; w < WORDS; w++) sm.mask[lane][w] = 0;
    const i32 kfirst = __shfl_sync(FULL, kv, 0);
    const i32 vfirst = __shfl_sync(FULL, v, 0);
    __syncwarp();

    // ---------------- phase A: fold committed colours, count the earlier pending ones
    if (DIST == 1) {
      for (i64 base = 0; base < total; base += 32) {
        const i64 e = base + lane;
        if (e < total) {
          const int j = search32<i64>(sm.excl, e);
          const i32 x = a.col[sm.rs[j] + (e - sm.excl[j])];
          visit(a, sm, j, x, kfirst, ident, vfirst);
        }
      }
    } else {
      for (i64 base = 0; base < total; base += 32) {
        const i64 e = base + lane;
        const bool ok = e < total;
        int j = 0;
        i32 u = 0;
        i64 us = 0, d2 = 0;
        if (ok) {
          j = search32<i64>(sm.excl, e);
          u = a.col[sm.rs[j] + (e - sm.excl[j])];
          us = a.rowptr[u];
          d2 = a.rowptr[u + 1] - us;
          atomicAdd((unsigned long long*)&sm.setsz[j], (unsigned long long)(d2 + 1));
        }
        i64 incl2 = d2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const i64 tt = __shfl_up_sync(FULL, incl2, o);
          if (lane >= o) incl2 += tt;
        }
        const i64 total2 = __shfl_sync(FULL, incl2, 31);
        __syncwarp();
        sm.excl2[lane] = incl2 - d2;
        sm.rs2[lane] = us;
        sm.own2[lane] = j;
        __syncwarp();
        if (ok && !PARTIAL) visit(a, sm, j, u, kfirst, ident, vfirst);
        for (i64 b2 = 0; b2 < total2; b2 += 32) {
          const i64 e2 = b2 + lane;
          if (e2 < total2) {
            const int k = search32<i64>(sm.excl2, e2);
            const int jj = sm.own2[k];
            const i32 x = a.col[sm.rs2[k] + (e2 - sm.excl2[k])];
            if (x != sm.v[jj]) visit(a, sm, jj, x, kfirst, ident, vfirst);
          }
        }
        __syncwarp();
      }
    }
    __syncwarp();

    unsigned long long t_a = 0;
    if (a.trace && lane == 0) t_a = gtimer();

    // ---------------- phase B: per-lane dataflow commit
    const u32 mydep = sm.dep[lane];
    bool done = !act;
    u32 donemask = __ballot_sync(FULL, done);
    unsigned ns = 64;
    while (donemask != FULL) {
      // commit every lane whose dependencies are all satisfied; repeat while the
      // in-chunk chain keeps advancing (no global traffic in this inner loop)
      for (;;) {
        const bool ready = !done && sm.pcnt[lane] == 0 && (mydep & ~donemask) == 0;
        int r = 1;
        if (ready) {
          u32 m[WORDS];
#pragma unroll
          for (int w = 0; w < WORDS; w++) m[w] = sm.mask[lane][w];
          for (u32 bits = mydep; bits; bits &= bits - 1) {
            const i32 c = sm.ccol[__ffs(bits) - 1];
            if (c <= FAST_COLORS) m[(c - 1) >> 5] |= 1u << ((c - 1) & 31);
          }
          r = first_free(m);
          if (r) {
            if (a.vtrace) a.vtrace[idx] = gtimer();
            st_relaxed(a.val + v, r);
            sm.ccol[lane] = r;
            done = true;
          }
        }
        u32 slow = __ballot_sync(FULL, ready && r == 0);
        while (slow) {
          const int l = __ffs(slow) - 1;
          slow &= slow - 1;
          const i32 c = slow_color<DIST, PARTIAL>(a, __shfl_sync(FULL, v, l), __shfl_sync(FULL, kv, l), lane);
          if (lane == l) {
            st_relaxed(a.val + v, c);
            sm.ccol[lane] = c;
            done = true;
          }
        }
        __syncwarp();
        const u32 nd = __ballot_sync(FULL, done);
        if (nd == donemask) break;
        donemask = nd;
      }
      if (donemask == FULL) break;
      // poll one sentinel per waiting lane (its largest-key pending earlier vertex);
      // adjacent lanes usually wait on adjacent vertices, so the loads coalesce
      bool need = false;
      if (!done && sm.pcnt[lane] > 0) need = ld_relaxed(a.val + (i32)(sm.sent[lane] & 0xffffffffu)) != PENDING;
      if (!__any_sync(FULL, need)) {
        __nanosleep(ns);
        ns = ns < NS_MAX ? ns * 2 : ns;
        continue;
      }
      ns = 64;
      // listed dependencies: one batch of independent loads, keep the still-pending
      const bool listed = need && !sm.povf[lane];
      if (listed) {
        const int n = sm.pcnt[lane];
        i32 xs[PL], cs[PL];
#pragma unroll
        for (int k = 0; k < PL; k++) {
          xs[k] = k < n ? sm.plist[lane][k] : 0;
          cs[k] = k < n ? ld_relaxed(a.val + xs[k]) : 0;
        }
        int w = 0;
        unsigned long long best = 0;
#pragma unroll
        for (int k = 0; k < PL; k++) {
          if (k >= n) break;
          if (cs[k] == PENDING) {
            sm.plist[lane][w++] = xs[k];
            const unsigned long long p = pack(key_of(a, xs[k]), xs[k]);
            best = p > best ? p : best;
          } else {
            forbid(sm, lane, cs[k]);
          }
        }
        sm.pcnt[lane] = w;
        sm.sent[lane] = best;
      }
      // overflowed lists: walk the whole set again (light lane-serially, heavy by the warp)
      const bool walk = need && !listed;
      const bool heavy = walk && sm.setsz[lane] > HEAVY;
      if (walk && !heavy) {
        int pend = 0;
        unsigned long long best = 0;
        walk_set<DIST, PARTIAL>(a, v, 0, 1, [&](i32 x) { revisit(a, sm, lane, x, kfirst, pend, best); });
        sm.pcnt[lane] = pend;
        sm.sent[lane] = best;
      }
      u32 hv = __ballot_sync(FULL, heavy);
      while (hv) {
        const int l = __ffs(hv) - 1;
        hv &= hv - 1;
        const i32 vl = __shfl_sync(FULL, v, l);
        int pend = 0;
        unsigned long long best = 0;
        walk_set<DIST, PARTIAL>(a, vl, lane, 32, [&](i32 x) { revisit(a, sm, l, x, kfirst, pend, best); });
        pend = __reduce_add_sync(FULL, pend);
        const u32 hi = __reduce_max_sync(FULL, (u32)(best >> 32));
        const u32 lo = __reduce_max_sync(FULL, (u32)(best >> 32) == hi ? (u32)best : 0u);
        if (lane == 0) {
          sm.pcnt[l] = pend;
          sm.sent[l] = ((unsigned long long)hi << 32) | lo;
        }
      }
      __syncwarp();
    }
    __syncwarp();
    if (a.trace && lane == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.trace[4 * chunk + 0] = t_claim;
      a.trace[4 * chunk + 1] = t_a;
      a.trace[4 * chunk + 2] = gtimer();
      a.trace[4 * chunk + 3] = smid;
    }
  }
}

}  // namespace

void launch_gs(const GsLaunch& L, cudaStream_t s) {
  // distance 1 in id order: the pre-scan-free kernel (color_gs_d1.cu)
  if (launch_gs_d1(L, s)) return;
  CHROMA_REQUIRE(!L.level_mode, CHROMA_ERUNTIME, "level schedules are distance-1 only");
  GsArgs a;
  a.rowptr = L.rowptr;
  a.col = L.col;
  a.val = L.val;
  a.old = L.old;
  a.wl = L.wl;
  a.wl_base = L.wl_base;
  a.nwl = L.nwl_dev;
  a.prio = L.prio;
  a.ticket = L.ticket;
  a.trace = nullptr;
  a.vtrace = nullptr;
  CUDA_CHECK(cudaMemsetAsync(L.ticket, 0, sizeof(unsigned long long), s));
  const i64 nchunks = (L.nwl_max + 31) / 32;
  static const char* trace_path = std::getenv("CHROMA_GS_TRACE");
  static const int bps_env = std::getenv("CHROMA_GS_BPS") ? std::atoi(std::getenv("CHROMA_GS_BPS")) : 0;
  DBuf<unsigned long long> tr, vtr;
  if (trace_path) {
    tr.alloc(4 * nchunks, s);
    tr.zero(s);
    a.trace = tr.p;
    vtr.alloc(32 * nchunks, s);
    vtr.zero(s);
    a.vtrace = vtr.p;
  }
  const int blocks_per_sm = bps_env > 0 ? bps_env : 8;
  int grid = (int)std::min<i64>((nchunks + WARPS - 1) / WARPS, (i64)num_sms() * blocks_per_sm);
  if (grid < 1) grid = 1;
  if (L.dist == 1)
    gs_kernel<1, false><<<grid, WARPS * 32, 0, s>>>(a);
  else if (L.partial)
    gs_kernel<2, true><<<grid, WARPS * 32, 0, s>>>(a);
  else
    gs_kernel<2, false><<<grid, WARPS * 32, 0, s>>>(a);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
  if (trace_path) {
    std::vector<unsigned long long> h((size_t)(4 * nchunks));
    CUDA_CHECK(cudaMemcpyAsync(h.data(), tr.p, sizeof(unsigned long long) * 4 * nchunks, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (FILE* f = std::fopen(trace_path, "wb")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
    std::vector<unsigned long long> hv((size_t)(32 * nchunks));
    CUDA_CHECK(cudaMemcpyAsync(hv.data(), vtr.p, sizeof(unsigned long long) * 32 * nchunks, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (FILE* f = std::fopen((std::string(trace_path) + ".v").c_str(), "wb")) {
      std::fwrite(hv.data(), sizeof(unsigned long long), hv.size(), f);
      std::fclose(f);
    }
  }
}

}  // namespace chroma
