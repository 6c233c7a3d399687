// Cut-edge conflict detection with the hashed-GID loser cascade.
//
// Reference: chroma/protocol.py:136-157 (D1: every ghost row, ascending, each row
// scanned in order, aborting once the ghost is uncoloured) and 160-194 (D2: every
// boundary_d2 vertex against its one-hop (full mode) and two-hop reach).  The
// reference scan is sequential and in place, so a loser uncoloured early hides
// later pairs (F4).  It is restated exactly (F5) as:
//   1. emit every equal-coloured pair of the scan as an event, in scan order
//      (two-pass count / exclusive-scan / ordered write, no sort needed);
//   2. the loser of each event is fixed by the cascade (degree, gid hash, gid);
//   3. event e fires iff neither endpoint was uncoloured by an earlier fired event
//      -- a recurrence over event order solved by Jacobi iteration to its unique
//      fixed point (each pass settles at least one more link of every chain);
//   4. fired events uncolour their losers; the count is the number of fired events.
// In free-running mode (sequential = false) every event fires (classic parallel
// detection: every conflicting pair loses one endpoint).
#include <cstdio>
#include <cstdlib>
#include <functional>

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/unique.h>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct DevDetect {
  const i64* rowptr;
  const i32* col;
  const i32* colors;
  const i64* gids;
  const i32* deg;
  const i32* rows;
  i64 nrows;
  bool rd;
};

__device__ __forceinline__ int2 make_event(const DevDetect& a, i32 v, i32 x) {
  const bool vl = v_loses(a.gids[v], a.gids[x], a.deg[v], a.deg[x], a.rd);
  return vl ? make_int2(v, x) : make_int2(x, v);
}

// Enumerates the scan sequence of row i in reference order and calls
// f(hit, x, ballot_prefix_base) warp-uniformly per 32-candidate step.
template <int DIST, bool PARTIAL, bool WRITE>
__global__ void k_events(DevDetect a, i64* cnt, const i64* off, int2* ev) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < a.nrows; i += nwarps) {
    if (WRITE && cnt[i] == 0) continue;
    const i32 v = a.rows[i];
    const i32 cv = a.colors[v];
    i64 pos = WRITE ? off[i] : 0;
    i64 count = 0;
    if (cv != 0) {
      const i64 rs = a.rowptr[v], re = a.rowptr[v + 1];
      if (DIST == 1) {
        for (i64 e0 = rs; e0 < re; e0 += 32) {
          const i64 e = e0 + lane;
          i32 x = 0;
          bool hit = false;
          if (e < re) {
            x = a.col[e];
            hit = a.colors[x] == cv;
          }
          const unsigned b = __ballot_sync(FULL, hit);
          if (WRITE && hit) ev[pos + __popc(b & lanemask_lt())] = make_event(a, v, x);
          pos += __popc(b);
          count += __popc(b);
        }
      } else {
        for (i64 j = rs; j < re; j++) {
          const i32 u = a.col[j];
          const i64 us = a.rowptr[u], ue = a.rowptr[u + 1];
          const i64 t0 = PARTIAL ? 0 : -1;
          for (i64 tb = t0; tb < ue - us; tb += 32) {
            const i64 t = tb + lane;
            i32 x = 0;
            bool hit = false;
            if (t < ue - us) {
              x = t < 0 ? u : a.col[us + t];
              hit = (t < 0 || x != v) && a.colors[x] == cv;
            }
            const unsigned b = __ballot_sync(FULL, hit);
            if (WRITE && hit) ev[pos + __popc(b & lanemask_lt())] = make_event(a, v, x);
            pos += __popc(b);
            count += __popc(b);
          }
        }
      }
    }
    if (!WRITE && lane == 0) cnt[i] = count;
  }
}

// Distance 1, rows of any length: a warp takes 32 consecutive detection rows; a lane
// walks its own row when it has at most 32 entries (most ghost rows hold a few
// back-edges), the warp walks the longer ones together.  Same events, same order.
template <bool WRITE>
__global__ void k_events_d1(DevDetect a, i64* cnt, const i64* off, int2* ev) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 b = warp * 32; b < a.nrows; b += nwarps * 32) {
    const i64 i = b + lane;
    i32 v = -1, cv = 0;
    i64 rs = 0, re = 0;
    if (i < a.nrows && (!WRITE || cnt[i] != 0)) {
      v = a.rows[i];
      cv = a.colors[v];
      if (cv != 0) {
        rs = a.rowptr[v];
        re = a.rowptr[v + 1];
      }
    }
    const bool lng = re - rs > 32;
    if (!lng && re > rs) {
      i64 pos = WRITE ? off[i] : 0, count = 0;
      for (i64 e0 = rs; e0 < re; e0 += 8) {
        i32 xs[8];
#pragma unroll
        for (int q = 0; q < 8; q++) xs[q] = e0 + q < re ? a.col[e0 + q] : -1;
        bool hs[8];
#pragma unroll
        for (int q = 0; q < 8; q++) hs[q] = xs[q] >= 0 && a.colors[xs[q]] == cv;
#pragma unroll
        for (int q = 0; q < 8; q++)
          if (hs[q]) {
            if (WRITE) ev[pos] = make_event(a, v, xs[q]);
            pos++;
            count++;
          }
      }
      if (!WRITE) cnt[i] = count;
    } else if (!lng && !WRITE && i < a.nrows) {
      cnt[i] = 0;
    }
    for (unsigned lm = __ballot_sync(FULL, lng); lm; lm &= lm - 1) {
      const int src = __ffs(lm) - 1;
      const i32 vl = __shfl_sync(FULL, v, src), cl = __shfl_sync(FULL, cv, src);
      const i64 ls = __shfl_sync(FULL, rs, src), le = __shfl_sync(FULL, re, src);
      i64 pos = WRITE ? off[b + src] : 0, count = 0;
      for (i64 e0 = ls; e0 < le; e0 += 32) {
        const i64 e = e0 + lane;
        i32 x = 0;
        bool hit = false;
        if (e < le) {
          x = a.col[e];
          hit = a.colors[x] == cl;
        }
        const unsigned bb = __ballot_sync(FULL, hit);
        if (WRITE && hit) ev[pos + __popc(bb & lanemask_lt())] = make_event(a, vl, x);
        pos += __popc(bb);
        count += __popc(bb);
      }
      if (!WRITE && lane == 0) cnt[b + src] = count;
    }
  }
}

__global__ void k_total(const i64* cnt, const i64* off, i64 n, i64* total) {
  *total = off[n - 1] + cnt[n - 1];
}

__global__ void __launch_bounds__(1024) k_resolve(const int2* ev, i64 E, uint8_t* fired, i32* kill,
                                                  i32* colors, unsigned long long* conflicts,
                                                  bool sequential) {
  __shared__ int changed;
  __shared__ unsigned long long fired_count;
  const i64 t = threadIdx.x, T = blockDim.x;
  if (t == 0) fired_count = 0;
  if (sequential) {
    for (i64 e = t; e < E; e += T) fired[e] = 1;
    __syncthreads();
    for (i64 it = 0; it <= E + 1; it++) {
      for (i64 e = t; e < E; e += T) {
        kill[ev[e].x] = INT32_MAX;
        kill[ev[e].y] = INT32_MAX;
      }
      __syncthreads();
      for (i64 e = t; e < E; e += T)
        if (fired[e]) atomicMin(&kill[ev[e].x], (i32)e);
      if (t == 0) changed = 0;
      __syncthreads();
      for (i64 e = t; e < E; e += T) {
        const uint8_t f = (kill[ev[e].x] >= (i32)e && kill[ev[e].y] >= (i32)e) ? 1 : 0;
        if (f != fired[e]) {
          fired[e] = f;
          changed = 1;
        }
      }
      __syncthreads();
      if (!changed) break;
      __syncthreads();
    }
  }
  unsigned long long mine = 0;
  for (i64 e = t; e < E; e += T) {
    if (!sequential || fired[e]) {
      colors[ev[e].x] = 0;
      mine++;
    }
  }
  atomicAdd(&fired_count, mine);
  __syncthreads();
  if (t == 0) *conflicts += fired_count;
}

// Grid-wide form of k_resolve for large event lists (cooperative launch, one
// 1024-thread CTA per SM): the same Jacobi fixed point over the event order, every
// sweep spread over the whole GPU with software grid barriers.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// kill64[v] = (tag(sweep) << 32 | smallest fired event with loser v) for the current
// sweep; a value with another sweep's tag reads as "no kill", so the per-sweep reset
// pass (and its barrier) of k_resolve is not needed.  Tags fall as sweeps advance, so
// the sweep's atomicMin always replaces an older value.
__device__ __forceinline__ unsigned long long kill_tag(i64 it) { return 0xFFFFFFFEull - (unsigned long long)it; }

__device__ __forceinline__ i32 kill_read(const unsigned long long* kill, i32 v, unsigned long long tag) {
  const unsigned long long k = kill[v];
  return (k >> 32) == tag ? (i32)(u32)k : INT32_MAX;
}

__global__ void __launch_bounds__(1024, 1) k_resolve_grid(const int2* ev, i64 E, uint8_t* fired,
                                                          unsigned long long* kill, i32* colors,
                                                          unsigned long long* conflicts, unsigned* bar, int* changed) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x, T = (i64)gridDim.x * blockDim.x;
  const unsigned nb = gridDim.x;
  for (i64 e = t; e < E; e += T) {
    fired[e] = 1;
    kill[ev[e].x] = ~0ull;  // a tag no sweep uses
    kill[ev[e].y] = ~0ull;
  }
  grid_sync(bar, nb);
  for (i64 it = 0; it <= E + 1; it++) {
    // three flags: this sweep's, the next one's (cleared now), and the previous
    // one's, which a block that just left the last barrier may still be reading
    int* ch = changed + it % 3;
    if (t == 0) changed[(it + 1) % 3] = 0;
    const unsigned long long tag = kill_tag(it);
    for (i64 e = t; e < E; e += T)
      if (fired[e]) atomicMin(kill + ev[e].x, (tag << 32) | (u32)e);
    grid_sync(bar, nb);
    bool mine = false;
    for (i64 e = t; e < E; e += T) {
      const int2 q = ev[e];
      const uint8_t f = (kill_read(kill, q.x, tag) >= (i32)e && kill_read(kill, q.y, tag) >= (i32)e) ? 1 : 0;
      if (f != fired[e]) {
        fired[e] = f;
        mine = true;
      }
    }
    if (__syncthreads_or(mine) && threadIdx.x == 0) atomicExch(ch, 1);
    grid_sync(bar, nb);
    if (!*(volatile int*)ch) break;
  }
  unsigned long long n = 0;
  for (i64 e = t; e < E; e += T)
    if (fired[e]) {
      colors[ev[e].x] = 0;
      n++;
    }
  n = __reduce_add_sync(0xffffffffu, (unsigned)n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(conflicts, n);
}

// Changed-side event emission (distance 1, sequential, incremental): an event needs
// a changed endpoint (see below), and the local CSR is symmetric (owned rows are
// complete, ghost rows hold the back-edges), so walking the rows of the changed
// vertices finds every scanned pair (v ghost, x in row(v)) with equal colours:
// from changed y, (y, x) when y is a ghost, (x, y) when x is.  Keys (v << 32 | x)
// sorted and de-duplicated are exactly the reference's scan order (ghost rows
// ascending, each row ascending).  WRITE = false counts; with WRITE, keys beyond cap
// are counted but not stored (the caller grows the buffer and emits again).
constexpr i64 SEG = 256;  // row entries per work item of the changed-side walk

// segments of the long (> 32 entries) source rows; short ones go to k_emit_short
__global__ void k_changed_nseg(const i64* rowptr, const i32* changed, i64 nch, i64* nseg, bool long_only) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nch; i += (i64)gridDim.x * blockDim.x) {
    const i32 y = changed[i];
    const i64 d = rowptr[y + 1] - rowptr[y];
    nseg[i] = long_only && d <= 32 ? 0 : (d + SEG - 1) / SEG;
  }
}

// Short source rows (<= 32 entries), one lane each; keys appended with one atomic
// per warp.  ROWS: sources are detection rows, emit (y, x); otherwise sources are
// changed vertices, emit (y, x) if y is a ghost and (x, y) if x is.
template <bool WRITE, bool ROWS>
__global__ void k_emit_short(const i64* rowptr, const i32* col, const i32* colors, const uint8_t* owned,
                             const i32* src, i64 nsrc, unsigned long long* cnt, u64* keys, unsigned long long cap) {
  const int lane = threadIdx.x & 31;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) - lane; b < nsrc; b += (i64)gridDim.x * blockDim.x) {
    const i64 i = b + lane;
    i32 y = -1, cy = 0;
    i64 rs = 0, re = 0;
    bool gy = ROWS;
    if (i < nsrc) {
      y = src[i];
      cy = colors[y];
      rs = rowptr[y];
      re = rowptr[y + 1];
      if (!ROWS) gy = !owned[y];
      if (re - rs > 32 || cy == 0) re = rs;  // long rows: k_changed_events
    }
    unsigned k = 0;
    for (int pass = 0; pass < (WRITE ? 2 : 1); pass++) {
      unsigned long long at = 0;
      if (pass == 1) {
        unsigned inc = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += t;
        }
        const unsigned tot = __shfl_sync(FULL, inc, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot) base = atomicAdd(cnt, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 31);
        at = base + inc - k;
      }
      for (i64 e0 = rs; e0 < re; e0 += 8) {
        i32 xs[8];
#pragma unroll
        for (int q = 0; q < 8; q++) xs[q] = e0 + q < re ? col[e0 + q] : -1;
        bool hs[8], gs[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          hs[q] = xs[q] >= 0 && colors[xs[q]] == cy;
          gs[q] = !ROWS && hs[q] && !owned[xs[q]];
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if (!hs[q]) continue;
          if (pass == 0) {
            k += (gy ? 1u : 0u) + (gs[q] ? 1u : 0u);
          } else {
            if (gy && at < cap) keys[at] = ((u64)(u32)y << 32) | (u32)xs[q];
            at += gy;
            if (gs[q] && at < cap) keys[at] = ((u64)(u32)xs[q] << 32) | (u32)y;
            at += gs[q];
          }
        }
      }
    }
    if (!WRITE) {
      const unsigned tot = __reduce_add_sync(FULL, k);
      if (lane == 0 && tot) atomicAdd(cnt, (unsigned long long)tot);
    }
  }
}

// A warp per item (changed vertex i, segment of SEG row entries): item j belongs to
// the last i with segoff[i] <= j.  Each warp takes a contiguous range of items (one
// binary search, then a warp-wide forward scan of segoff per item).  Four 32-entry
// steps of loads are in flight per lane; steps without an equal pair cost one ballot.
// Keys go to *cnt-indexed slots (one atomic per warp step with keys; the caller
// sorts them).  WRITE = false only counts.
template <bool WRITE, bool ROWS>
__global__ void k_changed_events(const i64* rowptr, const i32* col, const i32* colors, const uint8_t* owned,
                                 const i32* changed, i64 nch, const i64* segoff, i64 nitems,
                                 unsigned long long* cnt, u64* keys, unsigned long long cap) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  const i64 per = (nitems + nwarps - 1) / nwarps;
  const i64 j0 = warp * per, j1 = j0 + per < nitems ? j0 + per : nitems;
  if (j0 >= j1) return;
  // upper_bound(segoff, j0) - 1, searched by one lane
  i64 i = 0;
  if (lane == 0) {
    i64 lo = 0, hi = nch;
    while (hi - lo > 1) {
      const i64 mid = (lo + hi) >> 1;
      if (segoff[mid] <= j0) lo = mid; else hi = mid;
    }
    i = lo;
  }
  i = __shfl_sync(FULL, i, 0);
  unsigned long long mine = 0;
  for (i64 j = j0; j < j1; j++) {
    // advance to the last i with segoff[i] <= j (segoff is non-decreasing: the lanes
    // that pass form a prefix)
    for (;;) {
      const i64 t = i + 1 + lane;
      const unsigned b = __ballot_sync(FULL, t < nch && segoff[t] <= j);
      i += __popc(b);
      if (b != FULL) break;
    }
    const i32 y = changed[i];
    const i32 cy = colors[y];
    const bool gy = ROWS || !owned[y];
    const i64 rs = rowptr[y], re = cy == 0 ? rowptr[y] : rowptr[y + 1];
    const i64 s0 = rs + (j - segoff[i]) * SEG;
    const i64 s1 = s0 + SEG < re ? s0 + SEG : re;
    for (i64 e0 = s0; e0 < s1; e0 += 4 * 32) {
      i32 xs[4];
      bool eq[4];
#pragma unroll
      for (int q = 0; q < 4; q++) xs[q] = e0 + q * 32 + lane < s1 ? col[e0 + q * 32 + lane] : -1;
#pragma unroll
      for (int q = 0; q < 4; q++) eq[q] = xs[q] >= 0 && colors[xs[q]] == cy;
      bool gx[4];
#pragma unroll
      for (int q = 0; q < 4; q++) gx[q] = !ROWS && eq[q] && !owned[xs[q]];
      if (!WRITE) {
#pragma unroll
        for (int q = 0; q < 4; q++) mine += eq[q] ? (gy ? 1u : 0u) + (gx[q] ? 1u : 0u) : 0u;
        continue;
      }
      if (!__any_sync(FULL, eq[0] || eq[1] || eq[2] || eq[3])) continue;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const unsigned b1 = __ballot_sync(FULL, eq[q] && gy), b2 = __ballot_sync(FULL, gx[q]);
        const unsigned tot = __popc(b1) + __popc(b2);
        if (!tot) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(cnt, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 0);
        unsigned long long at = base + __popc(b1 & lt) + __popc(b2 & lt);
        if (eq[q] && gy) {
          if (at < cap) keys[at] = ((u64)(u32)y << 32) | (u32)xs[q];
          at++;
        }
        if (gx[q] && at < cap) keys[at] = ((u64)(u32)xs[q] << 32) | (u32)y;
      }
    }
  }
  if (!WRITE) {
    mine = __reduce_add_sync(FULL, (unsigned)mine);
    if (lane == 0 && mine) atomicAdd(cnt, mine);
  }
}

// vertices whose colour changed since the previous call (coloured now), listed in
// any order (the keys they emit are sorted): one atomic per warp step
__global__ void k_changed_list(const i32* colors, const i32* prev, i64 n, i32* out, i64* cnt) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = blockIdx.x * (i64)blockDim.x + threadIdx.x - lane; b < n; b += stride) {
    const i64 i = b + lane;
    bool ch = false;
    if (i < n) {
      const i32 c = colors[i];
      ch = c != 0 && c != prev[i];
    }
    const unsigned m = __ballot_sync(FULL, ch);
    if (!m) continue;
    i64 base = 0;
    if (lane == 0) base = (i64)atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)__popc(m));
    base = __shfl_sync(FULL, base, 0);
    if (ch) out[base + __popc(m & ((1u << lane) - 1u))] = (i32)i;
  }
}

// unique sorted keys -> events in scan order, loser by the cascade
__global__ void k_keys_to_events(DevDetect a, const u64* keys, i64 k, int2* ev) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < k; i += (i64)gridDim.x * blockDim.x) {
    const u64 key = keys[i];
    ev[i] = make_event(a, (i32)(key >> 32), (i32)(key & 0xffffffffu));
  }
}

// Incremental detection: an event (equal non-zero colours on a scanned pair) can
// only exist if one endpoint changed colour since the previous detection (which
// left no conflicting pair behind, and unchanged pairs keep their colours).  Mark
// every vertex within DIST hops of a changed, coloured vertex; the scan then visits
// only marked rows, in the same order, so the event sequence is unchanged.
template <int DIST>
__global__ void k_mark_changed(const i64* rowptr, const i32* col, const i32* colors, const i32* prev, i64 n,
                               uint8_t* mark) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 b = warp * 32; b < n; b += nwarps * 32) {
    const i64 i = b + lane;
    bool ch = false;
    if (i < n) {
      const i32 c = colors[i];
      ch = c != 0 && c != prev[i];
    }
    if (DIST == 1 && ch) {  // short rows: the lane marks its own row
      const i64 rs = rowptr[i], re = rowptr[i + 1];
      if (re - rs <= 32) {
        mark[i] = 1;
        for (i64 e = rs; e < re; e++) mark[col[e]] = 1;
        ch = false;
      }
    }
    unsigned m = __ballot_sync(FULL, ch);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const i32 v = (i32)(b + l);
      if (lane == 0) mark[v] = 1;
      const i64 rs = rowptr[v], re = rowptr[v + 1];
      if (DIST == 1) {
        for (i64 e = rs + lane; e < re; e += 32) mark[col[e]] = 1;
      } else {
        for (i64 e = rs; e < re; e++) {
          const i32 u = col[e];
          if (lane == 0) mark[u] = 1;
          for (i64 g = rowptr[u] + lane; g < rowptr[u + 1]; g += 32) mark[col[g]] = 1;
        }
      }
    }
  }
}

__global__ void k_mark_flags(const i32* rows, i64 n, const uint8_t* mark, uint8_t* flags) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flags[i] = mark[rows[i]];
}

// ---- free-running D1: pair-centric detection around changed vertices --------
// Without the reference's ordered replay (every conflicting pair loses its loser),
// only pairs touching a vertex whose colour changed since the previous detection
// can conflict.  Each such vertex scans its row; a cut pair (one owned, one ghost
// end) with equal non-zero colours uncolours its loser (degree / gid-hash cascade)
// on the loser's owner.  The count is the number of vertices uncoloured
// (atomicExch makes repeats idempotent).
constexpr i64 DET_HEAVY = 2048;
constexpr int DET_HEAVY_THREADS = 512;

__global__ void k_changed_split(const i32* colors, const i32* prev, i64 n, const i64* rowptr, i32* light,
                                i32* heavy, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + lane;
    bool ch = false, h = false;
    if (i < n) {
      const i32 c = colors[i];
      ch = c != 0 && (prev == nullptr || c != prev[i]);
      if (ch) h = rowptr[i + 1] - rowptr[i] > DET_HEAVY;
    }
    const unsigned mh = __ballot_sync(FULL, ch && h), ml = __ballot_sync(FULL, ch && !h);
    unsigned long long oh = 0, ol = 0;
    if (lane == 0) {
      if (ml) ol = atomicAdd(cnt, (unsigned long long)__popc(ml));
      if (mh) oh = atomicAdd(cnt + 1, (unsigned long long)__popc(mh));
    }
    ol = __shfl_sync(FULL, ol, 0);
    oh = __shfl_sync(FULL, oh, 0);
    const unsigned below = lanemask_lt();
    if (ch && h) heavy[oh + __popc(mh & below)] = (i32)i;
    else if (ch) light[ol + __popc(ml & below)] = (i32)i;
  }
}

struct FreeDet {
  const i64* rowptr;
  const i32* col;
  i32* colors;
  const uint8_t* owned;
  const i64* gids;
  const i32* deg;
  bool rd;
  bool kill_anywhere = false;            // list path: kill at the loser's owner (KillRoute)
  KillRoute kr;
};

// kill_anywhere (worklist-driven path): the loser is uncoloured at its owner --
// here if owned, else through KillRoute (same array for virtual ranks, NVLink for
// peers) -- and its owner's loser flag is raised; ghost copies are then refreshed
// by their owners alone (loser broadcast, exchange).  Otherwise (the full exchange
// rewrites every ghost each round) the loser's local entry is zeroed, ghost or not.
__device__ __forceinline__ int free_pair(const FreeDet& a, i32 x, bool ox, i32 cx, i32 y) {
  const bool oy = a.owned[y];
  if (ox == oy) return 0;  // owned-owned is proper by construction; ghost-ghost is the owners' business
  const i32 cy = ld_relaxed(a.colors + y);
  if (cy != cx) return 0;
  const i32 loser = v_loses(a.gids[x], a.gids[y], a.deg[x], a.deg[y], a.rd) ? x : y;
  if (!a.kill_anywhere) return atomicExch(a.colors + loser, 0) != 0 ? 1 : 0;
  const bool lo = loser == x ? ox : oy;
  if (lo) {
    if (atomicExch(a.colors + loser, 0) == 0) return 0;
    a.kr.flags[loser] = 1;
    return 1;
  }
  const i32 o = a.kr.owner_lid[loser];
  const i32 p = a.kr.owner_rank[loser];
  if (p < 0) {
    if (atomicExch(a.colors + o, 0) == 0) return 0;
    a.kr.flags[o] = 1;
  } else {
    if (atomicExch_system(a.kr.peer_colors[p] + o, 0) == 0) return 0;
    a.kr.peer_flag[p][o] = 1;
  }
  return 1;
}

// changed-vertex list -> light / heavy rows (warp-aggregated appends; two-hop walks
// count as heavy from a quarter of the one-hop threshold)
__global__ void k_split_list(const i32* list, const unsigned long long* n_dev, const i64* rowptr, const i32* colors,
                             i64 heavy_deg, i32* light, i32* heavy, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const i64 n = (i64)*n_dev;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + lane;
    bool ch = false, h = false;
    i32 x = 0;
    if (i < n) {
      x = list[i];
      ch = colors[x] != 0;
      if (ch) h = rowptr[x + 1] - rowptr[x] > heavy_deg;
    }
    const unsigned mh = __ballot_sync(FULL, ch && h), ml = __ballot_sync(FULL, ch && !h);
    unsigned long long oh = 0, ol = 0;
    if (lane == 0) {
      if (ml) ol = atomicAdd(cnt, (unsigned long long)__popc(ml));
      if (mh) oh = atomicAdd(cnt + 1, (unsigned long long)__popc(mh));
    }
    ol = __shfl_sync(FULL, ol, 0);
    oh = __shfl_sync(FULL, oh, 0);
    const unsigned below = lanemask_lt();
    if (ch && h) heavy[oh + __popc(mh & below)] = x;
    else if (ch) light[ol + __popc(ml & below)] = x;
  }
}

// Visit the colouring set of x -- N(x) (D1), N(x) and N2(x) (D2) or N2(x) (PD2) --
// with `stride` cooperating threads; f returns false to stop this thread's walk.
template <int DIST, bool PARTIAL, typename F>
__device__ __forceinline__ void walk_set(const FreeDet& a, i32 x, int t, int stride, F&& f) {
  const i64 rs = a.rowptr[x], re = a.rowptr[x + 1];
  if (DIST == 1) {
    for (i64 e = rs + t; e < re; e += stride)
      if (!f(a.col[e])) return;
  } else if (stride == 32) {
    for (i64 e = rs; e < re; e++) {
      const i32 u = a.col[e];
      if (!PARTIAL && t == 0 && !f(u)) return;
      const i64 ue = a.rowptr[u + 1];
      for (i64 g = a.rowptr[u] + t; g < ue; g += 32) {
        const i32 y = a.col[g];
        if (y != x && !f(y)) return;
      }
    }
  } else {
    for (i64 e = rs + t; e < re; e += stride) {
      const i32 u = a.col[e];
      if (!PARTIAL && !f(u)) return;
      const i64 ue = a.rowptr[u + 1];
      for (i64 g = a.rowptr[u]; g < ue; g++) {
        const i32 y = a.col[g];
        if (y != x && !f(y)) return;
      }
    }
  }
}

template <int DIST, bool PARTIAL>
__global__ void k_free_light(FreeDet a, const i32* list, const unsigned long long* n_dev,
                             unsigned long long* conflicts) {
  const int lane = threadIdx.x & 31;
  const i64 n = (i64)*n_dev;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  int mine = 0;
  for (i64 i = warp; i < n; i += nwarps) {
    const i32 x = list[i];
    const bool ox = a.owned[x];
    const i32 cx0 = ld_relaxed(a.colors + x);
    if (cx0 == 0) continue;
    walk_set<DIST, PARTIAL>(a, x, lane, 32, [&](i32 y) {
      const i32 cx = ox ? ld_relaxed(a.colors + x) : cx0;
      if (cx == 0) return false;  // an owned scanner already uncoloured by another pair
      mine += free_pair(a, x, ox, cx, y);
      return true;
    });
  }
  mine = __reduce_add_sync(FULL, mine);
  if (lane == 0 && mine) atomicAdd(conflicts, (unsigned long long)mine);
}

template <int DIST, bool PARTIAL>
__global__ void __launch_bounds__(DET_HEAVY_THREADS) k_free_heavy(FreeDet a, const i32* list,
                                                                  const unsigned long long* n_dev,
                                                                  unsigned long long* conflicts) {
  const int lane = threadIdx.x & 31;
  const i64 n = (i64)*n_dev;
  int mine = 0;
  for (i64 i = blockIdx.x; i < n; i += gridDim.x) {
    const i32 x = list[i];
    const bool ox = a.owned[x];
    const i32 cx0 = ld_relaxed(a.colors + x);
    if (cx0 == 0) continue;
    walk_set<DIST, PARTIAL>(a, x, threadIdx.x, DET_HEAVY_THREADS, [&](i32 y) {
      const i32 cx = ox ? ld_relaxed(a.colors + x) : cx0;
      if (cx == 0) return false;
      mine += free_pair(a, x, ox, cx, y);
      return true;
    });
  }
  mine = __reduce_add_sync(FULL, mine);
  if (lane == 0 && mine) atomicAdd(conflicts, (unsigned long long)mine);
}

#define FREE_DET_DISPATCH(KERNEL, GRID, BLOCK, ...)                                          \
  do {                                                                                      \
    if (A.dist == 1) KERNEL<1, false><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                  \
    else if (A.partial) KERNEL<2, true><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                \
    else KERNEL<2, false><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                              \
    count_launch();                                                                         \
  } while (0)

}  // namespace

static void run_detect_free_d1(const DetectArgs& A, i64 nv, DetectScratch& S, unsigned long long* conflicts,
                               cudaStream_t s) {
  S.chl.reserve(nv, s);
  S.chh.reserve(nv, s);
  S.nch.reserve(2, s);
  CUDA_CHECK(cudaMemsetAsync(S.nch.p, 0, 2 * sizeof(unsigned long long), s));
  k_changed_split<<<grid_for(nv, 256, num_sms() * 8), 256, 0, s>>>(
      A.colors, S.prev_valid ? S.prev.p : nullptr, nv, A.rowptr, S.chl.p, S.chh.p, S.nch.p);
  FreeDet a{A.rowptr, A.col, A.colors, A.owned_flag, A.gids, A.deg, A.recolor_degrees, false, KillRoute{}};
  k_free_heavy<1, false><<<num_sms() * 4, DET_HEAVY_THREADS, 0, s>>>(a, S.chh.p, S.nch.p + 1, conflicts);
  k_free_light<1, false><<<grid_for(nv * 32, 256, num_sms() * 16), 256, 0, s>>>(a, S.chl.p, S.nch.p, conflicts);
  count_launch(3);
  CUDA_CHECK(cudaGetLastError());
  S.prev.reserve(nv, s);
  CUDA_CHECK(cudaMemcpyAsync(S.prev.p, A.colors, sizeof(i32) * nv, cudaMemcpyDeviceToDevice, s));
  S.prev_valid = true;
}

void run_detect_free_lists(const DetectArgs& A, i64 nv, const FreeList* lists, int nlists, const KillRoute& kr,
                           DetectScratch& S, unsigned long long* conflicts, cudaStream_t s) {
  i64 cap = 0;
  for (int i = 0; i < nlists; i++) cap += lists[i].cap;
  S.chl.reserve(std::max<i64>(cap, 1), s);
  S.chh.reserve(std::max<i64>(cap, 1), s);
  S.nch.reserve(2, s);
  CUDA_CHECK(cudaMemsetAsync(S.nch.p, 0, 2 * sizeof(unsigned long long), s));
  for (int i = 0; i < nlists; i++) {
    if (lists[i].cap <= 0) continue;
    k_split_list<<<grid_for(lists[i].cap, 256, num_sms() * 8), 256, 0, s>>>(
        lists[i].ids, lists[i].n_dev, A.rowptr, A.colors, A.dist == 1 ? DET_HEAVY : DET_HEAVY / 32, S.chl.p,
        S.chh.p, S.nch.p);
    count_launch();
  }
  FreeDet a{A.rowptr, A.col, A.colors, A.owned_flag, A.gids, A.deg, A.recolor_degrees, true, kr};
  FREE_DET_DISPATCH(k_free_heavy, num_sms() * 4, DET_HEAVY_THREADS, a, S.chh.p, S.nch.p + 1, conflicts);
  FREE_DET_DISPATCH(k_free_light, grid_for(std::max<i64>(cap, 1) * 32, 256, num_sms() * 16), 256, a, S.chl.p,
                    S.nch.p, conflicts);
  CUDA_CHECK(cudaGetLastError());
}

static void resolve_events(const DetectArgs& A, DetectScratch& S, i64 E, unsigned long long* conflicts_dev,
                           i64 num_vertices, cudaStream_t s);

// Keyed D1 event emission from `src` (detection rows, or changed vertices): short
// rows by lanes, long rows in SEG-entry segments by warps; returns E, the events in
// S.ev in scan order.
static i64 keyed_events(const DetectArgs& A, const DevDetect& a, DetectScratch& S, const i32* src, i64 nsrc,
                        bool rows_mode, cudaStream_t s) {
  S.cnt.reserve(nsrc, s);
  S.off.reserve(nsrc, s);
  S.total.reserve(1, s);
  S.nch.reserve(1, s);
  // short rows by lanes (k_emit_short), long ones in segments (k_changed_events)
  k_changed_nseg<<<grid_for(nsrc, 256, num_sms() * 16), 256, 0, s>>>(A.rowptr, src, nsrc, S.cnt.p, true);
  count_launch();
  exclusive_scan_i64(S.cnt.p, S.off.p, nsrc, s);
  k_total<<<1, 1, 0, s>>>(S.cnt.p, S.off.p, nsrc, S.total.p);
  count_launch();
  CUDA_CHECK(cudaMemsetAsync(S.nch.p, 0, sizeof(unsigned long long), s));
  i64 nitems = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nitems, S.total.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  const int gs = grid_for(nsrc, 256, num_sms() * 16);
  const int gw = grid_for(std::max<i64>(nitems, 1) * 32, 256, num_sms() * 16);
  // one emission pass into a buffer sized by the previous call; a second, exact one
  // only when that was too small
  auto emit = [&](u64* keys, unsigned long long cap) {
    if (rows_mode) {
      k_emit_short<true, true><<<gs, 256, 0, s>>>(A.rowptr, A.col, A.colors, A.owned_flag, src, nsrc, S.nch.p, keys,
                                                  cap);
      if (nitems)
        k_changed_events<true, true><<<gw, 256, 0, s>>>(A.rowptr, A.col, A.colors, A.owned_flag, src, nsrc, S.off.p,
                                                        nitems, S.nch.p, keys, cap);
      count_launch(nitems ? 2 : 1);
    } else {
      k_emit_short<true, false><<<gs, 256, 0, s>>>(A.rowptr, A.col, A.colors, A.owned_flag, src, nsrc, S.nch.p, keys,
                                                   cap);
      if (nitems)
        k_changed_events<true, false><<<gw, 256, 0, s>>>(A.rowptr, A.col, A.colors, A.owned_flag, src, nsrc,
                                                         S.off.p, nitems, S.nch.p, keys, cap);
      count_launch(nitems ? 2 : 1);
    }
  };
  i64 cap = std::max<i64>(S.keys.n, (i64)1 << 20);
  S.keys.reserve(cap, s);
  emit(S.keys.p, (unsigned long long)cap);
  unsigned long long nku = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nku, S.nch.p, sizeof(nku), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  const i64 nk = (i64)nku;
  if (nk == 0) return 0;
  if (nk > cap) {
    S.keys.reserve(nk, s);
    CUDA_CHECK(cudaMemsetAsync(S.nch.p, 0, sizeof(unsigned long long), s));
    emit(S.keys.p, (unsigned long long)nk);
  }
  sort_u64(S.keys.p, nk, s);
  S.ukeys.reserve(nk, s);
  const i64 E = unique_u64(S.keys.p, nk, S.ukeys.p, s);
  CHROMA_REQUIRE(E < INT32_MAX, CHROMA_ERUNTIME, "too many conflict events");
  S.ev.reserve(E, s);
  k_keys_to_events<<<grid_for(E, 256, num_sms() * 16), 256, 0, s>>>(a, S.ukeys.p, E, S.ev.p);
  count_launch();
  return E;
}

void run_detect(const DetectArgs& A, i64 num_vertices, DetectScratch& S,
                unsigned long long* conflicts_dev, cudaStream_t s) {
  if (A.nrows <= 0) return;
  if (A.incremental && !A.sequential && A.dist == 1 && A.owned_flag) {
    run_detect_free_d1(A, num_vertices, S, conflicts_dev, s);
    return;
  }
  static const bool trace = std::getenv("CHROMA_DETECT_TRACE") != nullptr;
  cudaEvent_t te[6];
  int nte = 0;
  auto mark_t = [&]() {
    if (!trace) return;
    CUDA_CHECK(cudaEventCreate(&te[nte]));
    CUDA_CHECK(cudaEventRecord(te[nte++], s));
  };
  struct Report {
    std::function<void()> f;
    ~Report() { f(); }
  } report{[&]() {
    if (!trace || nte < 2) return;
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[detect] rows %lld", (long long)A.nrows);
    for (int i = 1; i < nte; i++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, te[i - 1], te[i]);
      std::fprintf(stderr, " | %.1f us", ms * 1e3);
    }
    std::fprintf(stderr, "\n");
    for (int i = 0; i < nte; i++) cudaEventDestroy(te[i]);
  }};
  mark_t();
  DevDetect a{A.rowptr, A.col, A.colors, A.gids, A.deg, A.rows, A.nrows, A.recolor_degrees};
  // remember this call's final colours for the next incremental call
  auto save_prev = [&]() {
    if (!A.incremental) return;
    S.prev.reserve(num_vertices, s);
    CUDA_CHECK(cudaMemcpyAsync(S.prev.p, A.colors, sizeof(i32) * num_vertices, cudaMemcpyDeviceToDevice, s));
    S.prev_valid = true;
  };
  static const bool no_keyed = std::getenv("CHROMA_DETECT_ROWSCAN") != nullptr;
  if (A.dist == 1 && A.owned_flag && A.sequential && !no_keyed) {
    // keyed emission: every equal-coloured scanned pair as a key (v << 32 | x),
    // sorted and de-duplicated into the reference's scan order
    const i32* src = A.rows;
    i64 nsrc = A.nrows;
    bool rows_mode = true;
    if (A.incremental && S.prev_valid) {
      // only rows around changed vertices can hold an event: walk from the changed side
      S.chl.reserve(num_vertices, s);
      S.narows.reserve(1, s);
      CUDA_CHECK(cudaMemsetAsync(S.narows.p, 0, sizeof(i64), s));
      k_changed_list<<<grid_for(num_vertices, 256, num_sms() * 16), 256, 0, s>>>(A.colors, S.prev.p, num_vertices,
                                                                                 S.chl.p, S.narows.p);
      count_launch();
      CUDA_CHECK(cudaMemcpyAsync(&nsrc, S.narows.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      src = S.chl.p;
      rows_mode = false;
    }
    mark_t();
    const i64 E = nsrc > 0 ? keyed_events(A, a, S, src, nsrc, rows_mode, s) : 0;
    mark_t();
    if (E > 0) resolve_events(A, S, E, conflicts_dev, num_vertices, s);
    mark_t();
    save_prev();
    return;
  }
  if (A.incremental && S.prev_valid) {
    S.mark.reserve(num_vertices, s);
    CUDA_CHECK(cudaMemsetAsync(S.mark.p, 0, num_vertices, s));
    const int gm = grid_for(num_vertices, 256, num_sms() * 16);
    if (A.dist == 1) k_mark_changed<1><<<gm, 256, 0, s>>>(A.rowptr, A.col, A.colors, S.prev.p, num_vertices, S.mark.p);
    else k_mark_changed<2><<<gm, 256, 0, s>>>(A.rowptr, A.col, A.colors, S.prev.p, num_vertices, S.mark.p);
    count_launch();
    S.arows.reserve(A.nrows, s);
    S.narows.reserve(1, s);
    // row flags reuse the fired buffer (sized later for events)
    S.fired.reserve(A.nrows, s);
    k_mark_flags<<<grid_for(A.nrows, 256, num_sms() * 16), 256, 0, s>>>(A.rows, A.nrows, S.mark.p, S.fired.p);
    count_launch();
    select_flagged_values(A.rows, S.fired.p, A.nrows, S.arows.p, S.narows.p, s);
    mark_t();
    i64 na = 0;
    CUDA_CHECK(cudaMemcpyAsync(&na, S.narows.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (na == 0) return;  // nothing changed: colours equal prev already
    a.rows = S.arows.p;
    a.nrows = na;
  }
  const i64 nrows = a.nrows;
  S.cnt.reserve(nrows, s);
  S.off.reserve(nrows, s);
  S.total.reserve(1, s);
  const int g = grid_for(nrows * 32, 256, num_sms() * 16);
  auto launch = [&](auto wr) {
    constexpr bool W = decltype(wr)::value;
    if (A.dist == 1) k_events_d1<W><<<grid_for(nrows, 256, num_sms() * 16), 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    else if (A.partial) k_events<2, true, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    else k_events<2, false, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    count_launch();
    CUDA_CHECK(cudaGetLastError());
  };
  launch(std::false_type{});
  exclusive_scan_i64(S.cnt.p, S.off.p, nrows, s);
  k_total<<<1, 1, 0, s>>>(S.cnt.p, S.off.p, nrows, S.total.p);
  count_launch();
  mark_t();
  i64 E = 0;
  CUDA_CHECK(cudaMemcpyAsync(&E, S.total.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (E == 0) {
    save_prev();
    return;
  }
  CHROMA_REQUIRE(E < INT32_MAX, CHROMA_ERUNTIME, "too many conflict events");
  S.ev.reserve(E, s);
  launch(std::true_type{});
  mark_t();
  resolve_events(A, S, E, conflicts_dev, num_vertices, s);
  mark_t();
  save_prev();
  mark_t();
}

// Resolve E ordered events in S.ev (fixed point over the event order, F5) and
// uncolour the fired losers; adds the number fired to *conflicts_dev.
static void resolve_events(const DetectArgs& A, DetectScratch& S, i64 E, unsigned long long* conflicts_dev,
                           i64 num_vertices, cudaStream_t s) {
  S.fired.reserve(E, s);
  S.kill.reserve(num_vertices, s);
  if (A.sequential && E > 32768) {
    S.result.reserve(4, s);
    CUDA_CHECK(cudaMemsetAsync(S.result.p, 0, 4 * sizeof(unsigned long long), s));
    unsigned* bar = reinterpret_cast<unsigned*>(S.result.p);
    int* changed = reinterpret_cast<int*>(S.result.p + 1);
    const int2* evp = S.ev.p;
    uint8_t* fp = S.fired.p;
    S.kill64.reserve(num_vertices, s);
    unsigned long long* kp = S.kill64.p;
    i32* cp = A.colors;
    void* args[] = {(void*)&evp, (void*)&E, (void*)&fp, (void*)&kp, (void*)&cp, (void*)&conflicts_dev, (void*)&bar,
                    (void*)&changed};
    CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_resolve_grid, dim3(num_sms()), dim3(1024), args, 0, s));
  } else {
    k_resolve<<<1, 1024, 0, s>>>(S.ev.p, E, S.fired.p, S.kill.p, A.colors, conflicts_dev, A.sequential);
  }
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace chroma
