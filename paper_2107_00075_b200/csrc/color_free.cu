// Free-running speculative colouring (AlgorithmConfig(algorithm="free")).
//
// The reference's two local modes are exact but inherently ordered (Gauss-Seidel,
// chroma/localcolor.py:161-165) or sweep-synchronous (Jacobi, 214-227).  The
// free-running mode keeps the paper's speculate-and-iterate structure (Alg. 1 of
// 2107.00075; the KokkosKernels VB kernel it runs on the GPU):
//
//   iteration 0   every pending vertex takes its first fit against whatever colours
//                 are visible (in place, no snapshot) -- one bandwidth-bound pass;
//   iteration k   (k >= 1, the few losers left) snapshot semantics: colours of
//                 pending neighbours are ignored and a vertex with r pending
//                 neighbours of larger id takes the (r+1)-th free colour instead of
//                 the first, so a dense core (an R-MAT hub clique) resolves in a few
//                 iterations instead of one vertex per iteration;
//   resolution    a vertex whose colour equals that of a larger-id member of its
//                 set loses (the reference's priority rule, chroma/localcolor.py:
//                 168-178), is uncoloured and goes to the next iteration.
//
// Tentative colours are stored negated until the resolution pass commits them, so
// "pending" is visible in the colour word itself (no side array).  The result is a
// proper colouring (every conflicting pair leaves its smaller endpoint uncoloured),
// not a bit-exact one.  Light vertices are processed one warp each, 32 per warp
// group (one atomic per group for the loser list); heavy rows (R-MAT hubs) one CTA
// each.  All passes are HBM/L2-bound gathers.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WORDS = 8;
constexpr int WIN = 32 * WORDS;
constexpr int HEAVY_THREADS = 512;

__device__ __forceinline__ i32 iabs(i32 x) { return x < 0 ? -x : x; }

// Visit the colouring set of v with `stride` cooperating threads, thread `t`.
template <int DIST, bool PARTIAL, typename F>
__device__ __forceinline__ void for_each_in_set(const i64* rowptr, const i32* col, i32 v, int t, int stride,
                                                F&& f) {
  const i64 rs = rowptr[v], re = rowptr[v + 1];
  if (DIST == 1) {
    // 4 column entries per thread in flight; the callback's gathers follow them
    constexpr int U = 4;
    for (i64 e0 = rs + t; e0 < re; e0 += (i64)U * stride) {
      i32 x[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const i64 e = e0 + (i64)u * stride;
        x[u] = e < re ? ld_stream(col + e) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; u++)
        if (x[u] >= 0) f(x[u]);
    }
  } else if (stride == 32) {
    for (i64 e = rs; e < re; e++) {
      const i32 u = col[e];
      if (!PARTIAL && t == 0) f(u);
      const i64 ue = rowptr[u + 1];
      for (i64 g = rowptr[u] + t; g < ue; g += 32) {
        const i32 x = col[g];
        if (x != v) f(x);
      }
    }
  } else {
    for (i64 e = rs + t; e < re; e += stride) {
      const i32 u = col[e];
      if (!PARTIAL) f(u);
      const i64 ue = rowptr[u + 1];
      for (i64 g = rowptr[u]; g < ue; g++) {
        const i32 x = col[g];
        if (x != v) f(x);
      }
    }
  }
}

// Accumulate forbidden colours [base, base+WIN) and (snapshot mode) the number of
// pending set members with larger id.
struct Acc {
  u32 m[WORDS];
  int rank;
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int w = 0; w < WORDS; w++) m[w] = 0;
    rank = 0;
  }
  __device__ __forceinline__ void add(i32 x, i32 v, i32 c, i32 base, bool snapshot) {
    if (snapshot && c <= 0) {
      rank += x > v;
      return;
    }
    const i32 o = iabs(c) - base;
    if (o >= 0 && o < WIN) m[o >> 5] |= 1u << (o & 31);
  }
};

// (skip+1)-th free colour of the window, 1-based; 0 (and skip reduced) if none.
__device__ __forceinline__ int pick(const u32* mw, int& skip) {
#pragma unroll
  for (int w = 0; w < WORDS; w++) {
    u32 z = ~mw[w];
    const int c = __popc(z);
    if (skip >= c) {
      skip -= c;
      continue;
    }
    for (int k = 0; k < skip; k++) z &= z - 1;
    return w * 32 + __ffs(z);
  }
  return 0;
}

// G lanes per vertex (G = 8 for short rows: four vertices in flight per warp; 32 for
// the rest).  Groups of a warp are independent: reductions use the group's lane mask.
template <int DIST, bool PARTIAL, int G>
__global__ void k_color_light(const i64* rowptr, const i32* col, i32* colors, const i32* list, const i64* n_dev,
                              bool snapshot, int rank_cap) {
  const int lane = threadIdx.x & 31, t = lane % G;
  const unsigned gmask = G == 32 ? FULL : ((1u << G) - 1) << (lane / G * G);
  const i64 n = *n_dev;
  const i64 grp = ((blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5) * (32 / G) + lane / G;
  const i64 ngrp = (((i64)gridDim.x * blockDim.x) >> 5) * (32 / G);
  for (i64 i = grp; i < n; i += ngrp) {
    const i32 v = list[i];
    int skip = -1;
    for (i32 base = 1;; base += WIN) {
      Acc a;
      a.clear();
      const bool count = skip < 0;
      for_each_in_set<DIST, PARTIAL>(rowptr, col, v, t, G, [&](i32 x) {
        a.add(x, v, ld_relaxed_nb(colors + x), base, snapshot && count);
      });
      if (count) skip = snapshot ? min((int)__reduce_add_sync(gmask, (unsigned)a.rank), rank_cap) : 0;
      u32 mw[WORDS];
#pragma unroll
      for (int w = 0; w < WORDS; w++) mw[w] = __reduce_or_sync(gmask, a.m[w]);
      const int r = pick(mw, skip);
      if (r) {
        if (t == 0) st_relaxed(colors + v, -(base + r - 1));
        break;
      }
    }
  }
}

template <int DIST, bool PARTIAL>
__global__ void __launch_bounds__(HEAVY_THREADS) k_color_heavy(const i64* rowptr, const i32* col, i32* colors,
                                                               const i32* list, const i64* n_dev, bool snapshot,
                                                               int rank_cap) {
  __shared__ u32 sm[WORDS];
  __shared__ int srank, sdone;
  const int t = threadIdx.x, lane = t & 31;
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x; i < n; i += gridDim.x) {
    const i32 v = list[i];
    int skip = -1;
    for (i32 base = 1;; base += WIN) {
      if (t < WORDS) sm[t] = 0;
      if (t == 0) srank = 0, sdone = 0;
      __syncthreads();
      Acc a;
      a.clear();
      const bool count = skip < 0;
      for_each_in_set<DIST, PARTIAL>(rowptr, col, v, t, HEAVY_THREADS, [&](i32 x) {
        a.add(x, v, ld_relaxed_nb(colors + x), base, snapshot && count);
      });
#pragma unroll
      for (int w = 0; w < WORDS; w++) {
        const u32 mw = __reduce_or_sync(FULL, a.m[w]);
        if (lane == 0 && mw) atomicOr(&sm[w], mw);
      }
      const int rk = __reduce_add_sync(FULL, a.rank);
      if (lane == 0 && rk) atomicAdd(&srank, rk);
      __syncthreads();
      if (count) skip = snapshot ? min(srank, rank_cap) : 0;
      __syncthreads();
      if (t == 0) {
        u32 mw[WORDS];
        for (int w = 0; w < WORDS; w++) mw[w] = sm[w];
        int s2 = skip;
        const int r = pick(mw, s2);
        if (r) {
          st_relaxed(colors + v, -(base + r - 1));
          sdone = 1;
        }
        srank = s2;  // carried into the next window
      }
      __syncthreads();
      const bool done = sdone;
      skip = srank;
      __syncthreads();
      if (done) break;
    }
  }
}

// Tiny rows (distance 1, degree <= 63): one thread per vertex.  First fit of a row of
// d entries is at most d + 1 <= 64, so one 64-bit mask covers it (no window loop,
// no lane reductions); column entries and colours are gathered in batches of 8 so
// a thread keeps 8 independent loads in flight.  Isolated vertices take colour 1.
constexpr int TB = 8;
__global__ void k_color_tiny(const i64* rowptr, const i32* col, i32* colors, const i32* list, const i64* n_dev) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = list[i];
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    u64 m = 0;
    for (i64 e0 = rs; e0 < re; e0 += TB) {
      i32 x[TB], c[TB];
#pragma unroll
      for (int u = 0; u < TB; u++) x[u] = e0 + u < re ? ld_stream(col + e0 + u) : -1;
#pragma unroll
      for (int u = 0; u < TB; u++) c[u] = x[u] >= 0 ? ld_relaxed_nb(colors + x[u]) : 0;
#pragma unroll
      for (int u = 0; u < TB; u++) {
        const i32 a = iabs(c[u]);
        if (a >= 1 && a <= 64) m |= 1ull << (a - 1);
      }
    }
    st_relaxed(colors + v, -__ffsll((long long)~m));
  }
}

__global__ void k_losers_tiny(const i64* rowptr, const i32* col, i32* colors, const i32* list, const i64* n_dev,
                              i32* next, unsigned long long* nnext) {
  const int lane = threadIdx.x & 31;
  const i64 n = *n_dev;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + lane;
    bool lose = false;
    i32 v = 0;
    if (i < n) {
      v = list[i];
      const i32 c = iabs(ld_relaxed_nb(colors + v));
      const i64 rs = rowptr[v], re = rowptr[v + 1];
      for (i64 e0 = rs; e0 < re && !lose; e0 += TB) {
        i32 x[TB], cx[TB];
#pragma unroll
        for (int u = 0; u < TB; u++) x[u] = e0 + u < re ? ld_stream(col + e0 + u) : -1;
#pragma unroll
        for (int u = 0; u < TB; u++) cx[u] = x[u] > v ? ld_relaxed_nb(colors + x[u]) : 0;
#pragma unroll
        for (int u = 0; u < TB; u++) lose |= x[u] > v && iabs(cx[u]) == c;
      }
      st_relaxed(colors + v, lose ? 0 : c);
    }
    const u32 m = __ballot_sync(FULL, lose);
    unsigned long long o = 0;
    if (lane == 0 && m) o = atomicAdd(nnext, (unsigned long long)__popc(m));
    o = __shfl_sync(FULL, o, 0);
    if (lose) next[o + __popc(m & ((1u << lane) - 1))] = v;
  }
}

// Resolution: v keeps its colour unless a larger-id member of its set has it.
// G lanes per vertex as above; losers are a small fraction, one atomic each.
template <int DIST, bool PARTIAL, int G>
__global__ void k_losers_light(const i64* rowptr, const i32* col, i32* colors, const i32* list, const i64* n_dev,
                               i32* next, unsigned long long* nnext) {
  const int lane = threadIdx.x & 31, t = lane % G;
  const unsigned gmask = G == 32 ? FULL : ((1u << G) - 1) << (lane / G * G);
  const i64 n = *n_dev;
  const i64 grp = ((blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5) * (32 / G) + lane / G;
  const i64 ngrp = (((i64)gridDim.x * blockDim.x) >> 5) * (32 / G);
  for (i64 i = grp; i < n; i += ngrp) {
    const i32 v = list[i];
    const i32 c = iabs(ld_relaxed(colors + v));
    bool hit = false;
    for_each_in_set<DIST, PARTIAL>(rowptr, col, v, t, G, [&](i32 x) {
      if (x > v && iabs(ld_relaxed_nb(colors + x)) == c) hit = true;
    });
    const bool any = __any_sync(gmask, hit);
    if (t == 0) {
      st_relaxed(colors + v, any ? 0 : c);
      if (any) next[atomicAdd(nnext, 1ull)] = v;
    }
  }
}

template <int DIST, bool PARTIAL>
__global__ void __launch_bounds__(HEAVY_THREADS) k_losers_heavy(const i64* rowptr, const i32* col, i32* colors,
                                                                const i32* list, const i64* n_dev, i32* next,
                                                                unsigned long long* nnext) {
  __shared__ int shit;
  const int t = threadIdx.x;
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x; i < n; i += gridDim.x) {
    const i32 v = list[i];
    if (t == 0) shit = 0;
    __syncthreads();
    const i32 c = iabs(ld_relaxed(colors + v));
    bool hit = false;
    for_each_in_set<DIST, PARTIAL>(rowptr, col, v, t, HEAVY_THREADS, [&](i32 x) {
      if (x > v && iabs(ld_relaxed_nb(colors + x)) == c) hit = true;
    });
    if (__any_sync(FULL, hit) && (t & 31) == 0) shit = 1;
    __syncthreads();
    if (t == 0) {
      st_relaxed(colors + v, shit ? 0 : c);
      if (shit) next[atomicAdd(nnext, 1ull)] = v;
    }
    __syncthreads();
  }
}

// worklist -> tiny / light / heavy lists by row length.  Each 256-thread block takes
// tiles of 256 x SPI entries; per-warp ballots are combined in shared memory so a
// tile costs one global atomic per class (appends are unordered).
constexpr int SPI = 8;
__global__ void __launch_bounds__(256) k_split(const i32* wl, const i64* n_dev, const i64* rowptr, i64 tiny_deg,
                                               i64 heavy_deg, i32* tiny, i32* light, i32* heavy,
                                               unsigned long long* cnt /* [light, heavy, tiny] */) {
  __shared__ u32 wtot[3][8];
  __shared__ unsigned long long base[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 below = (1u << lane) - 1;
  const i64 n = *n_dev;
  constexpr i64 TILE = 256 * SPI;
  i32* out[3] = {light, heavy, tiny};
  for (i64 t0 = (i64)blockIdx.x * TILE; t0 < n; t0 += (i64)gridDim.x * TILE) {
    i32 v[SPI];
    int cls[SPI];
    u32 run[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < SPI; k++) {
      const i64 i = t0 + (i64)k * 256 + threadIdx.x;
      v[k] = i < n ? wl[i] : -1;
    }
#pragma unroll
    for (int k = 0; k < SPI; k++) {
      const i64 d = v[k] >= 0 ? rowptr[v[k] + 1] - rowptr[v[k]] : 0;
      cls[k] = v[k] < 0 ? -1 : d > heavy_deg ? 1 : d <= tiny_deg ? 2 : 0;
#pragma unroll
      for (int c = 0; c < 3; c++) run[c] += __popc(__ballot_sync(FULL, cls[k] == c));
    }
    if (lane < 3) wtot[lane][warp] = run[lane];
    __syncthreads();
    if (threadIdx.x < 3) {
      u32 tot = 0;
      for (int w = 0; w < 8; w++) tot += wtot[threadIdx.x][w];
      base[threadIdx.x] = tot ? atomicAdd(cnt + threadIdx.x, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    unsigned long long o[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      o[c] = base[c];
      for (int w = 0; w < warp; w++) o[c] += wtot[c][w];
    }
#pragma unroll
    for (int k = 0; k < SPI; k++) {
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const u32 m = __ballot_sync(FULL, cls[k] == c);
        if (cls[k] == c) out[c][o[c] + __popc(m & below)] = v[k];
        o[c] += __popc(m);
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- heavy waves
// Heavy rows (hubs) form a dense core in which speculation serialises (all members
// see one snapshot and pick one colour; one keeps it per iteration).  They are
// coloured first, exactly, in waves of C = #CTAs vertices (one per CTA, one CTA per
// SM, cooperative launch): each CTA scans its member's row, recording the committed
// colours it sees (mask of WWORDS*32 colours) and which other members of the wave
// are in its set (members are marked in the colour word as -(slot+1)); then one warp
// replays the wave in slot order -- first fit over (row mask | colours chosen by
// earlier adjacent members) -- so no two adjacent hubs ever collide.  Light
// vertices are uncoloured or committed at this point, so they never interfere.
__device__ __forceinline__ u64 gtime() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int WWORDS = 64;            // 2048 colours per heavy mask
constexpr int MAXC = 160;             // >= #SMs
constexpr int AWORDS = (MAXC + 31) / 32;

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nb) {
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
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// First colour (1-based) free of row | extra over the WWORDS*32-colour mask, warp-wide;
// 0 if none.
__device__ __forceinline__ int first_free(const u32* row, const u32* extra, int lane) {
#pragma unroll
  for (int h = 0; h < WWORDS / 32; h++) {
    const int w = h * 32 + lane;
    const u32 fr = ~(row[w] | (extra ? extra[w] : 0u));
    const u32 bl = __ballot_sync(FULL, fr != 0);
    if (bl) {
      const int L = __ffs(bl) - 1;
      const u32 frL = __shfl_sync(FULL, fr, L);
      return (h * 32 + L) * 32 + __ffs(frL);
    }
  }
  return 0;
}

template <int DIST, bool PARTIAL>
__global__ void __launch_bounds__(HEAVY_THREADS, 1)
    k_heavy_waves(const i64* rowptr, const i32* col, i32* colors, const i32* heavy, i64 n, u32* gF, u32* gA,
                  int* gOvf, unsigned* bar, i32* light, unsigned long long* nlight, u64* gDbg) {
  __shared__ u32 sF[WWORDS];
  __shared__ u32 sA[AWORDS];
  __shared__ int sOvf;
  __shared__ u32 sW[MAXC][WWORDS + 1];  // +1: rows start in different banks
  __shared__ i32 sV[MAXC], sC[MAXC];
  __shared__ u32 sX[WWORDS];
  __shared__ u32 sAdj[MAXC * AWORDS];
  __shared__ int sOv[MAXC];
  const int b = blockIdx.x, C = gridDim.x, t = threadIdx.x, lane = t & 31;
  if (t < WWORDS) sX[t] = 0;
  if (t == 0 && b < n) st_relaxed(colors + heavy[b], -(b + 1));
  grid_barrier(bar, C);
  for (i64 base = 0; base < n; base += C) {
    const int m = (int)min((i64)C, n - base);
    const u64 t0 = (b == 0 && t == 0) ? gtime() : 0;
    if (b < m) {
      const i32 v = heavy[base + b];
      for (int i = t; i < WWORDS; i += blockDim.x) sF[i] = 0;
      if (t < AWORDS) sA[t] = 0;
      if (t == 0) sOvf = 0;
      __syncthreads();
      u32 r[WORDS];
#pragma unroll
      for (int w = 0; w < WORDS; w++) r[w] = 0;
      bool ovf = false;
      auto visit = [&](i32 c) {
        if (c < 0) {
          const int sl = -c - 1;
          atomicOr(&sA[sl >> 5], 1u << (sl & 31));
        } else if (c > 0) {
          const i32 o = c - 1;
          if (o < WIN) r[o >> 5] |= 1u << (o & 31);
          else if (o < WWORDS * 32) atomicOr(&sF[o >> 5], 1u << (o & 31));
          else ovf = true;
        }
      };
      if (DIST == 1) {
        // 8 independent gathers in flight per thread (hub rows are long)
        constexpr int U = 8;
        const i64 rs = rowptr[v], re = rowptr[v + 1];
        for (i64 e0 = rs + t; e0 < re; e0 += (i64)U * HEAVY_THREADS) {
          i32 x[U], c[U];
#pragma unroll
          for (int u = 0; u < U; u++) {
            const i64 e = e0 + (i64)u * HEAVY_THREADS;
            x[u] = e < re ? col[e] : -1;
          }
#pragma unroll
          for (int u = 0; u < U; u++) c[u] = x[u] >= 0 ? ld_relaxed(colors + x[u]) : 0;
#pragma unroll
          for (int u = 0; u < U; u++) visit(c[u]);
        }
      } else {
        for_each_in_set<DIST, PARTIAL>(rowptr, col, v, t, HEAVY_THREADS,
                                       [&](i32 x) { visit(ld_relaxed(colors + x)); });
      }
#pragma unroll
      for (int w = 0; w < WORDS; w++) {
        const u32 x = __reduce_or_sync(FULL, r[w]);
        if (lane == 0 && x) atomicOr(&sF[w], x);
      }
      if (__any_sync(FULL, ovf) && lane == 0) sOvf = 1;
      __syncthreads();
      for (int i = t; i < WWORDS; i += blockDim.x) gF[(i64)b * WWORDS + i] = sF[i];
      if (t < AWORDS) gA[b * AWORDS + t] = sA[t];
      if (t == 0) gOvf[b] = sOvf;
    }
    const u64 t1 = (b == 0 && t == 0) ? gtime() : 0; u64 t2 = 0;
    grid_barrier(bar, C);
    if (b == 0 && t == 0 && gDbg) { const u64 tn = gtime(); atomicAdd((unsigned long long*)(gDbg + 1), (unsigned long long)(tn - t1)); t2 = tn; }
    if (b == 0) {
      // stage the wave's masks and adjacency in shared memory, then replay it
      for (int i = t; i < m * WWORDS; i += blockDim.x) sW[i / WWORDS][i % WWORDS] = __ldcg(gF + i);
      for (int i = t; i < m * AWORDS; i += blockDim.x) sAdj[i] = __ldcg(gA + i);
      for (int i = t; i < m; i += blockDim.x) sOv[i] = __ldcg(gOvf + i), sV[i] = heavy[base + i];
      __syncthreads();
      if (t == 0 && gDbg) atomicAdd((unsigned long long*)(gDbg + 4), (unsigned long long)(gtime() - t2));
      // (a) provisional first fit of every member against its row mask, one warp each
      const int warp = t >> 5, nwarp = blockDim.x >> 5;
      const long long c0 = clock64();
      for (int j = warp; j < m; j += nwarp) {
        const int c = sOv[j] ? 0 : first_free(sW[j], nullptr, lane);
        if (lane == 0) sC[j] = c;
      }
      __syncthreads();
      // (b) ordered repair: member j keeps its pick unless an earlier adjacent member
      // holds that colour; then it takes the first colour free of both.  Either way
      // the result equals the sequential first fit in slot order.
      if (warp == 0) {
        for (int j = 0; j < m; j++) {
          const int cj = sC[j];
          if (cj == 0) continue;  // beyond the mask: constrains no one, finished later
          u32 adj[AWORDS];
#pragma unroll
          for (int q = 0; q < AWORDS; q++) adj[q] = sAdj[j * AWORDS + q];
          bool clash = false;
#pragma unroll
          for (int q = 0; q < AWORDS; q++) {
            const int k = q * 32 + lane;
            if (k < j && (adj[q] >> lane & 1) && sC[k] == cj) clash = true;
          }
          if (__any_sync(FULL, clash)) {
#pragma unroll
            for (int q = 0; q < AWORDS; q++) {
              const int k = q * 32 + lane;
              if (k < j && (adj[q] >> lane & 1)) {
                const int o = sC[k] - 1;
                if (o >= 0 && o < WWORDS * 32) atomicOr(&sX[o >> 5], 1u << (o & 31));
              }
            }
            __syncwarp();
            const int c = first_free(sW[j], sX, lane);
            __syncwarp();
            sX[lane] = 0;
            sX[lane + 32] = 0;
            if (lane == 0) sC[j] = c;
            __syncwarp();
          }
        }
      }
      const long long c1 = clock64();
      __syncthreads();
      for (int j = t; j < m; j += blockDim.x) {
        const i32 v = sV[j], c = sC[j];
        st_relaxed(colors + v, c);
        if (!c) light[atomicAdd(nlight, 1ull)] = v;  // beyond the mask: finish it speculatively
      }
      if (t == 0 && gDbg) {
        atomicAdd((unsigned long long*)(gDbg + 5), (unsigned long long)(c1 - c0));
        atomicAdd((unsigned long long*)(gDbg + 6), (unsigned long long)m);
      }
    }
    if (b == 0 && t == 0 && gDbg) { atomicAdd((unsigned long long*)(gDbg + 0), (unsigned long long)(t1 - t0)); atomicAdd((unsigned long long*)(gDbg + 2), (unsigned long long)(gtime() - t2)); }
    if (t == 0 && base + C + b < n) st_relaxed(colors + heavy[base + C + b], -(b + 1));
    const u64 t3 = (b == 0 && t == 0) ? gtime() : 0;
    grid_barrier(bar, C);
    if (b == 0 && t == 0 && gDbg) { const u64 tn = gtime(); atomicAdd((unsigned long long*)(gDbg + 3), (unsigned long long)(tn - t3)); }
  }
}

__global__ void k_degree_keys(const i32* v, i64 n, const i64* rowptr, u64* keys) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 x = v[i];
    const u64 d = (u64)(rowptr[x + 1] - rowptr[x]);
    keys[i] = ((u64)(0xffffffffu - (u32)(d > 0xffffffffull ? 0xffffffffull : d)) << 32) | (u32)x;
  }
}
__global__ void k_unkey(const u64* keys, i64 n, i32* v) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    v[i] = (i32)(keys[i] & 0xffffffffull);
}

#define FREE_DISPATCH(KERNEL, GRID, BLOCK, ...)                                              \
  do {                                                                                      \
    if (dist == 1) KERNEL<1, false><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                    \
    else if (partial) KERNEL<2, true><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                  \
    else KERNEL<2, false><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                              \
    count_launch();                                                                         \
    CUDA_CHECK(cudaGetLastError());                                                         \
  } while (0)

#define FREE_DISPATCH_G(KERNEL, G, GRID, BLOCK, ...)                                        \
  do {                                                                                      \
    if (dist == 1) KERNEL<1, false, G><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                 \
    else if (partial) KERNEL<2, true, G><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);               \
    else KERNEL<2, false, G><<<GRID, BLOCK, 0, s>>>(__VA_ARGS__);                           \
    count_launch();                                                                         \
    CUDA_CHECK(cudaGetLastError());                                                         \
  } while (0)

}  // namespace

void launch_free_split(const i32* wl, const i64* n_dev, i64 n_max, const i64* rowptr, i64 tiny_deg, i64 heavy_deg,
                       FreeLists& f, int p, cudaStream_t s) {
  CUDA_CHECK(cudaMemsetAsync(f.cnt + 3 * p, 0, 3 * sizeof(i64), s));
  if (n_max <= 0) return;
  k_split<<<grid_for(n_max, 256 * SPI, num_sms() * 8), 256, 0, s>>>(
      wl, n_dev, rowptr, tiny_deg, heavy_deg, f.tiny[p], f.light[p], f.heavy[p],
      reinterpret_cast<unsigned long long*>(f.cnt + 3 * p));
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

void launch_free_iteration(const i64* rowptr, const i32* col, i32* colors, FreeLists& f, int p, const i64* nmax,
                           int rank_cap, int dist, bool partial, cudaStream_t s) {
  const bool snapshot = rank_cap > 0;
  const int q = p ^ 1;
  const i64 nlight_max = nmax[0], nheavy_max = nmax[1], ntiny_max = nmax[2];
  CUDA_CHECK(cudaMemsetAsync(f.cnt + 3 * q, 0, 3 * sizeof(i64), s));
  auto* next_cnt = reinterpret_cast<unsigned long long*>(f.cnt + 3 * q);
  const i64* cnt = f.cnt + 3 * p;
  const int gh = (int)std::max<i64>(1, std::min<i64>(nheavy_max, num_sms() * 4));
  const int gl = grid_for(std::max<i64>(nlight_max, 1) * 32, 256, num_sms() * 16);
  const int gt = grid_for(std::max<i64>(ntiny_max, 1) * 8, 256, num_sms() * 16);
  if (nheavy_max > 0)
    FREE_DISPATCH(k_color_heavy, gh, HEAVY_THREADS, rowptr, col, colors, f.heavy[p], cnt + 1, snapshot, rank_cap);
  if (nlight_max > 0)
    FREE_DISPATCH_G(k_color_light, 32, gl, 256, rowptr, col, colors, f.light[p], cnt + 0, snapshot, rank_cap);
  // tiny rows exist for distance 1 only (launch_free_split); thread per vertex
  const bool tiny_thread = dist == 1 && !snapshot;
  const int gtt = grid_for(std::max<i64>(ntiny_max, 1), 256, num_sms() * 16);
  if (ntiny_max > 0 && tiny_thread) {
    k_color_tiny<<<gtt, 256, 0, s>>>(rowptr, col, colors, f.tiny[p], cnt + 2);
    count_launch();
  } else if (ntiny_max > 0) {
    FREE_DISPATCH_G(k_color_light, 8, gt, 256, rowptr, col, colors, f.tiny[p], cnt + 2, snapshot, rank_cap);
  }
  if (nheavy_max > 0)
    FREE_DISPATCH(k_losers_heavy, gh, HEAVY_THREADS, rowptr, col, colors, f.heavy[p], cnt + 1, f.heavy[q],
                  next_cnt + 1);
  if (nlight_max > 0)
    FREE_DISPATCH_G(k_losers_light, 32, gl, 256, rowptr, col, colors, f.light[p], cnt + 0, f.light[q], next_cnt + 0);
  if (ntiny_max > 0 && tiny_thread) {
    k_losers_tiny<<<gtt, 256, 0, s>>>(rowptr, col, colors, f.tiny[p], cnt + 2, f.tiny[q], next_cnt + 2);
    count_launch();
  } else if (ntiny_max > 0) {
    FREE_DISPATCH_G(k_losers_light, 8, gt, 256, rowptr, col, colors, f.tiny[p], cnt + 2, f.tiny[q], next_cnt + 2);
  }
}

}  // namespace chroma

namespace chroma {
void launch_free_heavy(const i64* rowptr, const i32* col, i32* colors, i32* heavy, i64 n, i32* light,
                       i64* nlight, int dist, bool partial, FreeWaveScratch& ws, cudaStream_t s) {
  if (n <= 0) return;
  // largest degree first (ties by id): balances the waves' row scans and is the
  // classic LDF order for the dense core
  ws.keys.reserve(n, s);
  k_degree_keys<<<grid_for(n, 256, num_sms() * 8), 256, 0, s>>>(heavy, n, rowptr, ws.keys.p);
  sort_u64(ws.keys.p, n, s);
  k_unkey<<<grid_for(n, 256, num_sms() * 8), 256, 0, s>>>(ws.keys.p, n, heavy);
  count_launch(2);
  const int C = std::min(num_sms(), MAXC);
  ws.F.reserve((i64)C * WWORDS, s);
  ws.A.reserve((i64)C * AWORDS, s);
  ws.ovf.reserve(C, s);
  ws.bar.reserve(2, s);
  CUDA_CHECK(cudaMemsetAsync(ws.bar.p, 0, 2 * sizeof(unsigned), s));
  u32* F = ws.F.p;
  u32* A = ws.A.p;
  int* ovf = ws.ovf.p;
  unsigned* bar = ws.bar.p;
  auto* nl = reinterpret_cast<unsigned long long*>(nlight);
  static const bool prof = std::getenv("CHROMA_FREE_TRACE") != nullptr;
  u64* dbg = nullptr;
  if (prof) {
    ws.dbg.reserve(7, s);
    CUDA_CHECK(cudaMemsetAsync(ws.dbg.p, 0, 7 * sizeof(u64), s));
    dbg = ws.dbg.p;
  }
  void* args[] = {(void*)&rowptr, (void*)&col, (void*)&colors, (void*)&heavy, (void*)&n, (void*)&F,
                  (void*)&A,      (void*)&ovf, (void*)&bar,    (void*)&light, (void*)&nl,  (void*)&dbg};
  const void* k = dist == 1 ? (const void*)k_heavy_waves<1, false>
                  : partial ? (const void*)k_heavy_waves<2, true>
                            : (const void*)k_heavy_waves<2, false>;
  CUDA_CHECK(cudaLaunchCooperativeKernel(k, dim3(C), dim3(HEAVY_THREADS), args, 0, s));
  count_launch();
  if (prof) {
    u64 h[7];
    CUDA_CHECK(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[free] waves=%lld cta0 scan %.1f us, barrier1 %.1f us, pick %.1f us, barrier2 %.1f us (stage %.1f us) loop %llu cycles / %llu picks\n",
                 (long long)((n + C - 1) / C), h[0] * 1e-3, h[1] * 1e-3, h[2] * 1e-3, h[3] * 1e-3, h[4] * 1e-3,
                 (unsigned long long)h[5], (unsigned long long)h[6]);
  }
}
}  // namespace chroma
