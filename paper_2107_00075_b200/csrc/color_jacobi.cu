// Jacobi (synchronous) speculative sweeps -- the reference's deterministic=False
// path, reproduced exactly:
//   chroma/localcolor.py:214-227 (D1): every pending vertex proposes first fit
//   against one snapshot; v loses iff an equal-coloured neighbour has a larger
//   local id or is outside the round (VB and EB select the same set, F3).
//   chroma/localcolor.py:292-303 (D2/PD2): same proposal over the distance-2
//   forbidden set; the net-based loser scan (230-271) keeps the largest member of
//   every equal-colour group of every net, which for a pending v is "v loses iff an
//   equal-coloured x in its forbidden set has x > v or is outside the round".
// One warp per pending vertex; colour windows of 256 are OR-reduced across lanes.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WORDS = 8;
constexpr int WIN = 32 * WORDS;

template <int DIST, bool PARTIAL, typename F>
__device__ __forceinline__ void for_each_in_set(const i64* rowptr, const i32* col, i32 v, int lane, F&& f) {
  const i64 rs = rowptr[v], re = rowptr[v + 1];
  if (DIST == 1) {
    for (i64 e = rs + lane; e < re; e += 32) f(col[e]);
  } else {
    for (i64 e = rs; e < re; e++) {
      const i32 u = col[e];
      if (!PARTIAL && lane == 0) f(u);
      const i64 us = rowptr[u], ue = rowptr[u + 1];
      for (i64 g = us + lane; g < ue; g += 32) {
        const i32 x = col[g];
        if (x != v) f(x);
      }
    }
  }
}

template <int DIST, bool PARTIAL>
__global__ void k_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pending,
                          const i64* np_dev, i32* prop) {
  const int lane = threadIdx.x & 31;
  const i64 np = *np_dev;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < np; i += nwarps) {
    const i32 v = pending[i];
    for (i32 base = 1;; base += WIN) {
      u32 m[WORDS];
#pragma unroll
      for (int w = 0; w < WORDS; w++) m[w] = 0;
      for_each_in_set<DIST, PARTIAL>(rowptr, col, v, lane, [&](i32 x) {
        const i32 o = colors[x] - base;
        if (o >= 0 && o < WIN) m[o >> 5] |= 1u << (o & 31);
      });
      int r = 0;
#pragma unroll
      for (int w = 0; w < WORDS; w++) {
        const u32 mw = __reduce_or_sync(FULL, m[w]);
        if (!r && mw != FULL) r = w * 32 + __ffs(~mw);
      }
      if (r) {
        if (lane == 0) prop[i] = base + r - 1;
        break;
      }
    }
  }
}

template <int DIST, bool PARTIAL>
__global__ void k_losers(const i64* rowptr, const i32* col, const i32* colors, const i32* pending,
                         const i64* np_dev, const uint8_t* in_round, uint8_t* lose) {
  const int lane = threadIdx.x & 31;
  const i64 np = *np_dev;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < np; i += nwarps) {
    const i32 v = pending[i];
    const i32 c = colors[v];
    bool hit = false;
    for_each_in_set<DIST, PARTIAL>(rowptr, col, v, lane, [&](i32 x) {
      if (colors[x] == c && (x > v || !in_round[x])) hit = true;
    });
    const bool any = __any_sync(FULL, hit);
    if (lane == 0) lose[i] = any ? 1 : 0;
  }
}

// ---------------------------------------------------------------- edge-based (EB)
// chroma/localcolor.py:181-195 (Kernel.EDGE_BASED, chosen when delta_max exceeds the
// threshold, 55-61): the same proposals and losers (F3), computed edge-parallel so a
// hub row is spread over many threads.  The pending rows' entries are flattened by an
// exclusive scan of their lengths (eoff); each thread takes EB_CHUNK consecutive
// entries, finds its first row by binary search and walks on (merge path).
constexpr int EB_CHUNK = 16;

__global__ void k_eb_lengths(const i64* rowptr, const i32* pending, i64 np, i64* len) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < np; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = pending[i];
    len[i] = rowptr[v + 1] - rowptr[v];
  }
}

__device__ __forceinline__ i64 eb_row_of(const i64* eoff, i64 np, i64 e) {
  i64 lo = 0, hi = np;  // last i with eoff[i] <= e
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (eoff[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// OR the colours of window [base, base + WIN) into the per-row masks of unresolved rows.
// Each thread ORs its entries into its own shared-memory mask and flushes it once per
// row segment; at the end of a chunk the lanes on the same row (a hub's entries span
// whole warps) combine their masks first, so a hub row takes one atomic per word per
// warp instead of one per entry.
constexpr int EB_THREADS = 256;
__global__ void __launch_bounds__(EB_THREADS) k_eb_masks(const i64* rowptr, const i32* col, const i32* colors,
                                                         const i32* pending, i64 np, const i64* eoff, i64 E,
                                                         i32 base, const i32* prop, u32* mask) {
  __shared__ u32 sm[EB_THREADS * (WORDS + 1)];
  u32* my = sm + threadIdx.x * (WORDS + 1);
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  auto flush_own = [&](i64 r) {
    for (int w = 0; w < WORDS; w++) {
      if (my[w]) atomicOr(mask + r * WORDS + w, my[w]);
      my[w] = 0;
    }
  };
  for (int w = 0; w < WORDS; w++) my[w] = 0;
  for (i64 wb = warp * 32 * EB_CHUNK; wb < E; wb += nwarps * 32 * EB_CHUNK) {
    const i64 c0 = wb + (i64)lane * EB_CHUNK;
    i64 cur = -1;  // the row my mask belongs to
    if (c0 < E) {
      i64 i = eb_row_of(eoff, np, c0);
      const i64 c1 = c0 + EB_CHUNK < E ? c0 + EB_CHUNK : E;
      cur = i;
      for (i64 e = c0; e < c1;) {
        while (i + 1 < np && eoff[i + 1] <= e) i++;
        if (i != cur) {
          flush_own(cur);
          cur = i;
        }
        const i64 re = i + 1 < np ? (eoff[i + 1] < c1 ? eoff[i + 1] : c1) : c1;  // this row's part of the chunk
        if (prop[i] != 0) {  // resolved in an earlier window
          e = re;
          continue;
        }
        const i64 rb = rowptr[pending[i]] - eoff[i];
        for (; e < re; e += 4) {
          i32 xs[4];
#pragma unroll
          for (int q = 0; q < 4; q++) xs[q] = e + q < re ? col[rb + e + q] : -1;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const i32 o = xs[q] >= 0 ? colors[xs[q]] - base : -1;
            if (o >= 0 && o < WIN) my[o >> 5] |= 1u << (o & 31);
          }
        }
        e = re;
      }
    }
    // lanes on the same row combine their masks; the group's first lane flushes
    const unsigned grp = __match_any_sync(0xffffffffu, (unsigned long long)cur);
    const bool lead = lane == __ffs(grp) - 1;
    for (int w = 0; w < WORDS; w++) {
      const u32 v = __reduce_or_sync(grp, my[w]);
      if (lead && cur >= 0 && v) atomicOr(mask + cur * WORDS + w, v);
      my[w] = 0;
    }
  }
}

// first free colour of the window per unresolved row; *left counts rows still full
__global__ void k_eb_pick(i64 np, i32 base, const u32* mask, i32* prop, unsigned long long* left) {
  unsigned long long full = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < np; i += (i64)gridDim.x * blockDim.x) {
    if (prop[i] != 0) continue;
    int r = 0;
#pragma unroll
    for (int w = 0; w < WORDS; w++) {
      const u32 mw = mask[i * WORDS + w];
      if (!r && mw != FULL) r = w * 32 + __ffs(~mw);
    }
    if (r) prop[i] = base + r - 1;
    else full++;
  }
  if (full) atomicAdd(left, full);
}

// v loses iff an equal-coloured neighbour has a larger id or is outside the round; one
// store per (thread, row segment) that found one
__global__ void k_eb_losers(const i64* rowptr, const i32* col, const i32* colors, const i32* pending, i64 np,
                            const i64* eoff, i64 E, const uint8_t* in_round, uint8_t* lose) {
  for (i64 c0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) * EB_CHUNK; c0 < E;
       c0 += (i64)gridDim.x * blockDim.x * EB_CHUNK) {
    i64 i = eb_row_of(eoff, np, c0);
    const i64 c1 = c0 + EB_CHUNK < E ? c0 + EB_CHUNK : E;
    for (i64 e = c0; e < c1;) {
      while (i + 1 < np && eoff[i + 1] <= e) i++;
      const i64 re = i + 1 < np ? (eoff[i + 1] < c1 ? eoff[i + 1] : c1) : c1;
      const i32 v = pending[i];
      const i32 cv = colors[v];
      const i64 rb = rowptr[v] - eoff[i];
      bool l = false;
      for (; e < re; e += 4) {
        i32 xs[4];
#pragma unroll
        for (int q = 0; q < 4; q++) xs[q] = e + q < re ? col[rb + e + q] : -1;
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (xs[q] >= 0 && colors[xs[q]] == cv && (xs[q] > v || !in_round[xs[q]])) l = true;
      }
      if (l) lose[i] = 1;
      e = re;
    }
  }
}

}  // namespace

static int warp_grid(i64 n) { return grid_for(n * 32, 256, num_sms() * 16); }

// Edge-based Jacobi sweep pieces (distance 1): proposals into prop, then (after the
// caller's commit) losers into lose.  np: exact pending count.
void launch_jacobi_eb(const i64* rowptr, const i32* col, i32* colors, const i32* pending, i64 np, i32* prop,
                      const uint8_t* in_round, uint8_t* lose, EbScratch& S, cudaStream_t s) {
  if (np <= 0) return;
  S.len.reserve(np + 1, s);
  S.eoff.reserve(np + 1, s);
  k_eb_lengths<<<grid_for(np, 256, num_sms() * 16), 256, 0, s>>>(rowptr, pending, np, S.len.p);
  CUDA_CHECK(cudaMemsetAsync(S.len.p + np, 0, sizeof(i64), s));
  exclusive_scan_i64(S.len.p, S.eoff.p, np + 1, s);
  i64 E = 0;
  CUDA_CHECK(cudaMemcpyAsync(&E, S.eoff.p + np, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  S.mask.reserve(np * WORDS, s);
  S.left.reserve(1, s);
  CUDA_CHECK(cudaMemsetAsync(prop, 0, sizeof(i32) * np, s));
  const int ge = grid_for(std::max<i64>((E + EB_CHUNK - 1) / EB_CHUNK, 1), 256, num_sms() * 16);
  const int gm = grid_for(std::max<i64>((E + EB_CHUNK - 1) / EB_CHUNK, 1), EB_THREADS, num_sms() * 8);
  static const bool trace = std::getenv("CHROMA_JACOBI_TRACE") != nullptr;
  static int ncall = 0;
  ncall++;
  const bool tr = trace && (ncall & (ncall - 1)) == 0;
  cudaEvent_t te[4];
  if (tr)
    for (auto& e : te) CUDA_CHECK(cudaEventCreate(&e));
  if (tr) CUDA_CHECK(cudaEventRecord(te[0], s));
  int nwin = 0;
  for (i32 base = 1;; base += WIN) {
    nwin++;
    CUDA_CHECK(cudaMemsetAsync(S.mask.p, 0, sizeof(u32) * WORDS * np, s));
    CUDA_CHECK(cudaMemsetAsync(S.left.p, 0, sizeof(unsigned long long), s));
    if (E > 0) k_eb_masks<<<gm, EB_THREADS, 0, s>>>(rowptr, col, colors, pending, np, S.eoff.p, E, base, prop, S.mask.p);
    k_eb_pick<<<grid_for(np, 256, num_sms() * 16), 256, 0, s>>>(np, base, S.mask.p, prop, S.left.p);
    count_launch(2);
    unsigned long long left = 0;
    CUDA_CHECK(cudaMemcpyAsync(&left, S.left.p, sizeof(left), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (!left) break;
  }
  // commit the proposals (chroma/localcolor.py:222), then the edge-parallel loser scan
  S.np.reserve(1, s);
  CUDA_CHECK(cudaMemcpyAsync(S.np.p, &np, sizeof(i64), cudaMemcpyHostToDevice, s));
  launch_scatter_idx_values(colors, pending, prop, S.np.p, np, s);
  CUDA_CHECK(cudaMemsetAsync(lose, 0, np, s));
  if (tr) CUDA_CHECK(cudaEventRecord(te[1], s));
  if (E > 0) k_eb_losers<<<ge, 256, 0, s>>>(rowptr, col, colors, pending, np, S.eoff.p, E, in_round, lose);
  count_launch(2);
  if (tr) {
    CUDA_CHECK(cudaEventRecord(te[2], s));
    CUDA_CHECK(cudaEventSynchronize(te[2]));
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, te[0], te[1]);
    cudaEventElapsedTime(&b, te[1], te[2]);
    std::fprintf(stderr, "[jacobi eb] call %d: pending %lld entries %lld windows %d: masks+pick %.1f us, losers %.1f us\n",
                 ncall, (long long)np, (long long)E, nwin, a * 1e3, b * 1e3);
    for (auto& e : te) cudaEventDestroy(e);
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_jacobi_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pending,
                           const i64* np_dev, i64 np_max, i32* prop, int dist, bool partial,
                           cudaStream_t s) {
  if (np_max <= 0) return;
  const int g = warp_grid(np_max);
  if (dist == 1) k_propose<1, false><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, prop);
  else if (partial) k_propose<2, true><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, prop);
  else k_propose<2, false><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, prop);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

void launch_jacobi_losers(const i64* rowptr, const i32* col, i32* colors, const i32* pending,
                          const i64* np_dev, i64 np_max, const i32* prop, const uint8_t* in_round,
                          uint8_t* lose, int dist, bool partial, cudaStream_t s) {
  if (np_max <= 0) return;
  // commit the proposals (colors[pending] = proposals, chroma/localcolor.py:222)
  launch_scatter_idx_values(colors, pending, prop, np_dev, np_max, s);
  const int g = warp_grid(np_max);
  if (dist == 1) k_losers<1, false><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, in_round, lose);
  else if (partial) k_losers<2, true><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, in_round, lose);
  else k_losers<2, false><<<g, 256, 0, s>>>(rowptr, col, colors, pending, np_dev, in_round, lose);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace chroma
