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

}  // namespace

static int warp_grid(i64 n) { return grid_for(n * 32, 256, num_sms() * 16); }

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
