// GPU properness checker (chroma/verify.py:61-112).
//   verify_d1: uncoloured vertices, then every edge (u, v>u) with equal non-zero colours.
//   verify_d2: uncoloured vertices in the endpoint mask, (full mode) the d1 edges, then
//              for every middle m every pair (i<j) of adj(m) with equal colours, both
//              endpoints in the mask.
// Counting is per row (warp per row; rows of <= 32 entries use __match_any_sync to
// find equal-colour groups in one step); listing re-walks only the rows that have
// violations and writes them at exclusive-scan offsets, which reproduces the
// reference's ordering without a sort.
#include <vector>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ unsigned lanemask_gt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_gt;" : "=r"(m));
  return m;
}

struct VArgs {
  const i64* rowptr;
  const i32* col;
  i64 n;
  const i32* colors;
  const uint8_t* mask;
};

__device__ __forceinline__ bool in_mask(const VArgs& a, i32 x) { return a.mask == nullptr || a.mask[x]; }

__global__ void k_uncolored(VArgs a, bool masked, uint8_t* flag) {
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < a.n; v += (i64)gridDim.x * blockDim.x)
    flag[v] = (a.colors[v] == 0 && (!masked || in_mask(a, (i32)v))) ? 1 : 0;
}

// CAT 1: d1 edges of row u; CAT 2: d2 pairs around middle m.
template <int CAT, bool WRITE>
__global__ void k_rows(VArgs a, i64* cnt, const i64* off, i64 base_pos, i64 cap, i64* out, int kind) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 r = warp; r < a.n; r += nwarps) {
    if (WRITE && cnt[r] == 0) continue;
    const i64 rs = a.rowptr[r], re = a.rowptr[r + 1];
    i64 pos = WRITE ? base_pos + off[r] : 0;
    i64 count = 0;
    if (CAT == 1) {
      const i32 cu = a.colors[r];
      if (cu != 0) {
        for (i64 e0 = rs; e0 < re; e0 += 32) {
          const i64 e = e0 + lane;
          i32 v = 0;
          bool hit = false;
          if (e < re) {
            v = a.col[e];
            hit = v > r && a.colors[v] == cu;
          }
          const unsigned b = __ballot_sync(FULL, hit);
          if (WRITE && hit) {
            const i64 p = pos + __popc(b & lanemask_lt());
            if (p < cap) {
              out[4 * p] = 1; out[4 * p + 1] = r; out[4 * p + 2] = v; out[4 * p + 3] = -1;
            }
          }
          pos += __popc(b);
          count += __popc(b);
        }
      }
    } else {
      const i64 d = re - rs;
      if (!WRITE && d <= 32) {
        i32 key = -1 - lane;
        if (lane < d) {
          const i32 u = a.col[rs + lane];
          const i32 c = a.colors[u];
          if (c != 0 && in_mask(a, u)) key = c;
        }
        const unsigned mt = __match_any_sync(FULL, key);
        const unsigned pairs = (key > 0) ? __popc(mt & lanemask_gt()) : 0;
        count = __reduce_add_sync(FULL, pairs);
      } else {
        for (i64 i = 0; i < d; i++) {
          const i32 u = a.col[rs + i];
          const i32 cu = a.colors[u];
          if (cu == 0 || !in_mask(a, u)) continue;
          for (i64 j0 = i + 1; j0 < d; j0 += 32) {
            const i64 j = j0 + lane;
            i32 w = 0;
            bool hit = false;
            if (j < d) {
              w = a.col[rs + j];
              hit = in_mask(a, w) && a.colors[w] == cu;
            }
            const unsigned b = __ballot_sync(FULL, hit);
            if (WRITE && hit) {
              const i64 p = pos + __popc(b & lanemask_lt());
              if (p < cap) {
                out[4 * p] = kind; out[4 * p + 1] = u; out[4 * p + 2] = w; out[4 * p + 3] = r;
              }
            }
            pos += __popc(b);
            count += __popc(b);
          }
        }
      }
    }
    if (!WRITE && lane == 0) cnt[r] = count;
  }
}

// Count-only verify_d1 (no listing): uncoloured vertices plus equal-coloured edges
// (u, v > u).  A warp takes 32 consecutive rows: a lane walks a row of <= 32 entries
// alone (8 column loads in flight), the warp walks the longer ones; one atomic per
// warp at the end.  Reads rowptr, col and the colour of every neighbour once.
__global__ void k_count_d1(VArgs a, unsigned long long* total) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  unsigned long long mine = 0;
  for (i64 b = warp * 32; b < a.n; b += nwarps * 32) {
    const i64 r = b + lane;
    i32 cu = 0;
    i64 rs = 0, re = 0;
    if (r < a.n) {
      cu = a.colors[r];
      rs = a.rowptr[r];
      re = a.rowptr[r + 1];
      if (cu == 0) {
        mine++;
        re = rs;
      }
    }
    const bool lng = re - rs > 32;
    if (!lng) {
      for (i64 e0 = rs; e0 < re; e0 += 8) {
        i32 vs[8];
#pragma unroll
        for (int q = 0; q < 8; q++) vs[q] = e0 + q < re ? __ldcs(a.col + e0 + q) : -1;
#pragma unroll
        for (int q = 0; q < 8; q++) mine += (vs[q] > r && a.colors[vs[q]] == cu) ? 1 : 0;
      }
    }
    for (unsigned lm = __ballot_sync(FULL, lng); lm; lm &= lm - 1) {
      const int src = __ffs(lm) - 1;
      const i64 rr = b + src;
      const i32 cl = __shfl_sync(FULL, cu, src);
      const i64 ls = __shfl_sync(FULL, rs, src), le = __shfl_sync(FULL, re, src);
      for (i64 e0 = ls; e0 < le; e0 += 128) {
        i32 vs[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const i64 e = e0 + q * 32 + lane;
          vs[q] = e < le ? __ldcs(a.col + e) : -1;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) mine += (vs[q] > rr && a.colors[vs[q]] == cl) ? 1 : 0;
      }
    }
  }
  mine = __reduce_add_sync(FULL, (unsigned)mine);
  if (lane == 0 && mine) atomicAdd(total, mine);
}

__global__ void k_write_uncolored(const i32* ids, const i64* nsel, i64 cap, i64* out) {
  const i64 n = *nsel;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n && i < cap; i += (i64)gridDim.x * blockDim.x) {
    out[4 * i] = 0; out[4 * i + 1] = ids[i]; out[4 * i + 2] = -1; out[4 * i + 3] = -1;
  }
}

__global__ void k_sum_last(const i64* cnt, const i64* off, i64 n, i64* total) {
  *total = n > 0 ? off[n - 1] + cnt[n - 1] : 0;
}

}  // namespace

i64 run_verify(const i64* rowptr, const i32* col, i64 n, const i32* colors, const uint8_t* mask,
               int mode, i64* rows_host, i64 cap, cudaStream_t s) {
  VArgs a{rowptr, col, n, colors, mask};
  const bool want_rows = rows_host != nullptr && cap > 0;
  if (mode == 0 && !want_rows) {  // the checker's common case: a count
    DBuf<unsigned long long> t;
    t.alloc(1, s);
    t.zero(s);
    k_count_d1<<<grid_for(n, 256, num_sms() * 16), 256, 0, s>>>(a, t.p);
    count_launch();
    unsigned long long h = 0;
    CUDA_CHECK(cudaMemcpyAsync(&h, t.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    return (i64)h;
  }
  DBuf<uint8_t> flag;
  DBuf<i32> unc;
  DBuf<i64> nunc, cnt1, off1, cnt2, off2, tot, out;
  flag.alloc(n + 1, s);
  unc.alloc(n + 1, s);
  nunc.alloc(1, s);
  tot.alloc(2, s);
  const int eg = grid_for(n, 256, num_sms() * 16);
  const int wg = grid_for(n * 32, 256, num_sms() * 16);
  k_uncolored<<<eg, 256, 0, s>>>(a, mode != 0, flag.p);
  count_launch();
  select_flagged(flag.p, n, unc.p, nunc.p, s);
  const bool do1 = mode == 0 || mode == 1;
  const bool do2 = mode >= 1;
  if (do1) {
    cnt1.alloc(n + 1, s);
    off1.alloc(n + 1, s);
    k_rows<1, false><<<wg, 256, 0, s>>>(a, cnt1.p, nullptr, 0, 0, nullptr, 1);
    count_launch();
    exclusive_scan_i64(cnt1.p, off1.p, n, s);
    k_sum_last<<<1, 1, 0, s>>>(cnt1.p, off1.p, n, tot.p);
    count_launch();
  }
  if (do2) {
    cnt2.alloc(n + 1, s);
    off2.alloc(n + 1, s);
    k_rows<2, false><<<wg, 256, 0, s>>>(a, cnt2.p, nullptr, 0, 0, nullptr, mode == 1 ? 2 : 3);
    count_launch();
    exclusive_scan_i64(cnt2.p, off2.p, n, s);
    k_sum_last<<<1, 1, 0, s>>>(cnt2.p, off2.p, n, tot.p + 1);
    count_launch();
  }
  CUDA_CHECK(cudaGetLastError());
  i64 h[3] = {0, 0, 0};
  CUDA_CHECK(cudaMemcpyAsync(&h[0], nunc.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaMemcpyAsync(&h[1], tot.p, 2 * sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (!do1) h[1] = 0;
  if (!do2) h[2] = 0;
  const i64 total = h[0] + h[1] + h[2];
  if (want_rows && total > 0) {
    const i64 nrows = std::min(total, cap);
    out.alloc(4 * nrows, s);
    k_write_uncolored<<<grid_for(std::max<i64>(h[0], 1), 256, num_sms() * 8), 256, 0, s>>>(unc.p, nunc.p, nrows, out.p);
    count_launch();
    if (do1 && h[1] > 0 && h[0] < nrows) {
      k_rows<1, true><<<wg, 256, 0, s>>>(a, cnt1.p, off1.p, h[0], nrows, out.p, 1);
      count_launch();
    }
    if (do2 && h[2] > 0 && h[0] + h[1] < nrows) {
      k_rows<2, true><<<wg, 256, 0, s>>>(a, cnt2.p, off2.p, h[0] + h[1], nrows, out.p, mode == 1 ? 2 : 3);
      count_launch();
    }
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaMemcpyAsync(rows_host, out.p, sizeof(i64) * 4 * nrows, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  return total;
}

// ---------------------------------------------------------------- colour stats
namespace {
__global__ void k_maxc(const i32* c, i64 n, int* mx) {
  int m = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    m = max(m, c[i]);
  m = __reduce_max_sync(FULL, m);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}
__global__ void k_hist(const i32* c, i64 n, int maxc, unsigned long long* h) {
  __shared__ unsigned long long sh[1024];
  const bool loc = maxc < 1024;
  if (loc)
    for (int i = threadIdx.x; i <= maxc; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 x = c[i];
    if (x > 0) {
      if (loc) atomicAdd(&sh[x], 1ull);
      else atomicAdd(&h[x], 1ull);
    }
  }
  __syncthreads();
  if (loc)
    for (int i = threadIdx.x; i <= maxc; i += blockDim.x)
      if (sh[i]) atomicAdd(&h[i], sh[i]);
}
}  // namespace

void run_color_stats(const i32* colors, i64 n, i64* num_colors, i64* max_color, i64* hist_host,
                     i64 hist_cap, cudaStream_t s) {
  DBuf<int> mx;
  mx.alloc(1, s);
  mx.zero(s);
  const int g = grid_for(std::max<i64>(n, 1), 256, num_sms() * 16);
  if (n > 0) {
    k_maxc<<<g, 256, 0, s>>>(colors, n, mx.p);
    count_launch();
  }
  int hm = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hm, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  DBuf<unsigned long long> h;
  h.alloc(hm + 1, s);
  h.zero(s);
  if (n > 0 && hm > 0) {
    k_hist<<<g, 256, 0, s>>>(colors, n, hm, h.p);
    count_launch();
  }
  std::vector<unsigned long long> hh(hm + 1);
  CUDA_CHECK(cudaMemcpyAsync(hh.data(), h.p, sizeof(unsigned long long) * (hm + 1), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  i64 k = 0;
  for (int c = 1; c <= hm; c++) k += hh[c] ? 1 : 0;
  *num_colors = k;
  *max_color = hm;
  if (hist_host)
    for (i64 c = 0; c < hist_cap; c++) hist_host[c] = c <= hm ? (i64)hh[c] : 0;
}

}  // namespace chroma
