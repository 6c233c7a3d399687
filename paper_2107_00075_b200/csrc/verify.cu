// GPU properness checker (chroma/verify.py:61-112).
//   verify_d1: uncoloured vertices, then every edge (u, v>u) with equal non-zero colours.
//   verify_d2: uncoloured vertices in the endpoint mask, (full mode) the d1 edges, then
//              for every middle m every pair (i<j) of adj(m) with equal colours, both
//              endpoints in the mask.
// Counting is per row (warp per row; rows of <= 32 entries use __match_any_sync to
// find equal-colour groups in one step); listing re-walks only the rows that have
// violations and writes them at exclusive-scan offsets, which reproduces the
// reference's ordering without a sort.
#include <cstdlib>
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
// (u, v > u).  Edge-tiled so the column stream is read with full-width coalesced loads
// whatever the degree skew: a CTA takes a tile of VT_TILE consecutive entries, stages
// the tile's slice of rowptr in shared memory (tile start rows from one pass over
// rowptr, loaded a tile ahead), and each
// thread takes VT_PER consecutive entries (two 16-byte loads), finds their rows by a
// binary search in shared memory and gathers the neighbours' colours from a 16-bit
// copy of the colour array.  The random colour loads bound it (one L1 wavefront each,
// ~1 per SM clock: scripts/gather_roofline.cu), so occupancy carries it.
// Colours >= 0xFFFF saturate in the copy; a saturated match re-checks the int32 colours.
// Reads rowptr, col and every neighbour's colour once (B = 8(n+1) + 4 nnz + 4n + 2 nnz
// gathered halfwords).
constexpr int VT_THREADS = 256;
constexpr int VT_PER = 8;
constexpr int VT_TILE = VT_THREADS * VT_PER;
constexpr int VT_MINB = 6;  // <= 40 registers: occupancy carries the gathers (A/B on C3:
                            // 8 entries x 6 CTAs 1.73 ms; 16 x 3 2.4 ms; 4 x 8 1.9 ms; row-wise 2.2 ms)
constexpr int VT_ROWS = 2048;  // rows of a tile staged in shared memory (more: global search)

__global__ void k_colors16(const i32* colors, i64 n, uint16_t* c16, unsigned long long* total) {
  unsigned long long zeros = 0;
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
    const i32 c = __ldcs(colors + v);
    c16[v] = (uint16_t)(c < 0 ? 0xFFFF : c > 0xFFFE ? 0xFFFF : c);
    zeros += c == 0;
  }
  zeros = __reduce_add_sync(FULL, (unsigned)zeros);
  if ((threadIdx.x & 31) == 0 && zeros) atomicAdd(total, zeros);
}

// largest r in [lo, hi] with rp[r] <= e
__device__ __forceinline__ i64 row_search(const i64* rp, i64 lo, i64 hi, i64 e) {
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    if (__ldg(rp + mid) <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// tile_row[t] = the row holding entry t * VT_TILE (t < ntiles), tile_row[ntiles] = n - 1:
// each non-empty row writes the tiles that start inside it (one pass over rowptr)
__global__ void k_tile_rows(const i64* rp, i64 n, i64 ntiles, i32* tile_row) {
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x) {
    const i64 rs = __ldg(rp + r), re = __ldg(rp + r + 1);
    for (i64 t = (rs + VT_TILE - 1) / VT_TILE; t * VT_TILE < re; t++) tile_row[t] = (i32)r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) tile_row[ntiles] = (i32)(n - 1);
}

__global__ void __launch_bounds__(VT_THREADS, VT_MINB) k_count_d1(const i64* rp, const i32* col, i64 n, const i32* tile_row,
                                                         const uint16_t* c16, const i32* c32, bool aligned,
                                                         unsigned long long* total) {
  __shared__ i32 s_off[VT_ROWS + 1];
  const i64 nnz = n > 0 ? __ldg(rp + n) : 0;
  unsigned long long mine = 0;
  // the next tile's row range is loaded one tile ahead, its columns before the staging
  i64 nlo = 0, nhi = 0;
  if ((i64)blockIdx.x * VT_TILE < nnz) {
    nlo = __ldg(tile_row + blockIdx.x);
    nhi = __ldg(tile_row + blockIdx.x + 1);
  }
  for (i64 t = blockIdx.x; t * VT_TILE < nnz; t += gridDim.x) {
    const i64 e0 = t * VT_TILE;
    const i64 e1 = min(e0 + (i64)VT_TILE, nnz);
    const int x0 = threadIdx.x * VT_PER;
    const int len = (int)(e1 - e0);
    i32 us[VT_PER];
    if (aligned && x0 + VT_PER <= len) {
      const int4* p4 = reinterpret_cast<const int4*>(col + e0 + x0);
#pragma unroll
      for (int q = 0; q < VT_PER / 4; q++) {
        const int4 w = __ldcs(p4 + q);
        us[4 * q] = w.x; us[4 * q + 1] = w.y; us[4 * q + 2] = w.z; us[4 * q + 3] = w.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < VT_PER; q++) us[q] = x0 + q < len ? __ldcs(col + e0 + x0 + q) : -1;
    }
    const i64 rlo = nlo, rhi = nhi;
    const i64 tn = t + gridDim.x;
    if (tn * VT_TILE < nnz) {
      nlo = __ldg(tile_row + tn);
      nhi = __ldg(tile_row + tn + 1);
    }
    const i64 nr = rhi - rlo + 1;
    const bool fits = nr <= VT_ROWS;
    if (fits) {
      for (i64 i = threadIdx.x; i <= nr; i += VT_THREADS) {
        const i64 o = __ldg(rp + rlo + i) - e0;
        s_off[i] = (i32)(o < 0 ? 0 : o > VT_TILE ? VT_TILE : o);
      }
    }
    __syncthreads();
    if (x0 < len) {
      // row (relative to rlo) of the first entry, then walk the row boundaries
      i64 ri;
      if (fits) {
        int lo = 0, hi = (int)nr - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_off[mid] <= x0) lo = mid;
          else hi = mid - 1;
        }
        ri = lo;
      } else {
        ri = row_search(rp, rlo, rhi, e0 + x0) - rlo;
      }
      auto off_at = [&](i64 i) -> i64 { return fits ? (i64)s_off[i] : min(__ldg(rp + rlo + i) - e0, (i64)VT_TILE); };
      i64 nxt = off_at(ri + 1);
      i32 rows[VT_PER];
#pragma unroll
      for (int q = 0; q < VT_PER; q++) {
        while (x0 + q >= nxt && x0 + q < len) nxt = off_at(++ri + 1);
        rows[q] = (i32)(rlo + ri);
      }
      // one gather per neighbour (each costs an L1 wavefront: ~1 per SM clock, measured
      // in scripts/gather_roofline.cu); the row's own colour once per row
      uint16_t cu[VT_PER], cv[VT_PER];
#pragma unroll
      for (int q = 0; q < VT_PER; q++) {
        const bool live = us[q] > rows[q];
        cv[q] = live ? __ldg(c16 + us[q]) : 0;
        cu[q] = q > 0 && rows[q] == rows[q - 1] ? cu[q - 1] : __ldg(c16 + rows[q]);
      }
#pragma unroll
      for (int q = 0; q < VT_PER; q++) {
        if (cu[q] != 0 && cu[q] == cv[q]) mine += cu[q] != 0xFFFF || __ldg(c32 + us[q]) == __ldg(c32 + rows[q]);
      }
    }
    __syncthreads();
  }
  mine = __reduce_add_sync(FULL, (unsigned)mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, mine);
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
    DBuf<uint16_t> c16;
    c16.alloc(n + 1, s);
    k_colors16<<<grid_for(n, 256, num_sms() * 8), 256, 0, s>>>(colors, n, c16.p, t.p);
    count_launch();
    const bool aligned = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
    i64 nnz = 0;
    CUDA_CHECK(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    const i64 ntiles = (nnz + VT_TILE - 1) / VT_TILE;
    DBuf<i32> trow;
    trow.alloc(ntiles + 1, s);
    k_tile_rows<<<grid_for(n, 256, num_sms() * 8), 256, 0, s>>>(rowptr, n, ntiles, trow.p);
    count_launch();
    k_count_d1<<<num_sms() * 12, VT_THREADS, 0, s>>>(rowptr, col, n, trow.p, c16.p, colors, aligned, t.p);
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
