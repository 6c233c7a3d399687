// The square G^2 of a bounded-degree local graph, for distance-2 colouring.
//
// The reference's distance-2 forbidden set of v (chroma/localcolor.py:136-158,
// _forbidden_d2 over two_hop_neighbors) is the colours of every x != v within two hops.
// That is exactly v's neighbourhood in G^2, so Gauss-Seidel and Jacobi distance-2
// colouring of G (chroma/localcolor.py:198-227, 274-303) are the distance-1 algorithms
// run on G^2 with the same worklist order: the same first-fit proposals, and the same
// loser rule ("an equal-coloured x in the forbidden set with x > v or outside the
// round").  For meshes (C4: 7-point stencil, 24 two-hop neighbours) G^2 has bounded
// degree, so the distance-1 machinery -- the level schedule and the cluster kernel
// (gs_levels.cu, gs_cluster.cu) or gs_chunked.cu -- replaces the two-hop dataflow
// kernel (color_gs.cu), which walked every two-hop set on every evaluation.
//
// Rows are built from the local graph for every local vertex (Jacobi's worklist holds
// uncoloured ghosts too, F7, and the reference takes their two-hop sets from the same
// local rows), or only where want[v] != 0; each row is sorted and duplicate-free.  One warp per
// row collects N(v) and N(u) for u in N(v) into shared memory (at most SQ_CAP), sorts
// them (bitonic) and keeps the first of each run.
#include "kernels.cuh"

namespace chroma {
namespace {

// warps per block: the candidate buffers (SQ_CAP ints per warp) stay within 32 KB
template <int SQ_CAP>
constexpr int sq_warps() { return SQ_CAP >= 4096 ? 2 : SQ_CAP >= 2048 ? 4 : 8; }

// WRITE = false: row lengths into len (and the max into *maxdeg, overflow into *ovf);
// WRITE = true: rows into col2 at off.
template <bool WRITE, int SQ_CAP, bool PARTIAL>
__global__ void __launch_bounds__(sq_warps<SQ_CAP>() * 32)
    k_square(const i64* rowptr, const i32* col, i64 nv, const uint8_t* want, i64* len, const i64* off, i32* col2,
             unsigned long long* maxdeg, unsigned* ovf) {
  constexpr int SQ_WARPS = sq_warps<SQ_CAP>();
  __shared__ i32 cand_all[SQ_WARPS][SQ_CAP];
  __shared__ int ncand_all[SQ_WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  i32* cand = cand_all[wid];
  int& ncand = ncand_all[wid];
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 v = warp; v < nv; v += nwarps) {
    if (want && !want[v]) {
      if (!WRITE && lane == 0) len[v] = 0;
      continue;
    }
    if (lane == 0) ncand = 0;
    __syncwarp();
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    bool over = false;
    for (i64 e = rs + lane; e < re; e += 32) {
      const i32 u = col[e];
      int k;
      if (!PARTIAL) {  // partial distance 2: the middles themselves are not forbidden
        k = atomicAdd(&ncand, 1);
        if (k < SQ_CAP) cand[k] = u;
        else over = true;
      }
      for (i64 f = rowptr[u]; f < rowptr[u + 1]; f++) {
        const i32 x = col[f];
        if (x == (i32)v) continue;
        k = atomicAdd(&ncand, 1);
        if (k < SQ_CAP) cand[k] = x;
        else over = true;
      }
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, over)) {
      if (lane == 0) {
        atomicOr(ovf, 1u);
        if (!WRITE) len[v] = 0;
      }
      continue;
    }
    const int K = ncand;
    // bitonic sort of the candidates padded to the next power of two (>= 64), then the
    // first of each run is kept
    int n2 = 64;
    while (n2 < K) n2 <<= 1;
    for (int i = K + lane; i < n2; i += 32) cand[i] = INT32_MAX;
    __syncwarp();
    for (int k = 2; k <= n2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < n2; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const i32 a = cand[i], b = cand[ixj];
            if ((a > b) == ((i & k) == 0)) {
              cand[i] = b;
              cand[ixj] = a;
            }
          }
        }
        __syncwarp();
      }
    const int PER = n2 / 32;  // lane l keeps positions [l * PER, (l + 1) * PER)
    auto keep = [&](int i) { return cand[i] != INT32_MAX && (i == 0 || cand[i] != cand[i - 1]); };
    int mine = 0;
    for (int q = 0; q < PER; q++) mine += keep(lane * PER + q);
    if (WRITE) {
      int inc = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      i64 at = off[v] + inc - mine;
      for (int q = 0; q < PER; q++)
        if (keep(lane * PER + q)) col2[at++] = cand[lane * PER + q];
    }
    const int U = __reduce_add_sync(0xffffffffu, mine);
    if (!WRITE && lane == 0) {
      len[v] = U;
      atomicMax(maxdeg, (unsigned long long)U);
    }
    __syncwarp();
  }
}

template <bool W, int CAP>
void launch_square(bool partial, const i64* rowptr, const i32* col, i64 nv, const uint8_t* want, i64* len,
                   const i64* off, i32* col2, unsigned long long* md, unsigned* ovf, cudaStream_t s) {
  constexpr int T = sq_warps<CAP>() * 32;
  const int g = grid_for(nv * 32, T, num_sms() * 16);
  if (partial) k_square<W, CAP, true><<<g, T, 0, s>>>(rowptr, col, nv, want, len, off, col2, md, ovf);
  else k_square<W, CAP, false><<<g, T, 0, s>>>(rowptr, col, nv, want, len, off, col2, md, ovf);
  count_launch();
}

template <bool W>
void launch_square_cap(int cap, bool partial, const i64* rowptr, const i32* col, i64 nv, const uint8_t* want,
                       i64* len, const i64* off, i32* col2, unsigned long long* md, unsigned* ovf, cudaStream_t s) {
  if (cap == 64) launch_square<W, 64>(partial, rowptr, col, nv, want, len, off, col2, md, ovf, s);
  else if (cap == 128) launch_square<W, 128>(partial, rowptr, col, nv, want, len, off, col2, md, ovf, s);
  else if (cap == 2048) launch_square<W, 2048>(partial, rowptr, col, nv, want, len, off, col2, md, ovf, s);
  else launch_square<W, 4096>(partial, rowptr, col, nv, want, len, off, col2, md, ovf, s);
}

}  // namespace

// G^2 (partial: two-hop only, the PD2 forbidden set) rows for the vertices with
// want[v] != 0 (all when want is null).  Returns false (nothing built) if a row would
// exceed the candidate capacity, or the rows would exceed max_entries in total.  The
// capacity follows the graph's maximum degree d: 64 when d + d(d - 1) <= 64, 128 up
// to d = 11, else 2048, retried at 4096 if a row overflows; each row sorts only the
// next power of two above its candidate count.
bool build_square(const i64* rowptr, const i32* col, i64 nv, i64 delta, bool partial, i64 max_entries,
                  const uint8_t* want, DBuf<i64>& rowptr2, DBuf<i32>& col2, i64& maxdeg, cudaStream_t s) {
  if (nv <= 0) return false;
  int cap = delta * delta <= 64 ? 64 : delta <= 11 ? 128 : 2048;
  DBuf<i64> len;
  len.alloc(nv + 1, s);
  DBuf<unsigned long long> md;
  md.alloc(2, s);
  unsigned* ovf = reinterpret_cast<unsigned*>(md.p + 1);
  unsigned long long h[2] = {0, 0};
  for (;;) {  // the wide capacity (fewer warps per SM) only if a row needs it
    md.zero(s);
    launch_square_cap<false>(cap, partial, rowptr, col, nv, want, len.p, nullptr, nullptr, md.p, ovf, s);
    CUDA_CHECK(cudaMemcpyAsync(h, md.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (!(h[1] & 0xffffffffull)) break;
    if (cap != 2048) return false;
    cap = 4096;
  }
  CUDA_CHECK(cudaMemsetAsync(len.p + nv, 0, sizeof(i64), s));
  DBuf<i64> rp;
  rp.alloc(nv + 1, s);
  exclusive_scan_i64(len.p, rp.p, nv + 1, s);
  i64 total = 0;
  CUDA_CHECK(cudaMemcpyAsync(&total, rp.p + nv, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (total > max_entries || total >= ((i64)1 << 31) * 4) return false;
  rowptr2 = std::move(rp);
  col2.alloc(std::max<i64>(total, 1), s);
  launch_square_cap<true>(cap, partial, rowptr, col, nv, want, nullptr, rowptr2.p, col2.p, md.p, ovf, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  maxdeg = (i64)h[0];
  return true;
}

}  // namespace chroma
