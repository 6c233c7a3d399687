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

}  // namespace

void run_detect(const DetectArgs& A, i64 num_vertices, DetectScratch& S,
                unsigned long long* conflicts_dev, cudaStream_t s) {
  if (A.nrows <= 0) return;
  DevDetect a{A.rowptr, A.col, A.colors, A.gids, A.deg, A.rows, A.nrows, A.recolor_degrees};
  S.cnt.reserve(A.nrows, s);
  S.off.reserve(A.nrows, s);
  S.total.reserve(1, s);
  const int g = grid_for(A.nrows * 32, 256, num_sms() * 16);
  auto launch = [&](auto wr) {
    constexpr bool W = decltype(wr)::value;
    if (A.dist == 1) k_events<1, false, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    else if (A.partial) k_events<2, true, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    else k_events<2, false, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
    count_launch();
    CUDA_CHECK(cudaGetLastError());
  };
  launch(std::false_type{});
  exclusive_scan_i64(S.cnt.p, S.off.p, A.nrows, s);
  k_total<<<1, 1, 0, s>>>(S.cnt.p, S.off.p, A.nrows, S.total.p);
  count_launch();
  i64 E = 0;
  CUDA_CHECK(cudaMemcpyAsync(&E, S.total.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (E == 0) return;
  CHROMA_REQUIRE(E < INT32_MAX, CHROMA_ERUNTIME, "too many conflict events");
  S.ev.reserve(E, s);
  launch(std::true_type{});
  S.fired.reserve(E, s);
  S.kill.reserve(num_vertices, s);
  k_resolve<<<1, 1024, 0, s>>>(S.ev.p, E, S.fired.p, S.kill.p, A.colors, conflicts_dev, A.sequential);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace chroma
