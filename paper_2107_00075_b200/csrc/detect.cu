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

__global__ void __launch_bounds__(1024, 1) k_resolve_grid(const int2* ev, i64 E, uint8_t* fired, i32* kill,
                                                          i32* colors, unsigned long long* conflicts, unsigned* bar,
                                                          int* changed) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x, T = (i64)gridDim.x * blockDim.x;
  const unsigned nb = gridDim.x;
  for (i64 e = t; e < E; e += T) fired[e] = 1;
  for (i64 it = 0; it <= E + 1; it++) {
    // three flags: this sweep's, the next one's (cleared now), and the previous
    // one's, which a block that just left the last barrier may still be reading
    int* ch = changed + it % 3;
    if (t == 0) changed[(it + 1) % 3] = 0;
    for (i64 e = t; e < E; e += T) {
      kill[ev[e].x] = INT32_MAX;
      kill[ev[e].y] = INT32_MAX;
    }
    grid_sync(bar, nb);
    for (i64 e = t; e < E; e += T)
      if (fired[e]) atomicMin(&kill[ev[e].x], (i32)e);
    grid_sync(bar, nb);
    bool mine = false;
    for (i64 e = t; e < E; e += T) {
      const uint8_t f = (kill[ev[e].x] >= (i32)e && kill[ev[e].y] >= (i32)e) ? 1 : 0;
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
    if (A.dist == 1) k_events<1, false, W><<<g, 256, 0, s>>>(a, S.cnt.p, S.off.p, S.ev.p);
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
  S.fired.reserve(E, s);
  S.kill.reserve(num_vertices, s);
  if (A.sequential && E > 32768) {
    S.result.reserve(4, s);
    CUDA_CHECK(cudaMemsetAsync(S.result.p, 0, 4 * sizeof(unsigned long long), s));
    unsigned* bar = reinterpret_cast<unsigned*>(S.result.p);
    int* changed = reinterpret_cast<int*>(S.result.p + 1);
    const int2* evp = S.ev.p;
    uint8_t* fp = S.fired.p;
    i32* kp = S.kill.p;
    i32* cp = A.colors;
    void* args[] = {(void*)&evp, (void*)&E, (void*)&fp, (void*)&kp, (void*)&cp, (void*)&conflicts_dev, (void*)&bar,
                    (void*)&changed};
    CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_resolve_grid, dim3(num_sms()), dim3(1024), args, 0, s));
  } else {
    k_resolve<<<1, 1024, 0, s>>>(S.ev.p, E, S.fired.p, S.kill.p, A.colors, conflicts_dev, A.sequential);
  }
  count_launch();
  CUDA_CHECK(cudaGetLastError());
  mark_t();
  save_prev();
  mark_t();
}

}  // namespace chroma
