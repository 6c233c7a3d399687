// build_local_graphs on the GPU (chroma/runtime.py:149-268).
//
// Exact layout (F8): local ids are [owned ascending gid | layer-1 ghosts ascending
// gid | layer-2 ghosts ascending gid]; every row is sorted by local id.
// Row content (F10): owned rows are complete; with one ghost layer a ghost row
// holds only its back-edges to owned vertices; with two layers layer-1 rows are
// complete and layer-2 rows hold only back-edges to layer 1.
//
// No sort is needed for the rows: the global rows are gid-sorted and the local id
// is monotone in gid inside each of the three classes, so a stable three-way
// partition of each row by class (owned < L1 < L2) is the lid-sorted row.  The
// class lists themselves come out sorted from an ordered compaction over gids.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/iterator/zip_iterator.h>

#include "world.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// partition_block (chroma/partition.py:49-58): owner[v] = r for v in [rn/P, (r+1)n/P)
__global__ void k_block_owner(i32* owner, i64 n, i32 P) {
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
    i64 r = (v * P) / n;
    while (r + 1 < P && ((r + 1) * n) / P <= v) r++;
    while (r > 0 && (r * n) / P > v) r--;
    owner[v] = (i32)r;
  }
}

// chk[0] += out-of-range owners, chk[1] = max degree, chk[2 + r] += |owned(r)|
// owner range, per-rank counts and the maximum degree.  Counts go through a block
// histogram (P <= 1024) or warp-aggregated atomics; the maximum is warp-reduced.
__global__ void k_owner_check(const i32* owner, i64 n, i32 P, const i64* off, unsigned long long* chk) {
  __shared__ unsigned h[1024];
  const bool local = P <= 1024;
  if (local)
    for (int i = threadIdx.x; i < P; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned long long bad = 0;
  unsigned dmax = 0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 v = b + (threadIdx.x & 31);
    i32 o = -1;
    if (v < n) {
      o = owner[v];
      if (o < 0 || o >= P) {
        bad++;
        o = -1;
      }
      const i64 d = off[v + 1] - off[v];
      dmax = max(dmax, d > 0xffffffffll ? 0xffffffffu : (unsigned)d);
    }
    if (P <= 4096) {
      const unsigned grp = __match_any_sync(0xffffffffu, o);
      if (o >= 0 && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) {
        if (local) atomicAdd(&h[o], (unsigned)__popc(grp));
        else atomicAdd(&chk[2 + o], (unsigned long long)__popc(grp));
      }
    }
  }
  dmax = __reduce_max_sync(0xffffffffu, dmax);
  const unsigned nbad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
  if ((threadIdx.x & 31) == 0) {
    if (nbad) atomicAdd(&chk[0], (unsigned long long)nbad);
    atomicMax(&chk[1], (unsigned long long)dmax);
  }
  __syncthreads();
  if (local)
    for (int i = threadIdx.x; i < P; i += blockDim.x)
      if (h[i]) atomicAdd(&chk[2 + i], (unsigned long long)h[i]);
}

// owned_lid[list[i]] = i (position of each owned gid inside its owner)
__global__ void k_scatter_pos(const i32* list, i64 k, i32* pos) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < k; i += (i64)gridDim.x * blockDim.x)
    pos[list[i]] = (i32)i;
}


// out[0] = min, out[1] = max, out[2] = count of the gids owned by ranks [lo, hi)
__global__ void k_owned_range(const i32* owner, i64 n, i32 lo, i32 hi, unsigned long long* out) {
  unsigned long long mn = ~0ull, mx = 0, c = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    if (owner[i] >= lo && owner[i] < hi) {
      mn = min(mn, (unsigned long long)i);
      mx = max(mx, (unsigned long long)i);
      c++;
    }
  mn = __reduce_min_sync(0xffffffffu, (unsigned)min(mn, 0xffffffffull));
  mx = __reduce_max_sync(0xffffffffu, (unsigned)mx);
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31) == 0) {
    if (c) {
      atomicMin(out, mn);
      atomicMax(out + 1, mx);
    }
    atomicAdd(out + 2, c);
  }
}

// out[0] = min, out[1] = max column over col[0, k)
__global__ void k_col_range(const i32* col, i64 k, unsigned* out) {
  unsigned mn = ~0u, mx = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < k; i += (i64)gridDim.x * blockDim.x) {
    const unsigned u = (unsigned)col[i];
    mn = min(mn, u);
    mx = max(mx, u);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

__global__ void k_flag_eq_i32(const i32* a, i64 n, i32 v, uint8_t* flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flag[i] = a[i] == v ? 1 : 0;
}
__global__ void k_flag_eq_u8(const uint8_t* a, i64 n, uint8_t v, uint8_t* flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flag[i] = a[i] == v ? 1 : 0;
}

// lid_of[list[i]] = base + i ; cls[list[i]] = c
__global__ void k_assign(const i32* list, i64 k, i32 base, uint8_t c, i32* lid_of, uint8_t* cls) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < k; i += (i64)gridDim.x * blockDim.x) {
    lid_of[list[i]] = base + (i32)i;
    cls[list[i]] = c;
  }
}

// For every row of `list`, neighbours u with cls[u] == 0 get cls[u] = to.
__global__ void k_mark_nbrs(const i32* list, i64 k, const i64* goff, const i32* gcol, uint8_t* cls,
                            uint8_t to) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < k; i += nwarps) {
    const i32 g = list[i];
    for (i64 e = goff[g] + lane; e < goff[g + 1]; e += 32) {
      const i32 u = gcol[e];
      if (cls[u] == 0) cls[u] = to;
    }
  }
}

// Which neighbours a local row keeps (chroma/runtime.py:186-200).
__device__ __forceinline__ bool keep_nbr(i64 lid, i64 oc, i64 l1, int gl, uint8_t cu) {
  if (lid < oc) return true;
  if (lid < oc + l1) return gl == 2 || cu == 1;
  return cu == 2;
}

__global__ void k_rowlen(const i32* lgids, i64 nl, i64 oc, i64 l1, int gl, const i64* goff,
                         const i32* gcol, const uint8_t* cls, i64* len) {
  // a warp takes 32 consecutive rows: complete rows (owned; layer 1 with two layers)
  // are a lane's length lookup, the partial ones are counted by the whole warp
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 b = warp * 32; b < nl; b += nwarps * 32) {
    const i64 lid = b + lane;
    i64 rs = 0, re = 0;
    bool partial = false;
    if (lid < nl) {
      const i32 g = lgids[lid];
      rs = goff[g];
      re = goff[g + 1];
      if (lid < oc || (lid < oc + l1 && gl == 2)) len[lid] = re - rs;
      else partial = true;
    }
    for (unsigned pm = __ballot_sync(FULL, partial); pm; pm &= pm - 1) {
      const int src = __ffs(pm) - 1;
      const i64 plid = b + src;
      const i64 prs = __shfl_sync(FULL, rs, src), pre = __shfl_sync(FULL, re, src);
      i64 c = 0;
      for (i64 e0 = prs; e0 < pre; e0 += 32) {
        const i64 e = e0 + lane;
        const bool k = e < pre && keep_nbr(plid, oc, l1, gl, cls[gcol[e]]);
        c += __popc(__ballot_sync(FULL, k));
      }
      if (lane == 0) len[plid] = c;
    }
  }
}

// Stable three-way partition of each kept row by class -> lid-sorted local row.
__global__ void k_fill(const i32* lgids, i64 nl, i64 oc, i64 l1, int gl, const i64* goff,
                       const i32* gcol, const uint8_t* cls, const i32* lid_of, const i64* lrow,
                       i32* lcol) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 lid = warp; lid < nl; lid += nwarps) {
    const i32 g = lgids[lid];
    const i64 rs = goff[g], re = goff[g + 1];
    i64 pos = lrow[lid];
    if (re - rs <= 32) {  // one chunk: load once, place all three classes from three ballots
      const i64 e = rs + lane;
      i32 u = 0;
      uint8_t cu = 0;
      if (e < re) {
        u = gcol[e];
        cu = cls[u];
      }
      const bool k = cu >= 1 && cu <= 3 && keep_nbr(lid, oc, l1, gl, cu);
      const unsigned b1 = __ballot_sync(FULL, k && cu == 1), b2 = __ballot_sync(FULL, k && cu == 2),
                     b3 = __ballot_sync(FULL, k && cu == 3);
      if (k) {
        const unsigned lt = lanemask_lt();
        const int off = cu == 1   ? __popc(b1 & lt)
                        : cu == 2 ? __popc(b1) + __popc(b2 & lt)
                                  : __popc(b1) + __popc(b2) + __popc(b3 & lt);
        lcol[pos + off] = lid_of[u];
      }
      continue;
    }
    // long row: count the kept owned / layer-1 entries, then place all three classes
    // in one more pass (rows of a world without ghosts keep every entry in order)
    i64 n1 = re - rs, n2 = 0;
    if (nl != oc) {
      n1 = 0;
      for (i64 e0 = rs; e0 < re; e0 += 32) {
        const i64 e = e0 + lane;
        uint8_t cu = 0;
        if (e < re) cu = cls[gcol[e]];
        const bool k = cu >= 1 && cu <= 3 && keep_nbr(lid, oc, l1, gl, cu);
        n1 += __popc(__ballot_sync(FULL, k && cu == 1));
        n2 += __popc(__ballot_sync(FULL, k && cu == 2));
      }
    }
    i64 p1 = pos, p2 = pos + n1, p3 = pos + n1 + n2;
    for (i64 e0 = rs; e0 < re; e0 += 32) {
      const i64 e = e0 + lane;
      i32 u = 0;
      uint8_t cu = 0;
      if (e < re) {
        u = gcol[e];
        cu = cls[u];
      }
      const bool k = cu >= 1 && cu <= 3 && keep_nbr(lid, oc, l1, gl, cu);
      const unsigned b1 = __ballot_sync(FULL, k && cu == 1), b2 = __ballot_sync(FULL, k && cu == 2),
                     b3 = __ballot_sync(FULL, k && cu == 3);
      if (k) {
        const unsigned lt = lanemask_lt();
        const i64 at = cu == 1 ? p1 + __popc(b1 & lt) : cu == 2 ? p2 + __popc(b2 & lt) : p3 + __popc(b3 & lt);
        lcol[at] = lid_of[u];
      }
      p1 += __popc(b1);
      p2 += __popc(b2);
      p3 += __popc(b3);
    }
  }
}

// boundary_d1 / edge counts (chroma/runtime.py:204-217)
__global__ void k_bound1(const i64* lrow, const i32* lcol, i64 nl, i64 oc, uint8_t* b1,
                         unsigned long long* ecount) {
  unsigned long long el = 0, eg = 0;
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < nl; v += (i64)gridDim.x * blockDim.x) {
    const i64 rs = lrow[v], re = lrow[v + 1];
    if (v < oc) {
      // rows are lid-sorted: owned neighbours form a prefix
      i64 lo = rs, hi = re;
      while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        if (lcol[mid] < oc) lo = mid + 1; else hi = mid;
      }
      el += (unsigned long long)(lo - rs);
      eg += (unsigned long long)(re - lo);
      b1[v] = (re > lo) ? 1 : 0;
    } else {
      eg += (unsigned long long)(re - rs);
    }
  }
  // one atomic pair per warp
  for (int o = 16; o > 0; o >>= 1) {
    el += __shfl_down_sync(0xffffffffu, el, o);
    eg += __shfl_down_sync(0xffffffffu, eg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&ecount[0], el);
    atomicAdd(&ecount[1], eg);
  }
}

// boundary_d2 = boundary_d1 u owned vertices with an owned boundary_d1 neighbour
// a warp per owned row: lanes test 32 owned neighbours at a time, stop at the first
// boundary_d1 one (rows are lid-sorted: owned neighbours form a prefix)
__global__ void k_bound2(const i64* lrow, const i32* lcol, i64 oc, const uint8_t* b1, uint8_t* b2) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 v = warp; v < oc; v += nwarps) {
    bool f = b1[v] != 0;
    const i64 re = lrow[v + 1];
    for (i64 e0 = lrow[v]; !f && e0 < re; e0 += 32) {
      const i64 e = e0 + lane;
      const i32 u = e < re ? lcol[e] : (i32)oc;
      const bool hit = u < oc && b1[u];
      f = __any_sync(FULL, hit);
      if (__any_sync(FULL, u >= oc)) break;
    }
    if (lane == 0) b2[v] = f ? 1 : 0;
  }
}

__global__ void k_local_meta(const i32* lgids, i64 nl, i64 oc, const i64* goff, const i32* owner,
                             i64* gids_out, i32* deg_out, i32* ghost_owner_out) {
  for (i64 lid = blockIdx.x * (i64)blockDim.x + threadIdx.x; lid < nl; lid += (i64)gridDim.x * blockDim.x) {
    const i32 g = lgids[lid];
    gids_out[lid] = g;
    deg_out[lid] = (i32)(goff[g + 1] - goff[g]);
    if (lid >= oc) ghost_owner_out[lid - oc] = owner[g];
  }
}

__global__ void k_reset(const i32* lgids, i64 nl, i32* lid_of, uint8_t* cls) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nl; i += (i64)gridDim.x * blockDim.x) {
    lid_of[lgids[i]] = -1;
    cls[lgids[i]] = 0;
  }
}

__global__ void k_shift_i64(const i64* in, i64* out, i64 n, i64 add) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = in[i] + add;
}
__global__ void k_shift_i32(const i32* in, i32* out, i64 n, i32 add) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = in[i] + add;
}
__global__ void k_ghost_lids(i32* out, i64 n, i32 first) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = first + (i32)i;
}
__global__ void k_set_range_u8(uint8_t* p, i64 lo, i64 hi, uint8_t v) {
  for (i64 i = lo + blockIdx.x * (i64)blockDim.x + threadIdx.x; i < hi; i += (i64)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_set_range_i32(i32* p, i64 lo, i64 hi, i32 v) {
  for (i64 i = lo + blockIdx.x * (i64)blockDim.x + threadIdx.x; i < hi; i += (i64)gridDim.x * blockDim.x)
    p[i] = v;
}

// One route per ghost slot of every local rank: src lid (owner side), dst lid, pair id.
__global__ void k_routes(const i64* gids, const i32* ghost_owner, i64 first_ghost_lid, i64 nghost,
                         const i32* owned_lid, const i64* rank_lid_off, i32 dst_rank, i32 P,
                         i32* src, i32* dst, i32* pair) {
  for (i64 s = blockIdx.x * (i64)blockDim.x + threadIdx.x; s < nghost; s += (i64)gridDim.x * blockDim.x) {
    const i64 lid = first_ghost_lid + s;
    const i32 o = ghost_owner[s];
    src[s] = (i32)(rank_lid_off[o] + owned_lid[gids[lid]]);
    dst[s] = (i32)lid;
    pair[s] = o * P + dst_rank;
  }
}

__global__ void k_route_heads(const i32* src, i64 n, uint8_t* head) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    head[i] = (i == 0 || src[i] != src[i - 1]) ? 1 : 0;
}
__global__ void k_route_off(const i32* head_pos, const i64* nheads, i64 n, i64* off) {
  const i64 k = *nheads;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i <= k; i += (i64)gridDim.x * blockDim.x)
    off[i] = i < k ? head_pos[i] : n;
}
__global__ void k_gather_i32(const i32* src, const i32* idx, const i64* n_dev, i32* out) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

// CHROMA_BUILD_TIMING=1 prints the device builder's phase times (synchronising)
struct PhaseTimer {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(cudaStream_t st) : s(st), on(std::getenv("CHROMA_BUILD_TIMING") != nullptr) {
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build] %-18s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }
int GW(i64 n) { return grid_for(std::max<i64>(n, 1) * 32, 256, num_sms() * 16); }

struct RankTmp {
  RankMeta m;
  DBuf<i32> lgids;
  DBuf<i64> lrow;
  DBuf<i32> lcol;
  DBuf<i64> gids;
  DBuf<i32> deg, ghost_owner, b1, b2;
};

}  // namespace

World* world_create(i64 n, const i64* h_off, const i64* h_col, i32 P, const i32* h_owner, i32 gl,
                    i32 lo, i32 hi, int device) {
  CHROMA_REQUIRE(gl == 1 || gl == 2, CHROMA_EVALUE, "ghost_layers must be 1 or 2");
  CHROMA_REQUIRE(P >= 1, CHROMA_EVALUE, "num_ranks must be >= 1");
  CHROMA_REQUIRE(n >= 0 && n < ((i64)1 << 31) - 1, CHROMA_EVALUE, "graph too large for int32 local ids");
  CHROMA_REQUIRE(0 <= lo && lo < hi && hi <= P, CHROMA_EVALUE, "bad local rank range");
  const i64 nnz = h_off[n];

  CUDA_CHECK(cudaSetDevice(device));
  retain_pool_memory(device);
  World* w = new World();
  try {
    w->device = device;
    CUDA_CHECK(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    cudaStream_t s = w->stream;
    w->P = P; w->rank_lo = lo; w->rank_hi = hi; w->gl = gl;
    w->n_global = n; w->m_global = nnz / 2;

    PhaseTimer ptm(s);
    DBuf<i64> goff;
    upload_large(goff, h_off, n + 1, s);
    // owner: uploaded (any PartitionMap) or computed (partition_block when h_owner is NULL);
    // validated on the device (chroma/partition.py:36-43, chroma/runtime.py:159-161)
    DBuf<i32> owner;
    if (h_owner) {
      upload_large(owner, h_owner, std::max<i64>(n, 1), s);
    } else {
      owner.alloc(std::max<i64>(n, 1), s);
      k_block_owner<<<G(n), 256, 0, s>>>(owner.p, n, P);
      count_launch();
    }
    {
      DBuf<unsigned long long> chk;
      chk.alloc(P + 2, s);
      chk.zero(s);
      k_owner_check<<<std::min(G(n), num_sms() * 4), 256, 0, s>>>(owner.p, n, P, goff.p, chk.p);
      count_launch();
      std::vector<unsigned long long> hc((size_t)P + 2);
      CUDA_CHECK(cudaMemcpyAsync(hc.data(), chk.p, sizeof(unsigned long long) * (P + 2), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      CHROMA_REQUIRE(hc[0] == 0, CHROMA_EVALUE, "owner out of range");
      if (P <= n && P <= 4096)
        for (i32 r = 0; r < P; r++)
          CHROMA_REQUIRE(hc[(size_t)r + 2] > 0, CHROMA_EVALUE, "empty rank with num_ranks <= num_vertices");
      w->delta_max = (i64)hc[1];
    }
    ptm.mark("offsets+owner");
    DBuf<i32> gcol;
    gcol.alloc(std::max<i64>(nnz, 1), s);
    {
      // columns [e0, e1) -> int32, range-checked on the device (ValueError like
      // chroma_csr_create): later window steps index the host row offsets with
      // column values read back from the device
      auto upload = [&](i64 e0, i64 e1) {
        if (e1 > e0) narrow_ids_checked(h_col + e0, e1 - e0, n, false, gcol.p + e0, s, "col_indices out of range");
      };
      // The builder reads the rows of the owned, layer-1 and (two layers) layer-2
      // vertices only.  When the owned gids of [lo, hi) are one contiguous range (block
      // partitions, one rank per process), only a gid window covering those rows
      // crosses PCIe: it starts at the owned range and grows, once per ghost layer, by
      // the neighbour range of the rows it added last.  Columns outside it are never read.
      bool windowed = false;
      static const bool no_window = std::getenv("CHROMA_NO_WINDOW") != nullptr;
      if (hi - lo < P && n > 0 && !no_window) {
        DBuf<unsigned long long> rr;
        rr.alloc(3, s);
        const unsigned long long init[3] = {~0ull, 0ull, 0ull};
        CUDA_CHECK(cudaMemcpyAsync(rr.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_owned_range<<<std::min(G(n), num_sms() * 4), 256, 0, s>>>(owner.p, n, lo, hi, rr.p);
        count_launch();
        unsigned long long hr[3];
        CUDA_CHECK(cudaMemcpyAsync(hr, rr.p, sizeof(hr), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (hr[2] > 0 && hr[1] - hr[0] + 1 == hr[2]) {
          windowed = true;
          i64 g0 = (i64)hr[0], g1 = (i64)hr[1] + 1;
          upload(h_off[g0], h_off[g1]);
          i64 p[2][2] = {{g0, g1}, {g1, g1}};  // rows added last (up to two pieces)
          DBuf<unsigned> cr;
          cr.alloc(2, s);
          for (int layer = 0; layer < gl; layer++) {
            const unsigned cinit[2] = {~0u, 0u};
            CUDA_CHECK(cudaMemcpyAsync(cr.p, cinit, sizeof(cinit), cudaMemcpyHostToDevice, s));
            for (auto& q : p) {
              const i64 e0 = h_off[q[0]], e1 = h_off[q[1]];
              if (e1 > e0) {
                k_col_range<<<std::min(G(e1 - e0), num_sms() * 4), 256, 0, s>>>(gcol.p + e0, e1 - e0, cr.p);
                count_launch();
              }
            }
            unsigned hc2[2];
            CUDA_CHECK(cudaMemcpyAsync(hc2, cr.p, sizeof(hc2), cudaMemcpyDeviceToHost, s));
            CUDA_CHECK(cudaStreamSynchronize(s));
            if (hc2[0] > hc2[1]) break;  // no neighbours: nothing further is read
            const i64 ng0 = std::min<i64>(g0, (i64)hc2[0]), ng1 = std::max<i64>(g1, (i64)hc2[1] + 1);
            upload(h_off[ng0], h_off[g0]);
            upload(h_off[g1], h_off[ng1]);
            p[0][0] = ng0; p[0][1] = g0;
            p[1][0] = g1; p[1][1] = ng1;
            g0 = ng0;
            g1 = ng1;
          }
        }
      }
      if (!windowed) upload(0, nnz);
    }
    ptm.mark("col h2d+convert");
    DBuf<i32> owned_lid, lid_of;
    owned_lid.alloc(std::max<i64>(n, 1), s);  // gid -> lid inside its owner (filled per rank below)
    lid_of.alloc(std::max<i64>(n, 1), s);
    launch_fill_i32(lid_of.p, n, -1, s);
    DBuf<uint8_t> cls, flag;
    cls.alloc(std::max<i64>(n, 1), s);
    cls.zero(s);
    flag.alloc(std::max<i64>(n, 1), s);
    DBuf<i64> cnt;
    cnt.alloc(4, s);
    DBuf<unsigned long long> ecount;
    ecount.alloc(2, s);

    std::vector<RankTmp> tmps((size_t)(hi - lo));
    auto count_of = [&](const i64* dptr) {
      i64 h = 0;
      CUDA_CHECK(cudaMemcpyAsync(&h, dptr, sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      return h;
    };
    ptm.mark("scratch");
    for (i32 r = lo; r < hi; r++) {
      RankTmp& T = tmps[(size_t)(r - lo)];
      T.m.rank = r;
      if (P == 1) {
        // one rank owns every vertex: no ghosts, the local graph is the graph itself
        // (lid = gid), boundary sets are empty, every edge is local
        T.lgids.alloc(std::max<i64>(n, 1), s);
        launch_iota_i32(T.lgids.p, n, 0, s);
        T.m.owned = n; T.m.ghost = 0; T.m.l1 = 0;
        T.m.nnz = nnz;
        T.lrow = std::move(goff);
        T.lcol = std::move(gcol);
        T.b1.alloc(1, s);
        T.b2.alloc(1, s);
        T.m.nb1 = T.m.nb2 = 0;
        T.m.e_local = nnz / 2;
        T.m.e_ghost = 0;
        T.gids.alloc(n + 1, s);
        T.deg.alloc(n + 1, s);
        T.ghost_owner.alloc(1, s);
        k_local_meta<<<G(n), 256, 0, s>>>(T.lgids.p, n, n, T.lrow.p, owner.p, T.gids.p, T.deg.p, T.ghost_owner.p);
        count_launch();
        continue;
      }
      T.lgids.alloc(std::max<i64>(n, 1), s);
      // owned (ascending gid)
      k_flag_eq_i32<<<G(n), 256, 0, s>>>(owner.p, n, r, flag.p);
      count_launch();
      select_flagged(flag.p, n, T.lgids.p, cnt.p, s);
      const i64 oc = count_of(cnt.p);
      k_assign<<<G(oc), 256, 0, s>>>(T.lgids.p, oc, 0, 1, lid_of.p, cls.p);
      k_scatter_pos<<<G(oc), 256, 0, s>>>(T.lgids.p, oc, owned_lid.p);
      count_launch(2);
      // layer 1 = neighbours of owned not owned (ascending gid)
      k_mark_nbrs<<<GW(oc), 256, 0, s>>>(T.lgids.p, oc, goff.p, gcol.p, cls.p, 2);
      count_launch();
      k_flag_eq_u8<<<G(n), 256, 0, s>>>(cls.p, n, 2, flag.p);
      count_launch();
      select_flagged(flag.p, n, T.lgids.p + oc, cnt.p, s);
      const i64 l1 = count_of(cnt.p);
      k_assign<<<G(l1), 256, 0, s>>>(T.lgids.p + oc, l1, (i32)oc, 2, lid_of.p, cls.p);
      count_launch();
      i64 l2 = 0;
      if (gl == 2) {
        k_mark_nbrs<<<GW(l1), 256, 0, s>>>(T.lgids.p + oc, l1, goff.p, gcol.p, cls.p, 3);
        count_launch();
        k_flag_eq_u8<<<G(n), 256, 0, s>>>(cls.p, n, 3, flag.p);
        count_launch();
        select_flagged(flag.p, n, T.lgids.p + oc + l1, cnt.p, s);
        l2 = count_of(cnt.p);
        k_assign<<<G(l2), 256, 0, s>>>(T.lgids.p + oc + l1, l2, (i32)(oc + l1), 3, lid_of.p, cls.p);
        count_launch();
      }
      const i64 nl = oc + l1 + l2;
      T.m.owned = oc; T.m.ghost = l1 + l2; T.m.l1 = l1;
      // rows
      DBuf<i64> len;
      len.alloc(nl + 1, s);
      k_rowlen<<<GW(nl), 256, 0, s>>>(T.lgids.p, nl, oc, l1, gl, goff.p, gcol.p, cls.p, len.p);
      count_launch();
      CUDA_CHECK(cudaMemsetAsync(len.p + nl, 0, sizeof(i64), s));
      T.lrow.alloc(nl + 1, s);
      exclusive_scan_i64(len.p, T.lrow.p, nl + 1, s);
      const i64 lnnz = count_of(T.lrow.p + nl);
      T.m.nnz = lnnz;
      T.lcol.alloc(std::max<i64>(lnnz, 1), s);
      k_fill<<<GW(nl), 256, 0, s>>>(T.lgids.p, nl, oc, l1, gl, goff.p, gcol.p, cls.p, lid_of.p, T.lrow.p, T.lcol.p);
      count_launch();
      // boundary sets and edge counts
      DBuf<uint8_t> b1f, b2f;
      b1f.alloc(oc + 1, s);
      b1f.zero(s);
      b2f.alloc(oc + 1, s);
      ecount.zero(s);
      k_bound1<<<G(nl), 256, 0, s>>>(T.lrow.p, T.lcol.p, nl, oc, b1f.p, ecount.p);
      count_launch();
      if (nl > oc) k_bound2<<<GW(oc), 256, 0, s>>>(T.lrow.p, T.lcol.p, oc, b1f.p, b2f.p);
      else CUDA_CHECK(cudaMemsetAsync(b2f.p, 0, oc + 1, s));  // no ghosts: no boundary
      count_launch();
      T.b1.alloc(oc + 1, s);
      T.b2.alloc(oc + 1, s);
      select_flagged(b1f.p, oc, T.b1.p, cnt.p + 1, s);
      select_flagged(b2f.p, oc, T.b2.p, cnt.p + 2, s);
      i64 hc[4];
      unsigned long long he[2];
      CUDA_CHECK(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaMemcpyAsync(he, ecount.p, sizeof(he), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      T.m.nb1 = oc > 0 ? hc[1] : 0;
      T.m.nb2 = oc > 0 ? hc[2] : 0;
      T.m.e_local = (i64)he[0] / 2;
      T.m.e_ghost = (i64)he[1] / 2;
      // gids, global degrees, ghost owners
      T.gids.alloc(nl + 1, s);
      T.deg.alloc(nl + 1, s);
      T.ghost_owner.alloc(T.m.ghost + 1, s);
      k_local_meta<<<G(nl), 256, 0, s>>>(T.lgids.p, nl, oc, goff.p, owner.p, T.gids.p, T.deg.p, T.ghost_owner.p);
      count_launch();
      k_reset<<<G(nl), 256, 0, s>>>(T.lgids.p, nl, lid_of.p, cls.p);
      count_launch();
    }

    ptm.mark("rank builds");
    // ---- concatenate (block-diagonal local graphs)
    i64 NL = 0, NNZ = 0, NG = 0, NB1 = 0, NB2 = 0;
    for (auto& T : tmps) {
      T.m.lid_off = NL; T.m.nnz_off = NNZ; T.m.ghost_off = NG; T.m.b1_off = NB1; T.m.b2_off = NB2;
      NL += T.m.owned + T.m.ghost;
      NNZ += T.m.nnz;
      NG += T.m.ghost;
      NB1 += T.m.nb1;
      NB2 += T.m.nb2;
    }
    CHROMA_REQUIRE(NL < INT32_MAX, CHROMA_EVALUE, "local vertex count exceeds int32");
    w->NL = NL; w->NNZ = NNZ; w->NGHOST = NG; w->NB1 = NB1; w->NB2 = NB2;
    w->g.device = device; w->g.stream = s; w->g.n = NL; w->g.nnz = NNZ;
    // a single rank at offset 0 hands its CSR over instead of copying it
    const bool take = tmps.size() == 1 && tmps[0].m.lid_off == 0 && tmps[0].m.nnz_off == 0;
    if (take) {
      w->g.rowptr = std::move(tmps[0].lrow);
      w->g.col = std::move(tmps[0].lcol);
    } else {
      w->g.rowptr.alloc(NL + 1, s);
      w->g.col.alloc(std::max<i64>(NNZ, 1), s);
    }
    w->gids.alloc(NL + 1, s);
    w->deg.alloc(NL + 1, s);
    w->colors.alloc(NL + 1, s);
    w->colors.zero(s);
    w->ghost_owner.alloc(NG + 1, s);
    w->ghosts.alloc(NG + 1, s);
    w->b1.alloc(NB1 + 1, s);
    w->b2.alloc(NB2 + 1, s);
    w->owned_flag.alloc(NL + 1, s);
    w->owned_flag.zero(s);
    w->rank_of.alloc(NL + 1, s);
    for (auto& T : tmps) {
      const RankMeta& m = T.m;
      const i64 nl = m.owned + m.ghost;
      if (!take) {
        k_shift_i64<<<G(nl), 256, 0, s>>>(T.lrow.p, w->g.rowptr.p + m.lid_off, nl, m.nnz_off);
        k_shift_i32<<<G(m.nnz), 256, 0, s>>>(T.lcol.p, w->g.col.p + m.nnz_off, m.nnz, (i32)m.lid_off);
      }
      CUDA_CHECK(cudaMemcpyAsync(w->gids.p + m.lid_off, T.gids.p, sizeof(i64) * nl, cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(w->deg.p + m.lid_off, T.deg.p, sizeof(i32) * nl, cudaMemcpyDeviceToDevice, s));
      if (m.ghost)
        CUDA_CHECK(cudaMemcpyAsync(w->ghost_owner.p + m.ghost_off, T.ghost_owner.p, sizeof(i32) * m.ghost,
                                   cudaMemcpyDeviceToDevice, s));
      k_ghost_lids<<<G(m.ghost), 256, 0, s>>>(w->ghosts.p + m.ghost_off, m.ghost, (i32)(m.lid_off + m.owned));
      k_shift_i32<<<G(m.nb1), 256, 0, s>>>(T.b1.p, w->b1.p + m.b1_off, m.nb1, (i32)m.lid_off);
      k_shift_i32<<<G(m.nb2), 256, 0, s>>>(T.b2.p, w->b2.p + m.b2_off, m.nb2, (i32)m.lid_off);
      k_set_range_u8<<<G(m.owned), 256, 0, s>>>(w->owned_flag.p, m.lid_off, m.lid_off + m.owned, 1);
      k_set_range_i32<<<G(nl), 256, 0, s>>>(w->rank_of.p, m.lid_off, m.lid_off + nl, m.rank - lo);
      count_launch(8);
      w->ranks.push_back(m);
    }
    if (!take) CUDA_CHECK(cudaMemcpyAsync(w->g.rowptr.p + NL, &NNZ, sizeof(i64), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    tmps.clear();

    ptm.mark("concatenate");
    // ---- local routing (virtual ranks: every route has both ends in this process)
    if (w->all_local() && NG > 0) {
      std::vector<i64> lid_off_h((size_t)P);
      for (auto& m : w->ranks) lid_off_h[(size_t)m.rank] = m.lid_off;
      DBuf<i64> rank_off;
      rank_off.upload(lid_off_h.data(), P, s);
      DBuf<i32> src, dst, pair;
      src.alloc(NG, s);
      dst.alloc(NG, s);
      pair.alloc(NG, s);
      for (auto& m : w->ranks) {
        k_routes<<<G(m.ghost), 256, 0, s>>>(w->gids.p, w->ghost_owner.p + m.ghost_off, m.lid_off + m.owned,
                                             m.ghost, owned_lid.p, rank_off.p, m.rank, P,
                                             src.p + m.ghost_off, dst.p + m.ghost_off, pair.p + m.ghost_off);
        count_launch();
      }
      auto zs = thrust::make_zip_iterator(thrust::make_tuple(thrust::device_pointer_cast(dst.p),
                                                             thrust::device_pointer_cast(pair.p)));
      thrust::stable_sort_by_key(thrust::cuda::par.on(s), thrust::device_pointer_cast(src.p),
                                 thrust::device_pointer_cast(src.p) + NG, zs);
      count_launch();
      DBuf<uint8_t> head;
      head.alloc(NG, s);
      k_route_heads<<<G(NG), 256, 0, s>>>(src.p, NG, head.p);
      count_launch();
      DBuf<i32> hpos;
      hpos.alloc(NG, s);
      select_flagged(head.p, NG, hpos.p, cnt.p, s);
      const i64 nr = count_of(cnt.p);
      w->nrouted = nr;
      w->st_off.alloc(nr + 1, s);
      k_route_off<<<G(nr + 1), 256, 0, s>>>(hpos.p, cnt.p, NG, w->st_off.p);
      w->routed.alloc(nr, s);
      k_gather_i32<<<G(nr), 256, 0, s>>>(src.p, hpos.p, cnt.p, w->routed.p);
      count_launch(2);
      w->st_dst = std::move(dst);
      w->st_pair = std::move(pair);
      w->last_sent.alloc(nr, s);
      w->pair_cnt.alloc((i64)P * P, s);
      w->pair_cnt.zero(s);
    } else {
      w->pair_cnt.alloc((i64)P * P, s);
      w->pair_cnt.zero(s);
    }
    ptm.mark("routing");
    w->stats.alloc(4 + P, s);  // [0] conflicts [1] bytes [2] msgs [3..3+P) recolored, [3+P] next worklist
    w->changed.alloc(NL + 1, s);
    world_reset_exchange(*w);
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaGetLastError());
  } catch (...) {
    world_destroy(w);
    throw;
  }
  return w;
}

void world_destroy(World* w) {
  if (!w) return;
  cudaSetDevice(w->device);
  cudaStream_t s = w->stream;
  if (s) cudaStreamSynchronize(s);
  halo_release_p2p(*w);
  delete w;  // the NCCL communicator is borrowed (chroma_comm), not owned
  if (s) cudaStreamDestroy(s);
}

void world_reset_exchange(World& w) {
  if (w.nrouted) launch_fill_i32(w.last_sent.p, w.nrouted, NEVER_SENT, w.stream);
  if (w.nrouted_remote) launch_fill_i32(w.last_sent_remote.p, w.nrouted_remote, NEVER_SENT, w.stream);
}

void world_exchange_local(World& w, bool changed_only, bool write_all) {
  launch_exchange_local(w.routed.p, w.nrouted, w.st_off.p, w.st_dst.p, w.st_pair.p, w.colors.p,
                        w.last_sent.p, changed_only, write_all, w.pair_cnt.p, (i64)w.P * w.P, w.stream);
}

}  // namespace chroma
