// Global hub pre-colouring for the free-running distance-1 path across ranks.
//
// On one rank the free mode colours the heavy rows (R-MAT hubs) first, exactly, in
// largest-degree-first waves (color_free.cu), so the dense core never speculates.
// Split over P ranks, every rank's waves run concurrently: the top hubs of
// different ranks take the same first colours, nearly every cross-rank hub pair
// collides, and the losers collide again round after round (the hubs form a near
// clique).  Here the hubs of ALL ranks are coloured once, before round 0, as one
// graph: every rank contributes its owned hubs' hub-neighbour lists (gid space),
// the lists are all-gathered (NCCL over NVLink between processes; already local for
// virtual ranks), and every rank colours the same hub subgraph H with the same
// deterministic wave kernel -- identical results everywhere, no exchange of the
// result needed.  Each rank then writes the hub colours into its owned hubs and
// into its ghost copies of remote hubs, so round 0's light colouring already
// avoids every hub colour and cross-rank conflicts are left to light vertices
// only.  A hub is a vertex whose global degree exceeds the threshold (owned rows
// are complete in the local graphs, so the owner and every ghost holder agree).
//
// This is a free-running extension (AlgorithmConfig(algorithm="free")); the
// reference's deterministic and Jacobi modes never take it.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <thrust/execution_policy.h>
#include <thrust/scan.h>

#include "world.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__global__ void k_flag_hubs(const uint8_t* owned_flag, const i32* deg, i64 n, i32 T, uint8_t* flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flag[i] = owned_flag[i] && deg[i] > T;
}

// one CTA per owned hub: number of hub neighbours, and the hub's gid
__global__ void k_hub_count(const i64* rowptr, const i32* col, const i32* deg, const i64* gids, const i32* hubs,
                            const i64* nh_dev, i32 T, i64* cnt, i64* hgid) {
  __shared__ int tot;
  const i64 nh = *nh_dev;
  for (i64 j = blockIdx.x; j < nh; j += gridDim.x) {
    const i32 v = hubs[j];
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    int c = 0;
    for (i64 e = rowptr[v] + threadIdx.x; e < rowptr[v + 1]; e += blockDim.x) c += deg[col[e]] > T;
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&tot, c);
    __syncthreads();
    if (threadIdx.x == 0) {
      cnt[j] = tot;
      hgid[j] = gids[v];
    }
    __syncthreads();
  }
}

// one CTA per owned hub: its hub neighbours' gids (row order is irrelevant to the
// wave kernel, which ORs masks)
__global__ void k_hub_fill(const i64* rowptr, const i32* col, const i32* deg, const i64* gids, const i32* hubs,
                           const i64* nh_dev, i32 T, const i64* off, i64* nbr) {
  __shared__ unsigned long long pos;
  const int lane = threadIdx.x & 31;
  const i64 nh = *nh_dev;
  for (i64 j = blockIdx.x; j < nh; j += gridDim.x) {
    const i32 v = hubs[j];
    if (threadIdx.x == 0) pos = 0;
    __syncthreads();
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    for (i64 b = rs + (threadIdx.x & ~31); b < re; b += blockDim.x) {
      const i64 e = b + lane;
      const i32 x = e < re ? col[e] : -1;
      const bool h = x >= 0 && deg[x] > T;
      const unsigned m = __ballot_sync(FULL, h);
      unsigned long long o = 0;
      if (lane == 0 && m) o = atomicAdd(&pos, (unsigned long long)__popc(m));
      o = __shfl_sync(FULL, o, 0);
      if (h) nbr[off[j] + (i64)o + __popc(m & ((1u << lane) - 1))] = gids[x];
    }
    __syncthreads();
  }
}

__global__ void k_hub_keys(const i64* hgid, i64 nh, u64* keys) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nh; i += (i64)gridDim.x * blockDim.x)
    keys[i] = ((u64)hgid[i] << 32) | (u64)i;
}

// gid -> H index by binary search over the sorted (gid << 32 | index) keys; -1 if absent
__device__ __forceinline__ i32 hub_index(const u64* keys, i64 nh, i64 gid) {
  i64 lo = 0, hi = nh;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if ((i64)(keys[mid] >> 32) < gid) lo = mid + 1;
    else hi = mid;
  }
  return lo < nh && (i64)(keys[lo] >> 32) == gid ? (i32)(keys[lo] & 0xffffffffu) : -1;
}

__global__ void k_hub_map(const i64* nbr, i64 ne, const u64* keys, i64 nh, i32* col, unsigned long long* missing) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < ne; i += (i64)gridDim.x * blockDim.x) {
    const i32 k = hub_index(keys, nh, nbr[i]);
    if (k < 0) atomicAdd(missing, 1ull);
    col[i] = k < 0 ? 0 : k;
  }
}

// every local vertex that is a hub (owned or ghost copy) takes H's colour
__global__ void k_hub_scatter(const i32* deg, const i64* gids, i64 n, i32 T, const u64* keys, i64 nh,
                              const i32* hcol, i32* colors) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    if (deg[i] <= T) continue;
    const i32 k = hub_index(keys, nh, gids[i]);
    if (k >= 0) colors[i] = hcol[k];
  }
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

#ifdef CHROMA_WITH_NCCL
#define HUB_NCCL(expr)                                                                          \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) throw Error(CHROMA_ECUDA, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#endif

}  // namespace

i64 hub_precolor(World& w, i32 T) {
  cudaStream_t s = w.stream;
  static const bool trace = std::getenv("CHROMA_FREE_TRACE") != nullptr;
  HubScratch& H = w.hub;
  // ---- this world's owned hubs and their hub-neighbour lists (gid space)
  H.flags.reserve(w.NL + 1, s);
  H.lhubs.reserve(w.NL + 1, s);
  H.nlh.reserve(1, s);
  k_flag_hubs<<<G(w.NL), 256, 0, s>>>(w.owned_flag.p, w.deg.p, w.NL, T, H.flags.p);
  count_launch();
  select_flagged(H.flags.p, w.NL, H.lhubs.p, H.nlh.p, s);
  i64 nh_local = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nh_local, H.nlh.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  H.lcnt.reserve(nh_local + 1, s);
  H.loff.reserve(nh_local + 1, s);
  H.lgid.reserve(nh_local + 1, s);
  const int gb = (int)std::max<i64>(1, std::min<i64>(nh_local, (i64)num_sms() * 8));
  i64 ne_local = 0;
  if (nh_local > 0) {
    k_hub_count<<<gb, 256, 0, s>>>(w.g.rowptr.p, w.g.col.p, w.deg.p, w.gids.p, H.lhubs.p, H.nlh.p, T, H.lcnt.p,
                                    H.lgid.p);
    count_launch();
    CUDA_CHECK(cudaMemsetAsync(H.lcnt.p + nh_local, 0, sizeof(i64), s));
    exclusive_scan_i64(H.lcnt.p, H.loff.p, nh_local + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(&ne_local, H.loff.p + nh_local, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  H.lnbr.reserve(ne_local + 1, s);
  if (nh_local > 0) {
    k_hub_fill<<<gb, 256, 0, s>>>(w.g.rowptr.p, w.g.col.p, w.deg.p, w.gids.p, H.lhubs.p, H.nlh.p, T, H.loff.p,
                                   H.lnbr.p);
    count_launch();
  }
  // ---- all-gather over the ranks of other processes (rank order = H order)
  const i64* hgid = H.lgid.p;
  const i64* hcnt = H.lcnt.p;
  const i64* hnbr = H.lnbr.p;
  i64 NH = nh_local, NE = ne_local;
  if (w.connected && w.P > 1) {
#ifdef CHROMA_WITH_NCCL
    const i32 P = w.P;
    DBuf<i64> sizes;
    sizes.alloc(2 * (i64)P + 2, s);
    const i64 mine[2] = {nh_local, ne_local};
    CUDA_CHECK(cudaMemcpyAsync(sizes.p + 2 * (i64)P, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    HUB_NCCL(ncclAllGather(sizes.p + 2 * (i64)P, sizes.p, 2, ncclInt64, w.comm, s));
    std::vector<i64> hs(2 * (size_t)P);
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), sizes.p, sizeof(i64) * 2 * P, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<i64> ho((size_t)P + 1, 0), eo((size_t)P + 1, 0);
    for (i32 p = 0; p < P; p++) {
      ho[(size_t)p + 1] = ho[(size_t)p] + hs[2 * (size_t)p];
      eo[(size_t)p + 1] = eo[(size_t)p] + hs[2 * (size_t)p + 1];
    }
    NH = ho[(size_t)P];
    NE = eo[(size_t)P];
    H.ggid.reserve(NH + 1, s);
    H.gcnt.reserve(NH + 1, s);
    H.gnbr.reserve(NE + 1, s);
    const i32 me = w.my_rank;
    if (nh_local) {
      CUDA_CHECK(cudaMemcpyAsync(H.ggid.p + ho[(size_t)me], H.lgid.p, sizeof(i64) * nh_local,
                                 cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(H.gcnt.p + ho[(size_t)me], H.lcnt.p, sizeof(i64) * nh_local,
                                 cudaMemcpyDeviceToDevice, s));
    }
    if (ne_local)
      CUDA_CHECK(cudaMemcpyAsync(H.gnbr.p + eo[(size_t)me], H.lnbr.p, sizeof(i64) * ne_local,
                                 cudaMemcpyDeviceToDevice, s));
    HUB_NCCL(ncclGroupStart());
    for (i32 p = 0; p < P; p++) {
      if (p == me) continue;
      const i64 rh = hs[2 * (size_t)p], re = hs[2 * (size_t)p + 1];
      if (nh_local) {
        HUB_NCCL(ncclSend(H.lgid.p, nh_local, ncclInt64, p, w.comm, s));
        HUB_NCCL(ncclSend(H.lcnt.p, nh_local, ncclInt64, p, w.comm, s));
      }
      if (ne_local) HUB_NCCL(ncclSend(H.lnbr.p, ne_local, ncclInt64, p, w.comm, s));
      if (rh) {
        HUB_NCCL(ncclRecv(H.ggid.p + ho[(size_t)p], rh, ncclInt64, p, w.comm, s));
        HUB_NCCL(ncclRecv(H.gcnt.p + ho[(size_t)p], rh, ncclInt64, p, w.comm, s));
      }
      if (re) HUB_NCCL(ncclRecv(H.gnbr.p + eo[(size_t)p], re, ncclInt64, p, w.comm, s));
    }
    HUB_NCCL(ncclGroupEnd());
    hgid = H.ggid.p;
    hcnt = H.gcnt.p;
    hnbr = H.gnbr.p;
#else
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  }
  if (NH == 0) return 0;
  CHROMA_REQUIRE(w.n_global < (1ll << 32) && NH < (1ll << 31), CHROMA_ERUNTIME, "hub index overflow");
  // ---- H as a CSR over hub indices
  H.rowptr.reserve(NH + 1, s);
  H.cntz.reserve(NH + 1, s);
  CUDA_CHECK(cudaMemcpyAsync(H.cntz.p, hcnt, sizeof(i64) * NH, cudaMemcpyDeviceToDevice, s));
  CUDA_CHECK(cudaMemsetAsync(H.cntz.p + NH, 0, sizeof(i64), s));
  exclusive_scan_i64(H.cntz.p, H.rowptr.p, NH + 1, s);
  H.keys.reserve(NH, s);
  k_hub_keys<<<G(NH), 256, 0, s>>>(hgid, NH, H.keys.p);
  count_launch();
  sort_u64(H.keys.p, NH, s);
  H.col.reserve(NE + 1, s);
  H.missing.reserve(1, s);
  H.missing.zero(s);
  if (NE) {
    k_hub_map<<<G(NE), 256, 0, s>>>(hnbr, NE, H.keys.p, NH, H.col.p, H.missing.p);
    count_launch();
  }
  // ---- colour H exactly (largest degree first waves), identically on every rank
  H.colors.reserve(NH + 1, s);
  H.colors.zero(s);
  H.list.reserve(NH + 1, s);
  launch_iota_i32(H.list.p, NH, 0, s);
  H.ovf.reserve(NH + 1, s);
  H.novf.reserve(1, s);
  H.novf.zero(s);
  launch_free_heavy(H.rowptr.p, H.col.p, H.colors.p, H.list.p, NH, H.ovf.p, H.novf.p, 1, false, H.fw, s);
  unsigned long long miss = 0;
  CUDA_CHECK(cudaMemcpyAsync(&miss, H.missing.p, sizeof(miss), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  CHROMA_REQUIRE(miss == 0, CHROMA_EPROTOCOL, "hub neighbour without a hub record (inconsistent degrees)");
  // ---- owned hubs and ghost copies of hubs take their colours (overflowed hubs stay
  // uncoloured and are coloured with the light vertices)
  k_hub_scatter<<<G(w.NL), 256, 0, s>>>(w.deg.p, w.gids.p, w.NL, T, H.keys.p, NH, H.colors.p, w.colors.p);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
  if (trace) {
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[hubs] %lld hubs (%lld local), %lld hub-hub entries (%lld local)\n", (long long)NH,
                 (long long)nh_local, (long long)NE, (long long)ne_local);
  }
  return NH;
}

}  // namespace chroma
