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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <thrust/execution_policy.h>
#include <thrust/scan.h>

#include "world.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// hub bitmap over every local lid (2 MB at 16.8 M lids: stays in L2 for the row
// scans below, unlike the 4-byte degree array) and the owned-hub flags
__global__ void k_flag_hubs(const uint8_t* owned_flag, const i32* deg, i64 n, i32 T, uint8_t* flag, u32* bits) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + (threadIdx.x & 31);
    const bool hub = i < n && deg[i] > T;
    const u32 m = __ballot_sync(FULL, hub);
    if (i < n) flag[i] = hub && owned_flag[i];
    if ((threadIdx.x & 31) == 0) bits[b >> 5] = m;
  }
}
__device__ __forceinline__ bool is_hub(const u32* bits, i32 x) { return bits[x >> 5] >> (x & 31) & 1u; }

// Hub rows are long and skewed (one R-MAT hub holds ~1e5 entries), so they are cut
// into units of UNIT entries and every CTA takes units, not hubs.
constexpr i64 UNIT = 8192;

__global__ void k_hub_units(const i64* rowptr, const i64* gids, const i32* hubs, i64 nh, i64* nunits, i64* hgid) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nh; j += (i64)gridDim.x * blockDim.x) {
    const i32 v = hubs[j];
    nunits[j] = (rowptr[v + 1] - rowptr[v] + UNIT - 1) / UNIT;
    hgid[j] = gids[v];
  }
}
__global__ void k_hub_unit_owner(const i64* ustart, i64 nh, i32* unit_hub) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nh; j += (i64)gridDim.x * blockDim.x)
    for (i64 u = ustart[j]; u < ustart[j + 1]; u++) unit_hub[u] = (i32)j;
}

// FILL = false: hub-neighbour count per hub (cnt zeroed); FILL = true: the
// neighbours' gids at cursor[j] (initialised to the hub's offset)
template <bool FILL>
__global__ void __launch_bounds__(256) k_hub_scan(const i64* rowptr, const i32* col, const u32* bits,
                                                  const i64* gids, const i32* hubs, const i32* unit_hub,
                                                  const i64* ustart, const i64* nunits_total, i64* cnt_or_cursor,
                                                  i32* nbr) {
  __shared__ int tot;
  const int lane = threadIdx.x & 31;
  const i64 U = *nunits_total;
  for (i64 u = blockIdx.x; u < U; u += gridDim.x) {
    const i32 j = unit_hub[u];
    const i32 v = hubs[j];
    const i64 rs = rowptr[v] + (u - ustart[j]) * UNIT;
    const i64 re = min(rowptr[v + 1], rs + UNIT);
    if (!FILL) {
      if (threadIdx.x == 0) tot = 0;
      __syncthreads();
    }
    int c = 0;
    // 4 entries per thread in flight
    for (i64 b = rs + (threadIdx.x & ~31) * 4; b < re; b += (i64)blockDim.x * 4) {
      i32 x[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const i64 e = b + k * 32 + lane;
        x[k] = e < re ? ld_stream(col + e) : -1;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const bool h = x[k] >= 0 && is_hub(bits, x[k]);
        if (!FILL) {
          c += h;
        } else {
          const unsigned m = __ballot_sync(FULL, h);
          unsigned long long o = 0;
          if (lane == 0 && m) o = atomicAdd((unsigned long long*)cnt_or_cursor + j, (unsigned long long)__popc(m));
          o = __shfl_sync(FULL, o, 0);
          if (h) nbr[o + __popc(m & ((1u << lane) - 1))] = (i32)gids[x[k]];
        }
      }
    }
    if (!FILL) {
      c = __reduce_add_sync(FULL, c);
      if (lane == 0 && c) atomicAdd(&tot, c);
      __syncthreads();
      if (threadIdx.x == 0 && tot) atomicAdd((unsigned long long*)cnt_or_cursor + j, (unsigned long long)tot);
      __syncthreads();
    }
  }
}

// gid -> H index through a table over global ids: only hub gids are ever written or
// read (the table is not initialised), and every read is checked against the hub's
// own gid
__global__ void k_hub_table(const i64* hgid, i64 nh, i32* table) {
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < nh; k += (i64)gridDim.x * blockDim.x)
    table[hgid[k]] = (i32)k;
}
__device__ __forceinline__ i32 hub_index(const i32* table, const i64* hgid, i64 nh, i64 gid) {
  const i32 k = table[gid];
  return k >= 0 && k < nh && hgid[k] == gid ? k : -1;
}

__global__ void k_hub_map(const i32* nbr, i64 ne, const i32* table, const i64* hgid, i64 nh, i32* col,
                          unsigned long long* missing) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < ne; i += (i64)gridDim.x * blockDim.x) {
    const i32 k = hub_index(table, hgid, nh, nbr[i]);
    if (k < 0) atomicAdd(missing, 1ull);
    col[i] = k < 0 ? 0 : k;
  }
}

// every local vertex that is a hub (owned or ghost copy) takes H's colour
__global__ void k_hub_scatter(const u32* bits, const i64* gids, i64 n, const i32* table, const i64* hgid, i64 nh,
                              const i32* hcol, i32* colors) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    if (!is_hub(bits, (i32)i)) continue;
    const i32 k = hub_index(table, hgid, nh, gids[i]);
    if (k >= 0) colors[i] = hcol[k];
  }
}

__global__ void k_diff(const i64* off, i64 n, i64* out) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x)
    out[j] = off[j + 1] - off[j];
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
  auto t0 = std::chrono::steady_clock::now();
  std::vector<double> marks;
  auto mark = [&]() {
    if (!trace) return;
    CUDA_CHECK(cudaStreamSynchronize(s));
    marks.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  };
  // gids travel as int32 (the hub-neighbour lists are the bulk of the all-gather)
  if (w.n_global >= (1ll << 31)) return 0;
  // ---- this world's owned hubs, their row units and hub-neighbour counts
  H.flags.reserve(w.NL + 1, s);
  H.lhubs.reserve(w.NL + 1, s);
  H.nlh.reserve(1, s);
  H.bits.reserve((w.NL + 31) / 32 + 1, s);
  k_flag_hubs<<<G(w.NL), 256, 0, s>>>(w.owned_flag.p, w.deg.p, w.NL, T, H.flags.p, H.bits.p);
  count_launch();
  select_flagged(H.flags.p, w.NL, H.lhubs.p, H.nlh.p, s);
  i64 nh_local = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nh_local, H.nlh.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  H.lcnt.reserve(nh_local + 1, s);
  H.loff.reserve(nh_local + 1, s);
  H.lgid.reserve(nh_local + 1, s);
  H.nunits.reserve(nh_local + 1, s);
  H.ustart.reserve(nh_local + 1, s);
  i64 ne_local = 0, units = 0;
  const int gs = num_sms() * 8;
  if (nh_local > 0) {
    k_hub_units<<<G(nh_local), 256, 0, s>>>(w.g.rowptr.p, w.gids.p, H.lhubs.p, nh_local, H.nunits.p, H.lgid.p);
    CUDA_CHECK(cudaMemsetAsync(H.nunits.p + nh_local, 0, sizeof(i64), s));
    exclusive_scan_i64(H.nunits.p, H.ustart.p, nh_local + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(&units, H.ustart.p + nh_local, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    H.unit_hub.reserve(units + 1, s);
    k_hub_unit_owner<<<G(nh_local), 256, 0, s>>>(H.ustart.p, nh_local, H.unit_hub.p);
    CUDA_CHECK(cudaMemsetAsync(H.lcnt.p, 0, sizeof(i64) * (nh_local + 1), s));
    k_hub_scan<false><<<gs, 256, 0, s>>>(w.g.rowptr.p, w.g.col.p, H.bits.p, w.gids.p, H.lhubs.p, H.unit_hub.p,
                                         H.ustart.p, H.ustart.p + nh_local, H.lcnt.p, nullptr);
    count_launch(3);
    exclusive_scan_i64(H.lcnt.p, H.loff.p, nh_local + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(&ne_local, H.loff.p + nh_local, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // ---- sizes of every rank (connected worlds); lists padded to the largest
  const bool gather = w.connected && w.P > 1;
  const i32 P = gather ? w.P : 1;
  std::vector<i64> hs(2 * (size_t)P, 0);
  hs[0] = nh_local;
  hs[1] = ne_local;
  if (gather) {
#ifdef CHROMA_WITH_NCCL
    DBuf<i64> sizes;
    sizes.alloc(2 * (i64)P + 2, s);
    const i64 mine[2] = {nh_local, ne_local};
    CUDA_CHECK(cudaMemcpyAsync(sizes.p + 2 * (i64)P, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    HUB_NCCL(ncclAllGather(sizes.p + 2 * (i64)P, sizes.p, 2, ncclInt64, w.comm, s));
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), sizes.p, sizeof(i64) * 2 * P, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
#else
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  }
  std::vector<i64> ho((size_t)P + 1, 0), eo((size_t)P + 1, 0);
  i64 maxH = 0, maxE = 0;
  for (i32 p = 0; p < P; p++) {
    ho[(size_t)p + 1] = ho[(size_t)p] + hs[2 * (size_t)p];
    eo[(size_t)p + 1] = eo[(size_t)p] + hs[2 * (size_t)p + 1];
    maxH = std::max(maxH, hs[2 * (size_t)p]);
    maxE = std::max(maxE, hs[2 * (size_t)p + 1]);
  }
  const i64 NH = ho[(size_t)P], NE = eo[(size_t)P];
  // ---- hub-neighbour gids (a cursor per hub, rows in any order)
  H.lnbr.reserve(maxE + 1, s);
  if (nh_local > 0) {
    CUDA_CHECK(cudaMemcpyAsync(H.lcnt.p, H.loff.p, sizeof(i64) * nh_local, cudaMemcpyDeviceToDevice, s));
    k_hub_scan<true><<<gs, 256, 0, s>>>(w.g.rowptr.p, w.g.col.p, H.bits.p, w.gids.p, H.lhubs.p, H.unit_hub.p,
                                        H.ustart.p, H.ustart.p + nh_local, H.lcnt.p, H.lnbr.p);
    count_launch();
  }
  mark();
  if (NH == 0) return 0;
  CHROMA_REQUIRE(NH < (1ll << 31), CHROMA_ERUNTIME, "hub index overflow");
  // per-hub counts (for H's row pointers) and gids, in H order = rank order
  H.cntz.reserve(NH + 1, s);
  H.ggid.reserve(NH + 1, s);
  const i32* hnbr = H.lnbr.p;
  if (nh_local) {
    // the fill advanced each cursor by the hub's count: count = cursor - offset,
    // recomputed as offset[j+1] - offset[j]
    k_diff<<<G(nh_local), 256, 0, s>>>(H.loff.p, nh_local, H.cntz.p + ho[0]);
    CUDA_CHECK(cudaMemcpyAsync(H.ggid.p, H.lgid.p, sizeof(i64) * nh_local, cudaMemcpyDeviceToDevice, s));
    count_launch();
  }
  if (gather) {
#ifdef CHROMA_WITH_NCCL
    // all-gather of equal-size (padded) blocks, then compaction into rank order
    H.pad64.reserve(2 * maxH * (i64)(P + 1) + 2, s);
    H.pad32.reserve(maxE * (i64)P + 1, s);
    i64* sendh = H.pad64.p + 2 * maxH * (i64)P;
    if (nh_local) {
      CUDA_CHECK(cudaMemcpyAsync(sendh, H.cntz.p, sizeof(i64) * nh_local, cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(sendh + maxH, H.ggid.p, sizeof(i64) * nh_local, cudaMemcpyDeviceToDevice, s));
    }
    HUB_NCCL(ncclGroupStart());
    HUB_NCCL(ncclAllGather(sendh, H.pad64.p, 2 * maxH, ncclInt64, w.comm, s));
    if (maxE) HUB_NCCL(ncclAllGather(H.lnbr.p, H.pad32.p, maxE, ncclInt32, w.comm, s));
    HUB_NCCL(ncclGroupEnd());
    H.gnbr.reserve(NE + 1, s);
    for (i32 p = 0; p < P; p++) {
      const i64 nh = hs[2 * (size_t)p], ne = hs[2 * (size_t)p + 1];
      if (nh) {
        CUDA_CHECK(cudaMemcpyAsync(H.cntz.p + ho[(size_t)p], H.pad64.p + 2 * maxH * p, sizeof(i64) * nh,
                                   cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(H.ggid.p + ho[(size_t)p], H.pad64.p + 2 * maxH * p + maxH, sizeof(i64) * nh,
                                   cudaMemcpyDeviceToDevice, s));
      }
      if (ne)
        CUDA_CHECK(cudaMemcpyAsync(H.gnbr.p + eo[(size_t)p], H.pad32.p + maxE * p, sizeof(i32) * ne,
                                   cudaMemcpyDeviceToDevice, s));
    }
    hnbr = H.gnbr.p;
#endif
  }
  mark();
  // ---- H as a CSR over hub indices
  H.rowptr.reserve(NH + 1, s);
  CUDA_CHECK(cudaMemsetAsync(H.cntz.p + NH, 0, sizeof(i64), s));
  exclusive_scan_i64(H.cntz.p, H.rowptr.p, NH + 1, s);
  H.table.reserve(w.n_global + 1, s);
  k_hub_table<<<G(NH), 256, 0, s>>>(H.ggid.p, NH, H.table.p);
  count_launch();
  H.col.reserve(NE + 1, s);
  H.missing.reserve(1, s);
  H.missing.zero(s);
  if (NE) {
    k_hub_map<<<G(NE), 256, 0, s>>>(hnbr, NE, H.table.p, H.ggid.p, NH, H.col.p, H.missing.p);
    count_launch();
  }
  mark();
  // ---- colour H exactly (largest degree first waves), identically on every rank
  H.colors.reserve(NH + 1, s);
  H.colors.zero(s);
  H.list.reserve(NH + 1, s);
  launch_iota_i32(H.list.p, NH, 0, s);
  H.ovf.reserve(NH + 1, s);
  H.novf.reserve(1, s);
  H.novf.zero(s);
  launch_free_heavy(H.rowptr.p, H.col.p, H.colors.p, H.list.p, NH, H.ovf.p, H.novf.p, 1, false, H.fw, s);
  mark();
  unsigned long long miss = 0;
  CUDA_CHECK(cudaMemcpyAsync(&miss, H.missing.p, sizeof(miss), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  CHROMA_REQUIRE(miss == 0, CHROMA_EPROTOCOL, "hub neighbour without a hub record (inconsistent degrees)");
  // ---- owned hubs and ghost copies of hubs take their colours (overflowed hubs stay
  // uncoloured and are coloured with the light vertices)
  k_hub_scatter<<<G(w.NL), 256, 0, s>>>(H.bits.p, w.gids.p, w.NL, H.table.p, H.ggid.p, NH, H.colors.p,
                                        w.colors.p);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
  if (trace) {
    mark();
    std::fprintf(stderr, "[hubs] %lld hubs (%lld local), %lld hub-hub entries (%lld local); us: extract %.0f "
                 "gather %.0f build %.0f waves %.0f scatter %.0f\n", (long long)NH, (long long)nh_local,
                 (long long)NE, (long long)ne_local, marks[0], marks[1] - marks[0], marks[2] - marks[1],
                 marks[3] - marks[2], marks[4] - marks[3]);
  }
  return NH;
}

}  // namespace chroma
