// Worklist-driven halo exchange for the free-running distance-1 path, and the NVLink
// peer-memory transport it uses between processes.
//
// After round 0 only the vertices an owner recoloured can change a ghost copy, so
// the exchange walks the worklist instead of every routed vertex (the reference
// re-scans its whole send map each round, chroma/runtime.py:271-308).  Each copy
// written is also appended to the receiver's changed-ghost list, which is exactly
// the ghost half of the next detection's changed set (detect.cu).
//
//  * virtual ranks (one process): plain stores into the same colour array;
//  * one rank per process: the owner stores the colour straight into the peer's
//    ghost slot over NVLink (cudaIpc-mapped peer region); a flag barrier over peer
//    memory then orders the stores before anyone's detection.  No NCCL launch, no pack/unpack,
//    no host round trip.  Round 0 (every boundary vertex changes) keeps the bulk
//    NCCL send/recv path.
// The reference's changed-only accounting (12 bytes per (vertex, destination) pair
// whose colour differs from the last one sent, one message per non-empty inbox) is
// kept per send entry.
#include <cstdlib>

#include "world.cuh"

namespace chroma {
namespace {

__global__ void k_route_index(const i32* routed, i64 n, i32* idx) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    idx[routed[i]] = (i32)i;
}

// (src, dst) message counters: shared per block, flushed with one atomic per pair
constexpr int PAIR_SHARED = 4096;

// virtual ranks: worklist vertex -> its ghost copies (same array) + changed flags
__global__ void k_xchg_local_list(const i32* wl, const i64* nwl_dev, const i32* route_idx, const i64* st_off,
                                  const i32* st_dst, const i32* st_pair, i32* colors, i32* last_sent,
                                  unsigned long long* pair_cnt, i64 npairs) {
  __shared__ unsigned sc[PAIR_SHARED];
  const bool local = npairs <= PAIR_SHARED;
  if (local)
    for (i64 k = threadIdx.x; k < npairs; k += blockDim.x) sc[k] = 0;
  __syncthreads();
  const i64 n = *nwl_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    const i32 r = route_idx[v];
    if (r < 0) continue;
    const i32 c = colors[v];
    const bool send = last_sent[r] != c;
    if (send) last_sent[r] = c;
    for (i64 t = st_off[r]; t < st_off[r + 1]; t++) {
      const i32 d = st_dst[t];
      colors[d] = c;
      if (send) {
        if (local) atomicAdd(&sc[st_pair[t]], 1u);
        else atomicAdd(&pair_cnt[st_pair[t]], 1ull);
      }
    }
  }
  __syncthreads();
  if (local)
    for (i64 k = threadIdx.x; k < npairs; k += blockDim.x)
      if (sc[k]) atomicAdd(&pair_cnt[k], (unsigned long long)sc[k]);
}

// one rank per process: worklist vertex -> peers' ghost slots over NVLink
__global__ void k_xchg_p2p(const i32* wl, const i64* nwl_dev, i64 lid_off, const i64* rs_off, const i32* rs_peer,
                           const i32* rs_rlid, i32* rs_last, const i32* colors, i32* const* peer_colors,
                           unsigned long long* pair_cnt, i32 P) {
  __shared__ unsigned sc[PAIR_SHARED];
  const bool local = P <= PAIR_SHARED;
  if (local)
    for (int k = threadIdx.x; k < P; k += blockDim.x) sc[k] = 0;
  __syncthreads();
  const i64 n = *nwl_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    const i64 o = v - lid_off;
    const i32 c = colors[v];
    for (i64 e = rs_off[o]; e < rs_off[o + 1]; e++) {
      const i32 p = rs_peer[e], r = rs_rlid[e];
      if (rs_last[e] != c) {
        rs_last[e] = c;
        if (local) atomicAdd(&sc[p], 1u);
        else atomicAdd(&pair_cnt[p], 1ull);
      }
      peer_colors[p][r] = c;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (local)
    for (int k = threadIdx.x; k < P; k += blockDim.x)
      if (sc[k]) atomicAdd(&pair_cnt[k], (unsigned long long)sc[k]);
}

// owned losers of the detection -> colour 0 in every ghost copy (virtual ranks)
__global__ void k_zero_local(const i32* list, const i64* n_dev, const i32* route_idx, const i64* st_off,
                             const i32* st_dst, i32* colors) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 r = route_idx[list[i]];
    if (r < 0) continue;
    for (i64 t = st_off[r]; t < st_off[r + 1]; t++) colors[st_dst[t]] = 0;
  }
}

// ... and over NVLink (the next NCCL allreduce orders these stores before anyone
// colours again)
__global__ void k_zero_p2p(const i32* list, const i64* n_dev, i64 lid_off, const i64* rs_off, const i32* rs_peer,
                           const i32* rs_rlid, i32* const* peer_colors) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 o = list[i] - lid_off;
    for (i64 e = rs_off[o]; e < rs_off[o + 1]; e++) peer_colors[rs_peer[e]][rs_rlid[e]] = 0;
  }
  __threadfence_system();
}

// all ranks: signal every peer, wait until every peer has signalled this epoch
__global__ void k_p2p_barrier(unsigned long long* const* peer_ctrl, unsigned long long* my_ctrl, int P, int me,
                              unsigned long long target) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();
  for (int p = 0; p < P; p++)
    if (p != me) atomicAdd_system(peer_ctrl[p] + 1, 1ull);
  volatile unsigned long long* arrivals = my_ctrl + 1;
  while (*arrivals < target) __nanosleep(100);
  __threadfence_system();
}

// after the bulk round-0 exchange every send entry carries its owner's colour
__global__ void k_init_rs_last(const i64* rs_off, i64 owned, i64 lid_off, const i32* colors, i32* rs_last) {
  for (i64 o = blockIdx.x * (i64)blockDim.x + threadIdx.x; o < owned; o += (i64)gridDim.x * blockDim.x) {
    const i32 c = colors[lid_off + o];
    for (i64 e = rs_off[o]; e < rs_off[o + 1]; e++) rs_last[e] = c;
  }
}

// virtual ranks: ghost lid -> owner lid (same array)
__global__ void k_kill_routes(const i32* routed, i64 nrouted, const i64* st_off, const i32* st_dst, i32* owner_lid) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nrouted; i += (i64)gridDim.x * blockDim.x)
    for (i64 t = st_off[i]; t < st_off[i + 1]; t++) owner_lid[st_dst[t]] = routed[i];
}

__global__ void k_clear_flags(const i32* list, const i64* n_dev, uint8_t* flags) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flags[list[i]] = 0;
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

}  // namespace

void halo_route_index(World& w) {
  cudaStream_t s = w.stream;
  if (w.route_idx.p && w.route_idx.n >= w.NL + 1) return;
  w.route_idx.alloc(w.NL + 1, s);
  launch_fill_i32(w.route_idx.p, w.NL + 1, -1, s);
  if (w.nrouted) {
    k_route_index<<<G(w.nrouted), 256, 0, s>>>(w.routed.p, w.nrouted, w.route_idx.p);
    count_launch();
  }
  if (!w.p2p) {
    // kill routes of virtual ranks: every ghost's owner entry lives in this array
    w.kill_lid.alloc(w.NL + 1, s);
    w.kill_rank.alloc(w.NL + 1, s);
    launch_fill_i32(w.kill_lid.p, w.NL + 1, -1, s);
    launch_fill_i32(w.kill_rank.p, w.NL + 1, -1, s);
    if (w.nrouted) {
      k_kill_routes<<<G(w.nrouted), 256, 0, s>>>(w.routed.p, w.nrouted, w.st_off.p, w.st_dst.p, w.kill_lid.p);
      count_launch();
    }
    w.gflag.alloc(w.NL + 1, s);
    w.gflag.zero(s);
  }
}

// the owned vertices flagged as losers since the last call (ascending) -> out,
// count -> *n_out (device); flags cleared
void halo_next_worklist(World& w, i32* out, i64* n_out) {
  cudaStream_t s = w.stream;
  if (w.p2p) {
    const RankMeta& m = w.ranks[0];
    select_flagged_base(w.my_flag + m.lid_off, m.owned, (i32)m.lid_off, out, n_out, s);
    k_clear_flags<<<G(m.owned), 256, 0, s>>>(out, n_out, w.my_flag);
  } else {
    select_flagged_base(w.gflag.p, w.NL, 0, out, n_out, s);
    k_clear_flags<<<G(w.NL), 256, 0, s>>>(out, n_out, w.gflag.p);
  }
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

KillRoute halo_kill_route(World& w) {
  KillRoute kr;
  kr.owner_lid = w.kill_lid.p;
  kr.owner_rank = w.kill_rank.p;
  kr.peer_colors = w.p2p ? w.peer_colors.p : nullptr;
  kr.peer_flag = w.p2p ? w.peer_flag.p : nullptr;
  kr.flags = w.p2p ? w.my_flag : w.gflag.p;
  return kr;
}

// all ranks have finished their kills (stores into peers are fenced by the barrier)
void halo_barrier(World& w) {
  if (!w.p2p) return;
  w.bar_epoch += (unsigned long long)(w.P - 1);
  k_p2p_barrier<<<1, 32, 0, w.stream>>>(w.peer_ctrl.p, w.my_ctrl, w.P, w.my_rank, w.bar_epoch);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

void halo_exchange_local_list(World& w, const i32* wl, const i64* nwl_dev, i64 nwl_max) {
  if (w.nrouted == 0 || nwl_max <= 0) return;
  k_xchg_local_list<<<G(nwl_max), 256, 0, w.stream>>>(wl, nwl_dev, w.route_idx.p, w.st_off.p, w.st_dst.p,
                                                       w.st_pair.p, w.colors.p, w.last_sent.p, w.pair_cnt.p, (i64)w.P * w.P);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

void halo_exchange_p2p(World& w, const i32* wl, const i64* nwl_dev, i64 nwl_max) {
  cudaStream_t s = w.stream;
  if (nwl_max > 0 && w.nsend > 0) {
    k_xchg_p2p<<<G(nwl_max), 256, 0, s>>>(wl, nwl_dev, w.ranks[0].lid_off, w.rs_off.p, w.rs_peer.p, w.rs_rlid.p,
                                          w.rs_last.p, w.colors.p, w.peer_colors.p, w.pair_cnt.p, w.P);
    count_launch();
  }
  CUDA_CHECK(cudaGetLastError());
  halo_barrier(w);
}

void halo_broadcast_losers(World& w, const i32* list, const i64* n_dev, i64 n_max) {
  if (n_max <= 0) return;
  cudaStream_t s = w.stream;
  if (w.p2p) {
    if (w.nsend > 0) {
      k_zero_p2p<<<G(n_max), 256, 0, s>>>(list, n_dev, w.ranks[0].lid_off, w.rs_off.p, w.rs_peer.p, w.rs_rlid.p,
                                          w.peer_colors.p);
      count_launch();
    }
  } else if (w.nrouted) {
    k_zero_local<<<G(n_max), 256, 0, s>>>(list, n_dev, w.route_idx.p, w.st_off.p, w.st_dst.p, w.colors.p);
    count_launch();
  }
  CUDA_CHECK(cudaGetLastError());
}

void halo_init_p2p_last(World& w) {
  const RankMeta& m = w.ranks[0];
  if (!w.p2p || m.owned == 0) return;
  k_init_rs_last<<<G(m.owned), 256, 0, w.stream>>>(w.rs_off.p, m.owned, m.lid_off, w.colors.p, w.rs_last.p);
  count_launch();
}

// ------------------------------------------------------------------ P2P setup
#ifdef CHROMA_WITH_NCCL
#define NCCL_OK(expr) ((expr) == ncclSuccess)

void halo_release_p2p(World& w) {
  for (void* b : w.peer_base)
    if (b) cudaIpcCloseMemHandle(b);
  w.peer_base.clear();
  if (w.ipc_base) {
    if (w.colors.borrowed) w.colors.release();
    cudaFree(w.ipc_base);
  }
  w.ipc_base = nullptr;
  w.my_ctrl = nullptr;
  w.my_flag = nullptr;
  w.p2p = false;
}

// Collective over w.comm: every rank ends with the same p2p decision.
void halo_setup_p2p(World& w, const std::vector<i32>& send_lids_abs, const std::vector<i32>& send_peer,
                    const std::vector<i32>& recv_lids_abs) {
  cudaStream_t s = w.stream;
  const i32 P = w.P, me = w.my_rank;
  const RankMeta& m = w.ranks[0];
  const bool disabled = std::getenv("CHROMA_NO_P2P") != nullptr;
  // 1. own region [ctrl 256 B | colours | changed flags (one byte per lid)]
  struct Info {
    cudaIpcMemHandle_t h;
    long long col_off, list_off;
    int ok;
  };
  Info mine{};
  const size_t ctrl = 256;
  const size_t col_bytes = ((sizeof(i32) * (size_t)(w.NL + 1)) + 255) / 256 * 256;
  const size_t list_bytes = (size_t)(w.NL + 1);
  mine.col_off = (long long)ctrl;
  mine.list_off = (long long)(ctrl + col_bytes);
  mine.ok = 0;
  if (!disabled && cudaMalloc(&w.ipc_base, ctrl + col_bytes + list_bytes) == cudaSuccess) {
    if (cudaIpcGetMemHandle(&mine.h, w.ipc_base) == cudaSuccess) mine.ok = 1;
  }
  cudaGetLastError();
  // 2. share (handle, offsets, ok) with every peer
  DBuf<char> sb, rb;
  sb.alloc(sizeof(Info), s);
  rb.alloc((i64)sizeof(Info) * P, s);
  CUDA_CHECK(cudaMemcpyAsync(sb.p, &mine, sizeof(Info), cudaMemcpyHostToDevice, s));
  if (!NCCL_OK(ncclAllGather(sb.p, rb.p, sizeof(Info), ncclChar, w.comm, s)))
    throw Error(CHROMA_ECUDA, "ncclAllGather (p2p setup) failed");
  std::vector<Info> all((size_t)P);
  CUDA_CHECK(cudaMemcpyAsync(all.data(), rb.p, sizeof(Info) * P, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  int ok = 1;
  for (auto& x : all) ok &= x.ok;
  // 3. open the peers' regions
  w.peer_base.assign((size_t)P, nullptr);
  if (ok) {
    for (i32 p = 0; p < P && ok; p++) {
      if (p == me) continue;
      if (cudaIpcOpenMemHandle(&w.peer_base[(size_t)p], all[(size_t)p].h, cudaIpcMemLazyEnablePeerAccess) !=
          cudaSuccess) {
        w.peer_base[(size_t)p] = nullptr;
        ok = 0;
      }
    }
    cudaGetLastError();
  }
  // 4. agree (min over ranks)
  DBuf<int> okd;
  okd.alloc(1, s);
  CUDA_CHECK(cudaMemcpyAsync(okd.p, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  if (!NCCL_OK(ncclAllReduce(okd.p, okd.p, 1, ncclInt32, ncclMin, w.comm, s)))
    throw Error(CHROMA_ECUDA, "ncclAllReduce (p2p setup) failed");
  CUDA_CHECK(cudaMemcpyAsync(&ok, okd.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (!ok) {
    halo_release_p2p(w);
    return;
  }
  // 5. remote lids: peer p's receive slots for my sends, in my send order
  std::vector<i32> rlid((size_t)std::max<i64>(w.nsend, 1));
  {
    DBuf<i32> rl_dev, rlid_dev;
    std::vector<i32> rl_local((size_t)std::max<i64>(w.nrecv, 1));
    for (i64 k = 0; k < w.nrecv; k++) rl_local[(size_t)k] = (i32)(recv_lids_abs[(size_t)k] - m.lid_off);
    rl_dev.upload(rl_local.data(), std::max<i64>(w.nrecv, 1), s);
    rlid_dev.alloc(std::max<i64>(w.nsend, 1), s);
    if (!NCCL_OK(ncclGroupStart())) throw Error(CHROMA_ECUDA, "ncclGroupStart failed");
    for (i32 p = 0; p < P; p++) {
      if (p == me) continue;
      if (w.recv_cnt[(size_t)p])
        ncclSend(rl_dev.p + w.recv_off[(size_t)p], w.recv_cnt[(size_t)p], ncclInt32, p, w.comm, s);
      if (w.send_cnt[(size_t)p])
        ncclRecv(rlid_dev.p + w.send_off[(size_t)p], w.send_cnt[(size_t)p], ncclInt32, p, w.comm, s);
    }
    if (!NCCL_OK(ncclGroupEnd())) throw Error(CHROMA_ECUDA, "remote lid exchange failed");
    CUDA_CHECK(cudaMemcpyAsync(rlid.data(), rlid_dev.p, sizeof(i32) * std::max<i64>(w.nsend, 1),
                               cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // 5b. owner lids of my ghosts: peer p's send lids for me, in my receive order
  std::vector<i32> olid((size_t)std::max<i64>(w.nrecv, 1));
  {
    DBuf<i32> sl_dev, ol_dev;
    std::vector<i32> sl_local((size_t)std::max<i64>(w.nsend, 1));
    for (i64 k = 0; k < w.nsend; k++) sl_local[(size_t)k] = (i32)(send_lids_abs[(size_t)k] - m.lid_off);
    sl_dev.upload(sl_local.data(), std::max<i64>(w.nsend, 1), s);
    ol_dev.alloc(std::max<i64>(w.nrecv, 1), s);
    if (!NCCL_OK(ncclGroupStart())) throw Error(CHROMA_ECUDA, "ncclGroupStart failed");
    for (i32 p = 0; p < P; p++) {
      if (p == me) continue;
      if (w.send_cnt[(size_t)p])
        ncclSend(sl_dev.p + w.send_off[(size_t)p], w.send_cnt[(size_t)p], ncclInt32, p, w.comm, s);
      if (w.recv_cnt[(size_t)p])
        ncclRecv(ol_dev.p + w.recv_off[(size_t)p], w.recv_cnt[(size_t)p], ncclInt32, p, w.comm, s);
    }
    if (!NCCL_OK(ncclGroupEnd())) throw Error(CHROMA_ECUDA, "owner lid exchange failed");
    CUDA_CHECK(cudaMemcpyAsync(olid.data(), ol_dev.p, sizeof(i32) * std::max<i64>(w.nrecv, 1),
                               cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  {
    std::vector<i32> kl((size_t)(w.NL + 1), -1), kp((size_t)(w.NL + 1), -1);
    for (i32 p = 0; p < P; p++)
      for (i64 k = w.recv_off[(size_t)p]; k < w.recv_off[(size_t)p + 1]; k++) {
        const i64 g = recv_lids_abs[(size_t)k];
        kl[(size_t)g] = olid[(size_t)k];
        kp[(size_t)g] = p;
      }
    w.kill_lid.upload(kl.data(), w.NL + 1, s);
    w.kill_rank.upload(kp.data(), w.NL + 1, s);
  }
  // 6. send entries grouped by owned lid (counting sort)
  std::vector<i64> off((size_t)m.owned + 1, 0);
  for (i64 k = 0; k < w.nsend; k++) off[(size_t)(send_lids_abs[(size_t)k] - m.lid_off) + 1]++;
  for (i64 o = 0; o < m.owned; o++) off[(size_t)o + 1] += off[(size_t)o];
  std::vector<i64> fill(off.begin(), off.end() - 1);
  std::vector<i32> ep((size_t)std::max<i64>(w.nsend, 1)), er((size_t)std::max<i64>(w.nsend, 1));
  for (i64 k = 0; k < w.nsend; k++) {
    const i64 o = send_lids_abs[(size_t)k] - m.lid_off;
    const i64 at = fill[(size_t)o]++;
    ep[(size_t)at] = send_peer[(size_t)k];
    er[(size_t)at] = rlid[(size_t)k];
  }
  w.rs_off.upload(off.data(), m.owned + 1, s);
  w.rs_peer.upload(ep.data(), std::max<i64>(w.nsend, 1), s);
  w.rs_rlid.upload(er.data(), std::max<i64>(w.nsend, 1), s);
  w.rs_last.alloc(std::max<i64>(w.nsend, 1), s);
  // 7. pointers: own colours move into the shared region
  char* base = (char*)w.ipc_base;
  CUDA_CHECK(cudaMemsetAsync(base, 0, ctrl, s));
  i32* region_colors = (i32*)(base + ctrl);
  CUDA_CHECK(cudaMemcpyAsync(region_colors, w.colors.p, sizeof(i32) * (size_t)(w.NL + 1), cudaMemcpyDeviceToDevice,
                             s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  w.colors.borrow(region_colors, w.NL + 1);
  w.my_ctrl = (unsigned long long*)base;
  w.my_flag = (uint8_t*)(base + mine.list_off);
  CUDA_CHECK(cudaMemsetAsync(w.my_flag, 0, list_bytes, s));
  std::vector<i32*> pc((size_t)P, nullptr);
  std::vector<uint8_t*> pl((size_t)P, nullptr);
  std::vector<unsigned long long*> pctl((size_t)P, nullptr);
  for (i32 p = 0; p < P; p++) {
    char* b = p == me ? base : (char*)w.peer_base[(size_t)p];
    pc[(size_t)p] = (i32*)(b + all[(size_t)p].col_off);
    pl[(size_t)p] = (uint8_t*)(b + all[(size_t)p].list_off);
    pctl[(size_t)p] = (unsigned long long*)b;
  }
  w.peer_colors.upload(pc.data(), P, s);
  w.peer_flag.upload(pl.data(), P, s);
  w.peer_ctrl.upload(pctl.data(), P, s);
  w.bar_epoch = 0;
  // everyone's control block is zero before anyone signals
  DBuf<int> z;
  z.alloc(1, s);
  if (!NCCL_OK(ncclAllReduce(z.p, z.p, 1, ncclInt32, ncclSum, w.comm, s)))
    throw Error(CHROMA_ECUDA, "ncclAllReduce (p2p setup) failed");
  CUDA_CHECK(cudaStreamSynchronize(s));
  w.p2p = true;
}
#else
void halo_release_p2p(World& w) { (void)w; }
void halo_setup_p2p(World& w, const std::vector<i32>&, const std::vector<i32>&, const std::vector<i32>&) {
  w.p2p = false;
}
#endif

}  // namespace chroma
