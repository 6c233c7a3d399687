// The speculate-and-iterate round loop (chroma/protocol.py:263-334) and the local
// colouring driver (chroma/localcolor.py:198-303), entirely device-side except for
// one small D2H of the round's counters (and of the conflict-event count).
//
// Per round, per the reference:
//   colour the worklist (round 0: every owned vertex; later: every uncoloured local
//   vertex, F7) -> restore ghosts -> exchange (changed-only accounting, F11) ->
//   snapshot ghosts -> detect -> allreduce -> stop on zero (F12: max_rounds+1 rounds).
// Device formulation: the exchange rewrites every routed ghost from its owner each
// round, which leaves every ghost equal to the owner's colour -- exactly the state
// restore + changed-only exchange produces -- so no snapshot buffer is needed.  In
// Gauss-Seidel mode ghost worklist entries are skipped: ghosts have larger local ids
// than every owned vertex, so their sequential recolouring can only affect other
// ghosts, which the restore/exchange overwrites.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include "world.cuh"

namespace chroma {
namespace {

__global__ void k_flag_worklist(const i32* colors, const uint8_t* owned_flag, i64 n, bool owned_only,
                                uint8_t* flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flag[i] = (colors[i] == 0 && (!owned_only || owned_flag[i])) ? 1 : 0;
}

// recolored_per_rank: owned entries of the worklist per local rank.  Worklists are
// ascending, so a thread's entries mostly share one rank: count runs in a register,
// flush into a block histogram on change, one global atomic per block and rank.
__global__ void k_count_recolored(const i32* wl, const i64* nwl, const uint8_t* owned_flag,
                                  const i32* rank_of, i32 rank_lo, i32 nlocal, unsigned long long* stats) {
  __shared__ unsigned long long h[256];
  const bool local_hist = nlocal <= 256;
  if (local_hist)
    for (int i = threadIdx.x; i < nlocal; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const i64 n = *nwl;
  i32 cur = -1;
  unsigned long long run = 0;
  auto flush = [&]() {
    if (run == 0) return;
    if (local_hist) atomicAdd(&h[cur], run);
    else atomicAdd(&stats[3 + rank_lo + cur], run);
    run = 0;
  };
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    if (!owned_flag[v]) continue;
    const i32 r = rank_of[v];
    if (r != cur) {
      flush();
      cur = r;
    }
    run++;
  }
  // last run: one shared atomic per warp and rank (lanes mostly share one rank)
  {
    const unsigned grp = __match_any_sync(0xffffffffu, cur);
    const unsigned tot = __reduce_add_sync(grp, (unsigned)run);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) run = tot;
    else run = 0;
  }
  flush();
  __syncthreads();
  if (local_hist)
    for (int i = threadIdx.x; i < nlocal; i += blockDim.x)
      if (h[i]) atomicAdd(&stats[3 + rank_lo + i], h[i]);
}

__global__ void k_set_u8_idx(uint8_t* flags, const i32* idx, const i64* n_dev, uint8_t v) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    flags[idx[i]] = v;
}

__global__ void k_gather_owned(const i64* gids, const i32* colors, i64 lo, i64 n, i32* out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[gids[lo + i]] = colors[lo + i];
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

i64 read_i64(const i64* d, cudaStream_t s) {
  i64 h = 0;
  CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  return h;
}

constexpr int MAX_SWEEPS = 10000;  // chroma/localcolor.py:34

i64 env_i64(const char* name, i64 dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoll(v) : dflt;
}

}  // namespace

// ------------------------------------------------------------------ colouring driver
void color_csr(const i64* rowptr, const i32* col, i64 nv, i32* colors, const i32* wl_in,
               const i64* nwl_dev, i64 nwl_max, bool wl_sorted_unique, int dist, bool partial,
               int algo, bool colors_nonneg, ColorScratch& S, cudaStream_t s, cudaEvent_t ev_k0,
               cudaEvent_t ev_k1) {
  if (nwl_max <= 0) return;
  S.nwl.reserve(1, s);
  S.ticket.reserve(1, s);
  const i32* wl = wl_in;
  const i64* nwl = nwl_dev;
  if (!wl_sorted_unique) {
    // the reference sorts the worklist (np.sort); duplicates are idempotent
    S.wl.reserve(nwl_max, s);
    CUDA_CHECK(cudaMemcpyAsync(S.wl.p, wl_in, sizeof(i32) * nwl_max, cudaMemcpyDeviceToDevice, s));
    auto b = thrust::device_pointer_cast(S.wl.p);
    thrust::sort(thrust::cuda::par.on(s), b, b + nwl_max);
    const i64 k = thrust::unique(thrust::cuda::par.on(s), b, b + nwl_max) - b;
    count_launch(2);
    CUDA_CHECK(cudaMemcpyAsync(S.nwl.p, &k, sizeof(i64), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    wl = S.wl.p;
    nwl = S.nwl.p;
    nwl_max = k;
  }
  if (algo == CHROMA_ALGO_FREE) {
    // color_free.cu: exact waves over heavy rows, then in-place first fit over the
    // light ones -> larger id keeps its colour -> the losers iterate until none is
    // left.  A distance-1 worklist without heavy rows (meshes, later rounds) has no
    // dense core to speculate around: it takes the ordered dataflow kernel instead,
    // which is conflict-free and uses the reference's colour count.
    for (auto& b : S.fl) b.reserve(nwl_max, s);
    S.fcnt.reserve(6, s);
    FreeLists f{{S.fl[0].p, S.fl[1].p}, {S.fl[2].p, S.fl[3].p}, {S.fl[4].p, S.fl[5].p}, S.fcnt.p};
    static const i64 heavy_deg = env_i64("CHROMA_FREE_HEAVY", 4096);
    static const i64 rank_cap = env_i64("CHROMA_FREE_RANKCAP", 0);
    static const bool trace = std::getenv("CHROMA_FREE_TRACE") != nullptr;
    if (ev_k0) CUDA_CHECK(cudaEventRecord(ev_k0, s));
    static const i64 tiny_deg = env_i64("CHROMA_FREE_TINY", 32);
    static const i64 tail_n = env_i64("CHROMA_FREE_TAIL", 4096);
    static const i64 tail_after = env_i64("CHROMA_FREE_TAIL_AFTER", 2);
    launch_free_split(wl, nwl, nwl_max, rowptr, dist == 1 ? tiny_deg : -1, heavy_deg, f, 0, s);
    i64 cnt[6];
    CUDA_CHECK(cudaMemcpyAsync(cnt, S.fcnt.p, 3 * sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (dist == 1 && cnt[1] == 0 && !S.keep_free) {  // no heavy rows
      algo = CHROMA_ALGO_GAUSS_SEIDEL;
      goto gauss_seidel;
    }
    {
    i32* cur = colors;
    if (!colors_nonneg) {
      S.val.reserve(nv, s);
      launch_clamp_nonneg(S.val.p, colors, nv, s);
      cur = S.val.p;
    }
    launch_scatter_const(cur, wl, nwl, nwl_max, 0, s);
    if (dist == 2) {
      // Distance 2: bounded-degree meshes are order-sensitive (first fit in id order
      // keeps the reference's colour count) -> the ordered kernel;
      // everything else -> net-centric speculation (color_net.cu).
      const i64 nexact = read_i64(nwl, s);
      if (worklist_max_degree(wl, nexact, rowptr, S.net, s) <= 26) {
        if (!colors_nonneg) launch_scatter_from(colors, S.val.p, wl, nwl, nwl_max, s);
        algo = CHROMA_ALGO_GAUSS_SEIDEL;
        goto gauss_seidel;
      }
      if (launch_free_net(rowptr, col, nv, cur, wl, nexact, partial, S.net, s)) {
        if (ev_k1) CUDA_CHECK(cudaEventRecord(ev_k1, s));
        if (!colors_nonneg) launch_scatter_from(colors, S.val.p, wl, nwl, nwl_max, s);
        return;
      }
    }
    if (cnt[1] > 0) {
      const auto tw0 = std::chrono::steady_clock::now();
      const i64 nh = cnt[1];
      launch_free_heavy(rowptr, col, cur, f.heavy[0], cnt[1], f.light[0], f.cnt, dist, partial, S.fw, s);
      CUDA_CHECK(cudaMemsetAsync(f.cnt + 1, 0, sizeof(i64), s));
      CUDA_CHECK(cudaMemcpyAsync(cnt, S.fcnt.p, 3 * sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      if (trace)
        std::fprintf(stderr, "[free] heavy waves (%lld vertices) %.1f us, light %lld\n", (long long)nh,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tw0).count(),
                     (long long)cnt[0]);
    }
    auto tl = std::chrono::steady_clock::now();
    for (int it = 0; it < MAX_SWEEPS; it++) {
      const int p = it & 1, q = p ^ 1;
      launch_free_iteration(rowptr, col, cur, f, p, cnt + 3 * p, it > 0 ? (int)rank_cap : 0, dist, partial, s);
      CUDA_CHECK(cudaMemcpyAsync(cnt + 3 * q, S.fcnt.p + 3 * q, 3 * sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      if (trace) {
        const auto tn = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[free] it=%d light %lld -> %lld heavy %lld -> %lld tiny %lld -> %lld (%.0f us)\n", it,
                     (long long)cnt[3 * p], (long long)cnt[3 * q], (long long)cnt[3 * p + 1],
                     (long long)cnt[3 * q + 1], (long long)cnt[3 * p + 2], (long long)cnt[3 * q + 2],
                     std::chrono::duration<double, std::micro>(tn - tl).count());
        tl = tn;
      }
      const i64 pend = cnt[3 * q] + cnt[3 * q + 1] + cnt[3 * q + 2];
      if (pend > 0 && it + 1 >= tail_after && pend <= tail_n) {
        // a small remainder that keeps colliding is a dense cluster: finish it
        // exactly with the wave kernel instead of iterating one layer at a time
        i32* dst = f.heavy[q];
        i64 k = cnt[3 * q + 1];
        CUDA_CHECK(cudaMemcpyAsync(dst + k, f.light[q], sizeof(i32) * cnt[3 * q], cudaMemcpyDeviceToDevice, s));
        k += cnt[3 * q];
        CUDA_CHECK(cudaMemcpyAsync(dst + k, f.tiny[q], sizeof(i32) * cnt[3 * q + 2], cudaMemcpyDeviceToDevice, s));
        k += cnt[3 * q + 2];
        CUDA_CHECK(cudaMemsetAsync(f.cnt + 3 * q, 0, 3 * sizeof(i64), s));
        launch_free_heavy(rowptr, col, cur, dst, k, f.light[q], f.cnt + 3 * q, dist, partial, S.fw, s);
        CUDA_CHECK(cudaMemcpyAsync(cnt + 3 * q, S.fcnt.p + 3 * q, 3 * sizeof(i64), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (trace) std::fprintf(stderr, "[free] tail waves over %lld, %lld left\n", (long long)k, (long long)cnt[3 * q]);
      }
      if (cnt[3 * q] == 0 && cnt[3 * q + 1] == 0 && cnt[3 * q + 2] == 0) {
        if (ev_k1) CUDA_CHECK(cudaEventRecord(ev_k1, s));
        if (!colors_nonneg) launch_scatter_from(colors, S.val.p, wl, nwl, nwl_max, s);
        return;
      }
    }
    throw Error(CHROMA_ERUNTIME, "speculative loop failed to settle");
    }
  }
gauss_seidel:
  if (algo == CHROMA_ALGO_GAUSS_SEIDEL) {
    GsLaunch L;
    L.rowptr = rowptr;
    L.col = col;
    if (colors_nonneg) {
      // protocol path: worklist colours are 0 and no colour is negative
      L.val = colors;
      L.old = nullptr;
      launch_scatter_const(colors, wl, nwl, nwl_max, PENDING, s);
    } else {
      S.val.reserve(nv, s);
      S.old.reserve(nv, s);
      CUDA_CHECK(cudaMemcpyAsync(S.old.p, colors, sizeof(i32) * nv, cudaMemcpyDeviceToDevice, s));
      launch_clamp_nonneg(S.val.p, colors, nv, s);
      launch_scatter_const(S.val.p, wl, nwl, nwl_max, PENDING, s);
      L.val = S.val.p;
      L.old = S.old.p;
    }
    L.wl = wl;
    L.nwl_dev = nwl;
    L.nwl_max = nwl_max;
    L.ticket = S.ticket.p;
    L.dist = dist;
    L.partial = partial;
    L.nv = nv;
    if (S.level_wl && dist == 1) {
      // same vertex set, claimed level by level or rank-interleaved (gs_levels.cu)
      S.level_n_dev.reserve(1, s);
      CUDA_CHECK(cudaMemcpyAsync(S.level_n_dev.p, &S.level_n, sizeof(i64), cudaMemcpyHostToDevice, s));
      L.wl = S.level_wl;
      L.nwl_dev = S.level_n_dev.p;
      L.nwl_max = S.level_n;
      L.level_mode = S.level_mode;
    }
    static const bool no_chunked = std::getenv("CHROMA_NO_CHUNKED") != nullptr;
    const bool cluster = S.level_wl && S.level_mode && S.cplan && dist == 1 && !L.old;
    // a level schedule without the cluster (too many vertices for its shared memory):
    // the level-ordered dataflow kernel; otherwise the chunked one
    const bool levels = S.level_wl && S.level_mode && !cluster;
    if (dist == 1 && !cluster && !levels && !no_chunked) {
      // chunked fixed point over the original worklist (gs_chunked.cu)
      const i64 nexact = wl_sorted_unique && nwl != nullptr ? read_i64(nwl, s) : nwl_max;
      GsLaunch C = L;
      C.wl = wl;
      C.nwl_dev = nwl;
      C.nwl_max = nexact;
      C.level_mode = false;
      if (ev_k0) CUDA_CHECK(cudaEventRecord(ev_k0, s));
      if (launch_gs_chunked(C, nexact, S.upper_zero, S.chunked, s)) {
        if (ev_k1) CUDA_CHECK(cudaEventRecord(ev_k1, s));
        if (!colors_nonneg) launch_scatter_from(colors, S.val.p, wl, nwl, nwl_max, s);
        return;
      }
    }
    if (ev_k0) CUDA_CHECK(cudaEventRecord(ev_k0, s));
    if (cluster) {
      launch_gs_cluster(*S.cplan, L.val, L.old, s);
    } else {
      if (S.level_wl && S.level_mode && S.cplan && S.cplan->chains) {
        // a schedule with runs is for the cluster kernel only: plain id order here
        L.wl = wl;
        L.nwl_dev = nwl;
        L.nwl_max = nwl_max;
        L.level_mode = false;
      }
      launch_gs(L, s);
    }
    if (ev_k1) CUDA_CHECK(cudaEventRecord(ev_k1, s));
    if (!colors_nonneg) launch_scatter_from(colors, S.val.p, wl, nwl, nwl_max, s);
    return;
  }
  // Jacobi sweeps (chroma/localcolor.py:214-227, 292-303); CHROMA_ALGO_JACOBI_EB takes
  // the edge-based kernels (chroma/localcolor.py:181-195) -- same losers (F3)
  const bool edge_based = algo == CHROMA_ALGO_JACOBI_EB;
  S.in_round.reserve(nv, s);
  CUDA_CHECK(cudaMemsetAsync(S.in_round.p, 0, nv, s));
  k_set_u8_idx<<<G(nwl_max), 256, 0, s>>>(S.in_round.p, wl, nwl, 1);
  count_launch();
  S.prop.reserve(nwl_max, s);
  S.flags.reserve(nwl_max, s);
  S.pend2.reserve(nwl_max, s);
  S.np2.reserve(1, s);
  S.val.reserve(nwl_max, s);
  CUDA_CHECK(cudaMemcpyAsync(S.val.p, wl, sizeof(i32) * nwl_max, cudaMemcpyDeviceToDevice, s));
  CUDA_CHECK(cudaMemcpyAsync(S.np2.p, nwl, sizeof(i64), cudaMemcpyDeviceToDevice, s));
  i32* pend = S.val.p;
  i64 np = read_i64(nwl, s);  // exact count: the compaction below takes a host length
  // after sweep 0, long pending rows are kept incrementally (jacobi_inc.cu): same
  // proposals and losers, rows not re-read every sweep
  static const bool no_inc = std::getenv("CHROMA_JACOBI_FULL") != nullptr;
  S.ji.on = false;
  static const bool jtrace = std::getenv("CHROMA_JACOBI_TRACE") != nullptr;
  for (int sweep = 0; sweep < MAX_SWEEPS; sweep++) {
    if (jtrace && (sweep < 8 || (sweep & (sweep - 1)) == 0 || np == 0)) {
      static auto jt = std::chrono::steady_clock::now();
      const auto tn = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[jacobi] sweep %d pending %lld%s (+%.0f us)\n", sweep, (long long)np,
                   S.ji.on ? " inc" : "", std::chrono::duration<double, std::micro>(tn - jt).count());
      jt = tn;
    }
    if (np == 0) return;
    if (S.ji.on) {
      jacobi_inc_propose(rowptr, col, colors, pend, S.np2.p, np, S.prop.p, S.ji, s);
      launch_scatter_idx_values(colors, pend, S.prop.p, S.np2.p, np, s);
      jacobi_inc_losers(rowptr, col, colors, pend, S.np2.p, np, S.in_round.p, S.flags.p, S.ji, s);
      jacobi_inc_update(colors, pend, S.np2.p, np, S.flags.p, S.ji, s);
    } else if (edge_based && dist == 1) {
      launch_jacobi_eb(rowptr, col, colors, pend, np, S.prop.p, S.in_round.p, S.flags.p, S.eb, s);
    } else {
      launch_jacobi_propose(rowptr, col, colors, pend, S.np2.p, np, S.prop.p, dist, partial, s);
      launch_jacobi_losers(rowptr, col, colors, pend, S.np2.p, np, S.prop.p, S.in_round.p, S.flags.p,
                           dist, partial, s);
    }
    select_flagged_values(pend, S.flags.p, np, S.pend2.p, S.np2.p, s);
    unsigned ovf = 0;
    CUDA_CHECK(cudaMemcpyAsync(&np, S.np2.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
    if (S.ji.on) CUDA_CHECK(cudaMemcpyAsync(&ovf, jacobi_inc_overflow_dev(S.ji), sizeof(ovf), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    launch_scatter_const(colors, S.pend2.p, S.np2.p, np, 0, s);
    std::swap(S.pend2, S.val);
    pend = S.val.p;
    if (ovf) S.ji.on = false;  // a colour fb cannot hold: full sweeps from here
    if (sweep == 0 && dist == 1 && np > 0 && !no_inc)
      jacobi_inc_init(rowptr, col, colors, pend, np, nv, S.ji, s);
  }
  // the reference raises after the last sweep even if it settled (chroma/localcolor.py:218-227)
  throw Error(CHROMA_ERUNTIME, "speculative loop failed to settle");
}

// ------------------------------------------------------------------ remote exchange
namespace {
__global__ void k_changed(const i32* routed, i64 n, const i32* colors, i32* last_sent, bool changed_only,
                          uint8_t* changed) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = routed[i];
    const i32 c = colors[v];
    const bool send = !changed_only || last_sent[i] != c;
    if (send) last_sent[i] = c;
    changed[v] = send ? 1 : 0;
  }
}
// send lists are grouped by peer: a thread's run of one peer is counted in a
// register and flushed into a shared counter when the peer changes, one global
// atomic per block and peer at the end
__global__ void k_pack(const i32* send_lids, const i32* send_peer, i64 n, const i32* colors,
                       const uint8_t* changed, i32* buf, unsigned long long* peer_cnt, i32 P) {
  __shared__ unsigned sc[1024];
  const bool local = P <= 1024;
  if (local)
    for (int k = threadIdx.x; k < P; k += blockDim.x) sc[k] = 0;
  __syncthreads();
  i32 cur = -1;
  unsigned run = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = send_lids[i];
    buf[i] = colors[v];
    if (changed[v]) {
      const i32 p = send_peer[i];
      if (p != cur) {
        if (run) {
          if (local) atomicAdd(&sc[cur], run);
          else atomicAdd(&peer_cnt[cur], (unsigned long long)run);
        }
        cur = p;
        run = 0;
      }
      run++;
    }
  }
  if (run) {
    if (local) atomicAdd(&sc[cur], run);
    else atomicAdd(&peer_cnt[cur], (unsigned long long)run);
  }
  __syncthreads();
  if (local)
    for (int k = threadIdx.x; k < P; k += blockDim.x)
      if (sc[k]) atomicAdd(&peer_cnt[k], (unsigned long long)sc[k]);
}
__global__ void k_unpack(const i32* recv_lids, i64 n, const i32* buf, i32* colors) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    colors[recv_lids[i]] = buf[i];
}
}  // namespace

#ifdef CHROMA_WITH_NCCL
#define NCCL_CHECK(expr)                                                                        \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) throw Error(CHROMA_ECUDA, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#endif

// Pack -> grouped NCCL send/recv over NVLink -> unpack, with the reference's
// changed-only accounting of this rank's sends added to stats[1..2].
static void exchange_remote(World& w, bool changed_only) {
#ifdef CHROMA_WITH_NCCL
  cudaStream_t s = w.stream;
  if (w.nrouted_remote)
    k_changed<<<G(w.nrouted_remote), 256, 0, s>>>(w.routed_remote.p, w.nrouted_remote, w.colors.p,
                                                   w.last_sent_remote.p, changed_only, w.changed.p);
  if (w.nsend)
    k_pack<<<G(w.nsend), 256, 0, s>>>(w.send_lids.p, w.send_peer.p, w.nsend, w.colors.p, w.changed.p,
                                       w.sendbuf.p, w.pair_cnt.p, w.P);
  count_launch(2);
  NCCL_CHECK(ncclGroupStart());
  for (i32 p = 0; p < w.P; p++) {
    if (p == w.my_rank) continue;
    if (w.send_cnt[p]) NCCL_CHECK(ncclSend(w.sendbuf.p + w.send_off[p], w.send_cnt[p], ncclInt32, p, w.comm, s));
    if (w.recv_cnt[p]) NCCL_CHECK(ncclRecv(w.recvbuf.p + w.recv_off[p], w.recv_cnt[p], ncclInt32, p, w.comm, s));
  }
  NCCL_CHECK(ncclGroupEnd());
  if (w.nrecv) {
    k_unpack<<<G(w.nrecv), 256, 0, s>>>(w.recv_lids.p, w.nrecv, w.recvbuf.p, w.colors.p);
    count_launch();
  }
  launch_pair_stats(w.pair_cnt.p, w.P, w.stats.p + 1, s);
  CUDA_CHECK(cudaGetLastError());
#else
  (void)w; (void)changed_only;
  throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
}

// Distance 2 without the partial (bipartite) restriction on a bounded-degree graph:
// the distance-1 kernels on the square G^2 (square.cu) -- identical forbidden sets,
// orders and loser rule (Gauss-Seidel, Jacobi; the free mode colours such graphs by
// Gauss-Seidel too).  Detection stays on G.  Builds G^2 on first use; returns whether
// (crow, ccol, cdist, cdelta) now describe it.
bool square_for(World& w, int dist, bool partial, int algo, bool owned_worklist, const i64*& crow, const i32*& ccol,
                int& cdist, i64& cdelta) {
  static const bool no_square = std::getenv("CHROMA_NO_SQUARE") != nullptr;
  if (dist != 2 || no_square) return false;
  // full D2: bounded degree (meshes); PD2: Gauss-Seidel and Jacobi while the two-hop
  // rows fit in memory (the free mode keeps the net-centric kernels, which read less)
  if (!partial ? w.delta_max > 11 : (algo == CHROMA_ALGO_FREE || w.delta_max > 128)) return false;
  // Gauss-Seidel rounds colour owned vertices only: the (large) partial rows of the
  // ghosts are not needed then
  const bool owned_only = partial && owned_worklist && algo == CHROMA_ALGO_GAUSS_SEIDEL;
  const int kind = !partial ? 1 : owned_only ? 3 : 2;
  if (w.sq_state != 0 && w.sq_kind != kind) {  // another square: rebuild
    w.sq_state = 0;
    w.sq_rowptr.release();
    w.sq_col.release();
  }
  if (w.sq_state == 0) {
    static const bool ltrace = std::getenv("CHROMA_LEVEL_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const i64 budget = (i64)(free_b / 2 / sizeof(i32));  // at most half the free memory
    i64 md = 0;
    w.sq_kind = kind;
    w.sq_state = build_square(w.g.rowptr.p, w.g.col.p, w.NL, w.delta_max, partial, budget,
                              owned_only ? w.owned_flag.p : nullptr, w.sq_rowptr, w.sq_col, md, w.stream) ? 1 : -1;
    w.sq_delta = md;
    if (ltrace)
      std::fprintf(stderr, "[square] %s%s, max degree %lld, %.2f ms\n", partial ? "partial, " : "",
                   w.sq_state == 1 ? "built" : "not applicable", (long long)md,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  if (w.sq_state != 1) return false;
  crow = w.sq_rowptr.p;
  ccol = w.sq_col.p;
  cdist = 1;
  cdelta = w.sq_delta;
  return true;
}

// ------------------------------------------------------------------ round loop
int run_distributed(World& w, int mode, bool rd, int algo, int max_rounds, i32* colors_out,
                    chroma_round_report* reports, i64* recolored, i64 cap, i64* n_reports,
                    bool out_on_device) {
  const int need = mode == CHROMA_MODE_D1 ? 1 : 2;
  CHROMA_REQUIRE(w.gl >= need, CHROMA_EVALUE, "mode needs more ghost layers than the world was built with");
  CHROMA_REQUIRE(max_rounds >= 1, CHROMA_EVALUE, "max_rounds must be >= 1");
  CHROMA_REQUIRE(w.all_local() || w.connected || w.P == 1, CHROMA_EVALUE,
                 "world holds a subset of ranks: call chroma_world_connect first");
  CUDA_CHECK(cudaSetDevice(w.device));
  cudaStream_t s = w.stream;
  const bool d2 = mode >= CHROMA_MODE_D2;
  const bool partial = mode == CHROMA_MODE_PD2;
  const int dist = d2 ? 2 : 1;
  world_reset_exchange(w);
  w.colors.zero(s);
  w.cs.wl.reserve(w.NL + 1, s);
  w.cs.nwl.reserve(1, s);
  w.cs.flags.reserve(w.NL + 1, s);
  const i64 nstats = 3 + w.P;  // allreduced; hs[nstats] is this process's next-worklist size
  std::vector<unsigned long long> hs((size_t)nstats + 1);
  // Free-running fast path (all modes): after round 0 the worklist is the owned
  // losers flagged by any rank's detection, the exchange walks only that worklist
  // (NVLink peer stores between processes), and the detection only the recoloured
  // owned vertices' sets, uncolouring each loser at its owner (halo_p2p.cu).
  static const bool no_fast = std::getenv("CHROMA_NO_FAST_FREE") != nullptr;
  static const bool no_levels = std::getenv("CHROMA_NO_LEVELS") != nullptr;
  static const bool no_cluster = std::getenv("CHROMA_NO_CLUSTER") != nullptr;
  static const bool no_chains = std::getenv("CHROMA_NO_CHAINS") != nullptr;
  // round-0 schedule: 0 auto (levels if the DAG is wide, else rank-interleaved for
  // virtual ranks, else id order), 1 levels only, 2 interleave only, 3 id order
  static const int sched = (int)env_i64("CHROMA_GS_SCHEDULE", 0);
  // Level frontiers expand row by row: hub rows (R-MAT) make a level step as slow as
  // its longest row and such DAGs are deep anyway, and the free mode only takes the
  // ordered kernel on hub-free worklists -- levels are built for bounded-degree graphs.
  static const i64 level_max_deg = env_i64("CHROMA_LEVEL_MAX_DEG", 1024);
  const bool fast = algo == CHROMA_ALGO_FREE && !no_fast && (!w.connected || w.p2p || w.P == 1);
  const bool is_jacobi = algo == CHROMA_ALGO_JACOBI || algo == CHROMA_ALGO_JACOBI_EB;
  // free-running D1 over several ranks: colour the hubs of all ranks first (hubs.cu)
  static const bool no_hubs = std::getenv("CHROMA_NO_HUBS") != nullptr;
  const i64 hub_deg = env_i64("CHROMA_HUB_DEG", 4096);  // read per call (tests vary it)
  const bool hubs_first = algo == CHROMA_ALGO_FREE && !d2 && w.P > 1 && !no_hubs &&
                          (w.all_local() || w.connected) && w.delta_max > hub_deg;
  if (fast) {
    halo_route_index(w);
    w.next_wl.reserve(w.NL + 1, s);
    w.nghost_dev.reserve(2, s);
    const unsigned long long ng[2] = {(unsigned long long)w.NGHOST, (unsigned long long)w.NB2};
    CUDA_CHECK(cudaMemcpyAsync(w.nghost_dev.p, ng, sizeof(ng), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  i64 nwl_host = w.NL;
  cudaEvent_t ev[8];
  for (auto& e : ev) CUDA_CHECK(cudaEventCreate(&e));
  w.t_total = w.t_color_kernel = w.t_color = w.t_comm = w.t_detect = 0;
  CUDA_CHECK(cudaEventRecord(ev[4], s));
  int status = CHROMA_OK;
  i64 round = 0;
  DetectArgs da;
  da.rowptr = w.g.rowptr.p;
  da.col = w.g.col.p;
  da.colors = w.colors.p;
  da.gids = w.gids.p;
  da.deg = w.deg.p;
  da.rows = d2 ? w.b2.p : w.ghosts.p;
  da.nrows = d2 ? w.NB2 : w.NGHOST;
  da.dist = dist;
  da.partial = partial;
  da.recolor_degrees = rd;
  da.sequential = algo != CHROMA_ALGO_FREE;
  da.incremental = true;
  da.owned_flag = w.owned_flag.p;
  w.det.prev_valid = false;
  const bool remote = w.connected && w.P > 1;
  const i64* crow = w.g.rowptr.p;
  const i32* ccol = w.g.col.p;
  int cdist = dist;
  i64 cdelta = w.delta_max;
  const bool use_sq = square_for(w, dist, partial, algo, true, crow, ccol, cdist, cdelta);
  const int lgraph = use_sq ? w.sq_kind : 0;
  if (w.level_n >= 0 && w.level_sq != lgraph) w.level_n = -1;  // a schedule of another graph
  bool hubs_done = false;
  // CHROMA_ROUND_TRACE[=r]: synchronised per-phase host timings of round r (default 0; dev aid)
  static const bool round_trace = std::getenv("CHROMA_ROUND_TRACE") != nullptr;
  static const i64 trace_round = env_i64("CHROMA_ROUND_TRACE", 0);
  auto rt_last = std::chrono::steady_clock::now();
  i64 rt_round = 0;
  auto rt_mark = [&](const char* what) {
    if (!round_trace || rt_round != trace_round) return;
    CUDA_CHECK(cudaStreamSynchronize(s));
    const auto tn = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[round%lld] %-18s %8.1f us\n", (long long)rt_round, what, std::chrono::duration<double, std::micro>(tn - rt_last).count());
    rt_last = tn;
  };
  for (;;) {
    if (round > max_rounds) {
      status = CHROMA_ENONCONV;
      break;
    }
    if (round >= cap) {
      status = CHROMA_ERUNTIME;
      break;
    }
    CUDA_CHECK(cudaMemsetAsync(w.stats.p, 0, sizeof(unsigned long long) * (nstats + 1), s));
    CUDA_CHECK(cudaEventRecord(ev[0], s));
    rt_round = round;
    rt_mark("start");
    if (round == 0 && hubs_first) {
      // hubs.cu: every rank's hubs coloured once, identically everywhere; the
      // round-0 worklist below then holds the light vertices only, and every round
      // keeps the speculative path (the ordered kernel's id chain is long on such
      // graphs even without the hubs)
      hubs_done = hub_precolor(w, (i32)hub_deg) > 0;
    }
    w.cs.keep_free = hubs_done;
    if (fast && round > 0) {
      // the previous detection's owned losers, ascending
      nwl_host = (i64)hs[(size_t)nstats];
      CUDA_CHECK(cudaMemcpyAsync(w.cs.wl.p, w.next_wl.p, sizeof(i32) * std::max<i64>(nwl_host, 1),
                                 cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(w.cs.nwl.p, &hs[(size_t)nstats], sizeof(i64), cudaMemcpyHostToDevice, s));
    } else {
      // worklist (ordered compaction: ascending local id)
      // Jacobi re-colours uncoloured ghosts too (F7); the other modes only owned ones
      k_flag_worklist<<<G(w.NL), 256, 0, s>>>(w.colors.p, w.owned_flag.p, w.NL,
                                              round == 0 || !is_jacobi, w.cs.flags.p);
      count_launch();
      select_flagged(w.cs.flags.p, w.NL, w.cs.wl.p, w.cs.nwl.p, s);
      nwl_host = w.NL;
    }
    k_count_recolored<<<grid_for(w.NL, 256, num_sms() * 16), 256, 0, s>>>(w.cs.wl.p, w.cs.nwl.p, w.owned_flag.p, w.rank_of.p, w.rank_lo,
                                              w.rank_hi - w.rank_lo, w.stats.p);
    count_launch();
    const bool gs_like = !is_jacobi;
    // round 0 colours every owned vertex: claim them by DAG level (cached per world)
    w.cs.level_wl = nullptr;
    // The schedule is built from round 0's full owned worklist and cached per world:
    // not when hubs were pre-coloured (the worklist then lacks them), and only for
    // bounded degree (the cluster kernel); other graphs take gs_chunked.cu.
    if (round == 0 && cdist == 1 && gs_like && !no_levels && !hubs_done && cdelta <= 32) {
      if (w.level_n < 0) {
        w.level_sq = lgraph;
        i64 owned = 0;
        std::vector<i64> counts;
        for (auto& m : w.ranks) {
          owned += m.owned;
          counts.push_back(m.owned);
        }
        i64 n = 0;
        // levels when the DAG is wide; else (virtual ranks) rank-interleaved id order
        // bounded degree <= 32: try the cluster kernel (gs_cluster.cu), which walks
        // narrow levels as cheaply as wide ones; otherwise only wide DAGs take levels
        const bool try_cluster = cdelta <= 32 && !no_cluster && w.NL <= cluster_max_vertices();
        // the cluster kernel resolves runs of adjacent consecutive ids in one level
        const bool chains = try_cluster && !no_chains;
        std::vector<i64> lsizes;
        static const bool ltrace = std::getenv("CHROMA_LEVEL_TRACE") != nullptr;
        const auto lt0 = std::chrono::steady_clock::now();
        w.level_mode = (sched == 0 || sched == 1) && cdelta <= level_max_deg &&
                       build_level_order(crow, ccol, w.NL, w.cs.wl.p, owned, w.level_wl, n, s,
                                         &lsizes, try_cluster ? 1 : -1, chains);
        const auto lt1 = std::chrono::steady_clock::now();
        if (w.level_mode && try_cluster &&
            !build_cluster_plan(crow, ccol, w.NL, cdelta, w.level_wl.p, n, lsizes, w.cplan, s,
                                chains, !hubs_done)) {
          // no cluster: keep the schedule only if it is wide enough for the dataflow
          // kernel (and has no runs, which only the cluster kernel evaluates)
          if (chains || (i64)lsizes.size() * 2048 > owned) w.level_mode = false;
        }
        if (ltrace) {
          CUDA_CHECK(cudaStreamSynchronize(s));
          const auto lt2 = std::chrono::steady_clock::now();
          std::fprintf(stderr, "[levels] build %.2f ms, cluster plan %.2f ms\n",
                       std::chrono::duration<double, std::milli>(lt1 - lt0).count(),
                       std::chrono::duration<double, std::milli>(lt2 - lt1).count());
        }
        w.level_n = w.level_mode ? n : 0;
        if (!w.level_mode && (sched == 0 || sched == 2) &&
            build_rank_interleave(w.cs.wl.p, counts, w.level_wl, n, s))
          w.level_n = n;
        // the colour array is untouched; restart the round's timing after the one-time build
        CUDA_CHECK(cudaEventRecord(ev[0], s));
      }
      if (w.level_n > 0) {
        w.cs.level_wl = w.level_wl.p;
        w.cs.level_n = w.level_n;
        w.cs.level_mode = w.level_mode;
        // a plan without ghost slots needs every ghost at 0 (no pre-coloured hubs)
        w.cs.cplan = w.level_mode && w.cplan.ok && !(w.cplan.zero_nm && hubs_done) ? &w.cplan : nullptr;
      }
    }
    rt_mark("hubs+worklist");
    w.cs.upper_zero = round == 0 && !hubs_done;  // nothing is coloured before round 0
    color_csr(crow, ccol, w.NL, w.colors.p, w.cs.wl.p, w.cs.nwl.p, nwl_host, true, cdist, partial,
              algo, true, w.cs, s, gs_like ? ev[6] : nullptr, gs_like ? ev[7] : nullptr);
    rt_mark("color");
    w.cs.level_wl = nullptr;
    w.cs.cplan = nullptr;
    w.cs.keep_free = false;
    w.cs.upper_zero = false;
    CUDA_CHECK(cudaEventRecord(ev[1], s));
    // exchange: every ghost takes its owner's colour; accounting is changed-only
    const bool listed = fast && round > 0;  // exchange and detection driven by lists
    if (w.nrouted) {
      if (listed) halo_exchange_local_list(w, w.cs.wl.p, w.cs.nwl.p, nwl_host);
      else world_exchange_local(w, round > 0, true);
      launch_pair_stats(w.pair_cnt.p, (i64)w.P * w.P, w.stats.p + 1, s);
    }
    if (remote) {
      if (listed) {
        halo_exchange_p2p(w, w.cs.wl.p, w.cs.nwl.p, nwl_host);
        launch_pair_stats(w.pair_cnt.p, w.P, w.stats.p + 1, s);
      } else {
        rt_mark("pre-exchange");
        exchange_remote(w, round > 0);
        rt_mark("exchange_remote");
        if (fast) halo_init_p2p_last(w);
        rt_mark("init_p2p_last");
      }
    }
    CUDA_CHECK(cudaEventRecord(ev[2], s));
    if (fast && w.NGHOST == 0) {
      // no cut edges: a locally proper colouring is final
    } else if (fast) {
      // Round 0 (every vertex changed): one side of each cut pair suffices -- the
      // ghost rows for D1 (every cut edge is in one; rows hold local edges only), the
      // owned boundary_d2 rows for D2/PD2.  Later rounds: a conflicting pair always
      // has a recoloured end, and that end's owner finds it, so only the worklist
      // is walked.  Losers are uncoloured at their owners (NVLink for peers).
      FreeList list;
      if (!listed) {
        if (d2) list = {w.b2.p, w.nghost_dev.p + 1, w.NB2};
        else list = {w.ghosts.p, w.nghost_dev.p, w.NGHOST};
      } else {
        list = {w.cs.wl.p, reinterpret_cast<const unsigned long long*>(w.cs.nwl.p), nwl_host};
      }
      run_detect_free_lists(da, w.NL, &list, 1, halo_kill_route(w), w.det, w.stats.p, s);
      rt_mark("detect");
      halo_barrier(w);  // every rank's kills have landed
      rt_mark("barrier");
      i64* next_cnt = reinterpret_cast<i64*>(w.stats.p + nstats);
      halo_next_worklist(w, w.next_wl.p, next_cnt);
      rt_mark("next_worklist");
      halo_broadcast_losers(w, w.next_wl.p, next_cnt, w.NL);
      rt_mark("broadcast_losers");
    } else {
      run_detect(da, w.NL, w.det, w.stats.p, s);
      rt_mark("detect");
    }
#ifdef CHROMA_WITH_NCCL
    if (remote)
      NCCL_CHECK(ncclAllReduce(w.stats.p, w.stats.p, nstats, ncclUint64, ncclSum, w.comm, s));
#endif
    rt_mark("allreduce");
    CUDA_CHECK(cudaEventRecord(ev[3], s));
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), w.stats.p, sizeof(unsigned long long) * (nstats + 1),
                               cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    float t01 = 0, t12 = 0, t23 = 0, tk = 0;
    if (gs_like && w.NL > 0) cudaEventElapsedTime(&tk, ev[6], ev[7]);
    w.t_color_kernel += tk * 1e-3;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t12, ev[1], ev[2]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    chroma_round_report& R = reports[round];
    R.round_index = round;
    R.conflicts = (int64_t)hs[0];
    R.bytes_sent = (int64_t)hs[1];
    R.messages_sent = (int64_t)hs[2];
    R.time_color_s = t01 * 1e-3;
    R.time_comm_s = t12 * 1e-3;
    R.time_detect_s = t23 * 1e-3;
    w.t_color += R.time_color_s;
    w.t_comm += R.time_comm_s;
    w.t_detect += R.time_detect_s;
    for (i32 r = 0; r < w.P; r++) recolored[round * w.P + r] = (i64)hs[(size_t)(3 + r)];
    round++;
    if (hs[0] == 0) break;
  }
  *n_reports = round;
  if (status == CHROMA_OK && colors_out) {
    if (w.all_local()) {
      DBuf<i32> out;
      i32* dst = colors_out;
      if (!out_on_device) {
        out.alloc(w.n_global + 1, s);
        dst = out.p;
      }
      for (auto& m : w.ranks) {
        k_gather_owned<<<G(m.owned), 256, 0, s>>>(w.gids.p, w.colors.p, m.lid_off, m.owned, dst);
        count_launch();
      }
      if (!out_on_device)
        CUDA_CHECK(cudaMemcpyAsync(colors_out, out.p, sizeof(i32) * w.n_global, cudaMemcpyDeviceToHost, s));
    } else {
      const RankMeta& m = w.ranks[0];
      CUDA_CHECK(cudaMemcpyAsync(colors_out, w.colors.p + m.lid_off, sizeof(i32) * m.owned,
                                 out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    }
  }
  CUDA_CHECK(cudaEventRecord(ev[5], s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  {
    float tt = 0;
    cudaEventElapsedTime(&tt, ev[4], ev[5]);
    w.t_total = tt * 1e-3;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return status;
}

// ------------------------------------------------------------------ connect (NCCL)
#ifdef CHROMA_WITH_NCCL
// Install the static halo routing computed by the host (dist.build_routing: ghost
// slots grouped by owner; owned lids each peer asked for) and create this rank's
// NCCL communicator.  All lists are in local ids of this process's single rank.
void world_connect(World& w, void* comm, i32 nranks, i32 rank, const i64* send_counts,
                   const i64* send_lids, const i64* recv_counts, const i64* recv_lids) {
  CHROMA_REQUIRE(nranks == w.P, CHROMA_EVALUE, "communicator size differs from num_ranks");
  CHROMA_REQUIRE(w.rank_hi - w.rank_lo == 1 && w.rank_lo == rank, CHROMA_EVALUE,
                 "connected worlds hold exactly their own rank");
  CUDA_CHECK(cudaSetDevice(w.device));
  cudaStream_t s = w.stream;
  const RankMeta& m = w.ranks[0];
  const i32 P = w.P;
  w.send_cnt.assign(send_counts, send_counts + P);
  w.recv_cnt.assign(recv_counts, recv_counts + P);
  CHROMA_REQUIRE(w.send_cnt[(size_t)rank] == 0 && w.recv_cnt[(size_t)rank] == 0, CHROMA_EPROTOCOL,
                 "a rank cannot route to itself");
  w.send_off.assign((size_t)P + 1, 0);
  w.recv_off.assign((size_t)P + 1, 0);
  for (i32 p = 0; p < P; p++) {
    w.send_off[(size_t)p + 1] = w.send_off[(size_t)p] + w.send_cnt[(size_t)p];
    w.recv_off[(size_t)p + 1] = w.recv_off[(size_t)p] + w.recv_cnt[(size_t)p];
  }
  w.nsend = w.send_off[(size_t)P];
  w.nrecv = w.recv_off[(size_t)P];
  CHROMA_REQUIRE(w.nrecv == m.ghost, CHROMA_EPROTOCOL, "every ghost slot must be received exactly once");
  std::vector<i32> sl((size_t)w.nsend), sp((size_t)w.nsend), rl((size_t)w.nrecv);
  std::vector<uint8_t> routed((size_t)m.owned + 1, 0), seen((size_t)m.ghost + 1, 0);
  for (i32 p = 0; p < P; p++)
    for (i64 k = w.send_off[(size_t)p]; k < w.send_off[(size_t)p + 1]; k++) {
      const i64 v = send_lids[k];
      CHROMA_REQUIRE(v >= 0 && v < m.owned, CHROMA_EPROTOCOL, "send list names a vertex this rank does not own");
      sl[(size_t)k] = (i32)(m.lid_off + v);
      sp[(size_t)k] = p;
      routed[(size_t)v] = 1;
    }
  for (i64 k = 0; k < w.nrecv; k++) {
    const i64 v = recv_lids[k];
    CHROMA_REQUIRE(v >= m.owned && v < m.owned + m.ghost && !seen[(size_t)(v - m.owned)], CHROMA_EPROTOCOL,
                   "receive list must cover each ghost slot once");
    seen[(size_t)(v - m.owned)] = 1;
    rl[(size_t)k] = (i32)(m.lid_off + v);
  }
  std::vector<i32> rt;
  for (i64 v = 0; v < m.owned; v++)
    if (routed[(size_t)v]) rt.push_back((i32)(m.lid_off + v));
  w.nrouted_remote = (i64)rt.size();
  w.routed_remote.upload(rt.data(), std::max<i64>(w.nrouted_remote, 1), s);
  w.last_sent_remote.alloc(std::max<i64>(w.nrouted_remote, 1), s);
  w.send_lids.upload(sl.data(), std::max<i64>(w.nsend, 1), s);
  w.send_peer.upload(sp.data(), std::max<i64>(w.nsend, 1), s);
  w.recv_lids.upload(rl.data(), std::max<i64>(w.nrecv, 1), s);
  w.sendbuf.alloc(std::max<i64>(w.nsend, 1), s);
  w.recvbuf.alloc(std::max<i64>(w.nrecv, 1), s);
  CUDA_CHECK(cudaMemsetAsync(w.changed.p, 0, w.NL + 1, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  w.comm = (ncclComm_t)comm;
  w.my_rank = rank;
  w.connected = true;
  world_reset_exchange(w);
  CUDA_CHECK(cudaStreamSynchronize(s));
  halo_release_p2p(w);
  halo_setup_p2p(w, sl, sp, rl);
}
#endif

}  // namespace chroma
