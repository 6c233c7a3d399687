// Incremental Jacobi sweeps (distance 1): the same proposals and losers as the
// reference's speculative loop (chroma/localcolor.py:214-227), without re-reading the
// rows of the long pending vertices every sweep.
//
// After sweep 0 every pending vertex is a loser reset to colour 0, and a vertex that
// leaves the pending set never changes again.  So for a pending v the forbidden set
// of a sweep is exactly the colours of its non-pending neighbours, a set that only
// grows, and an equal-coloured neighbour of v's proposal can only be another pending
// vertex (proposals avoid every other neighbour's colour).  For each pending vertex
// with a long row ("heavy", > JI_HEAVY entries; a warp each, a CTA each beyond
// JI_HUB entries) this file keeps
//   fb[slot]   the colours (1..1024) of its non-pending neighbours, and
//   list[slot] its pending neighbours,
// built once from the row and then updated from the list alone: after each sweep the
// neighbours that settled move their colour into fb and leave the list.  Proposals
// of heavy vertices are mex(fb); their loser test scans the list.  Light pending
// vertices keep the full-row kernels.  On R-MAT the pending set is dominated by hubs
// for hundreds of sweeps, whose rows were re-read every sweep before.
// A colour beyond 1024 (fb cannot hold it) switches the caller back to full sweeps
// before the next proposal; the state between sweeps is the reference's either way.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int JW = 32;          // fb words: colours 1..1024
constexpr int WIN = 256;        // colour window of the full-row proposal
constexpr i64 JI_HEAVY = 64;    // rows longer than this keep fb + list
constexpr i64 JI_HUB = 4096;    // ... handled by a whole CTA beyond this
constexpr int JI_CTA = 1024;

__global__ void k_i32_to_i64(const i32* a, i64 n, i64* b) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) b[i] = a[i];
}

// A cooperating group: a warp (G = 32) or a CTA (G = JI_CTA), one slot at a time.
template <int G>
struct Grp {
  __device__ static int tid() { return threadIdx.x & 31; }
  __device__ static i64 first() { return (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; }
  __device__ static i64 stride() { return ((i64)gridDim.x * blockDim.x) >> 5; }
  __device__ static void sync() { __syncwarp(); }
  __device__ static bool any(bool p) { return __any_sync(FULLM, p); }
  __device__ static int sum(int x, int*) { return __reduce_add_sync(FULLM, x); }
  // exclusive prefix of keep in the group; *total = group count
  __device__ static int prefix(bool keep, int* total, int*) {
    const unsigned b = __ballot_sync(FULLM, keep);
    *total = __popc(b);
    return __popc(b & ((1u << (threadIdx.x & 31)) - 1u));
  }
};
template <>
struct Grp<JI_CTA> {
  __device__ static int tid() { return threadIdx.x; }
  __device__ static i64 first() { return blockIdx.x; }
  __device__ static i64 stride() { return gridDim.x; }
  __device__ static void sync() { __syncthreads(); }
  __device__ static bool any(bool p) { return __syncthreads_or(p); }
  __device__ static int sum(int x, int* sm) {  // sm: 33 ints
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    x = __reduce_add_sync(FULLM, x);
    if (lane == 0) sm[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int y = __reduce_add_sync(FULLM, sm[lane]);
      if (lane == 0) sm[32] = y;
    }
    __syncthreads();
    const int r = sm[32];
    __syncthreads();
    return r;
  }
  __device__ static int prefix(bool keep, int* total, int* sm) {  // sm: 33 ints
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned b = __ballot_sync(FULLM, keep);
    if (lane == 0) sm[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {
      const int c = sm[lane];
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULLM, inc, o);
        if (lane >= o) inc += t;
      }
      sm[lane] = inc - c;
      if (lane == 31) sm[32] = inc;
    }
    __syncthreads();
    const int r = sm[wid] + __popc(b & ((1u << lane) - 1u));
    *total = sm[32];
    __syncthreads();
    return r;
  }
};

__device__ __forceinline__ void fb_set(u32* fb, i32 c, unsigned* ovf) {
  if (c <= 0) return;
  if (c > JW * 32) {
    atomicOr(ovf, 1u);
    return;
  }
  atomicOr(fb + ((c - 1) >> 5), 1u << ((c - 1) & 31));
}

// pending flags, heavy slots (class 0: warp, class 1: CTA) into act[c] (parity 0)
__global__ void k_ji_mark(const i64* rowptr, const i32* pend, i64 np, uint8_t* pendf, i32* hslot, i32* hv,
                          unsigned long long* cnt, i32* act0, i32* act1) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < np; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = pend[i];
    pendf[v] = 1;
    const i64 d = rowptr[v + 1] - rowptr[v];
    if (d > JI_HEAVY) {
      const i32 slot = (i32)atomicAdd(cnt, 1ull);
      hv[slot] = v;
      hslot[v] = slot;
      if (d > JI_HUB) act1[atomicAdd(cnt + 4, 1ull)] = slot;
      else act0[atomicAdd(cnt + 2, 1ull)] = slot;
    }
  }
}

// per slot: fb from the non-pending neighbours (group bitmap in shared memory), count
// of pending ones
template <int G>
__global__ void __launch_bounds__(G == JI_CTA ? JI_CTA : 256)
    k_ji_count(const i64* rowptr, const i32* col, const i32* colors, const uint8_t* pendf, const i32* hv,
               const i32* act, const unsigned long long* nact, u32* fb, i32* llen, unsigned* ovf) {
  using Gp = Grp<G>;
  __shared__ u32 sfb_all[G == JI_CTA ? JW : 8 * JW];
  __shared__ int sm[33];
  u32* sfb = sfb_all + (G == JI_CTA ? 0 : (threadIdx.x >> 5) * JW);
  const int t = Gp::tid();
  const i64 n = (i64)*nact;
  for (i64 k = Gp::first(); k < n; k += Gp::stride()) {
    const i32 h = act[k];
    const i32 v = hv[h];
    if (t < JW) sfb[t] = 0;
    Gp::sync();
    int c = 0;
    for (i64 e = rowptr[v] + t; e < rowptr[v + 1]; e += G) {
      const i32 u = col[e];
      if (pendf[u]) c++;
      else fb_set(sfb, colors[u], ovf);
    }
    c = Gp::sum(c, sm);
    Gp::sync();
    if (t < JW) fb[(i64)h * JW + t] = sfb[t];
    if (t == 0) llen[h] = c;
    bool full = true;
    for (int w = 0; w < JW; w++) full &= sfb[w] == FULLM;
    if (full && t == 0) atomicOr(ovf, 1u);
    Gp::sync();
  }
}

// per slot: its pending neighbours into list[loff[h] ...]
template <int G>
__global__ void __launch_bounds__(G == JI_CTA ? JI_CTA : 256)
    k_ji_fill(const i64* rowptr, const i32* col, const uint8_t* pendf, const i32* hv, const i32* act,
              const unsigned long long* nact, const i64* loff, i32* nb) {
  using Gp = Grp<G>;
  __shared__ int sm[33];
  const int t = Gp::tid();
  const i64 n = (i64)*nact;
  for (i64 k = Gp::first(); k < n; k += Gp::stride()) {
    const i32 h = act[k];
    const i32 v = hv[h];
    i64 at = loff[h];
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    for (i64 e0 = rs; e0 < re; e0 += G) {
      const i64 e = e0 + t;
      const i32 u = e < re ? col[e] : -1;
      const bool keep = u >= 0 && pendf[u];
      int tot = 0;
      const int pos = Gp::prefix(keep, &tot, sm);
      if (keep) nb[at + pos] = u;
      at += tot;
    }
  }
}

// heavy proposals: mex of fb (thread per active slot)
__global__ void k_ji_mex(const i32* act, const unsigned long long* nact, const u32* fb, i32* hprop) {
  const i64 n = (i64)*nact;
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) {
    const i32 h = act[k];
    const u32* f = fb + (i64)h * JW;
    i32 t = 0;
    for (int w = 0; w < JW && !t; w++) {
      const u32 x = f[w];
      if (x != FULLM) t = w * 32 + __ffs(~x);
    }
    hprop[h] = t;  // 0 cannot happen: a full fb switched the caller to full sweeps
  }
}

// light proposals (warp per pending vertex, full row); heavy ones copy their mex
__global__ void k_ji_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pend,
                             const i64* np_dev, const i32* hslot, const i32* hprop, i32* prop) {
  const int lane = threadIdx.x & 31;
  const i64 np = *np_dev;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < np; i += nwarps) {
    const i32 v = pend[i];
    const i32 h = hslot[v];
    if (h >= 0) {
      if (lane == 0) prop[i] = hprop[h];
      continue;
    }
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    for (i32 base = 1;; base += WIN) {
      u32 m[WIN / 32];
#pragma unroll
      for (int w = 0; w < WIN / 32; w++) m[w] = 0;
      for (i64 e = rs + lane; e < re; e += 32) {
        const i32 o = colors[col[e]] - base;
        if (o >= 0 && o < WIN) m[o >> 5] |= 1u << (o & 31);
      }
      int r = 0;
#pragma unroll
      for (int w = 0; w < WIN / 32; w++) {
        const u32 mw = __reduce_or_sync(FULLM, m[w]);
        if (!r && mw != FULLM) r = w * 32 + __ffs(~mw);
      }
      if (r) {
        if (lane == 0) prop[i] = base + r - 1;
        break;
      }
    }
  }
}

// heavy losers: an equal-coloured pending neighbour with a larger id
template <int G>
__global__ void __launch_bounds__(G == JI_CTA ? JI_CTA : 256)
    k_ji_hlose(const i32* act, const unsigned long long* nact, const i32* hv, const i64* loff, const i32* llen,
               const i32* nb, const i32* colors, uint8_t* hlose) {
  using Gp = Grp<G>;
  const int t = Gp::tid();
  const i64 n = (i64)*nact;
  for (i64 k = Gp::first(); k < n; k += Gp::stride()) {
    const i32 h = act[k];
    const i32 v = hv[h];
    const i32 c = colors[v];
    const i32* L = nb + loff[h];
    const i32 len = llen[h];
    bool hit = false;
    for (i32 j = t; j < len; j += G) {
      const i32 u = L[j];
      if (u > v && colors[u] == c) hit = true;
    }
    hit = Gp::any(hit);
    if (t == 0) hlose[h] = hit ? 1 : 0;
    Gp::sync();
  }
}

// light losers (full row, the reference rule); heavy ones copy
__global__ void k_ji_losers(const i64* rowptr, const i32* col, const i32* colors, const i32* pend,
                            const i64* np_dev, const uint8_t* in_round, const i32* hslot, const uint8_t* hlose,
                            uint8_t* lose) {
  const int lane = threadIdx.x & 31;
  const i64 np = *np_dev;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < np; i += nwarps) {
    const i32 v = pend[i];
    const i32 h = hslot[v];
    if (h >= 0) {
      if (lane == 0) lose[i] = hlose[h];
      continue;
    }
    const i32 c = colors[v];
    bool hit = false;
    for (i64 e = rowptr[v] + lane; e < rowptr[v + 1]; e += 32) {
      const i32 x = col[e];
      if (colors[x] == c && (x > v || !in_round[x])) hit = true;
    }
    hit = __any_sync(FULLM, hit);
    if (lane == 0) lose[i] = hit ? 1 : 0;
  }
}

// the settled leave the pending set
__global__ void k_ji_settle(const i32* pend, const i64* np_dev, const uint8_t* lose, uint8_t* pendf) {
  const i64 np = *np_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < np; i += (i64)gridDim.x * blockDim.x)
    if (!lose[i]) pendf[pend[i]] = 0;
}

// heavy losers stay: neighbours that settled move their colour into fb and leave the
// list (compacted in place, order kept); fb full or a colour > 1024 -> *ovf
template <int G>
__global__ void __launch_bounds__(G == JI_CTA ? JI_CTA : 256)
    k_ji_update(const i32* act, const unsigned long long* nact, const i32* hv, const i64* loff, i32* llen, i32* nb,
                const i32* colors, const uint8_t* pendf, const uint8_t* hlose, u32* fb, i32* act_next,
                unsigned long long* nact_next, unsigned* ovf) {
  using Gp = Grp<G>;
  __shared__ u32 sfb_all[G == JI_CTA ? JW : 8 * JW];
  __shared__ int sm[33];
  u32* sfb = sfb_all + (G == JI_CTA ? 0 : (threadIdx.x >> 5) * JW);
  const int t = Gp::tid();
  const i64 n = (i64)*nact;
  for (i64 k = Gp::first(); k < n; k += Gp::stride()) {
    const i32 h = act[k];
    if (!hlose[h]) continue;  // settled: done (uniform over the group)
    i32* L = nb + loff[h];
    u32* f = fb + (i64)h * JW;
    if (t < JW) sfb[t] = f[t];
    Gp::sync();
    const i32 len = llen[h];
    i32 at = 0;
    for (i32 j0 = 0; j0 < len; j0 += G) {
      const i32 j = j0 + t;
      const i32 u = j < len ? L[j] : -1;
      const bool keep = u >= 0 && pendf[u];
      if (u >= 0 && !keep) fb_set(sfb, colors[u], ovf);
      int tot = 0;
      const int pos = Gp::prefix(keep, &tot, sm);  // every read of this step precedes the writes
      if (keep) L[at + pos] = u;
      at += tot;
    }
    Gp::sync();
    if (t < JW) f[t] = sfb[t];
    bool full = true;
    for (int w = 0; w < JW; w++) full &= sfb[w] == FULLM;
    if (t == 0) {
      if (full) atomicOr(ovf, 1u);
      llen[h] = at;
      act_next[atomicAdd(nact_next, 1ull)] = h;
    }
    Gp::sync();
  }
}

int wgrid(i64 n) { return grid_for(std::max<i64>(n, 1) * 32, 256, num_sms() * 16); }
int tgrid(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 8); }
int cgrid(i64 n) { return (int)std::min<i64>(std::max<i64>(n, 1), num_sms() * 2); }

}  // namespace

bool jacobi_inc_init(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, i64 np, i64 nv,
                     JacobiIncScratch& S, cudaStream_t s) {
  S.on = false;
  if (np <= 0) return false;
  S.pendf.reserve(nv, s);
  S.hslot.reserve(nv, s);
  CUDA_CHECK(cudaMemsetAsync(S.pendf.p, 0, (size_t)nv, s));
  CUDA_CHECK(cudaMemsetAsync(S.hslot.p, 0xff, sizeof(i32) * (size_t)nv, s));
  S.hv.reserve(np, s);
  for (auto& a : S.act) a.reserve(np, s);
  S.cnt.reserve(8, s);
  S.cnt.zero(s);
  k_ji_mark<<<tgrid(np), 256, 0, s>>>(rowptr, pend, np, S.pendf.p, S.hslot.p, S.hv.p, S.cnt.p, S.act[0].p,
                                      S.act[2].p);
  count_launch();
  unsigned long long nh = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nh, S.cnt.p, sizeof(nh), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  S.nheavy = (i64)nh;
  S.fb.reserve(std::max<i64>(S.nheavy, 1) * JW, s);
  S.llen.reserve(S.nheavy + 1, s);
  S.loff.reserve(S.nheavy + 1, s);
  S.hprop.reserve(std::max<i64>(S.nheavy, 1), s);
  S.hlose.reserve(std::max<i64>(S.nheavy, 1), s);
  unsigned* ovf = reinterpret_cast<unsigned*>(S.cnt.p + 1);
  S.par = 0;
  if (S.nheavy > 0) {
    k_ji_count<32><<<wgrid(S.nheavy), 256, 0, s>>>(rowptr, col, colors, S.pendf.p, S.hv.p, S.act[0].p, S.cnt.p + 2,
                                                   S.fb.p, S.llen.p, ovf);
    k_ji_count<JI_CTA><<<cgrid(S.nheavy), JI_CTA, 0, s>>>(rowptr, col, colors, S.pendf.p, S.hv.p, S.act[2].p,
                                                          S.cnt.p + 4, S.fb.p, S.llen.p, ovf);
    count_launch(2);
    CUDA_CHECK(cudaMemsetAsync(S.llen.p + S.nheavy, 0, sizeof(i32), s));
    // list offsets (int64 scan of the int32 lengths)
    S.len64.reserve(S.nheavy + 1, s);
    k_i32_to_i64<<<tgrid(S.nheavy + 1), 256, 0, s>>>(S.llen.p, S.nheavy + 1, S.len64.p);
    count_launch();
    exclusive_scan_i64(S.len64.p, S.loff.p, S.nheavy + 1, s);
    i64 tot = 0;
    CUDA_CHECK(cudaMemcpyAsync(&tot, S.loff.p + S.nheavy, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    S.nb.reserve(std::max<i64>(tot, 1), s);
    k_ji_fill<32><<<wgrid(S.nheavy), 256, 0, s>>>(rowptr, col, S.pendf.p, S.hv.p, S.act[0].p, S.cnt.p + 2, S.loff.p,
                                                  S.nb.p);
    k_ji_fill<JI_CTA><<<cgrid(S.nheavy), JI_CTA, 0, s>>>(rowptr, col, S.pendf.p, S.hv.p, S.act[2].p, S.cnt.p + 4,
                                                         S.loff.p, S.nb.p);
    count_launch(2);
  }
  unsigned ov = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ov, ovf, sizeof(ov), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  S.on = ov == 0;
  return S.on;
}

void jacobi_inc_propose(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, const i64* np_dev,
                        i64 np, i32* prop, JacobiIncScratch& S, cudaStream_t s) {
  if (S.nheavy > 0) {
    for (int c = 0; c < 2; c++)
      k_ji_mex<<<tgrid(S.nheavy), 256, 0, s>>>(S.act[2 * c + S.par].p, S.cnt.p + 2 + 2 * c + S.par, S.fb.p,
                                               S.hprop.p);
    count_launch(2);
  }
  k_ji_propose<<<wgrid(np), 256, 0, s>>>(rowptr, col, colors, pend, np_dev, S.hslot.p, S.hprop.p, prop);
  count_launch();
}

void jacobi_inc_losers(const i64* rowptr, const i32* col, const i32* colors, const i32* pend, const i64* np_dev,
                       i64 np, const uint8_t* in_round, uint8_t* lose, JacobiIncScratch& S, cudaStream_t s) {
  if (S.nheavy > 0) {
    k_ji_hlose<32><<<wgrid(S.nheavy), 256, 0, s>>>(S.act[S.par].p, S.cnt.p + 2 + S.par, S.hv.p, S.loff.p, S.llen.p,
                                                   S.nb.p, colors, S.hlose.p);
    k_ji_hlose<JI_CTA><<<cgrid(S.nheavy), JI_CTA, 0, s>>>(S.act[2 + S.par].p, S.cnt.p + 4 + S.par, S.hv.p,
                                                          S.loff.p, S.llen.p, S.nb.p, colors, S.hlose.p);
    count_launch(2);
  }
  k_ji_losers<<<wgrid(np), 256, 0, s>>>(rowptr, col, colors, pend, np_dev, in_round, S.hslot.p, S.hlose.p, lose);
  count_launch();
}

// after the losers are known (before they are reset); the caller reads the overflow
// flag (jacobi_inc_overflow_dev) with its pending count
void jacobi_inc_update(const i32* colors, const i32* pend, const i64* np_dev, i64 np, const uint8_t* lose,
                       JacobiIncScratch& S, cudaStream_t s) {
  k_ji_settle<<<tgrid(np), 256, 0, s>>>(pend, np_dev, lose, S.pendf.p);
  count_launch();
  if (S.nheavy > 0) {
    const int p = S.par, q = p ^ 1;
    CUDA_CHECK(cudaMemsetAsync(S.cnt.p + 2 + q, 0, sizeof(unsigned long long), s));
    CUDA_CHECK(cudaMemsetAsync(S.cnt.p + 4 + q, 0, sizeof(unsigned long long), s));
    unsigned* ovf = reinterpret_cast<unsigned*>(S.cnt.p + 1);
    k_ji_update<32><<<wgrid(S.nheavy), 256, 0, s>>>(S.act[p].p, S.cnt.p + 2 + p, S.hv.p, S.loff.p, S.llen.p, S.nb.p,
                                                    colors, S.pendf.p, S.hlose.p, S.fb.p, S.act[q].p, S.cnt.p + 2 + q,
                                                    ovf);
    k_ji_update<JI_CTA><<<cgrid(S.nheavy), JI_CTA, 0, s>>>(S.act[2 + p].p, S.cnt.p + 4 + p, S.hv.p, S.loff.p,
                                                           S.llen.p, S.nb.p, colors, S.pendf.p, S.hlose.p, S.fb.p,
                                                           S.act[2 + q].p, S.cnt.p + 4 + q, ovf);
    count_launch(2);
    S.par = q;
  }
}

const unsigned* jacobi_inc_overflow_dev(const JacobiIncScratch& S) {
  return reinterpret_cast<const unsigned*>(S.cnt.p + 1);
}

}  // namespace chroma
