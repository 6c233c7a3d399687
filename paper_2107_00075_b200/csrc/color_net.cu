// Net-centric free-running colouring for distance 2 and partial distance 2.
//
// Reference semantics: chroma/localcolor.py:136-158 (_forbidden_d2 over
// two_hop_neighbors: the colours of N(v) ∪ N²(v) for D2, of N²(v) for PD2) and the
// net-based loser rule of _d2_losers (230-271): inside one net -- a middle vertex u
// and its adjacency (plus u itself for full D2) -- equal colours clash and the largest
// id keeps its colour.
//
// The vertex-centric walk re-reads every middle's row once per member (~1,040 two-hop
// visits per vertex on C5).  Here every middle u keeps a 256-colour mask of its net
// (4 x u64, one 32-byte sector), so a vertex's forbidden set is the OR of the masks
// of its own row -- |adj(v)| sector loads instead of Σ|adj(u)| colour gathers:
//   masks   every net's mask from the current colours (one pass over the CSR);
//   pick    each pending vertex ORs its nets' masks, takes the first free colour and
//           ORs it into those masks at once (later vertices of the same pass see it);
//   detect  per net, the largest pending id of each colour keeps it; the other
//           pending members of that colour are uncoloured and form the next worklist.
// Later iterations (few vertices) rebuild only the nets around the pending vertices.
// Colours above 256 fall back to the vertex-centric kernels (color_free.cu).
#include <cooperative_groups.h>
#include <cstdlib>

#include "kernels.cuh"

namespace chroma {
namespace cg = cooperative_groups;
namespace {

constexpr int NW = 4;                  // u64 words per net mask: colours 1..256
constexpr int NCOL = NW * 64;
constexpr unsigned FULLM = 0xffffffffu;
constexpr int GL = 8;                  // lanes per vertex in the pick pass

struct NetArgs {
  const i64* rowptr;
  const i32* col;
  i32* colors;
  unsigned long long* mask;   // [nv][NW]
  uint8_t* pend;              // pending this iteration
  const i32* wl;
  i64 nwl;
  bool full;                  // D2: the middle's own colour is in its net
  i32* next;                  // losers
  unsigned long long* nnext;
  unsigned* ovf;              // a colour above NCOL was needed
};

// words selected by compare, not by index: a dynamic index would put m[] in local memory
__device__ __forceinline__ unsigned long long word_at(const unsigned long long (&m)[NW], int k) {
  return k == 0 ? m[0] : k == 1 ? m[1] : k == 2 ? m[2] : m[3];
}

__device__ __forceinline__ void set_bit(unsigned long long (&m)[NW], i32 c) {
  const bool in = c >= 1 && c <= NCOL;
  const int w = (c - 1) >> 6;
  const unsigned long long b = in ? 1ull << ((c - 1) & 63) : 0ull;
#pragma unroll
  for (int k = 0; k < NW; k++) m[k] |= w == k ? b : 0ull;
}

// mask of net u from current colours, by one warp (rows are short; long rows loop)
__device__ __forceinline__ void build_mask(const NetArgs& a, i32 u, int lane) {
  unsigned long long m[NW] = {0, 0, 0, 0};
  const i64 rs = a.rowptr[u], re = a.rowptr[u + 1];
  for (i64 j = rs + lane; j < re; j += 32) set_bit(m, a.colors[a.col[j]]);
  if (a.full && lane == 0) set_bit(m, a.colors[u]);
#pragma unroll
  for (int w = 0; w < NW; w++) {
    const u32 lo = __reduce_or_sync(FULLM, (u32)m[w]), hi = __reduce_or_sync(FULLM, (u32)(m[w] >> 32));
    m[w] = ((unsigned long long)hi << 32) | lo;
  }
  if (lane < NW) a.mask[(i64)u * NW + lane] = word_at(m, lane);
}

// all nets, GL lanes per net (four nets per warp; rows of ~32 entries take four
// column loads per lane and three shuffle rounds)
__global__ void k_masks_all(NetArgs a, i64 nv) {
  const int lane = threadIdx.x & 31, sub = lane % GL;
  const i64 gi = (blockIdx.x * (i64)blockDim.x + threadIdx.x) / GL, ng = ((i64)gridDim.x * blockDim.x) / GL;
  for (i64 base = 0; base < nv; base += ng) {  // uniform trip count per warp
    const i64 u = base + gi;
    unsigned long long m[NW] = {0, 0, 0, 0};
    if (u < nv) {
      const i64 rs = a.rowptr[u], re = a.rowptr[u + 1];
      // four columns, then their four colours, in flight per lane
      for (i64 j = rs + sub; j < re; j += 4 * GL) {
        i32 us[4], cs[4];
#pragma unroll
        for (int q = 0; q < 4; q++) us[q] = j + q * GL < re ? __ldcs(a.col + j + q * GL) : -1;
#pragma unroll
        for (int q = 0; q < 4; q++) cs[q] = us[q] >= 0 ? a.colors[us[q]] : 0;
#pragma unroll
        for (int q = 0; q < 4; q++) set_bit(m, cs[q]);
      }
      if (a.full && sub == 0) set_bit(m, a.colors[u]);
    }
#pragma unroll
    for (int w = 0; w < NW; w++)
#pragma unroll
      for (int o = GL / 2; o >= 1; o >>= 1) m[w] |= __shfl_xor_sync(FULLM, m[w], o);
    if (u < nv && sub < NW) a.mask[u * NW + sub] = word_at(m, sub);
  }
}

// nets adjacent to the pending vertices (warp per pending vertex, its row's nets)
__global__ void k_masks_around(NetArgs a) {
  const int lane = threadIdx.x & 31;
  const i64 w0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = w0; i < a.nwl; i += nw) {
    const i32 v = a.wl[i];
    const i64 rs = a.rowptr[v], re = a.rowptr[v + 1];
    for (i64 j = rs; j < re; j++) build_mask(a, a.col[j], lane);
    if (a.full) build_mask(a, v, lane);
  }
}

// one pending vertex of a pick pass, as seen by one of its GL lanes: the parts that do
// not depend on colours (worklist entry, row bounds, the lane's first four nets), so
// the wave kernel can load the next wave's before the barrier
struct PickItem {
  i32 v;  // -1: no vertex for this group
  i64 rs, re;
  i32 us[4];
};

__device__ __forceinline__ void pick_load(const NetArgs& a, i64 i, i64 hi, int sub, PickItem& p) {
  p.v = -1;
  p.rs = p.re = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) p.us[q] = -1;
  if (i >= hi) return;
  p.v = a.wl[i];
  p.rs = a.rowptr[p.v];
  p.re = a.rowptr[p.v + 1];
#pragma unroll
  for (int q = 0; q < 4; q++) p.us[q] = p.rs + sub + q * GL < p.re ? a.col[p.rs + sub + q * GL] : -1;
}

// OR the vertex's nets' masks, take the first free colour, publish it into those nets;
// called by every lane of the warp (the shuffles use all lanes)
__device__ __forceinline__ void pick_finish(const NetArgs& a, const PickItem& p, int sub) {
  const bool act = p.v >= 0;
  unsigned long long m[NW] = {0, 0, 0, 0};
  if (act) {
    ulonglong4 qs[4];
#pragma unroll
    for (int q = 0; q < 4; q++)
      qs[q] = p.us[q] >= 0 ? *reinterpret_cast<const ulonglong4*>(a.mask + (i64)p.us[q] * NW) : make_ulonglong4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      m[0] |= qs[q].x;
      m[1] |= qs[q].y;
      m[2] |= qs[q].z;
      m[3] |= qs[q].w;
    }
    for (i64 j = p.rs + sub + 4 * GL; j < p.re; j += GL) {
      const i32 u = a.col[j];
      const ulonglong4 q = *reinterpret_cast<const ulonglong4*>(a.mask + (i64)u * NW);
      m[0] |= q.x;
      m[1] |= q.y;
      m[2] |= q.z;
      m[3] |= q.w;
    }
  }
#pragma unroll
  for (int w = 0; w < NW; w++)
#pragma unroll
    for (int o = GL / 2; o >= 1; o >>= 1) m[w] |= __shfl_xor_sync(FULLM, m[w], o);
  if (!act) return;
  i32 c = 0;
#pragma unroll
  for (int w = NW - 1; w >= 0; w--)
    if (~m[w]) c = w * 64 + __ffsll((long long)~m[w]);
  if (c == 0) {
    if (sub == 0) atomicOr(a.ovf, 1u);
    c = NCOL + 1;
  } else {
    // publish into the vertex's nets so later picks of this pass avoid it
    const unsigned long long bit = 1ull << ((c - 1) & 63);
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (p.us[q] >= 0) atomicOr(a.mask + (i64)p.us[q] * NW + ((c - 1) >> 6), bit);
    for (i64 j = p.rs + sub + 4 * GL; j < p.re; j += GL) atomicOr(a.mask + (i64)a.col[j] * NW + ((c - 1) >> 6), bit);
    if (a.full && sub == 0) atomicOr(a.mask + (i64)p.v * NW + ((c - 1) >> 6), bit);
  }
  if (sub == 0) a.colors[p.v] = c;
}

// pick for worklist positions [lo, hi): GL lanes per pending vertex
__global__ void k_pick(NetArgs a) {
  const int sub = (threadIdx.x & 31) % GL;
  const i64 gi = (blockIdx.x * (i64)blockDim.x + threadIdx.x) / GL, ng = ((i64)gridDim.x * blockDim.x) / GL;
  for (i64 base = 0; base < a.nwl; base += ng) {  // uniform trip count per warp
    PickItem p;
    pick_load(a, base + gi, a.nwl, sub, p);
    pick_finish(a, p, sub);
  }
}

// the first pass's waves in one cooperative launch, a grid barrier between waves (a
// wave's picks and mask updates are visible to the next one); each group's first item
// of the next wave is loaded before the barrier, so a wave's critical path starts at
// its mask loads
__global__ void k_pick_waves(NetArgs a, int waves) {
  cg::grid_group grid = cg::this_grid();
  const int sub = (threadIdx.x & 31) % GL;
  const i64 gi = (blockIdx.x * (i64)blockDim.x + threadIdx.x) / GL, ng = ((i64)gridDim.x * blockDim.x) / GL;
  PickItem p;
  pick_load(a, gi, a.nwl / waves, sub, p);
  for (int w = 0; w < waves; w++) {
    const i64 lo = a.nwl * w / waves, hi = a.nwl * (w + 1) / waves;
    pick_finish(a, p, sub);
    for (i64 base = lo + ng; base < hi; base += ng) {
      PickItem q;
      pick_load(a, base + gi, hi, sub, q);
      pick_finish(a, q, sub);
    }
    if (w + 1 < waves) pick_load(a, hi + gi, a.nwl * (w + 2) / waves, sub, p);
    grid.sync();
  }
}

__device__ __forceinline__ void lose(const NetArgs& a, i32 x) {
  if (atomicExch(a.colors + x, 0) != 0) {
    const unsigned long long k = atomicAdd(a.nnext, 1ull);
    a.next[k] = x;
  }
}

// detect on one net u by one warp: the largest pending id per colour survives
__device__ __forceinline__ void detect_net(const NetArgs& a, i32 u, int lane, i32* mx) {
  const i64 rs0 = a.rowptr[u], re0 = a.rowptr[u + 1];
  const i64 members = re0 - rs0 + (a.full ? 1 : 0);
  // mx[] holds -1 everywhere between nets (set at kernel start, restored after use)
  if (members <= 32) {  // one member per lane: the largest pending id per colour in mx[]
    i32 x = -1, key = 0;
    if (lane < members) {
      x = lane < re0 - rs0 ? a.col[rs0 + lane] : u;
      const uint8_t pd = a.pend[x];  // both gathers in flight together
      const i32 c = a.colors[x];
      if (pd && c >= 1 && c <= NCOL + 1) key = c;
    }
    if (key) atomicMax(mx + key, x);
    __syncwarp();
    const bool l = key && mx[key] > x;
    __syncwarp();
    if (key) mx[key] = -1;
    __syncwarp();
    if (l) lose(a, x);
    return;
  }
  if (members <= 64) {  // two members per lane, kept in registers for the loser test
    i32 xs[2], ks[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const i64 idx = lane + 32 * h;
      xs[h] = -1;
      ks[h] = 0;
      if (idx < members) {
        xs[h] = idx < re0 - rs0 ? a.col[rs0 + idx] : u;
        const uint8_t pd = a.pend[xs[h]];
        const i32 c = a.colors[xs[h]];
        if (pd && c >= 1 && c <= NCOL + 1) ks[h] = c;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (ks[h]) atomicMax(mx + ks[h], xs[h]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (ks[h] && mx[ks[h]] > xs[h]) lose(a, xs[h]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (ks[h]) mx[ks[h]] = -1;
    __syncwarp();
    return;
  }
  const i64 rs = a.rowptr[u], re = a.rowptr[u + 1];
  const i64 ext = a.full ? 1 : 0;  // the middle itself is a member of a D2 net
  for (i64 j = rs + lane; j < re + ext; j += 32) {
    const i32 x = j < re ? a.col[j] : u;
    if (!a.pend[x]) continue;
    const i32 c = a.colors[x];
    if (c >= 1 && c <= NCOL + 1) atomicMax(mx + c, x);
  }
  __syncwarp();
  // a settled member of the same colour cannot exist (the masks held it), so only
  // pending members clash
  for (i64 j = rs + lane; j < re + ext; j += 32) {
    const i32 x = j < re ? a.col[j] : u;
    if (!a.pend[x]) continue;
    const i32 c = a.colors[x];
    if (c >= 1 && c <= NCOL + 1 && mx[c] > x && a.colors[x] != 0) lose(a, x);
  }
  __syncwarp();
  for (int k = lane; k < NCOL + 2; k += 32) mx[k] = -1;
  __syncwarp();
}

__global__ void k_detect_all(NetArgs a, i64 nv) {
  __shared__ i32 mxs[8][NCOL + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = lane; k < NCOL + 2; k += 32) mxs[wid][k] = -1;
  __syncwarp();
  const i64 w0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 u = w0; u < nv; u += nw) detect_net(a, (i32)u, lane, mxs[wid]);
}

__global__ void k_detect_around(NetArgs a) {
  __shared__ i32 mxs[8][NCOL + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = lane; k < NCOL + 2; k += 32) mxs[wid][k] = -1;
  __syncwarp();
  const i64 w0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5, nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = w0; i < a.nwl; i += nw) {
    const i32 v = a.wl[i];
    const i64 rs = a.rowptr[v], re = a.rowptr[v + 1];
    for (i64 j = rs; j < re; j++) detect_net(a, a.col[j], lane, mxs[wid]);
    if (a.full) detect_net(a, v, lane, mxs[wid]);
  }
}

__global__ void k_zero_list(const i32* wl, i64 n, i32* colors) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) colors[wl[i]] = 0;
}

__global__ void k_max_deg(const i32* wl, i64 n, const i64* rowptr, unsigned long long* out) {
  unsigned long long m = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    const unsigned long long d = (unsigned long long)(rowptr[v + 1] - rowptr[v]);
    m = d > m ? d : m;
  }
  m = __reduce_max_sync(FULLM, (unsigned)m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_set_pend(const i32* wl, i64 n, uint8_t* pend, uint8_t val) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) pend[wl[i]] = val;
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

i64 net_waves() {
  static const i64 w = [] {
    const char* e = std::getenv("CHROMA_NET_WAVES");
    return e ? std::max<i64>(1, std::atoll(e)) : 1024;
  }();
  return w;
}

}  // namespace

// Colours the worklist (colours of its vertices must be 0; every other vertex keeps
// its colour).  Returns false if a colour above 256 was needed (worklist back at 0).
bool launch_free_net(const i64* rowptr, const i32* col, i64 nv, i32* colors, const i32* wl_in, i64 nwl,
                     bool partial, NetScratch& S, cudaStream_t s) {
  if (nwl <= 0) return true;
  S.mask.reserve(nv * NW, s);
  S.pend.reserve(nv, s);
  CUDA_CHECK(cudaMemsetAsync(S.pend.p, 0, nv, s));
  S.wl[0].reserve(nwl, s);
  S.wl[1].reserve(nwl, s);
  S.cnt.reserve(2, s);
  CUDA_CHECK(cudaMemcpyAsync(S.wl[0].p, wl_in, sizeof(i32) * nwl, cudaMemcpyDeviceToDevice, s));
  NetArgs a;
  a.rowptr = rowptr;
  a.col = col;
  a.colors = colors;
  a.mask = S.mask.p;
  a.pend = S.pend.p;
  a.full = !partial;
  a.ovf = reinterpret_cast<unsigned*>(S.cnt.p + 1);
  CUDA_CHECK(cudaMemsetAsync(S.cnt.p + 1, 0, sizeof(unsigned long long), s));
  const i64 small = std::max<i64>(nv / 32, 4096);
  int p = 0;
  i64 n = nwl;
  for (int it = 0; n > 0; it++) {
    CHROMA_REQUIRE(it < 10000, CHROMA_ERUNTIME, "speculative loop failed to settle");
    a.wl = S.wl[p].p;
    a.nwl = n;
    a.next = S.wl[p ^ 1].p;
    a.nnext = S.cnt.p;
    CUDA_CHECK(cudaMemsetAsync(S.cnt.p, 0, sizeof(unsigned long long), s));
    k_set_pend<<<G(n), 256, 0, s>>>(a.wl, n, a.pend, 1);
    const bool all = n > small;
    if (all) k_masks_all<<<num_sms() * 16, 256, 0, s>>>(a, nv);
    else k_masks_around<<<G(n * 32), 256, 0, s>>>(a);
    // the first pass picks in waves of ascending worklist position: each wave sees the
    // colours of the earlier ones in the masks, so fewer equal picks collide (the
    // colour count stays near sequential first fit's)
    const int waves = it == 0 ? (int)std::min<i64>(net_waves(), std::max<i64>(1, n / 1024)) : 1;
    if (waves > 1) {
      static int blocks[64] = {};  // co-resident blocks per SM, per device
      int dev = 0;
      CUDA_CHECK(cudaGetDevice(&dev));
      int& bps = blocks[dev & 63];
      if (!bps) CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_pick_waves, 256, 0));
      const int grid = std::min<i64>(std::max(1, bps) * num_sms(), std::max<i64>(1, (n / waves + 1) * GL / 256 + 1));
      int wv = waves;
      void* args[] = {&a, &wv};
      CUDA_CHECK(cudaLaunchCooperativeKernel((void*)k_pick_waves, grid, 256, args, 0, s));
    } else {
      k_pick<<<G(n * GL), 256, 0, s>>>(a);
    }
    if (all) k_detect_all<<<num_sms() * 16, 256, 0, s>>>(a, nv);
    else k_detect_around<<<G(n * 32), 256, 0, s>>>(a);
    k_set_pend<<<G(n), 256, 0, s>>>(a.wl, n, a.pend, 0);
    count_launch(6);
    unsigned long long h[2];
    CUDA_CHECK(cudaMemcpyAsync(h, S.cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if ((unsigned)h[1]) {
      k_zero_list<<<G(nwl), 256, 0, s>>>(wl_in, nwl, colors);
      count_launch();
      return false;
    }
    n = (i64)h[0];
    p ^= 1;
  }
  return true;
}

i64 worklist_max_degree(const i32* wl, i64 n, const i64* rowptr, NetScratch& S, cudaStream_t s) {
  if (n <= 0) return 0;
  S.cnt.reserve(2, s);
  CUDA_CHECK(cudaMemsetAsync(S.cnt.p, 0, sizeof(unsigned long long), s));
  k_max_deg<<<std::min(G(n), num_sms() * 4), 256, 0, s>>>(wl, n, rowptr, S.cnt.p);
  count_launch();
  unsigned long long h = 0;
  CUDA_CHECK(cudaMemcpyAsync(&h, S.cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  return (i64)h;
}

}  // namespace chroma
