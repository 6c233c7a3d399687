// Level-synchronous Gauss-Seidel first fit on one thread-block cluster.
//
// The reference colours the worklist in ascending id (chroma/localcolor.py:161-165):
// v's colour depends on its worklist neighbours u < v, so the work is a DAG whose
// longest path (C2 27-point 128^3: 890 levels; a 32-plane slab: 506; C1 grid 1000^2:
// 1999) bounds any exact evaluation.  The dataflow kernel (color_gs_d1.cu) resolves
// each level through global-memory flags -- a producer store, an L2 round trip and a
// poll, about 3 us per level.  Here the levels are walked by ONE cluster of CL CTAs
// (16 SMs, non-portable cluster size) and the colours live in distributed shared
// memory, one byte per vertex, dealt to the CTAs in blocks of B = 1024 ids
// round-robin (block b -> CTA b % CL), so every level's vertices spread evenly over
// the cluster while mesh neighbours x +- 1, x +- L mostly share a block.  A level
// costs a few shared / DSMEM gathers, a store and one barrier.cluster.
//
// The plan (built once per world together with the level schedule, gs_levels.cu):
//   * entries: the schedule without padding, level by level, grouped by owner CTA;
//   * items: each CTA's entries of a level in chunks of at most CAP, with their
//     rows copied out into fixed-width slots (DW >= max degree, -1 padded) and stored
//     transposed per item (slot k of entry t at item_base + k * n + t) so a warp's
//     gathers of one slot are one contiguous read;
//   * per CTA and level: the first item.
// A CTA streams its items through S shared-memory stages with cp.async, S - 1 items
// ahead of the one being coloured (items are static: only the colours are on the
// dependency chain).  Every CTA colours only vertices it owns, so each colour store
// is local; neighbours' colours are local or DSMEM loads.  First fit of a row of at
// most 32 entries is at most 33: a 64-bit mask, colours above 64 never block.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "world.cuh"

namespace cg = cooperative_groups;

namespace chroma {
namespace {

constexpr int S = 3;  // cp.async stages

__global__ void k_flag_valid(const i32* wl, i64 n, uint8_t* f) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    f[i] = wl[i] >= 0;
}

struct Own {
  int logB, logCL;
  __device__ __forceinline__ int owner(i64 x) const { return (int)((x >> logB) & ((1 << logCL) - 1)); }
  __device__ __forceinline__ i64 offset(i64 x) const {
    return ((x >> (logB + logCL)) << logB) | (x & ((1ll << logB) - 1));
  }
  __device__ __forceinline__ i32 loc(i64 x) const { return (i32)(((i64)owner(x) << 24) | offset(x)); }
};

// key of entry j: level << 36 | owner << 32 | id  (sorted: level, owner CTA, id)
__global__ void k_entry_keys(const i32* v, i64 nent, const i64* lstart, i64 L, Own own, u64* keys) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nent; j += (i64)gridDim.x * blockDim.x) {
    i64 lo = 0, hi = L;  // last level with lstart <= j
    while (hi - lo > 1) {
      const i64 mid = (lo + hi) >> 1;
      if (lstart[mid] <= j) lo = mid;
      else hi = mid;
    }
    keys[j] = ((u64)lo << 36) | ((u64)own.owner(v[j]) << 32) | (u32)v[j];
  }
}
__global__ void k_keys_to_ids(const u64* keys, i64 n, i32* v) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x)
    v[j] = (i32)(keys[j] & 0xffffffffu);
}

// bounds[l*(CL+1)+r] = first entry of level l owned by CTA >= r
__global__ void k_bounds(const u64* keys, i64 nent, i64 L, int CL, i64* bounds) {
  const i64 n = L * (CL + 1);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 l = i / (CL + 1);
    const int r = (int)(i % (CL + 1));
    const u64 key = ((u64)l << 36) + ((u64)r << 32);  // r = CL = 16 carries into the level bits
    i64 lo = 0, hi = nent;
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    bounds[i] = lo;
  }
}

// Slots of an entry: the neighbours whose colour can be non-zero when v is coloured
// in the protocol's round 0 -- worklist members below v (coloured in earlier levels)
// and vertices outside the worklist (fixed colours); worklist members above v still
// hold their pre-call colour, 0 on that path.
// zero_nm: every non-member holds colour 0 when the plan runs (the protocol's round
// 0 before any exchange: the non-members are the ghosts), so only lower members count
__device__ __forceinline__ bool keep_slot(i32 u, i32 v, const uint8_t* member, bool zero_nm) {
  return zero_nm ? u < v && member[u] : u < v || !member[u];
}
constexpr i32 LINK = 1 << 30, PREV = 1 << 29, ID_MASK = PREV - 1;  // entry flags (run links)

// level-ordered entries: is entry j's predecessor x - 1 on the same level (a run link)?
__device__ __forceinline__ bool same_level_prev(const i32* v, i64 j, const i64* lstart, i64 L) {
  if (j == 0 || v[j - 1] != v[j] - 1) return false;
  i64 lo = 0, hi = L;  // last level with lstart <= j
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (lstart[mid] <= j) lo = mid;
    else hi = mid;
  }
  return lstart[lo] < j;
}

// widest pruned row; the x - 1 slot of a run link is not a slot (the kernel takes
// that colour from the scan or, at an item start, from its own shared memory)
__global__ void k_slot_count(const i64* rowptr, const i32* col, const i32* v, i64 nent, const uint8_t* member,
                             const i64* lstart, i64 L, bool chains, bool zero_nm, unsigned* maxd) {
  unsigned m = 0;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nent; j += (i64)gridDim.x * blockDim.x) {
    const i32 x = v[j];
    const bool link = chains && same_level_prev(v, j, lstart, L);
    unsigned d = 0;
    for (i64 e = rowptr[x]; e < rowptr[x + 1]; e++) {
      const i32 u = col[e];
      d += keep_slot(u, x, member, zero_nm) && !(link && u == x - 1);
    }
    m = max(m, d);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(maxd, m);
}

__global__ void k_mark(const i32* v, i64 n, uint8_t* member) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) member[v[j]] = 1;
}

// rows of every entry into its item's transposed slots.  Entries are sorted by
// (level, owner, id) (keys); an adjacent x - 1 on the same level is a run link
// (gs_levels.cu): it gets no slot, and the entry id carries LINK (x - 1 is the
// previous entry of this item: the prefix scan supplies its colour) or PREV (x - 1
// ended this CTA's previous item of the level: read from own shared memory).
__global__ void k_fill_slots(const i64* rowptr, const i32* col, const u64* keys, const i32* ent_item,
                             const i32* item_a, const i32* item_n, const i64* item_o, i64 nent, int DW, Own own,
                             const uint8_t* member, i32* blob, bool zero_nm, i32 empty_off) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nent; j += (i64)gridDim.x * blockDim.x) {
    const i32 it = ent_item[j];
    const i64 a = item_a[it], n = (item_n[it] + 3) & ~3;  // n: the padded row length
    const i64 t = j - a;
    i32* hdr = blob + item_o[it];
    i32* nb = hdr + 4 + n;  // slot k of entry t at nb[k * n + t]
    const i32 x = (i32)(keys[j] & 0xffffffffu);
    const bool cand = j > 0 && (keys[j - 1] >> 36) == (keys[j] >> 36) && (i32)(keys[j - 1] & 0xffffffffu) == x - 1;
    bool adj = false;
    int k = 0;
    for (i64 e = rowptr[x]; e < rowptr[x + 1]; e++) {
      const i32 u = col[e];
      if (cand && u == x - 1) {
        adj = true;
        continue;
      }
      if (keep_slot(u, x, member, zero_nm)) nb[(i64)(k++) * n + t] = own.loc(u);
    }
    // empty slots: the zero byte past this CTA's colour slice
    const i32 empty = (i32)((u32)own.owner(x) << 24) | empty_off;
    for (; k < DW; k++) nb[(i64)k * n + t] = empty;
    hdr[4 + t] = x | (adj ? (t > 0 ? LINK : PREV) : 0);
    if (adj && t > 0) hdr[2] = 1;
  }
}

__global__ void k_item_hdr(const i32* item_n, const i32* item_l, const i64* item_o, i64 nitems, i32* blob) {
  for (i64 it = blockIdx.x * (i64)blockDim.x + threadIdx.x; it < nitems; it += (i64)gridDim.x * blockDim.x) {
    i32* h = blob + item_o[it];
    h[0] = item_n[it];
    h[1] = item_l[it];
    h[2] = 0;
    h[3] = (item_n[it] + 3) & ~3;
  }
}

__global__ void k_ent_item(const i32* item_a, const i32* item_n, i64 nitems, i32* ent_item) {
  for (i64 it = blockIdx.x; it < nitems; it += gridDim.x)
    for (i64 t = threadIdx.x; t < item_n[it]; t += blockDim.x) ent_item[item_a[it] + t] = (i32)it;
}

__device__ __forceinline__ u32 shl1(u32 c) {
  u32 r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(c));
  return r;
}

struct ClusterArgs {
  const i32* blob;      // items: [n, level, link, npad | ids x npad | slots DW x npad]
  const i64* item_o;    // per item: offset in blob (ints, multiple of 4)
  const i32* item_sz;   // per item: size (ints, multiple of 4)
  const i32* cta_item;  // [CL][L+1]: first item (global index) of level l for CTA r
  i64 L;
  i64 nv, per;  // per: bytes of colour slice per CTA
  int DW, CAP;
  bool chains;  // the schedule holds runs: entries may carry LINK / PREV
  Own own;
  i32* val;
  const i32* old;
};

template <int DW>
__global__ void __launch_bounds__(1024, 1) k_gs_cluster(ClusterArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int CL = (int)cluster.num_blocks();
  const int t = threadIdx.x;
  const i64 per_pad = (a.per + 15) / 16 * 16;
  unsigned char* col8 = smem;
  const i64 stage_bytes = ((i64)a.CAP * (a.DW + 1) + 4) * 4;  // one item: header, ids, slots
  unsigned char* stages = smem + per_pad + 16;
  const u32 mbar = (u32)__cvta_generic_to_shared(stages + (i64)S * stage_bytes);  // S mbarriers
  u32* tot = reinterpret_cast<u32*>(stages + (i64)S * stage_bytes + 32);         // scan: warp totals
  const u32 base8 = (u32)__cvta_generic_to_shared(col8);
  if (t == 0) {
    col8[per_pad] = 0;  // the byte empty slots read
    for (int q = 0; q < S; q++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar + 8 * q) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- my colour slice: pre-call colours (worklist entries: their old colour)
  const int lB = a.own.logB, lC = a.own.logCL;
  // four ids per thread and step (16-byte loads; a block of 2^lB ids is contiguous)
  auto pre = [&](i64 x) -> u32 {
    if (x >= a.nv) return 0;
    i32 c = a.val[x];
    if (c == PENDING) c = a.old ? a.old[x] : 0;
    return (c < 0 || c > 255) ? 0u : (u32)c;
  };
#pragma unroll 4
  for (i64 u = t; u < a.per / 4; u += blockDim.x) {
    const i64 o = 4 * u;
    const i64 x = ((((o >> lB) << lC) + r) << lB) | (o & ((1ll << lB) - 1));
    u32 w4;
    if (x + 3 < a.nv && !a.old) {
      const int4 c = *reinterpret_cast<const int4*>(a.val + x);
      auto b = [](i32 c) -> u32 { return (c == PENDING || c < 0 || c > 255) ? 0u : (u32)c; };
      w4 = b(c.x) | b(c.y) << 8 | b(c.z) << 16 | b(c.w) << 24;
    } else {
      w4 = pre(x) | pre(x + 1) << 8 | pre(x + 2) << 16 | pre(x + 3) << 24;
    }
    *reinterpret_cast<u32*>(col8 + o) = w4;
  }
  const i32* my_item = a.cta_item + (i64)r * (a.L + 1);
  const i32 k_begin = my_item[0], k_end = my_item[a.L];
  // items stream in by TMA bulk copies (one instruction per item, issued by thread
  // 0, completion on the stage's mbarrier), S - 1 items ahead; thread 0 reads the
  // next descriptor one item ahead of its issue (off the per-level chain)
  auto issue = [&](i32 k, i64 off, i32 sz) {
    if (t == 0 && k < k_end) {
      const int q = (k - k_begin) % S;
      const u32 dst = (u32)__cvta_generic_to_shared(stages + (i64)q * stage_bytes);
      const u32 bytes = (u32)sz * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar + 8 * q), "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(a.blob + off), "r"(bytes), "r"(mbar + 8 * q)
          : "memory");
    }
  };
  __syncthreads();  // barriers initialised
  for (int k = 0; k < S - 1; k++) {
    const i32 kk = k_begin + k;
    if (t == 0 && kk < k_end) issue(kk, a.item_o[kk], a.item_sz[kk]);
  }
  i64 nx_o = 0;
  i32 nx_sz = 0;
  if (t == 0 && k_begin + S - 1 < k_end) {
    nx_o = a.item_o[k_begin + S - 1];
    nx_sz = a.item_sz[k_begin + S - 1];
  }
  cluster.sync();
  // Level barriers, split and item-driven.  Every CTA passes L barriers (one per
  // level), in order; it arrives at level l's barrier once its stores of level l are
  // done and waits only right before its first gathers of a later level, so stage
  // hand-off, slot loads and address arithmetic overlap the barrier.  Items carry
  // their level, so the loop needs no per-level metadata from global memory.  The
  // colours are shared-memory stores of this CTA, completed in this SM's shared
  // memory by a CTA fence before the arrive; remote readers load them from there
  // after the wait.  A cluster-scope release (fence.acq_rel.cluster /
  // arrive.release) compiles to MEMBAR.ALL.GPU, which would also drain the cp.async
  // prefetches in flight -- a DRAM round trip per level -- so the arrive is relaxed.
  bool waiting = false;  // arrived at the last barrier, not yet waited
  i64 cur = 0;           // barriers arrived at
  auto wait_level = [&]() {
    if (waiting) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      waiting = false;
    }
  };
  auto close_levels_below = [&](i64 lv) {
    while (cur < lv) {
      wait_level();
      asm volatile("fence.acq_rel.cta;\n\tbarrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      waiting = true;
      cur++;
    }
  };
  for (i32 k = k_begin; k < k_end; k++) {
    {
      const int q = (k - k_begin) % S;
      const u32 par = (u32)((k - k_begin) / S) & 1u;
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n}" ::"r"(mbar + 8 * q),
          "r"(par)
          : "memory");
    }
    __syncthreads();  // stage k landed; every thread is past item k - 1
    const unsigned char* st = stages + (i64)((k - k_begin) % S) * stage_bytes;
    const i32* sh = reinterpret_cast<const i32*>(st);
    const i32 n = sh[0];
    const i32 lk = sh[1];
    const bool scan = sh[2] != 0;
    const i32 npad = sh[3];
    const i32* sv = sh + 4;
    const i32* snb = sv + npad;
    close_levels_below(lk);  // this CTA's stores of every earlier level are out
    const bool act = t < n;
    i32 v = 0;
    bool linked = false, prev = false;  // run link: x - 1 is the previous entry (LINK, PREV)
    // every slot's byte address in the cluster's shared window (mapa); slots hold
    // owner << 24 | offset, empty ones point at a zero byte of this CTA
    u32 ad[DW];
    if (act) {
      v = sv[t];
      linked = (v & LINK) != 0;
      prev = (v & PREV) != 0;
      v &= ID_MASK;
#pragma unroll
      for (int j = 0; j < DW; j++) {
        const u32 x = (u32)snb[j * npad + t];
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ad[j]) : "r"(base8 + (x & 0xffffffu)), "r"(x >> 24));
      }
    }
    wait_level();  // every level below lk is complete everywhere
    // first fit against the gathered colours: m0, and m1 (next free) for a run link.
    // Entry t's colour is f_t(colour of t - 1) with f_t(c) = c == p ? a : b, packed
    // as p | a << 8 | b << 16; an unlinked entry is the constant map (p = 0, colours
    // are >= 1).  Composition g o f = (f.p, g(f.a), g(f.b)).
    u32 f = 0;
    if (act) {
      int c[DW];
#pragma unroll
      for (int j = 0; j < DW; j++) asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=r"(c[j]) : "r"(ad[j]));
      u32 m0, m1;
      if (DW <= 28) {
        // first fit of <= DW + 1 neighbours (+ x - 1) is <= 31: a 32-bit mask with
        // bit c for colour c (bit 0 preset); PTX shl clamps, colours >= 32 drop out
        u32 m = 1;
#pragma unroll
        for (int j = 0; j < DW; j++) m |= shl1(c[j]);
        if (prev) m |= shl1(col8[a.own.offset(v - 1)]);
        m0 = (u32)__ffs(~m) - 1;
        m1 = (u32)__ffs(~m & ~(1u << m0)) - 1;
      } else {
        u64 m = 0;
#pragma unroll
        for (int j = 0; j < DW; j++)
          if (c[j] >= 1 && c[j] <= 64) m |= 1ull << (c[j] - 1);
        if (prev) {
          const int cp = col8[a.own.offset(v - 1)];
          if (cp >= 1 && cp <= 64) m |= 1ull << (cp - 1);
        }
        m0 = (u32)__ffsll((long long)~m);
        m1 = (u32)__ffsll((long long)(~m & ~(1ull << (m0 - 1))));
      }
      f = m0 << 8 | m0 << 16;
      if (linked) f = m0 | m1 << 8 | m0 << 16;
    }
    auto apply = [](u32 g, u32 c) -> u32 { return c == (g & 0xffu) ? (g >> 8) & 0xffu : g >> 16; };
    if (scan) {
      // runs: inclusive scan of map composition over the item
      const int lane = t & 31, w = t >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 q = __shfl_up_sync(0xffffffffu, f, o);
        if (lane >= o) f = (q & 0xffu) | apply(f, (q >> 8) & 0xffu) << 8 | apply(f, q >> 16) << 16;
      }
      if (((f >> 8) & 0xffu) == (f >> 16)) f &= ~0xffu;  // a == b: constant
      // across warps: entry 0 is unlinked, so the prefix of warps < w is a
      // constant reached from the nearest constant warp total
      if (lane == 31) tot[w] = f;
      __syncthreads();
      if (w > 0 && (f & 0xffu) != 0) {
        int k = w - 1;
        while ((tot[k] & 0xffu) != 0) k--;
        u32 cc = tot[k] >> 16;
        for (k++; k < w; k++) cc = apply(tot[k], cc);
        f = apply(f, cc) << 16;
      }
    }
    const u32 fb = f >> 16;
    if (act) col8[a.own.offset(v)] = (unsigned char)fb;
    if (t == 0) {
      issue(k + S - 1, nx_o, nx_sz);  // into item k - 1's stage (all threads are past it)
      if (k + S < k_end) {
        nx_o = a.item_o[k + S];
        nx_sz = a.item_sz[k + S];
      }
    }
  }
  close_levels_below(a.L);
  wait_level();
  // colours back to global memory once, at the end (no global stores inside the
  // level loop for the cluster barriers to drain): worklist entries still read PENDING
#pragma unroll 4
  for (i64 u = t; u < a.per / 4; u += blockDim.x) {
    const i64 o = 4 * u;
    const i64 x = ((((o >> lB) << lC) + r) << lB) | (o & ((1ll << lB) - 1));
    const u32 w4 = *reinterpret_cast<const u32*>(col8 + o);
    if (x + 3 < a.nv) {
      int4 c = *reinterpret_cast<const int4*>(a.val + x);
      c.x = c.x == PENDING ? (i32)(w4 & 0xffu) : c.x;
      c.y = c.y == PENDING ? (i32)((w4 >> 8) & 0xffu) : c.y;
      c.z = c.z == PENDING ? (i32)((w4 >> 16) & 0xffu) : c.z;
      c.w = c.w == PENDING ? (i32)(w4 >> 24) : c.w;
      *reinterpret_cast<int4*>(a.val + x) = c;
    } else {
      for (int i = 0; i < 4; i++)
        if (x + i < a.nv && a.val[x + i] == PENDING) a.val[x + i] = (i32)((w4 >> (8 * i)) & 0xffu);
    }
  }
}

using ClusterKernel = void (*)(ClusterArgs);
ClusterKernel cluster_kernel(int DW) {
  switch (DW) {
    case 4: return k_gs_cluster<4>;
    case 8: return k_gs_cluster<8>;
    case 12: return k_gs_cluster<12>;
    case 16: return k_gs_cluster<16>;
    case 20: return k_gs_cluster<20>;
    case 24: return k_gs_cluster<24>;
    case 28: return k_gs_cluster<28>;
    default: return k_gs_cluster<32>;
  }
}

}  // namespace

// ---------------------------------------------------------------- plan
// Largest vertex count whose colour bytes fit the cluster's shared memory (16 CTAs).
i64 cluster_max_vertices() {
  int dev = 0, max_smem = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return std::max<i64>(0, (i64)max_smem - 32 * 1024) * 16;
}

bool build_cluster_plan(const i64* rowptr, const i32* col, i64 nv, i64 max_deg, const i32* level_wl,
                        i64 level_n, const std::vector<i64>& level_sizes, ClusterPlan& plan, cudaStream_t s,
                        bool chains, bool zero_nm) {
  plan.ok = false;
  static const bool disabled = std::getenv("CHROMA_NO_CLUSTER") != nullptr;
  if (disabled || max_deg > 32 || nv <= 0 || level_n <= 0 || level_sizes.empty()) return false;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  int max_smem = 0;
  CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // ---- entries: the schedule without its padding (ids ascending within a level)
  DBuf<uint8_t> f;
  f.alloc(level_n, s);
  k_flag_valid<<<grid_for(level_n, 256, num_sms() * 8), 256, 0, s>>>(level_wl, level_n, f.p);
  count_launch();
  plan.v.alloc(level_n, s);
  DBuf<i64> nent_d;
  nent_d.alloc(1, s);
  select_flagged_values(level_wl, f.p, level_n, plan.v.p, nent_d.p, s);
  // worklist membership and the widest pruned row
  DBuf<uint8_t> member;
  member.alloc(nv + 1, s);
  member.zero(s);
  DBuf<unsigned> maxd;
  maxd.alloc(1, s);
  maxd.zero(s);
  // level boundaries in entry space
  std::vector<i64> lstart(1, 0);
  for (i64 sz : level_sizes) lstart.push_back(lstart.back() + sz);
  const i64 nent = lstart.back();
  const i64 L = (i64)lstart.size() - 1;
  if (chains && nv >= PREV) return false;
  DBuf<i64> ls_d;
  ls_d.upload(lstart.data(), L + 1, s);
  {
    i64 ne = 0;
    CUDA_CHECK(cudaMemcpyAsync(&ne, nent_d.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    k_mark<<<grid_for(std::max<i64>(ne, 1), 256, num_sms() * 8), 256, 0, s>>>(plan.v.p, ne, member.p);
    CHROMA_REQUIRE(ne == nent, CHROMA_ERUNTIME, "cluster plan: schedule size mismatch");
    k_slot_count<<<grid_for(std::max<i64>(ne, 1), 256, num_sms() * 8), 256, 0, s>>>(
        rowptr, col, plan.v.p, ne, member.p, ls_d.p, L, chains, zero_nm, maxd.p);
    count_launch(2);
  }
  unsigned hmaxd = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hmaxd, maxd.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  const int DW = (int)std::max<i64>(4, ((i64)hmaxd + 3) / 4 * 4);
  int CL = 0, CAP = 0;
  i64 per = 0;
  const int logB = 10;
  const i64 nblocks = (nv + (1ll << logB) - 1) >> logB;
  for (int cl : {16, 8}) {
    per = (nblocks + cl - 1) / cl << logB;  // colour bytes per CTA (whole blocks)
    const i64 per_pad = (per + 15) / 16 * 16;
    const i64 room = (i64)max_smem - per_pad - 16 - 1024 - 32 * 12;
    if (room <= 0 || per >= (1ll << 24)) continue;
    i64 cap = (room / (S * 4) - 4) / (DW + 1);
    cap = std::min<i64>(cap, 1024) / 32 * 32;
    if (cap < 64) continue;
    // a cluster of cl CTAs with this much shared memory must be schedulable
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3((unsigned)cap);
    cfg.dynamicSmemBytes = (size_t)(per_pad + 16 + S * (cap * (DW + 1) + 4) * 4 + 32 * 12);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const ClusterKernel kf = cluster_kernel(DW);
    cudaFuncAttributes fa;
    CUDA_CHECK(cudaFuncGetAttributes(&fa, kf));
    CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    max_smem - (int)fa.sharedSizeBytes));
    if (cl > 8) CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kf, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nclusters < 1) continue;
    CL = cl;
    CAP = (int)cap;
    break;
  }
  if (CL == 0) return false;
  // entries regrouped by (level, owner CTA, id)
  Own own;
  own.logB = logB;
  own.logCL = CL == 16 ? 4 : 3;
  DBuf<i64> bnd_d;
  DBuf<u64> keys;
  keys.alloc(std::max<i64>(nent, 1), s);
  k_entry_keys<<<grid_for(std::max<i64>(nent, 1), 256, num_sms() * 8), 256, 0, s>>>(plan.v.p, nent, ls_d.p, L, own,
                                                                                    keys.p);
  sort_u64(keys.p, nent, s);
  k_keys_to_ids<<<grid_for(std::max<i64>(nent, 1), 256, num_sms() * 8), 256, 0, s>>>(keys.p, nent, plan.v.p);
  bnd_d.alloc(L * (CL + 1), s);
  k_bounds<<<grid_for(L * (CL + 1), 256, num_sms() * 8), 256, 0, s>>>(keys.p, nent, L, CL, bnd_d.p);
  count_launch(3);
  std::vector<i64> bnd((size_t)(L * (CL + 1)));
  CUDA_CHECK(cudaMemcpyAsync(bnd.data(), bnd_d.p, sizeof(i64) * bnd.size(), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  // ---- items per CTA, grouped by CTA (each CTA's items are contiguous)
  std::vector<i32> ia, in, il, ci((size_t)CL * (L + 1));
  for (int r = 0; r < CL; r++)
    for (i64 l = 0; l < L; l++) {
      ci[(size_t)r * (L + 1) + l] = (i32)ia.size();
      const i64 b0 = bnd[(size_t)(l * (CL + 1) + r)], b1 = bnd[(size_t)(l * (CL + 1) + r + 1)];
      for (i64 x = b0; x < b1; x += CAP) {
        ia.push_back((i32)x);
        in.push_back((i32)std::min<i64>(CAP, b1 - x));
        il.push_back((i32)l);
      }
      if (l == L - 1) ci[(size_t)r * (L + 1) + L] = (i32)ia.size();
    }
  if (nent >= (1ll << 31) || (i64)ia.size() >= (1ll << 31)) return false;
  const i64 nitems = (i64)ia.size();
  // launch only the threads the largest item needs (whole warps)
  i32 maxn = 32;
  for (i32 x : in) maxn = std::max(maxn, x);
  plan.nthreads = (maxn + 31) / 32 * 32;
  // blob: per item [n, level, link, npad | ids | slots], rows padded to npad = n
  // rounded up to 4, so every item is a whole number of 16-byte units (TMA bulk copy)
  std::vector<i64> io((size_t)nitems);
  std::vector<i32> isz((size_t)nitems);
  i64 total = 0;
  for (i64 it = 0; it < nitems; it++) {
    io[(size_t)it] = total;
    isz[(size_t)it] = 4 + (in[(size_t)it] + 3) / 4 * 4 * (DW + 1);
    total += isz[(size_t)it];
  }
  DBuf<i32> item_a, item_n, item_l;
  item_a.upload(ia.data(), std::max<i64>(nitems, 1), s);
  item_n.upload(in.data(), std::max<i64>(nitems, 1), s);
  item_l.upload(il.data(), std::max<i64>(nitems, 1), s);
  plan.item_o.upload(io.data(), std::max<i64>(nitems, 1), s);
  plan.item_sz.upload(isz.data(), std::max<i64>(nitems, 1), s);
  plan.cta_item.upload(ci.data(), (i64)ci.size(), s);
  plan.blob.alloc(std::max<i64>(total, 4), s);
  k_item_hdr<<<grid_for(std::max<i64>(nitems, 1), 256, num_sms() * 8), 256, 0, s>>>(item_n.p, item_l.p,
                                                                                    plan.item_o.p, nitems, plan.blob.p);
  DBuf<i32> ent_item;
  ent_item.alloc(std::max<i64>(nent, 1), s);
  k_ent_item<<<(int)std::min<i64>(std::max<i64>(nitems, 1), (i64)num_sms() * 16), 256, 0, s>>>(
      item_a.p, item_n.p, nitems, ent_item.p);
  k_fill_slots<<<grid_for(std::max<i64>(nent, 1), 256, num_sms() * 8), 256, 0, s>>>(
      rowptr, col, keys.p, ent_item.p, item_a.p, item_n.p, plan.item_o.p, nent, DW, own, member.p, plan.blob.p,
      zero_nm, (i32)((per + 15) / 16 * 16));
  count_launch(3);
  CUDA_CHECK(cudaStreamSynchronize(s));
  plan.v.release();
  plan.CL = CL;
  plan.chains = chains;
  plan.zero_nm = zero_nm;
  plan.CAP = CAP;
  plan.DW = DW;
  plan.per = per;
  plan.logB = own.logB;
  plan.logCL = own.logCL;
  plan.nv = nv;
  plan.L = L;
  plan.smem = (size_t)((per + 15) / 16 * 16 + 16 + (i64)S * ((i64)CAP * (DW + 1) + 4) * 4 + 32 * 12);
  plan.ok = true;
  static const bool trace = std::getenv("CHROMA_LEVEL_TRACE") != nullptr;
  if (trace)
    std::fprintf(stderr, "[cluster] %d CTAs x %d (cap %d) threads, %lld levels, %lld entries, %lld items, DW %d, smem %zu%s\n",
                 CL, plan.nthreads, CAP, (long long)L, (long long)nent, (long long)nitems, DW, plan.smem, chains ? ", runs" : "");
  return true;
}

void launch_gs_cluster(const ClusterPlan& p, i32* val, const i32* old, cudaStream_t s) {
  ClusterArgs a;
  a.blob = p.blob.p;
  a.item_o = p.item_o.p;
  a.item_sz = p.item_sz.p;
  a.cta_item = p.cta_item.p;
  a.L = p.L;
  a.nv = p.nv;
  a.per = p.per;
  a.own.logB = p.logB;
  a.own.logCL = p.logCL;
  a.DW = p.DW;
  a.CAP = p.CAP;
  a.chains = p.chains;
  a.val = val;
  a.old = old;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(p.CL);
  cfg.blockDim = dim3((unsigned)(p.nthreads > 0 ? p.nthreads : p.CAP));
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, cluster_kernel(p.DW), a));
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace chroma
