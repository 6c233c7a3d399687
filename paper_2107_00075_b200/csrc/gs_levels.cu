// Level schedule for the ordered (Gauss-Seidel) kernel.
//
// The reference colours the worklist in ascending id (chroma/localcolor.py:161-165):
// v depends exactly on its worklist neighbours u < v.  The dataflow kernel
// (color_gs_d1.cu) evaluates that DAG in any order that claims dependencies
// first, but claiming chunks in id order limits the work in flight to a window
// of ids, while on a mesh the DAG's wavefront (all vertices of one longest-path
// level) spans nearly the whole id range: the window, not the DAG depth, sets
// the time.  Here the DAG's levels are computed once per graph (Kahn frontiers:
// level(v) = 1 + max level(u), u < v a worklist neighbour) and the worklist is
// laid out level by level, each level padded to whole 32-vertex chunks (entries
// -1), ids ascending inside a level.  Vertices of one level are never adjacent, so
// a chunk has no internal dependencies and everything it waits for was claimed
// earlier.  The colouring is unchanged (same DAG, same first-fit rule); only the
// evaluation order differs.  Deep, narrow DAGs (average level < 2048 vertices) keep
// the id order, where the kernel resolves chains inside a warp (C2: 890 levels of
// ~2,400 vertices -> levels; C1 and R-MAT -> id order).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "world.cuh"

namespace chroma {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// indeg[v] = number of worklist neighbours u < v (rows are sorted ascending)
__global__ void k_level_indeg(const i64* rowptr, const i32* col, const i32* wl, i64 n, const uint8_t* member,
                              i32* indeg, i32* level, i32* frontier, unsigned long long* nfront) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + lane;
    int d = 0;
    i32 v = -1;
    if (i < n) {
      v = wl[i];
      for (i64 e = rowptr[v]; e < rowptr[v + 1]; e++) {
        const i32 u = col[e];
        if (u >= v) break;
        d += member[u];
      }
      indeg[v] = d;
      level[v] = 0;
    }
    const bool src = i < n && d == 0;
    const unsigned m = __ballot_sync(FULL, src);
    unsigned long long o = 0;
    if (lane == 0 && m) o = atomicAdd(nfront, (unsigned long long)__popc(m));
    o = __shfl_sync(FULL, o, 0);
    if (src) frontier[o + __popc(m & ((1u << lane) - 1))] = v;
  }
}

// release the successors of one frontier; warp per vertex (rows may be long).
// Counters rotate over three slots so one launch per level suffices: this level's
// size is cnt[l%3] (recorded into sizes[l]), the next one accumulates in
// cnt[(l+1)%3], and cnt[(l+2)%3] is cleared for the level after.
__global__ void k_level_step(const i64* rowptr, const i32* col, const uint8_t* member, const i32* frontier,
                             unsigned long long* cnt, i64 lvl, i32* indeg, i32* level, i32* next,
                             unsigned long long* sizes) {
  const int lane = threadIdx.x & 31;
  const i64 n = (i64)cnt[lvl % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sizes[lvl] = (unsigned long long)n;
    cnt[(lvl + 2) % 3] = 0;
  }
  unsigned long long* nnext = cnt + (lvl + 1) % 3;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < n; i += nwarps) {
    const i32 v = frontier[i];
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    for (i64 e = re - 1 - lane; e >= rs; e -= 32) {
      const i32 x = col[e];
      if (x <= v) break;  // rows are sorted: only successors (x > v) from the top
      if (member[x] && atomicSub(indeg + x, 1) == 1) {
        level[x] = (i32)lvl + 1;
        next[atomicAdd(nnext, 1ull)] = x;
      }
    }
  }
}

__global__ void k_level_keys(const i32* wl, i64 n, const i32* level, u64* keys) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    keys[i] = ((u64)(u32)level[v] << 32) | (u32)v;
  }
}

// sorted (level, id) keys -> padded layout: level l starts at pstart[l]
__global__ void k_level_place(const u64* keys, i64 n, const i64* start, const i64* pstart, i32* out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 l = (i32)(keys[i] >> 32);
    out[pstart[l] + (i - start[l])] = (i32)(keys[i] & 0xffffffffu);
  }
}

__global__ void k_mark_members(const i32* wl, i64 n, uint8_t* member) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    member[wl[i]] = 1;
}

// ---- chain mode (cluster kernel only).  A "run" is a maximal interval of worklist
// ids h..t inside one 1024-id block (one owner CTA of gs_cluster.cu) in which every
// v > h is adjacent to v - 1.  Given every other lower neighbour's colour, first fit
// along a run is a composition of maps c -> (c == m0 ? m1 : m0) (m0, m1 = the two
// smallest colours free of the others), which the cluster kernel resolves by a
// prefix scan inside one level.  So a whole run takes one level:
// level(run) = 1 + max level(run') over runs holding a lower worklist neighbour of
// a member.  (Runs are id intervals, so the contracted graph is still a DAG; a run
// holds no edge other than its x - 1 links, see k_chain_cut.)  On
// the 27-point stencil the runs are the x-rows: 890 -> 382 levels at 128^3.
__global__ void k_chain_cont(const i64* rowptr, const i32* col, const i32* wl, i64 n, const uint8_t* member,
                             uint8_t* cont) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    bool c = false;
    if ((v & 1023) != 0 && member[v - 1])
      for (i64 e = rowptr[v + 1] - 1; e >= rowptr[v]; e--) {  // sorted row: v - 1 is the top lower entry
        const i32 u = col[e];
        if (u < v) {
          c = u == v - 1;
          break;
        }
      }
    cont[v] = c;
  }
}

// one CTA of 1024 threads per 1024-id block: head[x] = the last non-continuation id
// <= x (a max-scan); runlen[head] = length of the run
__global__ void __launch_bounds__(1024) k_run_heads(i64 nv, const uint8_t* member, const uint8_t* cont, i32* head,
                                                    i32* runlen) {
  __shared__ int wmax[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const i64 x = blockIdx.x * 1024ll + t;
  const bool c = x < nv && cont[x];
  int m = c ? -1 : t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, m, o);
    if (lane >= o) m = max(m, y);
  }
  if (lane == 31) wmax[w] = m;
  __syncthreads();
  int pre = -1;
  for (int k = 0; k < w; k++) pre = max(pre, wmax[k]);
  m = max(m, pre);
  __syncthreads();
  if (x < nv && member[x]) {
    const i32 h = (i32)(blockIdx.x * 1024ll + m);
    head[x] = h;
    const bool last = x + 1 >= nv || (t == 1023) || !cont[x + 1];
    if (last) runlen[h] = (i32)(x - h + 1);
  } else if (x < nv) {
    head[x] = -1;  // non-members (ghosts): k_run_step tests membership through head alone
  }
}

// the scan resolves only the x - 1 link: a run is cut at x if x has another lower
// neighbour inside its run (u in [head, x - 2]); cutting there leaves every
// remaining run free of such edges
__global__ void k_chain_cut(const i64* rowptr, const i32* col, const i32* wl, i64 n, const i32* head,
                            uint8_t* cont) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 x = wl[i];
    if (!cont[x]) continue;
    const i32 h = head[x];
    for (i64 e = rowptr[x]; e < rowptr[x + 1]; e++) {
      const i32 u = col[e];
      if (u >= x - 1) break;
      if (u >= h) {
        cont[x] = 0;
        break;
      }
    }
  }
}

// indeg[head] = lower worklist neighbours of the run's members outside the run
__global__ void k_run_indeg(const i64* rowptr, const i32* col, const i32* wl, i64 n, const uint8_t* member,
                            const i32* head, i32* indeg) {
  // warp-aligned: a run's members are consecutive in wl, so lanes mostly share h
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 b = (blockIdx.x * (i64)blockDim.x + threadIdx.x) & ~31ll; b < n; b += stride) {
    const i64 i = b + (threadIdx.x & 31);
    i32 h = -1;
    int d = 0;
    if (i < n) {
      const i32 x = wl[i];
      h = head[x];
      for (i64 e = rowptr[x]; e < rowptr[x + 1]; e++) {
        const i32 u = col[e];
        if (u >= h) break;
        d += member[u];
      }
    }
    const unsigned grp = __match_any_sync(FULL, h);
    d = (int)__reduce_add_sync(grp, (unsigned)d);
    if (h >= 0 && d && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) atomicAdd(indeg + h, d);
  }
}

__device__ __forceinline__ void expand_run(i32 h, i32 len, i32 lvl, i32* level, i32* out,
                                           unsigned long long* nout) {
  const unsigned long long b = atomicAdd(nout, (unsigned long long)len);
  for (i32 k = 0; k < len; k++) {
    out[b + k] = h + k;
    level[h + k] = lvl;
  }
}

__global__ void k_run_sources(const i32* wl, i64 n, const uint8_t* cont, const i32* indeg, const i32* runlen,
                              i32* level, i32* frontier, unsigned long long* nfront) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 v = wl[i];
    if (!cont[v] && indeg[v] == 0) expand_run(v, runlen[v], 0, level, frontier, nfront);
  }
}

// as k_level_step over runs: a run is released when its last outside dependency is
__global__ void k_run_step(const i64* rowptr, const i32* col, const uint8_t* member, const i32* head,
                           const i32* runlen, const i32* frontier, unsigned long long* cnt, i64 lvl, i32* indeg,
                           i32* level, i32* next, unsigned long long* sizes, i64 cap) {
  const int lane = threadIdx.x & 31;
  const i64 warp = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  // the warp's first frontier entry is loaded before the level size is known (the
  // buffer holds cap entries; the value is used only if warp < n): one dependent
  // load fewer per level
  const i32 v0 = warp < cap ? frontier[warp] : 0;
  const i64 n = (i64)cnt[lvl % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sizes[lvl] = (unsigned long long)n;
    cnt[(lvl + 2) % 3] = 0;
  }
  unsigned long long* nnext = cnt + (lvl + 1) % 3;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = warp; i < n; i += nwarps) {
    const i32 v = i == warp ? v0 : frontier[i];
    const i32 hv = head[v];
    const i64 rs = rowptr[v], re = rowptr[v + 1];
    // successors from the top of the sorted row, 32 at a time; lanes releasing the
    // same run combine their decrements (mesh rows hit a few runs many times)
    for (i64 base = re - 1; base >= rs; base -= 32) {
      const i64 e = base - lane;
      i32 h = -1;
      bool more = false;
      if (e >= rs) {
        const i32 x = col[e];
        if (x > v) {
          more = true;
          const i32 hx = head[x];  // -1 for non-members: one dependent load, not two
          if (hx >= 0 && hx != hv) h = hx;
        }
      }
      const unsigned grp = __match_any_sync(FULL, h);
      bool rel = false;
      i32 len = 0;
      unsigned long long b = 0;
      if (h >= 0 && lane == __ffs(grp) - 1) {
        const int c = __popc(grp);
        len = runlen[h];  // issued alongside the atomic, not after it
        rel = atomicSub(indeg + h, c) == c;
        if (rel) b = atomicAdd(nnext, (unsigned long long)len);
      }
      // released runs are written out by the whole warp (runs are up to 1024 ids)
      for (unsigned rm = __ballot_sync(FULL, rel); rm; rm &= rm - 1) {
        const int src = __ffs(rm) - 1;
        const i32 hh = __shfl_sync(FULL, h, src), ll = __shfl_sync(FULL, len, src);
        const unsigned long long bb = __shfl_sync(FULL, b, src);
        for (i32 k = lane; k < ll; k += 32) {
          next[bb + k] = hh + k;
          level[hh + k] = (i32)lvl + 1;
        }
      }
      if (!__all_sync(FULL, more)) break;
    }
  }
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

}  // namespace

bool build_level_order(const i64* rowptr, const i32* col, i64 nv, const i32* wl, i64 nwl, DBuf<i32>& out,
                       i64& nout, cudaStream_t s, std::vector<i64>* sizes_out, i64 min_width_override, bool chains) {
  const i64 min_width = min_width_override > 0 ? min_width_override : 2048;
  static const bool trace = std::getenv("CHROMA_LEVEL_TRACE") != nullptr;
  if (nwl < 4096) return false;
  const i64 max_levels = nwl / min_width;
  DBuf<uint8_t> member;
  DBuf<i32> indeg, level, fa, fb;
  DBuf<unsigned long long> cnt;
  member.alloc(nv + 1, s);
  member.zero(s);
  indeg.alloc(nv + 1, s);
  level.alloc(nv + 1, s);
  fa.alloc(nwl, s);
  fb.alloc(nwl, s);
  cnt.alloc(3, s);
  cnt.zero(s);
  DBuf<uint8_t> cont;
  DBuf<i32> head, runlen;
  k_mark_members<<<G(nwl), 256, 0, s>>>(wl, nwl, member.p);
  count_launch();
  if (chains) {
    cont.alloc(nv + 1, s);
    cont.zero(s);
    head.alloc(nv + 1, s);
    runlen.alloc(nv + 1, s);
    CUDA_CHECK(cudaMemsetAsync(indeg.p, 0, sizeof(i32) * (size_t)(nv + 1), s));
    k_chain_cont<<<G(nwl), 256, 0, s>>>(rowptr, col, wl, nwl, member.p, cont.p);
    k_run_heads<<<(unsigned)((nv + 1023) / 1024), 1024, 0, s>>>(nv, member.p, cont.p, head.p, runlen.p);
    k_chain_cut<<<G(nwl), 256, 0, s>>>(rowptr, col, wl, nwl, head.p, cont.p);
    k_run_heads<<<(unsigned)((nv + 1023) / 1024), 1024, 0, s>>>(nv, member.p, cont.p, head.p, runlen.p);
    k_run_indeg<<<G(nwl), 256, 0, s>>>(rowptr, col, wl, nwl, member.p, head.p, indeg.p);
    k_run_sources<<<G(nwl), 256, 0, s>>>(wl, nwl, cont.p, indeg.p, runlen.p, level.p, fa.p, cnt.p);
    count_launch(6);
  } else {
    k_level_indeg<<<grid_for(nwl, 256, num_sms() * 8), 256, 0, s>>>(rowptr, col, wl, nwl, member.p, indeg.p,
                                                                     level.p, fa.p, cnt.p);
    count_launch();
  }
  // frontier sizes land in a device array; the host checks every BATCH levels
  constexpr int BATCH = 64;
  const i64 cap_levels = max_levels + BATCH + 1;
  DBuf<unsigned long long> dsz;
  dsz.alloc(cap_levels + 1, s);
  dsz.zero(s);
  // host copy grows by BATCH per check (cap_levels is nwl when the caller allows any
  // depth: zero-filling that up front cost ~2 ms of host time per build)
  std::vector<unsigned long long> hsz;
  const auto tl0 = std::chrono::steady_clock::now();
  i32* buf[2] = {fa.p, fb.p};
  CUDA_CHECK(cudaMemsetAsync(cnt.p + 1, 0, 2 * sizeof(unsigned long long), s));
  i64 lvl = 0;
  bool done = false;
  const int grid = num_sms() * 8;
  while (!done) {
    for (int k = 0; k < BATCH; k++, lvl++) {
      const int p = (int)(lvl & 1);
      if (chains)
        k_run_step<<<grid, 256, 0, s>>>(rowptr, col, member.p, head.p, runlen.p, buf[p], cnt.p, lvl, indeg.p,
                                        level.p, buf[p ^ 1], dsz.p, nwl);
      else
        k_level_step<<<grid, 256, 0, s>>>(rowptr, col, member.p, buf[p], cnt.p, lvl, indeg.p, level.p,
                                          buf[p ^ 1], dsz.p);
    }
    count_launch(BATCH);
    hsz.resize((size_t)lvl);
    CUDA_CHECK(cudaMemcpyAsync(hsz.data() + (lvl - BATCH), dsz.p + (lvl - BATCH), sizeof(unsigned long long) * BATCH,
                               cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    done = hsz[(size_t)lvl - 1] == 0;
    if (!done && lvl > max_levels) {  // deep and narrow: id order is better
      if (trace) std::fprintf(stderr, "[levels] > %lld levels for %lld vertices: id order\n", (long long)max_levels,
                              (long long)nwl);
      return false;
    }
  }
  std::vector<i64> sizes;
  i64 seen = 0;
  for (i64 l = 0; l < lvl && hsz[(size_t)l] > 0; l++) {
    sizes.push_back((i64)hsz[(size_t)l]);
    seen += (i64)hsz[(size_t)l];
  }
  if ((i64)sizes.size() > max_levels) return false;
  CHROMA_REQUIRE(seen == nwl, CHROMA_ERUNTIME, "level schedule did not cover the worklist");
  const i64 L = (i64)sizes.size();
  if (sizes_out) *sizes_out = sizes;
  const auto tl1 = std::chrono::steady_clock::now();
  if (trace)
    std::fprintf(stderr, "[levels] %lld levels for %lld vertices%s, level loop %.2f ms\n", (long long)L,
                 (long long)nwl, chains ? " (runs)" : "",
                 std::chrono::duration<double, std::milli>(tl1 - tl0).count());
  std::vector<i64> start((size_t)L), pstart((size_t)L);
  i64 a = 0, b = 0;
  for (i64 l = 0; l < L; l++) {
    start[(size_t)l] = a;
    pstart[(size_t)l] = b;
    a += sizes[(size_t)l];
    b += (sizes[(size_t)l] + 31) / 32 * 32;
  }
  nout = b;
  DBuf<u64> keys;
  keys.alloc(nwl, s);
  k_level_keys<<<G(nwl), 256, 0, s>>>(wl, nwl, level.p, keys.p);
  count_launch();
  sort_u64(keys.p, nwl, s);
  DBuf<i64> st, pst;
  st.upload(start.data(), L, s);
  pst.upload(pstart.data(), L, s);
  out.alloc(nout, s);
  launch_fill_i32(out.p, nout, -1, s);
  k_level_place<<<G(nwl), 256, 0, s>>>(keys.p, nwl, st.p, pst.p, out.p);
  count_launch();
  CUDA_CHECK(cudaStreamSynchronize(s));
  return true;
}

}  // namespace chroma

namespace chroma {
namespace {
__global__ void k_place_chunks(const i32* wl, const i64* src, const i64* dst, const i32* len, i64 nchunks, i32* out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nchunks * 32; i += (i64)gridDim.x * blockDim.x) {
    const i64 c = i >> 5;
    const int l = (int)(i & 31);
    if (l < len[c]) out[dst[c] + l] = wl[src[c] + l];
  }
}
}  // namespace

// Virtual ranks share no edges: interleave their 32-vertex chunks round-robin so the
// claim window covers every rank's front at once (each rank keeps its id order,
// chunks never straddle ranks, the tail chunk of a rank is padded with -1).
bool build_rank_interleave(const i32* wl, const std::vector<i64>& rank_counts, DBuf<i32>& out, i64& nout,
                           cudaStream_t s) {
  if (rank_counts.size() < 2) return false;
  std::vector<i64> first(rank_counts.size()), nch(rank_counts.size());
  i64 acc = 0, maxch = 0;
  for (size_t r = 0; r < rank_counts.size(); r++) {
    first[r] = acc;
    acc += rank_counts[r];
    nch[r] = (rank_counts[r] + 31) / 32;
    maxch = std::max(maxch, nch[r]);
  }
  std::vector<i64> src, dst;
  std::vector<i32> len;
  i64 pos = 0;
  for (i64 k = 0; k < maxch; k++)
    for (size_t r = 0; r < rank_counts.size(); r++) {
      if (k >= nch[r]) continue;
      src.push_back(first[r] + 32 * k);
      dst.push_back(pos);
      len.push_back((i32)std::min<i64>(32, rank_counts[r] - 32 * k));
      pos += 32;
    }
  nout = pos;
  const i64 nc = (i64)src.size();
  DBuf<i64> ds, dd;
  DBuf<i32> dl;
  ds.upload(src.data(), nc, s);
  dd.upload(dst.data(), nc, s);
  dl.upload(len.data(), nc, s);
  out.alloc(nout, s);
  launch_fill_i32(out.p, nout, -1, s);
  k_place_chunks<<<grid_for(nc * 32, 256, num_sms() * 16), 256, 0, s>>>(wl, ds.p, dd.p, dl.p, nc, out.p);
  count_launch();
  CUDA_CHECK(cudaStreamSynchronize(s));
  return true;
}

}  // namespace chroma
