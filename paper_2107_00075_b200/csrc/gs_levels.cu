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

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 16); }

}  // namespace

bool build_level_order(const i64* rowptr, const i32* col, i64 nv, const i32* wl, i64 nwl, DBuf<i32>& out,
                       i64& nout, cudaStream_t s, std::vector<i64>* sizes_out, i64 min_width_override) {
  static const i64 min_width_env = [] {
    const char* e = std::getenv("CHROMA_LEVEL_MIN_WIDTH");
    return e ? std::atoll(e) : 2048ll;
  }();
  const i64 min_width = min_width_override > 0 ? min_width_override : min_width_env;
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
  k_mark_members<<<G(nwl), 256, 0, s>>>(wl, nwl, member.p);
  k_level_indeg<<<grid_for(nwl, 256, num_sms() * 8), 256, 0, s>>>(rowptr, col, wl, nwl, member.p, indeg.p,
                                                                   level.p, fa.p, cnt.p);
  count_launch(2);
  // frontier sizes land in a device array; the host checks every BATCH levels
  constexpr int BATCH = 64;
  const i64 cap_levels = max_levels + BATCH + 1;
  DBuf<unsigned long long> dsz;
  dsz.alloc(cap_levels + 1, s);
  dsz.zero(s);
  std::vector<unsigned long long> hsz((size_t)cap_levels + 1, 0);
  i32* buf[2] = {fa.p, fb.p};
  CUDA_CHECK(cudaMemsetAsync(cnt.p + 1, 0, 2 * sizeof(unsigned long long), s));
  i64 lvl = 0;
  bool done = false;
  const int grid = num_sms() * 8;
  while (!done) {
    for (int k = 0; k < BATCH; k++, lvl++) {
      const int p = (int)(lvl & 1);
      k_level_step<<<grid, 256, 0, s>>>(rowptr, col, member.p, buf[p], cnt.p, lvl, indeg.p, level.p, buf[p ^ 1],
                                        dsz.p);
    }
    count_launch(BATCH);
    CUDA_CHECK(cudaMemcpyAsync(hsz.data(), dsz.p, sizeof(unsigned long long) * (size_t)lvl, cudaMemcpyDeviceToHost,
                               s));
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
  if (trace) std::fprintf(stderr, "[levels] %lld levels for %lld vertices\n", (long long)L, (long long)nwl);
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
