// extern "C" boundary of libchroma_b200.so (declared in include/chroma_b200.h).
// Every call catches C++ exceptions and maps them to the reference's exception
// classes through status codes + a thread-local message.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "world.cuh"

namespace chroma {
int run_distributed(World& w, int mode, bool rd, int algo, int max_rounds, i32* colors_out,
                    chroma_round_report* reports, i64* recolored, i64 cap, i64* n_reports,
                    bool out_on_device);
#ifdef CHROMA_WITH_NCCL
void world_connect(World& w, void* comm, i32 nranks, i32 rank, const i64* send_counts,
                   const i64* send_lids, const i64* recv_counts, const i64* recv_lids);
#endif

static thread_local std::string t_err;
void set_last_error(const std::string& m) { t_err = m; }
}  // namespace chroma

using namespace chroma;

struct chroma_csr {
  Csr g;
  ColorScratch cs;
};
struct chroma_world {
  World* w = nullptr;
};
struct chroma_comm {
#ifdef CHROMA_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  int nranks = 0, rank = 0;
};

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return CHROMA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host out of memory");
    return CHROMA_ERUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CHROMA_ECUDA;
  }
}

static bool dev(uint32_t flags) { return (flags & CHROMA_DEVICE_PTRS) != 0; }

// int64 ids (host or device) -> int32 device array, range-checked against [0, n)
static void upload_ids(const int64_t* ids, i64 k, i64 n, bool on_device, DBuf<i32>& out, cudaStream_t s) {
  std::vector<int64_t> h;
  const int64_t* src = ids;
  if (on_device) {
    h.resize((size_t)k);
    if (k) CUDA_CHECK(cudaMemcpyAsync(h.data(), ids, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    src = h.data();
  }
  std::vector<i32> v((size_t)k);
  for (i64 i = 0; i < k; i++) {
    CHROMA_REQUIRE(src[i] >= 0 && src[i] < n, CHROMA_EVALUE, "vertex id out of range");
    v[(size_t)i] = (i32)src[i];
  }
  out.upload(v.data(), std::max<i64>(k, 1), s);
}

extern "C" {

const char* chroma_last_error(void) { return t_err.c_str(); }
const char* chroma_version(void) { return "chroma_b200 0.1 (sm_100a)"; }

int chroma_device_count(int* count) {
  return guarded([&] { CUDA_CHECK(cudaGetDeviceCount(count)); });
}

uint64_t chroma_gid_rand(int64_t gid) { return gid_rand(gid); }

int chroma_check_conflicts(int64_t v, int64_t u, int32_t* colors, const int64_t* gids,
                           const int64_t* degrees, int recolor_degrees, int* result) {
  return guarded([&] {
    const i32 cv = colors[v], cu = colors[u];
    if (cv == 0 || cu == 0 || cv != cu) {
      *result = 0;
      return;
    }
    CHROMA_REQUIRE(gids[v] != gids[u], CHROMA_EVALUE,
                   "conflict check on the same global vertex " + std::to_string(gids[v]));
    const bool vl = v_loses(gids[v], gids[u], degrees ? degrees[v] : 0, degrees ? degrees[u] : 0,
                            recolor_degrees != 0);
    colors[vl ? v : u] = 0;
    *result = 1;
  });
}

int64_t chroma_launch_count(void) { return launch_count(); }

// ---------------------------------------------------------------- CSR graphs
int chroma_csr_create(int64_t n, const int64_t* off, const int64_t* col, int device, uint32_t flags,
                      chroma_csr** out) {
  return guarded([&] {
    CHROMA_REQUIRE(n >= 0 && n < INT32_MAX, CHROMA_EVALUE, "graph too large for int32 ids");
    CUDA_CHECK(cudaSetDevice(device));
    retain_pool_memory(device);
    auto* h = new chroma_csr();
    try {
      h->g.device = device;
      CUDA_CHECK(cudaStreamCreateWithFlags(&h->g.stream, cudaStreamNonBlocking));
      cudaStream_t s = h->g.stream;
      if (dev(flags)) {
        h->g.rowptr.alloc(n + 1, s);
        CUDA_CHECK(cudaMemcpyAsync(h->g.rowptr.p, off, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
      } else {
        upload_large(h->g.rowptr, off, n + 1, s);
      }
      i64 nnz = 0;
      CUDA_CHECK(cudaMemcpyAsync(&nnz, h->g.rowptr.p + n, sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      CHROMA_REQUIRE(nnz >= 0, CHROMA_EVALUE, "row_offsets[n] must be >= 0");
      h->g.n = n;
      h->g.nnz = nnz;
      // narrowed and range-checked on the way in (upload.cu for host arrays)
      h->g.col.alloc(std::max<i64>(nnz, 1), s);
      narrow_ids_checked(col, nnz, n, dev(flags), h->g.col.p, s, "col_indices out of range");
      CUDA_CHECK(cudaStreamSynchronize(s));
    } catch (...) {
      // the buffers free on the stream: release them before the stream goes
      cudaStream_t st = h->g.stream;
      if (st) cudaStreamSynchronize(st);
      delete h;
      if (st) cudaStreamDestroy(st);
      throw;
    }
    *out = h;
  });
}

int chroma_csr_destroy(chroma_csr* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(h->g.device);
    cudaStream_t s = h->g.stream;
    cudaStreamSynchronize(s);
    delete h;
    cudaStreamDestroy(s);
  });
}

int chroma_serial_greedy(chroma_csr* h, const int64_t* order, int32_t* colors_out, uint32_t flags) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(h->g.device));
    cudaStream_t s = h->g.stream;
    const i64 n = h->g.n;
    ColorScratch& S = h->cs;
    S.val.reserve(n + 1, s);
    S.wl.reserve(n + 1, s);
    S.nwl.reserve(1, s);
    S.ticket.reserve(1, s);
    DBuf<i32> prio;
    if (order) {
      DBuf<i32> ord;
      upload_ids(order, n, n, dev(flags), ord, s);
      std::vector<i32> ho((size_t)n);
      CUDA_CHECK(cudaMemcpyAsync(ho.data(), ord.p, sizeof(i32) * n, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      std::vector<i32> pr((size_t)n, -1);
      for (i64 i = 0; i < n; i++) {
        CHROMA_REQUIRE(pr[(size_t)ho[(size_t)i]] < 0, CHROMA_EVALUE, "order is not a permutation of the vertices");
        pr[(size_t)ho[(size_t)i]] = (i32)i;
      }
      prio.upload(pr.data(), std::max<i64>(n, 1), s);
      CUDA_CHECK(cudaMemcpyAsync(S.wl.p, ord.p, sizeof(i32) * n, cudaMemcpyDeviceToDevice, s));
    }
    launch_fill_i32(S.val.p, n, PENDING, s);
    CUDA_CHECK(cudaMemcpyAsync(S.nwl.p, &n, sizeof(i64), cudaMemcpyHostToDevice, s));
    GsLaunch L;
    L.rowptr = h->g.rowptr.p;
    L.col = h->g.col.p;
    L.val = S.val.p;
    L.wl = order ? S.wl.p : nullptr;
    L.wl_base = 0;
    L.nwl_dev = S.nwl.p;
    L.nwl_max = n;
    L.prio = order ? prio.p : nullptr;
    L.ticket = S.ticket.p;
    L.dist = 1;
    L.nv = n;
    static const bool no_chunked = std::getenv("CHROMA_NO_CHUNKED") != nullptr;
    bool done = n == 0;
    if (!done && !order && !no_chunked) done = launch_gs_chunked(L, n, true, S.chunked, s);
    if (!done) launch_gs(L, s);
    CUDA_CHECK(cudaMemcpyAsync(colors_out, S.val.p, sizeof(i32) * n,
                               dev(flags) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int chroma_color(chroma_csr* h, int32_t* colors, const int64_t* worklist, int64_t nwl, int dist,
                 int partial, int algo, uint32_t flags) {
  return guarded([&] {
    CHROMA_REQUIRE(dist == 1 || dist == 2, CHROMA_EVALUE, "dist must be 1 or 2");
    if (nwl == 0) return;
    CUDA_CHECK(cudaSetDevice(h->g.device));
    cudaStream_t s = h->g.stream;
    const i64 n = h->g.n;
    DBuf<i32> wl, cols;
    upload_ids(worklist, nwl, n, dev(flags), wl, s);
    i32* cdev = colors;
    if (!dev(flags)) {
      cols.upload(colors, std::max<i64>(n, 1), s);
      cdev = cols.p;
    }
    DBuf<i64> nd;
    nd.upload(&nwl, 1, s);
    color_csr(h->g.rowptr.p, h->g.col.p, n, cdev, wl.p, nd.p, nwl, false, dist, partial != 0, algo, false,
              h->cs, s);
    if (!dev(flags)) CUDA_CHECK(cudaMemcpyAsync(colors, cols.p, sizeof(i32) * n, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int chroma_detect(chroma_csr* h, int32_t* colors, const int64_t* gids, const int64_t* degrees,
                  const int64_t* rows, int64_t nrows, int dist, int partial, int rd, int64_t* count,
                  uint32_t flags) {
  return guarded([&] {
    CHROMA_REQUIRE(!dev(flags), CHROMA_EVALUE, "chroma_detect takes host arrays");
    CHROMA_REQUIRE(dist == 1 || dist == 2, CHROMA_EVALUE, "dist must be 1 or 2");
    CUDA_CHECK(cudaSetDevice(h->g.device));
    cudaStream_t s = h->g.stream;
    const i64 n = h->g.n;
    DBuf<i32> c, r, d;
    DBuf<i64> gd;
    DBuf<unsigned long long> cnt;
    c.upload(colors, std::max<i64>(n, 1), s);
    gd.upload(gids, std::max<i64>(n, 1), s);
    std::vector<i32> dh((size_t)n);
    for (i64 i = 0; i < n; i++) {
      CHROMA_REQUIRE(degrees[i] >= INT32_MIN && degrees[i] <= INT32_MAX, CHROMA_EVALUE, "degree out of int32 range");
      dh[(size_t)i] = (i32)degrees[i];
    }
    d.upload(dh.data(), std::max<i64>(n, 1), s);
    upload_ids(rows, nrows, n, false, r, s);
    cnt.alloc(1, s);
    cnt.zero(s);
    DetectScratch S;
    DetectArgs a;
    a.rowptr = h->g.rowptr.p;
    a.col = h->g.col.p;
    a.colors = c.p;
    a.gids = gd.p;
    a.deg = d.p;
    a.rows = r.p;
    a.nrows = nrows;
    a.dist = dist;
    a.partial = partial != 0;
    a.recolor_degrees = rd != 0;
    a.sequential = true;
    run_detect(a, n, S, cnt.p, s);
    unsigned long long hc = 0;
    CUDA_CHECK(cudaMemcpyAsync(&hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(colors, c.p, sizeof(i32) * n, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    *count = (int64_t)hc;
  });
}

int chroma_verify(chroma_csr* h, const int32_t* colors, const uint8_t* mask, int mode, int64_t* nviol,
                  int64_t* rows, int64_t cap, uint32_t flags) {
  return guarded([&] {
    CHROMA_REQUIRE(mode >= 0 && mode <= 2, CHROMA_EVALUE, "verify mode must be 0, 1 or 2");
    CUDA_CHECK(cudaSetDevice(h->g.device));
    cudaStream_t s = h->g.stream;
    const i64 n = h->g.n;
    DBuf<i32> c;
    DBuf<uint8_t> m;
    const i32* cd = colors;
    const uint8_t* md = mask;
    if (!dev(flags)) {
      c.upload(colors, std::max<i64>(n, 1), s);
      cd = c.p;
      if (mask) {
        m.upload(mask, std::max<i64>(n, 1), s);
        md = m.p;
      }
    }
    *nviol = run_verify(h->g.rowptr.p, h->g.col.p, n, cd, md, mode, rows, cap, s);
  });
}

int chroma_color_stats(const int32_t* colors, int64_t n, int device, int64_t* num_colors, int64_t* max_color,
                       int64_t* hist, int64_t hist_cap, uint32_t flags) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    {
      DBuf<i32> c;
      const i32* cd = colors;
      if (!dev(flags)) {
        c.upload(colors, std::max<i64>(n, 1), s);
        cd = c.p;
      }
      run_color_stats(cd, n, num_colors, max_color, hist, hist_cap, s);
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
  });
}

// ---------------------------------------------------------------- worlds
int chroma_world_create(int64_t n, const int64_t* off, const int64_t* col, int32_t P, const int32_t* owner,
                        int32_t gl, int32_t lo, int32_t hi, int device, chroma_world** out) {
  return guarded([&] {
    auto* h = new chroma_world();
    try {
      h->w = world_create(n, off, col, P, owner, gl, lo, hi, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int chroma_world_destroy(chroma_world* h) {
  return guarded([&] {
    if (!h) return;
    world_destroy(h->w);
    delete h;
  });
}

int chroma_world_rank_info(chroma_world* h, int32_t rank, int64_t* info) {
  return guarded([&] {
    const World& w = *h->w;
    const RankMeta& m = w.meta(rank);
    std::fill(info, info + 16, 0);
    info[0] = m.owned; info[1] = m.ghost; info[2] = m.l1; info[3] = m.e_local; info[4] = m.e_ghost;
    info[5] = m.nnz; info[6] = m.nb1; info[7] = m.nb2; info[8] = w.delta_max; info[9] = w.n_global;
    info[10] = w.m_global; info[11] = w.gl; info[12] = m.lid_off;
  });
}

int chroma_world_rank_arrays(chroma_world* h, int32_t rank, int64_t* off, int64_t* col, int64_t* gids,
                             int32_t* ghost_owner, int64_t* b1, int64_t* b2) {
  return guarded([&] {
    World& w = *h->w;
    const RankMeta& m = w.meta(rank);
    cudaStream_t s = w.stream;
    CUDA_CHECK(cudaSetDevice(w.device));
    // every output pointer may be NULL (that array is not copied)
    const i64 nl = m.owned + m.ghost;
    std::vector<i64> o(off ? (size_t)nl + 1 : 0);
    std::vector<i32> c(col ? (size_t)m.nnz : 0), bb1(b1 ? (size_t)m.nb1 : 0), bb2(b2 ? (size_t)m.nb2 : 0);
    if (off)
      CUDA_CHECK(cudaMemcpyAsync(o.data(), w.g.rowptr.p + m.lid_off, sizeof(i64) * (nl + 1), cudaMemcpyDeviceToHost, s));
    if (col && m.nnz)
      CUDA_CHECK(cudaMemcpyAsync(c.data(), w.g.col.p + m.nnz_off, sizeof(i32) * m.nnz, cudaMemcpyDeviceToHost, s));
    if (gids) CUDA_CHECK(cudaMemcpyAsync(gids, w.gids.p + m.lid_off, sizeof(i64) * nl, cudaMemcpyDeviceToHost, s));
    if (ghost_owner && m.ghost)
      CUDA_CHECK(cudaMemcpyAsync(ghost_owner, w.ghost_owner.p + m.ghost_off, sizeof(i32) * m.ghost, cudaMemcpyDeviceToHost, s));
    if (b1 && m.nb1) CUDA_CHECK(cudaMemcpyAsync(bb1.data(), w.b1.p + m.b1_off, sizeof(i32) * m.nb1, cudaMemcpyDeviceToHost, s));
    if (b2 && m.nb2) CUDA_CHECK(cudaMemcpyAsync(bb2.data(), w.b2.p + m.b2_off, sizeof(i32) * m.nb2, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (off) for (i64 i = 0; i <= nl; i++) off[i] = o[(size_t)i] - m.nnz_off;
    if (col) for (i64 i = 0; i < m.nnz; i++) col[i] = (i64)c[(size_t)i] - m.lid_off;
    if (b1) for (i64 i = 0; i < m.nb1; i++) b1[i] = (i64)bb1[(size_t)i] - m.lid_off;
    if (b2) for (i64 i = 0; i < m.nb2; i++) b2[i] = (i64)bb2[(size_t)i] - m.lid_off;
  });
}

int chroma_nccl_unique_id(void* id_out) {
  return guarded([&] {
#ifdef CHROMA_WITH_NCCL
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    CHROMA_REQUIRE(r == ncclSuccess, CHROMA_ECUDA, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id_out, &id, sizeof(id));
#else
    (void)id_out;
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  });
}

int chroma_comm_create(const void* id_bytes, int32_t nranks, int32_t rank, int device, chroma_comm** out) {
  return guarded([&] {
#ifdef CHROMA_WITH_NCCL
    CUDA_CHECK(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    auto* c = new chroma_comm();
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      throw Error(CHROMA_ECUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
#else
    (void)id_bytes; (void)nranks; (void)rank; (void)device; (void)out;
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  });
}

int chroma_comm_create_all(int32_t ndev, const int* devices, chroma_comm** out) {
  return guarded([&] {
#ifdef CHROMA_WITH_NCCL
    CHROMA_REQUIRE(ndev >= 1, CHROMA_EVALUE, "ndev must be >= 1");
    std::vector<ncclComm_t> comms((size_t)ndev);
    ncclResult_t r = ncclCommInitAll(comms.data(), ndev, devices);
    if (r != ncclSuccess) throw Error(CHROMA_ECUDA, std::string("ncclCommInitAll: ") + ncclGetErrorString(r));
    for (int i = 0; i < ndev; i++) {
      auto* c = new chroma_comm();
      c->comm = comms[(size_t)i];
      c->nranks = ndev;
      c->rank = i;
      out[i] = c;
    }
#else
    (void)ndev; (void)devices; (void)out;
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  });
}

int chroma_comm_destroy(chroma_comm* c) {
  return guarded([&] {
#ifdef CHROMA_WITH_NCCL
    if (c) ncclCommDestroy(c->comm);
#endif
    delete c;
  });
}

int chroma_world_connect(chroma_world* h, chroma_comm* c, int32_t nranks, int32_t rank, const int64_t* sc,
                         const int64_t* sl, const int64_t* rc, const int64_t* rl) {
  return guarded([&] {
#ifdef CHROMA_WITH_NCCL
    CHROMA_REQUIRE(c && c->nranks == nranks && c->rank == rank, CHROMA_EVALUE, "communicator does not match");
    world_connect(*h->w, (void*)c->comm, nranks, rank, sc, sl, rc, rl);
#else
    (void)h; (void)c; (void)nranks; (void)rank; (void)sc; (void)sl; (void)rc; (void)rl;
    throw Error(CHROMA_ECUDA, "built without NCCL");
#endif
  });
}

int chroma_world_global_degrees(chroma_world* h, int32_t rank, int64_t* out) {
  return guarded([&] {
    World& w = *h->w;
    const RankMeta& m = w.meta(rank);
    CUDA_CHECK(cudaSetDevice(w.device));
    const i64 nl = m.owned + m.ghost;
    std::vector<i32> d((size_t)nl);
    CUDA_CHECK(cudaMemcpyAsync(d.data(), w.deg.p + m.lid_off, sizeof(i32) * nl, cudaMemcpyDeviceToHost, w.stream));
    CUDA_CHECK(cudaStreamSynchronize(w.stream));
    for (i64 i = 0; i < nl; i++) out[i] = d[(size_t)i];
  });
}

int chroma_world_reset_exchange(chroma_world* h) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(h->w->device));
    world_reset_exchange(*h->w);
    CUDA_CHECK(cudaStreamSynchronize(h->w->stream));
  });
}

int chroma_world_exchange(chroma_world* h, int32_t** colorings, int changed_only, int64_t* bytes,
                          int64_t* msgs) {
  return guarded([&] {
    World& w = *h->w;
    CHROMA_REQUIRE(w.all_local(), CHROMA_EVALUE, "exchange_boundary_colors needs every rank in this process");
    CUDA_CHECK(cudaSetDevice(w.device));
    cudaStream_t s = w.stream;
    for (auto& m : w.ranks)
      CUDA_CHECK(cudaMemcpyAsync(w.colors.p + m.lid_off, colorings[m.rank], sizeof(i32) * (m.owned + m.ghost),
                                 cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemsetAsync(w.stats.p, 0, sizeof(unsigned long long) * 3, s));
    if (w.nrouted) {
      world_exchange_local(w, changed_only != 0, false);
      launch_pair_stats(w.pair_cnt.p, (i64)w.P * w.P, w.stats.p + 1, s);
    }
    unsigned long long st[3];
    CUDA_CHECK(cudaMemcpyAsync(st, w.stats.p, sizeof(st), cudaMemcpyDeviceToHost, s));
    for (auto& m : w.ranks)
      CUDA_CHECK(cudaMemcpyAsync(colorings[m.rank], w.colors.p + m.lid_off, sizeof(i32) * (m.owned + m.ghost),
                                 cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    *bytes = (int64_t)st[1];
    *msgs = (int64_t)st[2];
  });
}

int chroma_world_color(chroma_world* h, int32_t rank, int32_t* colors, const int64_t* worklist, int64_t nwl,
                       int dist, int partial, int algo) {
  return guarded([&] {
    World& w = *h->w;
    const RankMeta& m = w.meta(rank);
    CHROMA_REQUIRE(dist == 1 || dist == 2, CHROMA_EVALUE, "dist must be 1 or 2");
    if (nwl == 0) return;
    CUDA_CHECK(cudaSetDevice(w.device));
    cudaStream_t s = w.stream;
    const i64 nl = m.owned + m.ghost;
    std::vector<i32> wl((size_t)nwl);
    for (i64 i = 0; i < nwl; i++) {
      CHROMA_REQUIRE(worklist[i] >= 0 && worklist[i] < nl, CHROMA_EVALUE, "worklist entry out of range");
      wl[(size_t)i] = (i32)(worklist[i] + m.lid_off);
    }
    DBuf<i32> dwl;
    dwl.upload(wl.data(), nwl, s);
    DBuf<i64> nd;
    nd.upload(&nwl, 1, s);
    CUDA_CHECK(cudaMemcpyAsync(w.colors.p + m.lid_off, colors, sizeof(i32) * nl, cudaMemcpyHostToDevice, s));
    const i64* crow = w.g.rowptr.p;
    const i32* ccol = w.g.col.p;
    int cdist = dist;
    i64 cdelta = w.delta_max;
    square_for(w, dist, partial != 0, algo, false, crow, ccol, cdist, cdelta);  // distance 2 as D1 on G^2
    color_csr(crow, ccol, w.NL, w.colors.p, dwl.p, nd.p, nwl, false, cdist, partial != 0, algo, false, w.cs, s);
    CUDA_CHECK(cudaMemcpyAsync(colors, w.colors.p + m.lid_off, sizeof(i32) * nl, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int chroma_world_detect(chroma_world* h, int32_t rank, int32_t* colors, const int64_t* degrees, int dist,
                        int partial, int rd, int64_t* count) {
  return guarded([&] {
    World& w = *h->w;
    const RankMeta& m = w.meta(rank);
    if (dist == 2)
      CHROMA_REQUIRE(w.gl >= 2, CHROMA_EVALUE, "distance-2 detection needs a second ghost layer");
    CUDA_CHECK(cudaSetDevice(w.device));
    cudaStream_t s = w.stream;
    const i64 nl = m.owned + m.ghost;
    CUDA_CHECK(cudaMemcpyAsync(w.colors.p + m.lid_off, colors, sizeof(i32) * nl, cudaMemcpyHostToDevice, s));
    const i32* degp = w.deg.p;
    if (degrees) {
      w.deg_override.reserve(w.NL + 1, s);
      std::vector<i32> d((size_t)nl);
      for (i64 i = 0; i < nl; i++) {
        CHROMA_REQUIRE(degrees[i] >= INT32_MIN && degrees[i] <= INT32_MAX, CHROMA_EVALUE, "degree out of int32 range");
        d[(size_t)i] = (i32)degrees[i];
      }
      CUDA_CHECK(cudaMemcpyAsync(w.deg_override.p + m.lid_off, d.data(), sizeof(i32) * nl, cudaMemcpyHostToDevice, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      degp = w.deg_override.p;
    }
    CUDA_CHECK(cudaMemsetAsync(w.stats.p, 0, sizeof(unsigned long long), s));
    DetectArgs a;
    a.rowptr = w.g.rowptr.p;
    a.col = w.g.col.p;
    a.colors = w.colors.p;
    a.gids = w.gids.p;
    a.deg = degp;
    a.rows = dist == 2 ? w.b2.p + m.b2_off : w.ghosts.p + m.ghost_off;
    a.nrows = dist == 2 ? m.nb2 : m.ghost;
    a.dist = dist;
    a.partial = partial != 0;
    a.recolor_degrees = rd != 0;
    a.sequential = true;
    run_detect(a, w.NL, w.det, w.stats.p, s);
    unsigned long long c = 0;
    CUDA_CHECK(cudaMemcpyAsync(&c, w.stats.p, sizeof(c), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(colors, w.colors.p + m.lid_off, sizeof(i32) * nl, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    *count = (int64_t)c;
  });
}

int chroma_run_distributed(chroma_world* h, int mode, int rd, int algo, int max_rounds, int32_t* colors_out,
                           chroma_round_report* reports, int64_t* recolored, int64_t cap, int64_t* n_reports,
                           uint32_t flags) {
  int st = CHROMA_OK;
  const int g = guarded([&] {
    CHROMA_REQUIRE(mode >= 0 && mode <= 3, CHROMA_EVALUE, "unknown mode");
    CHROMA_REQUIRE(algo >= 0 && algo <= 3, CHROMA_EVALUE, "unknown algorithm");
    st = run_distributed(*h->w, mode, rd != 0, algo, max_rounds, colors_out, reports, recolored, cap, n_reports,
                         dev(flags));
    if (st == CHROMA_ENONCONV) set_last_error("no convergence after " + std::to_string(max_rounds) + " rounds");
  });
  return g != CHROMA_OK ? g : st;
}

int chroma_world_last_timing(chroma_world* h, double* out) {
  return guarded([&] {
    const World& w = *h->w;
    out[0] = w.t_total;
    out[1] = w.t_color_kernel;
    out[2] = w.t_color;
    out[3] = w.t_comm;
    out[4] = w.t_detect;
  });
}

int chroma_world_colors_device(chroma_world* h, int32_t rank, int32_t** dev_ptr, int64_t* lid_offset) {
  return guarded([&] {
    const RankMeta& m = h->w->meta(rank);
    *dev_ptr = h->w->colors.p;
    *lid_offset = m.lid_off;
  });
}

}  // extern "C"
