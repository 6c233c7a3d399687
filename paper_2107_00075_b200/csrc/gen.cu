// Device generators of the BASELINE inputs, written straight
// into int64 CSR (chroma/graph.py:40-64 layout: sorted, simple, symmetric rows).
//
// The random generators are counter-based so that the device, the NumPy host path
// (graph.py) and the C oracle (oracle/chroma_oracle.c) build bit-identical graphs
// without sharing an RNG stream.  Every draw is mix64(key) with mix64 = the
// splitmix64 finaliser the reference already uses for gid_rand
// (chroma/protocol.py:79-88):
//   R-MAT (Graph500): edge e, level l: u = mix64((seed << 40) + e*scale + l) >> 32;
//     src bit = u >= T_ab, dst bit = (T_a <= u < T_ab) || u >= T_abc, bits shifted
//     in from the most significant level; T_* = floor(p * 2^32) are passed in.
//     Labels are relabelled by perm() below, self loops dropped, both directions
//     kept, duplicates removed (chroma/graph.py:166-179 preprocess).
//   random bipartite (PD2): row r, entry j: t = ((mix64((seed << 40) + r*k + j) >> 32)
//     * rows) >> 32; diagonal arcs dropped, duplicates removed
//     (chroma/graph.py:182-188), arc (r, t) -> edge (r, rows + t) (graph.py:388-399).
//   perm (label permutation on 2^bits ids): three rounds of x -> (x*m_i + k_i) mod
//     2^bits separated by x ^= x >> ceil(bits/2); m_i = mix64(8*seed + 2i) | 1,
//     k_i = mix64(8*seed + 2i + 1).  Each step is a bijection, so perm is one.
// The meshes (hex 6-point, 27-point stencil) are analytic: each row is emitted in
// ascending id order directly, no sort.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace chroma {
namespace {

__host__ __device__ __forceinline__ u64 mix64(u64 x) { return gid_rand((i64)x); }

struct Perm {
  u64 m[3], k[3], mask;
  int shift;
  bool on;
};

Perm make_perm(u64 seed, int bits, bool on) {
  Perm p;
  for (int i = 0; i < 3; i++) {
    p.m[i] = mix64(8 * seed + 2 * (u64)i) | 1ull;
    p.k[i] = mix64(8 * seed + 2 * (u64)i + 1);
  }
  p.mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  p.shift = (bits + 1) / 2;
  p.on = on && bits >= 1;
  return p;
}

__device__ __forceinline__ u64 perm_apply(const Perm& p, u64 x) {
  if (!p.on) return x;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    x = (x * p.m[i] + p.k[i]) & p.mask;
    if (i < 2) x ^= x >> p.shift;
  }
  return x;
}

// one thread per generated edge: both directions as keys src*n + dst; a dropped
// edge (self loop) writes the never-valid key n*n - 1 ... of vertex n-1 to itself
__global__ void k_rmat_keys(u64 seed, int scale, i64 m, u32 ta, u32 tab, u32 tabc, Perm perm, u64* keys) {
  const u64 n = 1ull << scale;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    u64 src = 0, dst = 0;
    const u64 base = (seed << 40) + (u64)e * (u64)scale;
    for (int l = 0; l < scale; l++) {
      const u32 u = (u32)(mix64(base + (u64)l) >> 32);
      src = (src << 1) | (u >= tab ? 1ull : 0ull);
      dst = (dst << 1) | (((u >= ta && u < tab) || u >= tabc) ? 1ull : 0ull);
    }
    src = perm_apply(perm, src);
    dst = perm_apply(perm, dst);
    const bool drop = src == dst;
    keys[2 * e] = drop ? n * n - 1 : src * n + dst;
    keys[2 * e + 1] = drop ? n * n - 1 : dst * n + src;
  }
}

__global__ void k_bip_keys(u64 seed, i64 rows, i64 k, u64* keys) {
  const u64 n = 2 * (u64)rows;
  const i64 m = rows * k;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    const u64 r = (u64)(e / k);
    const u64 t = ((mix64((seed << 40) + (u64)e) >> 32) * (u64)rows) >> 32;
    const bool drop = r == t;
    const u64 a = r, b = (u64)rows + t;
    keys[2 * e] = drop ? n * n - 1 : a * n + b;
    keys[2 * e + 1] = drop ? n * n - 1 : b * n + a;
  }
}

// sorted keys -> keep first of each run, drop self-loop keys; degree per source
__global__ void k_key_flags(const u64* keys, i64 nk, u64 n, uint8_t* keep, i64* deg) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x) {
    const u64 key = keys[i];
    const u64 s = key / n, d = key - s * n;
    const bool k = s != d && (i == 0 || keys[i - 1] != key);
    keep[i] = k ? 1 : 0;
    if (k) atomicAdd(reinterpret_cast<unsigned long long*>(deg + s), 1ull);
  }
}

__global__ void k_key_cols(const u64* keys, i64 nk, u64 n, i64* col) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nk; i += (i64)gridDim.x * blockDim.x) {
    const u64 key = keys[i];
    col[i] = (i64)(key % n);
  }
}

// ---------------------------------------------------------------- meshes
struct Box {
  i64 nx, ny, nz;
  int kind;  // 0: 6-point (hex mesh), 1: 26 neighbours (27-point stencil)
};

template <typename F>
__device__ __forceinline__ void box_row(const Box& b, i64 v, F&& emit) {
  const i64 x = v % b.nx, y = (v / b.nx) % b.ny, z = v / (b.nx * b.ny);
  // offsets in lexicographic (dz, dy, dx) order = ascending id delta
  for (int dz = -1; dz <= 1; dz++)
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        const int nzero = (dz != 0) + (dy != 0) + (dx != 0);
        if (nzero == 0) continue;
        if (b.kind == 0 && nzero != 1) continue;
        const i64 X = x + dx, Y = y + dy, Z = z + dz;
        if (X < 0 || Y < 0 || Z < 0 || X >= b.nx || Y >= b.ny || Z >= b.nz) continue;
        emit(X + b.nx * (Y + b.ny * Z));
      }
}

__global__ void k_box_deg(Box b, i64 n, i64* deg) {
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
    i64 d = 0;
    box_row(b, v, [&](i64) { d++; });
    deg[v] = d;
  }
}

__global__ void k_box_fill(Box b, i64 n, const i64* rowptr, i64* col) {
  for (i64 v = blockIdx.x * (i64)blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
    i64 k = rowptr[v];
    box_row(b, v, [&](i64 u) { col[k++] = u; });
  }
}

int G(i64 n) { return grid_for(std::max<i64>(n, 1), 256, num_sms() * 32); }

// deg[0..n) -> rowptr[0..n] (exclusive scan, rowptr[n] = total)
void deg_to_rowptr(const i64* deg, i64 n, i64* rowptr, cudaStream_t s) {
  CUDA_CHECK(cudaMemsetAsync(rowptr, 0, sizeof(i64), s));
  if (n == 0) return;
  size_t tb = 0;
  CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, deg, rowptr + 1, n, s));
  DBuf<uint8_t> tmp;
  tmp.alloc((i64)tb, s);
  CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.p, tb, deg, rowptr + 1, n, s));
  count_launch();
}

// keys (2 per generated edge, some dropped) -> CSR; col must hold nk entries
i64 keys_to_csr(DBuf<u64>& keys, i64 nk, u64 n, int key_bits, i64* rowptr, i64* col, cudaStream_t s) {
  DBuf<u64> alt;
  alt.alloc(std::max<i64>(nk, 1), s);
  cub::DoubleBuffer<u64> db(keys.p, alt.p);
  size_t tb = 0;
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, nk, 0, key_bits, s));
  {
    DBuf<uint8_t> tmp;
    tmp.alloc((i64)tb, s);
    CUDA_CHECK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, nk, 0, key_bits, s));
  }
  count_launch();
  u64* sorted = db.Current();
  u64* spare = db.Alternate();
  DBuf<uint8_t> keep;
  keep.alloc(std::max<i64>(nk, 1), s);
  DBuf<i64> deg;
  deg.alloc((i64)n + 1, s);
  deg.zero(s);
  k_key_flags<<<G(nk), 256, 0, s>>>(sorted, nk, n, keep.p, deg.p);
  count_launch();
  // compact the kept keys into the spare buffer
  DBuf<i64> nsel;
  nsel.alloc(1, s);
  tb = 0;
  CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tb, sorted, keep.p, spare, nsel.p, nk, s));
  {
    DBuf<uint8_t> tmp;
    tmp.alloc((i64)tb, s);
    CUDA_CHECK(cub::DeviceSelect::Flagged(tmp.p, tb, sorted, keep.p, spare, nsel.p, nk, s));
  }
  count_launch();
  i64 nnz = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nnz, nsel.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  k_key_cols<<<G(nnz), 256, 0, s>>>(spare, nnz, n, col);
  count_launch();
  deg_to_rowptr(deg.p, (i64)n, rowptr, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  return nnz;
}

int key_bits_for(u64 n) {
  int b = 0;
  while (b < 64 && (n * n - 1) >> b) b++;
  return b;
}

}  // namespace
}  // namespace chroma

using namespace chroma;

extern "C" {

int chroma_gen_rmat(int32_t scale, int64_t edge_factor, uint64_t seed, uint32_t t_a, uint32_t t_ab,
                    uint32_t t_abc, int permute, int device, int64_t* rowptr, int64_t* col, int64_t* nnz_out) {
  try {
    CHROMA_REQUIRE(scale >= 1 && scale <= 30, CHROMA_EVALUE, "R-MAT scale must be in [1, 30]");
    CHROMA_REQUIRE(edge_factor >= 1, CHROMA_EVALUE, "edge factor must be >= 1");
    CUDA_CHECK(cudaSetDevice(device));
    retain_pool_memory(device);
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const u64 n = 1ull << scale;
    const i64 m = edge_factor << scale;
    {
      DBuf<u64> keys;
      keys.alloc(2 * m, s);
      k_rmat_keys<<<G(m), 256, 0, s>>>(seed, scale, m, t_a, t_ab, t_abc, make_perm(seed, scale, permute != 0),
                                       keys.p);
      count_launch();
      *nnz_out = keys_to_csr(keys, 2 * m, n, key_bits_for(n), rowptr, col, s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    return CHROMA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CHROMA_ECUDA;
  }
}

int chroma_gen_random_bipartite(int64_t rows, int64_t nnz_per_row, uint64_t seed, int device, int64_t* rowptr,
                                int64_t* col, int64_t* nnz_out) {
  try {
    CHROMA_REQUIRE(rows >= 1 && rows <= ((i64)1 << 29), CHROMA_EVALUE, "rows must be in [1, 2^29]");
    CHROMA_REQUIRE(nnz_per_row >= 0, CHROMA_EVALUE, "nnz_per_row must be >= 0");
    CUDA_CHECK(cudaSetDevice(device));
    retain_pool_memory(device);
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const u64 n = 2 * (u64)rows;
    const i64 m = rows * nnz_per_row;
    {
      DBuf<u64> keys;
      keys.alloc(std::max<i64>(2 * m, 1), s);
      if (m) k_bip_keys<<<G(m), 256, 0, s>>>(seed, rows, nnz_per_row, keys.p);
      count_launch();
      *nnz_out = keys_to_csr(keys, 2 * m, n, key_bits_for(n), rowptr, col, s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    return CHROMA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CHROMA_ECUDA;
  }
}

// kind 0: gen_hex_mesh(nx, ny, nz) (chroma/graph.py:320-341); kind 1: 27-point
// stencil on nx*ny*nz (BASELINE C2).  rowptr: n+1, col: nnz (call with col NULL to
// get *nnz_out first).
int chroma_gen_box(int32_t kind, int64_t nx, int64_t ny, int64_t nz, int device, int64_t* rowptr, int64_t* col,
                   int64_t* nnz_out) {
  try {
    CHROMA_REQUIRE(kind == 0 || kind == 1, CHROMA_EVALUE, "box kind must be 0 (hex) or 1 (27-point)");
    CHROMA_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, CHROMA_EVALUE, "mesh dimensions must be >= 1");
    CHROMA_REQUIRE(nx * ny * nz < ((i64)1 << 31), CHROMA_EVALUE, "mesh dimensions overflow supported size");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const i64 n = nx * ny * nz;
    const Box b{nx, ny, nz, kind};
    {
      DBuf<i64> deg;
      deg.alloc(n, s);
      k_box_deg<<<G(n), 256, 0, s>>>(b, n, deg.p);
      count_launch();
      deg_to_rowptr(deg.p, n, rowptr, s);
      CUDA_CHECK(cudaMemcpyAsync(nnz_out, rowptr + n, sizeof(i64), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      if (col) {
        k_box_fill<<<G(n), 256, 0, s>>>(b, n, rowptr, col);
        count_launch();
      }
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    return CHROMA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CHROMA_ECUDA;
  }
}

}  // extern "C"
