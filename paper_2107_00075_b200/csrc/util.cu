// Small device utilities: fills, scatters, ordered compaction, scans.
#include <atomic>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "kernels.cuh"

namespace chroma {

static std::atomic<long long> g_launches{0};
void count_launch(int k) { g_launches += k; }
i64 launch_count() { return (i64)g_launches.load(); }

// Keep freed stream-ordered allocations in the device pool instead of returning
// them to the driver: worlds are rebuilt per call in the e2e path and the default
// release threshold (0) made every rebuild pay the page-mapping cost again.
void retain_pool_memory(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  done[device] = true;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

namespace {
__global__ void k_fill(i32* p, i64 n, i32 v) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_iota(i32* p, i64 n, i32 base) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    p[i] = base + (i32)i;
}
__global__ void k_scatter_const(i32* val, const i32* idx, const i64* n_dev, i32 v) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    val[idx[i]] = v;
}
__global__ void k_scatter_from(i32* dst, const i32* src, const i32* idx, const i64* n_dev) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 x = idx[i];
    dst[x] = src[x];
  }
}
__global__ void k_scatter_values(i32* dst, const i32* idx, const i32* values, const i64* n_dev) {
  const i64 n = *n_dev;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    dst[idx[i]] = values[i];
}
__global__ void k_clamp(i32* dst, const i32* src, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i32 c = src[i];
    dst[i] = c < 0 ? 0 : c;
  }
}
}  // namespace

static int ew_grid(i64 n) { return grid_for(n, 256, num_sms() * 16); }

void launch_fill_i32(i32* p, i64 n, i32 v, cudaStream_t s) {
  if (n <= 0) return;
  k_fill<<<ew_grid(n), 256, 0, s>>>(p, n, v);
  count_launch();
}
void launch_iota_i32(i32* p, i64 n, i32 base, cudaStream_t s) {
  if (n <= 0) return;
  k_iota<<<ew_grid(n), 256, 0, s>>>(p, n, base);
  count_launch();
}
void launch_scatter_const(i32* val, const i32* idx, const i64* n_dev, i64 n_max, i32 v, cudaStream_t s) {
  if (n_max <= 0) return;
  k_scatter_const<<<ew_grid(n_max), 256, 0, s>>>(val, idx, n_dev, v);
  count_launch();
}
void launch_scatter_from(i32* dst, const i32* src, const i32* idx, const i64* n_dev, i64 n_max,
                         cudaStream_t s) {
  if (n_max <= 0) return;
  k_scatter_from<<<ew_grid(n_max), 256, 0, s>>>(dst, src, idx, n_dev);
  count_launch();
}
void launch_scatter_idx_values(i32* dst, const i32* idx, const i32* values, const i64* n_dev,
                               i64 n_max, cudaStream_t s) {
  if (n_max <= 0) return;
  k_scatter_values<<<ew_grid(n_max), 256, 0, s>>>(dst, idx, values, n_dev);
  count_launch();
}
void launch_clamp_nonneg(i32* dst, const i32* src, i64 n, cudaStream_t s) {
  if (n <= 0) return;
  k_clamp<<<ew_grid(n), 256, 0, s>>>(dst, src, n);
  count_launch();
}

// Scratch (grow-only, per host thread AND device -- one process may drive several
// GPUs from a thread pool; intentionally never destroyed so no free runs after the
// CUDA context is gone).
template <typename T>
static DBuf<T>& per_device_scratch(DBuf<T>* (&slots)[64]) {
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) d = 0;
  if (!slots[d]) slots[d] = new DBuf<T>();
  return *slots[d];
}
static DBuf<uint8_t>& cub_tmp() {
  static thread_local DBuf<uint8_t>* b[64] = {};
  return per_device_scratch(b);
}
#define t_cub_tmp cub_tmp()

void select_flagged(const uint8_t* flags, i64 n, i32* out, i64* n_out, cudaStream_t s) {
  if (n <= 0) {
    CUDA_CHECK(cudaMemsetAsync(n_out, 0, sizeof(i64), s));
    return;
  }
  thrust::counting_iterator<i32> it(0);
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, n_out, n, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceSelect::Flagged(t_cub_tmp.p, bytes, it, flags, out, n_out, n, s));
  count_launch();
}

void select_flagged_base(const uint8_t* flags, i64 n, i32 base, i32* out, i64* n_out, cudaStream_t s) {
  if (n <= 0) {
    CUDA_CHECK(cudaMemsetAsync(n_out, 0, sizeof(i64), s));
    return;
  }
  thrust::counting_iterator<i32> it(base);
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, n_out, n, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceSelect::Flagged(t_cub_tmp.p, bytes, it, flags, out, n_out, n, s));
  count_launch();
}

void select_flagged_values(const i32* values, const uint8_t* flags, i64 n, i32* out, i64* n_out,
                           cudaStream_t s) {
  if (n <= 0) {
    CUDA_CHECK(cudaMemsetAsync(n_out, 0, sizeof(i64), s));
    return;
  }
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, values, flags, out, n_out, n, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceSelect::Flagged(t_cub_tmp.p, bytes, values, flags, out, n_out, n, s));
  count_launch();
}

void sort_i32(i32* keys, i64 n, cudaStream_t s) {
  if (n <= 1) return;
  static thread_local DBuf<i32>* alts[64] = {};
  DBuf<i32>* alt = &per_device_scratch(alts);
  alt->reserve(n, s);
  cub::DoubleBuffer<i32> db(keys, alt->p);
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, (int)n, 0, 32, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(t_cub_tmp.p, bytes, db, (int)n, 0, 32, s));
  count_launch();
  if (db.Current() != keys)
    CUDA_CHECK(cudaMemcpyAsync(keys, db.Current(), sizeof(i32) * n, cudaMemcpyDeviceToDevice, s));
}

void sort_u64(u64* keys, i64 n, cudaStream_t s) {
  if (n <= 1) return;
  static thread_local DBuf<u64>* alts[64] = {};
  DBuf<u64>* alt = &per_device_scratch(alts);
  alt->reserve(n, s);
  cub::DoubleBuffer<u64> db(keys, alt->p);
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, (int)n, 0, 64, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(t_cub_tmp.p, bytes, db, (int)n, 0, 64, s));
  count_launch();
  if (db.Current() != keys)
    CUDA_CHECK(cudaMemcpyAsync(keys, db.Current(), sizeof(u64) * n, cudaMemcpyDeviceToDevice, s));
}

namespace {
__global__ void k_narrow_checked(const i64* in, i32* out, i64 k, i64 n, unsigned* bad) {
  unsigned b = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < k; i += (i64)gridDim.x * blockDim.x) {
    const i64 x = in[i];
    b |= (x < 0 || x >= n) ? 1u : 0u;
    out[i] = (i32)x;
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}
}  // namespace

// int64 ids in [0, n) (host or device) -> int32 device array; ValueError (with
// `what`) if any id is out of range.  Host sources cross PCIe in 512 MB chunks.
void narrow_ids_checked(const i64* src, i64 k, i64 n, bool src_on_device, i32* out, cudaStream_t s,
                        const char* what) {
  if (k <= 0) return;
  if (!src_on_device && staged_upload_wanted(k * (i64)sizeof(i64))) {
    upload_narrow_host(src, k, n, out, s, what);
    return;
  }
  DBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  if (src_on_device) {
    k_narrow_checked<<<ew_grid(k), 256, 0, s>>>(src, out, k, n, bad.p);
    count_launch();
  } else {
    const i64 CH = (i64)1 << 26;
    DBuf<i64> tmp;
    tmp.alloc(std::min(k, CH), s);
    for (i64 b = 0; b < k; b += CH) {
      const i64 c = std::min(CH, k - b);
      CUDA_CHECK(cudaMemcpyAsync(tmp.p, src + b, sizeof(i64) * c, cudaMemcpyHostToDevice, s));
      k_narrow_checked<<<ew_grid(c), 256, 0, s>>>(tmp.p, out + b, c, n, bad.p);
      count_launch();
    }
  }
  unsigned hb = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  CHROMA_REQUIRE(hb == 0, CHROMA_EVALUE, what);
}

// distinct sorted keys of in[0..n) -> out; returns the count (one sync)
i64 unique_u64(const u64* in, i64 n, u64* out, cudaStream_t s) {
  if (n <= 0) return 0;
  static thread_local DBuf<i64>* cnts[64] = {};
  DBuf<i64>& c = per_device_scratch(cnts);
  c.reserve(1, s);
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, bytes, in, out, c.p, n, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceSelect::Unique(t_cub_tmp.p, bytes, in, out, c.p, n, s));
  count_launch();
  i64 k = 0;
  CUDA_CHECK(cudaMemcpyAsync(&k, c.p, sizeof(i64), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  return k;
}

void exclusive_scan_i64(const i64* in, i64* out, i64 n, cudaStream_t s) {
  if (n <= 0) return;
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
  t_cub_tmp.reserve((i64)bytes, s);
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t_cub_tmp.p, bytes, in, out, n, s));
  count_launch();
}

}  // namespace chroma
