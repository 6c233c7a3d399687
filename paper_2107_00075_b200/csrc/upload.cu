// Host -> device upload of the caller's CSR through a pinned staging ring.
//
// The reference's inputs are NumPy arrays (chroma/graph.py:24-60: int64 row_offsets and
// col_indices), i.e. pageable host memory.  cudaMemcpy from pageable memory goes through
// the driver's own bounce buffer at ~11 GB/s (C3: 4.2 GB of int64 columns in 380 ms).
// Here a few host threads each take every T-th chunk of the array, narrow it (int64 ids
// -> int32, range-checked) or copy it into one of their two pinned staging slots, and
// issue the DMA from the slot on their own stream while they fill the other slot: the
// copy runs at host-memory speed on T cores, the link carries half the bytes for
// columns, and pageable and pinned sources cost the same.
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"

namespace chroma {
namespace {

constexpr i64 STAGE_BYTES = (i64)4 << 20;  // per slot
constexpr int MAX_THREADS = 16;
constexpr int MAX_DEV = 64;

int upload_threads() {
  static const int t = [] {
    if (const char* e = std::getenv("CHROMA_UPLOAD_THREADS")) return std::max(1, std::min(MAX_THREADS, std::atoi(e)));
    cpu_set_t cs;
    int n = 0;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) n = CPU_COUNT(&cs);
    if (n <= 0) n = (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(MAX_THREADS, n));
  }();
  return t;
}

// per device (ranks of a one-process multi-GPU world upload concurrently)
struct Ring {
  std::mutex mu;            // one staged upload at a time per device
  std::vector<char*> slot;  // 2 per thread, pinned
  cudaStream_t st[MAX_THREADS] = {};
  cudaEvent_t ev[2 * MAX_THREADS] = {};
  cudaEvent_t start = nullptr;
};
Ring& ring(int dev) {
  static Ring* r[MAX_DEV] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (!r[dev]) r[dev] = new Ring;  // process lifetime (pinned memory is released at exit)
  return *r[dev];
}

// fill(dst_slot, first item, count) -> false if an item is out of range
template <class Fill>
void staged_h2d(i64 items, i64 out_elem, Fill fill, char* dst, cudaStream_t s) {
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  CHROMA_REQUIRE(dev >= 0 && dev < MAX_DEV, CHROMA_EVALUE, "device ordinal out of range");
  const int T = upload_threads();
  const i64 chunk = STAGE_BYTES / out_elem;
  const i64 nch = (items + chunk - 1) / chunk;
  const int nt = (int)std::min<i64>(T, nch);
  Ring& R = ring(dev);
  std::lock_guard<std::mutex> lk(R.mu);
  while ((int)R.slot.size() < 2 * nt) {
    void* p = nullptr;
    CUDA_CHECK(cudaHostAlloc(&p, STAGE_BYTES, cudaHostAllocDefault));
    R.slot.push_back((char*)p);
  }
  for (int t = 0; t < nt; t++) {
    if (!R.st[t]) CUDA_CHECK(cudaStreamCreateWithFlags(&R.st[t], cudaStreamNonBlocking));
    for (int k = 0; k < 2; k++)
      if (!R.ev[2 * t + k]) CUDA_CHECK(cudaEventCreateWithFlags(&R.ev[2 * t + k], cudaEventDisableTiming));
  }
  if (!R.start) CUDA_CHECK(cudaEventCreateWithFlags(&R.start, cudaEventDisableTiming));
  // the destination was allocated (stream-ordered) on s: copies start after that
  CUDA_CHECK(cudaEventRecord(R.start, s));
  std::atomic<bool> bad{false};
  std::atomic<int> failed{0};
  std::string err;
  std::mutex err_mu;
  auto work = [&](int t) {
    try {
      CUDA_CHECK(cudaSetDevice(dev));
      cudaStream_t ts = R.st[t];
      CUDA_CHECK(cudaStreamWaitEvent(ts, R.start, 0));
      int use = 0;
      for (i64 c = t; c < nch; c += nt, use++) {
        const int k = 2 * t + (use & 1);
        if (use >= 2) CUDA_CHECK(cudaEventSynchronize(R.ev[k]));  // the slot's last DMA is done
        const i64 b = c * chunk, cnt = std::min(chunk, items - b);
        if (!fill(R.slot[k], b, cnt)) bad.store(true, std::memory_order_relaxed);
        CUDA_CHECK(cudaMemcpyAsync(dst + b * out_elem, R.slot[k], (size_t)(cnt * out_elem), cudaMemcpyHostToDevice, ts));
        CUDA_CHECK(cudaEventRecord(R.ev[k], ts));
      }
      CUDA_CHECK(cudaStreamSynchronize(ts));
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> g(err_mu);
      if (!failed.fetch_add(1)) err = e.what();
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; t++) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  if (failed.load()) throw Error(CHROMA_ECUDA, "staged upload: " + err);
  if (bad.load()) throw Error(CHROMA_EVALUE, "");  // the caller words it
}

// int64 ids -> int32 with a range check, scalar; true iff every id is in [0, n)
bool narrow_scalar(const i64* x, i32* o, i64 cnt, i64 n) {
  unsigned long long any = 0;
  for (i64 i = 0; i < cnt; i++) {
    any |= (unsigned long long)x[i] >= (unsigned long long)n;
    o[i] = (i32)x[i];
  }
  return any == 0;
}

// the same, 8 ids per step; streaming stores into the staging slot (no read for
// ownership: the slot is only read again by the DMA engine).  o is 32-byte aligned.
__attribute__((target("avx2"))) bool narrow_avx2(const i64* x, i32* o, i64 cnt, i64 n) {
  const __m256i sign = _mm256_set1_epi64x(INT64_MIN);
  const __m256i lim = _mm256_set1_epi64x(n ^ INT64_MIN);  // unsigned x < n <=> (x^sign) < (n^sign)
  const __m256i lo = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i ok = _mm256_set1_epi64x(-1);
  i64 i = 0;
  for (; i + 8 <= cnt; i += 8) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)(x + i));
    const __m256i b = _mm256_loadu_si256((const __m256i*)(x + i + 4));
    ok = _mm256_and_si256(ok, _mm256_and_si256(_mm256_cmpgt_epi64(lim, _mm256_xor_si256(a, sign)),
                                               _mm256_cmpgt_epi64(lim, _mm256_xor_si256(b, sign))));
    const __m256i pa = _mm256_permutevar8x32_epi32(a, lo), pb = _mm256_permutevar8x32_epi32(b, lo);
    _mm256_stream_si256((__m256i*)(o + i), _mm256_permute2x128_si256(pa, pb, 0x20));
  }
  _mm_sfence();
  return _mm256_movemask_epi8(ok) == -1 && narrow_scalar(x + i, o + i, cnt - i, n);
}

const bool have_avx2 = __builtin_cpu_supports("avx2");

}  // namespace

bool staged_upload_wanted(i64 bytes) {
  static const bool off = [] {
    const char* e = std::getenv("CHROMA_UPLOAD");
    return e && std::string(e) == "direct";
  }();
  return !off && bytes >= 4 * STAGE_BYTES;
}

void upload_narrow_host(const i64* src, i64 k, i64 n, i32* out, cudaStream_t s, const char* what) {
  auto narrow = [src, n](char* slot, i64 b, i64 cnt) {
    return have_avx2 ? narrow_avx2(src + b, (i32*)slot, cnt, n) : narrow_scalar(src + b, (i32*)slot, cnt, n);
  };
  try {
    staged_h2d(k, sizeof(i32), narrow, (char*)out, s);
  } catch (const Error& e) {
    if (e.code == CHROMA_EVALUE && std::string(e.what()).empty()) throw Error(CHROMA_EVALUE, what);
    throw;
  }
}

void upload_bytes_host(const void* src, i64 bytes, void* out, cudaStream_t s) {
  const char* h = (const char*)src;
  auto copy = [h](char* slot, i64 b, i64 cnt) {
    std::memcpy(slot, h + b, (size_t)cnt);
    return true;
  };
  staged_h2d(bytes, 1, copy, (char*)out, s);
}

}  // namespace chroma
