// Shared definitions for libchroma_b200: status handling, device buffers, the
// hashed-GID loser rule (chroma/protocol.py:79-133) and small warp helpers.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <stdexcept>
#include <cuda_runtime.h>

#include "../../include/chroma_b200.h"

namespace chroma {

using i64 = int64_t;
using i32 = int32_t;
using u32 = uint32_t;
using u64 = uint64_t;

// A worklist vertex that has not committed its colour yet.  Colours are >= 0
// everywhere else, so a single compare distinguishes "pending" from "final".
constexpr i32 PENDING = -1;
// "never sent" sentinel of the changed-only exchange (chroma/runtime.py:287)
constexpr i32 NEVER_SENT = INT32_MIN;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define CUDA_CHECK(expr)                                                                    \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw ::chroma::Error(CHROMA_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                              " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define CHROMA_REQUIRE(cond, code, msg)                 \
  do {                                                  \
    if (!(cond)) throw ::chroma::Error((code), (msg));  \
  } while (0)

// Owning device buffer (stream-ordered allocation).
template <typename T>
struct DBuf {
  T* p = nullptr;
  i64 n = 0;
  cudaStream_t s = nullptr;
  bool borrowed = false;  // p belongs to someone else (e.g. an IPC-shared region)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; borrowed = o.borrowed;
      o.p = nullptr; o.n = 0; o.borrowed = false;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p && !borrowed) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    borrowed = false;
  }
  void borrow(T* ptr, i64 count) {
    release();
    p = ptr;
    n = count;
    borrowed = true;
  }
  void alloc(i64 count, cudaStream_t stream) {
    // free on the caller's (live) stream: a shared scratch may outlive the stream
    // it was first allocated on
    if (p && !borrowed) cudaFreeAsync(p, stream);
    p = nullptr;
    n = 0;
    borrowed = false;
    s = stream;
    n = count;
    if (count > 0) CUDA_CHECK(cudaMallocAsync(&p, sizeof(T) * (size_t)count, stream));
  }
  // grow-only scratch
  void reserve(i64 count, cudaStream_t stream) {
    if (count > n || !p) alloc(count > 0 ? count : 1, stream);
  }
  void zero(cudaStream_t stream) {
    if (n) CUDA_CHECK(cudaMemsetAsync(p, 0, sizeof(T) * (size_t)n, stream));
  }
  void upload(const T* h, i64 count, cudaStream_t stream) {
    alloc(count, stream);
    if (count) CUDA_CHECK(cudaMemcpyAsync(p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, stream));
  }
};

// ------------------------------------------------------------------ hashing
// chroma/protocol.py:79-88: splitmix64 finaliser of gid + golden gamma.
__host__ __device__ __forceinline__ u64 gid_rand(i64 gid) {
  u64 z = (u64)gid + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// chroma/protocol.py:99-133: which endpoint of an equal-coloured pair is uncoloured.
// Returns true when v loses.  (gv == gu is rejected by the callers' validation.)
__host__ __device__ __forceinline__ bool v_loses(i64 gv, i64 gu, i64 dv, i64 du, bool recolor_degrees) {
  if (recolor_degrees && dv != du) return dv < du;
  u64 hv = gid_rand(gv), hu = gid_rand(gu);
  if (hv != hu) return hv > hu;
  return gv > gu;
}

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ i32 ld_relaxed(const i32* p) {
  i32 v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// same load without the compiler memory barrier: independent loads around it may be
// batched (speculative gathers, where the value is only a hint until resolution)
__device__ __forceinline__ i32 ld_relaxed_nb(const i32* p) {
  i32 v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// streaming (evict-first) load of a CSR column entry: keeps the gathered colours in L2
__device__ __forceinline__ i32 ld_stream(const i32* p) { return __ldcs(p); }
__device__ __forceinline__ void st_relaxed(i32* p, i32 v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

inline int grid_for(i64 work, int block, int max_blocks) {
  i64 g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

int num_sms();

}  // namespace chroma
