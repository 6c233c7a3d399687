// Gather roofline of this B200: the rate at which an SM retires random element loads
// (one L1TEX wavefront per distinct 128-byte line a warp instruction touches), next to
// the streaming read bandwidth.  The colouring, detection and checker kernels are
// bound by the former (one random neighbour-colour load per CSR entry), not by HBM
// bytes; bench.py reports their time against both.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_roofline gather_roofline.cu
//   ./gather_roofline            -> one JSON line
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// PER independent random loads per thread per step, indices hashed (no index stream)
template <typename T, int PER>
__global__ void k_gather(const T* __restrict__ a, uint32_t mask, long long steps, unsigned long long* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (long long s = 0; s < steps; s++) {
    T v[PER];
#pragma unroll
    for (int q = 0; q < PER; q++) v[q] = __ldg(a + (mix(tid * 64u + (uint32_t)s * 4099u + q * 0x9e37u) & mask));
#pragma unroll
    for (int q = 0; q < PER; q++) acc += (uint32_t)v[q];
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_stream(const int4* __restrict__ a, long long n4, unsigned long long* sink) {
  uint32_t acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const int4 w = __ldcs(a + i);
    acc += w.x ^ w.y ^ w.z ^ w.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <typename T>
static int run_gather(const char* name, size_t bytes, int sms, double clk_hz, bool last) {
  T* a;
  unsigned long long* sink;
  const size_t n = bytes / sizeof(T);  // power of two
  CK(cudaMalloc(&a, bytes));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMalloc(&sink, 8));
  const int blocks = sms * 8, threads = 256;
  const long long steps = 64;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_gather<T, 16><<<blocks, threads>>>(a, (uint32_t)(n - 1), 4, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(e0));
    k_gather<T, 16><<<blocks, threads>>>(a, (uint32_t)(n - 1), steps, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double loads = (double)blocks * threads * steps * 16;
  const double rate = loads / (best * 1e-3);
  std::printf("\"%s\": {\"array_MB\": %.0f, \"gathers_per_s\": %.4g, \"per_sm_per_clk_at_max\": %.3f, \"ms\": %.3f}%s",
              name, bytes / 1e6, rate, rate / (sms * clk_hz), best, last ? "" : ", ");
  CK(cudaFree(a));
  CK(cudaFree(sink));
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"max_sm_mhz\": %d, ", p.name, p.multiProcessorCount, clk_khz / 1000);
  // u16 colour copy of C3 (33.5 MB), int32 colours of C3 (67 MB), a 256 MB array (beyond L2)
  if (run_gather<uint16_t>("gather_u16_32MB", 32u << 20, p.multiProcessorCount, clk_khz * 1e3, false)) return 1;
  if (run_gather<int32_t>("gather_i32_64MB", 64u << 20, p.multiProcessorCount, clk_khz * 1e3, false)) return 1;
  if (run_gather<int32_t>("gather_i32_256MB", 256u << 20, p.multiProcessorCount, clk_khz * 1e3, true)) return 1;
  // streaming read of 2 GB (the C3 column array's size)
  int4* s;
  unsigned long long* sink;
  const size_t sb = 2048u << 20;
  CK(cudaMalloc(&s, sb));
  CK(cudaMemset(s, 1, sb));
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_stream<<<p.multiProcessorCount * 8, 256>>>(s, sb / 16, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(e0));
    k_stream<<<p.multiProcessorCount * 8, 256>>>(s, sb / 16, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  std::printf(", \"stream_read_2GB\": {\"GBps\": %.1f, \"ms\": %.3f}}\n", sb / (best * 1e-3) / 1e9, best);
  return 0;
}
