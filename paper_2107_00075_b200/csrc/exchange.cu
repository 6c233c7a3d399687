// Ghost-colour exchange between ranks that live on the same device
// (chroma/runtime.py:271-308).  Every routed owned vertex is one entry with a list
// of destination ghost slots (CSR).  changed_only compares against last_sent
// exactly as the reference does (a vertex is sent iff its colour differs from the
// last broadcast, chroma/runtime.py:287-289); the byte / message accounting counts
// 12 bytes per (vertex, destination) pair sent and one message per non-empty
// (src rank, dst rank) inbox (chroma/runtime.py:294-307).
#include "kernels.cuh"

namespace chroma {
namespace {

// Per-(src, dst) counters are accumulated in shared memory (one global atomic per
// block and pair at the end): global atomics per entry on a handful of addresses
// serialise the whole kernel.
constexpr int SHARED_PAIRS = 4096;

__global__ void k_exchange(const i32* routed, i64 nrouted, const i64* st_off, const i32* st_dst,
                           const i32* st_pair, i32* colors, i32* last_sent, bool changed_only,
                           bool write_all, unsigned long long* pair_cnt, i64 npairs) {
  __shared__ unsigned sc[SHARED_PAIRS];
  const bool local = npairs <= SHARED_PAIRS;
  if (local)
    for (i64 k = threadIdx.x; k < npairs; k += blockDim.x) sc[k] = 0;
  __syncthreads();
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nrouted; i += (i64)gridDim.x * blockDim.x) {
    const i32 c = colors[routed[i]];
    const bool send = !changed_only || last_sent[i] != c;
    if (send) last_sent[i] = c;
    for (i64 t = st_off[i]; t < st_off[i + 1]; t++) {
      if (send || write_all) colors[st_dst[t]] = c;
      if (send) {
        if (local) atomicAdd(&sc[st_pair[t]], 1u);
        else atomicAdd(&pair_cnt[st_pair[t]], 1ull);
      }
    }
  }
  __syncthreads();
  if (local)
    for (i64 k = threadIdx.x; k < npairs; k += blockDim.x)
      if (sc[k]) atomicAdd(&pair_cnt[k], (unsigned long long)sc[k]);
}

// stats2[0] += 12 * pairs sent, stats2[1] += non-empty inboxes; clears pair_cnt
__global__ void k_pair_stats(unsigned long long* pair_cnt, i64 npairs, unsigned long long* stats2) {
  __shared__ unsigned long long b, m;
  if (threadIdx.x == 0) b = m = 0;
  __syncthreads();
  unsigned long long lb = 0, lm = 0;
  for (i64 i = threadIdx.x; i < npairs; i += blockDim.x) {
    const unsigned long long c = pair_cnt[i];
    lb += 12ull * c;
    lm += c ? 1 : 0;
    pair_cnt[i] = 0;
  }
  atomicAdd(&b, lb);
  atomicAdd(&m, lm);
  __syncthreads();
  if (threadIdx.x == 0) {
    stats2[0] += b;
    stats2[1] += m;
  }
}

}  // namespace

void launch_exchange_local(const i32* routed, i64 nrouted, const i64* st_off, const i32* st_dst,
                           const i32* st_pair, i32* colors, i32* last_sent, bool changed_only,
                           bool write_all, unsigned long long* pair_cnt, i64 npairs, cudaStream_t s) {
  if (nrouted <= 0) return;
  k_exchange<<<grid_for(nrouted, 256, num_sms() * 16), 256, 0, s>>>(
      routed, nrouted, st_off, st_dst, st_pair, colors, last_sent, changed_only, write_all, pair_cnt, npairs);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

void launch_pair_stats(unsigned long long* pair_cnt, i64 npairs, unsigned long long* stats2,
                       cudaStream_t s) {
  k_pair_stats<<<1, 256, 0, s>>>(pair_cnt, npairs, stats2);
  count_launch();
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace chroma
