// clip_shard.cu — K4: global output offsets of the sharded compacting clip.
//
// After the per-rank visible counts c_r have been allgathered (NCCL over NVLink, see
// paper_1110_5450_b200/shard.py), rank r's compacted rows start at the exclusive prefix
// sum_{r' < r} c_r'; the total is sum_r c_r.  One warp; P is the world size.
#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "clip_kernels.cuh"

namespace clipseg {

__global__ void shard_offsets_kernel(const int64_t* __restrict__ counts, int P, int rank, int64_t* __restrict__ offset,
                                     int64_t* __restrict__ total) {
  const int lane = threadIdx.x;
  long long before = 0, all = 0;
  for (int r = lane; r < P; r += 32) {
    const long long c = counts[r];
    all += c;
    before += (r < rank) ? c : 0;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    all += __shfl_xor_sync(0xFFFFFFFFu, all, d);
    before += __shfl_xor_sync(0xFFFFFFFFu, before, d);
  }
  if (lane == 0) {
    *offset = before;
    *total = all;
  }
}

cudaError_t launch_shard_offsets(const int64_t* d_counts, int P, int rank, int64_t* d_offset, int64_t* d_total,
                                 cudaStream_t s) {
  shard_offsets_kernel<<<1, 32, 0, s>>>(d_counts, P, rank, d_offset, d_total);
  return cudaGetLastError();
}

// Per-device launch state.  Function attributes and occupancy belong to a device (context),
// so both caches are keyed by the current device; a racing first use on two host threads
// computes and stores the same values (relaxed atomics, idempotent attribute writes).
namespace {
constexpr int kMaxDevices = 64;
std::atomic<int> g_sm_count[kMaxDevices];
std::mutex g_occ_mu;
std::map<std::pair<const void*, int>, int> g_occ;  // (kernel, device) -> resident blocks per SM
}  // namespace

int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  int sms = g_sm_count[dev].load(std::memory_order_relaxed);
  if (!sms) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    g_sm_count[dev].store(sms, std::memory_order_relaxed);
  }
  return sms;
}

cudaError_t kernel_occupancy(const void* kern, int threads, size_t smem, int* blocks_per_sm) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(kern, dev);
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    const auto it = g_occ.find(key);
    if (it != g_occ.end()) {
      *blocks_per_sm = it->second;
      return cudaSuccess;
    }
  }
  if (smem > 48 * 1024 &&
      (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  int b = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem)) != cudaSuccess) return e;
  if (b < 1) return cudaErrorInvalidConfiguration;  // the kernel cannot be resident at all
  std::lock_guard<std::mutex> g(g_occ_mu);
  g_occ[key] = b;
  *blocks_per_sm = b;
  return cudaSuccess;
}

}  // namespace clipseg
