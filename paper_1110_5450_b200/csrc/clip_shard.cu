// clip_shard.cu — K4: global output offsets of the sharded compacting clip.
//
// After the per-rank visible counts c_r have been allgathered (NCCL over NVLink, see
// paper_1110_5450_b200/shard.py), rank r's compacted rows start at the exclusive prefix
// sum_{r' < r} c_r'; the total is sum_r c_r.  One warp; P is the world size.
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

int device_sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    cached[dev] = sms;
  }
  return cached[dev];
}

}  // namespace clipseg
