// tma_probe2.cu — GPU probe of bulk tensor stores into SoA planes at arbitrary start rows,
// with a plain 2-D tensor map (the round-1 probe, scripts/tma_probe.cu,
// used an aliased 3-D map whose dim-2 stride overlapped dim 0, so its illegal instruction did
// not isolate the start-row question).  Not part of the library.
//   map: dims {n rows, P planes}, stride {ld * 4 B}; box {B rows, P planes};
//   shared source [P][B] floats, 128-byte aligned; store at global (x0, 0).
// For each box height B (multiple of 4: the inner box extent must be 16 bytes) and start row
// x0 (aligned and not), the probe checks the B x P stored values and that nothing else
// changed, then times K back-to-back stores of 32-row boxes against the same rows written
// by per-lane 4-byte stores.
// Result on B200 (driver 580, profiles/r02_tma_probe.txt): stores AND loads are correct at
// start rows whose byte offset is a multiple of 16 (x0 = 0, 4, 12) and raise "illegal
// instruction" at every other start row (x0 = 1, 2, 3, 37), for boxes of 4 and 32 rows —
// with a clean 2-D map the round-1 conclusion stands: a warp's compacted rows start at
// arbitrary rows, so a tile store would need per-row head/tail stores around 16-byte-aligned
// boxes, and the staged rows transposed to plane-major order first.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/tma_probe2.cu -o build/tma_probe2 -lcuda
// Run one case: build/tma_probe2 <box rows> <start row> <0 store | 1 load>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int P = 4;

__global__ void probe(const __grid_constant__ CUtensorMap map, int x0, int B) {
  extern __shared__ __align__(1024) float sm[];
  for (int i = threadIdx.x; i < P * B; i += blockDim.x) {
    const int c = i / B, r = i % B;
    sm[i] = (float)(c * 100000 + r);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(sm);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map), "r"(a),
                 "r"(x0), "r"(0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}

// the same box, loaded (global -> shared) at (x0, 0) and written back by the threads
__global__ void probe_load(const __grid_constant__ CUtensorMap map, int x0, int B, float* check) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned ba = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(sm);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(P * B * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(a), "l"(&map), "r"(ba), "r"(x0), "r"(0) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}"
               ::"r"(ba) : "memory");
  for (int i = threadIdx.x; i < P * B; i += blockDim.x) check[i] = sm[i];
}

// timing: every block stores `reps` boxes of 32 rows x P planes at rows base + 32 j + skew
__global__ void store_tma(const __grid_constant__ CUtensorMap map, int reps, int skew) {
  extern __shared__ __align__(1024) float sm[];
  for (int i = threadIdx.x; i < P * 32; i += blockDim.x) sm[i] = (float)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(sm);
    for (int j = 0; j < reps; ++j) {
      const int x = (blockIdx.x * reps + j) * 32 + skew;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map), "r"(a),
                   "r"(x), "r"(0)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void store_plain(float* out, long ld, int reps, int skew) {  // one warp per block, as the copy-out
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < reps; ++j) {
    const long x = (long)(blockIdx.x * reps + j) * 32 + skew + lane;
#pragma unroll
    for (int c = 0; c < P; ++c) out[c * ld + x] = (float)(c * 32 + lane);
  }
}

int one_case(int B, int x0, int load);

int main(int argc, char** argv) {
  if (argc == 4) return one_case(atoi(argv[1]), atoi(argv[2]), atoi(argv[3]));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const long ld = 1 << 16, n = 50000;
  float* d;
  CK(cudaMalloc(&d, sizeof(float) * ld * P));
  std::vector<float> h(ld * P);
  int bad_total = 0;
  for (int B : {4, 8, 32, 128}) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)P};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)B, P};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("B=%d encode 2-D {rows, planes}, stride ld*4: %d\n", B, (int)r);
    if (r != CUDA_SUCCESS) {
      bad_total++;
      continue;
    }
    for (int x0 : {0, 1, 2, 3, 37, 4093, 12345, (int)n - B + 1}) {
      CK(cudaMemset(d, 0xFF, sizeof(float) * ld * P));
      probe<<<1, 128, P * B * 4 + 1024>>>(map, x0, B);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("  B=%d x0=%d: launch error %s\n", B, x0, cudaGetErrorString(e));
        return 2;
      }
      CK(cudaMemcpy(h.data(), d, sizeof(float) * ld * P, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int c = 0; c < P; ++c)
        for (long x = 0; x < ld; ++x) {
          const float v = h[c * ld + x];
          const long rel = x - x0;
          const bool in = rel >= 0 && rel < B && x < n;  // rows past n are out of the map: not stored
          uint32_t bits;
          std::memcpy(&bits, &v, 4);
          if (in ? (v != (float)(c * 100000 + rel)) : (bits != 0xFFFFFFFFu)) bad++;
        }
      printf("  B=%d x0=%d: %s (%d bad)\n", B, x0, bad ? "WRONG" : "ok", bad);
      bad_total += bad != 0;
    }
  }
  // timing: 148 x 4 blocks, each 64 boxes of 32 rows (= 1.2M rows x 4 planes)
  {
    const int blocks = 148 * 4, reps = 64;
    const long rows = (long)blocks * reps * 32 + 64;
    float* o;
    CK(cudaMalloc(&o, sizeof(float) * rows * P));
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)P};
    const cuuint64_t strides[1] = {(cuuint64_t)rows * 4};
    const cuuint32_t box[2] = {32, P};
    const cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, o, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int skew : {0, 1}) {
      float ms_t = 0, ms_p = 0;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        store_tma<<<blocks, 32, P * 32 * 4 + 1024>>>(map, reps, skew);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms_t, a, b);
        cudaEventRecord(a);
        store_plain<<<blocks, 32>>>(o, rows, reps, skew);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms_p, a, b);
      }
      const double bytes = (double)blocks * reps * 32 * P * 4;
      printf("timing skew %d: tma %.3f ms (%.0f GB/s), per-lane stores %.3f ms (%.0f GB/s)\n", skew, ms_t,
             bytes / ms_t / 1e6, ms_p, bytes / ms_p / 1e6);
    }
  }
  printf("probe %s\n", bad_total ? "FAILED" : "passed");
  return bad_total ? 1 : 0;
}

// one probe case in its own process (an illegal instruction is sticky): B rows, start x0,
// load (1) or store (0); prints ok / WRONG / the launch error
int one_case(int B, int x0, int load) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const long ld = 1 << 16, n = 50000;
  float *d, *chk;
  CK(cudaMalloc(&d, sizeof(float) * ld * P));
  CK(cudaMalloc(&chk, sizeof(float) * P * B));
  std::vector<float> h(ld * P);
  for (int c = 0; c < P; ++c)
    for (long x = 0; x < ld; ++x) h[c * ld + x] = (float)(c * 100000 + x);
  CK(cudaMemcpy(d, h.data(), sizeof(float) * ld * P, cudaMemcpyHostToDevice));
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)P};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)B, P};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("%s B=%d x0=%d: encode error %d\n", load ? "load" : "store", B, x0, (int)r);
    return 1;
  }
  if (load) {
    probe_load<<<1, 128, P * B * 4 + 1024>>>(map, x0, B, chk);
  } else {
    CK(cudaMemset(d, 0xFF, sizeof(float) * ld * P));
    probe<<<1, 128, P * B * 4 + 1024>>>(map, x0, B);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s B=%d x0=%d (start byte offset %d mod 16): %s\n", load ? "load" : "store", B, x0, (x0 * 4) % 16,
           cudaGetErrorString(e));
    return 2;
  }
  int bad = 0;
  if (load) {
    std::vector<float> c(P * B);
    CK(cudaMemcpy(c.data(), chk, sizeof(float) * P * B, cudaMemcpyDeviceToHost));
    for (int cc = 0; cc < P; ++cc)
      for (int rr = 0; rr < B; ++rr)
        if (c[cc * B + rr] != (float)(cc * 100000 + x0 + rr)) bad++;
  } else {
    CK(cudaMemcpy(h.data(), d, sizeof(float) * ld * P, cudaMemcpyDeviceToHost));
    for (int c = 0; c < P; ++c)
      for (long x = 0; x < ld; ++x) {
        const float v = h[c * ld + x];
        const long rel = x - x0;
        const bool in = rel >= 0 && rel < B && x < n;
        uint32_t bits;
        std::memcpy(&bits, &v, 4);
        if (in ? (v != (float)(c * 100000 + rel)) : (bits != 0xFFFFFFFFu)) bad++;
      }
  }
  printf("%s B=%d x0=%d (start byte offset %d mod 16): %s (%d bad)\n", load ? "load" : "store", B, x0, (x0 * 4) % 16,
         bad ? "WRONG" : "ok", bad);
  return bad ? 1 : 0;
}
