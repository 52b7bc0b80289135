// tof_range.cu — K5 (NEXT-2): the paper's own per-pixel step over batched
// ToF frames: the range clip [r_min, r_max] of PAPER.md §5.2 (closed interval,
// recomputed per frame) as a 2-bit outcode, fused with phi = arctan(d sqrt(I)) of Eq. (5)
// for the kept pixels, plus the kept-pixel count per frame.
//
// HBM-bound map: 8 bytes in (d, I) and 5 out (phi, code) per pixel, 128-bit evict-first
// loads and stores; the per-frame counts are one warp reduction and one atomic per chunk.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "clip_kernels.cuh"

namespace clipseg {

namespace {

// code: 4 invalid (d <= 0, non-finite d or I, I < 0), else bit 0 = d < r_min, bit 1 = d > r_max
__device__ __forceinline__ uint32_t tof_code(float d, float I, float r_min, float r_max) {
  const bool invalid = !(d > 0.0f) || !(fabsf(d) <= FLT_MAX) || !(I >= 0.0f) || !(I <= FLT_MAX);
  return invalid ? 4u : ((uint32_t)(d < r_min) | ((uint32_t)(d > r_max) << 1));
}

// floor(i / ppf) for 0 <= i < 2^52 without a 64-bit integer division: a double-precision
// estimate (inv = 1 / ppf rounded) is off by at most one, fixed by the remainder's sign.
__device__ __forceinline__ int64_t frame_of(int64_t i, int64_t ppf, double inv) {
  int64_t q = (int64_t)((double)i * inv);
  const int64_t r = i - q * ppf;
  q += (r >= ppf) - (r < 0);
  return q;
}

// Eq. (5), phi = arctan(d sqrt(I)), in binary32 with its own error bound (DESIGN.md §13
// T-e/T-f): x = d * sqrt.approx(I); r = x or 1/x (MUFU.RCP + one Newton step) in [0, 1];
// atan(r) = r p(r^2) with a degree-8 minimax polynomial (|error| < 6e-9 on [0, 1], fitted
// by scripts/fit_atan.py); phi = r-branch or pi/2 - atan(1/x).  Measured bound of the whole
// chain (tests/test_gpu_tof.py sweep): < 4e-7 rad, inside the 1e-6 tolerance.  libm's
// atanf / IEEE sqrtf cost ~100 instructions per pixel here (issue-bound); this is ~25.
__device__ __forceinline__ float tof_phi(float d, float I) {
  float s, r0;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(I));
  const float x = __fmul_rn(d, s);
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(x));
  const float e = __fmaf_rn(-x, r0, 1.0f);
  const float inv = x <= FLT_MAX ? __fmaf_rn(r0, e, r0) : 0.0f;  // x = inf: the step would be inf * 0
  const bool big = x > 1.0f;
  const float r = big ? inv : x;
  const float z = __fmul_rn(r, r);
  float p = 0.002456725374445816f;
  p = __fmaf_rn(p, z, -0.014401361538426643f);
  p = __fmaf_rn(p, z, 0.039781230449838625f);
  p = __fmaf_rn(p, z, -0.07234858067414007f);
  p = __fmaf_rn(p, z, 0.10498946486203357f);
  p = __fmaf_rn(p, z, -0.14161229331516054f);
  p = __fmaf_rn(p, z, 0.1998590679144458f);
  p = __fmaf_rn(p, z, -0.3333259703029724f);
  p = __fmaf_rn(p, z, 0.9999998863836149f);
  const float a = __fmul_rn(r, p);
  return big ? __fsub_rn(1.5707963267948966f, a) : a;
}

// A warp owns chunks of kChunk = 32 lanes x kG vectors x 4 pixels; lane l loads vector
// (32 j + l) of the chunk for j < kG, so each 128-bit load instruction is fully coalesced and
// every lane has kG x 8 loads in flight.  A chunk inside one frame (the common case: frames
// are 41616 pixels) costs one frame lookup, one range load, one warp reduction and at most
// one atomic; chunks straddling a frame boundary or the end take a per-pixel path.
constexpr int kG = 4;
constexpr int64_t kChunk = 32 * kG * 4;

__global__ void __launch_bounds__(256) tof_range_phi_kernel(const float* __restrict__ d, const float* __restrict__ I,
                                                            int64_t n, int64_t ppf, const float* __restrict__ ranges,
                                                            float* __restrict__ phi, uint8_t* __restrict__ code,
                                                            int* __restrict__ kept, double inv_ppf) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  for (int64_t ch = warp_id; ch < nchunks; ch += nwarps) {
    const int64_t p0 = ch * kChunk;
    const bool full = p0 + kChunk <= n;
    float dv[kG][4], Iv[kG][4];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int64_t i = p0 + (int64_t)(32 * j + lane) * 4;
      if (full) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(d + i));
        const float4 b = __ldcs(reinterpret_cast<const float4*>(I + i));
        dv[j][0] = a.x; dv[j][1] = a.y; dv[j][2] = a.z; dv[j][3] = a.w;
        Iv[j][0] = b.x; Iv[j][1] = b.y; Iv[j][2] = b.z; Iv[j][3] = b.w;
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          dv[j][v] = i + v < n ? d[i + v] : 0.0f;
          Iv[j][v] = i + v < n ? I[i + v] : 0.0f;
        }
      }
    }
    const int64_t last = (full ? p0 + kChunk : n) - 1;
    const int64_t fa = frame_of(p0, ppf, inv_ppf), fb = frame_of(last, ppf, inv_ppf);
    if (full && fa == fb) {  // warp-uniform: the whole chunk lies in frame fa
      const float lo = __ldg(ranges + 2 * fa), hi = __ldg(ranges + 2 * fa + 1);
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int64_t i = p0 + (int64_t)(32 * j + lane) * 4;
        float pv[4];
        uint32_t cpack = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t c = tof_code(dv[j][v], Iv[j][v], lo, hi);
          const float ph = tof_phi(dv[j][v], Iv[j][v]);
          pv[v] = c == 0u ? ph : __int_as_float(0x7FC00000);
          cpack |= c << (8 * v);
          cnt += c == 0u;
        }
        __stcs(reinterpret_cast<float4*>(phi + i), make_float4(pv[0], pv[1], pv[2], pv[3]));
        if (code) __stcs(reinterpret_cast<unsigned int*>(code + i), cpack);
      }
      if (kept) {
        const int s = __reduce_add_sync(0xFFFFFFFFu, cnt);
        if (lane == 0 && s) atomicAdd(kept + fa, s);
      }
    } else {  // a frame boundary or the end inside the chunk: pixel by pixel
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int64_t i = p0 + (int64_t)(32 * j + lane) * 4;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (i + v >= n) continue;
          const int64_t f = frame_of(i + v, ppf, inv_ppf);
          const uint32_t c = tof_code(dv[j][v], Iv[j][v], __ldg(ranges + 2 * f), __ldg(ranges + 2 * f + 1));
          phi[i + v] = c == 0u ? tof_phi(dv[j][v], Iv[j][v]) : __int_as_float(0x7FC00000);
          if (code) code[i + v] = (uint8_t)c;
          if (kept && c == 0u) atomicAdd(kept + f, 1);
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_tof_range_phi(const float* d, const float* I, int64_t n, int64_t ppf, const float* ranges,
                                 float* phi, uint8_t* code, int* kept, cudaStream_t s) {
  const int64_t nframes = (n + ppf - 1) / ppf;
  if (kept) {
    const cudaError_t e = cudaMemsetAsync(kept, 0, (size_t)nframes * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  constexpr int NT = 256;
  int blocks_per_sm = 0;  // per device, cached (kernel_occupancy)
  const cudaError_t eo = kernel_occupancy((const void*)tof_range_phi_kernel, NT, 0, &blocks_per_sm);
  if (eo != cudaSuccess) return eo;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t want = (nchunks * 32 + NT - 1) / NT;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;  // persistent: one resident wave
  const int grid = (int)(want < cap ? want : cap);
  tof_range_phi_kernel<<<grid, NT, 0, s>>>(d, I, n, ppf, ranges, phi, code, kept, 1.0 / (double)ppf);
  return cudaGetLastError();
}

}  // namespace clipseg
