// tof_range.cu — K5 (NEXT-2): the paper's own per-pixel step over batched
// ToF frames: the range clip [r_min, r_max] of PAPER.md §5.2 (closed interval,
// recomputed per frame) as a 2-bit outcode, fused with phi = arctan(d sqrt(I)) of Eq. (5)
// for the kept pixels, plus the kept-pixel count per frame.
//
// HBM-bound map: 8 bytes in (d, I) and 5 out (phi, code) per pixel.  One thread owns 4
// consecutive pixels (128-bit loads / stores, evict-first); a warp owns 128 consecutive
// pixels, so with frames of >= 128 pixels (the paper's are 204^2) its pixels span at most
// two frames and the per-frame counts are two warp reductions and <= 2 atomics per warp.
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

template <bool COUNT_WARP>
__global__ void __launch_bounds__(256) tof_range_phi_kernel(const float* __restrict__ d, const float* __restrict__ I,
                                                            int64_t n, int64_t ppf, const float* __restrict__ ranges,
                                                            float* __restrict__ phi, uint8_t* __restrict__ code,
                                                            int* __restrict__ kept, double inv_ppf) {
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (n + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float4 nd = make_float4(0.f, 0.f, 0.f, 0.f), nI = nd;
  auto load = [&](int64_t gg, float4& a, float4& b) {  // group gg's 4 pixels (0 past the end)
    const int64_t i = gg * 4;
    if (i + 4 <= n) {
      a = __ldcs(reinterpret_cast<const float4*>(d + i));
      b = __ldcs(reinterpret_cast<const float4*>(I + i));
    } else {
      a = make_float4(i < n ? d[i] : 0.f, i + 1 < n ? d[i + 1] : 0.f, i + 2 < n ? d[i + 2] : 0.f, 0.f);
      b = make_float4(i < n ? I[i] : 0.f, i + 1 < n ? I[i + 1] : 0.f, i + 2 < n ? I[i + 2] : 0.f, 0.f);
    }
  };
  if (g < ngroups) load(g, nd, nI);
  // whole warps iterate together (the warp reductions need every lane)
  for (; g - lane < ngroups; g += stride) {
    const float dv[4] = {nd.x, nd.y, nd.z, nd.w}, Iv[4] = {nI.x, nI.y, nI.z, nI.w};
    if (g + stride < ngroups) load(g + stride, nd, nI);  // next group's loads in flight
    const int64_t i0 = g * 4;
    const bool live = g < ngroups;
    const int64_t f0 = frame_of(live ? i0 : 0, ppf, inv_ppf);
    const float lo0 = __ldg(ranges + 2 * f0), hi0 = __ldg(ranges + 2 * f0 + 1);
    float pv[4];
    uint32_t cpack = 0;
    int cnt_lo = 0, cnt_hi = 0;  // kept pixels in frame f0 / in later frames
    if (live && i0 + 4 <= n && i0 + 3 - f0 * ppf < ppf) {  // the common case: 4 pixels of frame f0
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint32_t c = tof_code(dv[v], Iv[v], lo0, hi0);
        const float ph = tof_phi(dv[v], Iv[v]);
        pv[v] = c == 0u ? ph : __int_as_float(0x7FC00000);
        cpack |= c << (8 * v);
        cnt_lo += c == 0u;
      }
    } else {  // the group crosses a frame boundary or the end
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const bool valid = live && i0 + v < n;
        const int64_t f = valid ? frame_of(i0 + v, ppf, inv_ppf) : f0;
        const float lo = __ldg(ranges + 2 * f), hi = __ldg(ranges + 2 * f + 1);
        const uint32_t c = tof_code(dv[v], Iv[v], lo, hi);
        const bool keep = valid && c == 0u;
        pv[v] = keep ? tof_phi(dv[v], Iv[v]) : __int_as_float(0x7FC00000);
        cpack |= c << (8 * v);
        if (keep) {
          if (COUNT_WARP) {
            if (f == f0) ++cnt_lo; else ++cnt_hi;
          } else if (kept) {
            atomicAdd(kept + f, 1);
          }
        }
      }
      if (!COUNT_WARP) cnt_lo = 0;
    }
    if (live) {
      if (i0 + 4 <= n) {
        __stcs(reinterpret_cast<float4*>(phi + i0), make_float4(pv[0], pv[1], pv[2], pv[3]));
        if (code) __stcs(reinterpret_cast<unsigned int*>(code + i0), cpack);
      } else {
        for (int v = 0; v < 4; ++v)
          if (i0 + v < n) {
            phi[i0 + v] = pv[v];
            if (code) code[i0 + v] = (uint8_t)(cpack >> (8 * v));
          }
      }
    }
    if (COUNT_WARP) {
      // the warp's 128 pixels span frames fw and fw + 1 at most (ppf >= 128)
      const int64_t fw = __shfl_sync(0xFFFFFFFFu, f0, 0);
      const int lo_c = (f0 == fw) ? cnt_lo : 0;
      const int hi_c = (f0 == fw) ? cnt_hi : cnt_lo + cnt_hi;
      const int s_lo = __reduce_add_sync(0xFFFFFFFFu, lo_c);
      const int s_hi = __reduce_add_sync(0xFFFFFFFFu, hi_c);
      if (lane == 0) {
        if (s_lo) atomicAdd(kept + fw, s_lo);
        if (s_hi) atomicAdd(kept + fw + 1, s_hi);
      }
    } else if (kept && cnt_lo) {
      atomicAdd(kept + f0, cnt_lo);  // the common-case group of the per-pixel-atomic variant
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
  static int blocks_per_sm = 0;  // cached device attribute (both instantiations are alike)
  if (!blocks_per_sm) {
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, tof_range_phi_kernel<true>, NT, 0);
    if (e != cudaSuccess || blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t ngroups = (n + 3) / 4;
  const int64_t want = (ngroups + NT - 1) / NT;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;  // persistent: one resident wave
  const int grid = (int)(want < cap ? want : cap);
  if (kept && ppf >= 128)
    tof_range_phi_kernel<true><<<grid, NT, 0, s>>>(d, I, n, ppf, ranges, phi, code, kept, 1.0 / (double)ppf);
  else
    tof_range_phi_kernel<false><<<grid, NT, 0, s>>>(d, I, n, ppf, ranges, phi, code, kept, 1.0 / (double)ppf);
  return cudaGetLastError();
}

}  // namespace clipseg
