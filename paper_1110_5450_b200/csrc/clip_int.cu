// clip_int.cu — K6 (NEXT-4): integer / pixel-coordinate 2D segment clipping
// against a closed integer window, with EXACT rational intersections.  The WEC formulation of
// the float path (PAPER.md:29-30 macros; DESIGN.md §3 R4-R5) in integers: per edge the WECs
// w0, w1 of both endpoints, trivial reject when both are negative, alpha = w0 / (w0 - w1)
// kept as a fraction num / den (den > 0) and compared by cross-multiplication; each clipped
// coordinate is p + round_half_up(d * num / den) (I4).  Coordinates are bounded by 2^30 (I1),
// so |w| <= 2^31, every cross product and d * num fit in 2^62, and each clipped coordinate's
// quotient is an fp64 estimate corrected by its exact int64 remainder (lerp_round): results
// are bit-exact by construction.
//
// HBM-bound map: 16 bytes in, 16 out + 1 flag byte per segment; one thread handles 4
// consecutive segments with 128-bit loads / stores on each of the 4 planes.
#include <cuda_runtime.h>

#include <cstdint>

#include "clip_int_math.cuh"
#include "clip_kernels.cuh"

namespace clipseg {

namespace {

using namespace intclip;

// in and out may be the same buffer (out == in, ld_out == ld_in: each thread reads its rows
// before writing them), so neither is __restrict__.
__global__ void __launch_bounds__(256) clip_int_kernel(const int32_t* in, int64_t ld_in, int64_t n,
                                                       int4 win, bool small_win, int32_t* out,
                                                       int64_t ld_out, uint8_t* __restrict__ flags) {
  const int64_t ngroups = (n + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += stride) {
    const int64_t i = 4 * g;
    // 128-bit loads are safe even for the ragged tail: ld >= n is a multiple of 4 elements
    int4 v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __ldcs(reinterpret_cast<const int4*>(in + c * ld_in + i));
    const int32_t* x0 = reinterpret_cast<const int32_t*>(&v[0]);
    const int32_t* y0 = reinterpret_cast<const int32_t*>(&v[1]);
    const int32_t* x1 = reinterpret_cast<const int32_t*>(&v[2]);
    const int32_t* y1 = reinterpret_cast<const int32_t*>(&v[3]);
    int32_t o[4][4];
    uint32_t fpack = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int32_t q[4];
      const uint32_t f = clip_int_one(x0[s], y0[s], x1[s], y1[s], win, small_win, q);
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c][s] = f == 1u ? q[c] : kFill;
      fpack |= f << (8 * s);
    }
    if (i + 4 <= n) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        __stcs(reinterpret_cast<int4*>(out + c * ld_out + i), make_int4(o[c][0], o[c][1], o[c][2], o[c][3]));
      if (flags) __stcs(reinterpret_cast<unsigned int*>(flags + i), fpack);
    } else {
      for (int s = 0; s < 4 && i + s < n; ++s) {
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c * ld_out + i + s] = o[c][s];
        if (flags) flags[i + s] = (uint8_t)(fpack >> (8 * s));
      }
    }
  }
}

}  // namespace

cudaError_t launch_clip_int(const int32_t* in, int64_t ld_in, int64_t n, const int32_t lo[2], const int32_t hi[2],
                            int32_t* out, int64_t ld_out, uint8_t* flags, cudaStream_t s) {
  constexpr int NT = 256;
  int blocks_per_sm = 0;  // per device, cached (kernel_occupancy)
  const cudaError_t e = kernel_occupancy((const void*)clip_int_kernel, NT, 0, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t ngroups = (n + 3) / 4;
  const int64_t want = (ngroups + NT - 1) / NT;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;  // persistent: one resident wave
  const int grid = (int)(want < cap ? want : cap);
  const bool small_win = lo[0] >= -kSmall && lo[1] >= -kSmall && hi[0] <= kSmall && hi[1] <= kSmall;
  clip_int_kernel<<<grid, NT, 0, s>>>(in, ld_in, n, make_int4(lo[0], lo[1], hi[0], hi[1]), small_win, out, ld_out,
                                      flags);
  return cudaGetLastError();
}

}  // namespace clipseg
