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

#include "clip_kernels.cuh"

namespace clipseg {

namespace {

constexpr int32_t kFill = INT32_MIN;
constexpr int64_t kCoordMax = (int64_t)1 << 30;

struct Frac {
  int64_t num, den;  // den > 0, 0 <= num <= den
};

// a < b for fractions with positive denominators (|num|, den <= 2^31: products < 2^62)
__device__ __forceinline__ bool frac_lt(Frac a, Frac b) { return a.num * b.den < b.num * a.den; }

// p + round_half_up(d * t): q = floor(d num / den), r = d num - q den in [0, den); +1 when
// 2r >= den.  No 64-bit integer division (a ~70-instruction software routine that made the
// kernel issue-bound): q is estimated as RN(RN(d num) * inv) with inv = RN(1 / den), whose
// relative error is below 2^-50, so |q_est - d num / den| < 2^31 * 2^-50 and floor() is off by
// at most one; the exact int64 remainder fixes that.
__device__ __forceinline__ int32_t lerp_round(int64_t p, int64_t d, Frac t, double inv) {
  const int64_t x = d * t.num;
  int64_t q = (int64_t)floor(__dmul_rn((double)x, inv));
  int64_t r = x - q * t.den;
  if (r < 0) { --q; r += t.den; }
  if (r >= t.den) { ++q; r -= t.den; }
  return (int32_t)(p + q + (2 * r >= t.den));
}

// Returns flag (0 invisible, 1 visible, 2 out of range) and writes q[4] when visible.
__device__ __forceinline__ uint32_t clip_int_one(int32_t x0, int32_t y0, int32_t x1, int32_t y1, int4 win,
                                                 int32_t q[4]) {
  const int64_t X0 = x0, Y0 = y0, X1 = x1, Y1 = y1;
  const bool range = (X0 >= -kCoordMax) & (X0 <= kCoordMax) & (Y0 >= -kCoordMax) & (Y0 <= kCoordMax) &
                     (X1 >= -kCoordMax) & (X1 <= kCoordMax) & (Y1 >= -kCoordMax) & (Y1 <= kCoordMax);
  if (!range) return 2u;
  Frac tin{0, 1}, tout{1, 1};
  bool reject = false;
  const int64_t w0s[4] = {X0 - win.x, Y0 - win.y, (int64_t)win.z - X0, (int64_t)win.w - Y0};
  const int64_t w1s[4] = {X1 - win.x, Y1 - win.y, (int64_t)win.z - X1, (int64_t)win.w - Y1};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t w0 = w0s[e], w1 = w1s[e];
    reject |= (w0 < 0) & (w1 < 0);
    if (w0 < 0 && w1 >= 0) {  // entering: alpha = -w0 / (w1 - w0)
      const Frac a{-w0, w1 - w0};
      if (frac_lt(tin, a)) tin = a;
    } else if (w1 < 0 && w0 >= 0) {  // leaving: alpha = w0 / (w0 - w1)
      const Frac a{w0, w0 - w1};
      if (frac_lt(a, tout)) tout = a;
    }
  }
  if (reject || frac_lt(tout, tin)) return 0u;
  const int64_t dx = X1 - X0, dy = Y1 - Y0;
  if (tin.num == 0) {
    q[0] = x0; q[1] = y0;
  } else {
    const double inv = __drcp_rn((double)tin.den);
    q[0] = lerp_round(X0, dx, tin, inv);
    q[1] = lerp_round(Y0, dy, tin, inv);
  }
  if (tout.num == tout.den) {
    q[2] = x1; q[3] = y1;
  } else {
    const double inv = __drcp_rn((double)tout.den);
    q[2] = lerp_round(X0, dx, tout, inv);
    q[3] = lerp_round(Y0, dy, tout, inv);
  }
  return 1u;
}

__global__ void __launch_bounds__(256) clip_int_kernel(const int32_t* __restrict__ in, int64_t ld_in, int64_t n,
                                                       int4 win, int32_t* __restrict__ out, int64_t ld_out,
                                                       uint8_t* __restrict__ flags) {
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
      const uint32_t f = clip_int_one(x0[s], y0[s], x1[s], y1[s], win, q);
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
  static int blocks_per_sm = 0;  // cached device attribute
  if (!blocks_per_sm) {
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, clip_int_kernel, NT, 0);
    if (e != cudaSuccess || blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t ngroups = (n + 3) / 4;
  const int64_t want = (ngroups + NT - 1) / NT;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;  // persistent: one resident wave
  const int grid = (int)(want < cap ? want : cap);
  clip_int_kernel<<<grid, NT, 0, s>>>(in, ld_in, n, make_int4(lo[0], lo[1], hi[0], hi[1]), out, ld_out, flags);
  return cudaGetLastError();
}

}  // namespace clipseg
