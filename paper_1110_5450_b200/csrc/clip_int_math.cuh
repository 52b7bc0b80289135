// clip_int_math.cuh — NEXT-4: the exact integer clip of one 2D int32 segment
// (rules I1-I6), shared by the dense kernel (clip_int.cu) and the packed compacting kernel
// (clip_compact.cu, IntOp).  See clip_int.cu for the derivation.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace clipseg {
namespace intclip {

constexpr int32_t kFill = INT32_MIN;
constexpr int64_t kCoordMax = (int64_t)1 << 30;
constexpr int32_t kSmall = 1 << 14;  // 32-bit path bound

template <typename I>
struct Frac {
  I num, den;  // den > 0, 0 <= num <= den
};

// a < b for fractions with positive denominators (|num|, den <= 2^31: products < 2^62;
// the 32-bit path has |num|, den <= 2^15: products < 2^30)
template <typename I>
__device__ __forceinline__ bool frac_lt(Frac<I> a, Frac<I> b) { return a.num * b.den < b.num * a.den; }

__device__ __forceinline__ double est_quot(int64_t x, double inv) { return floor(__dmul_rn((double)x, inv)); }
__device__ __forceinline__ double rcp(int64_t d) { return __drcp_rn((double)d); }

// p + round_half_up(d * t): q = floor(d num / den), r = d num - q den in [0, den); +1 when
// 2r >= den.  No integer division (64-bit division is a ~70-instruction software routine that
// made the kernel issue-bound): q is estimated as RN(RN(d num) * inv) with inv = RN(1 / den).
// 64-bit path: relative error < 3 * 2^-53 and |q| <= 2^31, so the estimate is within 2^-20 of
// d num / den; 32-bit path: relative error < 3 * 2^-24 and |q| <= 2^15, within 2^-7.  Either
// way floor() is off by at most one, and the exact integer remainder fixes it.
template <typename I, typename F>
__device__ __forceinline__ int32_t lerp_round(I p, I d, Frac<I> t, F inv) {
  const I x = d * t.num;
  I q = (I)est_quot(x, inv);
  I r = x - q * t.den;
  if (r < 0) { --q; r += t.den; }
  if (r >= t.den) { ++q; r -= t.den; }
  return (int32_t)(p + q + (2 * r >= t.den));
}

// Returns flag (0 invisible, 1 visible) and writes q[4] when visible.  I = int64_t for any
// coordinates in [-2^30, 2^30]; I = int32_t when every coordinate and window bound lies in
// [-2^14, 2^14] (|w|, den <= 2^15), the common pixel-coordinate case: all 32-bit arithmetic.
template <typename I>
__device__ __forceinline__ uint32_t clip_int_core(I X0, I Y0, I X1, I Y1, int4 win, int32_t q[4]) {
  Frac<I> tin{0, 1}, tout{1, 1};
  bool reject = false;
  const I w0s[4] = {X0 - (I)win.x, Y0 - (I)win.y, (I)win.z - X0, (I)win.w - Y0};
  const I w1s[4] = {X1 - (I)win.x, Y1 - (I)win.y, (I)win.z - X1, (I)win.w - Y1};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const I w0 = w0s[e], w1 = w1s[e];
    reject |= (w0 < 0) & (w1 < 0);
    if (w0 < 0 && w1 >= 0) {  // entering: alpha = -w0 / (w1 - w0)
      const Frac<I> a{-w0, w1 - w0};
      if (frac_lt(tin, a)) tin = a;
    } else if (w1 < 0 && w0 >= 0) {  // leaving: alpha = w0 / (w0 - w1)
      const Frac<I> a{w0, w0 - w1};
      if (frac_lt(a, tout)) tout = a;
    }
  }
  if (reject || frac_lt(tout, tin)) return 0u;
  const I dx = X1 - X0, dy = Y1 - Y0;
  if (tin.num == 0) {
    q[0] = (int32_t)X0; q[1] = (int32_t)Y0;
  } else {
    const auto inv = rcp(tin.den);
    q[0] = lerp_round(X0, dx, tin, inv);
    q[1] = lerp_round(Y0, dy, tin, inv);
  }
  if (tout.num == tout.den) {
    q[2] = (int32_t)X1; q[3] = (int32_t)Y1;
  } else {
    const auto inv = rcp(tout.den);
    q[2] = lerp_round(X0, dx, tout, inv);
    q[3] = lerp_round(Y0, dy, tout, inv);
  }
  return 1u;
}

// The 32-bit path without branches (every lane runs the same instructions: predicated selects
// instead of divergent ifs; measured thread efficiency 19.3 of 32 with the branchy core):
// t = 0 and t = 1 need no special case since lerp_round then returns p and p + d exactly.
__device__ __forceinline__ uint32_t clip_int_small(int32_t X0, int32_t Y0, int32_t X1, int32_t Y1, int4 win,
                                                   int32_t q[4]) {
  // Per axis, the sign of d decides which edge can be entered and which left (lo / hi for
  // d > 0, hi / lo for d < 0), and both alphas share the denominator |d| = w0 - w1: one
  // entering and one leaving candidate per axis instead of both tests on all four edges.
  // A d = 0 axis never yields a candidate unless the segment is rejected on it.
  int32_t in_n = 0, in_d = 1, out_n = 1, out_d = 1;
  bool reject = false;
  const int32_t p0s[2] = {X0, Y0}, p1s[2] = {X1, Y1}, los[2] = {win.x, win.y}, his[2] = {win.z, win.w};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int32_t p0 = p0s[k], p1 = p1s[k], lo = los[k], hi = his[k];
    reject |= ((p0 < lo) & (p1 < lo)) | ((p0 > hi) & (p1 > hi));
    const int32_t d = p1 - p0;
    const bool pos = d > 0;
    const int32_t ad = pos ? d : -d;
    const int32_t en = pos ? lo - p0 : p0 - hi;  // entering alpha = en / ad when en > 0
    const int32_t ln = pos ? hi - p0 : p0 - lo;  // leaving alpha = ln / ad
    const bool lea = pos ? p1 > hi : p1 < lo;
    const bool up_in = (en > 0) & (in_n * ad < en * in_d);
    const bool up_out = lea & (ln * out_d < out_n * ad);
    in_n = up_in ? en : in_n;
    in_d = up_in ? ad : in_d;
    out_n = up_out ? ln : out_n;
    out_d = up_out ? ad : out_d;
  }
  const uint32_t vis = !reject & !(out_n * in_d < in_n * out_d);
  const int32_t dx = X1 - X0, dy = Y1 - Y0;
  // inv = MUFU.RCP (relative error < 2^-22): the estimate stays within 1.5 * 2^-22 * 2^15 < 1
  // of d num / den, so one remainder fix still suffices (the correctly rounded __frcp_rn is a
  // ~10-instruction Newton sequence with a slow-path branch).
  float inv_in, inv_out;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_in) : "f"((float)in_d));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_out) : "f"((float)out_d));
  auto lerp = [](int32_t p, int32_t d, int32_t num, int32_t den, float inv) {
    const int32_t x = d * num;
    int32_t qq = __float2int_rd(__fmul_rn((float)x, inv));
    int32_t r = x - qq * den;
    qq += (r >= den) - (r < 0);
    r += (r < 0 ? den : 0) - (r >= den ? den : 0);
    return p + qq + (2 * r >= den);
  };
  q[0] = lerp(X0, dx, in_n, in_d, inv_in);
  q[1] = lerp(Y0, dy, in_n, in_d, inv_in);
  q[2] = lerp(X0, dx, out_n, out_d, inv_out);
  q[3] = lerp(Y0, dy, out_n, out_d, inv_out);
  return vis;
}

// Returns flag (0 invisible, 1 visible, 2 out of range) and writes q[4] when visible.
__device__ __forceinline__ uint32_t clip_int_one(int32_t x0, int32_t y0, int32_t x1, int32_t y1, int4 win,
                                                 bool small_win, int32_t q[4]) {
  // biased in unsigned arithmetic (no signed overflow near INT32_MAX): every coordinate lies in
  // [-2^14, 2^14] iff the largest biased value is <= 2^15
  const uint32_t m = max(max((uint32_t)x0 + (uint32_t)kSmall, (uint32_t)y0 + (uint32_t)kSmall),
                         max((uint32_t)x1 + (uint32_t)kSmall, (uint32_t)y1 + (uint32_t)kSmall));
  if (small_win && m <= 2u * kSmall) return clip_int_small(x0, y0, x1, y1, win, q);
  const int64_t X0 = x0, Y0 = y0, X1 = x1, Y1 = y1;
  const bool range = (X0 >= -kCoordMax) & (X0 <= kCoordMax) & (Y0 >= -kCoordMax) & (Y0 <= kCoordMax) &
                     (X1 >= -kCoordMax) & (X1 <= kCoordMax) & (Y1 >= -kCoordMax) & (Y1 <= kCoordMax);
  if (!range) return 2u;
  return clip_int_core<int64_t>(X0, Y0, X1, Y1, win, q);
}

// Two kept (in-range) segments per lane, the packed compacting kernel's rounds: the 32-bit
// path runs on both rows first (branch-free; its values are unused for a row outside its
// range), then one warp vote sends the rare warps holding a wide row to the 64-bit path
// for those rows only.
__device__ __forceinline__ bool int_small(int32_t x0, int32_t y0, int32_t x1, int32_t y1, bool small_win) {
  const uint32_t m = max(max((uint32_t)x0 + (uint32_t)kSmall, (uint32_t)y0 + (uint32_t)kSmall),
                         max((uint32_t)x1 + (uint32_t)kSmall, (uint32_t)y1 + (uint32_t)kSmall));
  return small_win && m <= 2u * kSmall;
}
__device__ __forceinline__ void clip_int_two(const int32_t (&a)[4], const int32_t (&b)[4], int4 win, bool small_win,
                                             int32_t (&qa)[4], int32_t (&qb)[4], bool& va, bool& vb) {
  const bool sa = int_small(a[0], a[1], a[2], a[3], small_win), sb = int_small(b[0], b[1], b[2], b[3], small_win);
  va = clip_int_small(a[0], a[1], a[2], a[3], win, qa) == 1u;
  vb = clip_int_small(b[0], b[1], b[2], b[3], win, qb) == 1u;
  if (!__all_sync(0xFFFFFFFFu, sa & sb)) {
    if (!sa) va = clip_int_core<int64_t>(a[0], a[1], a[2], a[3], win, qa) == 1u;
    if (!sb) vb = clip_int_core<int64_t>(b[0], b[1], b[2], b[3], win, qb) == 1u;
  }
}

}  // namespace intclip
}  // namespace clipseg
