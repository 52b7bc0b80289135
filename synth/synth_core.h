/* synth/synth_core.h — counter-based synthetic segment generator (G1).
 *
 * INPUT GENERATOR ONLY. This module holds none of the clipping arithmetic: it
 * produces seeded segment sets in the planar layout both the oracle/ tests and
 * the CUDA path consume, identically on host and device (every value below is
 * built from integer draws with exact conversions, so the host and device twins
 * are bit-identical).
 *
 * Draw j of segment i under seed s:  h(s,i,j) = mix64(s + (16 i + j + 1) * phi64)
 * with mix64 the splitmix64 finaliser.  Shapes follow BASELINE.json configs[0..4]
 * and SURVEY.md §8(d) (C1 uniform in [-1,2)^D, C2 inside/crossing/outside mixes,
 * C3 adversarial families, C4 3D uniform); the window the families are built
 * around is [0,1]^D.
 */
#pragma once
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

enum { SYN_UNIFORM = 0, SYN_MIX = 1, SYN_ADVERSARIAL = 2, SYN_HOMOG = 3 };
/* SYN_HOMOG (dim 4 only: x0,y0,z0,w0,x1,y1,z1,w1) tags */
enum { SYN_H_PERSPECTIVE = 0, SYN_H_AFFINE = 1, SYN_H_BEHIND = 2, SYN_H_ON_PLANE = 3, SYN_H_DEGENERATE = 4 };
enum { SYN_CAT_INSIDE = 0, SYN_CAT_CROSSING = 1, SYN_CAT_OUTSIDE = 2 };
#define SYN_TAG_NEAR 0x80u  /* adversarial tag bit: endpoint placed within tolerance of an edge */

SYN_HD uint64_t syn_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

SYN_HD uint64_t syn_h(uint64_t seed, int64_t i, int j) {
  return syn_mix64(seed + ((uint64_t)i * 16u + (uint64_t)j + 1u) * 0x9E3779B97F4A7C15ull);
}

/* ---- value construction, exact in the target type -------------------------------- */
template <typename T> struct SynT;

template <> struct SynT<float> {
  /* grid value in [-1,2): g * 2^-22, g integer in [-2^22, 2^23) (exact in fp32) */
  SYN_HD static float grid(uint64_t h) {
    int64_t g = (int64_t)(((h & 0xFFFFFFull) * 12582912ull) >> 24) - 4194304;
    return (float)g * 0x1p-22f;
  }
  /* unit offset in [0,1): 22-bit grid */
  SYN_HD static float unit(uint64_t h) { return (float)(h & 0x3FFFFFull) * 0x1p-22f; }
  /* far value in [-1024,1024): 2^-11 grid */
  SYN_HD static float far(uint64_t h) {
    return (float)((int64_t)(h & 0x3FFFFFull) - 2097152) * 0x1p-11f;
  }
  /* small offset below the fp32 tolerance 1e-6 (window extent 1): k*2^-40, k < 2^20 */
  SYN_HD static float tiny(uint64_t h) { return (float)(h & 0xFFFFFull) * 0x1p-40f; }
  /* x stepped by k ulps (x >= 0 on entry; k != 0, |k| <= 16) via the bit pattern */
  SYN_HD static float ulp_step(float x, int k) {
    uint32_t b; memcpy(&b, &x, 4);
    if (b == 0u) b = (k > 0) ? (uint32_t)k : (0x80000000u | (uint32_t)(-k));
    else b = (uint32_t)((int64_t)b + k);
    float r; memcpy(&r, &b, 4); return r;
  }
  /* positive w in [0.5, 2): (3k + 2^22) * 2^-23, k < 2^22 (exact) */
  SYN_HD static float wpos(uint64_t h) { return (float)(3u * (uint32_t)(h & 0x3FFFFFull) + 0x400000u) * 0x1p-23f; }
  SYN_HD static float min_sub() { return 0x1p-149f; }
  SYN_HD static float neg_zero() { uint32_t b = 0x80000000u; float r; memcpy(&r, &b, 4); return r; }
};

template <> struct SynT<double> {
  SYN_HD static double grid(uint64_t h) {
    int64_t g = (int64_t)((((h >> 12) * 3ull) >> 2)) - (int64_t)(1ull << 50);
    return (double)g * 0x1p-50;
  }
  SYN_HD static double unit(uint64_t h) { return (double)(h >> 12) * 0x1p-52; }
  SYN_HD static double far(uint64_t h) {
    return (double)((int64_t)(h >> 12) - (int64_t)(1ull << 51)) * 0x1p-41;
  }
  /* below the fp64 tolerance 1e-14: k*2^-67, k < 2^20 */
  SYN_HD static double tiny(uint64_t h) { return (double)(h & 0xFFFFFull) * 0x1p-67; }
  SYN_HD static double ulp_step(double x, int k) {
    uint64_t b; memcpy(&b, &x, 8);
    if (b == 0ull) b = (k > 0) ? (uint64_t)k : (0x8000000000000000ull | (uint64_t)(-k));
    else b = (uint64_t)((int64_t)b + k);
    double r; memcpy(&r, &b, 8); return r;
  }
  SYN_HD static double wpos(uint64_t h) { return (double)(3ull * (h >> 14) + (1ull << 50)) * 0x1p-51; }
  SYN_HD static double min_sub() { return 0x1p-1074; }
  SYN_HD static double neg_zero() { uint64_t b = 0x8000000000000000ull; double r; memcpy(&r, &b, 8); return r; }
};

/* Coordinate strictly outside [0,1] on the given side: side 0 -> [-1,0), side 1 -> (1,2]. */
template <typename T> SYN_HD T syn_beyond(uint64_t h, int side) {
  T u = SynT<T>::unit(h);
  return side ? (T)2 - u : u - (T)1;
}

/* One segment.  p[c], c = e*D + k (endpoint e, axis k) — the planar order x0,y0,[z0],x1,y1,[z1].
 * Returns the tag byte: category for MIX, family index (| SYN_TAG_NEAR) for ADVERSARIAL, 0 else. */
template <typename T, int D>
SYN_HD uint8_t syn_segment(int family, uint64_t seed, int64_t i, uint32_t p_in, uint32_t p_cross, T p[2 * D]) {
  typedef SynT<T> S;
  if (family == SYN_UNIFORM) {
    for (int c = 0; c < 2 * D; ++c) p[c] = S::grid(syn_h(seed, i, c));
    return 0;
  }
  const uint64_t h0 = syn_h(seed, i, 15);
  if (family == SYN_MIX) {
    const uint64_t u = h0 >> 32;
    const uint64_t sel = (h0 >> 1) & 0x7FFFFFFFull;
    if (u < (uint64_t)p_in) {                          /* inside: both endpoints in [0,1)^D */
      for (int c = 0; c < 2 * D; ++c) p[c] = S::unit(syn_h(seed, i, c));
      return SYN_CAT_INSIDE;
    }
    if (u < (uint64_t)p_in + (uint64_t)p_cross) {      /* crossing: inside endpoint + outer cell */
      const int ncell = (D == 2) ? 8 : 26, center = (D == 2) ? 4 : 13;
      int m = (int)(sel % (uint64_t)ncell);
      if (m >= center) m += 1;
      const int ein = (int)(h0 & 1u), eout = 1 - ein;
      for (int k = 0; k < D; ++k) {
        p[ein * D + k] = S::unit(syn_h(seed, i, k));
        const int digit = m % 3; m /= 3;
        const uint64_t hk = syn_h(seed, i, D + k);
        p[eout * D + k] = (digit == 1) ? S::unit(hk) : syn_beyond<T>(hk, digit == 2);
      }
      return SYN_CAT_CROSSING;
    }
    const int edge = (int)(sel % (uint64_t)(2 * D));   /* outside: both beyond one edge */
    const int ax = edge >> 1, side = edge & 1;
    for (int e = 0; e < 2; ++e)
      for (int k = 0; k < D; ++k) {
        const uint64_t hk = syn_h(seed, i, e * D + k);
        p[e * D + k] = (k == ax) ? syn_beyond<T>(hk, side) : S::grid(hk);
      }
    return SYN_CAT_OUTSIDE;
  }
  /* SYN_ADVERSARIAL (2D families; for D == 3 the third axis is grid-uniform) */
  const int f = (int)(i % 10);
  uint8_t tag = (uint8_t)f;
  for (int c = 0; c < 2 * D; ++c) p[c] = S::grid(syn_h(seed, i, c));
  const uint64_t h1 = syn_h(seed, i, 8), h2 = syn_h(seed, i, 9), h3 = syn_h(seed, i, 10);
  const uint64_t h4 = syn_h(seed, i, 11);
  T *P0 = p, *P1 = p + D;
  switch (f) {
    case 0: { /* F1 zero-length: inside / outside / on an edge / on a corner */
      const int s = (int)(h0 & 3u);
      T x, y;
      if (s == 0) { x = S::unit(h1); y = S::unit(h2); }
      else if (s == 1) { x = syn_beyond<T>(h1, (int)((h0 >> 2) & 1u)); y = S::grid(h2); }
      else if (s == 2) {
        const int e = (int)((h0 >> 2) & 3u);
        const T v = S::unit(h1), ev = (T)(e & 1);
        x = (e < 2) ? ev : v; y = (e < 2) ? v : ev;
      } else { x = (T)((h0 >> 2) & 1u); y = (T)((h0 >> 3) & 1u); }
      P0[0] = P1[0] = x; P0[1] = P1[1] = y;
      if (D == 3) P1[2] = P0[2] = S::unit(h3);
      break;
    }
    case 1: { /* F2 axis-parallel on / inside / outside an edge line */
      const int a = (int)(h0 & 1u), s = (int)((h0 >> 1) % 5u);
      T c;
      if (s < 2) c = (T)s;
      else if (s == 2) c = S::unit(h1);
      else c = syn_beyond<T>(h1, s == 4);
      P0[a] = P1[a] = c;
      break;
    }
    case 2: { /* F3 endpoints exactly on edges and corners */
      for (int e = 0; e < 2; ++e) {
        const uint64_t he = e ? h2 : h1;
        const int s = (int)((he >> 40) % 3u);
        T* P = e ? P1 : P0;
        if (s == 0) { P[0] = (T)(he & 1u); P[1] = (T)((he >> 1) & 1u); }
        else if (s == 1) {
          const int ed = (int)((he >> 2) & 3u);
          const T v = S::unit(he >> 4), ev = (T)(ed & 1);
          P[0] = (ed < 2) ? ev : v; P[1] = (ed < 2) ? v : ev;
        }
      }
      break;
    }
    case 3: { /* F4 collinear with an edge, spanning it */
      const int ed = (int)(h0 & 3u), a = ed >> 1;  /* a = axis held constant */
      const T ev = (T)(ed & 1);
      P0[a] = P1[a] = ev;
      P0[1 - a] = syn_beyond<T>(h1, 0);
      P1[1 - a] = syn_beyond<T>(h2, 1);
      break;
    }
    case 4: { /* F5 exact corner grazes (the line meets the window only at a corner) */
      const int cx = (int)(h0 & 1u), cy = (int)((h0 >> 1) & 1u);
      const T u = S::unit(h1), v = S::unit(h2);
      const T X = (T)cx, Y = (T)cy;
      /* direction (1, s) with s = -1 at corners (0,0),(1,1), s = +1 at (1,0),(0,1) */
      const T sx = cx ? (T)1 : (T)-1, sy = cy ? (T)1 : (T)-1;  /* outward normal signs */
      /* P0 = C + u*(-sy*?,...) : both endpoints outside, on the tangent line x*sx... */
      /* tangent direction t = (sy, -sx) (perpendicular to the diagonal normal (sx, sy)) */
      P0[0] = X + u * sy; P0[1] = Y - u * sx;
      P1[0] = X - v * sy; P1[1] = Y + v * sx;
      break;
    }
    case 5: { /* F6 near-boundary: one coordinate at edge +- k ulp or +- tiny */
      P0[0] = S::unit(h1); P0[1] = S::unit(h2);
      const int e = (int)(h0 & 1u), a = (int)((h0 >> 1) & 1u), side = (int)((h0 >> 2) & 1u);
      const int mode = (int)((h0 >> 3) & 1u), sgn = ((h0 >> 4) & 1u) ? 1 : -1;
      const T edge = (T)side;
      T v;
      if (mode == 0) v = S::ulp_step(edge, sgn * (1 + (int)((h0 >> 5) & 15u)));
      else v = sgn > 0 ? edge + S::tiny(h3) : edge - S::tiny(h3);
      (e ? P1 : P0)[a] = v;
      tag |= SYN_TAG_NEAR;
      break;
    }
    case 6: { /* F7 signed zeros and the smallest subnormal next to a zero edge (FTZ trap) */
      for (int c = 0; c < 4; ++c) {
        const int s = (int)((h0 >> (3 * c)) & 7u);
        T v;
        switch (s) {
          case 0: v = S::neg_zero(); break;
          case 1: v = (T)0; break;
          case 2: v = S::min_sub(); break;
          case 3: v = -S::min_sub(); break;
          case 4: v = (T)1; break;
          case 5: v = S::unit(syn_h(seed, i, c)); break;
          default: v = S::grid(syn_h(seed, i, c)); break;
        }
        p[(c >> 1) * D + (c & 1)] = v;
      }
      break;
    }
    case 7: { /* F8 reflection closed form: E on an edge, P_in inside, P_out = 2E - P_in */
      const int ed = (int)(h0 & 3u), a = ed >> 1, side = ed & 1;
      T E[2], Pin[2], Pout[2];
      E[a] = (T)side; E[1 - a] = S::unit(h1);
      Pin[a] = side ? S::unit(h2) : (T)1 - S::unit(h2);   /* strictly inside along a */
      Pin[1 - a] = S::unit(h3);
      for (int k = 0; k < 2; ++k) Pout[k] = (T)2 * E[k] - Pin[k];  /* exact on the grid */
      const int swap = (int)((h0 >> 2) & 1u);
      for (int k = 0; k < 2; ++k) { P0[k] = swap ? Pout[k] : Pin[k]; P1[k] = swap ? Pin[k] : Pout[k]; }
      if (D == 3) P1[2] = P0[2] = S::unit(h4);
      break;
    }
    case 8: /* F9 uniform C1 */
      break;
    default: /* F10 far coordinates, |p| <= 2^10 */
      for (int c = 0; c < 2 * D; ++c) p[c] = S::far(syn_h(seed, i, c));
      break;
  }
  return tag;
}

/* NEXT-1 input: one segment in homogeneous clip space, p = (x0,y0,z0,w0,x1,y1,z1,w1), around
 * the volume -w <= x,y,z <= w.  Mode (tag) from the segment's draw 15:
 *   60 % perspective: w in [0.5, 2), x,y,z = 2 g - 1 in [-3, 3) (g on the grid);
 *   10 % affine: w = 1 exactly (the 3D cuboid reduction), x,y,z as above;
 *   10 % behind: one endpoint with w in (-2, -0.5];
 *   10 % on planes: one endpoint exactly on a plane (x = +-w) or an edge/corner of the volume;
 *   10 % degenerate: an endpoint with w = 0 (the 4D origin, or a random direction), or a
 *        zero-length segment.
 * A nonzero p_persp sets the perspective share to p_persp / 2^32 instead (bench workloads). */
template <typename T>
SYN_HD uint8_t syn_homog(uint64_t seed, int64_t i, T p[8], uint32_t p_persp) {
  typedef SynT<T> S;
  const uint64_t h0 = syn_h(seed, i, 15);
  /* p_persp != 0 overrides the perspective share (p_persp / 2^32; the rest 6..9 equally) */
  const int m = p_persp == 0u ? (int)((h0 >> 32) % 10u)
                              : ((h0 >> 32) < (uint64_t)p_persp ? 0 : 6 + (int)((h0 >> 1) % 4u));
  for (int e = 0; e < 2; ++e) {
    for (int k = 0; k < 3; ++k) p[4 * e + k] = (T)2 * S::grid(syn_h(seed, i, 4 * e + k)) - (T)1;
    p[4 * e + 3] = (m == 6) ? (T)1 : S::wpos(syn_h(seed, i, 4 * e + 3));
  }
  const int e = (int)(h0 & 1u);
  T* P = p + 4 * e;
  if (m < 6) return SYN_H_PERSPECTIVE;
  if (m == 6) return SYN_H_AFFINE;
  if (m == 7) {
    P[3] = -P[3];
    return SYN_H_BEHIND;
  }
  if (m == 8) {
    const int a = (int)((h0 >> 1) % 3u), nb = (int)((h0 >> 3) & 3u);  /* axis, extra planes */
    for (int j = 0; j <= (nb == 3 ? 2 : nb); ++j) {
      const int ax = (a + j) % 3;
      P[ax] = ((h0 >> (5 + j)) & 1u) ? P[3] : -P[3];
    }
    return SYN_H_ON_PLANE;
  }
  const int s = (int)((h0 >> 1) & 3u);
  if (s == 0) { P[0] = P[1] = P[2] = P[3] = (T)0; }                      /* the 4D origin */
  else if (s == 1) { P[3] = (T)0; }                                       /* w = 0 direction */
  else { for (int k = 0; k < 4; ++k) p[4 * (1 - e) + k] = P[k]; }         /* zero length */
  return SYN_H_DEGENERATE;
}

/* ---- NEXT-2 input: batched ToF frames (distance d, intensity I per pixel) -------------
 * PAPER.md §5.2 clips pixels to [r_min, r_max] per frame; Eq. (5) fuses
 * them into phi = arctan(d sqrt(I)) under the inverse-square law I ~ 1/d^2.  Frames
 * are 204 x 204 in the paper.  Per pixel (global index i, draws j = 0..3):
 *   2 % dropouts (d = I = 0, the invalid sentinel); 40 % "hand" pixels within +-0.2 m of one
 *   of the frame's two hand distances; 58 % background, d uniform in [0.3, 7.5) m; d is a
 *   multiple of 2^-20 m; intensity I = rho / (d d), reflectivity rho in [0.2, 1) (the constant
 *   c of SPEC.md:400 makes I(1 m, rho = 1) = 1).
 * Per frame f: hand distances d1, d2 in [0.5, 1.5) and the clip range r_min = max(1e-3,
 * min(d1, d2) - r_th), r_max = max(d1, d2) + r_th with r_th = 0.1 m (§5.2 formulas;
 * r_th from Table 1 via SPEC.md:262). */
SYN_HD float syn_tof_hand(uint64_t seed, int64_t f, int which) {
  const uint64_t h = syn_h(seed ^ 0x70F0C11Bull, f, which);
  return 0.5f + (float)(h & 0xFFFFFull) * 0x1p-20f;   /* [0.5, 1.5) on a 2^-20 grid */
}

SYN_HD void syn_tof_range(uint64_t seed, int64_t f, float r[2]) {
  const float d1 = syn_tof_hand(seed, f, 0), d2 = syn_tof_hand(seed, f, 1);
  const float lo = (d1 < d2 ? d1 : d2) - 0.1f, hi = (d1 < d2 ? d2 : d1) + 0.1f;
  r[0] = lo > 1e-3f ? lo : 1e-3f;
  r[1] = hi;
}

SYN_HD void syn_tof_pixel(uint64_t seed, int64_t i, int64_t ppf, float* d, float* I) {
  const uint64_t h0 = syn_h(seed, i, 0), h1 = syn_h(seed, i, 1), h2 = syn_h(seed, i, 2);
  const uint32_t u = (uint32_t)(h0 >> 32) % 100u;
  if (u < 2u) { *d = 0.0f; *I = 0.0f; return; }
  float dist;
  if (u < 42u) {
    const float dh = syn_tof_hand(seed, i / ppf, (int)(h0 & 1u));
    /* hand pixel: dh + k 2^-20, |k 2^-20| < 0.2 (dh is on the 2^-20 grid: exact) */
    const int32_t k = (int32_t)(h1 % 419430ull) - 209715;
    dist = dh + (float)k * 0x1p-20f;
  } else {
    /* background: [0.3, 7.5) m on the 2^-20 grid */
    const uint32_t k = 314573u + (uint32_t)(h1 % 7549747ull);
    dist = (float)k * 0x1p-20f;
  }
  const float rho = 0.2f + (float)(h2 & 0xFFFFFull) * (0.8f * 0x1p-20f);
  *d = dist;
  *I = rho / (dist * dist);
}
