/* oracle/clip_homog_impl.h — NEXT-1: segment clipping in homogeneous clip space (rules H1..H10).
 *
 * TEST INFRASTRUCTURE ONLY (see clip_oracle.c).  Included twice by clip_oracle.c with
 * REAL = float / double (SFX, FMA as for clip_oracle_impl.h).
 *
 * PAPER.md only names the window-edge coordinates (\wec, \WEC); their
 * textbook home is Blinn & Newell's clipping in homogeneous coordinates (SURVEY.md §8(f)
 * NEXT-1).  DESIGN.md §12 states the rules and the readings:
 *
 *   a point P = (x, y, z, w) is inside the closed clip volume -w <= x, y, z <= w;
 *   H1  boundary coordinates (the WECs of the six planes): bl_k = RN(w + p_k) for the plane
 *       -w <= p_k, bh_k = RN(w - p_k) for p_k <= w;
 *   H2  outcode bit 2k = [bl_k < 0], bit 2k+1 = [bh_k < 0];
 *   H3  trivial reject (c0 & c1) != 0, trivial accept (c0 | c1) == 0 (Q = P bit for bit);
 *   H4  alpha = RN(b0 / RN(b0 - b1)) on EVERY plane an endpoint is outside of (entering when
 *       P0 is, exiting when P1 is) — unlike the cuboid (R4), an endpoint with w < 0 can be
 *       outside both planes of one axis, so each of the six planes has its own alpha;
 *   H5  t_in = max(0, alpha_in...), t_out = min(1, alpha_out...), compare-select in plane
 *       order (x low, x high, y low, y high, z low, z high);
 *   H6  visible iff no trivial reject and t_in <= t_out;
 *   H7  an inside endpoint is copied (all four components); a crossed endpoint takes
 *       q_w = RN(fma(t, RN(w1 - w0), w0)), then per axis k: snap q_k = -q_w when the low
 *       plane's alpha equals t, else q_w when the high plane's does, else q = RN(fma(t,
 *       RN(p1_k - p0_k), p0_k)) clamped into [-q_w, q_w] by comparisons;
 *   H8  invisible rows: canonical qNaN in every output component, flag 0;
 *   H9  a non-finite component makes the segment invisible;
 *   H10 compaction as R10;
 *   NDC (optional output, "the final divide"): ndc_k = RN(q_k / q_w), k < 3; an endpoint
 *       with q_w = 0 (only the 4D origin is inside with w = 0) gets qNaN.
 *
 * With w0 = w1 = 1 every step is the 3D cuboid rule R1..R8 with lo = -1, hi = 1
 * (RN(1 + x) = RN(x - (-1)), q_w = fma(t, 0, 1) = 1, snap to -1 / 1, clamp into [-1, 1]),
 * which is the pin of tests/test_oracle_homog.py.
 */

#define HCAT_(a, b) a##b
#define HCAT(a, b) HCAT_(a, b)
#define HNAME(x) HCAT(x, SFX)

static int HNAME(homog_one_)(const REAL P0[4], const REAL P1[4], REAL Q0[4], REAL Q1[4],
                             HNAME(oracle_htrace_) * tr) {
  REAL bl0[3], bh0[3], bl1[3], bh1[3];   /* boundary coordinates of the six planes */
  REAL a_in[6], a_out[6];                /* per plane j = 2k (low) / 2k + 1 (high) */
  int has_in[6] = {0, 0, 0, 0, 0, 0}, has_out[6] = {0, 0, 0, 0, 0, 0};
  unsigned c0 = 0, c1 = 0;
  REAL t_in = 0, t_out = 1;
  int k;

  if (tr) memset(tr, 0, sizeof(*tr));

  /* H9 */
  for (k = 0; k < 4; ++k)
    if (!isfinite(P0[k]) || !isfinite(P1[k])) goto invisible;

  /* H1 */
  for (k = 0; k < 3; ++k) {
    bl0[k] = P0[3] + P0[k];
    bh0[k] = P0[3] - P0[k];
    bl1[k] = P1[3] + P1[k];
    bh1[k] = P1[3] - P1[k];
  }

  /* H2 */
  for (k = 0; k < 3; ++k) {
    if (bl0[k] < 0) c0 |= 1u << (2 * k);
    if (bh0[k] < 0) c0 |= 1u << (2 * k + 1);
    if (bl1[k] < 0) c1 |= 1u << (2 * k);
    if (bh1[k] < 0) c1 |= 1u << (2 * k + 1);
  }
  if (tr) { tr->c0 = c0; tr->c1 = c1; }

  /* H3 */
  if ((c0 & c1) != 0) goto invisible;
  if ((c0 | c1) == 0) {
    for (k = 0; k < 4; ++k) { Q0[k] = P0[k]; Q1[k] = P1[k]; }
    if (tr) { tr->visible = 1; tr->t_in = t_in; tr->t_out = t_out; }
    return 1;
  }

  /* H4: plane j = 2k + s (s = 0 low, 1 high); (c0 & c1) == 0, so not both outside */
  for (k = 0; k < 6; ++k) {
    const REAL b0 = (k & 1) ? bh0[k >> 1] : bl0[k >> 1];
    const REAL b1 = (k & 1) ? bh1[k >> 1] : bl1[k >> 1];
    if (c0 & (1u << k)) {
      a_in[k] = b0 / (b0 - b1);
      has_in[k] = 1;
    }
    if (c1 & (1u << k)) {
      a_out[k] = b0 / (b0 - b1);
      has_out[k] = 1;
    }
  }

  /* H5 */
  for (k = 0; k < 6; ++k)
    if (has_in[k] && a_in[k] > t_in) t_in = a_in[k];
  for (k = 0; k < 6; ++k)
    if (has_out[k] && a_out[k] < t_out) t_out = a_out[k];
  if (tr) {
    tr->t_in = t_in; tr->t_out = t_out;
    for (k = 0; k < 6; ++k) {
      tr->has_in[k] = has_in[k]; tr->has_out[k] = has_out[k];
      tr->a_in[k] = has_in[k] ? a_in[k] : 0; tr->a_out[k] = has_out[k] ? a_out[k] : 0;
    }
  }

  /* H6 */
  if (!(t_in <= t_out)) goto invisible;

  /* H7: w first (the snap and clamp bounds of the other axes are its interpolated value) */
  {
    const REAL dw = P1[3] - P0[3];
    REAL qw0, qw1;
    if (c0 == 0) {
      for (k = 0; k < 4; ++k) Q0[k] = P0[k];
    } else {
      qw0 = FMA(t_in, dw, P0[3]);
      Q0[3] = qw0;
      for (k = 0; k < 3; ++k) {
        if (has_in[2 * k] && a_in[2 * k] == t_in) {
          Q0[k] = -qw0;
        } else if (has_in[2 * k + 1] && a_in[2 * k + 1] == t_in) {
          Q0[k] = qw0;
        } else {
          const REAL q = FMA(t_in, P1[k] - P0[k], P0[k]);
          Q0[k] = (q < -qw0) ? -qw0 : (q > qw0) ? qw0 : q;
        }
      }
    }
    if (c1 == 0) {
      for (k = 0; k < 4; ++k) Q1[k] = P1[k];
    } else {
      qw1 = FMA(t_out, dw, P0[3]);
      Q1[3] = qw1;
      for (k = 0; k < 3; ++k) {
        if (has_out[2 * k] && a_out[2 * k] == t_out) {
          Q1[k] = -qw1;
        } else if (has_out[2 * k + 1] && a_out[2 * k + 1] == t_out) {
          Q1[k] = qw1;
        } else {
          const REAL q = FMA(t_out, P1[k] - P0[k], P0[k]);
          Q1[k] = (q < -qw1) ? -qw1 : (q > qw1) ? qw1 : q;
        }
      }
    }
  }
  if (tr) tr->visible = 1;
  return 1;

invisible:
  /* H8 */
  for (k = 0; k < 4; ++k) { Q0[k] = HNAME(canonical_nan_)(); Q1[k] = HNAME(canonical_nan_)(); }
  if (tr) tr->visible = 0;
  return 0;
}

/* Output rows of one clipped segment: 8 homogeneous components (x0,y0,z0,w0,x1,y1,z1,w1),
 * or with ndc the 6 divided ones (x0/w0, y0/w0, z0/w0, x1/w1, ...). */
static void HNAME(homog_put_)(const REAL Q0[4], const REAL Q1[4], int ndc, REAL* out, int64_t ld_out, int64_t row) {
  int k;
  if (ndc) {  /* an endpoint at the 4D origin (q_w = 0) has no NDC image: qNaN */
    for (k = 0; k < 3; ++k) {
      out[k * ld_out + row] = Q0[3] == 0 ? HNAME(canonical_nan_)() : Q0[k] / Q0[3];
      out[(3 + k) * ld_out + row] = Q1[3] == 0 ? HNAME(canonical_nan_)() : Q1[k] / Q1[3];
    }
  } else {
    for (k = 0; k < 4; ++k) {
      out[k * ld_out + row] = Q0[k];
      out[(4 + k) * ld_out + row] = Q1[k];
    }
  }
}

/* Dense: in has 8 planes (x0,y0,z0,w0,x1,y1,z1,w1); out 8 planes, or 6 with ndc.
 * Invisible rows are canonical qNaN (NaN / NaN is the canonical NaN again under ndc). */
int HNAME(oracle_homog_clip_)(const REAL* in, int64_t ld_in, int64_t n, REAL* out, int64_t ld_out, uint8_t* flags,
                              int ndc) {
  int64_t i;
  int k;
  if (n < 0) return -1;
  for (i = 0; i < n; ++i) {
    REAL P0[4], P1[4], Q0[4], Q1[4];
    int vis;
    for (k = 0; k < 4; ++k) { P0[k] = in[k * ld_in + i]; P1[k] = in[(4 + k) * ld_in + i]; }
    vis = HNAME(homog_one_)(P0, P1, Q0, Q1, 0);
    if (!vis && ndc) {  /* H8 holds for the divided output too */
      for (k = 0; k < 6; ++k) out[k * ld_out + i] = HNAME(canonical_nan_)();
    } else {
      HNAME(homog_put_)(Q0, Q1, ndc, out, ld_out, i);
    }
    if (flags) flags[i] = (uint8_t)vis;
  }
  return 0;
}

/* H10: the visible segments in increasing input index and their count. */
int64_t HNAME(oracle_homog_compact_)(const REAL* in, int64_t ld_in, int64_t n, REAL* out, int64_t ld_out,
                                     int64_t* out_index, int64_t index_base, uint8_t* flags, int ndc) {
  int64_t i, count = 0;
  int k;
  if (n < 0) return -1;
  for (i = 0; i < n; ++i) {
    REAL P0[4], P1[4], Q0[4], Q1[4];
    int vis;
    for (k = 0; k < 4; ++k) { P0[k] = in[k * ld_in + i]; P1[k] = in[(4 + k) * ld_in + i]; }
    vis = HNAME(homog_one_)(P0, P1, Q0, Q1, 0);
    if (flags) flags[i] = (uint8_t)vis;
    if (!vis) continue;
    HNAME(homog_put_)(Q0, Q1, ndc, out, ld_out, count);
    if (out_index) out_index[count] = index_base + i;
    ++count;
  }
  return count;
}

/* One segment p = (x0,y0,z0,w0,x1,y1,z1,w1) -> q (8 homogeneous components) + trace. */
int HNAME(oracle_homog_one_)(const REAL p[8], REAL q[8], HNAME(oracle_htrace_) * tr) {
  return HNAME(homog_one_)(p, p + 4, q, q + 4, tr);
}

#undef HNAME
#undef HCAT
#undef HCAT_
