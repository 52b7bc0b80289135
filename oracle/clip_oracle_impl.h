/* oracle/clip_oracle_impl.h — the CLIP-R rules for one floating type.
 *
 * TEST INFRASTRUCTURE ONLY (see clip_oracle.c).  Included twice by clip_oracle.c,
 * once with REAL=float and once with REAL=double; SFX is the name suffix,
 * FMA the correctly rounded fused multiply-add of <math.h> (fmaf / fma).
 *
 * Every rule below is numbered as in DESIGN.md §3 "Readings" (R1..R10), which
 * restates SURVEY.md §8(c) rules CLIP-R.  The paper gives only the
 * vocabulary: \clip, \outcode, \wec / \WEC
 * (PAPER.md:29-30), and its only clip is the closed interval [r_min, r_max]
 * (§5.2), which fixes the window as CLOSED.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define NAME(x) CAT(x, SFX)

/* The one segment-level procedure.  P0, P1, Q0, Q1 have `dim` coordinates.
 * Returns 1 if visible, else 0.  `tr` (nullable) receives the intermediate values. */
static int NAME(clip_one_)(int dim, const REAL lo[], const REAL hi[], const REAL P0[], const REAL P1[],
                          REAL Q0[], REAL Q1[], NAME(oracle_trace_) * tr) {
  REAL wl0[3], wh0[3], wl1[3], wh1[3];   /* window-edge coordinates */
  REAL a_in[3], a_out[3];                /* WEC intersection parameters alpha */
  int has_in[3] = {0, 0, 0}, has_out[3] = {0, 0, 0};
  unsigned c0 = 0, c1 = 0;               /* outcodes */
  REAL t_in = 0, t_out = 1;
  int k;

  if (tr) memset(tr, 0, sizeof(*tr));

  /* R9: a non-finite coordinate makes the segment invisible (out of contract, defined). */
  for (k = 0; k < dim; ++k)
    if (!isfinite(P0[k]) || !isfinite(P1[k])) goto invisible;

  /* R1: window-edge coordinates, wl = p - lo (>= 0 inside the low edge), wh = hi - p. */
  for (k = 0; k < dim; ++k) {
    wl0[k] = P0[k] - lo[k];
    wh0[k] = hi[k] - P0[k];
    wl1[k] = P1[k] - lo[k];
    wh1[k] = hi[k] - P1[k];
  }

  /* R2: outcode bit 2k = outside the low edge of axis k, bit 2k+1 = outside the high edge
   * (L=1, R=2, B=4, T=8, N=16, F=32).  "Outside" is a negative WEC: the window is closed. */
  for (k = 0; k < dim; ++k) {
    if (wl0[k] < 0) c0 |= 1u << (2 * k);
    if (wh0[k] < 0) c0 |= 1u << (2 * k + 1);
    if (wl1[k] < 0) c1 |= 1u << (2 * k);
    if (wh1[k] < 0) c1 |= 1u << (2 * k + 1);
  }
  if (tr) { tr->c0 = c0; tr->c1 = c1; }

  /* R3: trivial reject (both endpoints outside one edge) and trivial accept (both inside). */
  if ((c0 & c1) != 0) goto invisible;
  if ((c0 | c1) == 0) {
    for (k = 0; k < dim; ++k) { Q0[k] = P0[k]; Q1[k] = P1[k]; }
    if (tr) { tr->visible = 1; tr->t_in = t_in; tr->t_out = t_out; }
    return 1;
  }

  /* R4: WEC intersection.  For an edge e with P0 outside it (entering) or P1 outside it
   * (exiting), alpha = w0 / (w0 - w1) where w0, w1 are the two endpoints' WECs for e. */
  for (k = 0; k < dim; ++k) {
    if (c0 & (3u << (2 * k))) {               /* P0 outside on axis k: entering */
      const int low = wl0[k] < 0;
      const REAL w0 = low ? wl0[k] : wh0[k];
      const REAL w1 = low ? wl1[k] : wh1[k];
      a_in[k] = w0 / (w0 - w1);
      has_in[k] = 1;
    }
    if (c1 & (3u << (2 * k))) {               /* P1 outside on axis k: exiting */
      const int low = wl1[k] < 0;
      const REAL w0 = low ? wl0[k] : wh0[k];
      const REAL w1 = low ? wl1[k] : wh1[k];
      a_out[k] = w0 / (w0 - w1);
      has_out[k] = 1;
    }
  }

  /* R5: t_in = max(0, entering alphas), t_out = min(1, exiting alphas), in axis order. */
  for (k = 0; k < dim; ++k)
    if (has_in[k] && a_in[k] > t_in) t_in = a_in[k];
  for (k = 0; k < dim; ++k)
    if (has_out[k] && a_out[k] < t_out) t_out = a_out[k];
  if (tr) {
    tr->t_in = t_in; tr->t_out = t_out;
    for (k = 0; k < dim; ++k) {
      tr->has_in[k] = has_in[k]; tr->has_out[k] = has_out[k];
      tr->a_in[k] = has_in[k] ? a_in[k] : 0; tr->a_out[k] = has_out[k] ? a_out[k] : 0;
    }
  }

  /* R6: visible iff the parameter range is non-empty (touching counts: closed window). */
  if (!(t_in <= t_out)) goto invisible;

  /* R7: endpoints.  An inside endpoint is copied.  A crossed endpoint snaps to the edge
   * on every axis whose alpha decided t; the other axes take fma(t, p1 - p0, p0),
   * clamped into the window by comparisons. */
  for (k = 0; k < dim; ++k) {
    const REAL d = P1[k] - P0[k];
    REAL q;
    if (c0 == 0) Q0[k] = P0[k];
    else if (has_in[k] && a_in[k] == t_in) Q0[k] = (wl0[k] < 0) ? lo[k] : hi[k];
    else {
      q = FMA(t_in, d, P0[k]);
      Q0[k] = (q < lo[k]) ? lo[k] : (q > hi[k]) ? hi[k] : q;
    }
    if (c1 == 0) Q1[k] = P1[k];
    else if (has_out[k] && a_out[k] == t_out) Q1[k] = (wl1[k] < 0) ? lo[k] : hi[k];
    else {
      q = FMA(t_out, d, P0[k]);
      Q1[k] = (q < lo[k]) ? lo[k] : (q > hi[k]) ? hi[k] : q;
    }
  }
  if (tr) tr->visible = 1;
  return 1;

invisible:
  /* R8: an invisible segment's outputs are the canonical quiet NaN, flag 0. */
  for (k = 0; k < dim; ++k) { Q0[k] = NAME(canonical_nan_)(); Q1[k] = NAME(canonical_nan_)(); }
  if (tr) tr->visible = 0;
  return 0;
}

/* Dense: every segment, planar layout in[c*ld_in + i], c = e*dim + k. */
int NAME(oracle_clip_)(int dim, const REAL lo[3], const REAL hi[3], const REAL* in, int64_t ld_in, int64_t n,
                       REAL* out, int64_t ld_out, uint8_t* flags) {
  int64_t i;
  int k;
  if (!window_ok_(dim) || n < 0) return -1;
  for (k = 0; k < dim; ++k)
    if (!isfinite(lo[k]) || !isfinite(hi[k]) || !(lo[k] <= hi[k])) return -1;
  for (i = 0; i < n; ++i) {
    REAL P0[3], P1[3], Q0[3], Q1[3];
    int vis;
    for (k = 0; k < dim; ++k) { P0[k] = in[k * ld_in + i]; P1[k] = in[(dim + k) * ld_in + i]; }
    vis = NAME(clip_one_)(dim, lo, hi, P0, P1, Q0, Q1, 0);
    for (k = 0; k < dim; ++k) { out[k * ld_out + i] = Q0[k]; out[(dim + k) * ld_out + i] = Q1[k]; }
    if (flags) flags[i] = (uint8_t)vis;
  }
  return 0;
}

/* R10 compaction: the visible segments in increasing input index, and their count.
 * out_index (nullable) receives index_base + i for each kept segment i. */
int64_t NAME(oracle_compact_)(int dim, const REAL lo[3], const REAL hi[3], const REAL* in, int64_t ld_in,
                              int64_t n, REAL* out, int64_t ld_out, int64_t* out_index, int64_t index_base,
                              uint8_t* flags) {
  int64_t i, count = 0;
  int k;
  if (!window_ok_(dim) || n < 0) return -1;
  for (k = 0; k < dim; ++k)
    if (!isfinite(lo[k]) || !isfinite(hi[k]) || !(lo[k] <= hi[k])) return -1;
  for (i = 0; i < n; ++i) {
    REAL P0[3], P1[3], Q0[3], Q1[3];
    int vis;
    for (k = 0; k < dim; ++k) { P0[k] = in[k * ld_in + i]; P1[k] = in[(dim + k) * ld_in + i]; }
    vis = NAME(clip_one_)(dim, lo, hi, P0, P1, Q0, Q1, 0);
    if (flags) flags[i] = (uint8_t)vis;
    if (!vis) continue;
    for (k = 0; k < dim; ++k) { out[k * ld_out + count] = Q0[k]; out[(dim + k) * ld_out + count] = Q1[k]; }
    if (out_index) out_index[count] = index_base + i;
    ++count;
  }
  return count;
}

/* One segment with its trace (t_in, t_out, alphas, outcodes), for worked examples. */
int NAME(oracle_clip_one_)(int dim, const REAL lo[3], const REAL hi[3], const REAL p[6], REAL q[6],
                           NAME(oracle_trace_) * tr) {
  if (!window_ok_(dim)) return -1;
  return NAME(clip_one_)(dim, lo, hi, p, p + dim, q, q + dim, tr);
}

#undef NAME
#undef CAT
#undef CAT_
