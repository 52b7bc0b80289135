/* oracle/clip_oracle.c — plain, slow, scalar CPU oracle of the segment-clipping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg / `--impl reference` arm may load or call this library.  The
 * product path (paper_1110_5450_b200/, libclipseg.so) never touches it; the two share
 * no code, headers or constants.
 *
 * What it computes: batched clipping of line segments against an axis-aligned CLOSED
 * window, by outcode classification with trivial accept/reject and the window-edge-
 * coordinate (WEC) intersection, written rule by rule (R1..R10 in clip_oracle_impl.h;
 * DESIGN.md §3 states each rule and the reading behind it).  PAPER.md defines no
 * clipping algorithm — it only names \clip, \outcode, \wec, \WEC
 * — so the rules are the textbook ones those names denote.
 *
 * Arithmetic: IEEE-754 binary32 / binary64, round-to-nearest-even, subnormals honoured.
 * Build with -ffp-contract=off and without fast-math: the only fused operation is the
 * explicit fma of R7.  Pins: tests/test_oracle_*.py (worked examples, exact rational
 * reference, exact grid classifier, brute-force sampling, closed forms, invariants,
 * metamorphic relations, an independent iterative Cohen-Sutherland clipper).
 *
 * NEXT-1 (clip_homog_impl.h): the same procedure in homogeneous clip space, -w <= x, y, z
 * <= w (Blinn & Newell's boundary coordinates), rules H1..H10; pinned by its reduction to
 * the 3D cuboid rules at w = 1 and by tests/test_oracle_homog.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  unsigned c0, c1;
  int visible;
  float t_in, t_out;
  float a_in[3], a_out[3];
  int has_in[3], has_out[3];
} oracle_trace_f32;

typedef struct {
  unsigned c0, c1;
  int visible;
  double t_in, t_out;
  double a_in[3], a_out[3];
  int has_in[3], has_out[3];
} oracle_trace_f64;

/* NEXT-1 trace: six planes (j = 2k low, 2k + 1 high) */
typedef struct {
  unsigned c0, c1;
  int visible;
  float t_in, t_out;
  float a_in[6], a_out[6];
  int has_in[6], has_out[6];
} oracle_htrace_f32;

typedef struct {
  unsigned c0, c1;
  int visible;
  double t_in, t_out;
  double a_in[6], a_out[6];
  int has_in[6], has_out[6];
} oracle_htrace_f64;

static int window_ok_(int dim) { return dim == 2 || dim == 3; }

static float canonical_nan_f32(void) {
  const uint32_t b = 0x7FC00000u;
  float r;
  memcpy(&r, &b, 4);
  return r;
}

static double canonical_nan_f64(void) {
  const uint64_t b = 0x7FF8000000000000ull;
  double r;
  memcpy(&r, &b, 8);
  return r;
}

#define REAL float
#define SFX f32
#define FMA fmaf
#include "clip_oracle_impl.h"
#include "clip_homog_impl.h"
#undef REAL
#undef SFX
#undef FMA

#define REAL double
#define SFX f64
#define FMA fma
#include "clip_oracle_impl.h"
#include "clip_homog_impl.h"
#undef REAL
#undef SFX
#undef FMA
