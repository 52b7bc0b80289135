// clip_kernels.cuh — internal launcher interface between the C ABI (clip_api.cu) and
// the sm_100a kernels (clip_dense.cu, clip_compact.cu, clip_shard.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "clip_int_math.cuh"
#include "clip_math.cuh"

namespace clipseg {

// A clip operation as the kernels see it: IN input planes, OUT output planes per segment,
// the per-call parameters, and the group clip of V segments (returns the visible bits;
// NAN_FILL writes R8's qNaN into invisible rows).
// The packed compacting kernel's optional third flag value: ops whose rules give flag 2 ("out
// of range", NEXT-4 I6) report those segments here (bit v); every other op reports none.
struct NoOutOfRange {
  template <typename T, int IN, int V>
  static __device__ __forceinline__ unsigned oor(const T (&)[IN][V]) { return 0u; }
};
template <typename T, int D> struct BoxOp : NoOutOfRange {  // axis-aligned closed box, D = 2, 3 (rules R1..R10)
  static constexpr int IN = 2 * D, OUT = 2 * D;
  static constexpr int GV = 4;  // whole groups (V <= 4)
  typedef Window<T, D> Params;
  template <int V, bool NAN_FILL>
  static __device__ __forceinline__ unsigned group(const T (&pl)[IN][V], const Params& w, T (&res)[OUT][V]) {
    return clip_group<T, D, V, NAN_FILL>(pl, w, res);
  }
  // packed compacting kernel: R3 alone (bit v: segment v is not rejected) and the clip of
  // one segment R3 kept
  // R3 alone (bit v set: segment v kept); KeepParams are prepared once per launch
#ifndef CLIPSEG_PK_KEEP
#define CLIPSEG_PK_KEEP 2  // fp32 R3 test: 0 min/max compares and selects, 1 sign bits (FMA pipe + LOP3),
                           // 2 min/max and one setp chain per segment (measured 5.65 -> 5.59 ms best at 1e9)
#endif
  typedef KeepPrep<T, D> KeepParams;
  static __device__ __forceinline__ KeepParams keep_params(const Params& w) { return keep_prep<T, D>(w); }
  template <int V>
  static __device__ __forceinline__ unsigned keep(const T (&pl)[IN][V], const Params& w, const KeepParams& kp) {
    if constexpr (sizeof(T) == 4 && CLIPSEG_PK_KEEP == 1) return box_keep_sign<D, V>(pl, kp);
    else if constexpr (sizeof(T) == 4 && CLIPSEG_PK_KEEP == 2) return box_keep_pred<D, V>(pl, w);
    else return box_keep<T, D, V>(pl, w);
  }
  static __device__ __forceinline__ bool clip_one(const T (&P)[IN], const Params& w, T (&Q)[OUT]) {
    return clip_kept<T, D, false>(P, w, Q);
  }
  static __device__ __forceinline__ void clip_two(const T (&Pa)[IN], const T (&Pb)[IN], const Params& w,
                                                  T (&Qa)[OUT], T (&Qb)[OUT], bool& va, bool& vb) {
    clip_kept2<T, D, false>(Pa, Pb, w, Qa, Qb, va, vb);
  }
  template <int NI>
  static __device__ __forceinline__ void clip_n(const T (&P)[NI][IN], const Params& w, T (&Q)[NI][OUT],
                                                bool (&vis)[NI]) {
    clip_keptN<T, D, NI>(P, w, Q, vis);
  }
  // deferred exceptional segments: the fast path's range test, the fast path alone (false:
  // the segment needs the rules) and the rules alone
  static constexpr bool kFastAlwaysDone = true;  // fast_try / fast_two never decline a row that passed fast_ok
  static __device__ __forceinline__ bool fast_ok(const T (&P)[IN], const Params& w) { return box_fast_ok<T, D>(P, w); }
  static __device__ __forceinline__ bool fast_ok2(const T (&P)[IN], const Params& w) { return box_fast_ok2<T, D>(P, w); }
  static __device__ __forceinline__ bool fast_try(const T (&P)[IN], const Params& w, T (&Q)[OUT], bool& vis) {
    vis = clip_fast<T, D, false, true>(P, w, Q);
    return true;
  }
  static __device__ __forceinline__ bool fast_two(const T (&Pa)[IN], const T (&Pb)[IN], const Params& w, T (&Qa)[OUT],
                                                  T (&Qb)[OUT], bool& va, bool& vb) {
    va = clip_fast<T, D, false, true>(Pa, w, Qa);
    vb = clip_fast<T, D, false, true>(Pb, w, Qb);
    return true;
  }
  static __device__ __forceinline__ bool exact(const T (&P)[IN], const Params& w, T (&Q)[OUT]) {
    return clip_exact<T, D>(P, w, Q);
  }
};
struct NoParams {
  int unused;
};

// NEXT-4: int32 2D segments against a closed integer window, exact rules
// I1-I6 (clip_int_math.cuh).  Packed compacting kernel only (the dense call has its own kernel).
struct IntWindow {
  int4 win;   // lo.x, lo.y, hi.x, hi.y
  int small;  // every window bound within [-2^14, 2^14]: the 32-bit path is allowed
};
struct IntOp {
  typedef int32_t T;
  static constexpr int IN = 4, OUT = 4;
  typedef IntWindow Params;
  struct KeepParams {
    int unused;
  };
  static __device__ __forceinline__ KeepParams keep_params(const Params&) { return KeepParams{0}; }
  // kept: every coordinate within I1's range and not trivially rejected (I2's both-outside test,
  // exact on integers); out-of-range segments are not kept and get flag 2 (oor)
  template <int V>
  static __device__ __forceinline__ unsigned keep(const int32_t (&pl)[IN][V], const Params& w, const KeepParams&) {
    unsigned m = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int32_t x0 = pl[0][v], y0 = pl[1][v], x1 = pl[2][v], y1 = pl[3][v];
      const bool rej = (max(x0, x1) < w.win.x) | (min(x0, x1) > w.win.z) | (max(y0, y1) < w.win.y) |
                       (min(y0, y1) > w.win.w);
      m |= ((!rej & in_range(x0, y0, x1, y1)) ? 1u : 0u) << v;
    }
    return m;
  }
  template <typename TT, int IIN, int V>
  static __device__ __forceinline__ unsigned oor(const TT (&pl)[IIN][V]) {
    unsigned m = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) m |= (in_range(pl[0][v], pl[1][v], pl[2][v], pl[3][v]) ? 0u : 1u) << v;
    return m;
  }
  static __device__ __forceinline__ bool in_range(int32_t x0, int32_t y0, int32_t x1, int32_t y1) {
    // |c| <= 2^30 for all four: biased into [0, 2^31] in unsigned arithmetic
    const uint32_t b = (uint32_t)intclip::kCoordMax;
    const uint32_t m = max(max((uint32_t)x0 + b, (uint32_t)y0 + b), max((uint32_t)x1 + b, (uint32_t)y1 + b));
    return m <= 2u * b;
  }
  static __device__ __forceinline__ bool clip_one(const int32_t (&P)[IN], const Params& w, int32_t (&Q)[OUT]) {
    return intclip::clip_int_one(P[0], P[1], P[2], P[3], w.win, w.small != 0, Q) == 1u;
  }
  static __device__ __forceinline__ void clip_two(const int32_t (&Pa)[IN], const int32_t (&Pb)[IN], const Params& w,
                                                  int32_t (&Qa)[OUT], int32_t (&Qb)[OUT], bool& va, bool& vb) {
#ifndef CLIPSEG_INT_TWO
#define CLIPSEG_INT_TWO 1  // 32-bit path on both rows, then a vote (0: two per-lane branching clips)
#endif
    if constexpr (CLIPSEG_INT_TWO) {
      intclip::clip_int_two(Pa, Pb, w.win, w.small != 0, Qa, Qb, va, vb);
    } else {
      va = clip_one(Pa, w, Qa);
      vb = clip_one(Pb, w, Qb);
    }
  }
  template <int NI>
  static __device__ __forceinline__ void clip_n(const int32_t (&P)[NI][IN], const Params& w, int32_t (&Q)[NI][OUT],
                                                bool (&vis)[NI]) {
#pragma unroll
    for (int i = 0; i < NI; ++i) vis[i] = clip_one(P[i], w, Q[i]);
  }
  static constexpr bool kFastAlwaysDone = true;
  static __device__ __forceinline__ bool fast_ok(const int32_t (&)[IN], const Params&) { return true; }
  static __device__ __forceinline__ bool fast_ok2(const int32_t (&)[IN], const Params&) { return true; }
  static __device__ __forceinline__ bool fast_two(const int32_t (&Pa)[IN], const int32_t (&Pb)[IN], const Params& w,
                                                  int32_t (&Qa)[OUT], int32_t (&Qb)[OUT], bool& va, bool& vb) {
    clip_two(Pa, Pb, w, Qa, Qb, va, vb);
    return true;
  }
  static __device__ __forceinline__ bool fast_try(const int32_t (&P)[IN], const Params& w, int32_t (&Q)[OUT], bool& vis) {
    vis = clip_one(P, w, Q);
    return true;
  }
  static __device__ __forceinline__ bool exact(const int32_t (&P)[IN], const Params& w, int32_t (&Q)[OUT]) {
    return clip_one(P, w, Q);
  }
};
#ifndef CLIPSEG_HOMOG_GV_F32
#define CLIPSEG_HOMOG_GV_F32 2      // segments per group_chunked call, fp32 homogeneous output
#endif
#ifndef CLIPSEG_HOMOG_GV_F32_NDC
#define CLIPSEG_HOMOG_GV_F32_NDC 1  // ... fp32 NDC output
#endif
#ifndef CLIPSEG_HOMOG_GV_F64
#define CLIPSEG_HOMOG_GV_F64 2
#endif
template <typename T, bool NDC> struct HomogOp : NoOutOfRange {  // NEXT-1: homogeneous clip space (rules H1..H10)
  static constexpr int IN = 8, OUT = NDC ? 6 : 8;
  // Segments clipped per call: the six-plane rules of 4 segments at once need more than 128
  // registers (spills at 80: 168 B); chunks of 2 (1 with the NDC divides) do not, measured
  // at 1e8 fp32 (profiles/ab_log.md): dense 1.43 -> 1.21 ms and compacting 1.78 -> 1.56 ms
  // homogeneous output, 1.66 -> 1.30 and 2.40 -> 2.02 ms NDC output; fp64 unchanged.
  static constexpr int GV = sizeof(T) == 8 ? CLIPSEG_HOMOG_GV_F64 : (NDC ? CLIPSEG_HOMOG_GV_F32_NDC : CLIPSEG_HOMOG_GV_F32);
  typedef NoParams Params;
  template <int V, bool NAN_FILL>
  static __device__ __forceinline__ unsigned group(const T (&pl)[IN][V], const Params&, T (&res)[OUT][V]) {
    return homog_group<T, V, NAN_FILL, NDC>(pl, res);
  }
  // packed compacting kernel: H3 alone and the clip of kept segments
  struct KeepParams {
    int unused;
  };
  static __device__ __forceinline__ KeepParams keep_params(const Params&) { return KeepParams{0}; }
  template <int V>
  static __device__ __forceinline__ unsigned keep(const T (&pl)[IN][V], const Params&, const KeepParams&) {
    return homog_keep<T, V>(pl);
  }
  static __device__ __forceinline__ bool clip_one(const T (&P)[IN], const Params&, T (&Q)[OUT]) {
    return homog_kept<T, NDC>(P, Q);
  }
  static __device__ __forceinline__ void clip_two(const T (&Pa)[IN], const T (&Pb)[IN], const Params&, T (&Qa)[OUT],
                                                  T (&Qb)[OUT], bool& va, bool& vb) {
    homog_kept2<T, NDC>(Pa, Pb, Qa, Qb, va, vb);
  }
  template <int NI>
  static __device__ __forceinline__ void clip_n(const T (&P)[NI][IN], const Params&, T (&Q)[NI][OUT], bool (&vis)[NI]) {
    homog_keptN<T, NDC, NI>(P, Q, vis);
  }
  static constexpr bool kFastAlwaysDone = false;  // homog_fast may decline (a crossed endpoint's q_w <= 0)
  static __device__ __forceinline__ bool fast_ok(const T (&P)[IN], const Params&) { return homog_fast_ok<T>(P); }
  static __device__ __forceinline__ bool fast_ok2(const T (&P)[IN], const Params&) { return homog_fast_ok<T>(P); }
  static __device__ __forceinline__ bool fast_two(const T (&Pa)[IN], const T (&Pb)[IN], const Params&, T (&Qa)[OUT],
                                                  T (&Qb)[OUT], bool& va, bool& vb) {
    bool ok = true;
    T qa[8], qb[8];
    va = homog_fast<T, true>(Pa, qa, ok);
    vb = homog_fast<T, true>(Pb, qb, ok);
    if (ok) {
      homog_emit<T, false, NDC>(qa, va, Qa);
      homog_emit<T, false, NDC>(qb, vb, Qb);
    }
    return ok;
  }
  static __device__ __forceinline__ bool fast_try(const T (&P)[IN], const Params&, T (&Q)[OUT], bool& vis) {
    bool ok = true;
    T q[8];
    vis = homog_fast<T, true>(P, q, ok);
    if (ok) homog_emit<T, false, NDC>(q, vis, Q);
    return ok;
  }
  static __device__ __forceinline__ bool exact(const T (&P)[IN], const Params&, T (&Q)[OUT]) {
    return homog_segment<T, false, NDC>(P, Q);
  }
};

// Op::group over V segments in chunks of Op::GV (a power of two): bounds the live state of ops
// whose per-segment work needs many registers (the homogeneous clipper's 6 planes).
template <class Op, bool NAN_FILL, typename T, int V>
__device__ __forceinline__ unsigned group_chunked(const T (&pl)[Op::IN][V], const typename Op::Params& w,
                                                  T (&res)[Op::OUT][V]) {
  constexpr int GV = Op::GV;
  if constexpr (GV >= V) {
    return Op::template group<V, NAN_FILL>(pl, w, res);
  } else {
    unsigned bits = 0;
#pragma unroll
    for (int h = 0; h < V / GV; ++h) {
      T pg[Op::IN][GV], rg[Op::OUT][GV];
#pragma unroll
      for (int c = 0; c < Op::IN; ++c)
#pragma unroll
        for (int j = 0; j < GV; ++j) pg[c][j] = pl[c][h * GV + j];
      bits |= Op::template group<GV, NAN_FILL>(pg, w, rg) << (h * GV);
#pragma unroll
      for (int c = 0; c < Op::OUT; ++c)
#pragma unroll
        for (int j = 0; j < GV; ++j) res[c][h * GV + j] = rg[c][j];
    }
    return bits;
  }
}

// Workspace of the compacting kernel: a 128-byte header (tile-claim counter) followed by
// one 64-bit look-back status word per tile.
constexpr size_t kWsHeaderBytes = 128;

template <typename T> __host__ __device__ constexpr int vec_elems() { return 16 / (int)sizeof(T); }
// Compacting kernel: a warp sub-tile is 32 lanes x 4 segments (fp64 lanes load two
// 128-bit vectors); a block tile is compact_subtiles() sub-tiles; compact_buffers() block
// tiles are staged in shared memory at once (the copy-out lags the compute by that many
// minus one).
template <typename T> __host__ __device__ constexpr int compact_items() { return 4 / vec_elems<T>(); }
#ifndef CLIPSEG_COMPUTE_WARPS  // tuning knobs of the headline (fp32, 2D) instantiation
#define CLIPSEG_COMPUTE_WARPS 16   // compute warps per block
#endif
#ifndef CLIPSEG_NSUB_F32_2D
#define CLIPSEG_NSUB_F32_2D 32     // sub-tiles (of 128 segments) per block tile
#endif
#ifndef CLIPSEG_NBUF_F32_2D
#define CLIPSEG_NBUF_F32_2D 3      // block tiles staged in shared memory at once
#endif
#ifndef CLIPSEG_MINB_F32_2D
#define CLIPSEG_MINB_F32_2D 1      // resident blocks per SM the register budget targets
#endif
// fp32 2D (the bench workload): one block per SM, 16 compute warps, 4096-segment tiles,
// 3 staged (~203 KB); fp32 3D: 11 warps, 2816-segment tiles; fp64: 8 compute warps and
// 1024-segment tiles, so the wider rows keep enough registers; homogeneous (8 input
// planes): fp32 8 warps x 2048-segment tiles, fp64 4 warps x 1024.
template <typename T, class Op> __host__ __device__ constexpr bool compact_headline() {
  return sizeof(T) == 4 && Op::IN == 4;
}
// The other instantiations, (compute warps, sub-tiles per tile, staged tiles), measured at
// 1e8 segments (scripts/kernel_probe.py): fp32 3D 11 x 22 x 3 (1.06 ms; 12 x 24 x 3 1.19 ms: 13
// warps cap ptxas at 128 registers and spill, 12 warps allow 159; 10 x 20 1.14, 11 x 33 1.10),
// fp64 2D 8 x 16 x 2 (2.03 ms vs 2.27 at 8 x 8 x 3); homogeneous fp32 without the register
// prefetch (see compact_prefetch): 15 x 15 x 3 (1.43 ms; 12 x 24 1.51, 16 x 16 1.53, 19 x 19
// 1.75), with the NDC divides 23 x 23 x 3 (1.48 ms; 19 x 19 1.53, 15 x 15 1.69, 12 x 24 2.0).
#ifndef CLIPSEG_F32_3D_W
#define CLIPSEG_F32_3D_W 11
#endif
#ifndef CLIPSEG_F32_3D_N
#define CLIPSEG_F32_3D_N 22
#endif
#ifndef CLIPSEG_F32_3D_B
#define CLIPSEG_F32_3D_B 3
#endif
#ifndef CLIPSEG_F64_2D_W
#define CLIPSEG_F64_2D_W 8
#endif
#ifndef CLIPSEG_F64_2D_N
#define CLIPSEG_F64_2D_N 16
#endif
#ifndef CLIPSEG_F64_2D_B
#define CLIPSEG_F64_2D_B 2
#endif
#ifndef CLIPSEG_F64_3D_W
#define CLIPSEG_F64_3D_W 8
#endif
#ifndef CLIPSEG_F64_3D_N
#define CLIPSEG_F64_3D_N 8
#endif
#ifndef CLIPSEG_F64_3D_B
#define CLIPSEG_F64_3D_B 2
#endif
#ifndef CLIPSEG_F32_H_W
#define CLIPSEG_F32_H_W 15
#endif
#ifndef CLIPSEG_F32_H_N
#define CLIPSEG_F32_H_N 15
#endif
#ifndef CLIPSEG_F32_HN_W  // homogeneous fp32 with the NDC divides (6 output planes)
#define CLIPSEG_F32_HN_W 23
#endif
#ifndef CLIPSEG_F32_HN_N
#define CLIPSEG_F32_HN_N 23
#endif
#ifndef CLIPSEG_F32_H_B
#define CLIPSEG_F32_H_B 3
#endif
#ifndef CLIPSEG_F64_H_W
#define CLIPSEG_F64_H_W 4
#endif
#ifndef CLIPSEG_F64_H_N
#define CLIPSEG_F64_H_N 8
#endif
#ifndef CLIPSEG_F64_H_B
#define CLIPSEG_F64_H_B 3
#endif
struct CompactKnobs {
  int warps, nsub, nbuf;
};
template <typename T, class Op> __host__ __device__ constexpr CompactKnobs compact_knobs() {
  return compact_headline<T, Op>() ? CompactKnobs{CLIPSEG_COMPUTE_WARPS, CLIPSEG_NSUB_F32_2D, CLIPSEG_NBUF_F32_2D}
         : Op::IN == 8 ? (sizeof(T) == 4 ? (Op::OUT == 6 ? CompactKnobs{CLIPSEG_F32_HN_W, CLIPSEG_F32_HN_N, CLIPSEG_F32_H_B}
                                                          : CompactKnobs{CLIPSEG_F32_H_W, CLIPSEG_F32_H_N, CLIPSEG_F32_H_B})
                                         : CompactKnobs{CLIPSEG_F64_H_W, CLIPSEG_F64_H_N, CLIPSEG_F64_H_B})
         : Op::IN == 6 ? (sizeof(T) == 4 ? CompactKnobs{CLIPSEG_F32_3D_W, CLIPSEG_F32_3D_N, CLIPSEG_F32_3D_B}
                                         : CompactKnobs{CLIPSEG_F64_3D_W, CLIPSEG_F64_3D_N, CLIPSEG_F64_3D_B})
                       : CompactKnobs{CLIPSEG_F64_2D_W, CLIPSEG_F64_2D_N, CLIPSEG_F64_2D_B};
}
template <typename T, class Op> __host__ __device__ constexpr int compact_warps() {
  return compact_knobs<T, Op>().warps;
}
template <typename T, class Op> __host__ __device__ constexpr int compact_subtiles() {
  return compact_knobs<T, Op>().nsub;
}
template <typename T, class Op> __host__ __device__ constexpr int compact_buffers() {
  return compact_knobs<T, Op>().nbuf;
}
#ifndef CLIPSEG_HOMOG_PREFETCH
#define CLIPSEG_HOMOG_PREFETCH 0
#endif
// Next-sub-tile loads in flight in a second register buffer — except for fp32 homogeneous
// rows (8 planes), whose registers buy more warps instead: 12 x 24 without the prefetch
// 1.77 ms vs 8 x 16 with it 1.79 ms at 1e8.
#ifndef CLIPSEG_F32_3D_PREFETCH
#define CLIPSEG_F32_3D_PREFETCH 1
#endif
#ifndef CLIPSEG_F32_2D_PREFETCH
#define CLIPSEG_F32_2D_PREFETCH 1
#endif
template <typename T, class Op> __host__ __device__ constexpr bool compact_prefetch() {
  return Op::IN == 8 && sizeof(T) == 4   ? CLIPSEG_HOMOG_PREFETCH != 0
         : Op::IN == 6 && sizeof(T) == 4 ? CLIPSEG_F32_3D_PREFETCH != 0
         : Op::IN == 4 && sizeof(T) == 4 ? CLIPSEG_F32_2D_PREFETCH != 0
                                         : true;
}
// Packed compacting kernel (clip_compact.cu): warp batches of PW sub-tiles; R3-rejected
// segments are dropped before the clip and the kept ones are clipped 32 at a time, one
// per lane.  Knobs: compute warps, sub-tiles per warp batch, staged tiles.
#ifndef CLIPSEG_PACKED_F32_2D
#define CLIPSEG_PACKED_F32_2D 1
#endif
#ifndef CLIPSEG_PK_WARPS
#define CLIPSEG_PK_WARPS 15
#endif
#ifndef CLIPSEG_PK_PW
#define CLIPSEG_PK_PW 2
#endif
#ifndef CLIPSEG_PK_ILP
#define CLIPSEG_PK_ILP 2  // kept rows clipped per lane per round while more than 32 remain
#endif
#ifndef CLIPSEG_PK_NBUF
#define CLIPSEG_PK_NBUF 3
#endif
// fp32 3D cuboid (C4): rows of 24 B; 10 compute warps with two sub-tiles (256 segments) per
// batch (staging 10 warps x 3 x 6 KB, 156 registers for the 48-float prefetch) measured
// 0.875 -> 0.832 ms at 1e8 against 15 warps x 128 segments (9 / 11 / 12 warps x 256: 0.93 /
// 0.887 / 0.894; two rows per lane: 0.8325; after the synchronisation clean-up 9 / 11 / 12
// warps x 256: 0.873 / 0.879 / 0.958 vs 0.775).
#ifndef CLIPSEG_PACKED_F32_3D
#define CLIPSEG_PACKED_F32_3D 1
#endif
#ifndef CLIPSEG_PK3_WARPS
#define CLIPSEG_PK3_WARPS 10
#endif
#ifndef CLIPSEG_PK3_PW
#define CLIPSEG_PK3_PW 2
#endif
#ifndef CLIPSEG_PK3_NBUF
#define CLIPSEG_PK3_NBUF 3
#endif
// fp32 homogeneous (NEXT-1): rows of 32 B, one sub-tile per warp batch (6 / 7 / 8 warps with
// two sub-tiles measured 1.43 / 1.25 / 1.33 ms against 1.15 at 1e8; 13 / 14 warps x 128:
// 1.30 / 1.23).
#ifndef CLIPSEG_PACKED_F32_H
#define CLIPSEG_PACKED_F32_H 1
#endif
#ifndef CLIPSEG_PKH_WARPS
#define CLIPSEG_PKH_WARPS 15
#endif
#ifndef CLIPSEG_PKH_PW
#define CLIPSEG_PKH_PW 1
#endif
#ifndef CLIPSEG_PKH_ILP
#define CLIPSEG_PKH_ILP CLIPSEG_PK_ILP
#endif
#ifndef CLIPSEG_PKH_NBUF
#define CLIPSEG_PKH_NBUF 3
#endif
// fp64 cuboids: 2D rows of 32 B, two sub-tiles of 64 segments per warp batch.
#ifndef CLIPSEG_PACKED_F64_2D
#define CLIPSEG_PACKED_F64_2D 1
#endif
#ifndef CLIPSEG_PKD_WARPS
#define CLIPSEG_PKD_WARPS 11
#endif
#ifndef CLIPSEG_PKD_PW
#define CLIPSEG_PKD_PW 2
#endif
template <typename T, class Op> __host__ __device__ constexpr bool compact_packed() {
  return (compact_headline<T, Op>() && CLIPSEG_PACKED_F32_2D != 0) ||
         (sizeof(T) == 4 && Op::IN == 6 && Op::OUT == 6 && CLIPSEG_PACKED_F32_3D != 0) ||
         (sizeof(T) == 4 && Op::IN == 8 && CLIPSEG_PACKED_F32_H != 0) ||
         (sizeof(T) == 8 && Op::IN == 4 && Op::OUT == 4 && CLIPSEG_PACKED_F64_2D != 0) ||
         std::is_same<Op, IntOp>::value;
}
// (compute warps, sub-tiles per warp batch, staged tiles, kept rows per lane per round),
// measured (scripts/ab.sh): two rows per lane pay for 2D fp32 (5.9 -> 5.6 ms at 1e9) and
// homogeneous fp32 (1.21 -> 1.17 ms at 1e8); one is faster for 3D fp32 (0.92 -> 0.89 ms)
// and fp64 (adversarial 0.72 -> 0.58 ms at 1e7).
struct PackedKnobs {
  int warps, pw, nbuf, ilp;
  bool defer;    // exceptional rows end the fast rounds and are finished in deferred passes
  bool b0tiles;  // block 0 processes tiles too, its scan warp interleaving the global scanner
  bool vfirst;   // deferred rounds vote on the range test before clipping (fp64: a wasted round costs
                 // C3 fp64 0.52 -> 0.61 ms at 1e7; fp32 clips first, see clip_compact.cu)
};
// Block 0 taking tiles (its scan warp runs the global scanner and its own tile duties,
// non-blocking): measured the headline 5.586 -> 5.624 ms best at 1e9 — the scanner, on whose
// latency every copy-out waits, then shares its SM with the compute warps — and, once the
// hot loop lost its needless warp synchronisation, 3D 0.775 -> 0.798 ms at 1e8 (before:
// 0.834 -> 0.829).  Off.
#ifndef CLIPSEG_PK_B0TILES
#define CLIPSEG_PK_B0TILES 0
#endif
#ifndef CLIPSEG_PK3_B0TILES
#define CLIPSEG_PK3_B0TILES 0
#endif
#ifndef CLIPSEG_PK_COPYW
#define CLIPSEG_PK_COPYW 0  // copy warps in the service warpgroup (0: compute warps copy their own batches)
#endif
#ifndef CLIPSEG_PK_REG_C
#define CLIPSEG_PK_REG_C 112  // registers per compute thread with copy warps (setmaxnreg)
#endif
#ifndef CLIPSEG_PK_REG_S
#define CLIPSEG_PK_REG_S 32   // registers per service thread with copy warps (512 x REG_C + 128 x REG_S <= 640 x 96: the CTA pool)
#endif
#ifndef CLIPSEG_PK_DEFER
#define CLIPSEG_PK_DEFER 1  // deferred passes for 2D fp32 / fp64 (measured: C3 fp32 1e7 0.237 -> 0.155 ms,
#endif                      // fp64 0.580 -> 0.523, headline unchanged)
#ifndef CLIPSEG_PK3_DEFER
#define CLIPSEG_PK3_DEFER 1  // 3D fp32 (10 warps x 256): with deferral and two rows per lane C4 0.801 -> 0.794 ms
#endif                       // (deferral alone 0.817, two rows alone 0.805)
#ifndef CLIPSEG_PKH_DEFER
#define CLIPSEG_PKH_DEFER 0  // homogeneous fp32: 1.17 -> 1.49 ms with deferral (spills)
#endif
#ifndef CLIPSEG_PK3_ILP
#define CLIPSEG_PK3_ILP 2
#endif
#ifndef CLIPSEG_PKD_ILP
#define CLIPSEG_PKD_ILP 1
#endif
template <typename T, class Op> __host__ __device__ constexpr PackedKnobs packed_knobs() {
  return Op::IN == 8      ? PackedKnobs{CLIPSEG_PKH_WARPS, CLIPSEG_PKH_PW, CLIPSEG_PKH_NBUF, CLIPSEG_PKH_ILP,
                                     CLIPSEG_PKH_DEFER != 0, CLIPSEG_PK_B0TILES != 0, false}
         : Op::IN == 6    ? PackedKnobs{CLIPSEG_PK3_WARPS, CLIPSEG_PK3_PW, CLIPSEG_PK3_NBUF, CLIPSEG_PK3_ILP,
                                     CLIPSEG_PK3_DEFER != 0, CLIPSEG_PK3_B0TILES != 0, false}
         : sizeof(T) == 8 ? PackedKnobs{CLIPSEG_PKD_WARPS, CLIPSEG_PKD_PW, 3, CLIPSEG_PKD_ILP, CLIPSEG_PK_DEFER != 0,
                                        CLIPSEG_PK_B0TILES != 0, true}
                          : PackedKnobs{CLIPSEG_PK_WARPS, CLIPSEG_PK_PW, CLIPSEG_PK_NBUF, CLIPSEG_PK_ILP,
                                        CLIPSEG_PK_DEFER != 0 && !std::is_same<Op, IntOp>::value,
                                        CLIPSEG_PK_B0TILES != 0, false};
}
template <typename T, class Op> __host__ __device__ constexpr int compact_min_blocks() {
  return compact_headline<T, Op>() ? CLIPSEG_MINB_F32_2D : 1;
}
// Smallest block tile over all (T, D) and both compacting kernels: the workspace is sized with it.
constexpr int64_t kMinCompactTile = 8 * 128;

template <typename T, class Op>
cudaError_t launch_dense(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                         int64_t ld_out, uint8_t* flags, cudaStream_t s);

template <typename T, class Op>
cudaError_t launch_compact(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                           int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags, int64_t* d_count,
                           void* ws, cudaStream_t s);

cudaError_t launch_shard_offsets(const int64_t* d_counts, int P, int rank, int64_t* d_offset, int64_t* d_total,
                                 cudaStream_t s);

// NEXT-2 (tof_range.cu): range clip + phi over batched frames of ppf pixels.
cudaError_t launch_tof_range_phi(const float* d, const float* I, int64_t n, int64_t ppf, const float* ranges,
                                 float* phi, uint8_t* code, int* kept, cudaStream_t s);

// NEXT-3 (cluster.cu): round-synchronous mutual-best region merging of nframes H x W frames.
// Two schedules (measured, scripts/cluster_probe.py, 204^2 frames): small batches run every
// round grid-wide (all SMs on each frame's rounds: 11.6 ms for 1 frame, 1.70 ms per frame at
// 16, 0.98 at 47), batches of >= kClusterPerFrameMin frames give each frame its own
// 1024-thread block with block barriers (1.03 ms per frame at 48, 0.79 at 64, 0.34 at 296).
// Each schedule processes at most cluster_part_frames() frames per launch; the workspace
// holds one part.
constexpr int64_t kClusterPerFrameMin = 64;
constexpr int64_t kClusterGridFrames = 64;
constexpr int64_t kClusterBlockFrames = 592;
__host__ __device__ constexpr int64_t cluster_part_frames(int64_t nframes) {
  return nframes >= kClusterPerFrameMin ? (nframes < kClusterBlockFrames ? nframes : kClusterBlockFrames)
                                        : (nframes < kClusterGridFrames ? nframes : kClusterGridFrames);
}
size_t cluster_workspace_bytes(int64_t n);
cudaError_t launch_cluster(const float* z, const float* phi, const uint8_t* valid, int64_t nframes, int H, int W,
                           double t_z, double t_phi, double alpha_z, double alpha_phi, int max_rounds, int* labels,
                           int* nregions, int* rounds_out, void* ws, cudaStream_t s);

// NEXT-4 (clip_int.cu): int32 2D segments, exact rational clipping, round-half-up endpoints.
cudaError_t launch_clip_int(const int32_t* in, int64_t ld_in, int64_t n, const int32_t lo[2], const int32_t hi[2],
                            int32_t* out, int64_t ld_out, uint8_t* flags, cudaStream_t s);

// Number of SMs of the current device (cached per device).
int device_sm_count();
// Resident blocks per SM of `kern` with `threads` threads and `smem` dynamic shared bytes on
// the current device, after raising the kernel's dynamic shared-memory limit on that device
// when smem > 48 KB.  Cached per (kernel, device); thread-safe.  Fails (no launch possible)
// rather than guessing when the kernel cannot be resident.
cudaError_t kernel_occupancy(const void* kern, int threads, size_t smem, int* blocks_per_sm);

}  // namespace clipseg
