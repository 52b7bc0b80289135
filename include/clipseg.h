/* include/clipseg.h — C ABI of the B200 segment-clipping library (libclipseg.so).
 *
 * The operation.  Batched clipping of line segments P0P1 against an axis-aligned,
 * CLOSED window [lo, hi] (2D or 3D) by outcode ("region code") classification with
 * trivial accept / trivial reject and the window-edge-coordinate (WEC) intersection
 * alpha = WEC(P0) / (WEC(P0) - WEC(P1)), producing each segment's clipped endpoints
 * and its visible flag, plus a stable compacting variant that returns only the visible
 * segments and their count.  PAPER.md names the operation only through its macros
 * \clip, \outcode, \wec, \WEC; its one clip is the closed
 * interval [r_min, r_max] of §5.2, which fixes "closed".  The exact
 * rule set (R1-R10: WEC, outcode bits, trivial cases, alpha per straddled edge,
 * t_in/t_out, visibility, endpoint snap/fma/clamp, canonical NaN, non-finite inputs,
 * stable compaction) is DESIGN.md §3 / SURVEY.md §8(c); results are bit-identical to
 * the CPU oracle (oracle/clip_oracle.c) on every input.
 *
 * Layout.  Planar structure-of-arrays: 2*dim planes of `ld` elements, plane
 * c = e*dim + k holds coordinate k of endpoint e, i.e. x0, y0, [z0], x1, y1, [z1];
 * segment i's coordinate sits at ptr[c*ld + i].  Requirements (else CLIP_EALIGN):
 * base pointers 16-byte aligned, ld*sizeof(element) a multiple of 16, ld >= n
 * (all ld elements of every plane must be addressable: kernels may read, never
 * write, the padding between n and ld); flags 4-byte aligned; out_index 8-byte aligned.
 * clip_plane_stride(n) gives the canonical ld (n rounded up to 32 elements, >= 32).
 *
 * Memory and streams.  Every pointer is a DEVICE pointer unless its name starts with
 * h_ or its comment says host; `win` is always a host pointer (copied into kernel
 * parameters).  Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream), except clip_segments_compact_host_* which returns when done.  The
 * caller owns every buffer, including workspaces; the library never allocates or
 * frees, keeps no state beyond cached device attributes, and is reentrant.
 *
 * Errors.  Functions return CLIP_OK (0) or a negative clip_status and never throw.
 * n < 0, a required pointer NULL, dim not in {2,3}, a non-finite window or lo > hi
 * -> CLIP_EINVAL (lo == hi is allowed: a degenerate window).  Misalignment ->
 * CLIP_EALIGN.  Workspace/staging too small -> CLIP_ENOSPACE.  A CUDA launch or
 * runtime error -> CLIP_ECUDA.  n == 0 is CLIP_OK with no kernel launch.
 */
#ifndef CLIPSEG_H_
#define CLIPSEG_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CLIP_OK = 0,
  CLIP_EINVAL = -1,
  CLIP_EALIGN = -2,
  CLIP_ENOSPACE = -3,
  CLIP_ECUDA = -4
} clip_status;

/* The clip window: lo[k] <= hi[k] for k < dim; entries k >= dim are ignored. */
typedef struct { float lo[3], hi[3]; int dim; } clip_window_f32;
typedef struct { double lo[3], hi[3]; int dim; } clip_window_f64;

/* Canonical plane stride (elements) for n segments: n rounded up to a multiple of 32, >= 32. */
int64_t clip_plane_stride(int64_t n);

/* Human-readable name of a status code (static string). */
const char* clip_status_string(int status);

/* ---- Dense clip (rules R1-R9): every segment -> clipped endpoints + flag --------------
 * in:    2*dim planes (ld_in), n segments.
 * out:   2*dim planes (ld_out); row i = clipped Q0,Q1 of segment i if visible, else the
 *        canonical quiet NaN (0x7FC00000 / 0x7FF8000000000000) in every plane.
 *        out == in (same ld) is allowed: each thread reads its segments before writing;
 *        any other overlap of out with in -> CLIP_EINVAL.
 * flags: n bytes (nullable): 1 visible, 0 invisible. */
int clip_segments_f32(const float* in, int64_t ld_in, int64_t n, const clip_window_f32* win,
                      float* out, int64_t ld_out, uint8_t* flags, void* stream);
int clip_segments_f64(const double* in, int64_t ld_in, int64_t n, const clip_window_f64* win,
                      double* out, int64_t ld_out, uint8_t* flags, void* stream);

/* ---- Stable compacting clip (R1-R10), one pass with a decoupled look-back scan --------
 * out:       2*dim planes (ld_out >= n): rows [0, count) hold the visible segments' clipped
 *            endpoints in increasing input index; rows >= count are not written.
 *            out must not overlap in.
 * out_index: (nullable) int64[count]: index_base + input index of each kept segment.
 * flags:     (nullable) n bytes, as in the dense call.
 * d_count:   one int64 in device memory receiving count (the caller synchronises).
 * workspace: device scratch of clip_compact_workspace_bytes(n) bytes (tile-claim counter
 *            and per-tile look-back status words).  It must be ZERO-FILLED before its first
 *            use (e.g. cudaMemsetAsync); every successful call leaves it zero-filled again,
 *            so one workspace serves any number of calls issued in order on one stream and
 *            a call is a single kernel launch (no per-call memset).  Calls that may run
 *            concurrently need distinct workspaces.  After a failed call, zero it again. */
size_t clip_compact_workspace_bytes(int64_t n);
int clip_segments_compact_f32(const float* in, int64_t ld_in, int64_t n, const clip_window_f32* win,
                              float* out, int64_t ld_out, int64_t* out_index, int64_t index_base,
                              uint8_t* flags, int64_t* d_count, void* workspace, size_t workspace_bytes,
                              void* stream);
int clip_segments_compact_f64(const double* in, int64_t ld_in, int64_t n, const clip_window_f64* win,
                              double* out, int64_t ld_out, int64_t* out_index, int64_t index_base,
                              uint8_t* flags, int64_t* d_count, void* workspace, size_t workspace_bytes,
                              void* stream);

/* ---- Sharded mode: global offsets from the per-shard visible counts ------------------
 * d_counts: P int64 counts (the allgathered c_r, rank order).  Writes
 * *d_offset = sum_{r' < rank} c_r' and *d_total = sum_r c_r (both device int64).
 * P >= 1, 0 <= rank < P, else CLIP_EINVAL. */
int clip_shard_offsets(const int64_t* d_counts, int P, int rank, int64_t* d_offset, int64_t* d_total,
                       void* stream);

/* ---- End-to-end compacting clip from/to HOST buffers (pipelined, blocking) ------------
 * h_in:    host planes (ld_in) of n segments; pinned (page-locked) memory gives full PCIe
 *          bandwidth, pageable memory works but serialises the copies.
 * h_out:   host planes (ld_out >= n) receiving rows [0, count) as in the device call.
 * h_flags: (nullable) n host bytes.  h_count: host int64 receiving count.
 * The input is streamed through the device in chunks of `chunk` segments: the H2D copy of
 * chunk j+1, the clip of chunk j and the D2H copy of chunk j-1 overlap on three streams.
 * d_staging: device scratch of clip_host_staging_bytes(dim, elem_bytes, chunk) bytes.
 * Returns when all results are in host memory (synchronises its own streams only). */
size_t clip_host_staging_bytes(int dim, int elem_bytes, int64_t chunk);
int clip_segments_compact_host_f32(const float* h_in, int64_t ld_in, int64_t n, const clip_window_f32* win,
                                   float* h_out, int64_t ld_out, uint8_t* h_flags, int64_t* h_count,
                                   int64_t chunk, void* d_staging, size_t staging_bytes);
int clip_segments_compact_host_f64(const double* h_in, int64_t ld_in, int64_t n, const clip_window_f64* win,
                                   double* h_out, int64_t ld_out, uint8_t* h_flags, int64_t* h_count,
                                   int64_t chunk, void* d_staging, size_t staging_bytes);

/* ---- NEXT-1: segments in homogeneous clip space (rules H1-H10) --------
 * The clip volume is the closed -w <= x, y, z <= w (Blinn & Newell; the textbook home of
 * the window-edge coordinates \wec / \WEC that PAPER.md:29-30 names).
 * in:    8 planes (ld_in): x0, y0, z0, w0, x1, y1, z1, w1.
 * ndc:   0 -> out has 8 planes: the clipped homogeneous endpoints (copied when inside,
 *             interpolated with the crossed plane snapped to -q_w / q_w and the other axes
 *             clamped into [-q_w, q_w] otherwise);
 *        1 -> out has 6 planes: the perspective-divided endpoints q_k / q_w (qNaN for an
 *             endpoint with q_w = 0, i.e. at the 4D origin).
 *        anything else -> CLIP_EINVAL.
 * Otherwise as the cuboid calls above: dense rows of invisible segments are canonical qNaN,
 * flags (nullable) 1/0, the compacting call keeps visible rows in input order with optional
 * global indices and a device count, workspace clip_compact_workspace_bytes(n), out must not
 * overlap in (compacting call), same status codes and alignment rules. */
int clip_homog_segments_f32(const float* in, int64_t ld_in, int64_t n, int ndc, float* out, int64_t ld_out,
                            uint8_t* flags, void* stream);
int clip_homog_segments_f64(const double* in, int64_t ld_in, int64_t n, int ndc, double* out, int64_t ld_out,
                            uint8_t* flags, void* stream);
int clip_homog_segments_compact_f32(const float* in, int64_t ld_in, int64_t n, int ndc, float* out,
                                    int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                                    int64_t* d_count, void* workspace, size_t workspace_bytes, void* stream);
int clip_homog_segments_compact_f64(const double* in, int64_t ld_in, int64_t n, int ndc, double* out,
                                    int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                                    int64_t* d_count, void* workspace, size_t workspace_bytes, void* stream);

/* ---- NEXT-2: the paper's per-pixel step — range clip + fused measure ---
 * PAPER.md §5.2: "pixels outside the range [r_min, r_max] will be ignored for
 * clustering", the range recomputed per frame; §4.2 Eq. (5): phi = arctan(d sqrt(I)).
 * d, I:    n pixels (device, 16-byte aligned): radial distance (m; 0 = invalid / dropout) and
 *          intensity, frames of pix_per_frame consecutive pixels (the last may be ragged).
 * ranges:  device float[2 * F], F = ceil(n / pix_per_frame): r_min, r_max of each frame.
 * phi:     n floats (16-byte aligned): arctan(d sqrt(I)) in binary32 for kept pixels, the
 *          canonical qNaN otherwise.  phi must not overlap d or I.
 * code:    (nullable, 4-byte aligned) n bytes: 4 invalid (d <= 0, non-finite d or I, I < 0),
 *          else bit 0 = d < r_min, bit 1 = d > r_max; kept iff 0 (closed interval).
 * kept:    (nullable, 4-byte aligned) int32[F]: kept pixels per frame (zeroed by the call).
 * Status: CLIP_EINVAL (n < 0 or n >= 2^52, pix_per_frame < 1, null d/I/ranges/phi), CLIP_EALIGN,
 * CLIP_ECUDA; n == 0 launches nothing. */
int clip_tof_range_phi_f32(const float* d, const float* I, int64_t n, int64_t pix_per_frame, const float* ranges,
                           float* phi, uint8_t* code, int32_t* kept, void* stream);

/* ---- NEXT-3: the paper's GPU hot path — mutual-best region merging ------
 * PAPER.md §4.1: every valid pixel starts as a region (id = row-major pixel
 * index + 1 within its frame); each round every region picks the 4-adjacent region that
 * passes Eq. (1) (|dz| <= t_z and |dphi| <= t_phi) with the smallest Eq. (2) difference
 * alpha_z |dz| + alpha_phi |dphi|, ties to the larger id (rule 2); mutual choices merge
 * (rule 3) into the larger id with pixel-count-weighted mean descriptors; all
 * choices of a round use the state at its start; rounds repeat until one merges nothing.
 * Table 1 parameters: t_z = 0.04 m, t_phi = 0.009 rad, alpha_z = 8/pi, alpha_phi = 4/3.
 * z, phi:   nframes * height * width binary32 values per pixel (device, row-major frames);
 * valid:    bytes, nonzero = the pixel is a region (0: invalid / clipped, label 0);
 * labels:   int32 per pixel: the id of its final region (0 for invalid pixels);
 * nregions: (nullable) int32[nframes] final region counts; d_rounds: (nullable) device int32:
 *           rounds run including the final one without merges (max_rounds if not converged);
 * workspace: clip_cluster_workspace_bytes(...) device bytes, 256-byte aligned (sized for one
 *           part: batches of more than 592 frames run as consecutive launches of at most
 *           592 frames each, reusing the workspace).
 * Limits: nframes * height * width < 2^30.  Status: CLIP_EINVAL (bad sizes, negative or
 * non-finite params, max_rounds < 1, null pointers), CLIP_EALIGN, CLIP_ENOSPACE, CLIP_ECUDA.
 * One launch per part of the batch runs every round on the device (no host round trips):
 * below 64 frames a grid-wide cooperative kernel (grid barriers between phases), from 64
 * frames one 1024-thread block per frame (block barriers). */
typedef struct {
  double t_z, t_phi, alpha_z, alpha_phi;
} clip_merge_params;
size_t clip_cluster_workspace_bytes(int64_t nframes, int height, int width);
int clip_cluster_frames(const float* z, const float* phi, const uint8_t* valid, int64_t nframes, int height,
                        int width, const clip_merge_params* params, int max_rounds, int32_t* labels,
                        int32_t* nregions, int32_t* d_rounds, void* workspace, size_t workspace_bytes,
                        void* stream);

/* ---- NEXT-4: integer / pixel-coordinate segments, exact clipping --------
 * SURVEY.md §8(f) NEXT-4; PAPER.md defines no integer variant (BJ:5 only mentions one), so
 * the rules are the float path's WEC rules (PAPER.md:29-30 macros) in exact rationals:
 * I1 every coordinate and window bound in [-2^30, 2^30]; I2 closed window lo <= hi;
 * I3 per edge the WECs w0, w1 of P0, P1 (x - lo, hi - x), trivial reject when both < 0,
 *    alpha = w0 / (w0 - w1) exact, t_in = max(0, entering), t_out = min(1, leaving),
 *    visible iff t_in <= t_out;
 * I4 Q_e,k = P0_k + floor(d_k t_e + 1/2) (round half up, exact);
 * I5 invisible rows hold INT32_MIN in all 4 planes; I6 flag 2 = a coordinate outside I1.
 * in, out: 4 int32 planes x0, y0, x1, y1 (ld_in / ld_out, same layout and alignment rules
 *          as the float calls; out == in with ld_out == ld_in allowed, any other overlap
 *          -> CLIP_EINVAL).
 * flags:   (nullable, 4-byte aligned) n bytes: 1 visible, 0 invisible, 2 out of range.
 * win:     host pointer; lo > hi or a bound outside [-2^30, 2^30] -> CLIP_EINVAL.
 * Results are bit-identical to the exact-rational oracle (oracle/int_oracle.py). */
typedef struct { int32_t lo[2], hi[2]; } clip_window_i32;
int clip_segments_i32(const int32_t* in, int64_t ld_in, int64_t n, const clip_window_i32* win, int32_t* out,
                      int64_t ld_out, uint8_t* flags, void* stream);

/* Compacting variant of the int32 clip (NEXT-4 widening; same rules I1-I6): rows [0, count)
 * of out hold the visible segments' clipped endpoints in increasing input index (rows >= count
 * are not written); out_index (nullable, int64[count]) = index_base + input index; flags
 * (nullable, n bytes) 1 visible / 0 invisible / 2 out of range, as clip_segments_i32; d_count:
 * one int64 in device memory; workspace: clip_compact_workspace_bytes(n) bytes, zero-filled
 * before its first use and left zero-filled by every call (as the float compacting calls).
 * out must not overlap in; same window, alignment and status rules as clip_segments_i32.
 * Results are bit-identical to the exact-rational oracle's visible rows in order. */
int clip_segments_compact_i32(const int32_t* in, int64_t ld_in, int64_t n, const clip_window_i32* win,
                              int32_t* out, int64_t ld_out, int64_t* out_index, int64_t index_base,
                              uint8_t* flags, int64_t* d_count, void* workspace, size_t workspace_bytes,
                              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CLIPSEG_H_ */
