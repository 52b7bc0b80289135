/* include/synth.h — C ABI of the seeded synthetic segment generator (libsynth.so).
 *
 * Input generator only (it holds none of the clipping arithmetic).  It serves both
 * the oracle tests and the CUDA path, so that both see bit-identical inputs; the
 * recipe is DESIGN.md "Input recipe" / SURVEY.md §8(d) "Generator G1".
 *
 * Layout: planar SoA, 2*dim planes of `ld` elements, plane c = e*dim + k holds
 * coordinate k of endpoint e (x0, y0, [z0], x1, y1, [z1]); element r of a plane is
 * the segment with global index i0 + r.  `tag` (nullable, n bytes) receives the
 * category (SYN_MIX: 0 inside, 1 crossing, 2 outside) or the adversarial family
 * index 0..9 with bit 0x80 set for near-boundary placements.
 *
 * family: 0 uniform grid in [-1,2)^dim, 1 inside/crossing/outside mix with
 * probabilities p_in/2^32 and p_cross/2^32 (the rest outside), 2 adversarial,
 * 3 homogeneous clip-space segments (dim must be 4: planes x0,y0,z0,w0,x1,y1,z1,w1;
 * tag = mode 0 perspective, 1 affine w = 1, 2 behind the eye, 3 on planes, 4 degenerate;
 * p_in != 0 sets the perspective share to p_in/2^32, the other modes share the rest).
 * Returns SYNTH_OK (0) or a negative status; device variants launch
 * asynchronously on `stream` (a cudaStream_t, NULL = legacy default stream).
 */
#ifndef SYNTH_H_
#define SYNTH_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define SYNTH_OK 0
#define SYNTH_EINVAL (-1)
#define SYNTH_ECUDA (-4)

int synth_fill_host_f32(int family, int dim, uint64_t seed, int64_t i0, int64_t n, float* planes, int64_t ld,
                        uint8_t* tag, uint32_t p_in, uint32_t p_cross, int nthreads);
int synth_fill_host_f64(int family, int dim, uint64_t seed, int64_t i0, int64_t n, double* planes, int64_t ld,
                        uint8_t* tag, uint32_t p_in, uint32_t p_cross, int nthreads);
int synth_fill_device_f32(int family, int dim, uint64_t seed, int64_t i0, int64_t n, float* planes, int64_t ld,
                          uint8_t* tag, uint32_t p_in, uint32_t p_cross, void* stream);
int synth_fill_device_f64(int family, int dim, uint64_t seed, int64_t i0, int64_t n, double* planes, int64_t ld,
                          uint8_t* tag, uint32_t p_in, uint32_t p_cross, void* stream);

/* NEXT-2 input: n pixels of batched ToF frames (ppf pixels per frame),
 * global pixel index i0 + r -> d[r] (meters, 0 = invalid), I[r] (intensity, I = rho / d^2);
 * synth_tof_ranges: the per-frame clip range r[2f] = r_min, r[2f+1] = r_max of frames
 * f0 .. f0 + nframes - 1 (host). */
int synth_tof_host(uint64_t seed, int64_t i0, int64_t n, int64_t ppf, float* d, float* I, int nthreads);
int synth_tof_device(uint64_t seed, int64_t i0, int64_t n, int64_t ppf, float* d, float* I, void* stream);
int synth_tof_ranges(uint64_t seed, int64_t f0, int64_t nframes, float* r);

#ifdef __cplusplus
}
#endif
#endif
