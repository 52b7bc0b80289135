// clip_dense.cu — K2: the dense clip (every segment -> clipped endpoints + flag).
//
// One thread owns V consecutive segments (V = 4 fp32 / 2 fp64): one 128-bit load per
// plane, the branch-free per-segment rules of clip_math.cuh, one 128-bit store per plane
// and one packed flag store.  Grid-stride over a persistent grid sized to the device's
// resident capacity (148 SMs x blocks/SM).  HBM-bound: 2*(2D*sizeof(T)) + 1 bytes moved
// per segment.
#include "clip_kernels.cuh"
#include "vec_io.cuh"

namespace clipseg {

#ifndef CLIPSEG_DENSE_HOMOG_PREFETCH
#define CLIPSEG_DENSE_HOMOG_PREFETCH 0  // fp32 homogeneous: 1.42 ms without vs 1.73 with (1e8)
#endif
#ifndef CLIPSEG_DENSE_3D_PREFETCH
#define CLIPSEG_DENSE_3D_PREFETCH 0  // fp32 3D: 0.884 ms without vs 0.968 with (1e8)
#endif
#ifndef CLIPSEG_DENSE_2D_PREFETCH
#define CLIPSEG_DENSE_2D_PREFETCH 1
#endif
#ifndef CLIPSEG_DENSE_F64_PREFETCH
#define CLIPSEG_DENSE_F64_PREFETCH 1
#endif
#ifndef CLIPSEG_DENSE_HOMOG_MINB
#define CLIPSEG_DENSE_HOMOG_MINB 3
#endif
// The next group's loads in flight while this one is clipped (registers for a second
// group) — except where the registers buy more than the overlap (measured per case).
template <typename T, class Op> __host__ __device__ constexpr bool dense_prefetch() {
  return sizeof(T) == 8   ? CLIPSEG_DENSE_F64_PREFETCH != 0
         : Op::IN == 8 ? CLIPSEG_DENSE_HOMOG_PREFETCH != 0
         : Op::IN == 6 ? CLIPSEG_DENSE_3D_PREFETCH != 0
                       : CLIPSEG_DENSE_2D_PREFETCH != 0;
}
template <typename T, class Op>
__global__ void __launch_bounds__(256, (Op::IN == 8 && sizeof(T) == 4) ? CLIPSEG_DENSE_HOMOG_MINB
                                                                          : (sizeof(T) == 4 ? 3 : 2))
    clip_dense_kernel(const T* in, int64_t ld_in, int64_t n, typename Op::Params w, T* out, int64_t ld_out,
                      uint8_t* flags) {
  constexpr int V = Vec16<T>::N, IN = Op::IN, OUT = Op::OUT;
  const int64_t ngroups = (n + V - 1) / V;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr bool PREFETCH = dense_prefetch<T, Op>();
  T nxt[PREFETCH ? IN : 1][V];
  if (PREFETCH && g < ngroups) {
#pragma unroll
    for (int c = 0; c < IN; ++c) load_vec<T, IN == 4>(in + c * ld_in + g * V, nxt[c]);
  }
  for (; g < ngroups; g += stride) {
    const int64_t i = g * V;
    T plane[IN][V];
    if constexpr (PREFETCH) {
#pragma unroll
      for (int c = 0; c < IN; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) plane[c][v] = nxt[c][v];
      if (g + stride < ngroups) {  // next group's loads in flight while this one is clipped
#pragma unroll
        for (int c = 0; c < IN; ++c) load_vec<T, IN == 4>(in + c * ld_in + (g + stride) * V, nxt[c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < IN; ++c) load_vec<T, IN == 4>(in + c * ld_in + i, plane[c]);
    }
    T res[OUT][V];
    const unsigned bits = group_chunked<Op, true>(plane, w, res);
    uint32_t vis = 0;  // one flag byte per segment
#pragma unroll
    for (int v = 0; v < V; ++v) vis |= ((bits >> v) & 1u) << (8 * v);
    if (i + V <= n) {
#pragma unroll
      for (int c = 0; c < OUT; ++c) store_vec<T>(out + c * ld_out + i, res[c]);
      if (flags) {
        if (V == 4) *reinterpret_cast<uint32_t*>(flags + i) = vis;
        else *reinterpret_cast<uint16_t*>(flags + i) = (uint16_t)vis;
      }
    } else {  // ragged tail: only rows < n are written
      for (int v = 0; v < V; ++v) {
        if (i + v < n) {
#pragma unroll
          for (int c = 0; c < OUT; ++c) out[c * ld_out + i + v] = res[c][v];
          if (flags) flags[i + v] = (uint8_t)((vis >> (8 * v)) & 1u);
        }
      }
    }
  }
}

template <typename T, class Op>
cudaError_t launch_dense(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                         int64_t ld_out, uint8_t* flags, cudaStream_t s) {
  constexpr int V = Vec16<T>::N, NT = 256;
  int blocks_per_sm = 0;  // per device, cached (kernel_occupancy)
  cudaError_t e = kernel_occupancy((const void*)clip_dense_kernel<T, Op>, NT, 0, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t ngroups = (n + V - 1) / V;
  const int64_t want = (ngroups + NT - 1) / NT;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;
  const int grid = (int)(want < cap ? want : cap);
  clip_dense_kernel<T, Op><<<grid, NT, 0, s>>>(in, ld_in, n, w, out, ld_out, flags);
  return cudaGetLastError();
}

#define INST(T, OP)                                                                                         \
  template cudaError_t launch_dense<T, OP>(const T*, int64_t, int64_t, const typename OP::Params&, T*, int64_t, \
                                           uint8_t*, cudaStream_t);
typedef BoxOp<float, 2> BoxF2;
typedef BoxOp<float, 3> BoxF3;
typedef BoxOp<double, 2> BoxD2;
typedef BoxOp<double, 3> BoxD3;
typedef HomogOp<float, false> HomF;
typedef HomogOp<float, true> HomFN;
typedef HomogOp<double, false> HomD;
typedef HomogOp<double, true> HomDN;
INST(float, BoxF2)
INST(float, BoxF3)
INST(double, BoxD2)
INST(double, BoxD3)
INST(float, HomF)
INST(float, HomFN)
INST(double, HomD)
INST(double, HomDN)
#undef INST

}  // namespace clipseg
