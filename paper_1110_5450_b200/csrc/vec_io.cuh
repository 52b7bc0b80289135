// vec_io.cuh — 128-bit streaming global loads/stores for the planar segment layout.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace clipseg {

template <typename T> struct Vec16;
template <> struct Vec16<float> {
  typedef float4 type;
  static constexpr int N = 4;
  static __device__ __forceinline__ void unpack(const float4& v, float (&a)[4]) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
  static __device__ __forceinline__ float4 pack(const float (&a)[4]) { return make_float4(a[0], a[1], a[2], a[3]); }
};
template <> struct Vec16<int32_t> {
  typedef int4 type;
  static constexpr int N = 4;
  static __device__ __forceinline__ void unpack(const int4& v, int32_t (&a)[4]) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
  static __device__ __forceinline__ int4 pack(const int32_t (&a)[4]) { return make_int4(a[0], a[1], a[2], a[3]); }
};
template <> struct Vec16<double> {
  typedef double2 type;
  static constexpr int N = 2;
  static __device__ __forceinline__ void unpack(const double2& v, double (&a)[2]) { a[0] = v.x; a[1] = v.y; }
  static __device__ __forceinline__ double2 pack(const double (&a)[2]) { return make_double2(a[0], a[1]); }
};

#ifndef CLIPSEG_LOAD_HINT
#define CLIPSEG_LOAD_HINT 2  // streaming loads of 2D segments: 0 evict-first, 1 .nc, 2 plain, 3 last-use
#endif
// Streaming loads (every byte is read once per launch).  PLAIN selects plain loads, measured
// ~2-7 % faster than evict-first ones for the 2D fp32 kernels (dense 0.617 -> 0.575 ms at 1e8)
// and slower for the 3D / homogeneous ones, which keep evict-first (profiles/r01_summary.md).
template <typename T, bool PLAIN = false>
__device__ __forceinline__ void load_vec(const T* p, T (&a)[Vec16<T>::N]) {
  typedef typename Vec16<T>::type V;
  const V* q = reinterpret_cast<const V*>(p);
  if (PLAIN) {
#if CLIPSEG_LOAD_HINT == 1
    Vec16<T>::unpack(__ldg(q), a);
#elif CLIPSEG_LOAD_HINT == 2
    Vec16<T>::unpack(*q, a);
#elif CLIPSEG_LOAD_HINT == 3
    Vec16<T>::unpack(__ldlu(q), a);
#else
    Vec16<T>::unpack(__ldcs(q), a);
#endif
  } else {
    Vec16<T>::unpack(__ldcs(q), a);
  }
}
template <typename T>
__device__ __forceinline__ void store_vec(T* p, const T (&a)[Vec16<T>::N]) {
#if defined(CLIPSEG_PLAIN_STORES)
  *reinterpret_cast<typename Vec16<T>::type*>(p) = Vec16<T>::pack(a);
#else
  __stcs(reinterpret_cast<typename Vec16<T>::type*>(p), Vec16<T>::pack(a));
#endif
}

}  // namespace clipseg
