/* synth/synth.cu — host and device entry points of the G1 generator (include/synth.h).
 * INPUT GENERATOR ONLY: no clipping arithmetic lives here (see synth_core.h). */
#include "synth_core.h"
#include "../include/synth.h"

#include <cuda_runtime.h>
#include <thread>
#include <vector>

namespace {

// D == 4 is the homogeneous family (syn_homog); D = 2, 3 the cuboid families.
template <typename T, int D>
SYN_HD uint8_t gen_one(int family, uint64_t seed, int64_t i, uint32_t p_in, uint32_t p_cross, T (&p)[2 * D]) {
  if constexpr (D == 4) return syn_homog<T>(seed, i, p, p_in);
  else return syn_segment<T, D>(family, seed, i, p_in, p_cross, p);
}

template <typename T, int D>
void fill_host_range(int family, uint64_t seed, int64_t i0, int64_t a, int64_t b, T* planes, int64_t ld,
                     uint8_t* tag, uint32_t p_in, uint32_t p_cross) {
  T p[2 * D];
  for (int64_t r = a; r < b; ++r) {
    const uint8_t t = gen_one<T, D>(family, seed, i0 + r, p_in, p_cross, p);
    for (int c = 0; c < 2 * D; ++c) planes[(int64_t)c * ld + r] = p[c];
    if (tag) tag[r] = t;
  }
}

template <typename T, int D>
int fill_host(int family, uint64_t seed, int64_t i0, int64_t n, T* planes, int64_t ld, uint8_t* tag,
              uint32_t p_in, uint32_t p_cross, int nthreads) {
  if (nthreads <= 1 || n < (1 << 16)) {
    fill_host_range<T, D>(family, seed, i0, 0, n, planes, ld, tag, p_in, p_cross);
    return SYNTH_OK;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t a = n * t / nthreads, b = n * (t + 1) / nthreads;
    th.emplace_back(fill_host_range<T, D>, family, seed, i0, a, b, planes, ld, tag, p_in, p_cross);
  }
  for (auto& x : th) x.join();
  return SYNTH_OK;
}

template <typename T, int D>
__global__ void fill_kernel(int family, uint64_t seed, int64_t i0, int64_t n, T* __restrict__ planes, int64_t ld,
                            uint8_t* __restrict__ tag, uint32_t p_in, uint32_t p_cross) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    T p[2 * D];
    const uint8_t t = gen_one<T, D>(family, seed, i0 + r, p_in, p_cross, p);
#pragma unroll
    for (int c = 0; c < 2 * D; ++c) planes[(int64_t)c * ld + r] = p[c];
    if (tag) tag[r] = t;
  }
}

template <typename T, int D>
int fill_device(int family, uint64_t seed, int64_t i0, int64_t n, T* planes, int64_t ld, uint8_t* tag,
                uint32_t p_in, uint32_t p_cross, void* stream) {
  if (n == 0) return SYNTH_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
  fill_kernel<T, D><<<grid, 256, 0, (cudaStream_t)stream>>>(family, seed, i0, n, planes, ld, tag, p_in, p_cross);
  return cudaGetLastError() == cudaSuccess ? SYNTH_OK : SYNTH_ECUDA;
}

int check(int family, int dim, int64_t i0, int64_t n, const void* planes, int64_t ld) {
  if (family < SYN_UNIFORM || family > SYN_HOMOG) return SYNTH_EINVAL;
  if (family == SYN_HOMOG ? dim != 4 : (dim != 2 && dim != 3)) return SYNTH_EINVAL;
  if (n < 0 || i0 < 0 || ld < n) return SYNTH_EINVAL;
  if (n > 0 && !planes) return SYNTH_EINVAL;
  return SYNTH_OK;
}

void tof_host_range(uint64_t seed, int64_t i0, int64_t a, int64_t b, int64_t ppf, float* d, float* I) {
  for (int64_t r = a; r < b; ++r) syn_tof_pixel(seed, i0 + r, ppf, d + r, I + r);
}

__global__ void tof_kernel(uint64_t seed, int64_t i0, int64_t n, int64_t ppf, float* __restrict__ d,
                           float* __restrict__ I) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    syn_tof_pixel(seed, i0 + r, ppf, d + r, I + r);
}

}  // namespace

extern "C" {

int synth_tof_host(uint64_t seed, int64_t i0, int64_t n, int64_t ppf, float* d, float* I, int nthreads) {
  if (n < 0 || i0 < 0 || ppf <= 0 || (n > 0 && (!d || !I))) return SYNTH_EINVAL;
  if (nthreads <= 1 || n < (1 << 16)) {
    tof_host_range(seed, i0, 0, n, ppf, d, I);
    return SYNTH_OK;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back(tof_host_range, seed, i0, n * t / nthreads, n * (t + 1) / nthreads, ppf, d, I);
  for (auto& x : th) x.join();
  return SYNTH_OK;
}

int synth_tof_device(uint64_t seed, int64_t i0, int64_t n, int64_t ppf, float* d, float* I, void* stream) {
  if (n < 0 || i0 < 0 || ppf <= 0 || (n > 0 && (!d || !I))) return SYNTH_EINVAL;
  if (n == 0) return SYNTH_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
  tof_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, i0, n, ppf, d, I);
  return cudaGetLastError() == cudaSuccess ? SYNTH_OK : SYNTH_ECUDA;
}

int synth_tof_ranges(uint64_t seed, int64_t f0, int64_t nframes, float* r) {
  if (nframes < 0 || f0 < 0 || (nframes > 0 && !r)) return SYNTH_EINVAL;
  for (int64_t f = 0; f < nframes; ++f) syn_tof_range(seed, f0 + f, r + 2 * f);
  return SYNTH_OK;
}

int synth_fill_host_f32(int family, int dim, uint64_t seed, int64_t i0, int64_t n, float* planes, int64_t ld,
                        uint8_t* tag, uint32_t p_in, uint32_t p_cross, int nthreads) {
  const int s = check(family, dim, i0, n, planes, ld);
  if (s) return s;
  if (dim == 4) return fill_host<float, 4>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads);
  return dim == 2 ? fill_host<float, 2>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads)
                  : fill_host<float, 3>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads);
}

int synth_fill_host_f64(int family, int dim, uint64_t seed, int64_t i0, int64_t n, double* planes, int64_t ld,
                        uint8_t* tag, uint32_t p_in, uint32_t p_cross, int nthreads) {
  const int s = check(family, dim, i0, n, planes, ld);
  if (s) return s;
  if (dim == 4) return fill_host<double, 4>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads);
  return dim == 2 ? fill_host<double, 2>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads)
                  : fill_host<double, 3>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, nthreads);
}

int synth_fill_device_f32(int family, int dim, uint64_t seed, int64_t i0, int64_t n, float* planes, int64_t ld,
                          uint8_t* tag, uint32_t p_in, uint32_t p_cross, void* stream) {
  const int s = check(family, dim, i0, n, planes, ld);
  if (s) return s;
  if (dim == 4) return fill_device<float, 4>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream);
  return dim == 2 ? fill_device<float, 2>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream)
                  : fill_device<float, 3>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream);
}

int synth_fill_device_f64(int family, int dim, uint64_t seed, int64_t i0, int64_t n, double* planes, int64_t ld,
                          uint8_t* tag, uint32_t p_in, uint32_t p_cross, void* stream) {
  const int s = check(family, dim, i0, n, planes, ld);
  if (s) return s;
  if (dim == 4) return fill_device<double, 4>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream);
  return dim == 2 ? fill_device<double, 2>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream)
                  : fill_device<double, 3>(family, seed, i0, n, planes, ld, tag, p_in, p_cross, stream);
}

}  // extern "C"
