// clip_api.cu — the extern "C" boundary declared in include/clipseg.h: argument
// validation, dispatch on (dtype, dim) to the sm_100a kernels, status codes, and the
// pipelined host-buffer entry points.  No torch types cross this boundary.
#include <clipseg.h>

#include <cmath>
#include <cstring>

#include "clip_kernels.cuh"

using namespace clipseg;

namespace {

template <typename T> struct WinT;
template <> struct WinT<float> { typedef clip_window_f32 type; };
template <> struct WinT<double> { typedef clip_window_f64 type; };

template <typename T>
int check_window(const typename WinT<T>::type* win) {
  if (!win || (win->dim != 2 && win->dim != 3)) return CLIP_EINVAL;
  for (int k = 0; k < win->dim; ++k) {
    if (!std::isfinite(win->lo[k]) || !std::isfinite(win->hi[k])) return CLIP_EINVAL;
    if (!(win->lo[k] <= win->hi[k])) return CLIP_EINVAL;
  }
  return CLIP_OK;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

template <typename T>
int check_planes(const T* p, int64_t ld, int64_t n) {
  if (!p) return CLIP_EINVAL;
  if (ld < n) return CLIP_EINVAL;
  if (!aligned(p, 16) || ((ld * (int64_t)sizeof(T)) % 16) != 0) return CLIP_EALIGN;
  return CLIP_OK;
}

// The kernels' fast path needs edges without -0 and with |edge| <= 2^58 (fp32) /
// 2^500 (fp64) (clip_math.cuh); other windows run every segment on the exact path.
template <typename T, int D>
Window<T, D> to_window(const typename WinT<T>::type* win) {
  Window<T, D> w;
  const double big = sizeof(T) == 4 ? 0x1p58 : 0x1p500;
  w.fast = 1;
  for (int k = 0; k < D; ++k) {
    w.lo[k] = win->lo[k];
    w.hi[k] = win->hi[k];
    for (const double e : {(double)win->lo[k], (double)win->hi[k]})
      if ((e == 0.0 && std::signbit(e)) || std::fabs(e) > big) w.fast = 0;
  }
  return w;
}

// Byte extent of `planes` planes of `ld` elements holding n rows each.
inline int64_t plane_bytes(int planes, int64_t ld, int64_t n, size_t esz) {
  return ((int64_t)(planes - 1) * ld + n) * (int64_t)esz;
}
// Element-wise (dense) kernels read a thread's rows before writing them, so in place
// (out == in with the same plane stride) is allowed; any other overlap would let one thread's
// stores race with another's loads.
inline bool overlap_ok(const void* in, int64_t in_bytes, const void* out, int64_t out_bytes, bool same_ld) {
  const char *ib = reinterpret_cast<const char*>(in), *ob = reinterpret_cast<const char*>(out);
  if (ib == ob) return same_ld;
  return !(ob < ib + in_bytes && ib < ob + out_bytes);
}

int status_of(cudaError_t e) { return e == cudaSuccess ? CLIP_OK : CLIP_ECUDA; }

template <typename T>
int dense(const T* in, int64_t ld_in, int64_t n, const typename WinT<T>::type* win, T* out, int64_t ld_out,
          uint8_t* flags, void* stream) {
  if (n < 0) return CLIP_EINVAL;
  int st = check_window<T>(win);
  if (st) return st;
  if (n == 0) return CLIP_OK;
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  const int planes = 2 * win->dim;
  if (!overlap_ok(in, plane_bytes(planes, ld_in, n, sizeof(T)), out, plane_bytes(planes, ld_out, n, sizeof(T)),
                  ld_in == ld_out))
    return CLIP_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (win->dim == 2)
    return status_of(launch_dense<T, BoxOp<T, 2>>(in, ld_in, n, to_window<T, 2>(win), out, ld_out, flags, s));
  return status_of(launch_dense<T, BoxOp<T, 3>>(in, ld_in, n, to_window<T, 3>(win), out, ld_out, flags, s));
}

template <typename T>
int compact(const T* in, int64_t ld_in, int64_t n, const typename WinT<T>::type* win, T* out, int64_t ld_out,
            int64_t* out_index, int64_t index_base, uint8_t* flags, int64_t* d_count, void* ws, size_t ws_bytes,
            void* stream) {
  if (n < 0 || !d_count) return CLIP_EINVAL;
  int st = check_window<T>(win);
  if (st) return st;
  if (!aligned(d_count, 8)) return CLIP_EALIGN;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n == 0) return status_of(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  if (out_index && !aligned(out_index, 8)) return CLIP_EALIGN;
  if (!ws) return CLIP_EINVAL;
  if (!aligned(ws, 16)) return CLIP_EALIGN;
  if (ws_bytes < clip_compact_workspace_bytes(n)) return CLIP_ENOSPACE;
  // out must not overlap in (the kernel reads tiles while others write compacted rows)
  const char *ib = reinterpret_cast<const char*>(in), *ob = reinterpret_cast<const char*>(out);
  const int dim = win->dim;
  const int64_t ibytes = ((int64_t)(2 * dim - 1) * ld_in + n) * (int64_t)sizeof(T);
  const int64_t obytes = ((int64_t)(2 * dim - 1) * ld_out + n) * (int64_t)sizeof(T);
  if (ob < ib + ibytes && ib < ob + obytes) return CLIP_EINVAL;
  if (dim == 2)
    return status_of(launch_compact<T, BoxOp<T, 2>>(in, ld_in, n, to_window<T, 2>(win), out, ld_out, out_index,
                                                    index_base, flags, d_count, ws, s));
  return status_of(launch_compact<T, BoxOp<T, 3>>(in, ld_in, n, to_window<T, 3>(win), out, ld_out, out_index,
                                                  index_base, flags, d_count, ws, s));
}

// ---- NEXT-1: homogeneous clip space (8 input planes; 8 output planes, or 6 with ndc) ----
template <typename T>
int homog_dense(const T* in, int64_t ld_in, int64_t n, int ndc, T* out, int64_t ld_out, uint8_t* flags,
                void* stream) {
  if (n < 0 || (ndc != 0 && ndc != 1)) return CLIP_EINVAL;
  if (n == 0) return CLIP_OK;
  int st;
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  if (!overlap_ok(in, plane_bytes(8, ld_in, n, sizeof(T)), out, plane_bytes(ndc ? 6 : 8, ld_out, n, sizeof(T)),
                  ld_in == ld_out))
    return CLIP_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const NoParams none{0};
  if (ndc) return status_of(launch_dense<T, HomogOp<T, true>>(in, ld_in, n, none, out, ld_out, flags, s));
  return status_of(launch_dense<T, HomogOp<T, false>>(in, ld_in, n, none, out, ld_out, flags, s));
}

template <typename T>
int homog_compact(const T* in, int64_t ld_in, int64_t n, int ndc, T* out, int64_t ld_out, int64_t* out_index,
                  int64_t index_base, uint8_t* flags, int64_t* d_count, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !d_count || (ndc != 0 && ndc != 1)) return CLIP_EINVAL;
  if (!aligned(d_count, 8)) return CLIP_EALIGN;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n == 0) return status_of(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
  int st;
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  if (out_index && !aligned(out_index, 8)) return CLIP_EALIGN;
  if (!ws) return CLIP_EINVAL;
  if (!aligned(ws, 16)) return CLIP_EALIGN;
  if (ws_bytes < clip_compact_workspace_bytes(n)) return CLIP_ENOSPACE;
  const char *ib = reinterpret_cast<const char*>(in), *ob = reinterpret_cast<const char*>(out);
  const int64_t ibytes = ((int64_t)7 * ld_in + n) * (int64_t)sizeof(T);
  const int64_t obytes = ((int64_t)(ndc ? 5 : 7) * ld_out + n) * (int64_t)sizeof(T);
  if (ob < ib + ibytes && ib < ob + obytes) return CLIP_EINVAL;
  const NoParams none{0};
  if (ndc)
    return status_of(launch_compact<T, HomogOp<T, true>>(in, ld_in, n, none, out, ld_out, out_index, index_base,
                                                         flags, d_count, ws, s));
  return status_of(launch_compact<T, HomogOp<T, false>>(in, ld_in, n, none, out, ld_out, out_index, index_base,
                                                        flags, d_count, ws, s));
}

// ---- pipelined host-buffer path -----------------------------------------------------
inline size_t round256(size_t x) { return (x + 255) & ~(size_t)255; }

struct StageLayout {
  size_t in_off, out_off, flags_off, count_off, ws_off, set_bytes;
};

StageLayout stage_layout(int dim, int elem, int64_t chunk) {
  StageLayout L;
  const int64_t ldc = clip_plane_stride(chunk);
  const size_t planes = (size_t)2 * dim * (size_t)ldc * (size_t)elem;
  L.in_off = 0;
  L.out_off = round256(planes);
  L.flags_off = L.out_off + round256(planes);
  L.count_off = L.flags_off + round256((size_t)ldc);
  L.ws_off = L.count_off + 256;
  L.set_bytes = L.ws_off + round256(clip_compact_workspace_bytes(chunk));
  return L;
}

// Streams and events of the pipelined host entry, per host thread and device: a call on
// another thread gets its own set (the entry stays reentrant), repeated calls reuse it.
// Created on first use; released when the thread exits.
struct HostPipe {
  cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr, sk = nullptr;
  cudaEvent_t h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {};
  bool ready = false;
  ~HostPipe() {
    if (!ready) return;
    for (int s = 0; s < 2; ++s) {
      cudaEventDestroy(h2d_done[s]);
      cudaEventDestroy(comp_done[s]);
      cudaEventDestroy(d2h_done[s]);
    }
    cudaStreamDestroy(sh);
    cudaStreamDestroy(sc);
    cudaStreamDestroy(sd);
    cudaStreamDestroy(sk);
  }
};
HostPipe* host_pipe() {
  constexpr int kMaxDev = 64;
  thread_local HostPipe pipes[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  HostPipe& p = pipes[dev];
  if (!p.ready) {
    bool ok = cudaStreamCreateWithFlags(&p.sh, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p.sc, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p.sd, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p.sk, cudaStreamNonBlocking) == cudaSuccess;
    for (int s = 0; s < 2 && ok; ++s)
      ok = cudaEventCreateWithFlags(&p.h2d_done[s], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p.comp_done[s], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p.d2h_done[s], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return nullptr;
    p.ready = true;
  }
  return &p;
}

template <typename T>
int compact_host(const T* h_in, int64_t ld_in, int64_t n, const typename WinT<T>::type* win, T* h_out,
                 int64_t ld_out, uint8_t* h_flags, int64_t* h_count, int64_t chunk, void* d_staging,
                 size_t staging_bytes) {
  if (n < 0 || chunk <= 0 || !h_count) return CLIP_EINVAL;
  int st = check_window<T>(win);
  if (st) return st;
  if (n > 0 && (!h_in || !h_out || ld_in < n || ld_out < n)) return CLIP_EINVAL;
  if (!d_staging) return CLIP_EINVAL;
  if (!aligned(d_staging, 256)) return CLIP_EALIGN;
  if (staging_bytes < clip_host_staging_bytes(win->dim, (int)sizeof(T), chunk)) return CLIP_ENOSPACE;
  *h_count = 0;
  if (n == 0) return CLIP_OK;

  const int dim = win->dim;
  const StageLayout L = stage_layout(dim, (int)sizeof(T), chunk);
  const int64_t ldc = clip_plane_stride(chunk);
  char* base = reinterpret_cast<char*>(d_staging);
  auto set_ptr = [&](int s, size_t off) { return base + (size_t)s * L.set_bytes + off; };

  // the pipeline's streams and events, created once per (host thread, device) and reused
  HostPipe* pipe = host_pipe();
  bool ok = pipe != nullptr;
  if (!ok) return CLIP_ECUDA;
  cudaStream_t sh = pipe->sh, sc = pipe->sc, sd = pipe->sd, sk = pipe->sk;
  cudaEvent_t* h2d_done = pipe->h2d_done;
  cudaEvent_t* comp_done = pipe->comp_done;
  cudaEvent_t* d2h_done = pipe->d2h_done;
  int rc = CLIP_OK;
  const int64_t nch = (n + chunk - 1) / chunk;
  int64_t written = 0;

  // H2D of chunk j into set j%2, then its clip (after the set's previous D2H drained).
  auto issue = [&](int64_t j) -> bool {
    const int s = (int)(j & 1);
    const int64_t a = j * chunk, m = (n - a < chunk) ? (n - a) : chunk;
    T* d_in = reinterpret_cast<T*>(set_ptr(s, L.in_off));
    T* d_out = reinterpret_cast<T*>(set_ptr(s, L.out_off));
    uint8_t* d_flags = reinterpret_cast<uint8_t*>(set_ptr(s, L.flags_off));
    int64_t* d_cnt = reinterpret_cast<int64_t*>(set_ptr(s, L.count_off));
    void* d_ws = set_ptr(s, L.ws_off);
    if (j >= 2 && cudaStreamWaitEvent(sh, comp_done[s], 0) != cudaSuccess) return false;
    if (cudaMemcpy2DAsync(d_in, (size_t)ldc * sizeof(T), h_in + a, (size_t)ld_in * sizeof(T), (size_t)m * sizeof(T),
                          (size_t)2 * dim, cudaMemcpyHostToDevice, sh) != cudaSuccess)
      return false;
    if (cudaEventRecord(h2d_done[s], sh) != cudaSuccess) return false;
    if (cudaStreamWaitEvent(sc, h2d_done[s], 0) != cudaSuccess) return false;
    if (j >= 2 && cudaStreamWaitEvent(sc, d2h_done[s], 0) != cudaSuccess) return false;
    if (compact<T>(d_in, ldc, m, win, d_out, ldc, nullptr, a, d_flags, d_cnt, d_ws, clip_compact_workspace_bytes(m),
                   sc) != CLIP_OK)
      return false;
    return cudaEventRecord(comp_done[s], sc) == cudaSuccess;
  };

  // the compacting kernel needs a zero-filled workspace on first use and leaves it zero:
  // clear both sets' workspaces once per call (the staging buffer is the caller's)
  for (int s = 0; s < 2 && ok; ++s)
    ok = cudaMemsetAsync(set_ptr(s, L.ws_off), 0, clip_compact_workspace_bytes(chunk), sc) == cudaSuccess;
  if (ok) ok = issue(0);
  for (int64_t j = 0; ok && j < nch; ++j) {
    const int s = (int)(j & 1);
    const int64_t a = j * chunk, m = (n - a < chunk) ? (n - a) : chunk;
    if (j + 1 < nch && !(ok = issue(j + 1))) break;
    // the visible count of chunk j sizes its D2H copy
    int64_t cnt = 0;
    ok = cudaStreamWaitEvent(sk, comp_done[s], 0) == cudaSuccess &&
         cudaMemcpyAsync(&cnt, set_ptr(s, L.count_off), sizeof(int64_t), cudaMemcpyDeviceToHost, sk) == cudaSuccess &&
         cudaStreamSynchronize(sk) == cudaSuccess;
    if (!ok) break;
    ok = cudaStreamWaitEvent(sd, comp_done[s], 0) == cudaSuccess;
    if (ok && cnt > 0)
      ok = cudaMemcpy2DAsync(h_out + written, (size_t)ld_out * sizeof(T), set_ptr(s, L.out_off),
                             (size_t)ldc * sizeof(T), (size_t)cnt * sizeof(T), (size_t)2 * dim,
                             cudaMemcpyDeviceToHost, sd) == cudaSuccess;
    if (ok && h_flags)
      ok = cudaMemcpyAsync(h_flags + a, set_ptr(s, L.flags_off), (size_t)m, cudaMemcpyDeviceToHost, sd) == cudaSuccess;
    if (ok) ok = cudaEventRecord(d2h_done[s], sd) == cudaSuccess;
    written += cnt;
  }
  if (ok) ok = cudaStreamSynchronize(sd) == cudaSuccess && cudaStreamSynchronize(sc) == cudaSuccess;
  if (!ok) {
    rc = CLIP_ECUDA;
    if (sh) cudaStreamSynchronize(sh);
    if (sc) cudaStreamSynchronize(sc);
    if (sd) cudaStreamSynchronize(sd);
  }
  if (rc == CLIP_OK) *h_count = written;
  return rc;
}

}  // namespace

extern "C" {

int64_t clip_plane_stride(int64_t n) {
  if (n <= 32) return 32;
  return (n + 31) / 32 * 32;
}

const char* clip_status_string(int status) {
  switch (status) {
    case CLIP_OK: return "CLIP_OK";
    case CLIP_EINVAL: return "CLIP_EINVAL: invalid argument";
    case CLIP_EALIGN: return "CLIP_EALIGN: misaligned pointer or plane stride";
    case CLIP_ENOSPACE: return "CLIP_ENOSPACE: workspace or staging buffer too small";
    case CLIP_ECUDA: return "CLIP_ECUDA: CUDA launch or runtime error";
    default: return "unknown clip status";
  }
}

int clip_segments_f32(const float* in, int64_t ld_in, int64_t n, const clip_window_f32* win, float* out,
                      int64_t ld_out, uint8_t* flags, void* stream) {
  return dense<float>(in, ld_in, n, win, out, ld_out, flags, stream);
}

int clip_segments_f64(const double* in, int64_t ld_in, int64_t n, const clip_window_f64* win, double* out,
                      int64_t ld_out, uint8_t* flags, void* stream) {
  return dense<double>(in, ld_in, n, win, out, ld_out, flags, stream);
}

size_t clip_compact_workspace_bytes(int64_t n) {
  // sized for the smallest block tile so one workspace serves every (dtype, dim)
  const int64_t tile = kMinCompactTile;
  const int64_t nt = n > 0 ? (n + tile - 1) / tile : 0;
  return kWsHeaderBytes + (size_t)nt * 8;
}

int clip_segments_compact_f32(const float* in, int64_t ld_in, int64_t n, const clip_window_f32* win, float* out,
                              int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                              int64_t* d_count, void* workspace, size_t workspace_bytes, void* stream) {
  return compact<float>(in, ld_in, n, win, out, ld_out, out_index, index_base, flags, d_count, workspace,
                        workspace_bytes, stream);
}

int clip_segments_compact_f64(const double* in, int64_t ld_in, int64_t n, const clip_window_f64* win, double* out,
                              int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                              int64_t* d_count, void* workspace, size_t workspace_bytes, void* stream) {
  return compact<double>(in, ld_in, n, win, out, ld_out, out_index, index_base, flags, d_count, workspace,
                         workspace_bytes, stream);
}

int clip_shard_offsets(const int64_t* d_counts, int P, int rank, int64_t* d_offset, int64_t* d_total, void* stream) {
  if (!d_counts || !d_offset || !d_total || P < 1 || rank < 0 || rank >= P) return CLIP_EINVAL;
  return status_of(launch_shard_offsets(d_counts, P, rank, d_offset, d_total, reinterpret_cast<cudaStream_t>(stream)));
}

size_t clip_host_staging_bytes(int dim, int elem_bytes, int64_t chunk) {
  if ((dim != 2 && dim != 3) || (elem_bytes != 4 && elem_bytes != 8) || chunk <= 0) return 0;
  return 2 * stage_layout(dim, elem_bytes, chunk).set_bytes;
}

int clip_segments_compact_host_f32(const float* h_in, int64_t ld_in, int64_t n, const clip_window_f32* win,
                                   float* h_out, int64_t ld_out, uint8_t* h_flags, int64_t* h_count, int64_t chunk,
                                   void* d_staging, size_t staging_bytes) {
  return compact_host<float>(h_in, ld_in, n, win, h_out, ld_out, h_flags, h_count, chunk, d_staging, staging_bytes);
}

int clip_segments_compact_host_f64(const double* h_in, int64_t ld_in, int64_t n, const clip_window_f64* win,
                                   double* h_out, int64_t ld_out, uint8_t* h_flags, int64_t* h_count, int64_t chunk,
                                   void* d_staging, size_t staging_bytes) {
  return compact_host<double>(h_in, ld_in, n, win, h_out, ld_out, h_flags, h_count, chunk, d_staging, staging_bytes);
}

int clip_tof_range_phi_f32(const float* d, const float* I, int64_t n, int64_t pix_per_frame, const float* ranges,
                           float* phi, uint8_t* code, int32_t* kept, void* stream) {
  if (n < 0 || n >= ((int64_t)1 << 52) || pix_per_frame < 1) return CLIP_EINVAL;
  if (n == 0) return CLIP_OK;
  if (!d || !I || !ranges || !phi) return CLIP_EINVAL;
  if (!aligned(d, 16) || !aligned(I, 16) || !aligned(phi, 16) || !aligned(ranges, 4)) return CLIP_EALIGN;
  if ((code && !aligned(code, 4)) || (kept && !aligned(kept, 4))) return CLIP_EALIGN;
  return status_of(launch_tof_range_phi(d, I, n, pix_per_frame, ranges, phi, code, reinterpret_cast<int*>(kept),
                                        reinterpret_cast<cudaStream_t>(stream)));
}

int clip_segments_i32(const int32_t* in, int64_t ld_in, int64_t n, const clip_window_i32* win, int32_t* out,
                      int64_t ld_out, uint8_t* flags, void* stream) {
  if (n < 0 || !win) return CLIP_EINVAL;
  const int64_t B = (int64_t)1 << 30;
  for (int k = 0; k < 2; ++k)
    if (win->lo[k] > win->hi[k] || win->lo[k] < -B || win->hi[k] > B) return CLIP_EINVAL;
  if (n == 0) return CLIP_OK;
  int st;
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  if (!overlap_ok(in, plane_bytes(4, ld_in, n, 4), out, plane_bytes(4, ld_out, n, 4), ld_in == ld_out))
    return CLIP_EINVAL;
  return status_of(launch_clip_int(in, ld_in, n, win->lo, win->hi, out, ld_out, flags,
                                   reinterpret_cast<cudaStream_t>(stream)));
}

int clip_segments_compact_i32(const int32_t* in, int64_t ld_in, int64_t n, const clip_window_i32* win, int32_t* out,
                              int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                              int64_t* d_count, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || !win || !d_count) return CLIP_EINVAL;
  const int64_t B = (int64_t)1 << 30;
  for (int k = 0; k < 2; ++k)
    if (win->lo[k] > win->hi[k] || win->lo[k] < -B || win->hi[k] > B) return CLIP_EINVAL;
  if (!aligned(d_count, 8)) return CLIP_EALIGN;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n == 0) return status_of(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
  int st;
  if ((st = check_planes(in, ld_in, n)) || (st = check_planes(out, ld_out, n))) return st;
  if (flags && !aligned(flags, 4)) return CLIP_EALIGN;
  if (out_index && !aligned(out_index, 8)) return CLIP_EALIGN;
  if (!workspace) return CLIP_EINVAL;
  if (!aligned(workspace, 16)) return CLIP_EALIGN;
  if (workspace_bytes < clip_compact_workspace_bytes(n)) return CLIP_ENOSPACE;
  // out must not overlap in (the kernel reads tiles while others write compacted rows)
  if (!overlap_ok(in, plane_bytes(4, ld_in, n, 4), out, plane_bytes(4, ld_out, n, 4), false)) return CLIP_EINVAL;
  const int32_t S = 1 << 14;
  IntWindow w;
  w.win = make_int4(win->lo[0], win->lo[1], win->hi[0], win->hi[1]);
  w.small = win->lo[0] >= -S && win->lo[1] >= -S && win->hi[0] <= S && win->hi[1] <= S;
  return status_of(launch_compact<int32_t, IntOp>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags, d_count,
                                                  workspace, s));
}

size_t clip_cluster_workspace_bytes(int64_t nframes, int height, int width) {
  if (nframes < 0 || height < 1 || width < 1) return 0;
  const int64_t part = cluster_part_frames(nframes);  // frames per launch
  return cluster_workspace_bytes(part * (int64_t)height * width) + 4096;
}

int clip_cluster_frames(const float* z, const float* phi, const uint8_t* valid, int64_t nframes, int height,
                        int width, const clip_merge_params* params, int max_rounds, int32_t* labels,
                        int32_t* nregions, int32_t* d_rounds, void* workspace, size_t workspace_bytes,
                        void* stream) {
  if (nframes < 0 || height < 1 || width < 1 || !params || max_rounds < 1) return CLIP_EINVAL;
  const int64_t n = nframes * (int64_t)height * width;
  if (n >= ((int64_t)1 << 31) / 2) return CLIP_EINVAL;  // int region and edge indices
  if (!(params->t_z >= 0) || !(params->t_phi >= 0) || !(params->alpha_z >= 0) || !(params->alpha_phi >= 0) ||
      !std::isfinite(params->t_z + params->t_phi + params->alpha_z + params->alpha_phi))
    return CLIP_EINVAL;
  if (n == 0) return CLIP_OK;
  if (!z || !phi || !valid || !labels || !workspace) return CLIP_EINVAL;
  if (!aligned(z, 4) || !aligned(phi, 4) || !aligned(labels, 4) || !aligned(workspace, 256) ||
      (nregions && !aligned(nregions, 4)) || (d_rounds && !aligned(d_rounds, 4)))
    return CLIP_EALIGN;
  if (workspace_bytes < clip_cluster_workspace_bytes(nframes, height, width)) return CLIP_ENOSPACE;
  return status_of(launch_cluster(z, phi, valid, nframes, height, width, params->t_z, params->t_phi,
                                  params->alpha_z, params->alpha_phi, max_rounds, labels, nregions, d_rounds,
                                  workspace, reinterpret_cast<cudaStream_t>(stream)));
}

int clip_homog_segments_f32(const float* in, int64_t ld_in, int64_t n, int ndc, float* out, int64_t ld_out,
                            uint8_t* flags, void* stream) {
  return homog_dense<float>(in, ld_in, n, ndc, out, ld_out, flags, stream);
}

int clip_homog_segments_f64(const double* in, int64_t ld_in, int64_t n, int ndc, double* out, int64_t ld_out,
                            uint8_t* flags, void* stream) {
  return homog_dense<double>(in, ld_in, n, ndc, out, ld_out, flags, stream);
}

int clip_homog_segments_compact_f32(const float* in, int64_t ld_in, int64_t n, int ndc, float* out, int64_t ld_out,
                                    int64_t* out_index, int64_t index_base, uint8_t* flags, int64_t* d_count,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  return homog_compact<float>(in, ld_in, n, ndc, out, ld_out, out_index, index_base, flags, d_count, workspace,
                              workspace_bytes, stream);
}

int clip_homog_segments_compact_f64(const double* in, int64_t ld_in, int64_t n, int ndc, double* out, int64_t ld_out,
                                    int64_t* out_index, int64_t index_base, uint8_t* flags, int64_t* d_count,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  return homog_compact<double>(in, ld_in, n, ndc, out, ld_out, out_index, index_base, flags, d_count, workspace,
                               workspace_bytes, stream);
}

}  // extern "C"
