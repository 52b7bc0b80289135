// cluster.cu — K6 (NEXT-3): the paper's GPU hot path, round-synchronous
// mutual-best merging of the 4-neighbourhood region graph (§4.1) with
// the §4.2 criterion (Eqs. (1)-(3)), for a batch of frames at once.
//
// One persistent cooperative kernel runs every round; grid-wide barriers separate the
// phases of a round (the paper's Find Mergepartner / Merge Regions / Update Values, Table 2):
//   A  live edges: move the endpoints absorbed last round to their survivors (one hop), drop
//      self-loops, append the edge to the next live list; Eq. (1) test and Eq. (2)
//      distance on the frozen means; per endpoint the minimum distance (64-bit atomicMin on
//      the non-negative double's bits);
//   B  live edges: among the allowed neighbours at that minimum, the largest id (rule 2);
//   C  live regions: mutual pairs (rule 3): the smaller id is absorbed (parent = partner), the
//      larger adds the partner's count and fp64 sums and refreshes its means; the survivors
//      and the unmatched form the next live list.
// The live lists shrink with the graph (append order is irrelevant: every decision is an
// order-free min / max / pair test), the per-round choice arrays are double-buffered so the
// next round's are reset while this round's are read, and a round that merges nothing ends
// the loop.  Finally pointer jumping resolves every pixel's surviving region id.  Region g of
// the batch is pixel g (frame g / P, id g % P + 1).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "clip_kernels.cuh"

namespace cg = cooperative_groups;

namespace clipseg {

namespace {

struct ClusterWs {  // views into the caller's workspace, n = nframes * P regions
  int* cnt;                     // pixels of region g
  int* parent;                  // g, or the region that absorbed g
  int* bestid[2];               // rule 2 choice (partner id, 0 = none), per round parity
  unsigned long long* bestd[2]; // minimum Eq. (2) distance (bits of a non-negative double)
  unsigned long long* ed;       // this round's live edges: Eq. (2) distance bits, ~0 if not allowed
  int* ea[2];                   // live edge lists (endpoints), per round parity
  int* eb[2];
  int* rl[2];                   // live region lists, per round parity
  int* counts;                  // [0..1] live edges, [2..3] live regions, [4..5] merges, [6] flag
  double* sz;                   // fp64 sums of the pixels' binary32 z and phi (DESIGN M-b)
  double* sp;
  double2* m;                   // means (sz / cnt, sp / cnt): one 16-byte load per endpoint
};

struct MergeParams {
  double t_z, t_phi, alpha_z, alpha_phi;
};

__device__ __forceinline__ bool eq1(const ClusterWs& w, int a, int b, const MergeParams& p, double* dist) {
  const double2 ma = w.m[a], mb = w.m[b];
  const double dz = fabs(__dsub_rn(ma.x, mb.x)), dp = fabs(__dsub_rn(ma.y, mb.y));
  *dist = __dadd_rn(__dmul_rn(p.alpha_z, dz), __dmul_rn(p.alpha_phi, dp));  // Eq. (2)
  return dz <= p.t_z && dp <= p.t_phi;                                         // Eq. (1)
}

// Warp-aggregated append: one atomic per warp; returns this lane's slot (if pred).
__device__ __forceinline__ int append_slot(int* counter, bool pred) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, pred);
  if (m == 0) return -1;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(act, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(256) cluster_kernel(const float* __restrict__ z, const float* __restrict__ phi,
                                                       const uint8_t* __restrict__ valid, int64_t nframes, int H,
                                                       int W, MergeParams prm, ClusterWs w, int max_rounds,
                                                       int* __restrict__ labels, int* __restrict__ nregions,
                                                       int* __restrict__ rounds_out) {
  cg::grid_group grid = cg::this_grid();
  const int64_t P = (int64_t)H * W, n = nframes * P;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  int* const ecount = w.counts;
  int* const rcount = w.counts + 2;
  int* const merges = w.counts + 4;
  int* const changed = w.counts + 6;

  // init: one region per valid pixel, the live lists of round 0
  for (int64_t g = t0; g < n; g += stride) {
    const bool v = valid[g] != 0;
    w.cnt[g] = v;
    w.parent[g] = (int)g;
    w.bestid[0][g] = 0;
    w.bestd[0][g] = ~0ull;
    const double zz = v ? (double)z[g] : 0.0, pp = v ? (double)phi[g] : 0.0;
    w.sz[g] = zz;
    w.sp[g] = pp;
    w.m[g] = make_double2(zz, pp);
    const int64_t q = g % P;
    const int x = (int)(q % W), y = (int)(q / W);
    const bool r = v && x + 1 < W && valid[g + 1] != 0, d = v && y + 1 < H && valid[g + W] != 0;
    int slot = append_slot(ecount + 0, r);
    if (r) {
      w.ea[0][slot] = (int)g;
      w.eb[0][slot] = (int)(g + 1);
    }
    slot = append_slot(ecount + 0, d);
    if (d) {
      w.ea[0][slot] = (int)g;
      w.eb[0][slot] = (int)(g + W);
    }
    slot = append_slot(rcount + 0, v);
    if (v) w.rl[0][slot] = (int)g;
  }
  grid.sync();

  int round = 0;
  for (; round < max_rounds; ++round) {
    const int cur = round & 1, nxt = cur ^ 1;
    // A: remap + compact the live edges; minimum Eq. (2) distance over allowed neighbours
    const int ne = ecount[cur];
    if (t0 == 0) rcount[nxt] = 0;  // last read by the previous round's phase C loop bound
    for (int64_t e = t0; e < ne; e += stride) {
      const int a = w.parent[w.ea[cur][e]], b = w.parent[w.eb[cur][e]];
      const bool live = a != b;
      const int slot = append_slot(ecount + nxt, live);
      if (!live) continue;
      w.ea[nxt][slot] = a;
      w.eb[nxt][slot] = b;
      double dist;
      const bool ok = eq1(w, a, b, prm, &dist);
      const unsigned long long bits = ok ? (unsigned long long)__double_as_longlong(dist) : ~0ull;
      w.ed[slot] = bits;  // phase B reads it back instead of recomputing from random means
      if (ok) {
        atomicMin(w.bestd[cur] + a, bits);
        atomicMin(w.bestd[cur] + b, bits);
      }
    }
    grid.sync();
    // B: the largest id among the neighbours at that distance (rule 2)
    const int ne2 = ecount[nxt];
    if (t0 == 0) ecount[cur] = 0;  // the list just read becomes the next round's output
    for (int64_t e = t0; e < ne2; e += stride) {
      const unsigned long long bits = w.ed[e];
      if (bits == ~0ull) continue;  // not allowed by Eq. (1)
      const int a = w.ea[nxt][e], b = w.eb[nxt][e];
      if (bits == w.bestd[cur][a]) atomicMax(w.bestid[cur] + a, (int)(b % P) + 1);
      if (bits == w.bestd[cur][b]) atomicMax(w.bestid[cur] + b, (int)(a % P) + 1);
    }
    grid.sync();
    // C: mutual pairs merge into the larger id (rule 3); the next live region list
    const int nr = rcount[cur];
    if (t0 == 0) merges[nxt] = 0;
    for (int64_t i = t0; i < nr; i += stride) {
      const int g = w.rl[cur][i];
      const int bi = w.bestid[cur][g];
      const int64_t base = g - g % P;
      const int me = (int)(g % P) + 1;
      const int pg = (int)(base + bi - 1);
      const bool mutual = bi != 0 && w.bestid[cur][pg] == me;
      const bool absorbed = mutual && me < bi;
      if (absorbed) {
        w.parent[g] = pg;  // its count and sums stay readable for the survivor
      } else if (mutual) {
        const int c = w.cnt[g] + w.cnt[pg];
        const double s1 = __dadd_rn(w.sz[g], w.sz[pg]), s2 = __dadd_rn(w.sp[g], w.sp[pg]);
        w.cnt[g] = c;
        w.sz[g] = s1;
        w.sp[g] = s2;
        w.m[g] = make_double2(__ddiv_rn(s1, (double)c), __ddiv_rn(s2, (double)c));
        atomicAdd(merges + cur, 1);
      }
      const int slot = append_slot(rcount + nxt, !absorbed);
      if (!absorbed) {
        w.rl[nxt][slot] = g;
        w.bestid[nxt][g] = 0;  // the next round's choices (last used two rounds ago)
        w.bestd[nxt][g] = ~0ull;
      }
    }
    grid.sync();
    if (merges[cur] == 0) break;  // the same value for every thread: uniform exit
  }
  if (t0 == 0 && rounds_out) atomicMax(rounds_out, round < max_rounds ? round + 1 : max_rounds);

  // labels: pointer jumping to the surviving region, then its id (0 for invalid pixels)
  for (;;) {
    if (t0 == 0) *changed = 0;
    grid.sync();
    int ch = 0;
    for (int64_t g = t0; g < n; g += stride) {
      const int p = w.parent[g], pp = w.parent[p];
      if (pp != p) {
        w.parent[g] = pp;
        ch = 1;
      }
    }
    if (ch) atomicOr(changed, 1);
    grid.sync();
    if (*changed == 0) break;
    grid.sync();  // everyone has read the flag before it is reset
  }
  for (int64_t g = t0; g < n; g += stride) {
    const bool v = valid[g] != 0;
    const int root = w.parent[g];
    labels[g] = v ? (int)(root % P) + 1 : 0;
    if (v && root == (int)g && nregions) atomicAdd(nregions + g / P, 1);
  }
}

// One block per frame: frames are independent, so a frame's rounds need only block-level
// barriers (__syncthreads) instead of grid-wide ones, and many frames run concurrently.  The
// phases and every decision are those of cluster_kernel, restricted to the frame's pixels;
// the frame's live lists live in its slice of the workspace, their counters in shared memory.
#ifndef CLIPSEG_CLUSTER_FRAME_THREADS
#define CLIPSEG_CLUSTER_FRAME_THREADS 1024
#endif
__global__ void __launch_bounds__(CLIPSEG_CLUSTER_FRAME_THREADS) cluster_frame_kernel(const float* __restrict__ z,
                                                              const float* __restrict__ phi,
                                                              const uint8_t* __restrict__ valid, int64_t nframes,
                                                              int H, int W, MergeParams prm, ClusterWs w,
                                                              int max_rounds, int* __restrict__ labels,
                                                              int* __restrict__ nregions, int* __restrict__ rounds_out) {
  __shared__ int ecount[2], rcount[2], merges[2], changed, roots;
  const int64_t P = (int64_t)H * W;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t f = blockIdx.x; f < nframes; f += gridDim.x) {
    const int64_t base = f * P;
    int* const ea0 = w.ea[0] + 2 * base;
    int* const ea1 = w.ea[1] + 2 * base;
    int* const eb0 = w.eb[0] + 2 * base;
    int* const eb1 = w.eb[1] + 2 * base;
    int* const rl0 = w.rl[0] + base;
    int* const rl1 = w.rl[1] + base;
    unsigned long long* const ed = w.ed + 2 * base;
    if (tid == 0) {
      ecount[0] = ecount[1] = rcount[0] = rcount[1] = merges[0] = merges[1] = roots = 0;
    }
    __syncthreads();
    for (int64_t q = tid; q < P; q += nt) {
      const int64_t g = base + q;
      const bool v = valid[g] != 0;
      w.cnt[g] = v;
      w.parent[g] = (int)g;
      w.bestid[0][g] = 0;
      w.bestd[0][g] = ~0ull;
      const double zz = v ? (double)z[g] : 0.0, pp = v ? (double)phi[g] : 0.0;
      w.sz[g] = zz;
      w.sp[g] = pp;
      w.m[g] = make_double2(zz, pp);
      const int x = (int)(q % W), y = (int)(q / W);
      const bool r = v && x + 1 < W && valid[g + 1] != 0, d = v && y + 1 < H && valid[g + W] != 0;
      int slot = append_slot(ecount + 0, r);
      if (r) {
        ea0[slot] = (int)g;
        eb0[slot] = (int)(g + 1);
      }
      slot = append_slot(ecount + 0, d);
      if (d) {
        ea0[slot] = (int)g;
        eb0[slot] = (int)(g + W);
      }
      slot = append_slot(rcount + 0, v);
      if (v) rl0[slot] = (int)g;
    }
    __syncthreads();
    int round = 0;
    for (; round < max_rounds; ++round) {
      const int cur = round & 1, nxt = cur ^ 1;
      int* const eac = cur ? ea1 : ea0;  // this round's lists (pointers, not indexed arrays:
      int* const ebc = cur ? eb1 : eb0;  // no local memory)
      int* const ean = cur ? ea0 : ea1;
      int* const ebn = cur ? eb0 : eb1;
      int* const rlc = cur ? rl1 : rl0;
      int* const rln = cur ? rl0 : rl1;
      const int ne = ecount[cur];
      if (tid == 0) rcount[nxt] = 0;
      for (int e = tid; e < ne; e += nt) {  // A
        const int a = w.parent[eac[e]], b = w.parent[ebc[e]];
        const bool live = a != b;
        const int slot = append_slot(ecount + nxt, live);
        if (!live) continue;
        ean[slot] = a;
        ebn[slot] = b;
        double dist;
        const bool ok = eq1(w, a, b, prm, &dist);
        const unsigned long long bits = ok ? (unsigned long long)__double_as_longlong(dist) : ~0ull;
        ed[slot] = bits;
        if (ok) {
          atomicMin(w.bestd[cur] + a, bits);
          atomicMin(w.bestd[cur] + b, bits);
        }
      }
      __syncthreads();
      const int ne2 = ecount[nxt];
      if (tid == 0) ecount[cur] = 0;
      for (int e = tid; e < ne2; e += nt) {  // B
        const unsigned long long bits = ed[e];
        if (bits == ~0ull) continue;
        const int a = ean[e], b = ebn[e];
        if (bits == w.bestd[cur][a]) atomicMax(w.bestid[cur] + a, (int)(b - base) + 1);
        if (bits == w.bestd[cur][b]) atomicMax(w.bestid[cur] + b, (int)(a - base) + 1);
      }
      __syncthreads();
      const int nr = rcount[cur];
      if (tid == 0) merges[nxt] = 0;
      for (int i = tid; i < nr; i += nt) {  // C
        const int g = rlc[i];
        const int bi = w.bestid[cur][g];
        const int me = (int)(g - base) + 1;
        const int pg = (int)(base + bi - 1);
        const bool mutual = bi != 0 && w.bestid[cur][pg] == me;
        const bool absorbed = mutual && me < bi;
        if (absorbed) {
          w.parent[g] = pg;
        } else if (mutual) {
          const int c = w.cnt[g] + w.cnt[pg];
          const double s1 = __dadd_rn(w.sz[g], w.sz[pg]), s2 = __dadd_rn(w.sp[g], w.sp[pg]);
          w.cnt[g] = c;
          w.sz[g] = s1;
          w.sp[g] = s2;
          w.m[g] = make_double2(__ddiv_rn(s1, (double)c), __ddiv_rn(s2, (double)c));
          atomicAdd(merges + cur, 1);
        }
        const int slot = append_slot(rcount + nxt, !absorbed);
        if (!absorbed) {
          rln[slot] = g;
          w.bestid[nxt][g] = 0;
          w.bestd[nxt][g] = ~0ull;
        }
      }
      __syncthreads();
      if (merges[cur] == 0) break;  // block-uniform
    }
    if (tid == 0 && rounds_out) atomicMax(rounds_out, round < max_rounds ? round + 1 : max_rounds);
    for (;;) {  // pointer jumping within the frame
      if (tid == 0) changed = 0;
      __syncthreads();
      int ch = 0;
      for (int64_t q = tid; q < P; q += nt) {
        const int64_t g = base + q;
        const int pp = w.parent[g], p2 = w.parent[pp];
        if (p2 != pp) {
          w.parent[g] = p2;
          ch = 1;
        }
      }
      if (ch) atomicOr(&changed, 1);
      __syncthreads();
      const int done = changed == 0;
      __syncthreads();
      if (done) break;
    }
    int mine = 0;
    for (int64_t q = tid; q < P; q += nt) {
      const int64_t g = base + q;
      const bool v = valid[g] != 0;
      const int root = w.parent[g];
      labels[g] = v ? (int)(root - base) + 1 : 0;
      mine += v && root == (int)g;
    }
    if (mine) atomicAdd(&roots, mine);
    __syncthreads();
    if (tid == 0 && nregions) nregions[f] = roots;
    __syncthreads();
  }
}

}  // namespace

size_t cluster_workspace_bytes(int64_t n) {
  // sums/means 4 x 8, choices 2 x (8 + 4), cnt/parent 2 x 4, edges 2 x 2 x 2 x 4, edge
  // distances 2 x 8, regions 2 x 4
  return (size_t)n * (32 + 24 + 8 + 32 + 16 + 8) + 16 * 256;
}

// One cooperative launch for frames [f0, f0 + nf) of the batch, workspace laid out for nf.
static cudaError_t launch_cluster_part(const float* z, const float* phi, const uint8_t* valid, int64_t nf, int H,
                                       int W, const MergeParams& prm, int max_rounds, int* labels, int* nregions,
                                       int* rounds_out, void* ws, bool per_frame, cudaStream_t s) {
  const int64_t n = nf * (int64_t)H * W;
  char* p = reinterpret_cast<char*>(ws);
  ClusterWs w;
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) & ~(size_t)255;
    return q;
  };
  w.sz = reinterpret_cast<double*>(take(8 * n));
  w.sp = reinterpret_cast<double*>(take(8 * n));
  w.m = reinterpret_cast<double2*>(take(16 * n));
  for (int q = 0; q < 2; ++q) {
    w.bestd[q] = reinterpret_cast<unsigned long long*>(take(8 * n));
    w.bestid[q] = reinterpret_cast<int*>(take(4 * n));
    w.ea[q] = reinterpret_cast<int*>(take(8 * n));
    w.eb[q] = reinterpret_cast<int*>(take(8 * n));
    w.rl[q] = reinterpret_cast<int*>(take(4 * n));
  }
  w.ed = reinterpret_cast<unsigned long long*>(take(16 * n));
  w.cnt = reinterpret_cast<int*>(take(4 * n));
  w.parent = reinterpret_cast<int*>(take(4 * n));
  w.counts = reinterpret_cast<int*>(take(64));
  const cudaError_t e = cudaMemsetAsync(w.counts, 0, 64, s);
  if (e != cudaSuccess) return e;
  int blocks_per_sm = 0;  // per device, cached (kernel_occupancy)
  const cudaError_t e2 = kernel_occupancy((const void*)cluster_kernel, 256, 0, &blocks_per_sm);
  if (e2 != cudaSuccess) return e2;
#ifndef CLIPSEG_CLUSTER_PIX_PER_BLOCK
#define CLIPSEG_CLUSTER_PIX_PER_BLOCK 512  // pixels per block (128..2048 measured alike; 8192 slower)
#endif
  const int64_t want = (n + CLIPSEG_CLUSTER_PIX_PER_BLOCK - 1) / CLIPSEG_CLUSTER_PIX_PER_BLOCK;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  MergeParams prm_copy = prm;
  if (per_frame) {  // one block per frame (a grid-stride loop over the part's frames)
    const int fgrid = (int)(nf < (1 << 20) ? nf : (1 << 20));
    cluster_frame_kernel<<<fgrid, CLIPSEG_CLUSTER_FRAME_THREADS, 0, s>>>(z, phi, valid, nf, H, W, prm_copy, w,
                                                                         max_rounds, labels, nregions, rounds_out);
    return cudaGetLastError();
  }
  void* args[] = {(void*)&z, (void*)&phi, (void*)&valid, (void*)&nf, (void*)&H, (void*)&W, (void*)&prm_copy,
                  (void*)&w, (void*)&max_rounds, (void*)&labels, (void*)&nregions, (void*)&rounds_out};
  return cudaLaunchCooperativeKernel((const void*)cluster_kernel, dim3(grid), dim3(256), args, 0, s);
}

cudaError_t launch_cluster(const float* z, const float* phi, const uint8_t* valid, int64_t nframes, int H, int W,
                           double t_z, double t_phi, double alpha_z, double alpha_phi, int max_rounds, int* labels,
                           int* nregions, int* rounds_out, void* ws, cudaStream_t s) {
  const MergeParams prm{t_z, t_phi, alpha_z, alpha_phi};
  if (nregions) {
    const cudaError_t e = cudaMemsetAsync(nregions, 0, (size_t)nframes * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  if (rounds_out) {
    const cudaError_t e = cudaMemsetAsync(rounds_out, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  // Frames are independent: batches run as consecutive launches of at most
  // cluster_part_frames() frames with the schedule chosen by the batch size (clip_kernels.cuh);
  // the workspace is sized for one part.
  const int64_t P = (int64_t)H * W;
  const bool per_frame = nframes >= kClusterPerFrameMin;
  const int64_t part = cluster_part_frames(nframes);
  for (int64_t f0 = 0; f0 < nframes; f0 += part) {
    const int64_t nf = nframes - f0 < part ? nframes - f0 : part;
    const cudaError_t e = launch_cluster_part(z + f0 * P, phi + f0 * P, valid + f0 * P, nf, H, W, prm, max_rounds,
                                              labels + f0 * P, nregions ? nregions + f0 : nullptr, rounds_out, ws,
                                              per_frame, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace clipseg
