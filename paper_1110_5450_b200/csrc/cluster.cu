// cluster.cu — K6 (NEXT-3): the paper's GPU hot path, round-synchronous
// mutual-best merging of the 4-neighbourhood region graph (§4.1) with
// the §4.2 criterion (Eqs. (1)-(3)), for a batch of frames at once.
//
// One persistent cooperative kernel runs every round; grid-wide barriers separate the
// phases of a round (the paper's Find Mergepartner / Merge Regions / Update Values, Table 2):
//   A  edges:   Eq. (1) test and Eq. (2) distance on the frozen means; per endpoint the
//               minimum distance (64-bit atomicMin on the non-negative double's bits);
//   B  edges:   among the allowed neighbours at that minimum, the largest id (rule 2);
//   C  regions: mutual pairs (rule 3): the smaller id is absorbed (parent = partner), the
//               larger id adds the partner's count and fp64 sums and refreshes its means;
//   D  regions / edges: reset the choices; edges of absorbed regions move to the survivor,
//               edges that became self-loops die.
// A round that merges nothing ends the loop.  Finally pointer jumping resolves every
// pixel's surviving region id.  Region g of the batch is pixel g (frame g / P, id g % P + 1).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "clip_kernels.cuh"

namespace cg = cooperative_groups;

namespace clipseg {

namespace {

struct ClusterWs {  // views into the caller's workspace, n = nframes * P regions
  int* cnt;                  // pixels of region g (0: not a region / absorbed)
  int* parent;               // g, or the region that absorbed g
  int* bestid;               // rule 2 choice (partner id), 0 = none
  int* ea;                   // edge endpoints (2 slots per pixel: right, down), -1 = dead
  int* eb;
  int* merges;               // [2] merged pairs of the current / next round
  int* changed;              // pointer-jumping flag
  double* sz;                // fp64 sums of the pixels' binary32 z and phi (DESIGN M-b)
  double* sp;
  double* mz;                // means sz / cnt, sp / cnt
  double* mp;
  unsigned long long* bestd; // minimum Eq. (2) distance (bits of a non-negative double)
};

struct MergeParams {
  double t_z, t_phi, alpha_z, alpha_phi;
};

__device__ __forceinline__ bool eq1(const ClusterWs& w, int a, int b, const MergeParams& p, double* dist) {
  const double dz = fabs(__dsub_rn(w.mz[a], w.mz[b])), dp = fabs(__dsub_rn(w.mp[a], w.mp[b]));
  *dist = __dadd_rn(__dmul_rn(p.alpha_z, dz), __dmul_rn(p.alpha_phi, dp));  // Eq. (2)
  return dz <= p.t_z && dp <= p.t_phi;                                         // Eq. (1)
}

__global__ void __launch_bounds__(256) cluster_kernel(const float* __restrict__ z, const float* __restrict__ phi,
                                                       const uint8_t* __restrict__ valid, int64_t nframes, int H,
                                                       int W, MergeParams prm, ClusterWs w, int max_rounds,
                                                       int* __restrict__ labels, int* __restrict__ nregions,
                                                       int* __restrict__ rounds_out) {
  cg::grid_group grid = cg::this_grid();
  const int64_t P = (int64_t)H * W, n = nframes * P, ne = 2 * n;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;

  // init: one region per valid pixel; edges to the right and lower valid neighbours
  for (int64_t g = t0; g < n; g += stride) {
    const bool v = valid[g] != 0;
    w.cnt[g] = v;
    w.parent[g] = (int)g;
    w.bestid[g] = 0;
    w.bestd[g] = ~0ull;
    const double zz = v ? (double)z[g] : 0.0, pp = v ? (double)phi[g] : 0.0;
    w.sz[g] = zz;
    w.sp[g] = pp;
    w.mz[g] = zz;
    w.mp[g] = pp;
    const int64_t q = g % P;
    const int x = (int)(q % W), y = (int)(q / W);
    const bool r = v && x + 1 < W && valid[g + 1] != 0, d = v && y + 1 < H && valid[g + W] != 0;
    w.ea[2 * g] = r ? (int)g : -1;
    w.eb[2 * g] = (int)(g + 1);
    w.ea[2 * g + 1] = d ? (int)g : -1;
    w.eb[2 * g + 1] = (int)(g + W);
  }
  if (t0 == 0) {
    w.merges[0] = 0;
    w.merges[1] = 0;
  }
  grid.sync();

  int round = 0;
  for (; round < max_rounds; ++round) {
    // A: minimum Eq. (2) distance over the allowed neighbours
    for (int64_t e = t0; e < ne; e += stride) {
      const int a = w.ea[e];
      if (a < 0) continue;
      const int b = w.eb[e];
      double dist;
      if (eq1(w, a, b, prm, &dist)) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(dist);
        atomicMin(w.bestd + a, bits);
        atomicMin(w.bestd + b, bits);
      }
    }
    grid.sync();
    // B: the largest id among the neighbours at that distance (rule 2)
    for (int64_t e = t0; e < ne; e += stride) {
      const int a = w.ea[e];
      if (a < 0) continue;
      const int b = w.eb[e];
      double dist;
      if (eq1(w, a, b, prm, &dist)) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(dist);
        if (bits == w.bestd[a]) atomicMax(w.bestid + a, (int)(b % P) + 1);
        if (bits == w.bestd[b]) atomicMax(w.bestid + b, (int)(a % P) + 1);
      }
    }
    grid.sync();
    // C: mutual pairs merge into the larger id (rules 3)
    for (int64_t g = t0; g < n; g += stride) {
      const int bi = w.bestid[g];
      if (bi == 0 || w.cnt[g] == 0) continue;
      const int64_t base = g - g % P, me = (int)(g % P) + 1, pg = base + bi - 1;
      if (w.bestid[pg] != me) continue;  // not mutual: wait
      if (me < bi) {
        w.parent[g] = (int)pg;  // absorbed; its count and sums stay readable for the survivor
      } else {
        const int c = w.cnt[g] + w.cnt[pg];
        const double s1 = __dadd_rn(w.sz[g], w.sz[pg]), s2 = __dadd_rn(w.sp[g], w.sp[pg]);
        w.cnt[g] = c;
        w.sz[g] = s1;
        w.sp[g] = s2;
        w.mz[g] = __ddiv_rn(s1, (double)c);
        w.mp[g] = __ddiv_rn(s2, (double)c);
        atomicAdd(w.merges + (round & 1), 1);
      }
    }
    grid.sync();
    // D: reset choices, retire absorbed regions, move their edges to the survivors
    for (int64_t g = t0; g < n; g += stride) {
      w.bestid[g] = 0;
      w.bestd[g] = ~0ull;
      if (w.parent[g] != (int)g && w.cnt[g] != 0) w.cnt[g] = 0;  // absorbed this round
    }
    for (int64_t e = t0; e < ne; e += stride) {
      const int a = w.ea[e];
      if (a < 0) continue;
      const int b = w.eb[e];
      const int a2 = w.parent[a], b2 = w.parent[b];  // one hop: a survivor's parent is itself
      if (a2 == b2) {
        w.ea[e] = -1;
      } else if (a2 != a || b2 != b) {
        w.ea[e] = a2;
        w.eb[e] = b2;
      }
    }
    if (t0 == 0) w.merges[(round + 1) & 1] = 0;
    grid.sync();
    if (w.merges[round & 1] == 0) break;  // the same value for every thread: uniform exit
  }
  if (t0 == 0 && rounds_out) *rounds_out = round < max_rounds ? round + 1 : max_rounds;

  // labels: pointer jumping to the surviving region, then its id (0 for invalid pixels)
  for (;;) {
    if (t0 == 0) *w.changed = 0;
    grid.sync();
    int ch = 0;
    for (int64_t g = t0; g < n; g += stride) {
      const int p = w.parent[g], pp = w.parent[p];
      if (pp != p) {
        w.parent[g] = pp;
        ch = 1;
      }
    }
    if (ch) atomicOr(w.changed, 1);
    grid.sync();
    if (*w.changed == 0) break;
    grid.sync();  // everyone has read the flag before it is reset
  }
  for (int64_t g = t0; g < n; g += stride) {
    const bool v = valid[g] != 0;
    const int root = w.parent[g];
    labels[g] = v ? (int)(root % P) + 1 : 0;
    if (v && root == (int)g && nregions) atomicAdd(nregions + g / P, 1);
  }
}

}  // namespace

size_t cluster_workspace_bytes(int64_t n) {
  return (size_t)n * (4 * 3 + 4 * 4 + 8 * 5) + 64;  // cnt/parent/bestid, ea/eb, sums/means/bestd
}

cudaError_t launch_cluster(const float* z, const float* phi, const uint8_t* valid, int64_t nframes, int H, int W,
                           double t_z, double t_phi, double alpha_z, double alpha_phi, int max_rounds, int* labels,
                           int* nregions, int* rounds_out, void* ws, cudaStream_t s) {
  const int64_t n = nframes * (int64_t)H * W;
  char* p = reinterpret_cast<char*>(ws);
  ClusterWs w;
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) & ~(size_t)255;
    return q;
  };
  w.sz = reinterpret_cast<double*>(take(8 * n));
  w.sp = reinterpret_cast<double*>(take(8 * n));
  w.mz = reinterpret_cast<double*>(take(8 * n));
  w.mp = reinterpret_cast<double*>(take(8 * n));
  w.bestd = reinterpret_cast<unsigned long long*>(take(8 * n));
  w.cnt = reinterpret_cast<int*>(take(4 * n));
  w.parent = reinterpret_cast<int*>(take(4 * n));
  w.bestid = reinterpret_cast<int*>(take(4 * n));
  w.ea = reinterpret_cast<int*>(take(8 * n));
  w.eb = reinterpret_cast<int*>(take(8 * n));
  w.merges = reinterpret_cast<int*>(take(16));
  w.changed = w.merges + 2;
  MergeParams prm{t_z, t_phi, alpha_z, alpha_phi};
  if (nregions) {
    const cudaError_t e = cudaMemsetAsync(nregions, 0, (size_t)nframes * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, cluster_kernel, 256, 0);
    if (e != cudaSuccess || blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t want = (2 * n + 255) / 256;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  void* args[] = {(void*)&z, (void*)&phi, (void*)&valid, (void*)&nframes, (void*)&H, (void*)&W, (void*)&prm,
                  (void*)&w, (void*)&max_rounds, (void*)&labels, (void*)&nregions, (void*)&rounds_out};
  return cudaLaunchCooperativeKernel((const void*)cluster_kernel, dim3(grid), dim3(256), args, 0, s);
}

}  // namespace clipseg
