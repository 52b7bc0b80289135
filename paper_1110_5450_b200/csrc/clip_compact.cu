// clip_compact.cu — K3: stable compacting clip in one pass (R1-R10).
//
// Single-pass stream compaction with tile aggregates published in global memory
// (decoupled look-back, Merrill & Garland), organised for sm_100a as a warp-specialised,
// software-pipelined persistent kernel.  Co-resident grid (cooperative launch):
//
//  * block 0 is the GLOBAL SCANNER: one warp walks the per-tile status words in tile order,
//    512 per probe, and turns every run of published aggregates (flag A) into inclusive
//    prefixes (flag P).  A tile's offset is thus known about one L2 round trip after the
//    last of its predecessors has published, with no redundant per-tile walks;
//
//  * every other block (one per SM) claims block tiles of BT = NSUB x 128 segments in
//    increasing order from an atomic counter (the first of its compute warps to start a
//    tile claims the block's next one, so claims follow the order blocks start computing;
//    the shapes per instantiation are in clip_kernels.cuh — fp32 2D: 16 compute warps, 32
//    sub-tiles, 3 staged tiles) and runs
//      - the compute warps.  Per sub-tile (32 lanes x 4 segments, one 128-bit load per plane
//        per lane; the next sub-tile's loads — across tile boundaries — in flight while this
//        one is clipped) a warp
//        classifies and clips its segments (clip_math.cuh), stores the flags, warp-scans the
//        visible counts and stages the visible rows, compacted, in its slot of stage buffer
//        k % NBUF.  The last warp to finish a tile publishes its aggregate (flag A).  Then
//        each warp copies ITS OWN staged rows of tile k - (NBUF-1), whose offset is known by
//        then, to their global rows (coalesced) — so compute warps neither wait for one
//        another nor, normally, for the offsets;
//      - 1 scan warp: once tile k's counts are in, it prefix-sums the NSUB sub-tile counts,
//        waits for the scanner's inclusive prefix of the tile and hands the offsets over.
//
// Hand-offs inside a block use shared-memory mbarriers (compute warps -> scan warp: one
// arrival per compute warp per tile; scan warp -> compute warps: 1; claiming warp -> all:
// the tile id, a ring of 8).  Status words are 64-bit: flag in bits 62-63 (0 not ready, 1 aggregate,
// 2 inclusive prefix), value in bits 0-61.  The scanner writes the total count.
#include <type_traits>

#include "clip_kernels.cuh"
#include "vec_io.cuh"

namespace clipseg {

#ifdef CLIPSEG_TRACE
// Debug build only (scripts/trace_compact.py): per-tile timeline in %globaltimer ns.
// slots: 0 claimed, 1 compute start, 2 aggregate published, 3 prefix wait start,
// 4 prefix seen by the block, 5 prefix published by the scanner, 6 copy start, 7 block id.
constexpr int kTraceTiles = 1 << 19;
__device__ unsigned long long g_trace[kTraceTiles * 8];
__device__ __forceinline__ unsigned long long trace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CLIP_TRACE(tile, slot, val)                                                \
  do {                                                                              \
    if ((tile) >= 0 && (tile) < kTraceTiles) g_trace[(tile) * 8 + (slot)] = (val); \
  } while (0)
#else
#define CLIP_TRACE(tile, slot, val) \
  do {                              \
  } while (0)
#endif

namespace {

constexpr unsigned long long kFlagA = 1ull << 62;
constexpr unsigned long long kFlagP = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;
#ifndef CLIPSEG_SCAN_PER_LANE
#define CLIPSEG_SCAN_PER_LANE 2  // scanner: lanes probe 2 tiles each (16: +1.6 % at 1e9, profiles/r01_summary.md)
#endif
#ifndef CLIPSEG_SCANNER_MAX_BACKOFF
#define CLIPSEG_SCANNER_MAX_BACKOFF 0  // scanner: longest sleep between empty probes (0: spin; block 0 computes nothing)
#endif
constexpr int kScanPerLane = CLIPSEG_SCAN_PER_LANE;  // scanner: 32 x this tiles per probe
#ifndef CLIPSEG_POLL_NS
#define CLIPSEG_POLL_NS 500        // scan warp: sleep between polls of its tile's prefix
#endif
#ifndef CLIPSEG_PRE_SLEEP_NS
#define CLIPSEG_PRE_SLEEP_NS 0     // compute warps: sleep between tests of a tile's offsets (0: suspending try_wait)
#endif
#ifndef CLIPSEG_SCAN_SLEEP_NS
#define CLIPSEG_SCAN_SLEEP_NS 256  // scan warp: sleep between tests of its mbarriers
#endif
#ifndef CLIPSEG_MUL_FLAGS
#define CLIPSEG_MUL_FLAGS 1  // measured -0.6 %
#endif
#ifndef CLIPSEG_IMAD_SELECT
#define CLIPSEG_IMAD_SELECT 1
#endif
#ifndef CLIPSEG_STORE_HINT
#define CLIPSEG_STORE_HINT 0       // copy-out stores: 0 evict-first (st.cs), 1 plain
#endif
// Claimed-tile ring: a slot is rewritten kTileRing iterations after its first use; it must
// exceed the copy lag (NBUF - 1) by enough that no warp still reads the old id.
constexpr int kTileRing = 8, kRingMask = kTileRing - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// One thread's shared-memory fetch-and-add (atomicAdd would wrap it in warp-aggregation code
// for a single active lane).
__device__ __forceinline__ int atom_add_shared(int* p, int v) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_addr(p)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void atom_or_shared_a(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// One thread's global 64-bit fetch-and-add (relaxed, gpu scope).
__device__ __forceinline__ unsigned long long atom_add_global(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
// release: the arriving thread's prior shared-memory writes are visible to the waiters
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(bar))
               : "memory");
}
// acquire: wait until the phase with the given parity has completed.  The suspend-time
// hint lets the hardware park the warp until the phase flips instead of spinning, so
// waiting warps leave the issue slots to the compute warps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// The same on 32-bit shared addresses computed once (no generic-to-shared conversion in the
// hot loop).
__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// Non-blocking: has the phase with the given parity completed?
__device__ __forceinline__ bool mbar_test_a(uint32_t a, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(a), "r"(parity)
      : "memory");
  return done != 0;
}

// Low-duty-cycle wait for the scan warp, which waits most of its life: a non-blocking phase
// test plus a real sleep, so it does not take issue slots from the compute warps it shares
// a scheduler with (a suspending try_wait is woken by every mbarrier event on the SM).
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t* bar, uint32_t parity, unsigned ns) {
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
  }
}

// Block 0's scan warp: walks the tile statuses in order and turns every run of published
// aggregates that follows the scanned prefix into inclusive prefixes.
__device__ __noinline__ void global_scanner(unsigned long long* status, int64_t ntiles, int lane, int64_t* d_count) {
  constexpr int M = kScanPerLane;
  int64_t base = 0;
  unsigned long long running = 0;
  unsigned backoff = 32;
  while (base < ntiles) {
    unsigned long long s[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int64_t idx = base + lane * M + j;
      s[j] = (idx < ntiles) ? ld_relaxed(status + idx) : 0ull;  // past the end: never ready
    }
    int myx = M;  // this lane's first not-ready tile
#pragma unroll
    for (int j = M - 1; j >= 0; --j)
      if ((s[j] >> 62) == 0u) myx = j;
    const unsigned xmask = __ballot_sync(0xFFFFFFFFu, myx < M);
    const int fl = xmask ? __ffs(xmask) - 1 : 32;
    const int ready = (fl == 32) ? 32 * M : fl * M + __shfl_sync(0xFFFFFFFFu, myx, fl & 31);
    if (ready == 0) {
      if (CLIPSEG_SCANNER_MAX_BACKOFF > 0) __nanosleep(backoff);
      backoff = backoff < CLIPSEG_SCANNER_MAX_BACKOFF ? 2 * backoff : CLIPSEG_SCANNER_MAX_BACKOFF;
      continue;
    }
    backoff = 32;
    unsigned long long vsum = 0;
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (lane * M + j < ready) vsum += s[j] & kValueMask;
    unsigned long long incl = vsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    unsigned long long run = running + incl - vsum;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if (lane * M + j < ready) {
        run += s[j] & kValueMask;
        st_relaxed(status + base + lane * M + j, kFlagP | run);
        CLIP_TRACE(base + lane * M + j, 5, trace_now());
      }
    }
    running += __shfl_sync(0xFFFFFFFFu, incl, 31);
    base += ready;
  }
  if (lane == 0) *d_count = (int64_t)running;
}

// A block's scan warp: for each of the block's tiles in claim order, once its compute warps'
// NSUB counts are in (mb_cnt), exclusive-prefix them, wait for the scanner's inclusive prefix
// of the tile and hand the offsets over (mb_pre).  It then zeroes the tile's status word: the
// scanner never reads a word again once it holds the prefix, so the workspace is all zero
// again when the launch ends and the next call needs no memset.
// s_tileof (nullable): receives each iteration's tile id in its slot, for consumers that
// outlive the tile ring.
template <int NSUB, int NBUF>
__device__ __forceinline__ void tile_scan_warp(int lane, int64_t ntiles, unsigned long long* status,
                                               const int64_t* s_tile, const int (*s_cnt)[NSUB], int (*s_pre)[NSUB],
                                               int64_t* s_prefix, int* s_done, uint64_t* mb_tile, uint64_t* mb_cnt,
                                               uint64_t* mb_pre, int64_t* s_tileof = nullptr, bool publish = false) {
  static_assert(NSUB <= 64, "two counts per lane");
  int b = 0;
  unsigned par = 0;  // bit q: parity of the next phase of mb_cnt[q] / mb_pre[q]
  for (int64_t k = 0;; ++k) {
    mbar_wait_sleepy(&mb_tile[k & kRingMask], (uint32_t)((k / kTileRing) & 1), CLIPSEG_SCAN_SLEEP_NS);
    const int64_t tile = s_tile[k & kRingMask];
    if (tile >= ntiles) break;
    mbar_wait_sleepy(&mb_cnt[b], (par >> b) & 1u, CLIPSEG_SCAN_SLEEP_NS);  // the compute warps' counts of tile k
    // lane holds counts lane and lane + 32, packed in the low / high 16 bits (a tile count
    // is below 2^16)
    const int c0 = (lane < NSUB) ? s_cnt[b][lane] : 0;
    const int c1 = (NSUB > 32 && lane + 32 < NSUB) ? s_cnt[b][lane + 32] : 0;
    const int c = c0 | (c1 << 16);
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    const int tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (lane < NSUB) s_pre[b][lane] = (incl & 0xFFFF) - c0;
    if (NSUB > 32 && lane + 32 < NSUB) s_pre[b][lane + 32] = (tot & 0xFFFF) + (incl >> 16) - c1;
    const int64_t total = (tot & 0xFFFF) + (tot >> 16);
    if (publish && lane == 0) st_relaxed(status + tile, kFlagA | (unsigned long long)total);  // the tile aggregate
    if (lane == 0) {
      CLIP_TRACE(tile, 3, trace_now());
      unsigned long long st;
      while (((st = ld_relaxed(status + tile)) >> 62) != 2u)  // the scanner's inclusive prefix
        __nanosleep(CLIPSEG_POLL_NS);  // it typically lands several microseconds after the aggregate
      CLIP_TRACE(tile, 4, trace_now());
      CLIP_TRACE(tile, 7, blockIdx.x);
      st_relaxed(status + tile, 0ull);  // consumed: leave the word clean for the next call
      s_prefix[b] = (int64_t)(st & kValueMask) - total;
      s_done[b] = 0;
      if (s_tileof) s_tileof[b] = tile;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&mb_pre[b]);  // tile k's offsets published
    par ^= 1u << b;
    b = (b + 1 == NBUF) ? 0 : b + 1;
  }
}

// Block 0's scan warp in the packed kernel: the global scanner above, interleaved with the
// tile duties of tile_scan_warp for block 0's own tiles, both non-blocking (mbarrier tests
// instead of waits), so block 0 computes tiles too instead of leaving one SM idle.  Its own
// tile's inclusive prefix is read back once the scanner's frontier has passed the tile.
template <int NSUB, int NBUF>
__device__ __forceinline__ void scanner_with_tiles(int lane, int64_t ntiles, unsigned long long* status,
                                                   int64_t* d_count, const int64_t* s_tile, const int (*s_cnt)[NSUB],
                                                   int (*s_pre)[NSUB], int64_t* s_prefix, int* s_done,
                                                   uint64_t* mb_tile, uint64_t* mb_cnt, uint64_t* mb_pre) {
  static_assert(NSUB <= 64, "two counts per lane");
  constexpr int M = kScanPerLane;
  int64_t base = 0;
  unsigned long long running = 0;
  int64_t k = 0, tile = 0, total = 0;
  int b = 0, state = 0;  // tile duty of iteration k: 0 claim, 1 counts, 2 prefix, 3 no tiles left
  unsigned par = 0;      // bit q: parity of the next phase of mb_cnt[q] / mb_pre[q]
  while (base < ntiles || state != 3) {
    if (base < ntiles) {  // ---- one scanner probe
      unsigned long long sv[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const int64_t idx = base + lane * M + j;
        sv[j] = (idx < ntiles) ? ld_relaxed(status + idx) : 0ull;
      }
      int myx = M;
#pragma unroll
      for (int j = M - 1; j >= 0; --j)
        if ((sv[j] >> 62) == 0u) myx = j;
      const unsigned xmask = __ballot_sync(0xFFFFFFFFu, myx < M);
      const int fl = xmask ? __ffs(xmask) - 1 : 32;
      const int ready = (fl == 32) ? 32 * M : fl * M + __shfl_sync(0xFFFFFFFFu, myx, fl & 31);
      if (ready > 0) {
        unsigned long long vsum = 0;
#pragma unroll
        for (int j = 0; j < M; ++j)
          if (lane * M + j < ready) vsum += sv[j] & kValueMask;
        unsigned long long incl = vsum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
          if (lane >= d) incl += y;
        }
        unsigned long long run = running + incl - vsum;
#pragma unroll
        for (int j = 0; j < M; ++j) {
          if (lane * M + j < ready) {
            run += sv[j] & kValueMask;
            st_relaxed(status + base + lane * M + j, kFlagP | run);
            CLIP_TRACE(base + lane * M + j, 5, trace_now());
          }
        }
        running += __shfl_sync(0xFFFFFFFFu, incl, 31);
        base += ready;
        __syncwarp();  // the published prefixes are visible to lane 0's read-back below
      }
    }
    // ---- block 0's own tile of iteration k
    if (state == 0 && mbar_test_a(smem_addr(&mb_tile[k & kRingMask]), (uint32_t)((k / kTileRing) & 1))) {
      tile = s_tile[k & kRingMask];
      state = tile >= ntiles ? 3 : 1;
    }
    if (state == 1 && mbar_test_a(smem_addr(&mb_cnt[b]), (par >> b) & 1u)) {
      const int c0 = (lane < NSUB) ? s_cnt[b][lane] : 0;
      const int c1 = (NSUB > 32 && lane + 32 < NSUB) ? s_cnt[b][lane + 32] : 0;
      const int c = c0 | (c1 << 16);
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += y;
      }
      const int tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
      if (lane < NSUB) s_pre[b][lane] = (incl & 0xFFFF) - c0;
      if (NSUB > 32 && lane + 32 < NSUB) s_pre[b][lane + 32] = (tot & 0xFFFF) + (incl >> 16) - c1;
      total = (tot & 0xFFFF) + (tot >> 16);
      state = 2;
    }
    if (state == 2 && tile < base) {  // the scanner has published the tile's inclusive prefix
      if (lane == 0) {
        const unsigned long long st = ld_relaxed(status + tile);
        st_relaxed(status + tile, 0ull);  // consumed: leave the word clean for the next call
        s_prefix[b] = (int64_t)(st & kValueMask) - total;
        s_done[b] = 0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mb_pre[b]);
      par ^= 1u << b;
      b = (b + 1 == NBUF) ? 0 : b + 1;
      ++k;
      state = 0;
    }
  }
  if (lane == 0) *d_count = (int64_t)running;
}

// Workspace header: [0] tile-claim counter, [1] finished-block counter.  The last block of
// the grid to finish resets both, so (with the status words zeroed by the scan warps) the
// workspace is all zero after every launch.  Called by one warp per block, after every other
// warp of the block has stopped touching the workspace (the scan warp is the block's last
// user: compute warps do not exit before their final copy-out, which waits on the scan warp).
__device__ __forceinline__ void block_exit(unsigned long long* ws, int lane) {
  if (lane == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(ws + 1, 1ull);
    if (done == (unsigned long long)gridDim.x - 1) {
      ws[0] = 0ull;
      ws[1] = 0ull;
    }
  }
}

}  // namespace

#ifndef CLIPSEG_PITCH_PAD
#define CLIPSEG_PITCH_PAD 0  // extra staged rows per plane beyond SUB + 1 (0: the scratch row only)
#endif
constexpr size_t kMaxSmemPerBlock = 227 * 1024 - 2048;  // dynamic smem budget (static smem aside)

template <typename T, class Op, bool INDEX> struct CompactShape {
  static constexpr int V = Vec16<T>::N;                 // segments per 128-bit vector
  static constexpr int IT = compact_items<T>();          // vectors per lane per sub-tile
  static constexpr int SUB = 32 * V * IT;                // 128 segments per sub-tile
  static constexpr int NSUB = compact_subtiles<T, Op>();  // sub-tiles per block tile
  static constexpr int BT = NSUB * SUB;
  static constexpr int PITCH = SUB + 1 + CLIPSEG_PITCH_PAD;  // staged plane pitch: rows + scratch row
  static constexpr int SLOT = Op::OUT * PITCH;           // staged elements per sub-tile
  // per staged tile: the rows, plus the local indices when out_index is requested
  static constexpr size_t kBufBytes = (size_t)NSUB * SLOT * sizeof(T) + (INDEX ? (size_t)NSUB * (SUB + 1) : 0);
  static constexpr int NBUF = (size_t)compact_buffers<T, Op>() * kBufBytes <= kMaxSmemPerBlock
                                  ? compact_buffers<T, Op>()
                                  : (int)(kMaxSmemPerBlock / kBufBytes);  // staged tiles in flight
  static constexpr size_t kStageBytes = (size_t)NBUF * NSUB * SLOT * sizeof(T);
  static constexpr size_t kSmemBytes = (size_t)NBUF * kBufBytes;
  static constexpr int kMinBlocks = compact_min_blocks<T, Op>();
  static constexpr int kComputeWarps = compact_warps<T, Op>();
  static constexpr bool kPrefetch = compact_prefetch<T, Op>();
  static constexpr int kThreads = (kComputeWarps + 1) * 32;  // + the scan warp
};

template <typename T, class Op, bool FLAGS, bool INDEX>
__global__ void __launch_bounds__(CompactShape<T, Op, INDEX>::kThreads, CompactShape<T, Op, INDEX>::kMinBlocks)
    clip_compact_kernel(
    const T* __restrict__ in, int64_t ld_in, int64_t n, typename Op::Params w, T* __restrict__ out, int64_t ld_out,
    int64_t* __restrict__ out_index, int64_t index_base, uint8_t* __restrict__ flags, int64_t* __restrict__ d_count,
    unsigned long long* __restrict__ ws, int64_t ntiles) {
  typedef CompactShape<T, Op, INDEX> S;
  constexpr int IN = Op::IN, OUT = Op::OUT;
  constexpr int V = S::V, IT = S::IT, SUB = S::SUB, NSUB = S::NSUB, BT = S::BT, SLOT = S::SLOT, NBUF = S::NBUF;
  constexpr int PITCH = S::PITCH;
  constexpr int kComputeWarps = S::kComputeWarps;
  constexpr int PER_WARP = NSUB / kComputeWarps;
  static_assert(NSUB % kComputeWarps == 0 && NSUB <= 64 && NBUF >= 2 && NBUF <= kTileRing - 2, "tile layout");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);            // [NBUF][NSUB][2D][SUB]
  uint8_t* lidx = smem_raw + S::kStageBytes;            // [NBUF][NSUB][SUB + 1]
  __shared__ int s_cnt[NBUF][NSUB], s_pre[NBUF][NSUB];
  __shared__ int64_t s_prefix[NBUF];
  __shared__ int s_done[NBUF];                           // compute warps finished with buffer b
  __shared__ int64_t s_tile[kTileRing];                  // tile of iteration k in slot k % ring
  __shared__ int s_claim[kTileRing];                     // compute warps that reached the slot
  __shared__ __align__(8) uint64_t mb_cnt[NBUF];         // compute warps -> scan warp
  __shared__ __align__(8) uint64_t mb_pre[NBUF];         // scan warp -> compute warps
  __shared__ __align__(8) uint64_t mb_tile[kTileRing];   // claiming warp -> all

  unsigned long long* counter = ws;
  unsigned long long* status = ws + kWsHeaderBytes / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int q = 0; q < NBUF; ++q) {
      s_done[q] = 0;
      mbar_init(&mb_cnt[q], kComputeWarps);
      mbar_init(&mb_pre[q], 1);
    }
    for (int q = 0; q < kTileRing; ++q) {
      s_claim[q] = 0;
      mbar_init(&mb_tile[q], 1);
    }
    if (blockIdx.x != 0) {
      s_tile[0] = (int64_t)atomicAdd(counter, 1ull);
      mbar_arrive(&mb_tile[0]);
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {  // block 0 only scans; it processes no tiles
    if (warp == kComputeWarps) {
      global_scanner(status, ntiles, lane, d_count);
      block_exit(ws, lane);
    }
    return;
  }

  if (warp == kComputeWarps) {
    tile_scan_warp<NSUB, NBUF>(lane, ntiles, status, s_tile, s_cnt, s_pre, s_prefix, s_done, mb_tile, mb_cnt, mb_pre);
    block_exit(ws, lane);
    return;
  }

  // -------------------------------------------------------------------- compute warps
  // Copies lag NBUF-1 tiles behind the compute: pend[q] is the tile of iteration k-1-q.
  int64_t pend[NBUF - 1];
  int pbuf[NBUF - 1];
  unsigned ppar[NBUF - 1];
#pragma unroll
  for (int q = 0; q < NBUF - 1; ++q) {
    pend[q] = ntiles;
    pbuf[q] = 0;
    ppar[q] = 0;
  }
  int b = 0;
  unsigned par = 0;
  // segments of sub-tile `sub` of tile t still in range (SUB for every full sub-tile)
  auto remaining = [&](int64_t t, int sub) -> int {
    const int64_t r = n - (t * BT + (int64_t)sub * SUB);
    return r >= SUB ? SUB : (r > 0 ? (int)r : 0);
  };
  auto load = [&](int64_t t, int sub, T (&dst)[IT][IN][V], const bool FULL) {
    const T* src = in + t * BT + (int64_t)sub * SUB;
    const int rem = FULL ? SUB : remaining(t, sub);
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int o = (32 * j + lane) * V;
      if (FULL || o < rem) {
#pragma unroll
        for (int c = 0; c < IN; ++c) load_vec<T, IN == 4>(src + c * ld_in + o, dst[j][c]);
      } else {
#pragma unroll
        for (int c = 0; c < IN; ++c)
#pragma unroll
          for (int v = 0; v < V; ++v) dst[j][c][v] = T(0);
      }
    }
  };
  // Sub-tile loads run one ahead of the clipping, across tile boundaries: the next tile is
  // claimed as this one starts, and its first sub-tile is loaded during this one's last.
  // PREFETCH: the next sub-tile's loads are in flight (in a second register buffer) while
  // this one is clipped; without it (wide homogeneous rows) the registers go to more warps.
  constexpr bool PREFETCH = S::kPrefetch;
  T buf[PREFETCH ? 2 : 1][IT][IN][V];
  mbar_wait(&mb_tile[0], 0u);
  int64_t tile = s_tile[0];
  if (PREFETCH && tile < ntiles) load(tile, warp, buf[0], false);
  for (int64_t k = 0;; ++k) {
    int64_t next = ntiles;
    if (tile < ntiles && lane == 0) {
      // the first compute warp to start tile k claims the tile of iteration k + 1
      const int q = (int)((k + 1) & kRingMask);
      const int order = atomicAdd(&s_claim[q], 1);
      if (order == 0) {
        s_tile[q] = (int64_t)atomicAdd(counter, 1ull);
        CLIP_TRACE(s_tile[q], 0, trace_now());
        mbar_arrive(&mb_tile[q]);
      } else if (order == kComputeWarps - 1) {
        s_claim[q] = 0;  // every warp has passed this slot; reused kTileRing iterations later
      }
    }
    if (tile < ntiles) {
      if (warp == 0 && lane == 0) CLIP_TRACE(tile, 1, trace_now());
      T* stg = stage + (size_t)b * NSUB * SLOT;
      uint8_t* lix = lidx + (size_t)b * NSUB * (SUB + 1);
      auto body = [&](const bool FULL) {
#pragma unroll
        for (int r = 0; r < PER_WARP; ++r) {
          const int sub = r * kComputeWarps + warp;
          // With an even PER_WARP, buf[r & 1] holds this sub-tile and the next one loads into
          // the other (static indices keep both in registers); with an odd one the current
          // sub-tile is copied out of buf[0] first.
          constexpr bool PING = (PER_WARP % 2) == 0;
          T held[IT][IN][V];
          if constexpr (!PREFETCH) {
            load(tile, sub, buf[0], FULL);
            if (r + 1 == PER_WARP) {
              mbar_wait(&mb_tile[(k + 1) & kRingMask], (uint32_t)(((k + 1) / kTileRing) & 1));
              next = s_tile[(k + 1) & kRingMask];
            }
          } else {
            const int cur = PING ? (r & 1) : 0;
            if (!PING) {
#pragma unroll
              for (int j = 0; j < IT; ++j)
#pragma unroll
                for (int c = 0; c < IN; ++c)
#pragma unroll
                  for (int v = 0; v < V; ++v) held[j][c][v] = buf[0][j][c][v];
            }
            T (&dst)[IT][IN][V] = PING ? buf[cur ^ 1] : buf[0];
            if (r + 1 < PER_WARP) {
              load(tile, sub + kComputeWarps, dst, FULL);
            } else {
              mbar_wait(&mb_tile[(k + 1) & kRingMask], (uint32_t)(((k + 1) / kTileRing) & 1));
              next = s_tile[(k + 1) & kRingMask];
              if (next < ntiles) load(next, warp, dst, false);
            }
          }
          const T (&plane)[IT][IN][V] = (PREFETCH && !PING) ? held : buf[PREFETCH ? (r & 1) : 0];
          const int rem = FULL ? SUB : remaining(tile, sub);
          uint8_t* fl = FLAGS ? flags + tile * BT + (int64_t)sub * SUB : nullptr;
          T res[IT][OUT][V];
          unsigned vis[IT];
#pragma unroll
          for (int j = 0; j < IT; ++j) {
            const int o = (32 * j + lane) * V;
            vis[j] = group_chunked<Op, false>(plane[j], w, res[j]);
            if (!FULL) vis[j] &= (o >= rem) ? 0u : (o + V <= rem ? (1u << V) - 1u : (1u << (rem - o)) - 1u);
            if (FLAGS) {
#if CLIPSEG_MUL_FLAGS
              // bit v of vis -> byte v with one multiply (the shifted copies never collide)
              const uint32_t packed = V == 4 ? (vis[j] * 0x204081u) & 0x01010101u : (vis[j] * 0x81u) & 0x0101u;
#else
              uint32_t packed = 0;
#pragma unroll
              for (int v = 0; v < V; ++v) packed |= ((vis[j] >> v) & 1u) << (8 * v);
#endif
              if (FULL || o + V <= rem) {
                if (V == 4) *reinterpret_cast<uint32_t*>(fl + o) = packed;
                else *reinterpret_cast<uint16_t*>(fl + o) = (uint16_t)packed;
              } else {
                for (int v = 0; v < V; ++v)
                  if (o + v < rem) fl[o + v] = (uint8_t)((vis[j] >> v) & 1u);
              }
            }
          }
          // warp scan of the visible counts (item j in bit field 8 j)
          unsigned cnt = 0;
#pragma unroll
          for (int j = 0; j < IT; ++j) cnt |= (unsigned)__popc(vis[j]) << (8 * j);
          unsigned incl = cnt;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += y;
          }
          const unsigned tot_f = __shfl_sync(0xFFFFFFFFu, incl, 31);
          const unsigned excl_f = incl - cnt;
          // stage the visible rows, compacted, at the front of this sub-tile's slot; an
          // invisible row goes to the slot's scratch row SUB, so the stores need no branch
          T* st = stg + sub * SLOT;
          int before = 0;
#pragma unroll
          for (int j = 0; j < IT; ++j) {
            int pos = before + (int)((excl_f >> (8 * j)) & 0xFFu);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const bool on = (vis[j] >> v) & 1u;
#if CLIPSEG_IMAD_SELECT
              // on ? pos : SUB as SUB + on * (pos - SUB): a multiply-add on the FMA pipe instead
              // of a select on the busier ALU pipe (measured -0.3 %)
              int at;
              asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(at) : "r"((int)on), "r"(pos - SUB), "r"(SUB));
              T* row = st + at;
#else
              T* row = st + (on ? pos : SUB);
#endif
#pragma unroll
              for (int c = 0; c < OUT; ++c) row[c * PITCH] = res[j][c][v];
              if (INDEX) lix[sub * (SUB + 1) + (on ? pos : SUB)] = (uint8_t)((32 * j + lane) * V + v);
              pos += on;
            }
            before += (int)((tot_f >> (8 * j)) & 0xFFu);
          }
          if (lane == 0) s_cnt[b][sub] = before;
        }
      };
      // (a second copy specialised for full tiles saves ~10% of the instructions but doubles
      // the hot loop's code, and the instruction-cache misses cost more: measured 7.5 vs 9.2 ms)
      body(false);
      // the last compute warp to finish publishes the tile aggregate (flag A) at once
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&s_done[b], 1) == kComputeWarps - 1;
      }
      last = __shfl_sync(0xFFFFFFFFu, last, 0);
      if (last) {
        __threadfence_block();
        int c = (lane < NSUB) ? ((volatile int*)s_cnt[b])[lane] : 0;
        if (NSUB > 32 && lane + 32 < NSUB) c += ((volatile int*)s_cnt[b])[lane + 32];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, d);
        if (lane == 0) {
          st_relaxed(status + tile, kFlagA | (unsigned long long)c);
          CLIP_TRACE(tile, 2, trace_now());
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mb_cnt[b]);  // counts of tile k published to the scan warp
    }
    // copy the rows of the oldest pending tile (iteration k - (NBUF-1)), then shift
    constexpr int Q = NBUF - 2;
    if (pend[Q] < ntiles) {
      const int pb = pbuf[Q];
      if (CLIPSEG_PRE_SLEEP_NS > 0) mbar_wait_sleepy(&mb_pre[pb], ppar[Q], CLIPSEG_PRE_SLEEP_NS);
      else mbar_wait(&mb_pre[pb], ppar[Q]);  // its offsets are published
      if (warp == 0 && lane == 0) CLIP_TRACE(pend[Q], 6, trace_now());
      const int64_t prefix = s_prefix[pb];
      const T* stg = stage + (size_t)pb * NSUB * SLOT;
      const uint8_t* lix = lidx + (size_t)pb * NSUB * (SUB + 1);
#pragma unroll
      for (int r = 0; r < PER_WARP; ++r) {
        const int sub = r * kComputeWarps + warp;  // the sub-tiles this warp staged
        const int cnt = s_cnt[pb][sub];
        const int64_t g0 = prefix + s_pre[pb][sub];
        const T* st = stg + sub * SLOT;
#pragma unroll
        for (int c = 0; c < OUT; ++c) {
          T* dst = out + c * ld_out + g0 + lane;
          const T* src = st + c * PITCH + lane;
#pragma unroll
          for (int q = 0; q < SUB / 32; ++q)
            if (q * 32 + lane < cnt) {
#if CLIPSEG_STORE_HINT == 1
              dst[q * 32] = src[q * 32];
#else
              __stcs(dst + q * 32, src[q * 32]);
#endif
            }
        }
        if (INDEX) {
          const int64_t ib = index_base + pend[Q] * BT + (int64_t)sub * SUB;
#pragma unroll
          for (int q = 0; q < SUB / 32; ++q) {
            const int e = q * 32 + lane;
            if (e < cnt) out_index[g0 + e] = ib + lix[sub * (SUB + 1) + e];
          }
        }
      }
    }
#pragma unroll
    for (int q = Q; q > 0; --q) {
      pend[q] = pend[q - 1];
      pbuf[q] = pbuf[q - 1];
      ppar[q] = ppar[q - 1];
    }
    pend[0] = tile;
    pbuf[0] = b;
    ppar[0] = (par >> b) & 1u;
    if (tile < ntiles) par ^= 1u << b;
    b = (b + 1 == NBUF) ? 0 : b + 1;
    tile = next;
    if (tile >= ntiles) {
      bool any = false;
#pragma unroll
      for (int q = 0; q <= Q; ++q) any |= pend[q] < ntiles;
      if (!any) break;
    }
  }
}

// ======================================================================================
// Packed variant (the headline 2D fp32 instantiation).  Same grid organisation as above
// (block 0 = global scanner; per block: compute warps + scan warp, dynamic tile claims,
// NBUF staged tiles, copy-out NBUF-1 tiles after the compute), but a compute warp owns a
// contiguous BATCH = PW x 128 segments of each tile and works on it in two phases:
//
//  1. R3 only (Op::keep) on its PW register-held sub-tiles; the kept segments are written,
//     in segment order, as rows of an array-of-structures list at the front of the warp's
//     staging region (plus their local indices), so the segments R3 rejects — about 40 % of
//     the headline workload — are never clipped.  The next tile's batch is then loaded
//     into the same registers, in flight during phase 2;
//  2. the kept rows are clipped 32 at a time, one per lane (Op::clip_one); ballot + popc
//     rank the visible ones and each is written back, as a row, at its rank in the same
//     region (rank <= list position, so the rows still to be read are never overwritten).
//
// The region then holds the batch's visible rows contiguously; NBUF-1 tiles later the warp
// copies them to their global rows (one shared-memory row load + 2·D coalesced stores per
// row, only ceil(count/32) rounds).  Flags go through a per-warp byte array (zeroed in
// phase 1, the visible ones set in phase 2, stored as words).
template <typename T, class Op, bool INDEX> struct PackedShape {
  static constexpr PackedKnobs K = packed_knobs<T, Op>();
  static constexpr int IN = Op::IN, OUT = Op::OUT;
  static constexpr int V = Vec16<T>::N;  // segments per 128-bit vector
  static constexpr int SUB = 32 * V;     // segments per sub-tile (one vector per plane per lane)
  static constexpr int PW = K.pw;        // sub-tiles per warp batch
  static constexpr int BATCH = PW * SUB; // segments per warp batch (local indices are bytes)
  static constexpr int W = K.warps;      // compute warps
  static constexpr int BT = W * BATCH;   // segments per block tile
  static constexpr size_t ROWB = (size_t)IN * sizeof(T);
  static constexpr size_t kRegion = (size_t)BATCH * IN;               // elements per warp region
  // staged tiles (the copy-out lags NBUF-1 tiles): the knob, or fewer when they do not fit
  static constexpr size_t kPerBuf = (size_t)W * (kRegion * sizeof(T) + (INDEX ? BATCH : 0));
  static constexpr size_t kFixed =
      (size_t)W * (BATCH / 32 + 1) * 4 + ((size_t)4 << (2 * V)) + (size_t)W * BATCH + (INDEX ? (size_t)W * BATCH : 0);
  static constexpr int NBUF = (size_t)K.nbuf * kPerBuf + kFixed <= kMaxSmemPerBlock
                                  ? K.nbuf
                                  : (int)((kMaxSmemPerBlock - kFixed) / kPerBuf);
  static constexpr size_t kStageBytes = (size_t)NBUF * W * kRegion * sizeof(T);
  // per warp: the visible bits of the batch's list, one word per 32 positions (+1 spare word)
  static constexpr int VBW = BATCH / 32 + 1;
  static constexpr size_t kVbOff = kStageBytes;                       // [W][VBW] u32
  static constexpr size_t kLutOff = kVbOff + (size_t)W * VBW * 4;     // [2^(2V)] u32: flags of (keep, bits)
  static constexpr size_t kExcOff = kLutOff + ((size_t)4 << (2 * V)); // [W][BATCH] u8 deferred list positions
  static constexpr size_t kIdxOff = kExcOff + (size_t)W * BATCH;      // [W][BATCH] list -> local index (INDEX)
  static constexpr size_t kLixOff = kIdxOff + (INDEX ? (size_t)W * BATCH : 0);  // [NBUF][W][BATCH] staged indices
  static constexpr size_t kSmemBytes = kLixOff + (INDEX ? (size_t)NBUF * W * BATCH : 0);
  // copy warps: a service warpgroup (the scan warp + COPYW copy warps) copies the staged
  // batches out, so compute warps neither copy nor wait for offsets (CLIPSEG_PK_COPYW)
  static constexpr int COPYW = compact_headline<T, Op>() ? CLIPSEG_PK_COPYW : 0;
  static constexpr int kThreads = (W + 1 + COPYW) * 32;
  static_assert(COPYW == 0 || ((W % 4) == 0 && ((1 + COPYW) % 4) == 0), "whole warpgroups for setmaxnreg");
  // the launch allocates the block kLaunchRegs per thread (per-SMSP share, 8-register granules);
  // setmaxnreg only moves registers inside that pool, so the split must fit it
  static constexpr int kLaunchRegs = ((16384 / ((((kThreads / 32) + 3) / 4) * 32)) / 8) * 8;
  static_assert(COPYW == 0 || W * 32 * CLIPSEG_PK_REG_C + (1 + COPYW) * 32 * CLIPSEG_PK_REG_S <= kThreads * kLaunchRegs,
                "register split exceeds the block's pool (setmaxnreg.inc would never return)");
  static_assert(BATCH <= 256, "local indices are bytes");
  static_assert(OUT <= IN, "rows are written back in place");
  static_assert(kSmemBytes <= kMaxSmemPerBlock, "shared memory");
  static_assert(BT >= kMinCompactTile, "workspace sizing");
};

// Shared memory by 32-bit shared-window address (computed once per kernel, so the hot loops
// carry no generic-to-shared conversions).  Rows of N elements: 128-bit accesses for rows of
// a multiple of 16 B (fp32 rows of 4 or 8, fp64 rows), 64-bit ones for fp32 rows of 6.
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
template <typename T, int N>
__device__ __forceinline__ void sts_row(uint32_t a, const T (&v)[N]);
template <typename T, int N>
__device__ __forceinline__ void lds_row(uint32_t a, T (&v)[N]);
template <int N>
__device__ __forceinline__ void sts_row(uint32_t a, const int32_t (&v)[N]) {  // int32 rows as their bit patterns
  float f[N];
#pragma unroll
  for (int i = 0; i < N; ++i) f[i] = __int_as_float(v[i]);
  sts_row<float, N>(a, f);
}
template <int N>
__device__ __forceinline__ void lds_row(uint32_t a, int32_t (&v)[N]) {
  float f[N];
  lds_row<float, N>(a, f);
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __float_as_int(f[i]);
}
template <typename T, int N>
__device__ __forceinline__ void sts_row(uint32_t a, const T (&v)[N]) {
  if constexpr (std::is_same<T, int32_t>::value) {
    sts_row<N>(a, v);
  } else if constexpr (sizeof(T) == 4 && N % 4 == 0) {  // 16-byte rows: 128-bit stores
#pragma unroll
    for (int i = 0; i < N; i += 4)
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a + 4 * i), "f"(v[i]), "f"(v[i + 1]),
                   "f"(v[i + 2]), "f"(v[i + 3])
                   : "memory");
  } else if constexpr (sizeof(T) == 4) {  // rows of 6 floats are only 8-byte aligned
    static_assert(N % 2 == 0, "row layout");
#pragma unroll
    for (int i = 0; i < N; i += 2)
      asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a + 4 * i), "f"(v[i]), "f"(v[i + 1]) : "memory");
  } else {
    static_assert(N % 2 == 0, "row layout");
#pragma unroll
    for (int i = 0; i < N; i += 2)
      asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a + 8 * i), "d"(v[i]), "d"(v[i + 1]) : "memory");
  }
}
template <typename T, int N>
__device__ __forceinline__ void lds_row(uint32_t a, T (&v)[N]) {
  if constexpr (std::is_same<T, int32_t>::value) {
    lds_row<N>(a, v);
  } else if constexpr (sizeof(T) == 4 && N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v[i]), "=f"(v[i + 1]), "=f"(v[i + 2]), "=f"(v[i + 3])
                   : "r"(a + 4 * i)
                   : "memory");
  } else if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < N; i += 2)
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v[i]), "=f"(v[i + 1]) : "r"(a + 4 * i) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 2)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[i]), "=d"(v[i + 1]) : "r"(a + 8 * i) : "memory");
  }
}

// Staged rows of the packed kernel.  Rows of a multiple of 16 bytes are stored in 16-byte
// slices: slice s of list row p sits at region + BATCH*16*s + 16*p, so a warp's accesses to
// 32 consecutive rows are contiguous in every slice — 32-byte rows at their own stride put
// twice the minimal wavefronts through the shared-memory banks (measured: homogeneous fp32
// 1.186 -> 1.155 ms, fp64 2D 0.896 -> 0.881 ms at 1e8 / 5e7).  Rows of 16 bytes (2D fp32,
// int32) are one slice, the plain array of rows; 24-byte rows (3D fp32) stay a plain array
// (sliced as 16 + 8 bytes they measured 0.873 -> 0.877 ms).  The layout is fixed by the list
// row's element count NIN; result rows (N <= NIN) use its slices.
template <typename T, int NIN, int BATCH> struct RowSlices {
  static constexpr int E = 16 / (int)sizeof(T);                // elements per slice
  static constexpr int RB = NIN * (int)sizeof(T);              // row bytes
  static constexpr bool PLAIN = RB % 16 != 0;                  // one slice: the array of rows
  static constexpr int NS = PLAIN ? 1 : RB / 16;               // slices
  static __host__ __device__ constexpr uint32_t stride(int) { return PLAIN ? (uint32_t)RB : 16u; }
  static __host__ __device__ constexpr uint32_t off(int s) { return (uint32_t)BATCH * 16u * (uint32_t)s; }
};
template <typename T, int NIN, int BATCH, int N>
__device__ __forceinline__ void sts_rowp(uint32_t region, int p, const T (&v)[N]) {
  if constexpr (std::is_same<T, int32_t>::value) {
    float f[N];
#pragma unroll
    for (int i = 0; i < N; ++i) f[i] = __int_as_float(v[i]);
    sts_rowp<float, NIN, BATCH, N>(region, p, f);
  } else if constexpr (RowSlices<T, NIN, BATCH>::PLAIN) {
    sts_row<T, N>(region + (uint32_t)p * RowSlices<T, NIN, BATCH>::stride(0), v);
  } else {
    typedef RowSlices<T, NIN, BATCH> L;
#pragma unroll
    for (int sl = 0; sl < L::NS; ++sl) {
      constexpr int E = L::E;
      const int i0 = sl * E;
      if (i0 < N) {
        const uint32_t a = region + L::off(sl) + (uint32_t)p * L::stride(sl);
        const int cnt = (N - i0 < E) ? N - i0 : E;
        if (cnt * (int)sizeof(T) == 16) {
          T x[E];
#pragma unroll
          for (int i = 0; i < E; ++i) x[i] = v[i0 + i < N ? i0 + i : i0];
          sts_row<T, E>(a, x);
        } else if constexpr (sizeof(T) == 4) {
          if (cnt == 2) {
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v[i0]), "f"(v[i0 + 1 < N ? i0 + 1 : i0]) : "memory");
          } else {
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v[i0]) : "memory");
          }
        } else {
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v[i0]) : "memory");
        }
      }
    }
  }
}
template <typename T, int NIN, int BATCH, int N>
__device__ __forceinline__ void lds_rowp(uint32_t region, int p, T (&v)[N]) {
  if constexpr (std::is_same<T, int32_t>::value) {
    float f[N];
    lds_rowp<float, NIN, BATCH, N>(region, p, f);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = __float_as_int(f[i]);
  } else if constexpr (RowSlices<T, NIN, BATCH>::PLAIN) {
    lds_row<T, N>(region + (uint32_t)p * RowSlices<T, NIN, BATCH>::stride(0), v);
  } else {
    typedef RowSlices<T, NIN, BATCH> L;
#pragma unroll
    for (int sl = 0; sl < L::NS; ++sl) {
      constexpr int E = L::E;
      const int i0 = sl * E;
      if (i0 < N) {
        const uint32_t a = region + L::off(sl) + (uint32_t)p * L::stride(sl);
        const int cnt = (N - i0 < E) ? N - i0 : E;
        if (cnt * (int)sizeof(T) == 16) {
          T x[E];
          lds_row<T, E>(a, x);
#pragma unroll
          for (int i = 0; i < E; ++i)
            if (i0 + i < N) v[i0 + i] = x[i];
        } else if constexpr (sizeof(T) == 4) {
          if (cnt == 2) {
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v[i0]), "=f"(v[i0 + 1 < N ? i0 + 1 : i0]) : "r"(a) : "memory");
          } else {
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[i0]) : "r"(a) : "memory");
          }
        } else {
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[i0]) : "r"(a) : "memory");
        }
      }
    }
  }
}

#ifndef CLIPSEG_PK_MAXNREG
#define CLIPSEG_PK_MAXNREG 0  // > 0: register cap instead of the launch bounds (A/B builds)
#endif
#if CLIPSEG_PK_MAXNREG > 0
#define CLIPSEG_PK_BOUNDS(...) __maxnreg__(CLIPSEG_PK_MAXNREG)
#else
#define CLIPSEG_PK_BOUNDS(...) __launch_bounds__(__VA_ARGS__, 1)
#endif
template <typename T, class Op, bool FLAGS, bool INDEX>
__global__ void CLIPSEG_PK_BOUNDS(PackedShape<T, Op, INDEX>::kThreads) clip_compact_packed_kernel(
    const T* __restrict__ in, int64_t ld_in, int64_t n, typename Op::Params w, T* __restrict__ out, int64_t ld_out,
    int64_t* __restrict__ out_index, int64_t index_base, uint8_t* __restrict__ flags, int64_t* __restrict__ d_count,
    unsigned long long* __restrict__ ws, int64_t ntiles) {
  typedef PackedShape<T, Op, INDEX> S;
  constexpr int IN = S::IN, OUT = S::OUT, V = S::V, SUB = S::SUB, PW = S::PW, BATCH = S::BATCH, W = S::W;
  constexpr int BT = S::BT, NBUF = S::NBUF;
  static_assert(NBUF >= 2 && NBUF <= kTileRing - 3, "tile ring");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cnt[NBUF][W], s_pre[NBUF][W];
  __shared__ int64_t s_prefix[NBUF];
  __shared__ int s_done[NBUF];
  __shared__ int64_t s_tile[kTileRing];
  __shared__ __align__(8) uint64_t mb_cnt[NBUF];
  __shared__ __align__(8) uint64_t mb_pre[NBUF];
  __shared__ __align__(8) uint64_t mb_tile[kTileRing];
  __shared__ __align__(8) uint64_t mb_free[NBUF];  // copy warps -> compute warps: buffer copied out
  constexpr int CW = S::COPYW;

  unsigned long long* counter = ws;
  unsigned long long* status = ws + kWsHeaderBytes / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  {  // flags of V segments from their kept mask (high V bits) and the kept ones' visible bits
    uint32_t* lut = reinterpret_cast<uint32_t*>(smem_raw + S::kLutOff);
    for (int e = threadIdx.x; e < (1 << (2 * V)); e += blockDim.x) {
      uint32_t kmask = (uint32_t)e >> V, bits = (uint32_t)e, f = 0;
      for (int v = 0; v < V; ++v)
        if ((kmask >> v) & 1u) {
          f |= (bits & 1u) << (8 * v);
          bits >>= 1;
        }
      lut[e] = f;
    }
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < NBUF; ++q) {
      s_done[q] = 0;
      mbar_init(&mb_cnt[q], W);
      mbar_init(&mb_pre[q], 1);
    }
    for (int q = 0; q < kTileRing; ++q) mbar_init(&mb_tile[q], 1);
    if (CW)
      for (int q = 0; q < NBUF; ++q) mbar_init(&mb_free[q], CW);
    if (S::K.b0tiles || blockIdx.x != 0) {  // the tiles of iterations 0 and 1
      s_tile[0] = (int64_t)atom_add_global(counter, 1ull);
      s_tile[1] = (int64_t)atom_add_global(counter, 1ull);
      mbar_arrive(&mb_tile[0]);
      mbar_arrive(&mb_tile[1]);
    }
  }
  __syncthreads();
  if (!S::K.b0tiles && blockIdx.x == 0) {
    if (warp == W) {
      global_scanner(status, ntiles, lane, d_count);
      block_exit(ws, lane);
    }
    return;
  }
  if (warp >= W) {  // ------------------------------------- service warpgroup: scan warp (+ copy warps)
    // warpgroup register split: the service warps give registers to the compute warps
    if constexpr (CW > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CLIPSEG_PK_REG_S));
    if (warp == W) {
      if (S::K.b0tiles && blockIdx.x == 0)
        scanner_with_tiles<W, NBUF>(lane, ntiles, status, d_count, s_tile, s_cnt, s_pre, s_prefix, s_done, mb_tile,
                                    mb_cnt, mb_pre);
      else
        tile_scan_warp<W, NBUF>(lane, ntiles, status, s_tile, s_cnt, s_pre, s_prefix, s_done, mb_tile, mb_cnt,
                                mb_pre);
      block_exit(ws, lane);
      return;
    }
    if constexpr (CW > 0) {  // ---------------------------------------------------- copy warps
      const int cw = warp - W - 1;
      const uint32_t sb = smem_addr(smem_raw);
      int bb = 0;
      unsigned ppar = 0;
      for (int64_t kk = 0;; ++kk) {
        mbar_wait_sleepy(&mb_tile[kk & kRingMask], (uint32_t)((kk / kTileRing) & 1), 128);
        const int64_t tk = s_tile[kk & kRingMask];
        if (tk >= ntiles) break;
        mbar_wait_a(smem_addr(&mb_pre[bb]), (ppar >> bb) & 1u);  // the tile's offsets
        ppar ^= 1u << bb;
        const int64_t prefix = s_prefix[bb];
        for (int w2 = cw; w2 < W; w2 += CW) {
          const int cnt = s_cnt[bb][w2];
          const int64_t g0 = prefix + s_pre[bb][w2];
          const uint32_t reg = sb + (uint32_t)(((size_t)bb * W + w2) * S::kRegion * sizeof(T));
          T* dst[OUT];
#pragma unroll
          for (int c = 0; c < OUT; ++c) dst[c] = out + c * ld_out + g0 + lane;
          const uint32_t slix = sb + (uint32_t)(S::kLixOff + ((size_t)bb * W + w2) * BATCH) + lane;
          const int64_t ib = INDEX ? index_base + tk * BT + (int64_t)w2 * BATCH : 0;
#pragma unroll
          for (int q = 0; q < BATCH / 32; ++q) {
            if (q * 32 >= cnt) break;
            if (q * 32 + lane < cnt) {
              T row[OUT];
              lds_rowp<T, IN, BATCH>(reg, q * 32 + lane, row);
#pragma unroll
              for (int c = 0; c < OUT; ++c) __stcs(dst[c] + q * 32, row[c]);
              if (INDEX) out_index[g0 + q * 32 + lane] = ib + lds_u8(slix + q * 32);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&mb_free[bb]);  // this buffer may be refilled
        bb = (bb + 1 == NBUF) ? 0 : bb + 1;
      }
    }
    return;
  }
  if constexpr (CW > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CLIPSEG_PK_REG_C));

  // ------------------------------------------------------------------ compute warps
  const typename Op::KeepParams kparams = Op::keep_params(w);
  const uint32_t sbase = smem_addr(smem_raw);
  const uint32_t lidx_a = sbase + (uint32_t)S::kIdxOff + warp * BATCH;    // list position -> local index (INDEX)
  const uint32_t vb_a = sbase + (uint32_t)S::kVbOff + warp * S::VBW * 4;  // visible bits of the list
  const uint32_t lut_a = sbase + (uint32_t)S::kLutOff;
  const uint32_t exc_a = sbase + (uint32_t)S::kExcOff + warp * BATCH;  // deferred (exceptional) list positions
  const uint32_t mbt_a = smem_addr(mb_tile), mbc_a = smem_addr(mb_cnt), mbp_a = smem_addr(mb_pre);
  const uint32_t mbf_a = smem_addr(mb_free);
  unsigned fpar = 0;  // bit q: parity of the next phase of mb_free[q] (copy-warp mode)
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t full_tiles = n / BT;  // tiles whose every batch is full
  const T* lane_in = in + (int64_t)warp * BATCH + lane * V;
  auto region_of = [&](int buf) -> uint32_t {
    return sbase + (uint32_t)(((size_t)buf * W + warp) * S::kRegion * sizeof(T));
  };
  // segments of this warp's batch of tile t before the end of the input (BATCH when full)
  auto batch_rem = [&](int64_t t) -> int {
    if (t < full_tiles) return BATCH;
    const int64_t r = n - (t * BT + (int64_t)warp * BATCH);
    return r >= BATCH ? BATCH : (r > 0 ? (int)r : 0);
  };
  T cur[PW][IN][V];
#ifndef CLIPSEG_PK_PLANEPTR
#define CLIPSEG_PK_PLANEPTR 0  // 1: per-plane base pointers held across the loop (fewer 64-bit address ops per load)
#endif
  const T* plane_in[CLIPSEG_PK_PLANEPTR ? IN : 1];
#pragma unroll
  for (int c = 0; c < (CLIPSEG_PK_PLANEPTR ? IN : 1); ++c) plane_in[c] = lane_in + c * ld_in;
  auto load = [&](int64_t t) {
    const T* src = lane_in + t * BT;
    const int rem = batch_rem(t);
    if (CLIPSEG_PK_PLANEPTR && rem == BATCH) {
      const int64_t off = t * BT;
#pragma unroll
      for (int c = 0; c < IN; ++c) {
        const T* sc = plane_in[CLIPSEG_PK_PLANEPTR ? c : 0] + off;
#pragma unroll
        for (int j = 0; j < PW; ++j) load_vec<T, IN == 4>(sc + j * SUB, cur[j][c]);
      }
    } else if (rem == BATCH) {  // warp-uniform: full batch, unpredicated loads
#pragma unroll
      for (int c = 0; c < IN; ++c) {
        const T* sc = src + c * ld_in;
#pragma unroll
        for (int j = 0; j < PW; ++j) load_vec<T, IN == 4>(sc + j * SUB, cur[j][c]);
      }
    } else {  // ragged tail: vectors past the end are not loaded (their segments are masked off)
#pragma unroll
      for (int j = 0; j < PW; ++j)
        if (j * SUB + lane * V < rem) {
#pragma unroll
          for (int c = 0; c < IN; ++c) load_vec<T, IN == 4>(src + c * ld_in + j * SUB, cur[j][c]);
        }
    }
  };
  // copy the visible rows of iteration kk (tile tk, buffer cb) to their global rows
  unsigned cpar = 0;  // bit q: parity of the next phase of mb_pre[q] this warp waits for
  auto copy_out = [&](int64_t tk, int cb) {
    mbar_wait_a(mbp_a + 8 * cb, (cpar >> cb) & 1u);
    cpar ^= 1u << cb;
    if (warp == 0 && lane == 0) CLIP_TRACE(tk, 6, trace_now());
    const int cnt = s_cnt[cb][warp];
    const int64_t g0 = s_prefix[cb] + s_pre[cb][warp];
    const uint32_t creg0 = region_of(cb);
    T* dst[OUT];  // per-plane row pointers, computed once per batch
#pragma unroll
    for (int c = 0; c < OUT; ++c) dst[c] = out + c * ld_out + g0 + lane;
    const uint32_t slix = sbase + (uint32_t)(S::kLixOff + ((size_t)cb * W + warp) * BATCH) + lane;
    const int64_t ib = INDEX ? index_base + tk * BT + (int64_t)warp * BATCH : 0;
#ifndef CLIPSEG_PK_COPY_CHUNK
#define CLIPSEG_PK_COPY_CHUNK 1  // copy-out rounds whose shared loads are issued before their stores
#endif
    constexpr int CH = CLIPSEG_PK_COPY_CHUNK;
#pragma unroll
    for (int q0 = 0; q0 < BATCH / 32; q0 += CH) {
      if (q0 * 32 >= cnt) break;
      T rows[CH][OUT];
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if ((q0 + u) * 32 + lane < cnt) lds_rowp<T, IN, BATCH>(creg0, (q0 + u) * 32 + lane, rows[u]);
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int q = q0 + u;
        if (q * 32 + lane < cnt) {
#pragma unroll
          for (int c = 0; c < OUT; ++c) {
#if CLIPSEG_STORE_HINT == 1
            dst[c][q * 32] = rows[u][c];
#else
            __stcs(dst[c] + q * 32, rows[u][c]);
#endif
          }
          if (INDEX) out_index[g0 + q * 32 + lane] = ib + lds_u8(slix + q * 32);
        }
      }
    }
  };
  // Claims: warp 0's lane 0 issues the fetch-and-add for iteration k + 3 during iteration k
  // and publishes its result (s_tile, mb_tile) at the start of iteration k + 1, so the atomic's
  // round trip overlaps a whole iteration of work instead of stalling the claiming warp.
  const bool claimer = warp == 0 && lane == 0;
  unsigned long long claimed = claimer ? atom_add_global(counter, 1ull) : 0ull;  // iteration 2
#pragma unroll
  for (int j = 0; j < PW; ++j)
#pragma unroll
    for (int c = 0; c < IN; ++c)
#pragma unroll
      for (int v = 0; v < V; ++v) cur[j][c][v] = T(0);
  mbar_wait_a(mbt_a, 0u);
  int64_t tile = s_tile[0];
  if (tile < ntiles) load(tile);
  int b = 0;                      // staging buffer of iteration k
  int64_t pend[NBUF - 1];         // tiles of iterations k-1, k-2, ... still staged
#pragma unroll
  for (int q = 0; q < NBUF - 1; ++q) pend[q] = ntiles;
  int64_t k = 0;
  for (; tile < ntiles; ++k) {
    if (claimer) {
      const int q = (int)((k + 2) & kRingMask);
      s_tile[q] = (int64_t)claimed;  // claimed during iteration k - 1 (before the loop for k = 0)
      CLIP_TRACE((int64_t)claimed, 0, trace_now());
      mbar_arrive_a(mbt_a + 8 * q);
      claimed = atom_add_global(counter, 1ull);  // iteration k + 3, published next iteration
    }
    const uint32_t region = region_of(b);
    const int rem = batch_rem(tile);
    if (warp == 0 && lane == 0) CLIP_TRACE(tile, 1, trace_now());
    // ---- phase 1: R3, and the kept rows listed in segment order
    unsigned keep[PW], oor[PW];
    unsigned cnt = 0;  // kept per sub-tile, byte j
#pragma unroll
    for (int j = 0; j < PW; ++j) {
      const int o = j * SUB + lane * V;
      oor[j] = FLAGS ? Op::template oor<T, IN, V>(cur[j]) : 0u;  // flag 2 segments (NEXT-4 I6), not kept
      keep[j] = Op::template keep<V>(cur[j], w, kparams);
      if (rem < BATCH) keep[j] &= (o >= rem) ? 0u : (o + V <= rem ? (1u << V) - 1u : (1u << (rem - o)) - 1u);
      cnt |= (unsigned)__popc(keep[j]) << (8 * j);
    }
    unsigned incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    const unsigned tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const unsigned excl = incl - cnt;
    if constexpr (CW > 0) {
      if (k >= NBUF) {  // the copy warps are done with this buffer's previous tile
        mbar_wait_a(mbf_a + 8 * b, (fpar >> b) & 1u);
        fpar ^= 1u << b;
      }
    }
    // (the previous use of this region, this warp's copy-out, is done: every lane has passed
    // the scan's shuffles above after consuming its copy-out loads)
    int before = 0;
    int kbase[PW];  // list position of this lane's first kept segment of sub-tile j
#pragma unroll
    for (int j = 0; j < PW; ++j) {
      int pos = before + (int)((excl >> (8 * j)) & 0xFFu);
      kbase[j] = pos;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const unsigned kv = (keep[j] >> v) & 1u;
        if (kv) {
          T row[IN];
#pragma unroll
          for (int c = 0; c < IN; ++c) row[c] = cur[j][c][v];
          sts_rowp<T, IN, BATCH>(region, pos, row);
          if (INDEX) sts_u8(lidx_a + pos, (uint32_t)(j * SUB + lane * V + v));
        }
        pos += kv;
      }
      before += (int)((tot >> (8 * j)) & 0xFFu);
    }
    const int nkept = before;
    __syncwarp();
    // the next tile's batch, in flight during phase 2
    mbar_wait_a(mbt_a + 8 * (int)((k + 1) & kRingMask), (uint32_t)(((k + 1) / kTileRing) & 1));
    const int64_t next = s_tile[(k + 1) & kRingMask];
    if (next < ntiles) load(next);
#ifndef CLIPSEG_PK_ILCOPY
#define CLIPSEG_PK_ILCOPY 0  // copy-out rounds interleaved with phase 2 when the offsets are already known
#endif
    // The pending copy-out (iteration k - (NBUF-1), buffer cb): when its offsets have already
    // arrived, one 32-row round of it runs in each phase-2 round, overlapping its shared
    // loads and global stores with the clip arithmetic; otherwise it runs (and waits) after.
    const int cb = (b + 1 == NBUF) ? 0 : b + 1;
    bool early = false;
    int ccnt = 0, cq = 0;
    uint32_t creg = 0;
    T* cdst[OUT];
    if (CLIPSEG_PK_ILCOPY && pend[NBUF - 2] < ntiles && !INDEX &&
        mbar_test_a(mbp_a + 8 * cb, (cpar >> cb) & 1u)) {
      early = true;
      cpar ^= 1u << cb;
      ccnt = s_cnt[cb][warp];
      creg = region_of(cb);
      const int64_t g0 = s_prefix[cb] + s_pre[cb][warp];
#pragma unroll
      for (int c = 0; c < OUT; ++c) cdst[c] = out + c * ld_out + g0 + lane;
    }
    auto copy_round = [&]() {  // warp-uniform: one 32-row round of the early copy-out
      if (cq * 32 < ccnt) {
        if (cq * 32 + lane < ccnt) {
          T row[OUT];
          lds_rowp<T, IN, BATCH>(creg, cq * 32 + lane, row);
#pragma unroll
          for (int c = 0; c < OUT; ++c) __stcs(cdst[c] + cq * 32, row[c]);
        }
        ++cq;
      }
    };
    // ---- phase 2: clip the kept rows (two per lane while more than 32 remain); each
    // visible row is written back at its rank, which is at most its list position, so rows
    // still to be read are never overwritten
    int rank = 0;
    const uint32_t slix = INDEX ? sbase + (uint32_t)(S::kLixOff + ((size_t)b * W + warp) * BATCH) : 0u;
    int p0 = 0;
    // Exceptional rows (CLIPSEG_PK_DEFER): the main rounds run the fast path only; the first
    // round holding a row outside its (cheap) range test ends them, and the batch's remaining
    // rows [dstart, nkept) are finished in three passes — A: each row that passes the finer
    // range test (Op::fast_ok2) is clipped by the fast path, its result left at its list
    // position and its visible bit in the bitmap, the others are queued; B: the queue is
    // clipped by the rules in dense rounds (results in place, bits OR-ed in); C: the rows are
    // compacted to their ranks in order.  A warp thus never runs the rules on a round whose
    // other lanes hold fast rows, and rows that only fail the cheap test (edge-touching WECs)
    // stay on the fast path.  CLIPSEG_PK_DEFER 0: the per-lane fallback inside the rounds.
    constexpr bool DEFER = S::K.defer;
    if constexpr (S::K.ilp >= 3) {  // NI rows per lane per round (this instantiation's knob)
      constexpr int NI = S::K.ilp;
      for (; nkept - p0 > 32 * (NI - 1); p0 += 32 * NI) {
        T rr[NI][IN], qq[NI][OUT];
        bool vv[NI], ac[NI];
        uint32_t id[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int p = p0 + 32 * i + lane;
          ac[i] = p < nkept;
          const int pr = ac[i] ? p : p0 + lane;  // an idle row re-clips the round's first one
          lds_rowp<T, IN, BATCH>(region, pr, rr[i]);
          id[i] = INDEX ? lds_u8(lidx_a + pr) : 0u;
        }
        Op::template clip_n<NI>(rr, w, qq, vv);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const bool v = vv[i] & ac[i];
          const unsigned m = __ballot_sync(0xFFFFFFFFu, v);
          if (v) {
            const int r = rank + __popc(m & lt_mask);
            sts_rowp<T, IN, BATCH>(region, r, qq[i]);
            if (INDEX) sts_u8(slix + r, id[i]);
          }
          if (FLAGS && lane == 0) sts_u32(vb_a + 4 * ((p0 >> 5) + i), m);
          rank += __popc(m);
        }
      }
    }
    bool brk = false;  // a main round met an exceptional row (DEFER)
    if constexpr (S::K.ilp >= 2) {  // (this instantiation's knob)
    for (; nkept - p0 > 32; p0 += 64) {
      const int pa = p0 + lane, pb = p0 + 32 + lane;
      const bool actb = pb < nkept;
      const int pbr = actb ? pb : pa;  // an idle second item re-clips the first (same path, no divergence)
      T ra[IN], rb[IN];
      lds_rowp<T, IN, BATCH>(region, pa, ra);
      lds_rowp<T, IN, BATCH>(region, pbr, rb);
      const uint32_t ida = INDEX ? lds_u8(lidx_a + pa) : 0u, idb = INDEX ? lds_u8(lidx_a + pbr) : 0u;
      T qa[OUT], qb[OUT];
      bool va, vb;
#ifdef CLIPSEG_ABL_NOMATH  // ablation builds only: the framework without the clip
      for (int c = 0; c < OUT; ++c) { qa[c] = ra[c]; qb[c] = rb[c]; }
      va = ra[0] < ra[2]; vb = rb[0] < rb[2];
#else
      if constexpr (DEFER) {
        // The fast path runs before the range test's vote (its values are dropped when a row
        // fails the test: nothing is stored before the vote), so the test's dependency chain
        // and the vote do not sit in front of the clip (measured: headline 5.476 -> 5.420 ms
        // best, mix 1/3 0.618 -> 0.610 ms at 1e8; C3, whose batches break out in their first
        // round, pays that round: 0.148 -> 0.155 ms.  Voting first only after a batch that
        // broke out cost the headline 0.8 %: 5 more registers.)
        const bool ok = Op::fast_ok(ra, w) & Op::fast_ok(rb, w);
        if constexpr (S::K.vfirst) {  // (this instantiation votes before clipping)
          if (!__all_sync(0xFFFFFFFFu, ok)) {
            brk = true;
            break;
          }
          if constexpr (Op::kFastAlwaysDone) {
            Op::fast_two(ra, rb, w, qa, qb, va, vb);
          } else if (!__all_sync(0xFFFFFFFFu, Op::fast_two(ra, rb, w, qa, qb, va, vb))) {
            brk = true;
            break;
          }
        } else {
          const bool done = Op::fast_two(ra, rb, w, qa, qb, va, vb);
          if (!__all_sync(0xFFFFFFFFu, ok & done)) {
            brk = true;
            break;
          }
        }
      } else {
        Op::clip_two(ra, rb, w, qa, qb, va, vb);
      }
#endif
      vb = vb & actb;
      // (the round's rows are all read before the ballots below, which every lane reaches only
      // after consuming its loads, and ranks stay below the next round's positions: no
      // __syncwarp needed between the reads and the stores)
      if (CLIPSEG_PK_ILCOPY) __syncwarp();
      if (early) {
        copy_round();
        copy_round();
      }
      const unsigned ma = __ballot_sync(0xFFFFFFFFu, va), mb = __ballot_sync(0xFFFFFFFFu, vb);
      const int rank_b = rank + __popc(ma);
      if (va) {
        const int r = rank + __popc(ma & lt_mask);
        sts_rowp<T, IN, BATCH>(region, r, qa);
        if (INDEX) sts_u8(slix + r, ida);
      }
      if (vb) {
        const int r = rank_b + __popc(mb & lt_mask);
        sts_rowp<T, IN, BATCH>(region, r, qb);
        if (INDEX) sts_u8(slix + r, idb);
      }
      if (FLAGS && lane == 0) {
        sts_u32(vb_a + 4 * (p0 >> 5), ma);
        sts_u32(vb_a + 4 * (p0 >> 5) + 4, mb);
      }
      rank = rank_b + __popc(mb);
    }
    }
    if (!brk) {
    for (; p0 < nkept; p0 += 32) {
      const int p = p0 + lane;
      const bool act = p < nkept;
      const int pr = act ? p : p0;  // an idle lane re-clips the round's first row
      T row[IN];
      lds_rowp<T, IN, BATCH>(region, pr, row);
      const uint32_t id = INDEX ? lds_u8(lidx_a + pr) : 0u;
      T res[OUT];
#ifdef CLIPSEG_ABL_NOMATH
      for (int c = 0; c < OUT; ++c) res[c] = row[c];
      const bool vis = (row[0] < row[2]) & act;
#else
      bool vis;
      if constexpr (DEFER) {
        const bool ok = Op::fast_ok(row, w);
        if constexpr (S::K.vfirst) {
          if (!__all_sync(0xFFFFFFFFu, ok)) break;
          if constexpr (Op::kFastAlwaysDone) {
            Op::fast_try(row, w, res, vis);
          } else if (!__all_sync(0xFFFFFFFFu, Op::fast_try(row, w, res, vis))) {
            break;
          }
        } else {
          const bool done = Op::fast_try(row, w, res, vis);
          if (!__all_sync(0xFFFFFFFFu, ok & done)) break;
        }
        vis = vis & act;
      } else {
        vis = Op::clip_one(row, w, res) & act;
      }
#endif
      if (CLIPSEG_PK_ILCOPY) __syncwarp();
      if (early) copy_round();
      const unsigned m = __ballot_sync(0xFFFFFFFFu, vis);
      if (vis) {
        const int r = rank + __popc(m & lt_mask);
        sts_rowp<T, IN, BATCH>(region, r, res);
        if (INDEX) sts_u8(slix + r, id);
      }
      if (FLAGS && lane == 0) sts_u32(vb_a + 4 * (p0 >> 5), m);
      rank += __popc(m);
    }
    }
    if (DEFER && p0 < nkept) {
      const int dstart = p0;
      int nexc = 0;
      __syncwarp();
      // pass A: the finer range test; fast rows clipped in place, the others queued.  Two rows
      // per lane while more than 32 remain; the fast path runs on every row (a row that fails
      // the test yields unused values), so the rounds are straight-line code.
      auto pass_a = [&](int p, bool act, const T (&row)[IN], bool done, const T (&res)[OUT], bool vis) -> unsigned {
        done = done && act && Op::fast_ok2(row, w);
        const bool q = act && !done;
        const unsigned qm = __ballot_sync(0xFFFFFFFFu, q);
        if (q) sts_u8(exc_a + nexc + __popc(qm & lt_mask), (uint32_t)p);
        nexc += __popc(qm);
        if (done) sts_rowp<T, IN, BATCH>(region, p, res);
        return __ballot_sync(0xFFFFFFFFu, done && vis);
      };
      int q0 = dstart;
      for (; nkept - q0 > 32; q0 += 64) {
        const int pa = q0 + lane, pb = q0 + 32 + lane;
        const bool actb = pb < nkept;
        T ra[IN], rb[IN], qa[OUT], qb[OUT];
        lds_rowp<T, IN, BATCH>(region, pa, ra);
        lds_rowp<T, IN, BATCH>(region, (actb ? pb : pa), rb);
        bool va, vb;
        const bool d = Op::fast_two(ra, rb, w, qa, qb, va, vb);
        const unsigned ma = pass_a(pa, true, ra, d, qa, va);
        const unsigned mb = pass_a(pb, actb, rb, d, qb, vb);
        if (lane == 0) {
          sts_u32(vb_a + 4 * (q0 >> 5), ma);
          sts_u32(vb_a + 4 * (q0 >> 5) + 4, mb);
        }
      }
      for (; q0 < nkept; q0 += 32) {
        const int p = q0 + lane;
        const bool act = p < nkept;
        T row[IN], res[OUT];
        lds_rowp<T, IN, BATCH>(region, (act ? p : q0), row);
        bool vis;
        const bool d = Op::fast_try(row, w, res, vis);
        const unsigned m = pass_a(p, act, row, d, res, vis);
        if (lane == 0) sts_u32(vb_a + 4 * (q0 >> 5), m);
      }
      __syncwarp();
      // pass B: the queued rows, by the rules, 32 per round (their results back in place)
      for (int e0 = 0; e0 < nexc; e0 += 32) {
        const int e = e0 + lane;
        const bool act = e < nexc;
        const int p = (int)lds_u8(exc_a + (act ? e : e0));
        T row[IN], res[OUT];
        lds_rowp<T, IN, BATCH>(region, p, row);
        const bool vis = Op::exact(row, w, res);
        if (act) {
          sts_rowp<T, IN, BATCH>(region, p, res);
          if (vis) atom_or_shared_a(vb_a + 4 * (p >> 5), 1u << (p & 31));
        }
      }
      __syncwarp();
      // pass C: rows dstart.. to their ranks, in order (rank <= position: in place)
      for (int q0 = dstart; q0 < nkept; q0 += 32) {
        const int p = q0 + lane;
        const bool act = p < nkept;
        T row[OUT];  // results (OUT elements) sit at the rows' list positions
        if (act) lds_rowp<T, IN, BATCH>(region, p, row);
        const bool vis = act && ((lds_u32(vb_a + 4 * (q0 >> 5)) >> lane) & 1u);
        const uint32_t id = (INDEX && act) ? lds_u8(lidx_a + p) : 0u;
        __syncwarp();
        const unsigned m = __ballot_sync(0xFFFFFFFFu, vis);
        if (vis) {
          const int r = rank + __popc(m & lt_mask);
          sts_rowp<T, IN, BATCH>(region, r, row);
          if (INDEX) sts_u8(slix + r, id);
        }
        rank += __popc(m);
      }
    }
    if (lane == 0) s_cnt[b][warp] = rank;
    // The tile's done test and total in one relaxed shared atomic word, (finished warps << 16)
    // | (their visible rows): the warp whose add completes the count holds the tile total in
    // the returned word (no fence, no other warp's counts to read), and the result is only
    // needed after the flags, so the atomic's latency is hidden.  Measured against a fenced
    // done count + lane-0 sum of the counts: 5.283 -> 5.265 ms best; against the same with the
    // done test broadcast to the warp and a warp reduction: 5.41 -> 5.27 ms.
    uint32_t done_old = 0;
    if (lane == 0) done_old = (uint32_t)atom_add_shared(&s_done[b], (1 << 16) | rank);
    __syncwarp();
    if (FLAGS) {
      // this lane's kept segments of sub-tile j sit at list positions kbase[j], kbase[j] + 1, ...:
      // their visible bits are a run of the bitmap, spread back to the kept slots by the table
      uint8_t* fl = flags + tile * BT + (int64_t)warp * BATCH;
#pragma unroll
      for (int j = 0; j < PW; ++j) {
        const int o = j * SUB + lane * V;
        const uint32_t wa = vb_a + 4 * (kbase[j] >> 5);
        const uint32_t run = __funnelshift_r(lds_u32(wa), lds_u32(wa + 4), kbase[j] & 31) & ((1u << V) - 1u);
        uint32_t f = lds_u32(lut_a + 4 * ((keep[j] << V) | run));
        if constexpr (V == 4) f |= ((oor[j] * 0x204081u) & 0x01010101u) << 1;  // out of range -> 2
        if (rem == BATCH || o + V <= rem) {
          if constexpr (V == 4) *reinterpret_cast<uint32_t*>(fl + o) = f;
          else *reinterpret_cast<uint16_t*>(fl + o) = (uint16_t)f;
        } else {
          for (int v = 0; v < V; ++v)
            if (o + v < rem) fl[o + v] = (uint8_t)(f >> (8 * v));
        }
      }
    }
    // the last compute warp to finish publishes the tile aggregate (flag A)
    if (lane == 0 && (done_old >> 16) == (uint32_t)(W - 1)) {
      st_relaxed(status + tile, kFlagA | (unsigned long long)((done_old & 0xFFFFu) + (uint32_t)rank));
      CLIP_TRACE(tile, 2, trace_now());
    }
    if (lane == 0) mbar_arrive_a(mbc_a + 8 * b);
    // copy out iteration k - (NBUF-1), NBUF-1 tiles behind: its offsets are known by now
    b = cb;  // buffer of iteration k + 1 == buffer of iteration k - (NBUF-1)
    if constexpr (CW == 0) {
      if (early) {
        while (cq * 32 < ccnt) copy_round();
      } else if (pend[NBUF - 2] < ntiles) {
        copy_out(pend[NBUF - 2], b);
      }
    }
#pragma unroll
    for (int q = NBUF - 2; q > 0; --q) pend[q] = pend[q - 1];
    pend[0] = tile;
    tile = next;
  }
  // drain: the last NBUF-1 iterations are still staged (oldest first)
  if constexpr (CW == 0) {
#pragma unroll
    for (int q = NBUF - 2; q >= 0; --q) {
      b = (b + 1 == NBUF) ? 0 : b + 1;
      if (pend[q] < ntiles) copy_out(pend[q], b);
    }
  }
}

template <typename T, class Op, bool FLAGS, bool INDEX>
static cudaError_t launch_packed_variant(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                                         int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                                         int64_t* d_count, unsigned long long* ws, int64_t ntiles, cudaStream_t s) {
  typedef PackedShape<T, Op, INDEX> S;
  auto kern = clip_compact_packed_kernel<T, Op, FLAGS, INDEX>;
  int blocks_per_sm = 0;
  cudaError_t e = kernel_occupancy((const void*)kern, S::kThreads, S::kSmemBytes, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;
  const int64_t want = S::K.b0tiles ? (ntiles > 1 ? ntiles : 1) : ntiles + 1;  // (block 0 computes too)
  const int grid = (int)(want < cap ? want : cap);
  void* args[] = {(void*)&in,     (void*)&ld_in,     (void*)&n,          (void*)&w,     (void*)&out,
                  (void*)&ld_out, (void*)&out_index, (void*)&index_base, (void*)&flags, (void*)&d_count,
                  (void*)&ws,     (void*)&ntiles};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(S::kThreads), args, S::kSmemBytes, s);
}

template <typename T, class Op, bool FLAGS, bool INDEX>
static cudaError_t launch_compact_variant(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                                         int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags,
                                         int64_t* d_count, unsigned long long* ws, int64_t ntiles, cudaStream_t s) {
  if constexpr (compact_packed<T, Op>()) {
    return launch_packed_variant<T, Op, FLAGS, INDEX>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags,
                                                      d_count, ws, ntiles, s);
  } else {
    typedef CompactShape<T, Op, INDEX> S;
    const size_t smem = S::kSmemBytes;
    auto kern = clip_compact_kernel<T, Op, FLAGS, INDEX>;
    int blocks_per_sm = 0;
    cudaError_t e = kernel_occupancy((const void*)kern, S::kThreads, smem, &blocks_per_sm);
    if (e != cudaSuccess) return e;
    // block 0 is the global scanner; the cooperative launch keeps every block resident, so
    // the scanner runs alongside the tiles it waits on
    const int64_t cap = (int64_t)device_sm_count() * blocks_per_sm;
    const int grid = (int)(ntiles + 1 < cap ? ntiles + 1 : cap);
    void* args[] = {(void*)&in,     (void*)&ld_in,     (void*)&n,          (void*)&w,     (void*)&out,
                    (void*)&ld_out, (void*)&out_index, (void*)&index_base, (void*)&flags, (void*)&d_count,
                    (void*)&ws,     (void*)&ntiles};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(S::kThreads), args, smem, s);
  }
}

// Block tile of the instantiation launch_compact uses for (T, Op).
template <typename T, class Op> constexpr int64_t compact_tile() {
  if constexpr (compact_packed<T, Op>()) return PackedShape<T, Op, false>::BT;
  else return CompactShape<T, Op, false>::BT;  // the tile size does not depend on out_index
}

// One launch per call: the workspace (header + one status word per tile) is all zero on
// entry — zero-filled once by the caller before its first use — and the kernel leaves it
// all zero again (tile_scan_warp, block_exit), so no per-call memset is needed.
template <typename T, class Op>
cudaError_t launch_compact(const T* in, int64_t ld_in, int64_t n, const typename Op::Params& w, T* out,
                           int64_t ld_out, int64_t* out_index, int64_t index_base, uint8_t* flags, int64_t* d_count,
                           void* ws, cudaStream_t s) {
  const int64_t ntiles = (n + compact_tile<T, Op>() - 1) / compact_tile<T, Op>();
  unsigned long long* wsp = reinterpret_cast<unsigned long long*>(ws);
  // flags / out_index are optional outputs: one instantiation per combination, so the
  // per-segment code carries no test for them
  if (flags && out_index)
    return launch_compact_variant<T, Op, true, true>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags,
                                                    d_count, wsp, ntiles, s);
  if (flags)
    return launch_compact_variant<T, Op, true, false>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags,
                                                     d_count, wsp, ntiles, s);
  if (out_index)
    return launch_compact_variant<T, Op, false, true>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags,
                                                     d_count, wsp, ntiles, s);
  return launch_compact_variant<T, Op, false, false>(in, ld_in, n, w, out, ld_out, out_index, index_base, flags,
                                                    d_count, wsp, ntiles, s);
}

#ifdef CLIPSEG_TRACE
extern "C" int clip_trace_read(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_trace, bytes) == cudaSuccess ? 0 : -4;
}
extern "C" int clip_trace_clear() {
  static unsigned long long* p = nullptr;
  if (cudaGetSymbolAddress((void**)&p, g_trace) != cudaSuccess) return -4;
  return cudaMemset(p, 0, sizeof(unsigned long long) * kTraceTiles * 8) == cudaSuccess ? 0 : -4;
}
#endif

#define INST(T, OP)                                                                                          \
  template cudaError_t launch_compact<T, OP>(const T*, int64_t, int64_t, const typename OP::Params&, T*, int64_t, \
                                             int64_t*, int64_t, uint8_t*, int64_t*, void*, cudaStream_t);
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
INST(int32_t, IntOp)
#undef INST

}  // namespace clipseg
