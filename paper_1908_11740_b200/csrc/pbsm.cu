// pbsm.cu — B200-native (sm_100a) PBSM filter step of arXiv 1908.11740.
//
// Four subsystems replace the reference's per-tile CPU kernels
// (/root/reference/pkg/src/sweepjoin/_kernels.pyx) for ALL tiles at once:
//
//  1. grid partitioning with class A/B/C/D labels
//       k_count    ← count_tiles   (_kernels.pyx:34-58) + RectBatch.validate
//                    (geometry.py:166-177) folded into the same pass
//       k_plan_*   ← compute_segment_offsets (partition.py:151-164) and
//                    build_task_queue (engine.py:84-100)
//       k_scatter  ← write_tiles   (_kernels.pyx:61-98)
//       k_guard    ← the write-overflow guard (partition.py:229-233)
//  2. per-tile segmented sort by x-lower        ← sort_segment (_kernels.pyx:188-228)
//  3. forward-scan mini-joins over the class combinations
//                                               ← do_sweep (_kernels.pyx:231-293)
//  4. count → emit pair writer                  ← sweep_count / sweep_collect
//                                                 (_kernels.pyx:304-341) and the
//                                                 aggregation (engine.py:293-309)
//  (2)-(4) are one kernel, k_join: a CTA stages a chunk of join tiles in shared
//  memory with TMA bulk copies, sorts every (tile, side) segment there, counts
//  its pairs, learns its output offset by a decoupled look-back over the
//  preceding chunks, and emits.  Tiles too large for one CTA's shared memory
//  are split into work items handled by the same kernel (nested loop).
//
// Duplicate avoidance.  The reference keeps a pair in tile T iff
// max(r.xl,s.xl) >= T.xl and max(r.yl,s.yl) >= T.yl (Eq. 1,
// geometry.py:64-72, _kernels.pyx:253-262).  Because tile_of() is monotone
// and consistent with the boundaries i/k (geometry.py:87-106), that holds in
// exactly the tile where at least one of r, s starts in T's column ("x-in")
// and at least one starts in T's row ("y-in") — the paper's class scheme
// (PAPER.md:651-733): of the 16 (R-class, S-class) combinations only AA, AB,
// AC, AD, BA, BC, CA, CB, DA qualify.  The scatter writes the label into the
// two always-zero top bits of xl, so no reference-point test runs in the join.
//
// All coordinate arithmetic is IEEE float64 with correctly rounded mul/div
// (no fast-math; tile boundaries are the exact doubles i/k), so the result
// set is bit-identical to the reference's.
//
// Memory layout in HBM: inputs are the reference's SoA
// columns; a tile-list entry is one 64-byte record {xl|label, xu, yl, yu, id}
// so the random scatter writes whole 32-byte sectors (no read-modify-write)
// and a chunk's entries are one contiguous byte range for the TMA bulk copy.

#include <cuda/atomic>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "../../include/pbsm.h"

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
typedef unsigned short u16;

namespace {

// ---------------------------------------------------------------- constants
constexpr int kPlanThreads = 256;
constexpr int kPlanPer = 16;                         // tiles per thread
constexpr int kPlanTile = kPlanThreads * kPlanPer;   // 4096 tiles per CTA
constexpr int kNV = 11;                              // plan scan lanes

constexpr int kJoinThreads = 256;
constexpr int kChunkB = 640;        // chunk bucket width in entries
constexpr int kLmax = 384;          // largest tile (|R_T|+|S_T|) on the chunk path
constexpr int kCap = kChunkB + kLmax;   // max entries staged per chunk CTA
constexpr int kMaxTiles = kCap / 2;     // a join tile holds >= 2 entries
constexpr int kLargeLead = kJoinThreads;  // lead-side entries per large work item

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTile = kScanThreads * kScanPer;

constexpr int kRectsPerThread = 4;  // ILP in the count / scatter passes

constexpr u64 kXOut = 1ull << 63;
constexpr u64 kYOut = 1ull << 62;
constexpr u64 kLabelMask = kXOut | kYOut;

constexpr u32 kSkip = 0x80000000u;  // cursor base of tiles whose list is not needed

constexpr u64 kFlagAgg = 1ull << 62;   // look-back: aggregate published
constexpr u64 kFlagPre = 2ull << 62;   // look-back: inclusive prefix published
constexpr u64 kValMask = (1ull << 62) - 1;

static_assert(kLmax <= kChunkB, "a small tile may cross at most one bucket boundary");

// ---------------------------------------------------------------- records
struct __align__(64) Rec {
  u64 xl_key;   // xl bits | class label (bit 63 x-out, bit 62 y-out)
  double xu, yl, yu;
  i64 id;
  u64 pad[3];
};
static_assert(sizeof(Rec) == 64, "record size");
static_assert(sizeof(Rec) == sizeof(pbsm_entry), "entry layout");

struct __align__(32) Half {  // the MBR half of a record: one sector
  u64 xl_key;
  double xu, yl, yu;
};

// ---------------------------------------------------------------- workspace
struct WsLayout {
  size_t hdr, bx, by, cnt_r, cnt_s, cur_r, cur_s, jrec, je, cstart, lrec, lpre, partials, total;
  u64 tiles;
  u64 nblocks;
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

inline WsLayout ws_layout(int kx, int ky, int row_lo, int row_hi) {
  WsLayout L;
  const u64 T = (u64)kx * (u64)(row_hi - row_lo);
  L.tiles = T;
  L.nblocks = (T + kPlanTile - 1) / kPlanTile;
  size_t o = 0;
  L.hdr = o; o = align_up(o + sizeof(pbsm_header), 256);
  L.bx = o; o = align_up(o + sizeof(double) * (kx + 1), 256);
  L.by = o; o = align_up(o + sizeof(double) * (ky + 1), 256);
  L.cnt_r = o; o = align_up(o + 4 * T, 256);
  L.cnt_s = o; o = align_up(o + 4 * T, 256);
  L.cur_r = o; o = align_up(o + 4 * T, 256);
  L.cur_s = o; o = align_up(o + 4 * T, 256);
  L.jrec = o; o = align_up(o + 16 * T, 256);
  L.je = o; o = align_up(o + 4 * (T + 1), 256);
  L.cstart = o; o = align_up(o + 4 * (T + 2), 256);
  L.lrec = o; o = align_up(o + 16 * T, 256);
  L.lpre = o; o = align_up(o + 4 * (T + 1), 256);
  L.partials = o; o = align_up(o + sizeof(u64) * kNV * (L.nblocks + 1), 256);
  L.total = o;
  return L;
}

struct Ws {
  pbsm_header* hdr;
  double* bx;
  double* by;
  u32 *cnt_r, *cnt_s, *cur_r, *cur_s, *je, *cstart, *lpre;
  uint4 *jrec, *lrec;   // {r_start, s_start, nR, nS}
  u64* partials;
  u64 tiles, nblocks;
};

inline Ws ws_bind(void* base, const WsLayout& L) {
  char* b = (char*)base;
  Ws w;
  w.hdr = (pbsm_header*)(b + L.hdr);
  w.bx = (double*)(b + L.bx);
  w.by = (double*)(b + L.by);
  w.cnt_r = (u32*)(b + L.cnt_r);
  w.cnt_s = (u32*)(b + L.cnt_s);
  w.cur_r = (u32*)(b + L.cur_r);
  w.cur_s = (u32*)(b + L.cur_s);
  w.jrec = (uint4*)(b + L.jrec);
  w.je = (u32*)(b + L.je);
  w.cstart = (u32*)(b + L.cstart);
  w.lrec = (uint4*)(b + L.lrec);
  w.lpre = (u32*)(b + L.lpre);
  w.partials = (u64*)(b + L.partials);
  w.tiles = L.tiles;
  w.nblocks = L.nblocks;
  return w;
}

// ---------------------------------------------------------------- helpers

// axis_tile_index (geometry.py:87-106) / tile_of (_kernels.pyx:20-31):
// floor(p*k) clamped to [0,k-1], then nudged against the materialised
// boundaries b[i] = i/k so it agrees with boundary comparisons exactly.
__device__ __forceinline__ int tile_of(double p, int k, const double* __restrict__ b) {
  long long i = (long long)__dmul_rn(p, (double)k);
  if (!(i >= 0)) i = 0;
  if (i > k - 1) i = k - 1;
  while (i > 0 && p < __ldg(b + i)) --i;
  while (i < k - 1 && p >= __ldg(b + i + 1)) ++i;
  return (int)i;
}

// Non-negative doubles order like their bit patterns; -0.0 is mapped to +0.0
// so the two top bits are free for the class label.
__device__ __forceinline__ u64 xl_bits(double xl) {
  return xl == 0.0 ? 0ull : (u64)__double_as_longlong(xl);
}

__device__ __forceinline__ double key_x(u64 key) {
  return __longlong_as_double((long long)(key & ~kLabelMask));
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one u64 per thread; returns the exclusive
// prefix, *total receives the block sum.  NT = blockDim.x.
template <int NT>
__device__ __forceinline__ u64 block_excl_scan(u64 v, u64* total, u64* sh /* >= NT/32+1 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64 inc = warp_incl_scan<u64>(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    u64 s = lane < NT / 32 ? sh[lane] : 0ull;
    u64 si = warp_incl_scan<u64>(s);
    if (lane < NT / 32) sh[lane] = si - s;
    if (lane == NT / 32 - 1) sh[NT / 32] = si;
  }
  __syncthreads();
  u64 r = inc - v + sh[wid];
  *total = sh[NT / 32];
  __syncthreads();
  return r;
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier, one elected thread issues
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---------------------------------------------------------------- init
__global__ void k_bounds(double* bx, int kx, double* by, int ky) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  // tile_boundary (geometry.py:82-84): i / k, correctly rounded
  if (i <= kx) bx[i] = __ddiv_rn((double)i, (double)kx);
  if (i <= ky) by[i] = __ddiv_rn((double)i, (double)ky);
}

// ---------------------------------------------------------------- 1a count
// count_tiles (_kernels.pyx:34-58) for all rectangles; each thread keeps
// kRectsPerThread rectangles in flight.  The same pass applies
// RectBatch.validate (geometry.py:166-177): inverted or out-of-[0,1]
// rectangles raise error bits the host turns into the reference's ValueError.
__global__ void __launch_bounds__(256) k_count(const double* __restrict__ xl,
                                               const double* __restrict__ xu,
                                               const double* __restrict__ yl,
                                               const double* __restrict__ yu, i64 n,
                                               int kx, int ky, int row_lo, int row_hi,
                                               const double* __restrict__ bx,
                                               const double* __restrict__ by,
                                               u32* __restrict__ cnt, int side,
                                               pbsm_header* hdr) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  u32 bad = 0;
  for (i64 base = blockIdx.x * (i64)blockDim.x + threadIdx.x; base < n;
       base += stride * kRectsPerThread) {
    double a[kRectsPerThread], b[kRectsPerThread], c[kRectsPerThread], d[kRectsPerThread];
#pragma unroll
    for (int u = 0; u < kRectsPerThread; ++u) {
      const i64 i = base + u * stride;
      if (i < n) {
        a[u] = __ldg(xl + i);
        b[u] = __ldg(xu + i);
        c[u] = __ldg(yl + i);
        d[u] = __ldg(yu + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kRectsPerThread; ++u) {
      const i64 i = base + u * stride;
      if (i >= n) continue;
      if (!(a[u] <= b[u]) || !(c[u] <= d[u])) bad |= PBSM_ERR_INVERTED;
      if (a[u] < 0.0 || c[u] < 0.0 || b[u] > 1.0 || d[u] > 1.0) bad |= PBSM_ERR_RANGE;
      const int c0 = tile_of(a[u], kx, bx);
      const int c1 = tile_of(b[u], kx, bx);
      const int r0 = max(tile_of(c[u], ky, by), row_lo);
      const int r1 = min(tile_of(d[u], ky, by), row_hi - 1);
      for (int row = r0; row <= r1; ++row) {
        u32* rowp = cnt + (size_t)(row - row_lo) * kx;
        for (int col = c0; col <= c1; ++col) atomicAdd(rowp + col, 1u);
      }
    }
  }
  if (bad) atomicOr(&hdr->error, bad << (2 * side));
}

// ---------------------------------------------------------------- 1c scatter
// write_tiles (_kernels.pyx:61-98): copy each rectangle into every tile it
// overlaps, labelled with its class there.  Only tiles where both inputs are
// non-empty get a list (the others cannot produce a pair: build_task_queue
// joins only those, engine.py:97); their cursors start at kSkip and the write
// is skipped, but the cursor still advances so k_guard can check every tile.
__global__ void __launch_bounds__(256) k_scatter(const i64* __restrict__ ids,
                                                 const double* __restrict__ xl,
                                                 const double* __restrict__ xu,
                                                 const double* __restrict__ yl,
                                                 const double* __restrict__ yu, i64 n,
                                                 int kx, int ky, int row_lo, int row_hi,
                                                 const double* __restrict__ bx,
                                                 const double* __restrict__ by,
                                                 u32* __restrict__ cursor, Rec* __restrict__ out,
                                                 i64 capacity, pbsm_header* hdr) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  u32 bad = 0;
  for (i64 base = blockIdx.x * (i64)blockDim.x + threadIdx.x; base < n;
       base += stride * kRectsPerThread) {
    double a[kRectsPerThread], b[kRectsPerThread], c[kRectsPerThread], d[kRectsPerThread];
    i64 id[kRectsPerThread];
#pragma unroll
    for (int u = 0; u < kRectsPerThread; ++u) {
      const i64 i = base + u * stride;
      if (i < n) {
        a[u] = __ldg(xl + i);
        b[u] = __ldg(xu + i);
        c[u] = __ldg(yl + i);
        d[u] = __ldg(yu + i);
        id[u] = __ldg(ids + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kRectsPerThread; ++u) {
      const i64 i = base + u * stride;
      if (i >= n) continue;
      const int c0 = tile_of(a[u], kx, bx);
      const int c1 = tile_of(b[u], kx, bx);
      const int rr0 = tile_of(c[u], ky, by);
      const int r0 = max(rr0, row_lo);
      const int r1 = min(tile_of(d[u], ky, by), row_hi - 1);
      const u64 xk = xl_bits(a[u]);
      for (int row = r0; row <= r1; ++row) {
        u32* rowp = cursor + (size_t)(row - row_lo) * kx;
        const u64 ylab = (row != rr0) ? kYOut : 0ull;
        for (int col = c0; col <= c1; ++col) {
          const u32 pos = atomicAdd(rowp + col, 1u);
          if (pos >= kSkip) continue;  // not a join tile
          if ((i64)pos >= capacity) {
            bad |= PBSM_ERR_SCATTER_OVERFLOW;
            continue;
          }
          Half h;
          h.xl_key = xk | ylab | ((col != c0) ? kXOut : 0ull);
          h.xu = b[u];
          h.yl = c[u];
          h.yu = d[u];
          Rec* r = out + pos;
          *reinterpret_cast<Half*>(r) = h;
          Half t;
          t.xl_key = (u64)id[u];
          t.xu = 0.0;
          t.yl = 0.0;
          t.yu = 0.0;
          *reinterpret_cast<Half*>(&r->id) = t;
        }
      }
    }
  }
  if (bad) atomicOr(&hdr->error, bad);
}

// write guard (partition.py:229-233): every cursor must end exactly where the
// count pass said (the plan stored the expected end in cnt[]).
__global__ void k_guard(const u32* __restrict__ cur_r, const u32* __restrict__ end_r,
                        const u32* __restrict__ cur_s, const u32* __restrict__ end_s, u64 T,
                        pbsm_header* hdr) {
  bool bad = false;
  for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < T;
       t += (u64)gridDim.x * blockDim.x)
    bad |= (cur_r[t] != end_r[t]) || (cur_s[t] != end_s[t]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&hdr->error, PBSM_ERR_OFFSET_MISMATCH);
}

// ---------------------------------------------------------------- 1b plan
// Per tile t the plan scans nine lanes at once:
//   0 |R_T|  1 |S_T|                         (A_R, A_S: PartitionedDataset totals)
//   2 small-join flag  3 small-join entries  (→ join tile list + CTA chunks)
//   4 large-join flag  5 large-join items    (→ large tile list)
//   6 |R_T| 7 |S_T| of small join tiles   ┐ tile-list offsets (compute_segment_
//   9 |R_T| 10 |S_T| of large join tiles  ┘ offsets, partition.py:151-164)
//   8 |R_T|·|S_T| of join tiles              (upper bound on the pair count)
// A join tile has both inputs non-empty (build_task_queue, engine.py:97).
// Small join tiles take the front of each tile list in tile order, so a
// chunk of consecutive small tiles is one contiguous range per input; large
// tiles follow in a second region.
__device__ __forceinline__ void tile_vals(u32 a, u32 b, u64 v[kNV]) {
  const bool join = a != 0u && b != 0u;
  const u32 w = a + b;
  const bool small = join && w <= (u32)kLmax;
  const bool large = join && !small;
  const u32 lead = a >= b ? a : b;
  v[0] = a;
  v[1] = b;
  v[2] = small;
  v[3] = small ? w : 0u;
  v[4] = large;
  v[5] = large ? (lead + kLargeLead - 1) / kLargeLead : 0u;
  v[6] = small ? a : 0u;
  v[7] = small ? b : 0u;
  v[8] = join ? (u64)a * (u64)b : 0ull;
  v[9] = large ? a : 0u;
  v[10] = large ? b : 0u;
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_reduce(const u32* __restrict__ cr,
                                                              const u32* __restrict__ cs,
                                                              u64 T, u64* __restrict__ partials,
                                                              pbsm_header* hdr) {
  __shared__ u64 sh[kPlanThreads / 32][kNV];
  __shared__ u32 shmax[kPlanThreads / 32];
  u64 acc[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) acc[q] = 0;
  u32 mx = 0;
  const u64 base = (u64)blockIdx.x * kPlanTile;
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = base + (u64)i * kPlanThreads + threadIdx.x;
    if (t < T) {
      const u32 a = cr[t], b = cs[t];
      u64 v[kNV];
      tile_vals(a, b, v);
#pragma unroll
      for (int q = 0; q < kNV; ++q) acc[q] += v[q];
      if (a && b) mx = max(mx, a + b);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kNV; ++q) {
    u64 v = acc[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[wid][q] = v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if (lane == 0) shmax[wid] = mx;
  __syncthreads();
  if (threadIdx.x < kNV) {
    u64 s = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) s += sh[w][threadIdx.x];
    partials[(u64)blockIdx.x * kNV + threadIdx.x] = s;
  }
  if (threadIdx.x == 0) {
    u32 m = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) m = max(m, shmax[w]);
    atomicMax((unsigned long long*)&hdr->max_tile, (unsigned long long)m);
  }
}

// single CTA: exclusive scan of the per-CTA partial sums, totals → header
__global__ void __launch_bounds__(1024) k_plan_partials(u64* __restrict__ partials, u64 nb,
                                                        pbsm_header* hdr, u32* je, u32* lpre,
                                                        u32* cstart) {
  __shared__ u64 sh[33];
  u64 carry[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) carry[q] = 0;
  for (u64 base = 0; base < nb; base += 1024) {
    const u64 i = base + threadIdx.x;
#pragma unroll
    for (int q = 0; q < kNV; ++q) {
      const u64 v = i < nb ? partials[i * kNV + q] : 0ull;
      u64 tot;
      const u64 ex = block_excl_scan<1024>(v, &tot, sh);
      if (i < nb) partials[i * kNV + q] = carry[q] + ex;
      carry[q] += tot;
    }
  }
  if (threadIdx.x == 0) {
    hdr->a_r = (i64)carry[0];
    hdr->a_s = (i64)carry[1];
    hdr->n_join = (i64)carry[2];
    hdr->w_join = (i64)carry[3];
    hdr->n_large = (i64)carry[4];
    hdr->n_items = (i64)carry[5];
    hdr->list_r = (i64)(carry[6] + carry[9]);
    hdr->list_s = (i64)(carry[7] + carry[10]);
    partials[nb * kNV + 0] = carry[6];   // small-region sizes, read by k_plan_apply
    partials[nb * kNV + 1] = carry[7];
    hdr->pair_bound = (i64)carry[8];
    hdr->n_chunks = 0;
    hdr->pairs = 0;
    if (carry[0] >= kSkip || carry[1] >= kSkip || carry[3] >= kSkip || carry[5] >= kSkip ||
        carry[6] + carry[9] >= kSkip || carry[7] + carry[10] >= kSkip)
      hdr->error |= PBSM_ERR_TOTAL_RANGE;
    je[carry[2]] = (u32)carry[3];      // sentinel: end of the last join tile
    lpre[carry[4]] = (u32)carry[5];    // sentinel: total large work items
    cstart[0] = 0;
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_apply(
    u32* __restrict__ cr, u32* __restrict__ cs, u64 T, u64 nb, const u64* __restrict__ partials,
    u32* __restrict__ cur_r, u32* __restrict__ cur_s, uint4* __restrict__ jrec,
    u32* __restrict__ je, uint4* __restrict__ lrec, u32* __restrict__ lpre) {
  __shared__ u32 sa[kPlanTile];
  __shared__ u32 sb[kPlanTile];
  __shared__ u64 shs[33];
  const u64 base = (u64)blockIdx.x * kPlanTile;
  for (int i = threadIdx.x; i < kPlanTile; i += kPlanThreads) {
    const u64 t = base + i;
    sa[i] = t < T ? cr[t] : 0u;
    sb[i] = t < T ? cs[t] : 0u;
  }
  __syncthreads();
  u32 a[kPlanPer], b[kPlanPer];
  u64 acc[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) acc[q] = 0;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    a[i] = sa[threadIdx.x * kPlanPer + i];
    b[i] = sb[threadIdx.x * kPlanPer + i];
    u64 v[kNV];
    tile_vals(a[i], b[i], v);
#pragma unroll
    for (int q = 0; q < kNV; ++q) acc[q] += v[q];
  }
  u64 pre[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) {
    u64 tot;
    pre[q] = block_excl_scan<kPlanThreads>(acc[q], &tot, shs) +
             partials[(u64)blockIdx.x * kNV + q];
  }
  const u64 small_r = partials[nb * kNV + 0], small_s = partials[nb * kNV + 1];
  // (block_excl_scan ends with a barrier, so sa/sb may be overwritten now:
  // they receive the cursor starts; the expected cursor ends go back into
  // cnt[] for k_guard.)
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = base + (u64)threadIdx.x * kPlanPer + i;
    u64 v[kNV];
    tile_vals(a[i], b[i], v);
    const u32 r0 = v[2] ? (u32)pre[6] : v[4] ? (u32)(small_r + pre[9]) : kSkip;
    const u32 s0 = v[2] ? (u32)pre[7] : v[4] ? (u32)(small_s + pre[10]) : kSkip;
    sa[threadIdx.x * kPlanPer + i] = r0;
    sb[threadIdx.x * kPlanPer + i] = s0;
    if (t < T) {
      if (v[2]) {
        jrec[pre[2]] = make_uint4(r0, s0, a[i], b[i]);
        je[pre[2]] = (u32)pre[3];
      }
      if (v[4]) {
        lrec[pre[4]] = make_uint4(r0, s0, a[i], b[i]);
        lpre[pre[4]] = (u32)pre[5];
      }
    }
#pragma unroll
    for (int q = 0; q < kNV; ++q) pre[q] += v[q];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPlanTile; i += kPlanThreads) {
    const u64 t = base + i;
    if (t < T) {
      const u32 r0 = sa[i], s0 = sb[i];
      cr[t] = r0 + cr[t];   // expected end of tile t's R cursor
      cs[t] = s0 + cs[t];
      cur_r[t] = r0;
      cur_s[t] = s0;
    }
  }
}

// chunk c = the join tiles whose exclusive entry prefix lies in [c*B, (c+1)*B);
// a chunk holds < B + kLmax = kCap entries.
__global__ void k_chunks(const u32* __restrict__ je, u32* __restrict__ cstart, pbsm_header* hdr) {
  const i64 nj = hdr->n_join;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < nj;
       j += (i64)gridDim.x * blockDim.x) {
    const i64 c = je[j] / kChunkB;
    const i64 cp = j == 0 ? -1 : (i64)(je[j - 1] / kChunkB);
    for (i64 cc = cp + 1; cc <= c; ++cc) cstart[cc] = (u32)j;
    if (j == nj - 1) {
      cstart[c + 1] = (u32)nj;
      hdr->n_chunks = c + 1;
    }
  }
}

// ---------------------------------------------------------------- generic scan
// exclusive scan of u32 counts into u64 bases; base[n] = total (ε refinement)
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const u32* __restrict__ in, u64 n,
                                                              u64* __restrict__ partials) {
  __shared__ u64 sh[kScanThreads / 32];
  u64 acc = 0;
  const u64 base = (u64)blockIdx.x * kScanTile;
  for (int i = 0; i < kScanPer; ++i) {
    const u64 t = base + (u64)i * kScanThreads + threadIdx.x;
    if (t < n) acc += in[t];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 s = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) s += sh[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024) k_scan_partials(u64* __restrict__ partials, u64 nb,
                                                        u64* __restrict__ out, u64 n) {
  __shared__ u64 sh[33];
  u64 carry = 0;
  for (u64 base = 0; base < nb; base += 1024) {
    const u64 i = base + threadIdx.x;
    const u64 v = i < nb ? partials[i] : 0ull;
    u64 tot;
    const u64 ex = block_excl_scan<1024>(v, &tot, sh);
    if (i < nb) partials[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const u32* __restrict__ in, u64 n,
                                                             const u64* __restrict__ partials,
                                                             u64* __restrict__ out) {
  __shared__ u32 sv[kScanTile];
  __shared__ u64 shs[33];
  const u64 base = (u64)blockIdx.x * kScanTile;
  for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
    const u64 t = base + i;
    sv[i] = t < n ? in[t] : 0u;
  }
  __syncthreads();
  u64 acc = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) acc += sv[threadIdx.x * kScanPer + i];
  u64 tot;
  u64 pre = block_excl_scan<kScanThreads>(acc, &tot, shs) + partials[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const u64 t = base + (u64)threadIdx.x * kScanPer + i;
    const u32 v = sv[threadIdx.x * kScanPer + i];
    if (t < n) out[t] = pre;
    pre += v;
  }
}

// ---------------------------------------------------------------- 2-4 join
struct JoinArgs {
  const uint4* jrec;
  const u32* cstart;
  const uint4* lrec;
  const u32* lpre;
  const Rec* rl;
  const Rec* sl;
  u32* ticket;
  u64* status;     // [n_units] decoupled look-back words (emit mode)
  i64* pairs;      // (r_id, s_id) int64 pairs
  i64 capacity;    // pairs the buffer holds
  i64 n_chunks;
  i64 n_units;
  pbsm_header* hdr;
};

struct ChunkSmem {
  Rec recs[kCap];      // TMA landing zone: the chunk's R range then its S range
  u64 key[kCap];       // label|xl bits per loaded entry
  double sxl[kCap];    // per segment: [x-in sorted by xl | x-out]
  double syl[kCap];
  double syu[kCap];
  u16 sidx[kCap];      // sorted position → loaded entry
  u16 seg[kCap];       // position → chunk-local tile
  unsigned char syin[kCap];
  u16 tR0[kMaxTiles], tS0[kMaxTiles], tNR[kMaxTiles], tNS[kMaxTiles];
  u16 tNinR[kMaxTiles], tNinS[kMaxTiles];
  u64 bar;
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  int unit, nt, NR, NS;
};

struct LargeSmem {
  Rec other[kCap];
  u64 bar;
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  int unit;
};

union JoinSmem {
  ChunkSmem c;
  LargeSmem l;
};

// Decoupled look-back (one thread): publish this unit's count, accumulate the
// predecessors' published values until an inclusive prefix is found, publish
// ours.  Units are handed out by an atomic ticket in launch order, so every
// predecessor is resident or finished — the spin cannot deadlock.
__device__ u64 lookback(u64* status, i64 unit, u64 count, pbsm_header* hdr) {
  cuda::atomic_ref<u64, cuda::thread_scope_device> me(status[unit]);
  if (unit == 0) {
    me.store(kFlagPre | count, cuda::memory_order_release);
    return 0;
  }
  me.store(kFlagAgg | count, cuda::memory_order_release);
  u64 excl = 0;
  i64 j = unit - 1;
  u64 spins = 0;
  while (true) {
    cuda::atomic_ref<u64, cuda::thread_scope_device> st(status[j]);
    const u64 v = st.load(cuda::memory_order_acquire);
    const u64 flag = v & ~kValMask;
    if (flag == 0) {
      // a predecessor that never publishes is a bug; never hang the GPU on it
      if (++spins > (1ull << 24)) {
        atomicOr(&hdr->error, PBSM_ERR_INTERNAL);
        break;
      }
      __nanosleep(64);
      continue;
    }
    excl += v & kValMask;
    if (flag == kFlagPre) break;
    --j;
  }
  me.store(kFlagPre | (excl + count), cuda::memory_order_release);
  return excl;
}

// One leader element of the forward scan (Alg. 1, _kernels.pyx:231-293,
// reformulated per element).  In the reference, when r.xl < s.xl the R
// element scans S, otherwise S scans R (ties advance S, :245); so R leads the
// pairs with s.xl in (r.xl, r.xu] and S leads those with r.xl in [s.xl, s.xu].
// Only x-in entries are sorted and searched; an x-out leader (class C/D)
// starts left of the tile, so its x-overlap with an x-in partner reduces to
// partner.xl <= leader.xu: a prefix of the partner's sorted x-in run
// (mini-joins AC, AD, BC, CA, CB, DA).  A candidate is kept iff the y-ranges
// overlap and at least one side is y-in, which rejects BB/BD/DB and with the
// x rule above leaves exactly the nine class combinations AA AB AC AD BA BC CA
// CB DA.
template <bool EMIT>
__device__ __forceinline__ u32 sweep_one(const ChunkSmem& S, int p, i64* out) {
  const int lt = S.seg[p];
  const int rb = S.tR0[lt], sb = S.tS0[lt];
  const bool lead_r = p < sb;
  const double mxl = S.sxl[p], myl = S.syl[p], myu = S.syu[p];
  const bool yme = S.syin[p];
  const double mxu = S.recs[S.sidx[p]].xu;
  int k, hi;
  if (lead_r) {
    k = sb;
    hi = sb + S.tNinS[lt];
    if (p - rb < S.tNinR[lt]) {
      // upper_bound(S x-in run, r.xl): first s with s.xl > r.xl
      int b = hi;
      while (k < b) {
        const int m = (k + b) >> 1;
        if (S.sxl[m] <= mxl) k = m + 1; else b = m;
      }
    }
  } else {
    k = rb;
    hi = rb + S.tNinR[lt];
    if (p - sb < S.tNinS[lt]) {
      // lower_bound(R x-in run, s.xl): first r with r.xl >= s.xl
      int b = hi;
      while (k < b) {
        const int m = (k + b) >> 1;
        if (S.sxl[m] < mxl) k = m + 1; else b = m;
      }
    }
  }
  u32 c = 0;
  i64 my_id = 0;
  if (EMIT) my_id = S.recs[S.sidx[p]].id;
  for (; k < hi; ++k) {
    if (S.sxl[k] > mxu) break;
    if (myl <= S.syu[k] && S.syl[k] <= myu && (yme || S.syin[k])) {
      if (EMIT) {
        const i64 oid = S.recs[S.sidx[k]].id;
        *reinterpret_cast<longlong2*>(out + 2 * (i64)c) =
            lead_r ? make_longlong2(my_id, oid) : make_longlong2(oid, my_id);
      }
      ++c;
    }
  }
  return c;
}

template <bool EMIT>
__device__ void join_chunk(ChunkSmem& S, const JoinArgs& A, int c) {
  const int tid = threadIdx.x;
  const u32 j0 = A.cstart[c], j1 = A.cstart[c + 1];
  const int nt = (int)(j1 - j0);
  if (tid == 0) {
    const uint4 first = A.jrec[j0], last = A.jrec[j1 - 1];
    const int NR = (int)(last.x + last.z - first.x);
    const int NS = (int)(last.y + last.w - first.y);
    // a chunk never exceeds the staging buffer by construction (k_chunks);
    // if it somehow did, flag it and contribute 0 pairs (the look-back chain
    // must still be fed, so no early return)
    const bool fits = NR > 0 && NS > 0 && NR + NS <= kCap && nt <= kMaxTiles;
    if (!fits) atomicOr(&A.hdr->error, PBSM_ERR_INTERNAL);
    S.nt = fits ? nt : 0;
    S.NR = fits ? NR : 0;
    S.NS = fits ? NS : 0;
    if (fits) {
      // TMA: two bulk copies (the chunk's R and S ranges are contiguous
      // because small join tiles get consecutive list offsets in tile order)
      mbar_init(&S.bar, 1);
      mbar_expect_tx(&S.bar, (u32)(NR + NS) * (u32)sizeof(Rec));
      bulk_g2s(&S.recs[0], A.rl + first.x, (u32)NR * (u32)sizeof(Rec), &S.bar);
      bulk_g2s(&S.recs[NR], A.sl + first.y, (u32)NS * (u32)sizeof(Rec), &S.bar);
    }
  }
  __syncthreads();
  const int NR = S.NR, N = S.NR + S.NS;
  // tile table + position → tile map, while the copies are in flight
  {
    const uint4 first = A.jrec[j0];
    for (int lt = tid; lt < S.nt; lt += kJoinThreads) {
      const uint4 r = A.jrec[j0 + lt];
      const int r0 = (int)(r.x - first.x), s0 = NR + (int)(r.y - first.y);
      S.tR0[lt] = (u16)r0;
      S.tS0[lt] = (u16)s0;
      S.tNR[lt] = (u16)r.z;
      S.tNS[lt] = (u16)r.w;
      for (int e = 0; e < (int)r.z; ++e) S.seg[r0 + e] = (u16)lt;
      for (int e = 0; e < (int)r.w; ++e) S.seg[s0 + e] = (u16)lt;
    }
  }
  if (N > 0) mbar_wait(&S.bar, 0);
  for (int e = tid; e < N; e += kJoinThreads) S.key[e] = S.recs[e].xl_key;
  __syncthreads();

  // ---- 2: segmented sort (sort_segment, _kernels.pyx:188-228) by rank
  // counting inside each (tile, side) segment.  x-in entries are ordered by
  // (xl, load position) — a strict total order, so ranks are a permutation;
  // x-out entries keep load order after the x-in run.
  for (int e = tid; e < N; e += kJoinThreads) {
    const int lt = S.seg[e];
    const bool is_r = e < NR;
    const int a = is_r ? S.tR0[lt] : S.tS0[lt];
    const int b = a + (is_r ? S.tNR[lt] : S.tNS[lt]);
    const u64 ke = S.key[e];
    const bool in_e = !(ke & kXOut);
    const u64 xe = ke & ~kLabelMask;
    int n_in = 0, less = 0, out_before = 0;
    for (int j = a; j < b; ++j) {
      const u64 kj = S.key[j];
      const bool in_j = !(kj & kXOut);
      const u64 xj = kj & ~kLabelMask;
      n_in += in_j;
      less += in_j & ((xj < xe) | ((xj == xe) & (j < e)));
      out_before += (!in_j) & (j < e);
    }
    const int p = a + (in_e ? less : n_in + out_before);
    S.sxl[p] = __longlong_as_double((long long)xe);
    S.syl[p] = S.recs[e].yl;
    S.syu[p] = S.recs[e].yu;
    S.syin[p] = (ke & kYOut) ? 0 : 1;
    S.sidx[p] = (u16)e;
    if (e == a) {
      if (is_r) S.tNinR[lt] = (u16)n_in;
      else S.tNinS[lt] = (u16)n_in;
    }
  }
  __syncthreads();

  // ---- 3/4: forward-scan mini-joins: count, look-back, emit
  u32 cnt = 0;
  for (int p = tid; p < N; p += kJoinThreads) cnt += sweep_one<false>(S, p, nullptr);
  u64 total;
  const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
  if (!EMIT) {
    if (tid == 0 && total) atomicAdd((unsigned long long*)&A.hdr->pairs, total);
    return;
  }
  if (tid == 0) {
    const u64 b = lookback(A.status, c, total, A.hdr);
    S.base = b;
    if (c == A.n_units - 1) A.hdr->pairs = (i64)(b + total);
  }
  __syncthreads();
  const i64 start = (i64)(S.base + excl);
  if (start + (i64)cnt > A.capacity) {
    if (cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
    return;
  }
  i64* out = A.pairs + 2 * start;
  for (int p = tid; p < N; p += kJoinThreads) out += 2 * (i64)sweep_one<true>(S, p, out);
}

// Large join tiles (|R_T|+|S_T| > kLmax): the larger side is split into work
// items of kLargeLead entries, one per thread; the other side streams through
// shared memory.  Every (lead, other) pair is tested with the full
// closed-interval predicate (intersects, geometry.py:59-61) and the class rule
// (>= 1 x-in and >= 1 y-in ⇔ Eq. 1 owner tile).
template <bool EMIT>
__device__ __forceinline__ u32 large_pass(const LargeSmem& S, int n, bool have, const Half& me,
                                          bool lead_r, i64 my_id, i64* out) {
  u32 c = 0;
  if (!have) return 0;
  const double mxl = key_x(me.xl_key);
  const bool mxin = !(me.xl_key & kXOut), myin = !(me.xl_key & kYOut);
  for (int k = 0; k < n; ++k) {
    const Rec& o = S.other[k];
    const u64 ok = o.xl_key;
    const double oxl = key_x(ok);
    if (mxl <= o.xu && oxl <= me.xu && me.yl <= o.yu && o.yl <= me.yu &&
        (mxin || !(ok & kXOut)) && (myin || !(ok & kYOut))) {
      if (EMIT) {
        *reinterpret_cast<longlong2*>(out + 2 * (i64)c) =
            lead_r ? make_longlong2(my_id, o.id) : make_longlong2(o.id, my_id);
      }
      ++c;
    }
  }
  return c;
}

template <bool EMIT>
__device__ void join_large(LargeSmem& S, const JoinArgs& A, i64 unit) {
  const int tid = threadIdx.x;
  const i64 item = unit - A.n_chunks;
  // item → large tile (binary search over the work-item prefix)
  int lo = 0, hi = (int)A.hdr->n_large;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if ((i64)A.lpre[m] <= item) lo = m + 1; else hi = m;
  }
  const int lj = lo - 1;
  const uint4 rec = A.lrec[lj];
  const u32 nR = rec.z, nS = rec.w;
  const bool lead_r = nR >= nS;
  const u32 no = lead_r ? nS : nR;
  const Rec* L = lead_r ? A.rl + rec.x : A.sl + rec.y;
  const Rec* O = lead_r ? A.sl + rec.y : A.rl + rec.x;
  const u32 nl = lead_r ? nR : nS;
  const u32 a = (u32)(item - (i64)A.lpre[lj]) * kLargeLead + tid;
  const bool have = a < nl;
  Half me;
  i64 my_id = 0;
  if (have) {
    me = *reinterpret_cast<const Half*>(L + a);
    my_id = L[a].id;
  }
  if (tid == 0) mbar_init(&S.bar, 1);
  __syncthreads();
  u32 phase = 0;
  u32 cnt = 0;
  const int passes = EMIT ? 2 : 1;
  i64* out = nullptr;
  bool ok = true;
  for (int pass = 0; pass < passes; ++pass) {
    for (u32 ob = 0; ob < no; ob += kCap) {
      const int n = (int)min((u32)kCap, no - ob);
      __syncthreads();  // previous piece fully consumed
      if (tid == 0) {
        mbar_expect_tx(&S.bar, (u32)n * (u32)sizeof(Rec));
        bulk_g2s(&S.other[0], O + ob, (u32)n * (u32)sizeof(Rec), &S.bar);
      }
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
      if (pass == 0) {
        cnt += large_pass<false>(S, n, have, me, lead_r, my_id, nullptr);
      } else if (ok) {
        out += 2 * (i64)large_pass<true>(S, n, have, me, lead_r, my_id, out);
      }
    }
    if (pass == 0) {
      u64 total;
      const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
      if (!EMIT) {
        if (tid == 0 && total) atomicAdd((unsigned long long*)&A.hdr->pairs, total);
        return;
      }
      if (tid == 0) {
        const u64 b = lookback(A.status, unit, total, A.hdr);
        S.base = b;
        if (unit == A.n_units - 1) A.hdr->pairs = (i64)(b + total);
      }
      __syncthreads();
      const i64 start = (i64)(S.base + excl);
      ok = start + (i64)cnt <= A.capacity;
      if (!ok && cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
      out = A.pairs + 2 * start;
    }
  }
}

template <bool EMIT>
__global__ void __launch_bounds__(kJoinThreads, 2) k_join(JoinArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  JoinSmem& U = *reinterpret_cast<JoinSmem*>(smem_raw);
  __shared__ int s_unit;
  if (threadIdx.x == 0) s_unit = (int)atomicAdd(A.ticket, 1u);
  __syncthreads();
  const int unit = s_unit;
  if (unit < A.n_chunks) join_chunk<EMIT>(U.c, A, unit);
  else join_large<EMIT>(U.l, A, unit);
}

// ---------------------------------------------------------------- ε refinement
// _refine_pairs (engine.py:201-206): keep a candidate (row i of P, row j of Q)
// iff dx*dx + dy*dy <= eps^2 with every operation rounded on its own (numpy
// semantics: no FMA contraction), then map row indices to ids (:298-300).
__device__ __forceinline__ bool within_eps(const i64* __restrict__ cand, i64 i,
                                           const double* __restrict__ px,
                                           const double* __restrict__ py,
                                           const double* __restrict__ qx,
                                           const double* __restrict__ qy, double eps_sq) {
  const i64 a = cand[2 * i], b = cand[2 * i + 1];
  const double dx = __dsub_rn(px[a], qx[b]);
  const double dy = __dsub_rn(py[a], qy[b]);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= eps_sq;
}

__global__ void k_refine_flag(const i64* __restrict__ cand, i64 n, const double* __restrict__ px,
                              const double* __restrict__ py, const double* __restrict__ qx,
                              const double* __restrict__ qy, double eps_sq,
                              u32* __restrict__ flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    flag[i] = within_eps(cand, i, px, py, qx, qy, eps_sq) ? 1u : 0u;
}

__global__ void k_refine_compact(const i64* __restrict__ cand, i64 n,
                                 const u32* __restrict__ flag, const u64* __restrict__ base,
                                 const i64* __restrict__ p_ids, const i64* __restrict__ q_ids,
                                 i64* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    if (flag[i]) {
      const u64 o = base[i];
      out[2 * o] = p_ids[cand[2 * i]];
      out[2 * o + 1] = q_ids[cand[2 * i + 1]];
    }
  }
}

// ---------------------------------------------------------------- host glue
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

inline bool grid_ok(int kx, int ky, int row_lo, int row_hi) {
  return kx >= 1 && ky >= 1 && kx <= 65535 && ky <= 65535 && row_lo >= 0 && row_lo < row_hi &&
         row_hi <= ky && (u64)kx * (u64)(row_hi - row_lo) < (1ull << 32) - 2;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct ScanLayout {
  size_t cnt, base, partials, total;
  u64 n, nb;
};
inline ScanLayout scan_layout(i64 n) {
  ScanLayout L;
  L.n = (u64)n;
  L.nb = (L.n + kScanTile - 1) / kScanTile;
  size_t o = 0;
  L.cnt = o; o = align_up(o + 4 * (L.n + 1), 256);
  L.base = o; o = align_up(o + 8 * (L.n + 1), 256);
  L.partials = o; o = align_up(o + 8 * (L.nb + 1), 256);
  L.total = o;
  return L;
}

// join scratch: [ticket | status[n_units]]
inline size_t join_scratch(i64 n_units) { return 256 + align_up(8 * (size_t)(n_units + 1), 256); }

int set_smem_attrs() {
  static bool done = false;
  if (done) return 0;
  cudaError_t e;
  e = cudaFuncSetAttribute(k_join<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(JoinSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_join<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(JoinSmem));
  if (e != cudaSuccess) return (int)e;
  done = true;
  return 0;
}

int launch_join(bool emit, void* ws, int kx, int ky, int row_lo, int row_hi,
                const pbsm_entry* r_list, const pbsm_entry* s_list, i64 n_chunks, i64 n_items,
                void* scratch, int64_t* pairs, i64 capacity, cudaStream_t s) {
  int rc = set_smem_attrs();
  if (rc) return rc;
  const WsLayout L = ws_layout(kx, ky, row_lo, row_hi);
  Ws w = ws_bind(ws, L);
  const i64 n_units = n_chunks + n_items;
  // write guard first (reads the cursors the scatter left behind)
  const unsigned gb = (unsigned)std::max<i64>(1, std::min<i64>((i64)((L.tiles + 255) / 256),
                                                                (i64)num_sms() * 8));
  k_guard<<<gb, 256, 0, s>>>(w.cur_r, w.cnt_r, w.cur_s, w.cnt_s, L.tiles, w.hdr);
  cudaMemsetAsync(&w.hdr->pairs, 0, sizeof(int64_t), s);
  if (n_units == 0) return launch_status();
  cudaMemsetAsync(scratch, 0, join_scratch(n_units), s);
  JoinArgs A;
  A.jrec = w.jrec;
  A.cstart = w.cstart;
  A.lrec = w.lrec;
  A.lpre = w.lpre;
  A.rl = reinterpret_cast<const Rec*>(r_list);
  A.sl = reinterpret_cast<const Rec*>(s_list);
  A.ticket = (u32*)scratch;
  A.status = (u64*)((char*)scratch + 256);
  A.pairs = (i64*)pairs;
  A.capacity = capacity;
  A.n_chunks = n_chunks;
  A.n_units = n_units;
  A.hdr = w.hdr;
  if (emit)
    k_join<true><<<(unsigned)n_units, kJoinThreads, sizeof(JoinSmem), s>>>(A);
  else
    k_join<false><<<(unsigned)n_units, kJoinThreads, sizeof(JoinSmem), s>>>(A);
  return launch_status();
}

}  // namespace

// ======================================================================== ABI
extern "C" {

int32_t pbsm_abi_version(void) { return PBSM_ABI_VERSION; }

const char* pbsm_build_info(void) {
  return "pbsm sm_100a v2: count+validate / plan / scatter(64B records, join tiles only) / "
         "guard / fused TMA-staged sort+sweep join with decoupled look-back; "
         "kCap=1024 kLmax=384";
}

int64_t pbsm_workspace_bytes(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi) {
  if (!grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  return (int64_t)ws_layout(kx, ky, row_lo, row_hi).total;
}

int pbsm_init(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  const WsLayout L = ws_layout(kx, ky, row_lo, row_hi);
  Ws w = ws_bind(ws, L);
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(w.hdr, 0, sizeof(pbsm_header), s);
  cudaMemsetAsync(w.cnt_r, 0, 4 * L.tiles, s);
  cudaMemsetAsync(w.cnt_s, 0, 4 * L.tiles, s);
  const int m = std::max(kx, ky) + 1;
  k_bounds<<<(m + 255) / 256, 256, 0, s>>>(w.bx, kx, w.by, ky);
  return launch_status();
}

int pbsm_count(const double* xl, const double* xu, const double* yl, const double* yu, int64_t n,
               int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
               void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1))
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  const i64 per_block = 256 * kRectsPerThread;
  const i64 blocks = std::min<i64>((n + per_block - 1) / per_block, (i64)num_sms() * 8);
  k_count<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(xl, xu, yl, yu, n, kx, ky, row_lo,
                                                           row_hi, w.bx, w.by,
                                                           side ? w.cnt_s : w.cnt_r, side,
                                                           w.hdr);
  return launch_status();
}

int pbsm_plan(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  cudaStream_t s = as_stream(stream);
  k_plan_reduce<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles,
                                                              w.partials, w.hdr);
  k_plan_partials<<<1, 1024, 0, s>>>(w.partials, w.nblocks, w.hdr, w.je, w.lpre, w.cstart);
  k_plan_apply<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles,
                                                             w.nblocks, w.partials, w.cur_r, w.cur_s,
                                                             w.jrec, w.je, w.lrec, w.lpre);
  const i64 blocks = std::min<i64>((i64)((w.tiles + 255) / 256), (i64)num_sms() * 8);
  k_chunks<<<(unsigned)std::max<i64>(blocks, 1), 256, 0, s>>>(w.je, w.cstart, w.hdr);
  return launch_status();
}

int pbsm_read_header(void* ws, pbsm_header* out, void* stream) {
  if (!ws || !out) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(out, ws, sizeof(pbsm_header), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return (int)e;
  e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? 0 : (int)e;
}

int pbsm_scatter(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                 const double* yu, int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky,
                 int32_t row_lo, int32_t row_hi, pbsm_entry* out, int64_t capacity,
                 void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!ids || !xl || !xu || !yl || !yu || (!out && capacity > 0)) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  const i64 per_block = 256 * kRectsPerThread;
  const i64 blocks = std::min<i64>((n + per_block - 1) / per_block, (i64)num_sms() * 8);
  k_scatter<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      (const i64*)ids, xl, xu, yl, yu, n, kx, ky, row_lo, row_hi, w.bx, w.by,
      side ? w.cur_s : w.cur_r, reinterpret_cast<Rec*>(out), capacity, w.hdr);
  return launch_status();
}

int64_t pbsm_join_scratch_bytes(int64_t n_chunks, int64_t n_items) {
  if (n_chunks < 0 || n_items < 0) return PBSM_E_ARG;
  return (int64_t)join_scratch(n_chunks + n_items);
}

int pbsm_join_count(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                    const pbsm_entry* r_list, const pbsm_entry* s_list, int64_t n_chunks,
                    int64_t n_items, void* scratch, void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || n_chunks < 0 || n_items < 0)
    return PBSM_E_ARG;
  return launch_join(false, ws, kx, ky, row_lo, row_hi, r_list, s_list, n_chunks, n_items,
                     scratch, nullptr, 0, as_stream(stream));
}

int pbsm_join_emit(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const pbsm_entry* r_list, const pbsm_entry* s_list, int64_t n_chunks,
                   int64_t n_items, void* scratch, int64_t* pairs, int64_t capacity,
                   void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || n_chunks < 0 || n_items < 0 ||
      capacity < 0 || (capacity > 0 && !pairs))
    return PBSM_E_ARG;
  return launch_join(true, ws, kx, ky, row_lo, row_hi, r_list, s_list, n_chunks, n_items,
                     scratch, pairs, capacity, as_stream(stream));
}

int64_t pbsm_refine_scratch_bytes(int64_t n_cand) {
  if (n_cand < 0) return PBSM_E_ARG;
  return (int64_t)scan_layout(n_cand).total;
}

int64_t pbsm_refine_result_offset(int64_t n_cand) {
  if (n_cand < 0) return PBSM_E_ARG;
  const ScanLayout SL = scan_layout(n_cand);
  return (int64_t)(SL.base + 8 * SL.n);
}

int pbsm_refine(const int64_t* cand, int64_t n_cand, const double* px, const double* py,
                const double* qx, const double* qy, const int64_t* p_ids, const int64_t* q_ids,
                double eps_sq, void* scratch, int64_t* out, void* stream) {
  if (n_cand < 0 || !scratch) return PBSM_E_ARG;
  const ScanLayout SL = scan_layout(n_cand);
  cudaStream_t s = as_stream(stream);
  u64* base = (u64*)((char*)scratch + SL.base);
  if (n_cand == 0) {
    cudaMemsetAsync(base, 0, sizeof(u64), s);
    return launch_status();
  }
  if (!cand || !px || !py || !qx || !qy || !p_ids || !q_ids || !out) return PBSM_E_ARG;
  u32* flag = (u32*)((char*)scratch + SL.cnt);
  u64* part = (u64*)((char*)scratch + SL.partials);
  const unsigned blocks = (unsigned)std::min<i64>((n_cand + 255) / 256, (i64)num_sms() * 16);
  k_refine_flag<<<blocks, 256, 0, s>>>((const i64*)cand, n_cand, px, py, qx, qy, eps_sq, flag);
  k_scan_reduce<<<(unsigned)SL.nb, kScanThreads, 0, s>>>(flag, SL.n, part);
  k_scan_partials<<<1, 1024, 0, s>>>(part, SL.nb, base, SL.n);
  k_scan_apply<<<(unsigned)SL.nb, kScanThreads, 0, s>>>(flag, SL.n, part, base);
  k_refine_compact<<<blocks, 256, 0, s>>>((const i64*)cand, n_cand, flag, base,
                                          (const i64*)p_ids, (const i64*)q_ids, (i64*)out);
  return launch_status();
}

}  // extern "C"
