// pbsm.cu — B200-native (sm_100a) PBSM filter step of arXiv 1908.11740.
//
// Four subsystems replace the reference's per-tile CPU kernels
// (/root/reference/pkg/src/sweepjoin/_kernels.pyx) for ALL tiles at once:
//
//  1. grid partitioning with class A/B/C/D labels
//       k_count    ← count_tiles   (_kernels.pyx:34-58)
//       k_plan_*   ← compute_segment_offsets (partition.py:151-164) and
//                    build_task_queue (engine.py:84-100)
//       k_scatter  ← write_tiles   (_kernels.pyx:61-98)
//  2. per-tile segmented sort by x-lower        ← sort_segment (_kernels.pyx:188-228)
//  3. forward-scan mini-joins over the class combinations
//                                               ← do_sweep (_kernels.pyx:231-293)
//  4. two-pass count → emit pair writer         ← sweep_count / sweep_collect
//                                                 (_kernels.pyx:304-341) and the
//                                                 aggregation (engine.py:293-309)
//  (2)-(4) are fused in k_join_chunk: a CTA stages a chunk of small tiles in
//  shared memory, sorts every (tile, side) segment there and sweeps it.
//  Tiles too large for one CTA's shared memory go to k_join_large.
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

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "../../include/pbsm.h"

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;

namespace {

// ---------------------------------------------------------------- constants
constexpr int kPlanThreads = 256;
constexpr int kPlanPer = 16;                         // tiles per thread
constexpr int kPlanTile = kPlanThreads * kPlanPer;   // 4096 tiles per CTA
constexpr int kNV = 6;                               // plan scan lanes

constexpr int kJoinThreads = 256;
constexpr int kChunkB = 1024;       // chunk bucket width in entries
constexpr int kLmax = 512;          // largest tile (|R_T|+|S_T|) on the chunk path
constexpr int kCap = kChunkB + kLmax;   // max entries staged per chunk CTA
constexpr int kEPT = kCap / kJoinThreads;  // entries per thread in the load
constexpr int kMaxTilesPerChunk = kCap / 2 + 1;
constexpr int kLargeLead = 256;     // lead-side entries per large-tile work item
constexpr int kLargeStage = 1024;   // other-side entries staged per round

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTile = kScanThreads * kScanPer;

constexpr u64 kXOut = 1ull << 63;
constexpr u64 kYOut = 1ull << 62;
constexpr u64 kLabelMask = kXOut | kYOut;

static_assert(kCap % kJoinThreads == 0, "kCap must be a multiple of the CTA size");
static_assert(kLmax <= kChunkB, "a small tile may cross at most one bucket boundary");

// ---------------------------------------------------------------- workspace
struct WsLayout {
  size_t hdr, bx, by, cnt_r, cnt_s, off_r, off_s, jlist, je, cstart, llist, lpre,
      partials, total;
  u64 tiles;
  u64 nblocks;
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

inline WsLayout ws_layout(int kx, int ky, int row_lo, int row_hi) {
  WsLayout L;
  u64 T = (u64)kx * (u64)(row_hi - row_lo);
  L.tiles = T;
  L.nblocks = (T + kPlanTile - 1) / kPlanTile;
  size_t o = 0;
  L.hdr = o; o = align_up(o + sizeof(pbsm_header), 256);
  L.bx = o; o = align_up(o + sizeof(double) * (kx + 1), 256);
  L.by = o; o = align_up(o + sizeof(double) * (ky + 1), 256);
  L.cnt_r = o; o = align_up(o + 4 * T, 256);
  L.cnt_s = o; o = align_up(o + 4 * T, 256);
  L.off_r = o; o = align_up(o + 4 * T, 256);
  L.off_s = o; o = align_up(o + 4 * T, 256);
  L.jlist = o; o = align_up(o + 4 * T, 256);
  L.je = o; o = align_up(o + 4 * (T + 1), 256);
  L.cstart = o; o = align_up(o + 4 * (T + 2), 256);
  L.llist = o; o = align_up(o + 4 * T, 256);
  L.lpre = o; o = align_up(o + 4 * (T + 1), 256);
  L.partials = o; o = align_up(o + sizeof(u64) * kNV * (L.nblocks + 1), 256);
  L.total = o;
  return L;
}

struct Ws {
  pbsm_header* hdr;
  double* bx;
  double* by;
  u32 *cnt_r, *cnt_s, *off_r, *off_s, *jlist, *je, *cstart, *llist, *lpre;
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
  w.off_r = (u32*)(b + L.off_r);
  w.off_s = (u32*)(b + L.off_s);
  w.jlist = (u32*)(b + L.jlist);
  w.je = (u32*)(b + L.je);
  w.cstart = (u32*)(b + L.cstart);
  w.llist = (u32*)(b + L.llist);
  w.lpre = (u32*)(b + L.lpre);
  w.partials = (u64*)(b + L.partials);
  w.tiles = L.tiles;
  w.nblocks = L.nblocks;
  return w;
}

struct __align__(32) Entry {
  u64 xl_key;
  double xu, yl, yu;
};
static_assert(sizeof(Entry) == sizeof(pbsm_entry), "entry layout");

struct __align__(32) Box {
  double xl, xu, yl, yu;
};

// ---------------------------------------------------------------- helpers

// axis_tile_index (geometry.py:87-106) / tile_of (_kernels.pyx:20-31):
// floor(p*k) clamped to [0,k-1], then nudged against the materialised
// boundaries b[i] = i/k so it agrees with boundary comparisons exactly.
__device__ __forceinline__ int tile_of(double p, int k, const double* __restrict__ b) {
  long long i = (long long)__dmul_rn(p, (double)k);
  if (i < 0) i = 0;
  else if (i > k - 1) i = k - 1;
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

__device__ __forceinline__ int upper_bound_u32(const u32* a, int n, u32 v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- init
__global__ void k_bounds(double* bx, int kx, double* by, int ky) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  // tile_boundary (geometry.py:82-84): i / k, correctly rounded
  if (i <= kx) bx[i] = __ddiv_rn((double)i, (double)kx);
  if (i <= ky) by[i] = __ddiv_rn((double)i, (double)ky);
}

// ---------------------------------------------------------------- 1a count
// count_tiles (_kernels.pyx:34-58), all rectangles, one thread per rectangle.
__global__ void __launch_bounds__(256) k_count(const double* __restrict__ xl,
                                               const double* __restrict__ xu,
                                               const double* __restrict__ yl,
                                               const double* __restrict__ yu, i64 n,
                                               int kx, int ky, int row_lo, int row_hi,
                                               const double* __restrict__ bx,
                                               const double* __restrict__ by,
                                               u32* __restrict__ cnt) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const int c0 = tile_of(__ldg(xl + i), kx, bx);
    const int c1 = tile_of(__ldg(xu + i), kx, bx);
    int r0 = tile_of(__ldg(yl + i), ky, by);
    int r1 = tile_of(__ldg(yu + i), ky, by);
    r0 = max(r0, row_lo);
    r1 = min(r1, row_hi - 1);
    for (int row = r0; row <= r1; ++row) {
      u32* base = cnt + (size_t)(row - row_lo) * kx;
      for (int col = c0; col <= c1; ++col) atomicAdd(base + col, 1u);
    }
  }
}

// ---------------------------------------------------------------- 1c scatter
// write_tiles (_kernels.pyx:61-98): copy each rectangle into every tile it
// overlaps, at a cursor that starts at the tile's exclusive offset.  After the
// pass off[t] is the END of tile t; the join kernels check
// end[t] - cnt[t] == end[t-1], the device form of the write guard
// (partition.py:229-233).
__global__ void __launch_bounds__(256) k_scatter(const i64* __restrict__ ids,
                                                 const double* __restrict__ xl,
                                                 const double* __restrict__ xu,
                                                 const double* __restrict__ yl,
                                                 const double* __restrict__ yu, i64 n,
                                                 int kx, int ky, int row_lo, int row_hi,
                                                 const double* __restrict__ bx,
                                                 const double* __restrict__ by,
                                                 u32* __restrict__ cursor,
                                                 Entry* __restrict__ out,
                                                 i64* __restrict__ out_ids, i64 capacity,
                                                 pbsm_header* hdr) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const double a = __ldg(xl + i), b = __ldg(xu + i), c = __ldg(yl + i), d = __ldg(yu + i);
    const i64 id = __ldg(ids + i);
    const int c0 = tile_of(a, kx, bx);
    const int c1 = tile_of(b, kx, bx);
    const int rr0 = tile_of(c, ky, by);
    const int r1 = min(tile_of(d, ky, by), row_hi - 1);
    const int r0 = max(rr0, row_lo);
    const u64 xk = xl_bits(a);
    for (int row = r0; row <= r1; ++row) {
      u32* base = cursor + (size_t)(row - row_lo) * kx;
      const u64 ylab = (row != rr0) ? kYOut : 0ull;
      for (int col = c0; col <= c1; ++col) {
        const u32 pos = atomicAdd(base + col, 1u);
        if ((i64)pos >= capacity) {
          atomicOr(&hdr->error, PBSM_ERR_SCATTER_OVERFLOW);
          continue;
        }
        Entry e;
        e.xl_key = xk | ylab | ((col != c0) ? kXOut : 0ull);
        e.xu = b;
        e.yl = c;
        e.yu = d;
        out[pos] = e;
        out_ids[pos] = id;
      }
    }
  }
}

// ---------------------------------------------------------------- 1b plan
// Per tile t the plan scans six lanes at once:
//   0 |R_T|  1 |S_T|  (→ CSR offsets, compute_segment_offsets partition.py:151-164)
//   2 small-join flag  3 small-join entries   (→ join tile list + chunk buckets)
//   4 large-join flag  5 large-join work items (→ large tile list)
// A join tile has both inputs non-empty (build_task_queue, engine.py:97).
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
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_reduce(const u32* __restrict__ cr,
                                                              const u32* __restrict__ cs,
                                                              u64 T, u64* __restrict__ partials,
                                                              pbsm_header* hdr) {
  __shared__ u64 sh[kPlanThreads / 32][kNV];
  __shared__ u32 shmax[kPlanThreads / 32];
  u64 acc[kNV] = {0, 0, 0, 0, 0, 0};
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
  u64 carry[kNV] = {0, 0, 0, 0, 0, 0};
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
    hdr->join_tiles_all = (i64)(carry[2] + carry[4]);
    hdr->n_chunks = 0;
    if (carry[0] > 0xffffffffull || carry[1] > 0xffffffffull || carry[3] > 0xffffffffull ||
        carry[5] > 0xffffffffull)
      hdr->error |= PBSM_ERR_TOTAL_RANGE;
    je[carry[2]] = (u32)carry[3];      // sentinel: end of the last join tile
    lpre[carry[4]] = (u32)carry[5];    // sentinel: total large work items
    cstart[0] = 0;
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_apply(
    const u32* __restrict__ cr, const u32* __restrict__ cs, u64 T,
    const u64* __restrict__ partials, u32* __restrict__ off_r, u32* __restrict__ off_s,
    u32* __restrict__ jlist, u32* __restrict__ je, u32* __restrict__ llist,
    u32* __restrict__ lpre) {
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
  u64 acc[kNV] = {0, 0, 0, 0, 0, 0};
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
  // (block_excl_scan ends with a barrier, so sa/sb may be overwritten now)
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = base + (u64)threadIdx.x * kPlanPer + i;
    u64 v[kNV];
    tile_vals(a[i], b[i], v);
    sa[threadIdx.x * kPlanPer + i] = (u32)pre[0];
    sb[threadIdx.x * kPlanPer + i] = (u32)pre[1];
    if (t < T) {
      if (v[2]) {
        jlist[pre[2]] = (u32)t;
        je[pre[2]] = (u32)pre[3];
      }
      if (v[4]) {
        llist[pre[4]] = (u32)t;
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
      off_r[t] = sa[i];
      off_s[t] = sb[i];
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
// exclusive scan of u32 counts into u64 bases; base[n] = total → hdr->pairs
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
                                                        u64* __restrict__ out, u64 n,
                                                        pbsm_header* hdr) {
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
  if (threadIdx.x == 0) {
    out[n] = carry;
    if (hdr) hdr->pairs = (i64)carry;
  }
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
  const u32* jlist;
  const u32* je;
  const u32* cstart;
  const u32* llist;
  const u32* lpre;
  const u32* cnt_r;
  const u32* cnt_s;
  const u32* off_r;   // tile END after the scatter
  const u32* off_s;
  const Entry* rl;
  const Entry* sl;
  const i64* rid;
  const i64* sid;
  u32* unit_cnt;       // [n_chunks + n_items]
  const u64* unit_base;
  i64* pairs;
  i64 pair_base;
  i64 capacity;
  i64 n_chunks;
  pbsm_header* hdr;
};

struct ChunkSmem {
  Box sorted[kCap];            // per tile: [R x-in sorted by xl | R x-out | S x-in sorted | S x-out]
  u64 key[kCap];               // label|xl bits as loaded
  i64 ids[kCap];               // ids in sorted order (emit only)
  unsigned short seg[kCap];    // chunk-local tile of each loaded entry
  unsigned char yin[kCap];     // y-in flag in sorted order
  u32 tE[kMaxTilesPerChunk + 1];
  u32 tR[kMaxTilesPerChunk];
  u32 tS[kMaxTilesPerChunk];
  u32 tRs[kMaxTilesPerChunk];
  u32 tSs[kMaxTilesPerChunk];
  unsigned short tNinR[kMaxTilesPerChunk];
  unsigned short tNinS[kMaxTilesPerChunk];
  u64 scan[33];
  int nt, N;
};

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
__device__ __forceinline__ u32 sweep_one(const ChunkSmem& S, int p, int lt, i64* out) {
  const int base = (int)S.tE[lt];
  const int nR = (int)S.tR[lt];
  const int ninR = S.tNinR[lt], ninS = S.tNinS[lt];
  const int q = p - base;
  const Box me = S.sorted[p];
  const bool yme = S.yin[p];
  int k, hi;
  bool lead_r;
  if (q < nR) {
    lead_r = true;
    const int lo = base + nR;
    hi = lo + ninS;
    k = lo;
    if (q < ninR) {
      // upper_bound(S x-in run, r.xl): first s with s.xl > r.xl
      int b = hi;
      while (k < b) {
        const int m = (k + b) >> 1;
        if (S.sorted[m].xl <= me.xl) k = m + 1; else b = m;
      }
    }
  } else {
    lead_r = false;
    const int lo = base;
    hi = lo + ninR;
    k = lo;
    if (q - nR < ninS) {
      // lower_bound(R x-in run, s.xl): first r with r.xl >= s.xl
      int b = hi;
      while (k < b) {
        const int m = (k + b) >> 1;
        if (S.sorted[m].xl < me.xl) k = m + 1; else b = m;
      }
    }
  }
  u32 c = 0;
  for (; k < hi; ++k) {
    const Box o = S.sorted[k];
    if (o.xl > me.xu) break;
    if (me.yl <= o.yu && o.yl <= me.yu && (yme || S.yin[k])) {
      if (EMIT) {
        out[2 * (i64)c] = lead_r ? S.ids[p] : S.ids[k];
        out[2 * (i64)c + 1] = lead_r ? S.ids[k] : S.ids[p];
      }
      ++c;
    }
  }
  return c;
}

template <bool EMIT>
__global__ void __launch_bounds__(kJoinThreads, 2) k_join_chunk(JoinArgs A) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  ChunkSmem& S = *reinterpret_cast<ChunkSmem*>(smem_raw);
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  const u32 j0 = A.cstart[c], j1 = A.cstart[c + 1];
  const int nt = (int)(j1 - j0);
  const u32 e0 = A.je[j0];

  // ---- tile table of the chunk (task list: build_task_queue engine.py:84-100)
  for (int lt = tid; lt < nt; lt += kJoinThreads) {
    const u32 t = A.jlist[j0 + lt];
    const u32 nR = A.cnt_r[t], nS = A.cnt_s[t];
    const u32 endR = A.off_r[t], endS = A.off_s[t];
    const u32 rs = endR - nR, ss = endS - nS;
    const u32 prevR = t == 0 ? 0u : A.off_r[t - 1];
    const u32 prevS = t == 0 ? 0u : A.off_s[t - 1];
    if (rs != prevR || ss != prevS) atomicOr(&A.hdr->error, PBSM_ERR_OFFSET_MISMATCH);
    S.tE[lt] = A.je[j0 + lt] - e0;
    S.tR[lt] = nR;
    S.tS[lt] = nS;
    S.tRs[lt] = rs;
    S.tSs[lt] = ss;
    if (lt == nt - 1) {
      S.tE[nt] = A.je[j0 + lt] - e0 + nR + nS;
      S.N = (int)(A.je[j0 + lt] - e0 + nR + nS);
    }
  }
  __syncthreads();
  const int N = S.N;

  // ---- stage the chunk: one 256-bit load per entry, kept in registers
  Entry ent[kEPT];
  i64 eid[kEPT];
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    const int e = tid + i * kJoinThreads;
    if (e < N) {
      const int lt = upper_bound_u32(S.tE, nt, (u32)e) - 1;
      const int q = e - (int)S.tE[lt];
      const int nR = (int)S.tR[lt];
      if (q < nR) {
        const u32 g = S.tRs[lt] + q;
        ent[i] = A.rl[g];
        if (EMIT) eid[i] = A.rid[g];
      } else {
        const u32 g = S.tSs[lt] + (q - nR);
        ent[i] = A.sl[g];
        if (EMIT) eid[i] = A.sid[g];
      }
      S.key[e] = ent[i].xl_key;
      S.seg[e] = (unsigned short)lt;
    }
  }
  __syncthreads();

  // ---- 2: segmented sort (sort_segment, _kernels.pyx:188-228) by rank
  // counting inside each (tile, side) segment.  x-in entries are ordered by
  // (xl, load position) — a strict total order, so ranks are a permutation;
  // x-out entries keep load order after the x-in run.
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    const int e = tid + i * kJoinThreads;
    if (e < N) {
      const int lt = S.seg[e];
      const int base = (int)S.tE[lt];
      const int nR = (int)S.tR[lt];
      int a, b;
      if (e < base + nR) { a = base; b = base + nR; }
      else { a = base + nR; b = a + (int)S.tS[lt]; }
      const u64 ke = S.key[e];
      const bool in_e = !(ke & kXOut);
      const u64 xe = ke & ~kLabelMask;
      int n_in = 0, less = 0, out_before = 0;
      for (int j = a; j < b; ++j) {
        const u64 kj = S.key[j];
        if (!(kj & kXOut)) {
          ++n_in;
          const u64 xj = kj & ~kLabelMask;
          less += (xj < xe) || (xj == xe && j < e);
        } else {
          out_before += (j < e);
        }
      }
      const int rank = in_e ? less : n_in + out_before;
      const int p = a + rank;
      Box bx;
      bx.xl = __longlong_as_double((long long)xe);
      bx.xu = ent[i].xu;
      bx.yl = ent[i].yl;
      bx.yu = ent[i].yu;
      S.sorted[p] = bx;
      S.yin[p] = (ke & kYOut) ? 0 : 1;
      if (EMIT) S.ids[p] = eid[i];
      if (e == a) {
        if (a == base) S.tNinR[lt] = (unsigned short)n_in;
        else S.tNinS[lt] = (unsigned short)n_in;
      }
    }
  }
  __syncthreads();

  // ---- 3/4: forward-scan mini-joins, count (then emit)
  const int per = (N + kJoinThreads - 1) / kJoinThreads;
  const int p0 = min(N, tid * per), p1 = min(N, p0 + per);
  int lt0 = 0;
  if (p0 < p1) lt0 = upper_bound_u32(S.tE, nt, (u32)p0) - 1;
  u32 cnt = 0;
  {
    int lt = lt0;
    for (int p = p0; p < p1; ++p) {
      while ((u32)p >= S.tE[lt + 1]) ++lt;
      cnt += sweep_one<false>(S, p, lt, nullptr);
    }
  }
  u64 total;
  const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
  if (!EMIT) {
    if (tid == 0) A.unit_cnt[c] = (u32)total;
    return;
  }
  const i64 start = (i64)A.unit_base[c] + (i64)excl;
  if (start + (i64)cnt > A.capacity) {
    if (cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
    return;
  }
  i64* out = A.pairs + 2 * (A.pair_base + start);
  int lt = lt0;
  for (int p = p0; p < p1; ++p) {
    while ((u32)p >= S.tE[lt + 1]) ++lt;
    out += 2 * (i64)sweep_one<true>(S, p, lt, out);
  }
}

// Large join tiles (|R_T|+|S_T| > kLmax): the larger side is split into
// work items of kLargeLead entries, one per thread; the other side streams
// through shared memory.  Every (lead, other) pair is tested with the full
// closed-interval predicate (intersects, geometry.py:59-61) and the class
// rule (>=1 x-in and >=1 y-in ⇔ Eq. 1 owner tile).
struct LargeSmem {
  Entry other[kLargeStage];
  i64 oid[kLargeStage];
  u64 scan[33];
};

template <bool EMIT>
__device__ __forceinline__ u32 large_pass(const LargeSmem& S, int n, bool have, const Entry& me,
                                          bool lead_r, i64 my_id, i64* out) {
  u32 c = 0;
  if (!have) return 0;
  const double mxl = key_x(me.xl_key);
  const bool mxin = !(me.xl_key & kXOut), myin = !(me.xl_key & kYOut);
  for (int k = 0; k < n; ++k) {
    const Entry o = S.other[k];
    const double oxl = key_x(o.xl_key);
    const bool oxin = !(o.xl_key & kXOut), oyin = !(o.xl_key & kYOut);
    if (mxl <= o.xu && oxl <= me.xu && me.yl <= o.yu && o.yl <= me.yu && (mxin || oxin) &&
        (myin || oyin)) {
      if (EMIT) {
        out[2 * (i64)c] = lead_r ? my_id : S.oid[k];
        out[2 * (i64)c + 1] = lead_r ? S.oid[k] : my_id;
      }
      ++c;
    }
  }
  return c;
}

template <bool EMIT>
__global__ void __launch_bounds__(kLargeLead) k_join_large(JoinArgs A) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  LargeSmem& S = *reinterpret_cast<LargeSmem*>(smem_raw);
  const int item = blockIdx.x;
  const int tid = threadIdx.x;
  // item → large tile (binary search over the work-item prefix)
  int lo = 0, hi = (int)A.hdr->n_large;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (A.lpre[m] <= (u32)item) lo = m + 1; else hi = m;
  }
  const int lj = lo - 1;
  const u32 t = A.llist[lj];
  const u32 nR = A.cnt_r[t], nS = A.cnt_s[t];
  const u32 rs = A.off_r[t] - nR, ss = A.off_s[t] - nS;
  if (tid == 0) {
    const u32 prevR = t == 0 ? 0u : A.off_r[t - 1];
    const u32 prevS = t == 0 ? 0u : A.off_s[t - 1];
    if (rs != prevR || ss != prevS) atomicOr(&A.hdr->error, PBSM_ERR_OFFSET_MISMATCH);
  }
  const bool lead_r = nR >= nS;
  const u32 nl = lead_r ? nR : nS, no = lead_r ? nS : nR;
  const Entry* L = lead_r ? A.rl + rs : A.sl + ss;
  const Entry* O = lead_r ? A.sl + ss : A.rl + rs;
  const i64* Lid = lead_r ? A.rid + rs : A.sid + ss;
  const i64* Oid = lead_r ? A.sid + ss : A.rid + rs;
  const u32 a = (u32)(item - (int)A.lpre[lj]) * kLargeLead + tid;
  const bool have = a < nl;
  Entry me;
  i64 my_id = 0;
  if (have) {
    me = L[a];
    if (EMIT) my_id = Lid[a];
  }
  u32 cnt = 0;
  for (u32 ob = 0; ob < no; ob += kLargeStage) {
    const int n = (int)min((u32)kLargeStage, no - ob);
    __syncthreads();
    for (int k = tid; k < n; k += kLargeLead) {
      S.other[k] = O[ob + k];
    }
    __syncthreads();
    cnt += large_pass<false>(S, n, have, me, lead_r, my_id, nullptr);
  }
  u64 total;
  const u64 excl = block_excl_scan<kLargeLead>((u64)cnt, &total, S.scan);
  const i64 unit = A.n_chunks + item;
  if (!EMIT) {
    if (tid == 0) A.unit_cnt[unit] = (u32)total;
    return;
  }
  const i64 start = (i64)A.unit_base[unit] + (i64)excl;
  const bool ok = start + (i64)cnt <= A.capacity;
  if (!ok && cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
  i64* out = A.pairs + 2 * (A.pair_base + start);
  for (u32 ob = 0; ob < no; ob += kLargeStage) {
    const int n = (int)min((u32)kLargeStage, no - ob);
    __syncthreads();
    for (int k = tid; k < n; k += kLargeLead) {
      S.other[k] = O[ob + k];
      S.oid[k] = Oid[ob + k];
    }
    __syncthreads();
    if (ok) out += 2 * (i64)large_pass<true>(S, n, have, me, lead_r, my_id, out);
  }
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

int g_num_sms = 0;
inline int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

struct ScratchLayout {
  size_t cnt, base, partials, total;
  u64 n, nb;
};
inline ScratchLayout scratch_layout(i64 n_chunks, i64 n_items) {
  ScratchLayout L;
  L.n = (u64)(n_chunks + n_items);
  L.nb = (L.n + kScanTile - 1) / kScanTile;
  size_t o = 0;
  L.cnt = o; o = align_up(o + 4 * (L.n + 1), 256);
  L.base = o; o = align_up(o + 8 * (L.n + 1), 256);
  L.partials = o; o = align_up(o + 8 * (L.nb + 1), 256);
  L.total = o;
  return L;
}

bool g_attr_set = false;
int set_smem_attrs() {
  if (g_attr_set) return 0;
  cudaError_t e;
  e = cudaFuncSetAttribute(k_join_chunk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ChunkSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_join_chunk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ChunkSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_join_large<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(LargeSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_join_large<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(LargeSmem));
  if (e != cudaSuccess) return (int)e;
  g_attr_set = true;
  return 0;
}

JoinArgs make_args(const Ws& w, const pbsm_entry* r_list, const pbsm_entry* s_list,
                   i64 n_chunks, const ScratchLayout& SL, void* scratch) {
  JoinArgs A;
  A.jlist = w.jlist;
  A.je = w.je;
  A.cstart = w.cstart;
  A.llist = w.llist;
  A.lpre = w.lpre;
  A.cnt_r = w.cnt_r;
  A.cnt_s = w.cnt_s;
  A.off_r = w.off_r;
  A.off_s = w.off_s;
  A.rl = reinterpret_cast<const Entry*>(r_list);
  A.sl = reinterpret_cast<const Entry*>(s_list);
  A.rid = nullptr;
  A.sid = nullptr;
  A.unit_cnt = (u32*)((char*)scratch + SL.cnt);
  A.unit_base = (const u64*)((char*)scratch + SL.base);
  A.pairs = nullptr;
  A.pair_base = 0;
  A.capacity = 0;
  A.n_chunks = n_chunks;
  A.hdr = w.hdr;
  return A;
}

}  // namespace

// ======================================================================== ABI
extern "C" {

int32_t pbsm_abi_version(void) { return PBSM_ABI_VERSION; }

const char* pbsm_build_info(void) {
  return "pbsm sm_100a: count/plan/scatter + chunk sort-sweep + large nested-loop; "
         "kCap=1536 kLmax=512";
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
  const i64 blocks = std::min<i64>((n + 255) / 256, (i64)num_sms() * 16);
  k_count<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(xl, xu, yl, yu, n, kx, ky, row_lo,
                                                           row_hi, w.bx, w.by,
                                                           side ? w.cnt_s : w.cnt_r);
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
                                                             w.partials, w.off_r, w.off_s,
                                                             w.jlist, w.je, w.llist, w.lpre);
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
                 int32_t row_lo, int32_t row_hi, pbsm_entry* out, int64_t* out_ids,
                 int64_t capacity, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1))
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!ids || !xl || !xu || !yl || !yu || ((!out || !out_ids) && capacity > 0)) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  const i64 blocks = std::min<i64>((n + 255) / 256, (i64)num_sms() * 16);
  k_scatter<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      (const i64*)ids, xl, xu, yl, yu, n, kx, ky, row_lo, row_hi, w.bx, w.by,
      side ? w.off_s : w.off_r, reinterpret_cast<Entry*>(out), (i64*)out_ids, capacity, w.hdr);
  return launch_status();
}

int64_t pbsm_join_scratch_bytes(int64_t n_chunks, int64_t n_items) {
  if (n_chunks < 0 || n_items < 0) return PBSM_E_ARG;
  return (int64_t)scratch_layout(n_chunks, n_items).total;
}

int pbsm_join_count(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                    const pbsm_entry* r_list, const pbsm_entry* s_list, int64_t n_chunks,
                    int64_t n_items, void* scratch, void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || n_chunks < 0 || n_items < 0)
    return PBSM_E_ARG;
  int rc = set_smem_attrs();
  if (rc) return rc;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  const ScratchLayout SL = scratch_layout(n_chunks, n_items);
  cudaStream_t s = as_stream(stream);
  JoinArgs A = make_args(w, r_list, s_list, n_chunks, SL, scratch);
  if (n_chunks > 0)
    k_join_chunk<false><<<(unsigned)n_chunks, kJoinThreads, sizeof(ChunkSmem), s>>>(A);
  if (n_items > 0) {
    k_join_large<false><<<(unsigned)n_items, kLargeLead, sizeof(LargeSmem), s>>>(A);
  }
  const u64 n = SL.n;
  if (n > 0) {
    u32* cnt = (u32*)((char*)scratch + SL.cnt);
    u64* base = (u64*)((char*)scratch + SL.base);
    u64* part = (u64*)((char*)scratch + SL.partials);
    k_scan_reduce<<<(unsigned)SL.nb, kScanThreads, 0, s>>>(cnt, n, part);
    k_scan_partials<<<1, 1024, 0, s>>>(part, SL.nb, base, n, w.hdr);
    k_scan_apply<<<(unsigned)SL.nb, kScanThreads, 0, s>>>(cnt, n, part, base);
  } else {
    cudaMemsetAsync(&w.hdr->pairs, 0, sizeof(int64_t), s);
  }
  return launch_status();
}

int pbsm_join_emit(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const pbsm_entry* r_list, const int64_t* r_ids, const pbsm_entry* s_list,
                   const int64_t* s_ids, int64_t n_chunks, int64_t n_items, const void* scratch,
                   int64_t* pairs, int64_t pair_base, int64_t capacity, void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || n_chunks < 0 || n_items < 0 ||
      pair_base < 0 || capacity < 0)
    return PBSM_E_ARG;
  if (capacity > 0 && !pairs) return PBSM_E_ARG;
  int rc = set_smem_attrs();
  if (rc) return rc;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  const ScratchLayout SL = scratch_layout(n_chunks, n_items);
  cudaStream_t s = as_stream(stream);
  JoinArgs A = make_args(w, r_list, s_list, n_chunks, SL, const_cast<void*>(scratch));
  A.rid = (const i64*)r_ids;
  A.sid = (const i64*)s_ids;
  A.pairs = (i64*)pairs;
  A.pair_base = pair_base;
  A.capacity = capacity;
  if (n_chunks > 0)
    k_join_chunk<true><<<(unsigned)n_chunks, kJoinThreads, sizeof(ChunkSmem), s>>>(A);
  if (n_items > 0) {
    k_join_large<true><<<(unsigned)n_items, kLargeLead, sizeof(LargeSmem), s>>>(A);
  }
  return launch_status();
}

int64_t pbsm_refine_scratch_bytes(int64_t n_cand) {
  if (n_cand < 0) return PBSM_E_ARG;
  return (int64_t)scratch_layout(n_cand, 0).total;
}

int pbsm_refine(const int64_t* cand, int64_t n_cand, const double* px, const double* py,
                const double* qx, const double* qy, const int64_t* p_ids, const int64_t* q_ids,
                double eps_sq, void* scratch, int64_t* out, void* stream) {
  if (n_cand < 0 || !scratch) return PBSM_E_ARG;
  const ScratchLayout SL = scratch_layout(n_cand, 0);
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
  k_scan_partials<<<1, 1024, 0, s>>>(part, SL.nb, base, SL.n, nullptr);
  k_scan_apply<<<(unsigned)SL.nb, kScanThreads, 0, s>>>(flag, SL.n, part, base);
  k_refine_compact<<<blocks, 256, 0, s>>>((const i64*)cand, n_cand, flag, base,
                                          (const i64*)p_ids, (const i64*)q_ids, (i64*)out);
  return launch_status();
}

int64_t pbsm_refine_result_offset(int64_t n_cand) {
  if (n_cand < 0) return PBSM_E_ARG;
  const ScratchLayout SL = scratch_layout(n_cand, 0);
  return (int64_t)(SL.base + 8 * SL.n);
}

}  // extern "C"
