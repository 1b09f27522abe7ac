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
//  (2)-(4) run as per-tile mini-joins chosen by a cost model in the plan:
//       k_join_nested  small tiles (the default for the BASELINE configs): a CTA
//                      stages a chunk of consecutive tiles with cp.async, one
//                      lane per entry of each tile's larger side tests the
//                      other side, hits go to per-warp lists, one atomic
//                      reserves the chunk's output range, then it emits
//       k_join         medium tiles: TMA-staged chunk, per-(tile, side) rank
//                      sort by x-lower + the forward scan (Alg. 1); large
//                      tiles: work items of 256 lead x 2048 other entries
//  The output range is reserved with one atomic per unit (the reference's pair
//  list is unordered) or, in ordered mode, by a decoupled look-back.
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
#ifndef PBSM_PLAN_PER
#define PBSM_PLAN_PER 4
#endif
#ifndef PBSM_PLAN_MINB
#define PBSM_PLAN_MINB 4
#endif
constexpr int kPlanPer = PBSM_PLAN_PER;               // tiles per thread
constexpr int kPlanTile = kPlanThreads * kPlanPer;   // 1024 tiles per CTA
constexpr int kNV = 12;                              // plan scan lanes (see tile_vals)
constexpr int kNTot = kNV;                           // partials row stride

constexpr int kJoinThreads = 256;
#ifndef PBSM_CHUNK_B
#define PBSM_CHUNK_B 256
#endif
#ifndef PBSM_LMAX
#define PBSM_LMAX 128
#endif
#ifndef PBSM_NESTED_MAX
#define PBSM_NESTED_MAX 1024
#endif
constexpr int kChunkB = PBSM_CHUNK_B;   // chunk bucket width in entries
constexpr int kLmax = PBSM_LMAX;        // largest tile (|R_T|+|S_T|) staged by one CTA
constexpr int kNestedMax = PBSM_NESTED_MAX;  // nested strategy iff |R_T|*|S_T| <= this
constexpr int kCap = kChunkB + kLmax;   // max entries staged per chunk CTA
constexpr int kMaxTiles = kCap / 2;     // a join tile holds >= 2 entries
#ifndef PBSM_CHUNK_BN
#define PBSM_CHUNK_BN 384
#endif
constexpr int kChunkBN = PBSM_CHUNK_BN;  // bucket width of the nested chunks
constexpr int kCapN = kChunkBN + kLmax;  // max entries of a nested chunk
#ifndef PBSM_NESTED_THREADS
#define PBSM_NESTED_THREADS 256
#endif
constexpr int kNT = PBSM_NESTED_THREADS;  // threads of a nested-join CTA
#ifndef PBSM_NESTED_ROWS
#define PBSM_NESTED_ROWS 1  // 1: lane per lead entry; 0: pair-flattened lanes
#endif
constexpr int kMaxTilesN = kCapN / 2;
static_assert(kCapN <= 512 && kLmax <= 128, "nested row descriptors: 9-bit positions, 7-bit counts");
constexpr int kLargeLead = kJoinThreads;  // lead-side entries per large work item
#ifndef PBSM_LARGE_OTHER
#define PBSM_LARGE_OTHER 2048
#endif
constexpr int kLargeOther = PBSM_LARGE_OTHER;  // other-side entries per large work item

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTile = kScanThreads * kScanPer;

#ifndef PBSM_BIN_DIRECT
#define PBSM_BIN_DIRECT 0
#endif
#ifndef PBSM_REC_HINT  // record stores: 1 L2 evict_first policy, 0 plain, 2 st.cs
#define PBSM_REC_HINT 1
#endif
#ifndef PBSM_PART_MINB
#define PBSM_PART_MINB 4
#endif
#ifndef PBSM_BINS
#define PBSM_BINS 256
#endif
constexpr int kBins = PBSM_BINS;                  // row bands of the binned scatter
constexpr int kBinSlots = kBins + 1;        // + one slot for rectangles outside the strip
#ifndef PBSM_MAX_PART_BLOCKS
#define PBSM_MAX_PART_BLOCKS 16384
#endif
constexpr int kMaxPartBlocks = PBSM_MAX_PART_BLOCKS;  // grid cap of the count / bin passes
#ifndef PBSM_BIN_TILE
#define PBSM_BIN_TILE 1024
#endif
constexpr int kBinTile = PBSM_BIN_TILE;              // rectangles staged per bin-copy step

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
static_assert(sizeof(pbsm_header) % 4 == 0 && sizeof(pbsm_header) <= 256 * 4, "header reset");
static_assert(sizeof(Rec) == sizeof(pbsm_entry), "entry layout");

struct __align__(32) Half {  // the MBR half of a record: one sector
  u64 xl_key;
  double xu, yl, yu;
};

// ---------------------------------------------------------------- workspace
struct WsLayout {
  size_t hdr, bx, by, cnt_r, cnt_s, cur_r, cur_s, jrec[2], cdesc[2], lrec, lpre,
      partials, bc[2], bo, bscan, total;
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
  for (int q = 0; q < 2; ++q) {  // 0 = nested tiles, 1 = sorted tiles
    L.jrec[q] = o; o = align_up(o + 16 * T, 256);
    L.cdesc[q] = o; o = align_up(o + 16 * (T + 2), 256);
  }
  L.lrec = o; o = align_up(o + 16 * T, 256);
  L.lpre = o; o = align_up(o + 4 * (T + 1), 256);
  L.partials = o; o = align_up(o + sizeof(u64) * kNTot * (L.nblocks + 1), 256);
  for (int q = 0; q < 2; ++q) {  // per-(band, block) rectangle counts of each input
    L.bc[q] = o; o = align_up(o + 4 * (size_t)kBinSlots * kMaxPartBlocks, 256);
  }
  L.bo = o; o = align_up(o + 8 * ((size_t)kBinSlots * kMaxPartBlocks + 1), 256);
  L.bscan = o; o = align_up(o + 8 * (((size_t)kBinSlots * kMaxPartBlocks) / 4096 + 2), 256);
  L.total = o;
  return L;
}

struct Ws {
  pbsm_header* hdr;
  double* bx;
  double* by;
  u32 *cnt_r, *cnt_s, *cur_r, *cur_s, *lpre;
  uint4* cdesc[2];  // chunk c: {first tile j0, r_start, s_start, -}; [n_chunks] = ends
  uint4* jrec[2];   // {r_start, s_start, nR, nS}
  uint4* lrec;
  u64* partials;
  u32* bc[2];
  u64* bo;
  u64* bscan;
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
  for (int q = 0; q < 2; ++q) {
    w.jrec[q] = (uint4*)(b + L.jrec[q]);
    w.cdesc[q] = (uint4*)(b + L.cdesc[q]);
  }
  w.lrec = (uint4*)(b + L.lrec);
  w.lpre = (u32*)(b + L.lpre);
  w.partials = (u64*)(b + L.partials);
  for (int q = 0; q < 2; ++q) w.bc[q] = (u32*)(b + L.bc[q]);
  w.bo = (u64*)(b + L.bo);
  w.bscan = (u64*)(b + L.bscan);
  w.tiles = L.tiles;
  w.nblocks = L.nblocks;
  return w;
}

// ---------------------------------------------------------------- helpers

// axis_tile_index (geometry.py:87-106) / tile_of (_kernels.pyx:20-31):
// floor(p*k) clamped to [0,k-1], then nudged against the materialised
// boundaries b[i] = i/k so it agrees with boundary comparisons exactly.
//
// Fast path (no table access): f = fl(p*k) is within 2^-53*k < 7.3e-12 of
// p*k for k <= 65535, and fl(i/k) within 1.2e-16 of i/k.  So when f is more
// than 1e-9 away from the nearest integer, p is at least ~1.5e-14 away from
// both boundaries of division floor(f): the nudge loops would not move, and
// floor(f) is the exact answer.  Otherwise — p within ~1e-9/k of a boundary,
// or p = 1.0 — the reference's loop runs on the table.
__device__ __forceinline__ int tile_of(double p, int k, const double* __restrict__ b) {
  const double f = __dmul_rn(p, (double)k);
  // round f to the nearest integer without a conversion instruction: adding
  // 1.5*2^52 leaves round(f) in the low mantissa bits (|f| < 2^31 here)
  const double kMagic = 6755399441055744.0;
  const double t = __dadd_rn(f, kMagic);
  const double r = __dsub_rn(t, kMagic);
  const double dlt = __dsub_rn(f, r);  // f - round(f), exact
  const int ri = (int)__double2loint(t);
  const int i0 = ri - (dlt < 0.0 ? 1 : 0);  // floor(f)
  if (fabs(dlt) > 1e-9 && i0 >= 0 && i0 < k) return i0;
  // clipped coordinates sit exactly on the domain edges (0.0 / 1.0) and are
  // common (clipped clusters): the reference loop settles at 0 for p <= 0
  // and at k-1 for p >= 1 (b[1] = 1/k > 0, b[k-1] < 1)
  if (p <= 0.0) return 0;
  if (p >= 1.0) return k - 1;
  long long i = (long long)f;
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


// Block-wide exclusive scan of NV u64 lanes at once (two barriers for all
// lanes).  v[] is replaced by the exclusive prefixes, tot[] gets the sums.
template <int NT, int NV, typename T>
__device__ __forceinline__ void block_excl_scan_multi(T v[NV], T tot[NV],
                                                      T (*sh)[NV] /* [NT/32] */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    inc[q] = warp_incl_scan<T>(v[q]);
    if (lane == 31) sh[wid][q] = inc[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    T before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      const T x = sh[w][q];
      before += w < wid ? x : (T)0;
      all += x;
    }
    v[q] = inc[q] - v[q] + before;
    tot[q] = all;
  }
  __syncthreads();
}

// 32-bit variant (one shuffle per step instead of two)
template <int NT>
__device__ __forceinline__ u32 block_excl_scan32(u32 v, u32* total, u32* sh /* >= NT/32+1 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 inc = warp_incl_scan<u32>(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const u32 s = lane < NT / 32 ? sh[lane] : 0u;
    const u32 si = warp_incl_scan<u32>(s);
    if (lane < NT / 32) sh[lane] = si - s;
    if (lane == NT / 32 - 1) sh[NT / 32] = si;
  }
  __syncthreads();
  const u32 r = inc - v + sh[wid];
  *total = sh[NT / 32];
  return r;  // (callers sync before sh is reused)
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
// One launch for the whole per-join reset (a memset per buffer cost a host
// API call each while the GPU sat idle at the start of the join): zero the
// header and both inputs' per-tile counters, build the boundary tables.
__global__ void k_init(pbsm_header* hdr, u32* cnt_r, u32* cnt_s, u64 T, double* bx, int kx,
                       double* by, int ky) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 nt = (u64)gridDim.x * blockDim.x;
  if (tid < sizeof(pbsm_header) / 4) reinterpret_cast<u32*>(hdr)[tid] = 0u;
  // tile_boundary (geometry.py:82-84): i / k, correctly rounded
  for (u64 i = tid; i <= (u64)max(kx, ky); i += nt) {
    if (i <= (u64)kx) bx[i] = __ddiv_rn((double)i, (double)kx);
    if (i <= (u64)ky) by[i] = __ddiv_rn((double)i, (double)ky);
  }
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  const u64 nv = T / 4;  // the counter arrays are 256-byte aligned
  for (u64 i = tid; i < nv; i += nt) {
    reinterpret_cast<uint4*>(cnt_r)[i] = z;
    reinterpret_cast<uint4*>(cnt_s)[i] = z;
  }
  for (u64 i = 4 * nv + tid; i < T; i += nt) {
    cnt_r[i] = 0u;
    cnt_s[i] = 0u;
  }
}

// ---------------------------------------------------------------- 1a count
// count_tiles (_kernels.pyx:34-58) for all rectangles, one per thread and
// loop step with the next one prefetched; block b takes a contiguous input
// range and also counts its rectangles per row band (binned scatter, below).
// The same pass applies
// RectBatch.validate (geometry.py:166-177): inverted or out-of-[0,1]
// rectangles raise error bits the host turns into the reference's ValueError.
// one rectangle of the row-band copy: 40 bytes, so a band run of a few
// rectangles covers whole sectors (five separate 8-byte columns would write
// partial sectors at every run)
struct BRec {
  i64 id;
  double xl, xu, yl, yu;
};
static_assert(sizeof(BRec) == 40, "band record");

// band of a rectangle in the binned scatter: its first tile row inside the
// strip, in kBins equal row bands; rectangles that miss the strip → kBins.
// Any monotone map into [0, kBins) works as long as the count and bin passes
// agree, so a float multiply replaces the 64-bit division (which cost ~10% of
// k_count's instructions).
__device__ __forceinline__ int band_of(int r0, int r1, int row_lo, int row_hi) {
  if (r0 > r1) return kBins;
  const float scale = (float)kBins / (float)(row_hi - row_lo);
  return min((int)((float)(r0 - row_lo) * scale), kBins - 1);
}

// the contiguous input range of block b in the count and bin passes
__device__ __forceinline__ void part_range(i64 n, i64& beg, i64& end) {
  const i64 per = (n + gridDim.x - 1) / gridDim.x;
  beg = min(n, (i64)blockIdx.x * per);
  end = min(n, beg + per);
}


// ---- cp.async (16/8-byte async global → shared copies)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Per-tile counter / cursor atomics, tagged with an L2 evict_last policy so
// the counter lines outlive the streamed input and record lines around them
// (measured: cfg2 scatter 585 -> 550 µs, cfg4 count 1.41 -> 1.31 ms;
// PBSM_ATOM_HINT=0 gives plain atomics).
#ifndef PBSM_ATOM_HINT
#define PBSM_ATOM_HINT 1
#endif
__device__ __forceinline__ void cnt_inc(u32* p) {
#if PBSM_ATOM_HINT
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.global.add.L2::cache_hint.u32 [%0], 1, %1;" ::"l"(p), "l"(pol) : "memory");
#else
  atomicAdd(p, 1u);
#endif
}
__device__ __forceinline__ u32 cur_inc(u32* p) {
#if PBSM_ATOM_HINT
  u64 pol;
  u32 old;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], 1, %2;"
               : "=r"(old) : "l"(p), "l"(pol) : "memory");
  return old;
#else
  return atomicAdd(p, 1u);
#endif
}

__global__ void __launch_bounds__(256, PBSM_PART_MINB) k_count(const double* __restrict__ xl,
                                               const double* __restrict__ xu,
                                               const double* __restrict__ yl,
                                               const double* __restrict__ yu, i64 n,
                                               int kx, int ky, int row_lo, int row_hi,
                                               const double* __restrict__ bx,
                                               const double* __restrict__ by,
                                               u32* __restrict__ cnt, int side,
                                               u32* __restrict__ band_cnt,
                                               pbsm_header* hdr) {
  __shared__ u32 hist[kBinSlots];
  for (int g = threadIdx.x; g < kBinSlots; g += blockDim.x) hist[g] = 0;
  __syncthreads();
  i64 beg, end;
  part_range(n, beg, end);
  i64 i = beg + threadIdx.x;
  u32 bad = 0;
  // software pipeline: the next rectangle's loads are in flight while this
  // one is binned (streamed once: evict-first keeps the counters in L2)
  double a = 0, b = 0, c = 0, d = 0;
  if (i < end) {
    a = __ldcs(xl + i);
    b = __ldcs(xu + i);
    c = __ldcs(yl + i);
    d = __ldcs(yu + i);
  }
  for (; i < end; i += blockDim.x) {
    const i64 nx = i + blockDim.x;
    double na = 0, nb = 0, nc = 0, nd = 0;
    if (nx < end) {
      na = __ldcs(xl + nx);
      nb = __ldcs(xu + nx);
      nc = __ldcs(yl + nx);
      nd = __ldcs(yu + nx);
    }
    if (!(a <= b) || !(c <= d)) bad |= PBSM_ERR_INVERTED;
    if (a < 0.0 || c < 0.0 || b > 1.0 || d > 1.0) bad |= PBSM_ERR_RANGE;
    const int c0 = tile_of(a, kx, bx);
    const int c1 = tile_of(b, kx, bx);
    const int r0 = max(tile_of(c, ky, by), row_lo);
    const int r1 = min(tile_of(d, ky, by), row_hi - 1);
    atomicAdd_block(&hist[band_of(r0, r1, row_lo, row_hi)], 1u);
    u32* t00 = cnt + (size_t)(r0 - row_lo) * kx + c0;
    const int ec = c1 - c0, er = r1 - r0;  // extents - 1 (er < 0: outside the strip)
    if ((ec | er) == 0) {
      cnt_inc(t00);
    } else if (ec <= 1 && er <= 1 && er >= 0) {  // 2 or 4 tiles, no loop
      cnt_inc(t00);
      if (ec) cnt_inc(t00 + 1);
      if (er) cnt_inc(t00 + kx);
      if (ec & er) cnt_inc(t00 + kx + 1);
    } else {
      for (int row = r0; row <= r1; ++row) {
        u32* rowp = cnt + (size_t)(row - row_lo) * kx;
        for (int col = c0; col <= c1; ++col) cnt_inc(rowp + col);
      }
    }
    a = na;
    b = nb;
    c = nc;
    d = nd;
  }
  if (bad) atomicOr(&hdr->error, bad << (2 * side));
  __syncthreads();
  // band-major: all blocks' counts of band 0, then band 1, ...
  for (int g = threadIdx.x; g < kBinSlots; g += blockDim.x)
    band_cnt[(size_t)g * gridDim.x + blockIdx.x] = hist[g];
}

// Binned scatter, step 1 (only for inputs whose tile lists are large): copy
// the rectangles into row-band order.  Block b re-reads its range of the count
// pass in steps of kBinTile rectangles, counting-sorts each step by band in
// shared memory and writes every band run contiguously at that band's next
// slot for this block (band-major prefix of the count pass' band counts).
// The scatter then reads this copy, so at any moment the GPU writes the tile
// lists of one or two bands — a window that stays in L2 — instead of
// scattering 64-byte records over the whole list.
__global__ void __launch_bounds__(256) k_bin_copy(const i64* __restrict__ ids,
                                                  const double* __restrict__ xl,
                                                  const double* __restrict__ xu,
                                                  const double* __restrict__ yl,
                                                  const double* __restrict__ yu, i64 n,
                                                  int ky, int row_lo, int row_hi,
                                                  const double* __restrict__ by,
                                                  const u64* __restrict__ band_off,
                                                  BRec* __restrict__ out) {
  constexpr int kPer = kBinTile / 256;
  __shared__ u32 cursor[kBinSlots];
  __shared__ u32 hist[kBinSlots];
#if !PBSM_BIN_DIRECT
  __shared__ u32 start[kBinSlots + 1];
#endif
#if !PBSM_BIN_DIRECT
  __shared__ i64 s_id[kBinTile];
  __shared__ double s_xl[kBinTile], s_xu[kBinTile], s_yl[kBinTile], s_yu[kBinTile];
  __shared__ u16 s_band[kBinTile];
  __shared__ u64 scan_sh[256 / 32 + 1];
#endif
  for (int g = threadIdx.x; g < kBinSlots; g += blockDim.x)
    cursor[g] = (u32)band_off[(size_t)g * gridDim.x + blockIdx.x];
  i64 beg, end;
  part_range(n, beg, end);
  for (i64 t0 = beg; t0 < end; t0 += kBinTile) {
    for (int g = threadIdx.x; g < kBinSlots; g += blockDim.x) hist[g] = 0;
    __syncthreads();
    i64 id[kPer];
    double a[kPer], b[kPer], c[kPer], d[kPer];
    int band[kPer];
    u32 rank[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const i64 i = t0 + threadIdx.x + u * 256;
      band[u] = -1;
      if (i < end) {
        id[u] = ids ? __ldcs(ids + i) : i;
        a[u] = __ldcs(xl + i);
        b[u] = __ldcs(xu + i);
        c[u] = __ldcs(yl + i);
        d[u] = __ldcs(yu + i);
        const int r0 = max(tile_of(c[u], ky, by), row_lo);
        const int r1 = min(tile_of(d[u], ky, by), row_hi - 1);
        band[u] = band_of(r0, r1, row_lo, row_hi);
        rank[u] = atomicAdd_block(&hist[band[u]], 1u);
      }
    }
    __syncthreads();
#if PBSM_BIN_DIRECT
    // each record straight to its band's frontier for this block; the
    // frontier lines (kBinSlots per block) stay in L2 and merge there
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (band[u] < 0) continue;
      BRec r;
      r.id = id[u];
      r.xl = a[u];
      r.xu = b[u];
      r.yl = c[u];
      r.yu = d[u];
      out[cursor[band[u]] + rank[u]] = r;
    }
    __syncthreads();
#else
    // exclusive scan of the step's band histogram (kBinSlots <= 2 per thread)
    {
      const int g0 = 2 * threadIdx.x;
      const u32 h0 = g0 < kBinSlots ? hist[g0] : 0u, h1 = g0 + 1 < kBinSlots ? hist[g0 + 1] : 0u;
      u64 tot;
      const u32 ex = (u32)block_excl_scan<256>((u64)(h0 + h1), &tot, scan_sh);
      if (g0 < kBinSlots) start[g0] = ex;
      if (g0 + 1 < kBinSlots) start[g0 + 1] = ex + h0;
      if (threadIdx.x == 0) start[kBinSlots] = (u32)tot;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (band[u] < 0) continue;
      const u32 p = start[band[u]] + rank[u];
      s_id[p] = id[u];
      s_xl[p] = a[u];
      s_xu[p] = b[u];
      s_yl[p] = c[u];
      s_yu[p] = d[u];
      s_band[p] = (u16)band[u];
    }
    __syncthreads();
    // band runs out, consecutive threads → consecutive slots of a run
    const int m = (int)start[kBinSlots];
    for (int e = threadIdx.x; e < m; e += 256) {
      const int g = s_band[e];
      const u32 dst = cursor[g] + (u32)(e - (int)start[g]);
      BRec r;
      r.id = s_id[e];
      r.xl = s_xl[e];
      r.xu = s_xu[e];
      r.yl = s_yl[e];
      r.yu = s_yu[e];
      out[dst] = r;
    }
    __syncthreads();
#endif
    for (int g = threadIdx.x; g < kBinSlots; g += blockDim.x) cursor[g] += hist[g];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- 1c scatter
// one 64-byte record = two full 32-byte sectors (no read-modify-write), stored
// as 256-bit writes with an L2 evict-first policy so the streaming record
// writes do not push the cursor array out of L2
__device__ __forceinline__ u64 l2_evict_first_policy() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void st256_hint(void* p, u64 a, u64 b, u64 c, u64 d, u64 pol) {
#if PBSM_REC_HINT == 1
  asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "l"(a),
               "l"(b), "l"(c), "l"(d), "l"(pol)
               : "memory");
#elif PBSM_REC_HINT == 2
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c),
               "l"(d)
               : "memory");
#else
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c),
               "l"(d)
               : "memory");
#endif
}

__device__ __forceinline__ void write_rec(Rec* r, u64 key, double xu, double yl, double yu,
                                          i64 id, u64 pol) {
  st256_hint(r, key, (u64)__double_as_longlong(xu), (u64)__double_as_longlong(yl),
             (u64)__double_as_longlong(yu), pol);
  st256_hint(&r->id, (u64)id, 0ull, 0ull, 0ull, pol);
}

// write_tiles (_kernels.pyx:61-98): copy each rectangle into every tile it
// overlaps, labelled with its class there.  Only tiles where both inputs are
// non-empty get a list (the others cannot produce a pair: build_task_queue
// joins only those, engine.py:97); their cursors start at kSkip and the write
// is skipped, but the cursor still advances so k_guard can check every tile.
// Input of the scatter: the caller's SoA columns, or the row-band copy.
struct ScatterIn {
  const i64* ids;
  const double *xl, *xu, *yl, *yu;
  const BRec* band;  // non-null: read the row-band copy instead
  template <bool BANDED>
  __device__ __forceinline__ void load(i64 i, double& a, double& b, double& c, double& d,
                                       i64& id) const {
    if (BANDED) {
      const BRec* r = band + i;
      id = __ldcs(&r->id);
      a = __ldcs(&r->xl);
      b = __ldcs(&r->xu);
      c = __ldcs(&r->yl);
      d = __ldcs(&r->yu);
    } else {
      id = ids ? __ldcs(ids + i) : i;  // no id column: the row index (see pbsm_map_ids)
      a = __ldcs(xl + i);
      b = __ldcs(xu + i);
      c = __ldcs(yl + i);
      d = __ldcs(yu + i);
    }
  }
};

// 5 resident CTAs per SM measured best for the SoA input (cfg3: 4.77 vs 4.91
// ms at 4), 4 for the 40-byte band records (cfg4: 6.65 vs 7.02 ms at 5)
template <bool BANDED>
#ifndef PBSM_SCAT_MINB
#define PBSM_SCAT_MINB 5
#endif
__global__ void __launch_bounds__(256, BANDED ? 4 : PBSM_SCAT_MINB) k_scatter(ScatterIn in, i64 n,
                                                 int kx, int ky, int row_lo, int row_hi,
                                                 const double* __restrict__ bx,
                                                 const double* __restrict__ by,
                                                 u32* __restrict__ cursor, Rec* __restrict__ out,
                                                 i64 capacity, pbsm_header* hdr) {
  u32 bad = 0;
  const u64 pol = l2_evict_first_policy();
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  double pa = 0, pb = 0, pc = 0, pd = 0;
  i64 pid = 0;
  if (i < n) in.load<BANDED>(i, pa, pb, pc, pd, pid);  // software pipeline: next one in flight
  for (; i < n; i += stride) {
    const double a = pa, b = pb, c = pc, d = pd;
    const i64 id = pid;
    if (i + stride < n) in.load<BANDED>(i + stride, pa, pb, pc, pd, pid);
    const int c0 = tile_of(a, kx, bx);
    const int c1 = tile_of(b, kx, bx);
    const int rr0 = tile_of(c, ky, by);
    const int r0 = max(rr0, row_lo);
    const int r1 = min(tile_of(d, ky, by), row_hi - 1);
    if (r0 > r1) continue;  // entirely outside this strip
    const u64 xk = xl_bits(a);
    const int nc = c1 - c0 + 1, nr = r1 - r0 + 1;
    if (nc * nr == 1) {  // one tile: most rectangles
      const u32 p = cur_inc(cursor + (size_t)(r0 - row_lo) * kx + c0);
      if (p < kSkip) {
        if ((i64)p < capacity) write_rec(out + p, xk | ((r0 != rr0) ? kYOut : 0ull), b, c, d, id, pol);
        else bad |= PBSM_ERR_SCATTER_OVERFLOW;
      }
      continue;
    }
    if (nc <= 2 && nr <= 2) {
      // 2 or 4 tiles: their cursor atomics back to back (no branches in
      // between) so the latencies overlap, then the record writes
      u32* t00 = cursor + (size_t)(r0 - row_lo) * kx + c0;
      u32* t01 = nc == 2 ? t00 + 1 : t00 + kx;   // second tile: right, or above
      u32 pos[4];
      int rows[4], cols[4];
      rows[0] = r0;
      cols[0] = c0;
      rows[1] = nc == 2 ? r0 : r0 + 1;
      cols[1] = nc == 2 ? c0 + 1 : c0;
      int ns = 2;
      if (nc == 2 && nr == 2) {
        ns = 4;
        pos[0] = cur_inc(t00);
        pos[1] = cur_inc(t00 + 1);
        pos[2] = cur_inc(t00 + kx);
        pos[3] = cur_inc(t00 + kx + 1);
        rows[2] = rows[3] = r0 + 1;
        cols[2] = c0;
        cols[3] = c0 + 1;
      } else {
        pos[0] = cur_inc(t00);
        pos[1] = cur_inc(t01);
        pos[2] = pos[3] = kSkip;
        rows[2] = rows[3] = cols[2] = cols[3] = 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q >= ns || pos[q] >= kSkip) continue;  // absent / not a join tile
        if ((i64)pos[q] >= capacity) {
          bad |= PBSM_ERR_SCATTER_OVERFLOW;
          continue;
        }
        const u64 key = xk | ((rows[q] != rr0) ? kYOut : 0ull) | ((cols[q] != c0) ? kXOut : 0ull);
        write_rec(out + pos[q], key, b, c, d, id, pol);
      }
      continue;
    }
    for (int row = r0; row <= r1; ++row) {
      u32* rowp = cursor + (size_t)(row - row_lo) * kx;
      const u64 ylab = (row != rr0) ? kYOut : 0ull;
      for (int col = c0; col <= c1; ++col) {
        const u32 p = cur_inc(rowp + col);
        if (p >= kSkip) continue;  // not a join tile
        if ((i64)p >= capacity) {
          bad |= PBSM_ERR_SCATTER_OVERFLOW;
          continue;
        }
        write_rec(out + p, xk | ylab | ((col != c0) ? kXOut : 0ull), b, c, d, id, pol);
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
// Per tile t the plan scans twelve lanes at once (one exclusive scan each):
//   0 |R_T|  1 |S_T|                          all tiles (A_R, A_S totals)
//   2..4   nested tiles: flag, |R_T|, |S_T|
//   5..7   sorted tiles: flag, |R_T|, |S_T|
//   8..11  large tiles:  flag, work items, |R_T|, |S_T|
// A join tile has both inputs non-empty (build_task_queue, engine.py:97);
// its strategy comes from the cost model in include/pbsm.h.  The |R_T| /
// |S_T| lanes of the three strategies give the tile-list offsets
// (compute_segment_offsets, partition.py:151-164): each input's list holds
// the nested tiles, then the sorted tiles, then the large tiles, each region
// in tile order — so a chunk of consecutive nested (or sorted) tiles is one
// contiguous range per input, fetched by one bulk async copy.  Within a CTA the
// lanes are u32 (a CTA's sums never exceed the u32-checked totals); the
// per-CTA partial sums are u64.
enum TileKind { kNone = 0, kNested = 1, kSorted = 2, kLarge = 3 };
enum Lane { L_A, L_B, L_NF, L_NA, L_NB, L_SF, L_SA, L_SB, L_LF, L_LI, L_LA, L_LB };

__device__ __forceinline__ int tile_kind(u32 a, u32 b, i64 nested_max) {
  if (a == 0u || b == 0u) return kNone;
  if (a + b > (u32)kLmax) return kLarge;
  return (i64)((u64)a * (u64)b) <= nested_max ? kNested : kSorted;
}

__device__ __forceinline__ void tile_vals(u32 a, u32 b, i64 nm, u32 v[kNV]) {
  const int kind = tile_kind(a, b, nm);
  const u32 lead = a >= b ? a : b, other = a >= b ? b : a;
#pragma unroll
  for (int q = 0; q < kNV; ++q) v[q] = 0;
  v[L_A] = a;
  v[L_B] = b;
  if (kind == kNested) {
    v[L_NF] = 1;
    v[L_NA] = a;
    v[L_NB] = b;
  } else if (kind == kSorted) {
    v[L_SF] = 1;
    v[L_SA] = a;
    v[L_SB] = b;
  } else if (kind == kLarge) {
    v[L_LF] = 1;
    v[L_LI] = ((lead + kLargeLead - 1) / kLargeLead) * ((other + kLargeOther - 1) / kLargeOther);
    v[L_LA] = a;
    v[L_LB] = b;
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_reduce(const u32* __restrict__ cr,
                                                              const u32* __restrict__ cs,
                                                              u64 T, i64 nm,
                                                              u64* __restrict__ partials,
                                                              pbsm_header* hdr) {
  __shared__ u32 sh[kPlanThreads / 32][kNV];
  __shared__ u32 shmax[kPlanThreads / 32];
  __shared__ u64 shb[kPlanThreads / 32];
  u32 acc[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) acc[q] = 0;
  u32 mx = 0;
  u64 bound = 0;
  const u64 base = (u64)blockIdx.x * kPlanTile;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = base + (u64)i * kPlanThreads + threadIdx.x;
    const u32 a = t < T ? cr[t] : 0u, b = t < T ? cs[t] : 0u;
    u32 v[kNV];
    tile_vals(a, b, nm, v);
#pragma unroll
    for (int q = 0; q < kNV; ++q) acc[q] += v[q];
    if (a && b) {
      mx = max(mx, a + b);
      bound += (u64)a * (u64)b;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kNV; ++q) {
    u32 v = acc[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[wid][q] = v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
    bound += __shfl_down_sync(0xffffffffu, bound, o);
  }
  if (lane == 0) {
    shmax[wid] = mx;
    shb[wid] = bound;
  }
  __syncthreads();
  if (threadIdx.x < kNV) {
    u64 s = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) s += sh[w][threadIdx.x];
    partials[(u64)threadIdx.x * (gridDim.x + 1) + blockIdx.x] = s;
  }
  if (threadIdx.x == 0) {
    u32 m = 0;
    u64 bs = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) {
      m = max(m, shmax[w]);
      bs += shb[w];
    }
    if (m) atomicMax((unsigned long long*)&hdr->max_tile, (unsigned long long)m);
    if (bs) atomicAdd((unsigned long long*)&hdr->pair_bound, (unsigned long long)bs);
  }
}

// one CTA per scan lane: exclusive scan of lane q's per-CTA partial sums (a
// lane-major row, so loads and stores are coalesced; 4 consecutive values per
// thread, 4096 per block-scan step).  The lane total goes after the row (read
// by k_plan_apply); the last CTA to finish writes the header.
constexpr int kPartThreads = 1024;
__global__ void __launch_bounds__(kPartThreads) k_plan_partials(u64* __restrict__ partials, u64 nb,
                                                                 pbsm_header* hdr, uint4* cd_n,
                                                                 uint4* cd_s, u32* lpre) {
  __shared__ u64 sh[kPartThreads / 32 + 1];
  __shared__ bool last;
  u64* row = partials + (u64)blockIdx.x * (nb + 1);
  u64 carry = 0;
  for (u64 base = 0; base < nb; base += 4 * kPartThreads) {
    const u64 i0 = base + 4 * (u64)threadIdx.x;
    u64 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u < nb ? row[i0 + u] : 0ull;
    u64 tot;
    u64 run = carry + block_excl_scan<kPartThreads>(v[0] + v[1] + v[2] + v[3], &tot, sh);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u < nb) row[i0 + u] = run;
      run += v[u];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    row[nb] = carry;
    __threadfence();
    last = atomicAdd(&hdr->pad, 1u) == (u32)(kNV - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  hdr->pad = 0;  // the lane counter, ready for the next plan
  {
    u64 c[kNV];
    for (int qq = 0; qq < kNV; ++qq) c[qq] = __ldcg(partials + (u64)qq * (nb + 1) + nb);
    hdr->a_r = (i64)c[L_A];
    hdr->a_s = (i64)c[L_B];
    hdr->n_nested = (i64)c[L_NF];
    hdr->w_nested = (i64)(c[L_NA] + c[L_NB]);
    hdr->n_sorted = (i64)c[L_SF];
    hdr->w_sorted = (i64)(c[L_SA] + c[L_SB]);
    hdr->n_large = (i64)c[L_LF];
    hdr->n_items = (i64)c[L_LI];
    const u64 lr = c[L_NA] + c[L_SA] + c[L_LA], ls = c[L_NB] + c[L_SB] + c[L_LB];
    hdr->list_r = (i64)lr;
    hdr->list_s = (i64)ls;
    // chunk counts and the closing descriptors (see k_plan_apply)
    const u64 wn = c[L_NA] + c[L_NB], ws = c[L_SA] + c[L_SB];
    const u64 chn = wn ? (wn - 1) / kChunkBN + 1 : 0, chs = ws ? (ws - 1) / kChunkB + 1 : 0;
    hdr->chunks_nested = (i64)chn;
    hdr->chunks_sorted = (i64)chs;
    cd_n[chn] = make_uint4((u32)c[L_NF], (u32)c[L_NA], (u32)c[L_NB], 0u);
    cd_s[chs] = make_uint4((u32)c[L_SF], (u32)(c[L_NA] + c[L_SA]), (u32)(c[L_NB] + c[L_SB]), 0u);
    hdr->pairs = 0;
    if (c[L_A] >= kSkip || c[L_B] >= kSkip || lr >= kSkip || ls >= kSkip || c[L_LI] >= kSkip)
      hdr->error |= PBSM_ERR_TOTAL_RANGE;
    lpre[c[L_LF]] = (u32)c[L_LI];
  }
}

struct PlanOut {
  u32 *cur_r, *cur_s;
  uint4* jrec[2];
  uint4* cdesc[2];
  uint4* lrec;
  u32* lpre;
};

// the lanes k_plan_apply scans: every lane but the two totals (L_A, L_B)
constexpr int kNA = kNV - 2;
__global__ void __launch_bounds__(kPlanThreads, PBSM_PLAN_MINB) k_plan_apply(u32* __restrict__ cr,
                                                             u32* __restrict__ cs, u64 T, u64 nb,
                                                             i64 nm,
                                                             const u64* __restrict__ partials,
                                                             PlanOut P) {
  __shared__ u32 sa[kPlanTile];   // counts, then the tiles' list starts
  __shared__ u32 sb[kPlanTile];
  __shared__ u32 ca[kPlanTile];   // counts (for the expected cursor ends)
  __shared__ u32 cb[kPlanTile];
  __shared__ u32 shs[kPlanThreads / 32][kNA];
  __shared__ u64 shp[2][kNV];  // this CTA's global prefixes, the totals
  const u64 base = (u64)blockIdx.x * kPlanTile;
  // lane-major partials: lane q of CTA b at q * (nb + 1) + b, totals at q * (nb + 1) + nb;
  // fetched first so their latency overlaps the count loads
  if (threadIdx.x < 2 * kNV) {
    const int q = threadIdx.x % kNV;
    shp[threadIdx.x / kNV][q] = partials[(u64)q * (nb + 1) + (threadIdx.x < kNV ? blockIdx.x : nb)];
  }
  for (int i = threadIdx.x; i < kPlanTile; i += kPlanThreads) {
    const u64 t = base + i;
    const u32 x = t < T ? cr[t] : 0u, y = t < T ? cs[t] : 0u;
    sa[i] = x;
    sb[i] = y;
    ca[i] = x;
    cb[i] = y;
  }
  __syncthreads();
  u32 a[kPlanPer], b[kPlanPer];
  u32 pre[kNA];  // in-CTA exclusive prefixes of lanes 2..11 (u32: a CTA's sums fit)
#pragma unroll
  for (int q = 0; q < kNA; ++q) pre[q] = 0;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    a[i] = sa[threadIdx.x * kPlanPer + i];
    b[i] = sb[threadIdx.x * kPlanPer + i];
    u32 v[kNV];
    tile_vals(a[i], b[i], nm, v);
#pragma unroll
    for (int q = 0; q < kNA; ++q) pre[q] += v[q + 2];
  }
  {
    u32 tot[kNA];
    block_excl_scan_multi<kPlanThreads, kNA, u32>(pre, tot, shs);
  }
  // global prefix of lane q = this CTA's u64 partial + the u32 running
  // in-CTA prefix (the scan's barriers made shp visible); only the active
  // strategy's lanes advance per tile
  auto g = [&](int q) -> u64 { return shp[0][q] + pre[q - 2]; };
  const u64 rs_base = shp[1][L_NA], ss_base = shp[1][L_NB];
  const u64 rl_base = shp[1][L_NA] + shp[1][L_SA], sl_base = shp[1][L_NB] + shp[1][L_SB];
  // (the scan ended with a barrier, so sa/sb may be overwritten now: they
  // receive the list starts)
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = base + (u64)threadIdx.x * kPlanPer + i;
    const int kind = tile_kind(a[i], b[i], nm);
    u32 r0 = kSkip, s0 = kSkip;
    // chunks: consecutive tiles of one strategy whose LAST entry falls in the
    // same bucket of B entries; a tile starts chunk c when its end is in
    // bucket c and its start (the previous tile's end) is not.  A tile holds
    // <= kLmax <= B entries, so it crosses at most one bucket boundary and a
    // chunk holds < B + kLmax entries.  The plan's last CTA writes the
    // closing descriptor and the chunk counts (k_plan_partials).
    // (one branch per strategy: the bucket widths stay compile-time
    // constants — a runtime divisor cost a 64-bit division per tile)
    if (kind == kNested) {
      r0 = (u32)g(L_NA);
      s0 = (u32)g(L_NB);
      if (t < T) {
        const u32 jj = (u32)g(L_NF);
        P.jrec[0][jj] = make_uint4(r0, s0, a[i], b[i]);
        const u64 st = g(L_NA) + g(L_NB);
        const u64 ce = (st + a[i] + b[i] - 1) / kChunkBN;
        if (st == 0 || (st - 1) / kChunkBN < ce) P.cdesc[0][ce] = make_uint4(jj, r0, s0, 0u);
      }
      pre[L_NF - 2] += 1u;
      pre[L_NA - 2] += a[i];
      pre[L_NB - 2] += b[i];
    } else if (kind == kSorted) {
      r0 = (u32)(rs_base + g(L_SA));
      s0 = (u32)(ss_base + g(L_SB));
      if (t < T) {
        const u32 jj = (u32)g(L_SF);
        P.jrec[1][jj] = make_uint4(r0, s0, a[i], b[i]);
        const u64 st = g(L_SA) + g(L_SB);
        const u64 ce = (st + a[i] + b[i] - 1) / kChunkB;
        if (st == 0 || (st - 1) / kChunkB < ce) P.cdesc[1][ce] = make_uint4(jj, r0, s0, 0u);
      }
      pre[L_SF - 2] += 1u;
      pre[L_SA - 2] += a[i];
      pre[L_SB - 2] += b[i];
    } else if (kind == kLarge) {
      r0 = (u32)(rl_base + g(L_LA));
      s0 = (u32)(sl_base + g(L_LB));
      if (t < T) {
        P.lrec[g(L_LF)] = make_uint4(r0, s0, a[i], b[i]);
        P.lpre[g(L_LF)] = (u32)g(L_LI);
      }
      u32 v[kNV];
      tile_vals(a[i], b[i], nm, v);
      pre[L_LF - 2] += 1u;
      pre[L_LI - 2] += v[L_LI];
      pre[L_LA - 2] += a[i];
      pre[L_LB - 2] += b[i];
    }
    sa[threadIdx.x * kPlanPer + i] = r0;
    sb[threadIdx.x * kPlanPer + i] = s0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPlanTile; i += kPlanThreads) {
    const u64 t = base + i;
    if (t < T) {
      const u32 r0 = sa[i], s0 = sb[i];
      cr[t] = r0 + ca[i];   // expected end of tile t's R cursor (for k_guard)
      cs[t] = s0 + cb[i];
      P.cur_r[t] = r0;
      P.cur_s[t] = s0;
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
  const uint4* jrec[2];    // [0] nested tiles, [1] sorted tiles
  const uint4* cdesc[2];
  const uint4* lrec;
  const u32* lpre;
  const Rec* rl;
  const Rec* sl;
  u32* ticket;
  u64* status;     // [n_units] decoupled look-back words (ordered emit)
  unsigned long long* total;  // running pair total (unordered emit / count)
  int ordered;
  i64* pairs;      // (r_id, s_id) int64 pairs
  i64 capacity;    // pairs the buffer holds
  i64 n_units;
  pbsm_header* hdr;
  int bounded;     // grids are upper bounds: units past the plan's counts exit
  // write guard folded into the nested join (g_tiles > 0): cursor ends vs
  // the counted ends, every tile (partition.py:229-233)
  const u32 *g_cur_r, *g_end_r, *g_cur_s, *g_end_s;
  u64 g_tiles;
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

#ifndef PBSM_LARGE_HITS
#define PBSM_LARGE_HITS 4096
#endif
constexpr int kLargeHitCap = PBSM_LARGE_HITS;  // hits of a large work item kept for the emit
struct LargeSmem {
  Rec other[kCap];
  u32 hit[kLargeHitCap];        // lead thread | other index (in the item) << 8
  i64 lead_id[kJoinThreads];
  u64 bar;
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  u32 nhit;
  int unit;
};

union JoinSmem {
  ChunkSmem c;
  LargeSmem l;
};

// Decoupled look-back (one thread): publish this unit's count, accumulate the
// predecessors' published values until an inclusive prefix is found, publish
// ours.  Units are handed out by an atomic ticket in launch order, so every
// predecessor is resident or finished — the spin cannot deadlock (and is
// bounded anyway, so a bug can never hang the GPU).
__device__ u64 lookback_thread(u64* status, i64 unit, u64 count, pbsm_header* hdr) {
  cuda::atomic_ref<u64, cuda::thread_scope_device> me(status[unit]);
  if (unit == 0) {
    me.store(kFlagPre | count, cuda::memory_order_release);
    return 0;
  }
  me.store(kFlagAgg | count, cuda::memory_order_release);
  u64 excl = 0;
  i64 j = unit - 1;
  u64 spins = 0;
  while (j >= 0) {
    cuda::atomic_ref<u64, cuda::thread_scope_device> st(status[j]);
    const u64 v = st.load(cuda::memory_order_acquire);
    const u64 flag = v & ~kValMask;
    if (flag == 0) {
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

// Output range of one work unit, after its count pass.  Default: one atomic
// on the running pair total — no unit ever waits for another, and the pair
// list is a permutation of the reference's, which is itself unordered
// (engine.py:61-62; with m > 1 threads its order varies run to run).  With
// A.ordered the decoupled look-back gives every unit the exclusive prefix
// of the units before it, i.e. a deterministic chunk-major order.
__device__ __forceinline__ u64 reserve(const JoinArgs& A, i64 unit, u64 total) {
  if (!A.ordered) return atomicAdd(A.total, total);
  const u64 b = lookback_thread(A.status, unit, total, A.hdr);
  if (unit == A.n_units - 1) A.hdr->pairs = (i64)(b + total);
  return b;
}

// ---- nested mini-joins (small tiles)
// For a tile this small, testing all |R_T|·|S_T| pairs costs less than the
// per-tile sort it would need: the larger side leads (one thread per lead
// entry, so lanes stay busy on lopsided tiles), the smaller side is scanned.
// A pair is kept iff the closed rectangles intersect (intersects,
// geometry.py:59-61) and at least one entry is x-in and one is y-in — the
// nine valid class combinations AA AB AC AD BA BC CA CB DA,
// i.e. exactly the tile that passes Eq. 1 for the pair.
__device__ __forceinline__ bool pair_ok(u64 ka, double axu, double ayl, double ayu, u64 kb,
                                        double bxu, double byl, double byu) {
  const double axl = key_x(ka), bxl = key_x(kb);
  // label bits set = "out"; the pair needs one x-in and one y-in: (ka & kb)
  // must have neither label bit set
  return (axl <= bxu) & (bxl <= axu) & (ayl <= byu) & (byl <= ayu) &
         (((ka & kb) & kLabelMask) == 0ull);
}

// Stage a chunk of consecutive tiles of one strategy: TMA bulk copies of its
// R range and S range (contiguous, see k_plan_apply) into `recs`, plus the
// tile table.  Returns false (and flags) if the chunk breaks a plan invariant.
template <typename Smem>
__device__ __forceinline__ void stage_chunk(Smem& S, const JoinArgs& A, int which, int c) {
  const int tid = threadIdx.x;
  const uint4* jrec = A.jrec[which];
  const uint4 d0 = A.cdesc[which][c], d1 = A.cdesc[which][c + 1];
  const u32 j0 = d0.x;
  const int nt = (int)(d1.x - d0.x);
  if (tid == 0) {
    const int NR = (int)(d1.y - d0.y);
    const int NS = (int)(d1.z - d0.z);
    // a chunk never exceeds the staging buffer by construction (k_plan_apply);
    // if it somehow did, flag it and contribute 0 pairs (no early return:
    // the ordered mode's look-back chain must still be fed)
    const bool fits = nt > 0 && NR > 0 && NS > 0 && NR + NS <= kCap && nt <= kMaxTiles;
    if (!fits) atomicOr(&A.hdr->error, PBSM_ERR_INTERNAL);
    S.nt = fits ? nt : 0;
    S.NR = fits ? NR : 0;
    S.NS = fits ? NS : 0;
    if (fits) {
      mbar_init(&S.bar, 1);
      mbar_expect_tx(&S.bar, (u32)(NR + NS) * (u32)sizeof(Rec));
      bulk_g2s(&S.recs[0], A.rl + d0.y, (u32)NR * (u32)sizeof(Rec), &S.bar);
      bulk_g2s(&S.recs[NR], A.sl + d0.z, (u32)NS * (u32)sizeof(Rec), &S.bar);
    }
  }
  __syncthreads();
  // tile table, while the copies are in flight
  const int NR = S.NR;
  for (int lt = tid; lt < S.nt; lt += kJoinThreads) {
    const uint4 r = jrec[j0 + lt];
    S.tR0[lt] = (u16)(r.x - d0.y);
    S.tS0[lt] = (u16)(NR + (int)(r.y - d0.z));
    S.tNR[lt] = (u16)r.z;
    S.tNS[lt] = (u16)r.w;
  }
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
__device__ void join_sorted(ChunkSmem& S, const JoinArgs& A, i64 unit, int c) {
  const int tid = threadIdx.x;
  stage_chunk(S, A, 1, c);
  const int NR = S.NR, N = S.NR + S.NS;
  // position → tile map (the table is complete for this thread's tiles)
  for (int lt = tid; lt < S.nt; lt += kJoinThreads) {
    for (int e = 0; e < (int)S.tNR[lt]; ++e) S.seg[S.tR0[lt] + e] = (u16)lt;
    for (int e = 0; e < (int)S.tNS[lt]; ++e) S.seg[S.tS0[lt] + e] = (u16)lt;
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
    if (tid == 0 && total) atomicAdd(A.total, total);
    return;
  }
  if (tid == 0) S.base = reserve(A, unit, total);
  __syncthreads();
  const i64 start = (i64)(S.base + excl);
  if (start + (i64)cnt > A.capacity) {
    if (cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
    return;
  }
  i64* out = A.pairs + 2 * start;
  for (int p = tid; p < N; p += kJoinThreads) out += 2 * (i64)sweep_one<true>(S, p, out);
}

// Large join tiles (|R_T|+|S_T| > kLmax): work items of kLargeLead entries of
// the larger side (one per thread) × kLargeOther entries of the other side,
// which stream through shared memory.  Every (lead, other) pair is tested with the full
// closed-interval predicate (intersects, geometry.py:59-61) and the class rule
// (>= 1 x-in and >= 1 y-in ⇔ Eq. 1 owner tile).
// LIST: also record each hit (lead thread, other index k0 + k) in the block's
// hit list while it has room
template <bool EMIT, bool LIST>
__device__ __forceinline__ u32 large_pass(LargeSmem& S, int n, bool have, const Half& me,
                                          bool lead_r, i64 my_id, i64* out, u32 k0) {
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
      if (LIST) {
        const u32 h = atomicAdd_block(&S.nhit, 1u);
        if (h < (u32)kLargeHitCap) S.hit[h] = threadIdx.x | ((k0 + (u32)k) << 8);
      }
      ++c;
    }
  }
  return c;
}

template <bool EMIT>
__device__ void join_large(LargeSmem& S, const JoinArgs& A, i64 unit, i64 item) {
  const int tid = threadIdx.x;
  // item → large tile: the last tile whose work-item prefix is <= item.
  // 32-ary search, every warp on its own (same addresses): each step the
  // lanes probe 32 evenly spaced prefixes at once, so the dependent chain is
  // log32 instead of log2 loads long (the binary search was ~12% of the
  // kernel's stall samples on cfg2)
  int lo = 0, hi = (int)A.hdr->n_large;  // lpre[0] = 0 <= item
  const int lane = tid & 31;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int m = lo + lane * step;
    const unsigned le = __ballot_sync(0xffffffffu, m < hi && (i64)__ldg(A.lpre + m) <= item);
    lo += (31 - __clz(le)) * step;  // prefixes are non-decreasing: le is a lane prefix
    hi = min(hi, lo + step);
  }
  const int lj = lo;
  const uint4 rec = A.lrec[lj];
  const u32 nR = rec.z, nS = rec.w;
  const bool lead_r = nR >= nS;
  const u32 no = lead_r ? nS : nR;
  const Rec* L = lead_r ? A.rl + rec.x : A.sl + rec.y;
  const Rec* O = lead_r ? A.sl + rec.y : A.rl + rec.x;
  const u32 nl = lead_r ? nR : nS;
  // work item = (block of kLargeLead lead entries) × (block of kLargeOther
  // other entries), so a huge tile spreads over many CTAs both ways
  const u32 nob = (no + kLargeOther - 1) / kLargeOther;
  const u32 li = (u32)(item - (i64)A.lpre[lj]);
  const u32 a = (li / nob) * kLargeLead + tid;
  const u32 o_beg = (li % nob) * kLargeOther, o_end = min(no, o_beg + kLargeOther);
  const bool have = a < nl;
  Half me;
  i64 my_id = 0;
  if (have) {
    me = *reinterpret_cast<const Half*>(L + a);
    my_id = L[a].id;
  }
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    S.nhit = 0;
  }
  S.lead_id[tid] = my_id;
  __syncthreads();
  u32 phase = 0;
  u32 cnt = 0;
  const int passes = EMIT ? 2 : 1;
  i64* out = nullptr;
  bool ok = true;
  for (int pass = 0; pass < passes; ++pass) {
    for (u32 ob = o_beg; ob < o_end; ob += kCap) {
      const int n = (int)min((u32)kCap, o_end - ob);
      __syncthreads();  // previous piece fully consumed
      if (tid == 0) {
        mbar_expect_tx(&S.bar, (u32)n * (u32)sizeof(Rec));
        bulk_g2s(&S.other[0], O + ob, (u32)n * (u32)sizeof(Rec), &S.bar);
      }
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
      if (pass == 0) {
        cnt += large_pass<false, EMIT>(S, n, have, me, lead_r, my_id, nullptr, ob - o_beg);
      } else if (ok) {
        out += 2 * (i64)large_pass<true, false>(S, n, have, me, lead_r, my_id, out, 0);
      }
    }
    if (pass == 0) {
      u64 total;
      const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
      if (!EMIT) {
        if (tid == 0 && total) atomicAdd(A.total, total);
        return;
      }
      if (tid == 0) S.base = reserve(A, unit, total);
      __syncthreads();
      if (total <= (u64)kLargeHitCap) {
        // every hit is in the list: emit from it (no second pass over the
        // other side), one coalesced 16-byte store per hit
        if ((i64)(S.base + total) > A.capacity) {
          if (tid == 0 && total) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
          return;
        }
        i64* o = A.pairs + 2 * (i64)S.base;
        for (u32 h = tid; h < (u32)total; h += kJoinThreads) {
          const u32 v = S.hit[h];
          const i64 lid = S.lead_id[v & 0xffu];
          const i64 oid = O[o_beg + (v >> 8)].id;
          *reinterpret_cast<longlong2*>(o + 2 * (i64)h) =
              lead_r ? make_longlong2(lid, oid) : make_longlong2(oid, lid);
        }
        return;
      }
      const i64 start = (i64)(S.base + excl);
      ok = start + (i64)cnt <= A.capacity;
      if (!ok && cnt) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
      out = A.pairs + 2 * start;
    }
  }
}

// ---- nested mini-joins: one CTA per chunk of small tiles
// Two lane mappings (PBSM_NESTED_ROWS): the row form (default) gives a lane
// each entry of a tile's larger side and loops over the smaller side; the
// flat form numbers every (r, s) pair of the chunk and gives lane q pair q.
// Hits are ballot-compacted into per-warp lists and emitted after the
// chunk's single output reservation (one coalesced 16-byte store per hit).
//
// Staging: per-thread 16-byte async copies (cp.async) land each 64-byte list
// record directly in the layout the pair tests read — {xl|label, xu} and
// {yl, yu} in two 16-byte arrays, the id in a third — so there is no
// transpose pass, and 32 lanes reading 32 consecutive entries hit 512
// contiguous bytes (4 wavefronts).  The pad words are never fetched.
constexpr int kHitCap = 128;  // hits per warp kept (packed entry positions) for the emit

struct TileInfo {  // one 16-byte shared-memory read per pair test
  u32 p0;          // first pair index of the tile
  u32 rs0;         // chunk-local position of the tile's first R | first S << 16
  u32 ns;          // |S_T|
  float inv_ns;    // 1 / |S_T|
};

struct NestedBuf {               // one staged chunk
  ulonglong2 ax[kCapN];          // {xl | label, xu} per staged entry (R range, then S range)
  double2 ay[kCapN];             // {yl, yu}
  i64 aid[kCapN];                // id
  uint4 jr[kMaxTilesN];          // tile records {r_start, s_start, |R_T|, |S_T|}
};

struct NestedSmem {
  NestedBuf buf;
  // row form: per lead entry pos | o0 << 9 | |other| << 18 | R-leads << 25
  // (positions < kCapN = 512; |other| <= 64: the smaller side of a tile of
  // <= kLmax = 128 entries)
  u32 lead[PBSM_NESTED_ROWS ? kCapN : 1];
  // flat form: tile table, pair-prefix boundaries (tb[nt] = pair total) and
  // 32 sentinels (no bounds check per warp-step)
  TileInfo ti[PBSM_NESTED_ROWS ? 1 : kMaxTilesN];
  u32 tb[PBSM_NESTED_ROWS ? 1 : kMaxTilesN + 33];
  u64 wtot[kNT / 32 + 1];
  u32 scan32[kNT / 32 + 1];
  u32 hits[kNT / 32][kHitCap];  // pass-1 hits: r position | s position << 16
  u64 base;
};

// first tile of pair q0: binary search over the boundaries (the same
// addresses in every lane: broadcast reads)
__device__ __forceinline__ int nested_tile_of(const NestedSmem& S, int nt, u32 q0) {
  int lo = 0, hi = nt;  // last lt with tb[lt] <= q0
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (S.tb[m] <= q0) lo = m; else hi = m;
  }
  return lo;
}

// Tiles of one warp-step: lane j reads boundary tb[lt + 1 + j]; the in-step
// boundaries (at most 31: tiles hold >= 1 pair and tb[lt] <= q0) become a
// position bitmask, and lane L's tile is lt + (boundaries at positions <= L).
// Returns lane's tile; advances lt to the tile of the step's last pair.
__device__ __forceinline__ int nested_step_tile(const NestedSmem& S, int nt, u32 q0, int& lt,
                                                int lane) {
  const int j = lt + 1 + lane;
  const u32 d = S.tb[j] - q0;  // tb[nt + 1 ..] = ~0
  if (__shfl_sync(0xffffffffu, d, 0) >= 32u) return lt;  // the whole step in tile lt
  const unsigned bits = __reduce_or_sync(0xffffffffu, d < 32u ? (1u << d) : 0u);
  const int mine = lt + __popc(bits & (0xffffffffu >> (31 - lane)));
  lt += __popc(bits);
  return mine;
}

// pair q (in tile t) → chunk-local positions of its r and s entries
__device__ __forceinline__ void nested_pair(const NestedSmem& S, int t, u32 q, int& pr, int& ps) {
  const TileInfo ti = S.ti[t];
  const u32 local = q - ti.p0;
  // local / ns: local < 2^16 and |local/ns - integer| >= 0.5/ns, so the
  // float estimate of (local + 0.5) / ns truncates to the exact quotient
  const u32 r = (u32)__float2int_rz(((float)local + 0.5f) * ti.inv_ns);
  pr = (int)(ti.rs0 & 0xffffu) + (int)r;
  ps = (int)(ti.rs0 >> 16) + (int)(local - r * ti.ns);
}

__device__ __forceinline__ bool nested_hit(const NestedBuf& B, int pr, int ps) {
  const ulonglong2 rx = B.ax[pr], sx = B.ax[ps];
  const double2 ry = B.ay[pr], sy = B.ay[ps];
  return pair_ok(rx.x, __longlong_as_double((long long)rx.y), ry.x, ry.y, sx.x,
                 __longlong_as_double((long long)sx.y), sy.x, sy.y);
}

// chunk c's ranges: tiles [d0.x, d0.x + nt), R entries from d0.y, S from d0.z
struct NestedChunk {
  uint4 d0;
  int nt, NR, NS;
  bool ok;
};

// all threads: the chunk descriptor (broadcast loads) and its plan check
__device__ __forceinline__ NestedChunk nested_desc(const JoinArgs& A, i64 c) {
  NestedChunk k;
  k.d0 = A.cdesc[0][c];
  const uint4 d1 = A.cdesc[0][c + 1];
  k.nt = (int)(d1.x - k.d0.x);
  k.NR = (int)(d1.y - k.d0.y);
  k.NS = (int)(d1.z - k.d0.z);
  k.ok = k.nt > 0 && k.NR > 0 && k.NS > 0 && k.NR + k.NS <= kCapN && k.nt <= kMaxTilesN;
  return k;
}

// a chunk that breaks the plan invariants (never, by construction of
// k_plan_apply): flag it and contribute 0 pairs (no early return: the ordered
// look-back chain must still be fed)
__device__ __forceinline__ void nested_check(const JoinArgs& A, NestedChunk& k) {
  if (!k.ok) {
    if (threadIdx.x == 0) atomicOr(&A.hdr->error, PBSM_ERR_INTERNAL);
    k.nt = k.NR = k.NS = 0;
  }
}

// all threads: async copies of the chunk's entries (coords + id; the pad is
// skipped) and tile records into B
__device__ __forceinline__ void nested_stage(NestedBuf& B, const JoinArgs& A,
                                             const NestedChunk& k) {
  const int N = k.NR + k.NS;
  for (int e = threadIdx.x; e < N; e += kNT) {
    const Rec* src = e < k.NR ? A.rl + k.d0.y + e : A.sl + k.d0.z + (e - k.NR);
    const unsigned char* g = reinterpret_cast<const unsigned char*>(src);
    cp_async16(&B.ax[e], g);
    cp_async16(&B.ay[e], g + 16);
    cp_async8(&B.aid[e], g + 32);
  }
  for (int t = threadIdx.x; t < k.nt; t += kNT) cp_async16(&B.jr[t], A.jrec[0] + k.d0.x + t);
}

// Row form: one lane per entry of each tile's larger ("lead") side, looping
// over the tile's other side (<= 32 entries with the default cost model,
// |R_T|*|S_T| <= 1024; <= 64 for any nested tile, |R_T|+|S_T| <= 128).  No per-pair index arithmetic; a warp runs max(|other|)
// steps over its 32 lead entries.  body(hit, pr, ps, ballot) is called by
// every lane of every step.
template <typename Body>
__device__ __forceinline__ void nested_rows(const NestedSmem& S, const NestedBuf& B, u32 e_beg,
                                            u32 e_end, u32 e_step, int lane, Body&& body) {
  for (u32 g = e_beg; g < e_end; g += e_step) {
    const u32 ei = g + lane;
    const bool valid = ei < e_end;
    const u32 d = valid ? S.lead[ei] : 0u;
    const u32 pos = d & 511u, o0 = (d >> 9) & 511u, nO = valid ? (d >> 18) & 127u : 0u;
    const bool lr = (d >> 25) & 1u;
    const ulonglong2 mx = B.ax[pos];
    const double2 my = B.ay[pos];
    const double mxu = __longlong_as_double((long long)mx.y);
    const u32 steps = __reduce_max_sync(0xffffffffu, nO);
    for (u32 j = 0; j < steps; ++j) {
      bool hit = false;
      if (j < nO) {
        const ulonglong2 ox = B.ax[o0 + j];
        const double2 oy = B.ay[o0 + j];
        hit = pair_ok(mx.x, mxu, my.x, my.y, ox.x, __longlong_as_double((long long)ox.y), oy.x,
                      oy.y);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      body(hit, lr ? pos : o0 + j, lr ? o0 + j : pos, m);
    }
  }
}

// Pair-flattened form (PBSM_NESTED_ROWS=0): every (r, s) pair of every tile
// gets an index (tile-major, then r, then s); lane q of a warp-step tests pair q.
template <typename Body>
__device__ __forceinline__ void nested_flat(const NestedSmem& S, const NestedBuf& B, int nt,
                                            u32 q_beg, u32 q_end, int lt, int lane,
                                            Body&& body) {
  for (u32 q0 = q_beg; q0 < q_end; q0 += 32u) {
    const u32 q = q0 + lane;
    const int t = nested_step_tile(S, nt, q0, lt, lane);
    bool hit = false;
    int pr = 0, ps = 0;
    if (q < q_end) {
      nested_pair(S, t, q, pr, ps);
      hit = nested_hit(B, pr, ps);
    }
    body(hit, (u32)pr, (u32)ps, __ballot_sync(0xffffffffu, hit));
  }
}

// One staged chunk (B landed and visible): tables, count, reserve, emit.
template <bool EMIT>
__device__ __forceinline__ void nested_chunk(NestedSmem& S, const NestedBuf& B,
                                             const JoinArgs& A, const NestedChunk& k, i64 c) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = k.nt, NR = k.NR;
  constexpr int kTPT = (kMaxTilesN + kNT - 1) / kNT;
  constexpr int kW = kNT / 32;
  const unsigned lt_mask = (1u << lane) - 1u;
  // per-tile table (kTPT consecutive tiles per thread)
  uint4 tr[kTPT];
  u32 w = 0;
#pragma unroll
  for (int h = 0; h < kTPT; ++h) {
    const int t = kTPT * tid + h;
    tr[h] = t < nt ? B.jr[t] : make_uint4(0, 0, 0, 0);
    w += PBSM_NESTED_ROWS ? max(tr[h].z, tr[h].w) : tr[h].z * tr[h].w;
  }
  u32 W;  // rows: lead entries of the chunk; flat: pairs of the chunk
  u32 pre = block_excl_scan32<kNT>(w, &W, S.scan32);
#pragma unroll
  for (int h = 0; h < kTPT; ++h) {
    const int t = kTPT * tid + h;
    if (t >= nt) continue;
    const u32 r0 = tr[h].x - k.d0.y, s0 = (u32)NR + (tr[h].y - k.d0.z);
    if (PBSM_NESTED_ROWS) {
      const bool lr = tr[h].z >= tr[h].w;
      const u32 nL = lr ? tr[h].z : tr[h].w, nO = lr ? tr[h].w : tr[h].z;
      const u32 l0 = lr ? r0 : s0, o0 = lr ? s0 : r0;
      const u32 d = (o0 << 9) | (nO << 18) | ((u32)lr << 25);
      for (u32 i = 0; i < nL; ++i) S.lead[pre + i] = (l0 + i) | d;
      pre += nL;
    } else {
      TileInfo ti;
      ti.p0 = pre;
      ti.rs0 = r0 | (s0 << 16);
      ti.ns = tr[h].w;
      ti.inv_ns = 1.0f / (float)tr[h].w;
      S.ti[t] = ti;
      S.tb[t] = pre;
      pre += tr[h].z * tr[h].w;
    }
  }
  if (!PBSM_NESTED_ROWS && tid <= 32) S.tb[nt + tid] = tid == 0 ? W : 0xffffffffu;
  __syncthreads();
  // flat form: each warp owns one contiguous, 32-aligned slice of the pair
  // index space (its tile only moves forward); row form: warps take groups
  // of 32 lead entries round-robin (the groups' step counts differ, so
  // interleaving balances the warps before the barrier)
  const u32 per = ((W + kW - 1) / kW + 31u) & ~31u;
  const u32 w_beg = PBSM_NESTED_ROWS ? 32u * warp : min(W, (u32)warp * per);
  const u32 w_end = PBSM_NESTED_ROWS ? W : min(W, w_beg + per);
  const int lt_beg = (!PBSM_NESTED_ROWS && w_beg < W) ? nested_tile_of(S, nt, w_beg) : 0;
  // pass 1: count, keeping the warp's hits (ballot-compacted) in its list
  u32 wcnt = 0;
  auto count = [&](bool hit, u32 pr, u32 ps, unsigned m) {
    if (EMIT && hit) {
      const u32 o = wcnt + __popc(m & lt_mask);
      if (o < kHitCap) S.hits[warp][o] = pr | (ps << 16);
    }
    wcnt += __popc(m);
  };
  if (PBSM_NESTED_ROWS) nested_rows(S, B, w_beg, w_end, 32u * kW, lane, count);
  else nested_flat(S, B, nt, w_beg, w_end, lt_beg, lane, count);
  if (lane == 0) S.wtot[warp] = wcnt;
  __syncthreads();
  if (tid == 0) {
    u64 t = 0;
    for (int v = 0; v < kW; ++v) {
      const u64 x = S.wtot[v];
      S.wtot[v] = t;
      t += x;
    }
    if (!EMIT) {
      if (t) atomicAdd(A.total, t);
    } else {
      S.base = reserve(A, c, t);
      if ((i64)(S.base + t) > A.capacity) {
        if (t) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
        S.base = ~0ull;  // nothing written
      }
    }
  }
  if (!EMIT) return;
  __syncthreads();
  if (S.base == ~0ull) return;
  // pass 2: emit the warp's hits at its offset — from the hit list (one
  // coalesced 16-byte store per hit, nothing re-tested), or, for a warp whose
  // hits overflowed the list, by re-testing its slice (same order)
  i64* out = A.pairs + 2 * (i64)(S.base + S.wtot[warp]);
  if (wcnt <= (u32)kHitCap) {
    for (u32 i = lane; i < wcnt; i += 32u) {
      const u32 v = S.hits[warp][i];
      *reinterpret_cast<longlong2*>(out + 2 * (i64)i) =
          make_longlong2(B.aid[v & 0xffffu], B.aid[v >> 16]);
    }
    return;
  }
  auto emit = [&](bool hit, u32 pr, u32 ps, unsigned m) {
    if (hit) {
      const i64 o = __popc(m & lt_mask);
      *reinterpret_cast<longlong2*>(out + 2 * o) = make_longlong2(B.aid[pr], B.aid[ps]);
    }
    out += 2 * (i64)__popc(m);
  };
  if (PBSM_NESTED_ROWS) nested_rows(S, B, w_beg, w_end, 32u * kW, lane, emit);
  else nested_flat(S, B, nt, w_beg, w_end, lt_beg, lane, emit);
}

// One CTA per chunk (chunks handed out by ticket in the ordered mode, whose
// look-back needs launch order).  Static shared memory: the compiler then
// addresses it with constant offsets.  (A persistent variant that staged chunk
// i+1 with cp.async while joining chunk i was measured slower twice: more
// resident CTAs beat the deeper pipeline.)
template <bool EMIT>
#ifndef PBSM_NESTED_MINB
#define PBSM_NESTED_MINB (1536 / kNT)
#endif
__global__ void __launch_bounds__(kNT, PBSM_NESTED_MINB) k_join_nested(JoinArgs A, i64 n_chunks) {
  __shared__ __align__(128) NestedSmem S;
  if (A.g_tiles) {  // the write guard, a grid-stride slice per CTA (all CTAs)
    bool bad = false;
    for (u64 t = blockIdx.x * (u64)kNT + threadIdx.x; t < A.g_tiles; t += (u64)gridDim.x * kNT)
      bad |= (A.g_cur_r[t] != A.g_end_r[t]) || (A.g_cur_s[t] != A.g_end_s[t]);
    if (bad) atomicOr(&A.hdr->error, PBSM_ERR_OFFSET_MISMATCH);
  }
  __shared__ int s_unit;
  if (A.ordered) {
    if (threadIdx.x == 0) s_unit = (int)atomicAdd(A.ticket, 1u);
    __syncthreads();
  }
  const i64 c = A.ordered ? s_unit : blockIdx.x;
  // (cdesc holds tiles + 2 entries, so the descriptor load is in bounds
  // even for a unit past the plan's count: load it alongside the count)
  const i64 n_plan = A.bounded ? (i64)A.hdr->chunks_nested : n_chunks;
  NestedChunk k = nested_desc(A, c);
  if (c >= n_plan) return;
  nested_check(A, k);
  nested_stage(S.buf, A, k);
  cp_async_wait_all();
  __syncthreads();
  nested_chunk<EMIT>(S, S.buf, A, k, c);
}

template <bool EMIT>
#ifndef PBSM_JOIN_MINB
#define PBSM_JOIN_MINB 2
#endif
__global__ void __launch_bounds__(kJoinThreads, PBSM_JOIN_MINB) k_join(JoinArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  JoinSmem& U = *reinterpret_cast<JoinSmem*>(smem_raw);
  // ordered mode hands out units by ticket (launch order, for the look-back);
  // otherwise any CTA may take any unit
  __shared__ int s_unit;
  if (A.ordered) {
    if (threadIdx.x == 0) s_unit = (int)atomicAdd(A.ticket, 1u);
    __syncthreads();
  }
  const int local = A.ordered ? s_unit : (int)blockIdx.x;
  // units of this launch: [sorted chunks | large items]; the look-back ids
  // continue after the nested chunks (k_join_nested)
  const i64 cn = A.hdr->chunks_nested, cs = A.hdr->chunks_sorted;
  if (A.bounded && local >= cs + A.hdr->n_items) return;
  const i64 unit = cn + local;
  if (local < cs) join_sorted<EMIT>(U.c, A, unit, local);
  else join_large<EMIT>(U.l, A, unit, local - cs);
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

// ---------------------------------------------------------------- input formats
// SJB1 body (io.py:113-141 in the reference): packed little-endian records
// {id u64, x_l f64, y_l f64, x_u f64, y_u f64} (40 bytes) → the SoA columns
// of RectBatch, with load_mbr_binary's check (lower <= upper on both axes;
// NaN fails it) as an error flag.
__global__ void k_unpack_records(const u64* __restrict__ rec, i64 n, i64* __restrict__ ids,
                                 double* __restrict__ xl, double* __restrict__ xu,
                                 double* __restrict__ yl, double* __restrict__ yu,
                                 u32* __restrict__ bad) {
  bool b = false;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const u64* r = rec + 5 * i;
    const double a = __longlong_as_double((long long)__ldcs(r + 1));
    const double c = __longlong_as_double((long long)__ldcs(r + 2));
    const double bb = __longlong_as_double((long long)__ldcs(r + 3));
    const double d = __longlong_as_double((long long)__ldcs(r + 4));
    ids[i] = (i64)__ldcs(r);
    xl[i] = a;
    yl[i] = c;
    xu[i] = bb;
    yu[i] = d;
    b |= !(a <= bb) || !(c <= d);
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1u);
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

// header → page-locked host memory (see pbsm_read_header)
__global__ void k_publish_header(const pbsm_header* __restrict__ hdr, pbsm_header* out) {
  static_assert(sizeof(pbsm_header) % 8 == 0, "header words");
  const int i = threadIdx.x;
  if (i < (int)(sizeof(pbsm_header) / 8))
    reinterpret_cast<volatile u64*>(out)[i] = __ldcg(reinterpret_cast<const u64*>(hdr) + i);
}

// row indices → ids in a pair list (scatter run without the id columns)
__global__ void k_map_ids(i64* __restrict__ pairs, i64 n, const i64* __restrict__ r_ids,
                          const i64* __restrict__ s_ids) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
    reinterpret_cast<longlong2*>(pairs)[i] = make_longlong2(__ldg(r_ids + p.x), __ldg(s_ids + p.y));
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

// grid of the count and bin passes (the same n → the same block ranges)
// (swept: 32 blocks per SM of >= 2048 rectangles — finer than the 8 per SM
// before — took the cfg3 count pass from 1.09 to 0.97 ms, cfg2 273 -> 255 µs)
#ifndef PBSM_PART_GRID
#define PBSM_PART_GRID 32  // blocks per SM
#endif
unsigned part_blocks(i64 n) {
  return (unsigned)std::max<i64>(1, std::min<i64>((n + 2047) / 2048,
                                                  std::min<i64>(kMaxPartBlocks, num_sms() * PBSM_PART_GRID)));
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

int launch_join(bool emit, bool ordered, void* ws, int kx, int ky, int row_lo, int row_hi,
                const pbsm_entry* r_list, const pbsm_entry* s_list, const pbsm_header* plan,
                void* scratch, int64_t* pairs, i64 capacity, cudaStream_t s,
                i64 max_nested = -1, i64 max_other = -1) {
  int rc = set_smem_attrs();
  if (rc) return rc;
  const WsLayout L = ws_layout(kx, ky, row_lo, row_hi);
  Ws w = ws_bind(ws, L);
  const bool bounded = plan == nullptr;  // sizes from the device header, grids = bounds
  const i64 cn = bounded ? max_nested : plan->chunks_nested;
  const i64 rest = bounded ? max_other : plan->chunks_sorted + plan->n_items;
  const i64 n_units = cn + rest;
  // the write guard (reads the cursors the scatter left behind) runs inside
  // the nested join when there is one, else as its own kernel
  const bool fused_guard = cn > 0;
  if (!fused_guard) {
    const unsigned gb = (unsigned)std::max<i64>(1, std::min<i64>((i64)((L.tiles + 255) / 256),
                                                                  (i64)num_sms() * 8));
    k_guard<<<gb, 256, 0, s>>>(w.cur_r, w.cnt_r, w.cur_s, w.cnt_s, L.tiles, w.hdr);
  }
  cudaMemsetAsync(&w.hdr->pairs, 0, sizeof(int64_t), s);
  if (n_units == 0) return launch_status();
  if (ordered) cudaMemsetAsync(scratch, 0, join_scratch(n_units), s);
  JoinArgs A;
  for (int q = 0; q < 2; ++q) {
    A.jrec[q] = w.jrec[q];
    A.cdesc[q] = w.cdesc[q];
  }
  A.lrec = w.lrec;
  A.lpre = w.lpre;
  A.rl = reinterpret_cast<const Rec*>(r_list);
  A.sl = reinterpret_cast<const Rec*>(s_list);
  A.ticket = (u32*)scratch;
  A.status = (u64*)((char*)scratch + 256);
  A.pairs = (i64*)pairs;
  A.capacity = capacity;
  A.n_units = n_units;
  A.hdr = w.hdr;
  A.total = (unsigned long long*)&w.hdr->pairs;
  A.ordered = ordered ? 1 : 0;
  A.bounded = bounded ? 1 : 0;
  A.g_cur_r = w.cur_r;
  A.g_end_r = w.cnt_r;
  A.g_cur_s = w.cur_s;
  A.g_end_s = w.cnt_s;
  A.g_tiles = fused_guard ? L.tiles : 0;
  if (cn > 0) {
    // one CTA per chunk (the ordered look-back takes tickets in launch order)
    if (emit)
      k_join_nested<true><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
    else
      k_join_nested<false><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
  }
  if (rest > 0) {
    // the sorted/large launch keeps its own ticket (the look-back ids follow
    // the nested chunks', whose kernel has finished by then)
    if (ordered) cudaMemsetAsync(scratch, 0, 4, s);
    if (emit)
      k_join<true><<<(unsigned)rest, kJoinThreads, sizeof(JoinSmem), s>>>(A);
    else
      k_join<false><<<(unsigned)rest, kJoinThreads, sizeof(JoinSmem), s>>>(A);
  }
  return launch_status();
}

}  // namespace

// ======================================================================== ABI
extern "C" {

int32_t pbsm_abi_version(void) { return PBSM_ABI_VERSION; }

#define PBSM_STR2(x) #x
#define PBSM_STR(x) PBSM_STR2(x)
const char* pbsm_build_info(void) {
  return "pbsm sm_100a abi4: count+validate / plan / scatter (64B records, join tiles only) / "
         "guard / mini-joins: nested (cp.async-staged) | sort+forward-scan, large (TMA-staged), "
         "count->emit; B=" PBSM_STR(PBSM_CHUNK_B) " Bn=" PBSM_STR(PBSM_CHUNK_BN) " Lmax=" PBSM_STR(
             PBSM_LMAX) " nested<=" PBSM_STR(PBSM_NESTED_MAX);
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
  const i64 blocks = std::max<i64>(1, std::min<i64>((i64)(L.tiles / 4 + 255) / 256,
                                                     (i64)num_sms() * 4));
  k_init<<<(unsigned)blocks, 256, 0, s>>>(w.hdr, w.cnt_r, w.cnt_s, L.tiles, w.bx, kx, w.by, ky);
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
  k_count<<<part_blocks(n), 256, 0, as_stream(stream)>>>(xl, xu, yl, yu, n, kx, ky, row_lo,
                                                         row_hi, w.bx, w.by,
                                                         side ? w.cnt_s : w.cnt_r, side,
                                                         w.bc[side], w.hdr);
  return launch_status();
}

int pbsm_plan(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
              int64_t nested_max, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  cudaStream_t s = as_stream(stream);
  const i64 nm = nested_max < 0 ? (i64)kNestedMax : (i64)nested_max;
  k_plan_reduce<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles, nm,
                                                              w.partials, w.hdr);
  k_plan_partials<<<kNV, kPartThreads, 0, s>>>(w.partials, w.nblocks, w.hdr, w.cdesc[0],
                                                w.cdesc[1], w.lpre);
  PlanOut P;
  P.cur_r = w.cur_r;
  P.cur_s = w.cur_s;
  for (int q = 0; q < 2; ++q) {
    P.jrec[q] = w.jrec[q];
    P.cdesc[q] = w.cdesc[q];
  }
  P.lrec = w.lrec;
  P.lpre = w.lpre;
  k_plan_apply<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles,
                                                             w.nblocks, nm, w.partials, P);
  return launch_status();
}

int pbsm_read_header(void* ws, pbsm_header* out, void* stream) {
  if (!ws || !out) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  // page-locked destination (device-accessible under UVA): one tiny kernel
  // stores the header straight into host memory over PCIe, which returns
  // sooner than a copy-engine transfer; pageable memory takes the copy
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, out);
  if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer == (void*)out) {
    k_publish_header<<<1, 32, 0, s>>>(reinterpret_cast<const pbsm_header*>(ws), out);
    e = cudaGetLastError();
  } else {
    cudaGetLastError();  // (clear a failed attribute query)
    e = cudaMemcpyAsync(out, ws, sizeof(pbsm_header), cudaMemcpyDeviceToHost, s);
  }
  if (e != cudaSuccess) return (int)e;
  e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? 0 : (int)e;
}

static int scatter_impl(const int64_t* ids, const double* xl, const double* xu,
                        const double* yl, const double* yu, const void* band, int64_t n,
                        int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                        int32_t row_hi, pbsm_entry* out, int64_t capacity, void* stream) {
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
#ifndef PBSM_SCAT_GRID
#define PBSM_SCAT_GRID 32  // blocks per SM (swept 8-1000 on cfg2/cfg3: 32 best)
#endif
  const i64 blocks = std::min<i64>((n + 255) / 256, (i64)num_sms() * PBSM_SCAT_GRID);
  ScatterIn in{(const i64*)ids, xl, xu, yl, yu, reinterpret_cast<const BRec*>(band)};
  if (band)
    k_scatter<true><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        in, n, kx, ky, row_lo, row_hi, w.bx, w.by, side ? w.cur_s : w.cur_r,
        reinterpret_cast<Rec*>(out), capacity, w.hdr);
  else
    k_scatter<false><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        in, n, kx, ky, row_lo, row_hi, w.bx, w.by, side ? w.cur_s : w.cur_r,
        reinterpret_cast<Rec*>(out), capacity, w.hdr);
  return launch_status();
}

int pbsm_scatter(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                 const double* yu, int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky,
                 int32_t row_lo, int32_t row_hi, pbsm_entry* out, int64_t capacity,
                 void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu || (!out && capacity > 0)) return PBSM_E_ARG;
  return scatter_impl(ids, xl, xu, yl, yu, nullptr, n, side, ws, kx, ky, row_lo, row_hi, out,
                      capacity, stream);
}

int pbsm_scatter_banded(const void* band, int64_t n, int32_t side, void* ws, int32_t kx,
                        int32_t ky, int32_t row_lo, int32_t row_hi, pbsm_entry* out,
                        int64_t capacity, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!band || (!out && capacity > 0)) return PBSM_E_ARG;
  return scatter_impl(nullptr, nullptr, nullptr, nullptr, nullptr, band, n, side, ws, kx, ky,
                      row_lo, row_hi, out, capacity, stream);
}

int pbsm_bin(const int64_t* ids, const double* xl, const double* xu, const double* yl,
             const double* yu, int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky,
             int32_t row_lo, int32_t row_hi, void* band, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1))
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu || !band) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  cudaStream_t s = as_stream(stream);
  const unsigned nb = part_blocks(n);
  const u64 m = (u64)kBinSlots * nb;
  const u64 sb = (m + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<(unsigned)sb, kScanThreads, 0, s>>>(w.bc[side], m, w.bscan);
  k_scan_partials<<<1, 1024, 0, s>>>(w.bscan, sb, w.bo, m);
  k_scan_apply<<<(unsigned)sb, kScanThreads, 0, s>>>(w.bc[side], m, w.bscan, w.bo);
  k_bin_copy<<<nb, 256, 0, s>>>((const i64*)ids, xl, xu, yl, yu, n, ky, row_lo, row_hi, w.by,
                                w.bo, reinterpret_cast<BRec*>(band));
  return launch_status();
}

int64_t pbsm_join_scratch_bytes(int64_t n_units) {
  if (n_units < 0) return PBSM_E_ARG;
  return (int64_t)join_scratch(n_units);
}

int pbsm_join_count(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                    const pbsm_entry* r_list, const pbsm_entry* s_list,
                    const pbsm_header* plan, void* scratch, void* stream) {
  if (!ws || !scratch || !plan || !grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  return launch_join(false, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, plan, scratch,
                     nullptr, 0, as_stream(stream));
}

int pbsm_join_emit(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const pbsm_entry* r_list, const pbsm_entry* s_list,
                   const pbsm_header* plan, void* scratch, int64_t* pairs, int64_t capacity,
                   int32_t ordered, void* stream) {
  if (!ws || !scratch || !plan || !grid_ok(kx, ky, row_lo, row_hi) || capacity < 0 ||
      (capacity > 0 && !pairs))
    return PBSM_E_ARG;
  return launch_join(true, ordered != 0, ws, kx, ky, row_lo, row_hi, r_list, s_list, plan,
                     scratch, pairs, capacity, as_stream(stream));
}

int pbsm_join_emit_bounded(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                           const pbsm_entry* r_list, const pbsm_entry* s_list,
                           int64_t max_nested_chunks, int64_t max_other_units, void* scratch,
                           int64_t* pairs, int64_t capacity, void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || capacity < 0 ||
      (capacity > 0 && !pairs) || max_nested_chunks < 0 || max_other_units < 0 ||
      max_nested_chunks > 0x7fffffff || max_other_units > 0x7fffffff)
    return PBSM_E_ARG;
  return launch_join(true, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, nullptr, scratch,
                     pairs, capacity, as_stream(stream), max_nested_chunks, max_other_units);
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

int pbsm_map_ids(int64_t* pairs, int64_t n, const int64_t* r_ids, const int64_t* s_ids,
                 void* stream) {
  if (n < 0) return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!pairs || !r_ids || !s_ids) return PBSM_E_ARG;
  const unsigned blocks = (unsigned)std::min<i64>((n + 255) / 256, (i64)num_sms() * 8);
  k_map_ids<<<blocks, 256, 0, as_stream(stream)>>>((i64*)pairs, n, (const i64*)r_ids,
                                                    (const i64*)s_ids);
  return launch_status();
}

int pbsm_unpack_records(const void* records, int64_t n, int64_t* ids, double* xl, double* xu,
                        double* yl, double* yu, uint32_t* bad, void* stream) {
  if (n < 0 || !bad) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(uint32_t), s);
  if (n == 0) return launch_status();
  if (!records || !ids || !xl || !xu || !yl || !yu || ((uintptr_t)records & 7u)) return PBSM_E_ARG;
  const unsigned blocks = (unsigned)std::min<i64>((n + 255) / 256, (i64)num_sms() * 8);
  k_unpack_records<<<blocks, 256, 0, s>>>((const u64*)records, n, (i64*)ids, xl, xu, yl, yu, bad);
  return launch_status();
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
