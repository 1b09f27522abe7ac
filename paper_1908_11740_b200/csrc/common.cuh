// common.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: constants, records, workspace layout, tile_of, scans, TMA/cp.async helpers.
#pragma once

// ---------------------------------------------------------------- constants
constexpr int kPlanThreads = 256;
#ifndef PBSM_PLAN_PER
#define PBSM_PLAN_PER 8  // tiles per thread (4 → 8: cfg2 plan 86 → 83 µs, cfg3 191 → 182 µs)
#endif
#ifndef PBSM_PLAN_MINB
#define PBSM_PLAN_MINB 4
#endif
constexpr int kPlanPer = PBSM_PLAN_PER;               // tiles per thread
constexpr int kPlanTile = kPlanThreads * kPlanPer;   // 1024 tiles per CTA
constexpr int kNV = 13;                              // plan scan lanes (see tile_vals)
constexpr int kNTot = kNV + 3;  // partials rows: kNV scan lanes + per-CTA max tile, pair bound, max huge side

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
static_assert(kCapN <= 512 && kLmax <= 256, "nested row descriptors: 9-bit positions, 8-bit counts");
constexpr int kLargeLead = kJoinThreads;  // lead-side entries per large work item
#ifndef PBSM_LARGE_OTHER
#define PBSM_LARGE_OTHER 1024  // (a bitmap row of 32 words per lead thread; 256-2048 time alike, r03f)
#endif
constexpr int kLargeOther = PBSM_LARGE_OTHER;  // other-side entries per large work item
constexpr int kSweepLeaders = 256;    // leaders per sweep work item (sweep.cuh)
#ifndef PBSM_SWEEP_MIN
#define PBSM_SWEEP_MIN (1ll << 26)
#endif
// A large tile whose |R_T|*|S_T| exceeds this is sorted + swept (sweep.cuh);
// smaller ones are brute-forced in work items of 256 x 1024 entries, which
// on a GPU beats the sort + scan (bounded cost, no divergence) below ~10^8
// pair tests per tile
constexpr long long kSweepMin = PBSM_SWEEP_MIN;
__host__ __device__ __forceinline__ bool is_huge(unsigned a, unsigned b, long long sweep_min) {
  return (long long)((unsigned long long)a * (unsigned long long)b) > sweep_min;
}
constexpr int kSortWindow = 4096;     // entries per shared-memory sort window (sweep.cuh)

#ifndef PBSM_JOIN_PDL
#define PBSM_JOIN_PDL 1  // k_join launched as a programmatic dependent of the nested join (cfg2 join 332 -> 320 µs)
#endif

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
  size_t hdr, bx, by, cnt_r, cnt_s, cur_r, cur_s, jrec[2], cdesc[2], lrec, lpre, lwin,
      partials, bc[2], bo, bscan, litem, total;
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
  L.lwin = o; o = align_up(o + 4 * (T + 1), 256);
  L.partials = o; o = align_up(o + sizeof(u64) * kNTot * (L.nblocks + 1), 256);
  for (int q = 0; q < 2; ++q) {  // per-(band, block) rectangle counts of each input
    L.bc[q] = o; o = align_up(o + 4 * (size_t)kBinSlots * kMaxPartBlocks, 256);
  }
  L.bo = o; o = align_up(o + 8 * ((size_t)kBinSlots * kMaxPartBlocks + 1), 256);
  L.bscan = o; o = align_up(o + 8 * (((size_t)kBinSlots * kMaxPartBlocks) / 4096 + 2), 256);
  // large work item → its tile (the first `tiles` items; later ones search lpre)
  L.litem = o; o = align_up(o + 4 * T, 256);
  L.total = o;
  return L;
}

struct Ws {
  pbsm_header* hdr;
  double* bx;
  double* by;
  u32 *cnt_r, *cnt_s, *cur_r, *cur_s, *lpre, *lwin, *litem;
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
  w.lwin = (u32*)(b + L.lwin);
  w.partials = (u64*)(b + L.partials);
  for (int q = 0; q < 2; ++q) w.bc[q] = (u32*)(b + L.bc[q]);
  w.bo = (u64*)(b + L.bo);
  w.bscan = (u64*)(b + L.bscan);
  w.litem = (u32*)(b + L.litem);
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
