// sweep.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after join.cuh's types).
// Contents: subsystems 2 + 3 for the LARGE tiles (|R_T|+|S_T| > LMAX): a
// segmented sort of every large tile's R and S lists by x-lower
// (sort_segment, _kernels.pyx:188-228) in global memory, then the forward-scan
// plane sweep (Alg. 1, do_sweep _kernels.pyx:231-293) with one leader element
// per thread and binary-searched scan starts.
//
// Sort.  The large tiles' entries of one input are one contiguous range of its
// tile list (the list layout is [nested | sorted | large], each in tile
// order), i.e. a sequence of segments, one per large tile.  Sort key of an
// entry: (xl with the x-out label, list position) — x-in entries (label bit
// 63 clear) order by xl, x-out entries follow; the list position makes the
// order total.  k_lsort_win sorts every 4096-entry window of every segment
// (windows counted from the segment start) in shared memory (bitonic);
// k_lmerge then merges runs of width w, 2w, ... within each segment — every
// element finds its rank in the partner run by binary search and moves
// straight to its final slot (no merge-path partitioning) — until w >= the
// longest segment.  k_lgather writes the sorted copy (SoA:
// key, xu, yl, yu, id) the sweep reads.
//
// Sweep.  Work item = 256 consecutive sorted entries of one side of one
// large tile, one leader per thread.  As in the reference, a pair is found
// from the side with the smaller x-lower (r leads iff r.xl < s.xl, ties to
// s, _kernels.pyx:245): an x-in R leader scans S's x-in run from the first
// s.xl > r.xl, an x-in S leader scans R's x-in run from the first
// r.xl >= s.xl, while partner.xl <= leader.xu; an x-out leader (class C/D,
// starts left of the tile) scans the partner's x-in run from its start (all
// of them have xl >= the tile's left edge > leader.xl).  A candidate is kept
// iff the y-ranges overlap and at least one side is y-in — with the x rule
// exactly the nine class combinations AA AB AC AD BA BC CA CB DA, so the
// reference-point test (Eq. 1) never runs.  Count → one reservation per item
// → emit (second scan).
#pragma once

constexpr int kSortWin = kSortWindow;  // entries sorted per CTA in shared memory
constexpr int kSortThreads = 512;
static_assert(kSweepLeaders == kJoinThreads, "one leader per thread");

struct LargeSort {
  u64 *keyA, *keyB;   // sort keys (xl_key with the y-out bit cleared)
  u32 *posA, *posB;   // list positions
  u64* sk;            // sorted copy: key (xl_key with both labels)
  double *sxu, *syl, *syu;
  i64* sid;
  i64 cap;            // entries the arrays hold (R's large entries, then S's)
  int passes;         // merge passes launched (widths 4096 << p)
};

inline size_t large_sort_bytes(i64 cap) { return 72 * (size_t)cap + 10 * 256; }

inline LargeSort large_sort_bind(void* base, i64 cap) {
  char* b = (char*)base;
  LargeSort L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* p = b + o;
    o = align_up(o + bytes, 256);
    return p;
  };
  L.keyA = (u64*)take(8 * cap);
  L.keyB = (u64*)take(8 * cap);
  L.posA = (u32*)take(4 * cap);
  L.posB = (u32*)take(4 * cap);
  L.sk = (u64*)take(8 * cap);
  L.sxu = (double*)take(8 * cap);
  L.syl = (double*)take(8 * cap);
  L.syu = (double*)take(8 * cap);
  L.sid = (i64*)take(8 * cap);
  L.cap = cap;
  L.passes = 0;
  return L;
}

// The large-tile ranges of the two lists (header of the plan): R's large
// entries start at list position rl0, S's at sl0; combined index e < LR is
// R's entry rl0 + e, e >= LR is S's entry sl0 + (e - LR).
struct LargeGeo {
  i64 LR, LS, rl0, sl0, n_large;
};
__device__ __forceinline__ LargeGeo large_geo(const pbsm_header* hdr) {
  LargeGeo g;
  g.LR = hdr->large_r;
  g.LS = hdr->large_s;
  g.rl0 = hdr->list_r - g.LR;
  g.sl0 = hdr->list_s - g.LS;
  g.n_large = hdr->n_large;
  return g;
}

// the plan invariants the sort relies on; false → flag (the caller re-runs)
__device__ __forceinline__ bool large_fits(const LargeGeo& g, const pbsm_header* hdr,
                                           const LargeSort& L) {
  return g.LR + g.LS <= L.cap && hdr->max_huge <= ((i64)kSortWin << L.passes);
}

__device__ __forceinline__ const Rec* large_rec(const Rec* rl, const Rec* sl, const LargeGeo& g,
                                                i64 e) {
  return e < g.LR ? rl + g.rl0 + e : sl + g.sl0 + (e - g.LR);
}

// (key, pos) total order
__device__ __forceinline__ bool klt(u64 ka, u32 pa, u64 kb, u32 pb) {
  return ka < kb || (ka == kb && pa < pb);
}

// Window c (of the plan's numbering) → its segment [seg_lo, seg_hi) and its
// entries [beg, end) in the combined index space; false past the last window.
__device__ __forceinline__ bool sort_window(const uint4* __restrict__ lrec,
                                            const u32* __restrict__ lwin, const LargeGeo& g,
                                            i64 c, i64& seg_lo, i64& seg_hi, i64& beg,
                                            i64& end) {
  if (g.n_large == 0 || c >= (i64)__ldg(lwin + g.n_large)) return false;
  int lo_t = 0, hi_t = (int)g.n_large;  // the last tile whose first window is <= c
  const int lane = threadIdx.x & 31;
  while (hi_t - lo_t > 1) {
    const int step = (hi_t - lo_t + 31) >> 5;
    const int m = lo_t + lane * step;
    const unsigned le = __ballot_sync(0xffffffffu, m < hi_t && (i64)__ldg(lwin + m) <= c);
    lo_t += (31 - __clz(le)) * step;
    hi_t = min(hi_t, lo_t + step);
  }
  const uint4 r = lrec[lo_t];
  const i64 wr = (r.z + kSortWin - 1) / kSortWin;
  const i64 j = c - (i64)__ldg(lwin + lo_t);
  const bool s_side = j >= wr;
  seg_lo = s_side ? g.LR + ((i64)r.y - g.sl0) : (i64)r.x - g.rl0;
  seg_hi = seg_lo + (s_side ? r.w : r.z);
  beg = seg_lo + (s_side ? j - wr : j) * kSortWin;
  end = min(seg_hi, beg + kSortWin);
  return true;
}

// Sort every 4096-entry window of every segment (windows aligned to the
// segment start; the plan numbered them, lwin[t] = first window of large
// tile t, R's windows then S's) by (key, position) in shared memory.
__global__ void __launch_bounds__(kSortThreads) k_lsort_win(const Rec* __restrict__ rl,
                                                           const Rec* __restrict__ sl,
                                                           const uint4* __restrict__ lrec,
                                                           const u32* __restrict__ lwin,
                                                           pbsm_header* __restrict__ hdr,
                                                           LargeSort L) {
  extern __shared__ __align__(16) unsigned char ls_raw[];
  u64* sk = reinterpret_cast<u64*>(ls_raw);
  u32* sp = reinterpret_cast<u32*>(sk + kSortWin);
  const LargeGeo g = large_geo(hdr);
  if (!large_fits(g, hdr, L)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&hdr->error, PBSM_ERR_SCATTER_OVERFLOW);
    return;
  }
  i64 seg_lo, seg_hi, beg, end;
  if (!sort_window(lrec, lwin, g, blockIdx.x, seg_lo, seg_hi, beg, end)) return;
  const int n = (int)(end - beg);
  int np = 1;  // bitonic width: the next power of two >= n
  while (np < n) np <<= 1;
  for (int i = threadIdx.x; i < np; i += kSortThreads) {
    if (i < n) {
      const i64 e = beg + i;
      sk[i] = large_rec(rl, sl, g, e)->xl_key & ~kYOut;
      sp[i] = (u32)e;
    } else {
      sk[i] = ~0ull;
      sp[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < np; i += kSortThreads) {
        const int p = i ^ jj;
        if (p > i) {
          const bool up = (i & k) == 0;
          const u64 a_k = sk[i], b_k = sk[p];
          const u32 a_p = sp[i], b_p = sp[p];
          if (klt(b_k, b_p, a_k, a_p) == up) {
            sk[i] = b_k; sk[p] = a_k;
            sp[i] = b_p; sp[p] = a_p;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += kSortThreads) {
    L.keyA[beg + i] = sk[i];
    L.posA[beg + i] = sp[i];
  }
}

// one merge pass: runs of width w (from the segment start) merged pairwise,
// src → dst; a CTA per sort window, a thread per entry
__global__ void __launch_bounds__(256) k_lmerge(const uint4* __restrict__ lrec,
                                                const u32* __restrict__ lwin,
                                                const pbsm_header* __restrict__ hdr, LargeSort L,
                                                int pass) {
  const LargeGeo g = large_geo(hdr);
  if (!large_fits(g, hdr, L)) return;
  i64 lo, hi, beg, end;
  if (!sort_window(lrec, lwin, g, blockIdx.x, lo, hi, beg, end)) return;
  const u64* sk = (pass & 1) ? L.keyB : L.keyA;
  const u32* sp = (pass & 1) ? L.posB : L.posA;
  u64* dk = (pass & 1) ? L.keyA : L.keyB;
  u32* dp = (pass & 1) ? L.posA : L.posB;
  const i64 w = (i64)kSortWin << pass;
  for (i64 e = beg + threadIdx.x; e < end; e += blockDim.x) {
    const u64 k = sk[e];
    const u32 p = sp[e];
    if (hi - lo <= w) {  // the whole segment is one run already
      dk[e] = k;
      dp[e] = p;
      continue;
    }
    // runs of width w from the segment start; merge run r with run r ^ 1
    const i64 run = (e - lo) / w;
    const i64 own_lo = lo + run * w;
    const i64 bud = run ^ 1;
    const i64 b_lo = min(hi, lo + bud * w), b_hi = min(hi, lo + bud * w + w);
    const i64 out_lo = lo + (run & ~1ll) * w;
    i64 a = b_lo, b = b_hi;  // rank in the buddy run: elements (key, pos) below mine
    while (a < b) {
      const i64 m = (a + b) >> 1;
      if (klt(sk[m], sp[m], k, p)) a = m + 1; else b = m;
    }
    const i64 out = out_lo + (e - own_lo) + (a - b_lo);
    dk[out] = k;
    dp[out] = p;
  }
}

// the sorted copy the sweep reads (SoA), from the final pass' positions
__global__ void __launch_bounds__(256) k_lgather(const Rec* __restrict__ rl,
                                                 const Rec* __restrict__ sl,
                                                 const uint4* __restrict__ lrec,
                                                 const u32* __restrict__ lwin,
                                                 const pbsm_header* __restrict__ hdr,
                                                 LargeSort L) {
  const LargeGeo g = large_geo(hdr);
  if (!large_fits(g, hdr, L)) return;
  i64 lo, hi, beg, end;
  if (!sort_window(lrec, lwin, g, blockIdx.x, lo, hi, beg, end)) return;
  const u32* sp = (L.passes & 1) ? L.posB : L.posA;
  for (i64 e = beg + threadIdx.x; e < end; e += blockDim.x) {
    const Rec* r = large_rec(rl, sl, g, sp[e]);
    L.sk[e] = r->xl_key;
    L.sxu[e] = r->xu;
    L.syl[e] = r->yl;
    L.syu[e] = r->yu;
    L.sid[e] = r->id;
  }
}

// number of x-in entries of a sorted segment [lo, hi): x-out keys (bit 63) follow
__device__ __forceinline__ i64 xin_count(const LargeSort& L, i64 lo, i64 hi) {
  i64 a = lo, b = hi;
  while (a < b) {
    const i64 m = (a + b) >> 1;
    if (L.sk[m] & kXOut) b = m; else a = m + 1;
  }
  return a - lo;
}

// The CTA's 256 leaders are consecutive sorted entries, so their scan ranges
// overlap: the union of the ranges streams through shared memory in pieces
// of kSweepPiece partner entries (coalesced loads), and each leader scans its
// own range inside each piece.  Hits are kept in a list for the emit; if the
// list overflows, a second pass re-scans and emits directly.
constexpr int kSweepPiece = 1024;
constexpr int kSweepHits = 4096;

struct SweepSmem {
  u64 pk[kSweepPiece];       // partner piece: key (xl_key with labels)
  double2 py[kSweepPiece];   // {yl, yu}
  u32 hit_p[kSweepHits];     // hit: partner index (combined)
  unsigned char hit_l[kSweepHits];  // hit: leader thread
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  i64 pin_n;                 // partner's sorted x-in run length
  long long ulo, uhi;        // union of the leaders' scan ranges
  u32 nhit;
};

// [start, end) of one leader's scan in the partner's sorted x-in run
// [plo, plo + pn): from the first partner the leader leads (R: s.xl > r.xl;
// S: r.xl >= s.xl; an x-out leader: the run start) to the first partner
// with xl > leader.xu
__device__ __forceinline__ void sweep_range(const LargeSort& L, u64 mk, double mxu, bool lead_r,
                                            i64 plo, i64 pn, i64& k0, i64& k1) {
  const double mxl = key_x(mk);
  i64 a = plo, b = plo + pn;
  if (!(mk & kXOut)) {
    while (a < b) {
      const i64 m = (a + b) >> 1;
      const double x = key_x(L.sk[m]);
      if (lead_r ? (x <= mxl) : (x < mxl)) a = m + 1; else b = m;
    }
  }
  k0 = a;
  b = plo + pn;
  while (a < b) {  // first partner with xl > mxu
    const i64 m = (a + b) >> 1;
    if (key_x(L.sk[m]) <= mxu) a = m + 1; else b = m;
  }
  k1 = a;
}
