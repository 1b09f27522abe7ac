// units.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after common.cuh / partition.cuh / join.cuh).
// Contents: the unit pipeline — cell histogram, unit map, unit-major bins,
// per-unit partition + nested mini-joins while the unit's tile lists are hot
// in L2, and the deferred large tiles.
//
// Why: the tile-list pipeline (partition.cuh / join.cuh) scatters every
// tile-list entry to a random place in a ~1-GB list (one L2 atomic with return
// + one 64-byte record write per entry, DRAM-row bound) and the join reads the
// lists back from HBM.  Here the scatter to tiles happens per UNIT — one tile
// row × a column range holding a few thousand records — inside one CTA:
// shared-memory counters replace the per-tile global atomics, the unit's lists
// are written to and read from a slice of scratch that is still in L2, and the
// only HBM round trip left is the unit-major copy of the input (36 B/record).
//
//   k_ucount  (P1)  count_tiles at CELL granularity (tile row × column group
//                   of CW columns, <= 32768 cells: a shared-memory histogram)
//                   + RectBatch.validate + Σ tiles covered (A_R / A_S)
//   k_umap          cells → units: per row, consecutive cells merged until a
//                   unit holds ~target records; units where one input is
//                   empty are dead (no pair possible, nothing binned); bases
//                   of the unit-major bins; largest-first order (the
//                   reference's task queue is largest-first, engine.py:97-99)
//   k_ubin    (P2)  each rectangle → every live unit it overlaps: its 32-byte
//                   MBR and its row index, at an atomic cursor per unit
//   k_ujoin   (P3)  one CTA per unit: count_tiles over the unit's tiles
//                   (shared memory), compute_segment_offsets (block scan),
//                   write_tiles into the unit's slice of scratch (class label
//                   in the top bits of xl, as the tile-list pipeline), then
//                   the nested mini-joins of its small tiles, chunk by chunk
//                   (count → reserve → emit); tiles of more than LMAX
//                   entries are queued
//   k_ularge  (P4)  the queued tiles: work items of 256 lead × 2048 other
//                   entries over all SMs (persistent CTAs, item ticket)
#pragma once

// other-side entries per deferred large work item of the unit pipeline (its own
// constant: the tile-list pipeline's kLargeOther follows its bitmap rows)
constexpr int kULargeOther = 2048;

constexpr int kUnitMaxW = 4096;        // widest unit, in tile columns
constexpr int kUnitMaxCells = 32768;   // cells of the P1 histogram (128 KB of shared memory)
constexpr int kUnitMaxG = 64;          // column groups per tile row
constexpr u32 kDeadUnit = 0xffffffffu;
constexpr int kUCountThreads = 1024;
constexpr int kUMapThreads = 1024;
constexpr int kUJoinThreads = 256;     // = kNT: the nested chunk code's CTA shape
#ifndef PBSM_UNIT_TARGET
#define PBSM_UNIT_TARGET 3072          // records (R + S) per unit
#endif
constexpr u64 kDefItemBits = 40;       // def_packed: tiles << 40 | items

static_assert(kUJoinThreads == kNT, "the unit join reuses the nested-chunk CTA shape");

struct __align__(32) URec {  // one binned record / one tile-list entry
  u64 xl;                     // xl bits (| class label in a tile list)
  double xu, yl, yu;
};
static_assert(sizeof(URec) == 32, "URec");

struct UnitDesc {  // one unit: tile row × columns [ca, cb)
  u32 row, ca, cb, nR, nS, baseR, baseS, pad;
};
static_assert(sizeof(UnitDesc) == 32, "UnitDesc");

struct UGeo {
  int kx, ky, row_lo, row_hi, rows, G, CW, cells;
};

// Column groups: G per row, CW columns each, with rows*G <= kUnitMaxCells and
// CW <= kUnitMaxW (a unit never spans more than kUnitMaxW columns).
inline bool unit_geometry(int kx, int ky, int row_lo, int row_hi, UGeo& g) {
  if (!grid_ok(kx, ky, row_lo, row_hi)) return false;
  const int rows = row_hi - row_lo;
  int G = std::min(std::min(kUnitMaxG, kUnitMaxCells / rows), kx);
  if (G < 1) return false;
  const int CW = (kx + G - 1) / G;
  if (CW > kUnitMaxW) return false;
  G = (kx + CW - 1) / CW;  // no empty trailing group
  g.kx = kx;
  g.ky = ky;
  g.row_lo = row_lo;
  g.row_hi = row_hi;
  g.rows = rows;
  g.G = G;
  g.CW = CW;
  g.cells = rows * G;
  return g.cells <= kUnitMaxCells;
}

struct ULayout {
  size_t hdr, bx, by, bhist[2], first[2], cont[2], cell_unit, unR, unS, row_live, row_nR,
      row_nS, units, order, blk_base[2], ccur[2], cls, total;
  int nb;  // P1 / P2 blocks (a 1024-thread CTA per SM)
};

inline ULayout ulayout(const UGeo& g, int nb) {
  ULayout L;
  L.nb = nb;
  const size_t C = (size_t)g.cells, Rw = (size_t)g.rows;
  size_t o = 0;
  L.hdr = o; o = align_up(o + sizeof(pbsm_uheader), 256);
  L.bx = o; o = align_up(o + sizeof(double) * (g.kx + 1), 256);
  L.by = o; o = align_up(o + sizeof(double) * (g.ky + 1), 256);
  for (int q = 0; q < 2; ++q) { L.bhist[q] = o; o = align_up(o + 4 * C * nb, 256); }
  for (int q = 0; q < 2; ++q) { L.first[q] = o; o = align_up(o + 4 * C, 256); }
  for (int q = 0; q < 2; ++q) { L.cont[q] = o; o = align_up(o + 4 * C, 256); }
  L.cls = o; o = align_up(o + 4 * 64, 256);
  L.cell_unit = o; o = align_up(o + 4 * C, 256);
  L.unR = o; o = align_up(o + 4 * C, 256);
  L.unS = o; o = align_up(o + 4 * C, 256);
  L.row_live = o; o = align_up(o + 4 * (Rw + 1), 256);
  L.row_nR = o; o = align_up(o + 8 * (Rw + 1), 256);
  L.row_nS = o; o = align_up(o + 8 * (Rw + 1), 256);
  L.units = o; o = align_up(o + sizeof(UnitDesc) * C, 256);
  L.order = o; o = align_up(o + 4 * C, 256);
  for (int q = 0; q < 2; ++q) { L.blk_base[q] = o; o = align_up(o + 4 * C * nb, 256); }
  for (int q = 0; q < 2; ++q) { L.ccur[q] = o; o = align_up(o + 4 * C, 256); }
  L.total = o;
  return L;
}

struct UWs {
  pbsm_uheader* hdr;
  double *bx, *by;
  u32 *bhist[2], *first[2], *cont[2], *cell_unit, *unR, *unS, *row_live, *order,
      *blk_base[2], *ccur[2], *cls;
  u64 *row_nR, *row_nS;
  UnitDesc* units;
  int nb;
};

inline UWs ubind(void* base, const ULayout& L) {
  char* b = (char*)base;
  UWs w;
  w.hdr = (pbsm_uheader*)(b + L.hdr);
  w.bx = (double*)(b + L.bx);
  w.by = (double*)(b + L.by);
  for (int q = 0; q < 2; ++q) {
    w.bhist[q] = (u32*)(b + L.bhist[q]);
    w.first[q] = (u32*)(b + L.first[q]);
    w.cont[q] = (u32*)(b + L.cont[q]);
    w.blk_base[q] = (u32*)(b + L.blk_base[q]);
    w.ccur[q] = (u32*)(b + L.ccur[q]);
  }
  w.cls = (u32*)(b + L.cls);
  w.cell_unit = (u32*)(b + L.cell_unit);
  w.unR = (u32*)(b + L.unR);
  w.unS = (u32*)(b + L.unS);
  w.row_live = (u32*)(b + L.row_live);
  w.row_nR = (u64*)(b + L.row_nR);
  w.row_nS = (u64*)(b + L.row_nS);
  w.units = (UnitDesc*)(b + L.units);
  w.order = (u32*)(b + L.order);
  w.nb = L.nb;
  return w;
}

// the join scratch: [slots: URec × n | row index per slot: u32 × n |
// deferred tiles: uint4 × d | their item bases: u32 × d | queued chunks: uint4 × q]
struct UScratch {
  URec* ent;
  u32* eidx;
  uint4* dtile;
  u32* ditem;
  uint4* queue;
  u64 slots, dcap, qcap;
};
inline u64 udef_capacity(u64 slots) { return slots / (kLmax + 1) + 16; }
inline u64 uqueue_capacity(u64 slots) { return slots / 64 + 64; }
inline size_t uscratch_bytes(u64 slots) {
  const u64 d = udef_capacity(slots), q = uqueue_capacity(slots);
  return align_up(32 * slots, 256) + align_up(4 * slots, 256) + align_up(16 * d, 256) +
         align_up(4 * d, 256) + align_up(16 * q, 256);
}
inline UScratch uscratch_bind(void* base, u64 slots) {
  char* b = (char*)base;
  UScratch s;
  s.slots = slots;
  s.dcap = udef_capacity(slots);
  s.qcap = uqueue_capacity(slots);
  size_t o = 0;
  s.ent = (URec*)(b + o); o += align_up(32 * slots, 256);
  s.eidx = (u32*)(b + o); o += align_up(4 * slots, 256);
  s.dtile = (uint4*)(b + o); o += align_up(16 * s.dcap, 256);
  s.ditem = (u32*)(b + o); o += align_up(4 * s.dcap, 256);
  s.queue = (uint4*)(b + o);
  return s;
}

// P1 / P2 decomposition: block b of `nb` owns records [b*per, (b+1)*per) —
// the same ranges in both passes, so P2 can place each record exactly where
// P1's per-block counts say (no global atomic per record).
__host__ __device__ inline i64 upart_per(i64 n, int nb) { return (n + nb - 1) / nb; }
inline int upart_blocks(i64 n, int max_nb) {
  return (int)std::max<i64>(1, std::min<i64>((n + 8191) / 8192, max_nb));
}

// ---------------------------------------------------------------- init
__global__ void k_uinit(pbsm_uheader* hdr, u32* z, u64 nz, u32* cls, double* bx, int kx,
                        double* by, int ky) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 nt = (u64)gridDim.x * blockDim.x;
  if (tid < sizeof(pbsm_uheader) / 4) reinterpret_cast<u32*>(hdr)[tid] = 0u;
  if (tid < 64) cls[tid] = 0u;
  for (u64 i = tid; i <= (u64)max(kx, ky); i += nt) {
    if (i <= (u64)kx) bx[i] = __ddiv_rn((double)i, (double)kx);
    if (i <= (u64)ky) by[i] = __ddiv_rn((double)i, (double)ky);
  }
  for (u64 i = tid; i < nz; i += nt) z[i] = 0u;  // cont[2] (contiguous)
}

// ---------------------------------------------------------------- P1 cell counts
// count_tiles (_kernels.pyx:34-58) at cell granularity.  For every tile row a
// record covers, it counts once in `first` at the cell of its first covered
// column group there (a shared-memory histogram per block, written out as the
// block's row of bhist) and once in `cont` at each later group it covers
// (rare: a direct RED).  A unit made of cells [a, b) of a row then holds
// Σ first[a..b) + cont[a] records — each record once.  Validation
// (RectBatch.validate, geometry.py:166-177) rides along, and Σ tiles covered
// gives A_R / A_S (PartitionedDataset.total_assigned).
template <typename F>
__device__ __forceinline__ void urec_cells(double a, double b, double c, double d, const UGeo& g,
                                           const double* bx, const double* by, F&& f) {
  const int r0 = max(tile_of(c, g.ky, by), g.row_lo);
  const int r1 = min(tile_of(d, g.ky, by), g.row_hi - 1);
  if (r0 > r1) return;
  const int c0 = tile_of(a, g.kx, bx), c1 = tile_of(b, g.kx, bx);
  f(r0, r1, c0, c1, c0 / g.CW, c1 / g.CW);
}

__global__ void __launch_bounds__(kUCountThreads, 1) k_ucount(
    const double* __restrict__ xl, const double* __restrict__ xu, const double* __restrict__ yl,
    const double* __restrict__ yu, i64 n, UGeo g, const double* __restrict__ bx,
    const double* __restrict__ by, u32* __restrict__ bhist, u32* __restrict__ cont,
    pbsm_uheader* hdr, int side) {
  extern __shared__ u32 uhist[];
  for (int c = threadIdx.x; c < g.cells; c += kUCountThreads) uhist[c] = 0u;
  __syncthreads();
  const i64 per = upart_per(n, gridDim.x);
  const i64 beg = min(n, (i64)blockIdx.x * per), end = min(n, beg + per);
  u64 acov = 0;
  u32 bad = 0;
  i64 i = beg + threadIdx.x;
  double a = 0, b = 0, c = 0, d = 0;
  if (i < end) {
    a = __ldcs(xl + i);
    b = __ldcs(xu + i);
    c = __ldcs(yl + i);
    d = __ldcs(yu + i);
  }
  for (; i < end; i += kUCountThreads) {
    const i64 nx = i + kUCountThreads;
    double na = 0, nb = 0, nc = 0, nd = 0;
    if (nx < end) {
      na = __ldcs(xl + nx);
      nb = __ldcs(xu + nx);
      nc = __ldcs(yl + nx);
      nd = __ldcs(yu + nx);
    }
    if (!(a <= b) || !(c <= d)) bad |= PBSM_ERR_INVERTED;
    if (a < 0.0 || c < 0.0 || b > 1.0 || d > 1.0) bad |= PBSM_ERR_RANGE;
    urec_cells(a, b, c, d, g, bx, by, [&](int r0, int r1, int c0, int c1, int j0, int j1) {
      acov += (u64)(c1 - c0 + 1) * (u64)(r1 - r0 + 1);
      for (int r = r0; r <= r1; ++r) {
        const int base = (r - g.row_lo) * g.G;
        atomicAdd_block(&uhist[base + j0], 1u);
        for (int j = j0 + 1; j <= j1; ++j) atomicAdd(&cont[base + j], 1u);
      }
    });
    a = na;
    b = nb;
    c = nc;
    d = nd;
  }
  if (bad) atomicOr(&hdr->error, bad << (2 * side));
#pragma unroll
  for (int o = 16; o; o >>= 1) acov += __shfl_down_sync(0xffffffffu, acov, o);
  if ((threadIdx.x & 31) == 0 && acov)
    atomicAdd(reinterpret_cast<unsigned long long*>(side ? &hdr->a_s : &hdr->a_r), acov);
  __syncthreads();
  u32* out = bhist + (size_t)blockIdx.x * g.cells;
  for (int cc = threadIdx.x; cc < g.cells; cc += kUCountThreads) out[cc] = uhist[cc];
}

// cell totals of `first` (Σ over the P1 blocks of each side)
__global__ void k_ucell_sum(const u32* __restrict__ bhR, int nbR, const u32* __restrict__ bhS,
                            int nbS, int cells, u32* __restrict__ fR, u32* __restrict__ fS) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * cells) return;
  const int side = t >= cells, c = side ? t - cells : t;
  const u32* h = side ? bhS : bhR;
  const int nb = side ? nbS : nbR;
  u32 v = 0;
  for (int b = 0; b < nb; ++b) v += __ldcs(h + (size_t)b * cells + c);
  (side ? fS : fR)[c] = v;
}

// ---------------------------------------------------------------- unit map
// Per tile row (a warp each): consecutive cells are merged into a unit until
// adding the next cell would pass `target` records or kUnitMaxW columns.  A
// unit with an empty input side can produce no pair (build_task_queue joins
// only tiles with both inputs, engine.py:97): it is dead, and nothing is
// binned into it.  Then (k_umap_scan, one CTA) prefixes over rows, and
// (k_umap_write) the descriptors, the cell → unit map, the largest-first
// order (size classes, as the reference's largest-first task queue,
// engine.py:97-99) and each P1 block's first slot in every unit.
constexpr int kMapRowsPerBlock = 8;  // 256 threads, a warp per row

__device__ __forceinline__ int size_class(u32 v) { return 31 - __clz(max(v, 1u)); }

__global__ void __launch_bounds__(256) k_umap_rows(UGeo g, const u32* __restrict__ fR,
                                                   const u32* __restrict__ cR,
                                                   const u32* __restrict__ fS,
                                                   const u32* __restrict__ cS, u32 target,
                                                   u32* __restrict__ cell_local,
                                                   u32* __restrict__ unR, u32* __restrict__ unS,
                                                   u32* __restrict__ row_live,
                                                   u64* __restrict__ row_nR,
                                                   u64* __restrict__ row_nS, u32* cls,
                                                   pbsm_uheader* hdr) {
  __shared__ u32 sf[kMapRowsPerBlock][4][kUnitMaxG];
  __shared__ u32 hist[32];
  __shared__ u32 bmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kMapRowsPerBlock + warp;
  if (threadIdx.x < 32) hist[threadIdx.x] = 0u;
  if (threadIdx.x == 0) bmax = 0u;
  __syncthreads();
  u32 mx = 0;
  if (row < g.rows) {
    const int base = row * g.G;
    for (int j = lane; j < g.G; j += 32) {
      sf[warp][0][j] = fR[base + j];
      sf[warp][1][j] = cR[base + j];
      sf[warp][2][j] = fS[base + j];
      sf[warp][3][j] = cS[base + j];
    }
    __syncwarp();
    if (lane == 0) {
      u32 live = 0;
      u64 tR = 0, tS = 0;
      int start = 0;
      u32 nR = sf[warp][1][0] + sf[warp][0][0], nS = sf[warp][3][0] + sf[warp][2][0];
      auto close = [&](int a, int b) {
        const bool ok = nR && nS;
        for (int j = a; j < b; ++j) cell_local[base + j] = ok ? live : kDeadUnit;
        if (ok) {
          unR[base + live] = nR;
          unS[base + live] = nS;
          tR += nR;
          tS += nS;
          mx = max(mx, nR + nS);
          atomicAdd_block(&hist[size_class(nR + nS)], 1u);
          ++live;
        }
      };
      for (int j = 1; j < g.G; ++j) {
        const u32 a = sf[warp][0][j], b = sf[warp][2][j];
        const bool wide = (j + 1 - start) * g.CW > kUnitMaxW;
        if ((nR + nS > 0 && nR + nS + a + b > target) || wide) {
          close(start, j);
          start = j;
          nR = sf[warp][1][j] + a;
          nS = sf[warp][3][j] + b;
        } else {
          nR += a;
          nS += b;
        }
      }
      close(start, g.G);
      row_live[row] = live;
      row_nR[row] = tR;
      row_nS[row] = tS;
    }
  }
  if (lane == 0 && mx) atomicMax_block(&bmax, mx);
  __syncthreads();
  if (threadIdx.x < 32 && hist[threadIdx.x]) atomicAdd(&cls[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0 && bmax)
    atomicMax(reinterpret_cast<unsigned long long*>(&hdr->max_unit), (u64)bmax);
}

// One CTA: exclusive prefixes over rows (units, R records, S records) and
// over the size classes (descending: largest first); totals → header.
__global__ void __launch_bounds__(kUMapThreads) k_umap_scan(UGeo g, u32* __restrict__ row_live,
                                                            u64* __restrict__ row_nR,
                                                            u64* __restrict__ row_nS, u32* cls,
                                                            pbsm_uheader* hdr) {
  __shared__ u64 sh[kUMapThreads / 32][3];
  __shared__ u64 carry[3];
  const int tid = threadIdx.x;
  if (tid < 3) carry[tid] = 0;
  __syncthreads();
  for (int r0 = 0; r0 < g.rows; r0 += kUMapThreads) {
    const int r = r0 + tid;
    u64 v[3] = {r < g.rows ? row_live[r] : 0u, r < g.rows ? row_nR[r] : 0ull,
                r < g.rows ? row_nS[r] : 0ull};
    u64 tot[3];
    block_excl_scan_multi<kUMapThreads, 3, u64>(v, tot, sh);
    if (r < g.rows) {
      row_live[r] = (u32)(carry[0] + v[0]);
      row_nR[r] = carry[1] + v[1];
      row_nS[r] = carry[2] + v[2];
    }
    __syncthreads();
    if (tid < 3) carry[tid] += tot[tid];
    __syncthreads();
  }
  if (tid == 0) {
    u32 run = 0;
    for (int c = 31; c >= 0; --c) {  // class cursors (cls[32 + c]), largest class first
      cls[32 + c] = run;
      run += cls[c];
    }
    hdr->n_units = (i64)carry[0];
    hdr->bin_r = (i64)carry[1];
    hdr->bin_s = (i64)carry[2];
    hdr->cells = g.cells;
    hdr->group_cols = g.CW;
    if (carry[1] > 0xffffffffull || carry[2] > 0xffffffffull)
      atomicOr(&hdr->error, PBSM_ERR_TOTAL_RANGE);
  }
}

// Per row (a warp): the live units' descriptors, the cell → unit map, the
// order slots, and for every P1 block b and side the block's first slot in
// the unit (exclusive prefix over blocks of the block's `first` counts in the
// unit's cells), plus the continuation cursors after the `first` records.
__global__ void __launch_bounds__(256) k_umap_write(
    UGeo g, u32* __restrict__ cell_unit, const u32* __restrict__ unR, const u32* __restrict__ unS,
    const u32* __restrict__ row_live, const u64* __restrict__ row_nR,
    const u64* __restrict__ row_nS, u32* cls, UnitDesc* __restrict__ units,
    u32* __restrict__ order, const u32* __restrict__ bhR, int nbR, const u32* __restrict__ bhS,
    int nbS, u32* __restrict__ bbR, u32* __restrict__ bbS, u32* __restrict__ ccR,
    u32* __restrict__ ccS) {
  __shared__ u32 hist[32], hbase[32];
  __shared__ u32 uid[kMapRowsPerBlock][kUnitMaxG];
  __shared__ unsigned char ucls[kMapRowsPerBlock][kUnitMaxG];
  __shared__ u32 urank[kMapRowsPerBlock][kUnitMaxG];
  __shared__ int nun[kMapRowsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kMapRowsPerBlock + warp;
  if (threadIdx.x < 32) hist[threadIdx.x] = 0u;
  if (lane == 0) nun[warp] = 0;
  __syncthreads();
  if (row < g.rows) {
    const int base = row * g.G;
    const u32 u0 = row_live[row];
    u64 bR = row_nR[row], bS = row_nS[row];
    int a = 0, k = 0;
    while (a < g.G) {
      const u32 loc = cell_unit[base + a];  // local id (k_umap_rows)
      int b = a + 1;
      while (b < g.G && cell_unit[base + b] == loc) ++b;
      if (loc == kDeadUnit) {
        a = b;
        continue;
      }
      const u32 id = u0 + loc;
      const u32 nR = unR[base + loc], nS = unS[base + loc];
      if (lane == 0) {
        UnitDesc u;
        u.row = (u32)(row + g.row_lo);
        u.ca = (u32)(a * g.CW);
        u.cb = (u32)min(g.kx, b * g.CW);
        u.nR = nR;
        u.nS = nS;
        u.baseR = (u32)bR;
        u.baseS = (u32)bS;
        u.pad = 0;
        units[id] = u;
        const int c = size_class(nR + nS);
        uid[warp][k] = id;
        ucls[warp][k] = (unsigned char)c;
        urank[warp][k] = atomicAdd_block(&hist[c], 1u);
      }
      // each P1 block's first slot in this unit, both sides (lanes over blocks)
      for (int side = 0; side < 2; ++side) {
        const u32* bh = side ? bhS : bhR;
        const int nb = side ? nbS : nbR;
        u32* bbp = side ? bbS : bbR;
        u32 carry = (u32)(side ? bS : bR);
        for (int b0 = 0; b0 < nb; b0 += 32) {
          const int blk = b0 + lane;
          u32 v = 0;
          if (blk < nb)
            for (int j = a; j < b; ++j) v += bh[(size_t)blk * g.cells + base + j];
          const u32 inc = warp_incl_scan<u32>(v);
          if (blk < nb) bbp[(size_t)blk * g.cells + id] = carry + inc - v;
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) (side ? ccS : ccR)[id] = carry;  // continuation records follow
      }
      bR += nR;
      bS += nS;
      ++k;
      a = b;
    }
    if (lane == 0) nun[warp] = k;
    __syncwarp();
    for (int j = lane; j < g.G; j += 32) {
      const u32 loc = cell_unit[base + j];
      cell_unit[base + j] = loc == kDeadUnit ? kDeadUnit : u0 + loc;
    }
  }
  __syncthreads();
  // largest-first order: one global cursor bump per size class and block
  if (threadIdx.x < 32 && hist[threadIdx.x])
    hbase[threadIdx.x] = atomicAdd(&cls[32 + threadIdx.x], hist[threadIdx.x]);
  __syncthreads();
  for (int k = lane; k < nun[warp]; k += 32)
    order[hbase[ucls[warp][k]] + urank[warp][k]] = uid[warp][k];
}

// ---------------------------------------------------------------- P2 bins
#ifndef PBSM_UBIN_MODE
#define PBSM_UBIN_MODE 0
#endif
#ifndef PBSM_UBIN_NOIDX
#define PBSM_UBIN_NOIDX 0
#endif
#ifndef PBSM_UBIN_NOREC
#define PBSM_UBIN_NOREC 0
#endif
#ifndef PBSM_UBIN_IDXHINT
#define PBSM_UBIN_IDXHINT 1  // row-index stores: L2 evict_last (their sectors fill slowly)
#endif
#ifndef PBSM_UBIN_RECHINT
#define PBSM_UBIN_RECHINT 1  // record stores: L2 evict_first (full sectors, never re-read soon)
#endif
__device__ __forceinline__ void st_u32_hint(u32* p, u32 v, u64 pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_urec(URec* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)),
               "l"(__double_as_longlong(c)), "l"(__double_as_longlong(d))
               : "memory");
}

__device__ __forceinline__ void st_urec_hint(URec* p, double a, double b, double c, double d,
                                             u64 pol) {
  asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
               "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)),
               "l"(__double_as_longlong(c)), "l"(__double_as_longlong(d)), "l"(pol)
               : "memory");
}

// Each rectangle → every live unit it overlaps, into the unit-major bins.
// Block b owns the same records as in P1, so its `first` records of unit u
// go to [bb[b][u], ...) at a shared-memory cursor (no global atomic, no
// contention on the hot units of clustered data); a record's later units in a
// row (it crosses a column-group boundary; rare) take a global cursor.
__global__ void __launch_bounds__(kUCountThreads, 1) k_ubin(
    const double* __restrict__ xl, const double* __restrict__ xu, const double* __restrict__ yl,
    const double* __restrict__ yu, i64 n, UGeo g, const double* __restrict__ bx,
    const double* __restrict__ by, const u32* __restrict__ cell_unit,
    const u32* __restrict__ bb, u32* __restrict__ ccur, URec* __restrict__ bin,
    u32* __restrict__ bidx, i64 cap, pbsm_uheader* hdr) {
  extern __shared__ u32 bcur[];
  u64 pol_keep, pol_drop;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_drop));
  const u32 U = (u32)hdr->n_units;
  const u32* mine = bb + (size_t)blockIdx.x * g.cells;
  for (u32 u = threadIdx.x; u < U; u += kUCountThreads) bcur[u] = mine[u];
  __syncthreads();
  const i64 per = upart_per(n, gridDim.x);
  const i64 beg = min(n, (i64)blockIdx.x * per), end = min(n, beg + per);
  u32 bad = 0;
  i64 i = beg + threadIdx.x;
  double pa = 0, pb = 0, pc = 0, pd = 0;
  if (i < end) {
    pa = __ldcs(xl + i);
    pb = __ldcs(xu + i);
    pc = __ldcs(yl + i);
    pd = __ldcs(yu + i);
  }
  for (; i < end; i += kUCountThreads) {
    const double a = pa, b = pb, c = pc, d = pd;
    const i64 nx = i + kUCountThreads;
    if (nx < end) {
      pa = __ldcs(xl + nx);
      pb = __ldcs(xu + nx);
      pc = __ldcs(yl + nx);
      pd = __ldcs(yu + nx);
    }
    urec_cells(a, b, c, d, g, bx, by, [&](int r0, int r1, int, int, int j0, int j1) {
      for (int r = r0; r <= r1; ++r) {
        const u32* cu = cell_unit + (r - g.row_lo) * g.G;
        u32 prev = __ldg(cu + j0);
        if (prev != kDeadUnit) {
#if PBSM_UBIN_MODE == 1  // diagnostic: one global cursor per unit (block 0's base row)
          const u32 slot = atomicAdd(const_cast<u32*>(bb) + prev, 1u);
#else
          const u32 slot = atomicAdd_block(&bcur[prev], 1u);
#endif
          if ((i64)slot < cap) {
#if !PBSM_UBIN_NOREC
#if PBSM_UBIN_RECHINT
            st_urec_hint(bin + slot, a, b, c, d, pol_drop);
#else
            st_urec(bin + slot, a, b, c, d);
#endif
#endif
#if !PBSM_UBIN_NOIDX
#if PBSM_UBIN_IDXHINT
            st_u32_hint(bidx + slot, (u32)i, pol_keep);
#else
            bidx[slot] = (u32)i;
#endif
#endif
          } else {
            bad |= PBSM_ERR_SCATTER_OVERFLOW;
          }
        }
        for (int j = j0 + 1; j <= j1; ++j) {
          const u32 u = __ldg(cu + j);
          if (u == prev || u == kDeadUnit) {
            prev = u;
            continue;
          }
          prev = u;
          const u32 slot = atomicAdd(ccur + u, 1u);
          if ((i64)slot < cap) {
            st_urec(bin + slot, a, b, c, d);
            bidx[slot] = (u32)i;
          } else {
            bad |= PBSM_ERR_SCATTER_OVERFLOW;
          }
        }
      }
    });
  }
  if (bad) atomicOr(&hdr->error, bad);
}

// ---------------------------------------------------------------- P3 unit join
// The unit's scratch region (32-byte slots, 4-slot = 128-byte aligned):
//   [tile records of its small tiles: uint4 {r_off, s_off, nR | nS << 8, -}]
//   [chunk descriptors: uint4 {first small tile, r_off, s_off, -}, + closing]
//   [small tiles' R entries | small tiles' S entries]   (tile order)
//   [deferred tiles' R entries | deferred tiles' S entries]
// Offsets are absolute slot indices.  A chunk = consecutive small tiles whose
// last entry falls in the same bucket of kChunkBN entries (as in k_plan_apply),
// so its R and S entries are two contiguous slot ranges.
struct UJoinArgs {
  UGeo g;
  const double* bx;
  const double* by;
  const UnitDesc* units;
  const u32* order;
  pbsm_uheader* hdr;
  const URec* bin[2];
  const u32* bidx[2];
  i64 bcap[2];
  const i64* ids[2];
  UScratch sc;
  i64* pairs;
  i64 capacity;
};

struct UNestBuf {          // one staged chunk
  ulonglong2 ax[kCapN];    // {xl | label, xu} per entry (R range, then S range)
  double2 ay[kCapN];       // {yl, yu}
  u32 aidx[kCapN];         // row index
  uint4 jr[kMaxTilesN];    // tile records
};

struct UNestSmem {
  UNestBuf buf;
  u32 lead[kCapN];         // lead entry pos | o0 << 9 | |other| << 18 | R-leads << 25
  u64 wtot[kNT / 32 + 1];
  u32 scan32[kNT / 32 + 1];
  u32 hits[kNT / 32][kHitCap];
  u64 base;
};

constexpr int kUL = 8;  // plan lanes: small R/S/tiles, deferred R/S/tiles/items, chunks
struct UJoinSmem {
  union {
    u32 cnt[2][kUnitMaxW];  // phases A-C: per-tile counts, then cursors
    UNestSmem nest;         // phase D
  } u;
  u32 shs[kUJoinThreads / 32][kUL];
  u32 tot[kUL];
  u64 base;                 // the unit's first slot (~0: not allocated)
  u32 dt0, di0;             // first deferred tile / item of the unit
  u32 wrote[kUJoinThreads / 32];
};

__device__ __forceinline__ URec ld_urec(const URec* p) {
  URec r;
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(r.xl), "=l"(*reinterpret_cast<u64*>(&r.xu)),
                 "=l"(*reinterpret_cast<u64*>(&r.yl)), "=l"(*reinterpret_cast<u64*>(&r.yu))
               : "l"(p));
  return r;
}

__device__ __forceinline__ u32 large_items(u32 a, u32 b) {
  const u32 lead = a >= b ? a : b, other = a >= b ? b : a;
  return ((lead + kLargeLead - 1) / kLargeLead) * ((other + kULargeOther - 1) / kULargeOther);
}

__device__ __forceinline__ i64 map_id(const i64* ids, u32 row) { return ids ? __ldg(ids + row) : (i64)row; }

// Nested mini-joins of one staged chunk (row form: one lane per entry of a
// tile's larger side, looping over its other side), hits ballot-compacted
// into per-warp lists, one reservation per chunk, ids looked up at the emit.
// Same tests as nested_chunk (join.cuh) on the unit layout.
__device__ __forceinline__ void unit_chunk(UNestSmem& S, const UJoinArgs& A, int nt, int NR,
                                           u32 R0, u32 S0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kNT / 32;
  const unsigned lt_mask = (1u << lane) - 1u;
  const UNestBuf& B = S.buf;
  uint4 tr = make_uint4(0, 0, 0, 0);
  u32 w = 0;
  if (tid < nt) {
    tr = B.jr[tid];
    w = max(tr.z & 0xffu, tr.z >> 8);
  }
  u32 W;
  const u32 pre = block_excl_scan32<kNT>(w, &W, S.scan32);
  if (tid < nt) {
    const u32 nr = tr.z & 0xffu, ns = tr.z >> 8;
    const u32 r0 = tr.x - R0, s0 = (u32)NR + (tr.y - S0);
    const bool lr = nr >= ns;
    const u32 nL = lr ? nr : ns, nO = lr ? ns : nr;
    const u32 l0 = lr ? r0 : s0, o0 = lr ? s0 : r0;
    const u32 d = (o0 << 9) | (nO << 18) | ((u32)lr << 25);
    for (u32 i = 0; i < nL; ++i) S.lead[pre + i] = (l0 + i) | d;
  }
  __syncthreads();
  u32 wcnt = 0;
  for (u32 g0 = 32u * warp; g0 < W; g0 += 32u * kW) {
    const u32 ei = g0 + lane;
    const bool valid = ei < W;
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
      if (hit) {
        const u32 o = wcnt + __popc(m & lt_mask);
        const u32 pr = lr ? pos : o0 + j, ps = lr ? o0 + j : pos;
        if (o < (u32)kHitCap) S.hits[warp][o] = pr | (ps << 16);
      }
      wcnt += __popc(m);
    }
  }
  if (lane == 0) S.wtot[warp] = wcnt;
  __syncthreads();
  if (tid == 0) {
    u64 t = 0;
    for (int v = 0; v < kW; ++v) {
      const u64 x = S.wtot[v];
      S.wtot[v] = t;
      t += x;
    }
    S.base = t ? atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->pairs), t) : 0ull;
    if (t && (i64)(S.base + t) > A.capacity) {
      atomicOr(&A.hdr->jerror, PBSM_ERR_PAIR_OVERFLOW);
      S.base = ~0ull;
    }
  }
  __syncthreads();
  if (S.base == ~0ull || wcnt == 0) return;
  i64* out = A.pairs + 2 * (i64)(S.base + S.wtot[warp]);
  if (wcnt <= (u32)kHitCap) {
    for (u32 i = lane; i < wcnt; i += 32u) {
      const u32 v = S.hits[warp][i];
      *reinterpret_cast<longlong2*>(out + 2 * (i64)i) =
          make_longlong2(map_id(A.ids[0], B.aidx[v & 0xffffu]), map_id(A.ids[1], B.aidx[v >> 16]));
    }
    return;
  }
  // more hits than the list holds: re-test the warp's slice in the same order
  for (u32 g0 = 32u * warp; g0 < W; g0 += 32u * kW) {
    const u32 ei = g0 + lane;
    const bool valid = ei < W;
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
      if (hit) {
        const u32 pr = lr ? pos : o0 + j, ps = lr ? o0 + j : pos;
        *reinterpret_cast<longlong2*>(out + 2 * (i64)__popc(m & lt_mask)) =
            make_longlong2(map_id(A.ids[0], B.aidx[pr]), map_id(A.ids[1], B.aidx[ps]));
      }
      out += 2 * (i64)__popc(m);
    }
  }
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}

#ifndef PBSM_UJOIN_MINB
#define PBSM_UJOIN_MINB 4
#endif
#ifndef PBSM_UNIT_ILP
#define PBSM_UNIT_ILP 4
#endif
constexpr int kUB = PBSM_UNIT_ILP;     // unit records per thread in flight (phases A, C)
#ifndef PBSM_LOCAL_CHUNKS
#define PBSM_LOCAL_CHUNKS 16
#endif
constexpr int kLocalChunks = PBSM_LOCAL_CHUNKS;  // more → queued for k_uchunks
__device__ __forceinline__ void unit_stage_and_join(UNestSmem& N, const UJoinArgs& A,
                                                    const uint4* cdesc, const uint4* jrec,
                                                    u32 c);
__global__ void __launch_bounds__(kUJoinThreads, PBSM_UJOIN_MINB) k_ujoin(UJoinArgs A) {
  __shared__ __align__(128) UJoinSmem S;
  const int tid = threadIdx.x;
  if ((i64)blockIdx.x >= A.hdr->n_units) return;
  const UnitDesc ud = A.units[A.order[blockIdx.x]];
  const int W = (int)(ud.cb - ud.ca), ca = (int)ud.ca, row = (int)ud.row;
  const int nR = (int)ud.nR, N = (int)(ud.nR + ud.nS);
  if ((i64)ud.baseR + ud.nR > A.bcap[0] || (i64)ud.baseS + ud.nS > A.bcap[1]) {
    if (tid == 0) atomicOr(&A.hdr->jerror, PBSM_ERR_SCATTER_OVERFLOW);
    return;
  }
  const URec* bin[2] = {A.bin[0] + ud.baseR, A.bin[1] + ud.baseS};
  const u32* bidx[2] = {A.bidx[0] + ud.baseR, A.bidx[1] + ud.baseS};
  const int kx = A.g.kx;
  u32* cnt0 = S.u.cnt[0];
  u32* cnt1 = S.u.cnt[1];
  for (int t = tid; t < W; t += kUJoinThreads) {
    cnt0[t] = 0u;
    cnt1[t] = 0u;
  }
  __syncthreads();
  // ---- A: count_tiles over the unit's tiles (_kernels.pyx:34-58); kUB
  // records per thread in flight (the unit's records come from HBM)
  for (int e0 = tid; e0 < N; e0 += kUB * kUJoinThreads) {
    URec r[kUB];
#pragma unroll
    for (int q = 0; q < kUB; ++q) {
      const int e = e0 + q * kUJoinThreads;
      if (e < N) r[q] = ld_urec(e >= nR ? bin[1] + (e - nR) : bin[0] + e);
    }
#pragma unroll
    for (int q = 0; q < kUB; ++q) {
      const int e = e0 + q * kUJoinThreads;
      if (e >= N) break;
      const int c0 = tile_of(__longlong_as_double((long long)r[q].xl), kx, A.bx);
      const int c1 = tile_of(r[q].xu, kx, A.bx);
      const int lo = max(c0, ca) - ca, hi = min(c1, ca + W - 1) - ca;
      u32* cn = e >= nR ? cnt1 : cnt0;
      for (int t = lo; t <= hi; ++t) atomicAdd_block(cn + t, 1u);
    }
  }
  __syncthreads();
  // ---- B: compute_segment_offsets + the unit's task plan (build_task_queue,
  // engine.py:84-100): small tiles (|R_T|+|S_T| <= LMAX) → nested chunks
  // here; larger tiles → the deferred queue (k_ularge)
  const int tpt = (W + kUJoinThreads - 1) / kUJoinThreads;
  const int t0 = min(W, tid * tpt), t1 = min(W, t0 + tpt);
  u32 v[kUL];
#pragma unroll
  for (int q = 0; q < kUL; ++q) v[q] = 0;
  for (int t = t0; t < t1; ++t) {
    const u32 a = cnt0[t], b = cnt1[t];
    if (a == 0u || b == 0u) continue;
    if (a + b <= (u32)kLmax) {
      v[0] += a;
      v[1] += b;
      v[2] += 1u;
    } else {
      v[3] += a;
      v[4] += b;
      v[5] += 1u;
      v[6] += large_items(a, b);
    }
  }
  {
    u32 tot[kUL];
    block_excl_scan_multi<kUJoinThreads, kUL, u32>(v, tot, S.shs);
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < kUL; ++q) S.tot[q] = tot[q];
      const u32 small = tot[0] + tot[1];
      const u32 nch = small ? (small - 1) / kChunkBN + 1 : 0u;
      const u64 jslots = ((u64)tot[2] + 1) / 2, cslots = ((u64)nch + 2) / 2;
      const u64 region = align_up(align_up(jslots, 4) + align_up(cslots, 4) + small + tot[3] + tot[4], 4);
      u64 base = atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->scratch_used), region);
      if (base + region > A.sc.slots) {
        atomicOr(&A.hdr->jerror, PBSM_ERR_SCATTER_OVERFLOW);
        base = ~0ull;
      }
      S.base = base;
      S.tot[7] = nch;
      S.dt0 = S.di0 = 0;
      if (tot[5]) {
        const u64 p = atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->def_packed),
                                ((u64)tot[5] << kDefItemBits) | (u64)tot[6]);
        const u64 dt = p >> kDefItemBits, di = p & ((1ull << kDefItemBits) - 1);
        if (dt + tot[5] > A.sc.dcap || di + tot[6] > 0xffffffffull) {
          atomicOr(&A.hdr->jerror, PBSM_ERR_SCATTER_OVERFLOW);
          S.base = ~0ull;
        }
        S.dt0 = (u32)dt;
        S.di0 = (u32)di;
      }
    }
  }
  __syncthreads();
  const u64 base = S.base;
  if (base == ~0ull) return;
  const u32 tsR = S.tot[0], tsS = S.tot[1], tsT = S.tot[2], tdR = S.tot[3];
  const u32 nch = S.tot[7];
  const u64 jslots = align_up(((u64)tsT + 1) / 2, 4), cslots = align_up(((u64)nch + 2) / 2, 4);
  uint4* jrec = reinterpret_cast<uint4*>(A.sc.ent + base);
  uint4* cdesc = reinterpret_cast<uint4*>(A.sc.ent + base + jslots);
  const u64 sbase = base + jslots + cslots;              // small R entries
  const u64 dbase = sbase + tsR + tsS;                   // deferred R entries
  for (int t = t0; t < t1; ++t) {
    const u32 a = cnt0[t], b = cnt1[t];
    u32 ro = 0xffffffffu, so = 0xffffffffu;
    if (a && b) {
      if (a + b <= (u32)kLmax) {
        ro = (u32)(sbase + v[0]);
        so = (u32)(sbase + tsR + v[1]);
        const u32 st = v[0] + v[1], en = st + a + b;
        jrec[v[2]] = make_uint4(ro, so, a | (b << 8), en);
        const u32 ce = (en - 1) / kChunkBN;
        if (st == 0 || (st - 1) / kChunkBN < ce) cdesc[ce] = make_uint4(v[2], ro, so, 0u);
        v[0] += a;
        v[1] += b;
        v[2] += 1u;
      } else {
        ro = (u32)(dbase + v[3]);
        so = (u32)(dbase + tdR + v[4]);
        A.sc.dtile[S.dt0 + v[5]] = make_uint4(ro, so, a, b);
        A.sc.ditem[S.dt0 + v[5]] = S.di0 + v[6];
        v[3] += a;
        v[4] += b;
        v[5] += 1u;
        v[6] += large_items(a, b);
      }
    }
    cnt0[t] = ro;
    cnt1[t] = so;
  }
  if (tid == 0 && nch) cdesc[nch] = make_uint4(tsT, (u32)(sbase + tsR), (u32)(sbase + tsR + tsS), 0u);
  __syncthreads();
  // ---- C: write_tiles (_kernels.pyx:61-98) into the unit's slots, labelled
  // with the entry's class in each tile (x-out: starts left of the tile's
  // column; y-out: starts below this row)
  u32 wrote = 0;
  for (int e0 = tid; e0 < N; e0 += kUB * kUJoinThreads) {
    URec rr[kUB];
    u32 ix[kUB];
#pragma unroll
    for (int q = 0; q < kUB; ++q) {
      const int e = e0 + q * kUJoinThreads;
      if (e < N) {
        const int side = e >= nR;
        const int k = side ? e - nR : e;
        rr[q] = ld_urec(bin[side] + k);
        ix[q] = __ldg(bidx[side] + k);
      }
    }
#pragma unroll
    for (int q = 0; q < kUB; ++q) {
      const int e = e0 + q * kUJoinThreads;
      if (e >= N) break;
      const URec& r = rr[q];
      const double xl = __longlong_as_double((long long)r.xl);
      const int c0 = tile_of(xl, kx, A.bx), c1 = tile_of(r.xu, kx, A.bx);
      const u64 key = xl_bits(xl) | ((tile_of(r.yl, A.g.ky, A.by) != row) ? kYOut : 0ull);
      const int lo = max(c0, ca), hi = min(c1, ca + W - 1);
      u32* cn = e >= nR ? cnt1 : cnt0;
      for (int c = lo; c <= hi; ++c) {
        if (cn[c - ca] == 0xffffffffu) continue;  // not a join tile
        const u32 slot = atomicAdd_block(cn + (c - ca), 1u);
        st_urec(A.sc.ent + slot,
                __longlong_as_double((long long)(key | (c != c0 ? kXOut : 0ull))), r.xu, r.yl,
                r.yu);
        A.sc.eidx[slot] = ix[q];
        ++wrote;
      }
    }
  }
  // write guard (partition.py:229-233): the unit's entries written == counted
#pragma unroll
  for (int o = 16; o; o >>= 1) wrote += __shfl_down_sync(0xffffffffu, wrote, o);
  if ((tid & 31) == 0) S.wrote[tid >> 5] = wrote;
  __syncthreads();
  if (tid == 0) {
    u32 w = 0;
    for (int q = 0; q < kUJoinThreads / 32; ++q) w += S.wrote[q];
    if (w != tsR + tsS + tdR + S.tot[4]) atomicOr(&A.hdr->jerror, PBSM_ERR_OFFSET_MISMATCH);
  }
  // ---- D: the nested mini-joins, chunk by chunk (the counters are dead:
  // their shared memory becomes the staging buffer).  A unit with many chunks
  // queues them for k_uchunks instead, so one heavy unit does not serialise
  // its chunks on one SM.
  if (nch > (u32)kLocalChunks) {
    __syncthreads();
    if (tid == 0) {
      const u64 q0 = atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->nq), (u64)nch);
      S.base = q0 + nch <= A.sc.qcap ? q0 : ~0ull;
      if (S.base == ~0ull) atomicOr(&A.hdr->jerror, PBSM_ERR_SCATTER_OVERFLOW);
    }
    __syncthreads();
    if (S.base != ~0ull)
      for (u32 c = tid; c < nch; c += kUJoinThreads)
        A.sc.queue[S.base + c] = make_uint4((u32)(base + jslots), c, (u32)base, 0u);
    return;
  }
  for (u32 c = 0; c < nch; ++c) {
    __syncthreads();  // previous chunk consumed (and, for c = 0, the slots written)
    unit_stage_and_join(S.u.nest, A, cdesc, jrec, c);
  }
}

// stage chunk c of a unit (descriptors cdesc, tile records jrec) and join it
__device__ __forceinline__ void unit_stage_and_join(UNestSmem& N, const UJoinArgs& A,
                                                    const uint4* cdesc, const uint4* jrec,
                                                    u32 c) {
  const int tid = threadIdx.x;
  const uint4 d0 = cdesc[c], d1 = cdesc[c + 1];
  const int nt = (int)(d1.x - d0.x), NR = (int)(d1.y - d0.y), NS = (int)(d1.z - d0.z);
  if (nt <= 0 || nt > kMaxTilesN || NR <= 0 || NS <= 0 || NR + NS > kCapN) {
    if (tid == 0) atomicOr(&A.hdr->jerror, PBSM_ERR_INTERNAL);
    return;
  }
  UNestBuf& B = N.buf;
  for (int e = tid; e < NR + NS; e += kUJoinThreads) {
    const u32 slot = e < NR ? d0.y + e : d0.z + (e - NR);
    const char* g = reinterpret_cast<const char*>(A.sc.ent + slot);
    cp_async16(&B.ax[e], g);
    cp_async16(&B.ay[e], g + 16);
    cp_async4(&B.aidx[e], A.sc.eidx + slot);
  }
  if (tid < nt) cp_async16(&B.jr[tid], jrec + d0.x + tid);
  cp_async_wait_all();
  __syncthreads();
  unit_chunk(N, A, nt, NR, d0.y, d0.z);
}

// The chunks heavy units queued: persistent CTAs take them by ticket.
__global__ void __launch_bounds__(kUJoinThreads, 6) k_uchunks(UJoinArgs A) {
  __shared__ __align__(128) UNestSmem N;
  __shared__ i64 tk;
  const i64 nq = *reinterpret_cast<volatile i64*>(&A.hdr->nq);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) tk = (i64)atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->qticket), 1ull);
    __syncthreads();
    const i64 t = tk;
    if (t >= nq) return;
    const uint4 q = A.sc.queue[t];
    unit_stage_and_join(N, A, reinterpret_cast<const uint4*>(A.sc.ent + q.x),
                        reinterpret_cast<const uint4*>(A.sc.ent + q.z), q.y);
  }
}

// ---------------------------------------------------------------- P4 deferred tiles
// Tiles of more than LMAX entries, queued by the units: work items of
// kLargeLead lead entries (one per thread) × kULargeOther entries of the other
// side (streamed through shared memory), every pair tested with the closed
// predicate and the class rule, count → reserve → emit (hits kept in a list;
// a second pass re-tests if the list overflows).  Persistent CTAs take items
// by ticket.
constexpr int kULargeHitCap = 4096;  // hits of a deferred-tile work item kept for the emit
struct ULargeSmem {
  URec other[kCap];
  u32 oidx[kCap];
  u32 hit[kULargeHitCap];  // lead thread | other index (in the item) << 8
  u32 lead_idx[kJoinThreads];
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  u32 nhit;
  i64 item;
};

template <bool LIST>
__device__ __forceinline__ u32 ularge_pass(ULargeSmem& S, int n, bool have, const URec& me,
                                           bool lead_r, u32 my_idx, i64* out, u32 k0,
                                           const UJoinArgs& A) {
  u32 c = 0;
  if (!have) return 0;
  const double mxl = key_x(me.xl);
  const bool mxin = !(me.xl & kXOut), myin = !(me.xl & kYOut);
  for (int k = 0; k < n; ++k) {
    const URec& o = S.other[k];
    const u64 ok = o.xl;
    const double oxl = key_x(ok);
    if (mxl <= o.xu && oxl <= me.xu && me.yl <= o.yu && o.yl <= me.yu &&
        (mxin || !(ok & kXOut)) && (myin || !(ok & kYOut))) {
      if (out) {
        const i64 a = map_id(A.ids[lead_r ? 0 : 1], my_idx), b = map_id(A.ids[lead_r ? 1 : 0], S.oidx[k]);
        *reinterpret_cast<longlong2*>(out + 2 * (i64)c) =
            lead_r ? make_longlong2(a, b) : make_longlong2(b, a);
      }
      if (LIST) {
        const u32 h = atomicAdd_block(&S.nhit, 1u);
        if (h < (u32)kULargeHitCap) S.hit[h] = threadIdx.x | ((k0 + (u32)k) << 8);
      }
      ++c;
    }
  }
  return c;
}

__global__ void __launch_bounds__(kJoinThreads, 2) k_ularge(UJoinArgs A) {
  extern __shared__ __align__(128) unsigned char ul_raw[];
  ULargeSmem& S = *reinterpret_cast<ULargeSmem*>(ul_raw);
  const int tid = threadIdx.x;
  const u64 packed = *reinterpret_cast<volatile u64*>(&A.hdr->def_packed);
  const i64 n_tiles = (i64)(packed >> kDefItemBits);
  const i64 n_items = (i64)(packed & ((1ull << kDefItemBits) - 1));
  if (blockIdx.x == 0 && tid == 0) {
    A.hdr->n_def_tiles = n_tiles;
    A.hdr->n_def_items = n_items;
  }
  if (n_items == 0) return;
  const URec* ent = A.sc.ent;
  for (;;) {
    __syncthreads();
    if (tid == 0) S.item = (i64)atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->work), 1ull);
    __syncthreads();
    const i64 item = S.item;
    if (item >= n_items) return;
    // item → tile: the last deferred tile whose item base is <= item (bases
    // are allocated in tile order, so they increase): 32-ary search per warp
    int lo = 0, hi = (int)n_tiles;
    const int lane = tid & 31;
    while (hi - lo > 1) {
      const int step = (hi - lo + 31) >> 5;
      const int m = lo + lane * step;
      const unsigned le = __ballot_sync(0xffffffffu, m < hi && (i64)__ldg(A.sc.ditem + m) <= item);
      lo += (31 - __clz(le)) * step;
      hi = min(hi, lo + step);
    }
    const uint4 rec = A.sc.dtile[lo];
    const u32 nR = rec.z, nS = rec.w;
    const bool lead_r = nR >= nS;
    const u32 no = lead_r ? nS : nR, nl = lead_r ? nR : nS;
    const u32 L = lead_r ? rec.x : rec.y, O = lead_r ? rec.y : rec.x;
    const u32 nob = (no + kULargeOther - 1) / kULargeOther;
    const u32 li = (u32)(item - (i64)A.sc.ditem[lo]);
    const u32 a = (li / nob) * kLargeLead + tid;
    const u32 o_beg = (li % nob) * kULargeOther, o_end = min(no, o_beg + kULargeOther);
    const bool have = a < nl;
    URec me;
    u32 my_idx = 0;
    if (have) {
      me = ld_urec(ent + L + a);
      my_idx = A.sc.eidx[L + a];
    }
    if (tid == 0) S.nhit = 0;
    u32 cnt = 0;
    bool ok = true;
    i64* out = nullptr;
    for (int pass = 0; pass < 2; ++pass) {
      for (u32 ob = o_beg; ob < o_end; ob += kCap) {
        const int n = (int)min((u32)kCap, o_end - ob);
        __syncthreads();  // previous piece consumed
        for (int k = tid; k < n; k += kJoinThreads) {
          S.other[k] = ld_urec(ent + O + ob + k);
          S.oidx[k] = A.sc.eidx[O + ob + k];
        }
        __syncthreads();
        if (pass == 0) cnt += ularge_pass<true>(S, n, have, me, lead_r, my_idx, nullptr,
                                                 ob - o_beg, A);
        else if (ok) out += 2 * (i64)ularge_pass<false>(S, n, have, me, lead_r, my_idx, out, 0, A);
      }
      if (pass == 1) break;
      u64 total;
      const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
      if (tid == 0) {
        S.base = total ? atomicAdd(reinterpret_cast<unsigned long long*>(&A.hdr->pairs), total) : 0ull;
        if (total && (i64)(S.base + total) > A.capacity) {
          atomicOr(&A.hdr->jerror, PBSM_ERR_PAIR_OVERFLOW);
          S.base = ~0ull;
        }
      }
      S.lead_idx[tid] = my_idx;
      __syncthreads();
      if (S.base == ~0ull || total == 0) break;
      if (total <= (u64)kULargeHitCap) {
        i64* o = A.pairs + 2 * (i64)S.base;
        for (u32 h = tid; h < (u32)total; h += kJoinThreads) {
          const u32 hv = S.hit[h];
          const u32 ki = o_beg + (hv >> 8);
          const i64 lid = map_id(A.ids[lead_r ? 0 : 1], S.lead_idx[hv & 0xffu]);
          const i64 oid = map_id(A.ids[lead_r ? 1 : 0], A.sc.eidx[O + ki]);
          *reinterpret_cast<longlong2*>(o + 2 * (i64)h) =
              lead_r ? make_longlong2(lid, oid) : make_longlong2(oid, lid);
        }
        break;
      }
      out = A.pairs + 2 * (i64)(S.base + excl);
    }
  }
}

// the header → page-locked host memory (pbsm_read_uheader)
__global__ void k_publish_uheader(const pbsm_uheader* __restrict__ hdr, pbsm_uheader* out) {
  static_assert(sizeof(pbsm_uheader) % 8 == 0, "header words");
  const int i = threadIdx.x;
  if (i < (int)(sizeof(pbsm_uheader) / 8))
    reinterpret_cast<volatile u64*>(out)[i] = __ldcg(reinterpret_cast<const u64*>(hdr) + i);
}
