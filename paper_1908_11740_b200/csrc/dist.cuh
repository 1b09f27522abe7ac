// dist.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after common.cuh / partition.cuh).
// Contents: the multi-GPU plumbing around the join:
//   * strip routing — every rectangle of a rank's slice packed, per
//     destination strip, into one send buffer of 40-byte records for a single
//     all_to_all (the distributed PBSM input distribution);
//   * the canonical pair order — a stable LSD radix sort of (r_id, s_id)
//     int64 pairs, lexicographic, the parity form of the reference's
//     unordered list (engine.py:61-62, 293-300).
#pragma once

// ---------------------------------------------------------------- routing
constexpr int kRouteThreads = 256;
constexpr int kRouteTile = 4096;   // rectangles per routing block
constexpr int kMaxRanks = 1024;    // strips (ranks) a routing call supports

struct RouteLayout {
  size_t by, cnt, base, part, total;
  u64 nb, m;  // blocks, world * blocks counters
};
inline RouteLayout route_layout(i64 n, int ky, int world) {
  RouteLayout L;
  L.nb = (u64)std::max<i64>(1, (n + kRouteTile - 1) / kRouteTile);
  L.m = (u64)world * L.nb;
  const u64 sb = (L.m + kScanTile - 1) / kScanTile;
  size_t o = 0;
  L.by = o; o = align_up(o + 8 * ((size_t)ky + 1), 256);
  L.cnt = o; o = align_up(o + 4 * (L.m + 1), 256);
  L.base = o; o = align_up(o + 8 * (L.m + 1), 256);
  L.part = o; o = align_up(o + 8 * (sb + 1), 256);
  L.total = o;
  return L;
}

__global__ void k_bounds(double* __restrict__ b, int k) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= k; i += gridDim.x * blockDim.x)
    b[i] = __ddiv_rn((double)i, (double)k);  // tile_boundary, geometry.py:82-84
}

// strips [g0, g1] a rectangle with tile rows [r0, r1] meets (cuts strictly
// increasing: every strip non-empty)
__device__ __forceinline__ int strip_of(int r, const int* cuts, int world) {
  int lo = 0, hi = world;  // last g with cuts[g] <= r
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (cuts[m] <= r) lo = m; else hi = m;
  }
  return lo;
}

template <bool PACK>
__global__ void __launch_bounds__(kRouteThreads) k_route(
    const i64* __restrict__ ids, const double* __restrict__ xl, const double* __restrict__ xu,
    const double* __restrict__ yl, const double* __restrict__ yu, i64 n, int ky,
    const double* __restrict__ by, const int* __restrict__ cuts_g, int world,
    u32* __restrict__ cnt, const u64* __restrict__ base, u64* __restrict__ out) {
  __shared__ int cuts[kMaxRanks + 1];
  __shared__ u32 cur[kMaxRanks];
  for (int g = threadIdx.x; g <= world; g += kRouteThreads) cuts[g] = cuts_g[g];
  for (int g = threadIdx.x; g < world; g += kRouteThreads)
    cur[g] = PACK ? (u32)(base[(size_t)g * gridDim.x + blockIdx.x] -
                          base[(size_t)g * gridDim.x]) : 0u;
  __syncthreads();
  const i64 beg = (i64)blockIdx.x * kRouteTile, end = min(n, beg + kRouteTile);
  for (i64 i = beg + threadIdx.x; i < end; i += kRouteThreads) {
    const double c = yl[i], d = yu[i];
    const int g0 = strip_of(tile_of(c, ky, by), cuts, world);
    const int g1 = strip_of(tile_of(d, ky, by), cuts, world);
    for (int g = g0; g <= g1; ++g) {
      const u32 slot = atomicAdd_block(&cur[g], 1u);
      if (PACK) {
        // SJB1 record order {id, x_l, y_l, x_u, y_u} (io.py:113-141), so the
        // receiver unpacks with k_unpack_records
        u64* r = out + 5 * (base[(size_t)g * gridDim.x] + slot);
        r[0] = (u64)(ids ? ids[i] : i);
        r[1] = (u64)__double_as_longlong(xl[i]);
        r[2] = (u64)__double_as_longlong(c);
        r[3] = (u64)__double_as_longlong(xu[i]);
        r[4] = (u64)__double_as_longlong(d);
      }
    }
  }
  if (!PACK) {
    __syncthreads();
    // destination-major: all blocks' counts for strip 0, then strip 1, ...
    for (int g = threadIdx.x; g < world; g += kRouteThreads)
      cnt[(size_t)g * gridDim.x + blockIdx.x] = cur[g];
  }
}

// per-destination totals and starts from the scanned counters
__global__ void k_route_totals(const u64* __restrict__ base, u64 nb, int world, u64 m,
                               i64* __restrict__ dest) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < world; g += gridDim.x * blockDim.x) {
    const u64 a = base[(u64)g * nb], b = (g + 1 < world) ? base[(u64)(g + 1) * nb] : base[m];
    dest[g] = (i64)(b - a);
  }
}

// ---------------------------------------------------------------- pair sort
// Stable LSD radix sort of n (r_id, s_id) int64 pairs into lexicographic
// order, 8-bit digits: digit d < 8 is byte d of s_id, d >= 8 byte d-8 of
// r_id, each with the sign bit flipped (signed order → unsigned order).
// Digits on which every key agrees are skipped (the host reads the digit
// histogram first: ids below 2^24 sort in 6 passes instead of 16).
constexpr int kSortT = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortT * kSortItems;  // pairs per block per pass
constexpr int kSortWarps = kSortT / 32;

__device__ __forceinline__ u32 pair_digit(u64 r_id, u64 s_id, int d) {
  const u64 w = (d < 8 ? s_id : r_id) ^ (1ull << 63);
  return (u32)(w >> (8 * (d & 7))) & 0xffu;
}

__global__ void __launch_bounds__(kSortT) k_pair_digits(const ulonglong2* __restrict__ p, i64 n,
                                                        u32* __restrict__ hist) {
  __shared__ u32 h[16 * 256];
  for (int i = threadIdx.x; i < 16 * 256; i += kSortT) h[i] = 0u;
  __syncthreads();
  for (i64 i = blockIdx.x * (i64)kSortT + threadIdx.x; i < n; i += (i64)gridDim.x * kSortT) {
    const ulonglong2 v = p[i];
#pragma unroll
    for (int d = 0; d < 16; ++d) atomicAdd_block(&h[d * 256 + pair_digit(v.x, v.y, d)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * 256; i += kSortT)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// per-block digit counts, digit-major (cnt[digit * nb + block])
__global__ void __launch_bounds__(kSortT) k_pair_count(const ulonglong2* __restrict__ p, i64 n,
                                                       int d, u32* __restrict__ cnt) {
  __shared__ u32 h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const i64 beg = (i64)blockIdx.x * kSortTile, end = min(n, beg + kSortTile);
  for (i64 i = beg + threadIdx.x; i < end; i += kSortT) {
    const ulonglong2 v = p[i];
    atomicAdd_block(&h[pair_digit(v.x, v.y, d)], 1u);
  }
  __syncthreads();
  cnt[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: warp w ranks its 512 consecutive pairs step by step
// (__match_any_sync per 32-pair step, a running per-(warp, digit) count),
// the warps' counts are scanned per digit, and every pair lands at
// base[digit][block] + warp offset + its rank
__global__ void __launch_bounds__(kSortT) k_pair_scatter(const ulonglong2* __restrict__ in,
                                                         ulonglong2* __restrict__ out, i64 n,
                                                         int d, const u64* __restrict__ base) {
  __shared__ u32 wc[kSortWarps][256];
  __shared__ u64 bb[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortT) (&wc[0][0])[i] = 0u;
  bb[threadIdx.x] = base[(size_t)threadIdx.x * gridDim.x + blockIdx.x];
  __syncthreads();
  const i64 w0 = (i64)blockIdx.x * kSortTile + (i64)warp * (kSortTile / kSortWarps);
  ulonglong2 v[kSortItems];
  u32 rk[kSortItems];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int s = 0; s < kSortItems; ++s) {
    const i64 i = w0 + 32 * s + lane;
    const bool ok = i < n;
    v[s] = ok ? in[i] : make_ulonglong2(0ull, 0ull);
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (act == 0u) {
      rk[s] = 0u;
      continue;
    }
    const u32 dg = pair_digit(v[s].x, v[s].y, d);
    const unsigned peers = __match_any_sync(0xffffffffu, ok ? dg : 0x100u) & act;
    u32 before = 0;
    if (ok) before = wc[warp][dg];
    __syncwarp();
    if (ok) {
      rk[s] = before + __popc(peers & lt);
      if ((peers & lt) == 0u) wc[warp][dg] = before + __popc(peers);  // the group's leader
    }
    __syncwarp();
  }
  __syncthreads();
  {  // exclusive scan of the warps' counts, per digit (thread = digit)
    u32 run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const u32 c = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kSortItems; ++s) {
    const i64 i = w0 + 32 * s + lane;
    if (i < n) {
      const u32 dg = pair_digit(v[s].x, v[s].y, d);
      out[bb[dg] + wc[warp][dg] + rk[s]] = v[s];
    }
  }
}

inline u64 pair_sort_blocks(i64 n) { return (u64)std::max<i64>(1, (n + kSortTile - 1) / kSortTile); }

struct PairSortLayout {
  size_t cnt, base, part, total;
  u64 nb, m;
};
inline PairSortLayout pair_sort_layout(i64 n) {
  PairSortLayout L;
  L.nb = pair_sort_blocks(n);
  L.m = 256 * L.nb;
  const u64 sb = (L.m + kScanTile - 1) / kScanTile;
  size_t o = 0;
  L.cnt = o; o = align_up(o + 4 * (L.m + 1), 256);
  L.base = o; o = align_up(o + 8 * (L.m + 1), 256);
  L.part = o; o = align_up(o + 8 * (sb + 1), 256);
  L.total = o;
  return L;
}

// ---------------------------------------------------------------- public partition()
// partition() / PartitionedDataset (partition.py:75-111, 243-263) on the
// device: every (tile, rectangle) assignment as a (tile, row) key pair, the
// keys radix-sorted (stable: rows ascending inside a tile — exactly the
// reference's order, whose writers own contiguous input slices in slice order,
// partition.py:130-133, 201-227), the coordinates gathered in that order and
// the CSR offsets found at the tile boundaries of the sorted keys.
template <typename F>
__device__ __forceinline__ void rect_tiles(double a, double b, double c, double d, int kx, int ky,
                                           const double* bx, const double* by, F&& f) {
  const int c0 = tile_of(a, kx, bx), c1 = tile_of(b, kx, bx);
  const int r0 = tile_of(c, ky, by), r1 = tile_of(d, ky, by);
  // tiles_overlapping (partition.py:114-127): rows ascending, then columns
  for (int row = r0; row <= r1; ++row)
    for (int col = c0; col <= c1; ++col) f((u64)row * (u64)kx + (u64)col);
}

__global__ void k_assign_count(const double* __restrict__ xl, const double* __restrict__ xu,
                               const double* __restrict__ yl, const double* __restrict__ yu,
                               i64 n, int kx, int ky, const double* __restrict__ bx,
                               const double* __restrict__ by, u32* __restrict__ per) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const int c0 = tile_of(xl[i], kx, bx), c1 = tile_of(xu[i], kx, bx);
    const int r0 = tile_of(yl[i], ky, by), r1 = tile_of(yu[i], ky, by);
    per[i] = (u32)((c1 - c0 + 1) * (r1 - r0 + 1));
  }
}

__global__ void k_assign_write(const double* __restrict__ xl, const double* __restrict__ xu,
                               const double* __restrict__ yl, const double* __restrict__ yu,
                               i64 n, int kx, int ky, const double* __restrict__ bx,
                               const double* __restrict__ by, const u64* __restrict__ start,
                               ulonglong2* __restrict__ keys) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    u64 o = start[i];
    rect_tiles(xl[i], xu[i], yl[i], yu[i], kx, ky, bx, by,
               [&](u64 t) { keys[o++] = make_ulonglong2(t, (u64)i); });
  }
}

// sorted (tile, row) keys → SoA copies + offsets[t] = first position of tile t
__global__ void k_assign_gather(const ulonglong2* __restrict__ keys, i64 a, u64 tiles,
                                const i64* __restrict__ ids, const double* __restrict__ xl,
                                const double* __restrict__ xu, const double* __restrict__ yl,
                                const double* __restrict__ yu, i64* __restrict__ o_ids,
                                double* __restrict__ o_xl, double* __restrict__ o_xu,
                                double* __restrict__ o_yl, double* __restrict__ o_yu,
                                i64* __restrict__ offsets) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i <= a;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 t = i < a ? keys[i].x : tiles;
    const u64 prev = i > 0 ? keys[i - 1].x + 1 : 0;  // tiles (prev, t] start here
    for (u64 q = prev; q <= t; ++q) offsets[q] = i;
    if (i < a) {
      const i64 r = (i64)keys[i].y;
      o_ids[i] = ids ? ids[r] : r;
      o_xl[i] = xl[r];
      o_xu[i] = xu[r];
      o_yl[i] = yl[r];
      o_yu[i] = yu[r];
    }
  }
}

struct AssignLayout {
  size_t bx, by, per, start, part, total;
  u64 nb;
};
inline AssignLayout assign_layout(i64 n, int kx, int ky) {
  AssignLayout L;
  L.nb = ((u64)n + kScanTile - 1) / kScanTile;
  size_t o = 0;
  L.bx = o; o = align_up(o + 8 * ((size_t)kx + 1), 256);
  L.by = o; o = align_up(o + 8 * ((size_t)ky + 1), 256);
  L.per = o; o = align_up(o + 4 * ((size_t)n + 1), 256);
  L.start = o; o = align_up(o + 8 * ((size_t)n + 1), 256);
  L.part = o; o = align_up(o + 8 * (L.nb + 1), 256);
  L.total = o;
  return L;
}
