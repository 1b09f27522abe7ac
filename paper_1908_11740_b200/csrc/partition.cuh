// partition.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: subsystem 1: init, count (+ validation), row-band copy, scatter, write guard, plan, generic scan.
#pragma once

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
// PBSM_SCAT_FILTER: the scatter reads a tile's cursor first and skips the
// atomic for tiles without a list (cursor base kSkip: one input empty there —
// 43% of cfg2's assignments); a cursor's join / non-join status never
// changes during the scatter, so a plain L2 load classifies it
#ifndef PBSM_SCAT_FILTER
#define PBSM_SCAT_FILTER 0
#endif
// write guard predicate: a tile's cursor ended where the plan said (with the
// filter, a list-less tile's cursor is never advanced: it stays at kSkip)
__device__ __forceinline__ bool cursor_done(u32 cur, u32 end) {
#if PBSM_SCAT_FILTER
  return cur < kSkip ? cur == end : cur == kSkip;
#else
  return cur == end;
#endif
}
__device__ __forceinline__ u32 cur_inc(u32* p) {
#if PBSM_SCAT_FILTER
  if (__ldcg(p) >= kSkip) return kSkip;
#endif
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

// Points mode (PTS, the ε-distance join): the input is the point columns
// px = xl, py = yl only (xu, yu unused) and each rectangle is the side-ε square
// around its point, clip(p ∓ half, 0, 1) — computed here with the reference's
// numpy arithmetic (engine.py:342-350), never materialised.
__device__ __forceinline__ double clip01(double v) { return fmin(fmax(v, 0.0), 1.0); }
template <bool PTS>
__device__ __forceinline__ void load_mbr(const double* __restrict__ xl,
                                         const double* __restrict__ xu,
                                         const double* __restrict__ yl,
                                         const double* __restrict__ yu, i64 i, double half,
                                         double& a, double& b, double& c, double& d) {
  if (PTS) {
    const double px = __ldcs(xl + i), py = __ldcs(yl + i);
    a = clip01(__dsub_rn(px, half));
    b = clip01(__dadd_rn(px, half));
    c = clip01(__dsub_rn(py, half));
    d = clip01(__dadd_rn(py, half));
  } else {
    a = __ldcs(xl + i);
    b = __ldcs(xu + i);
    c = __ldcs(yl + i);
    d = __ldcs(yu + i);
  }
}

template <bool PTS>
__global__ void __launch_bounds__(256, PBSM_PART_MINB) k_count(const double* __restrict__ xl,
                                               const double* __restrict__ xu,
                                               const double* __restrict__ yl,
                                               const double* __restrict__ yu, i64 n,
                                               int kx, int ky, int row_lo, int row_hi,
                                               const double* __restrict__ bx,
                                               const double* __restrict__ by,
                                               u32* __restrict__ cnt, int side,
                                               u32* __restrict__ band_cnt,
                                               pbsm_header* hdr, double half) {
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
  if (i < end) load_mbr<PTS>(xl, xu, yl, yu, i, half, a, b, c, d);
  for (; i < end; i += blockDim.x) {
    const i64 nx = i + blockDim.x;
    double na = 0, nb = 0, nc = 0, nd = 0;
    if (nx < end) load_mbr<PTS>(xl, xu, yl, yu, nx, half, na, nb, nc, nd);
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

// pt = the point {px, py} bits of an ε-join entry (pad[1], pad[2]: one
// 16-byte-aligned pair the join stages with the rest), else zero
__device__ __forceinline__ void write_rec(Rec* r, u64 key, double xu, double yl, double yu,
                                          i64 id, u64 pol, ulonglong2 pt) {
  st256_hint(r, key, (u64)__double_as_longlong(xu), (u64)__double_as_longlong(yl),
             (u64)__double_as_longlong(yu), pol);
  st256_hint(&r->id, (u64)id, 0ull, pt.x, pt.y, pol);
}

// Compact nested entries (the shipped driver's default where it applies):
// the NESTED region of a tile list — positions [0, nested_end), every entry of
// a tile the nested mini-join tests — is written as ONE 32-byte sector
// {xl | label, xu, yl, yu32 | row << 32}: yu rounded toward zero to float32
// (yu32 <= yu < next float32) and the entry's row index.  The scatter then
// stores one sector per nested entry instead of two (the scatter is bound by
// its scattered per-lane memory operations); the nested join
// decides a y-test against yu32 and reads the exact yu from the input column
// in the rare case it falls inside yu32's float32 gap, and looks the hit's id
// up by row at the emit.  Sorted / large tiles keep the 64-byte record.
struct SplitOut {
  Half* rec32;            // null: one 64-byte format for every entry
  i64 cap32;              // entries rec32 holds
  const i64* nested_end;  // &hdr->nested_r / nested_s (written by the plan)
};

__device__ __forceinline__ u64 yu_row_word(double yu, i64 row) {
  return ((u64)(u32)row << 32) | (u64)__float_as_uint(__double2float_rz(yu));
}

// one list entry at position p: a compact 32-byte sector in the nested
// region (split format), else the 64-byte record; past a capacity → error bit
__device__ __forceinline__ void put_entry(Rec* out, i64 capacity, const SplitOut& sp, u64 nend,
                                          u32 p, u64 key, double xu, double yl, double yu,
                                          i64 id, i64 row, u64 pol, ulonglong2 pt, u32& bad) {
  if (sp.rec32 && (u64)p < nend) {
    if ((i64)p < sp.cap32)
      st256_hint(sp.rec32 + p, key, (u64)__double_as_longlong(xu),
                 (u64)__double_as_longlong(yl), yu_row_word(yu, row), pol);
    else
      bad |= PBSM_ERR_SCATTER_OVERFLOW;
    return;
  }
  if ((i64)p < capacity) write_rec(out + p, key, xu, yl, yu, id, pol, pt);
  else bad |= PBSM_ERR_SCATTER_OVERFLOW;
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
  double half;       // points mode: square half-side (see load_mbr)
  SplitOut split;
  template <bool BANDED, bool PTS>
  __device__ __forceinline__ void load(i64 i, double& a, double& b, double& c, double& d,
                                       i64& id, ulonglong2& pt) const {
    if (PTS) {
      id = ids ? __ldcs(ids + i) : i;
      const double px = __ldcs(xl + i), py = __ldcs(yl + i);
      pt = make_ulonglong2((u64)__double_as_longlong(px), (u64)__double_as_longlong(py));
      a = clip01(__dsub_rn(px, half));
      b = clip01(__dadd_rn(px, half));
      c = clip01(__dsub_rn(py, half));
      d = clip01(__dadd_rn(py, half));
    } else if (BANDED) {
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
template <bool BANDED, bool PTS>
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
  const u64 nend = in.split.rec32 ? (u64)__ldcg(in.split.nested_end) : 0ull;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  double pa = 0, pb = 0, pc = 0, pd = 0;
  i64 pid = 0;
  ulonglong2 ppt = make_ulonglong2(0ull, 0ull);
  if (i < n) in.load<BANDED, PTS>(i, pa, pb, pc, pd, pid, ppt);  // software pipeline: next one in flight
  for (; i < n; i += stride) {
    const double a = pa, b = pb, c = pc, d = pd;
    const i64 id = pid;
    const ulonglong2 pt = ppt;
    if (i + stride < n) in.load<BANDED, PTS>(i + stride, pa, pb, pc, pd, pid, ppt);
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
      if (p < kSkip)
        put_entry(out, capacity, in.split, nend, p, xk | ((r0 != rr0) ? kYOut : 0ull), b, c, d,
                  id, i, pol, pt, bad);
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
        const u64 key = xk | ((rows[q] != rr0) ? kYOut : 0ull) | ((cols[q] != c0) ? kXOut : 0ull);
        put_entry(out, capacity, in.split, nend, pos[q], key, b, c, d, id, i, pol, pt, bad);
      }
      continue;
    }
    for (int row = r0; row <= r1; ++row) {
      u32* rowp = cursor + (size_t)(row - row_lo) * kx;
      const u64 ylab = (row != rr0) ? kYOut : 0ull;
      for (int col = c0; col <= c1; ++col) {
        const u32 p = cur_inc(rowp + col);
        if (p >= kSkip) continue;  // not a join tile
        put_entry(out, capacity, in.split, nend, p, xk | ylab | ((col != c0) ? kXOut : 0ull), b,
                  c, d, id, i, pol, pt, bad);
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
    bad |= !cursor_done(cur_r[t], end_r[t]) || !cursor_done(cur_s[t], end_s[t]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&hdr->error, PBSM_ERR_OFFSET_MISMATCH);
}

// ---------------------------------------------------------------- 1b plan
// Per tile t the plan scans thirteen lanes at once (one exclusive scan each):
//   0 |R_T|  1 |S_T|                          all tiles (A_R, A_S totals)
//   2..4   nested tiles: flag, |R_T|, |S_T|
//   5..7   sorted tiles: flag, |R_T|, |S_T|
//   8..12  large tiles:  flag, sweep work items (256 leaders of one side
//          each), |R_T|, |S_T|, sort windows (4096 entries of one side each)
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
enum Lane { L_A, L_B, L_NF, L_NA, L_NB, L_SF, L_SA, L_SB, L_LF, L_LI, L_LA, L_LB, L_LW };

__device__ __forceinline__ int tile_kind(u32 a, u32 b, i64 nested_max) {
  if (a == 0u || b == 0u) return kNone;
  if (a + b > (u32)kLmax) return kLarge;
  return (i64)((u64)a * (u64)b) <= nested_max ? kNested : kSorted;
}

__device__ __forceinline__ void tile_vals(u32 a, u32 b, i64 nm, u32 v[kNV], i64 sm) {
  const int kind = tile_kind(a, b, nm);
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
    v[L_LA] = a;
    v[L_LB] = b;
    if (is_huge(a, b, sm)) {  // sort + sweep: leader blocks of each side, sort windows
      v[L_LI] = (a + kSweepLeaders - 1) / kSweepLeaders + (b + kSweepLeaders - 1) / kSweepLeaders;
      v[L_LW] = (a + kSortWindow - 1) / kSortWindow + (b + kSortWindow - 1) / kSortWindow;
    } else {  // brute force: lead blocks × other blocks
      const u32 lead = a >= b ? a : b, other = a >= b ? b : a;
      v[L_LI] = ((lead + kLargeLead - 1) / kLargeLead) * ((other + kLargeOther - 1) / kLargeOther);
    }
  }
}

// The plan kernels give thread j of CTA c the kPlanPer = 8 CONSECUTIVE tiles
// from c * kPlanTile + 8 j: two 16-byte loads per counter array put all of a
// thread's counts in flight at once (with one 4-byte load per tile and step
// both kernels sat on their first loads: 59% / 24% of their stall samples),
// and k_plan_apply writes its four outputs back the same way, with no
// shared-memory staging.  Tiles past T read as empty.
static_assert(kPlanPer == 8, "plan kernels: two uint4 per thread and array");
__device__ __forceinline__ void plan_load8(const u32* __restrict__ c, u64 t0, u64 T, u32 v[8]) {
  if (t0 + 8 <= T && (t0 & 3) == 0) {
    const uint4 x = *reinterpret_cast<const uint4*>(c + t0);
    const uint4 y = *reinterpret_cast<const uint4*>(c + t0 + 4);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t0 + i < T ? c[t0 + i] : 0u;
  }
}
__device__ __forceinline__ void plan_store8(u32* __restrict__ c, u64 t0, u64 T, const u32 v[8]) {
  if (t0 + 8 <= T && (t0 & 3) == 0) {
    *reinterpret_cast<uint4*>(c + t0) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(c + t0 + 4) = make_uint4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (t0 + i < T) c[t0 + i] = v[i];
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_plan_reduce(const u32* __restrict__ cr,
                                                              const u32* __restrict__ cs,
                                                              u64 T, i64 nm, i64 sm,
                                                              u64* __restrict__ partials,
                                                              pbsm_header* hdr) {
  __shared__ u32 sh[kPlanThreads / 32][kNV];
  __shared__ u32 shmax[kPlanThreads / 32];
  __shared__ u32 shhuge[kPlanThreads / 32];
  __shared__ u64 shb[kPlanThreads / 32];
  u32 acc[kNV];
#pragma unroll
  for (int q = 0; q < kNV; ++q) acc[q] = 0;
  u32 mx = 0, mh = 0;
  u64 bound = 0;
  const u64 t0 = (u64)blockIdx.x * kPlanTile + (u64)threadIdx.x * kPlanPer;
  u32 av[kPlanPer], bv[kPlanPer];
  plan_load8(cr, t0, T, av);
  plan_load8(cs, t0, T, bv);
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u32 a = av[i], b = bv[i];
    u32 v[kNV];
    tile_vals(a, b, nm, v, sm);
#pragma unroll
    for (int q = 0; q < kNV; ++q) acc[q] += v[q];
    if (a && b) {
      mx = max(mx, a + b);
      bound += (u64)a * (u64)b;
      if (a + b > (u32)kLmax && is_huge(a, b, sm)) mh = max(mh, max(a, b));
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
    mh = max(mh, __shfl_down_sync(0xffffffffu, mh, o));
    bound += __shfl_down_sync(0xffffffffu, bound, o);
  }
  if (lane == 0) {
    shmax[wid] = mx;
    shhuge[wid] = mh;
    shb[wid] = bound;
  }
  __syncthreads();
  if (threadIdx.x < kNV) {
    u64 s = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) s += sh[w][threadIdx.x];
    partials[(u64)threadIdx.x * (gridDim.x + 1) + blockIdx.x] = s;
  }
  if (threadIdx.x == 0) {
    u32 m = 0, h = 0;
    u64 bs = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) {
      m = max(m, shmax[w]);
      h = max(h, shhuge[w]);
      bs += shb[w];
    }
    // into two extra partials rows, reduced by k_plan_partials (a header
    // atomic per CTA queued ~4000 same-address atomics at one L2 slice)
    partials[(u64)kNV * (gridDim.x + 1) + blockIdx.x] = m;
    partials[(u64)(kNV + 1) * (gridDim.x + 1) + blockIdx.x] = bs;
    partials[(u64)(kNV + 2) * (gridDim.x + 1) + blockIdx.x] = h;
  }
}

// one CTA per scan lane: exclusive scan of lane q's per-CTA partial sums (a
// lane-major row, so loads and stores are coalesced; 4 consecutive values per
// thread, 4096 per block-scan step).  The lane total goes after the row (read
// by k_plan_apply); the last CTA to finish writes the header.
constexpr int kPartThreads = 1024;
__global__ void __launch_bounds__(kPartThreads) k_plan_partials(u64* __restrict__ partials, u64 nb,
                                                                 pbsm_header* hdr, uint4* cd_n,
                                                                 uint4* cd_s, u32* lpre,
                                                                 u32* lwin, i64 sm) {
  __shared__ u64 sh[kPartThreads / 32 + 1];
  __shared__ bool last;
  u64* row = partials + (u64)blockIdx.x * (nb + 1);
  u64 carry = 0;
  if (blockIdx.x == kNV) {
    // the extra CTA: max tile and pair bound over the plan CTAs' rows
    const u64* rb = row + (nb + 1);
    const u64* rh = rb + (nb + 1);
    u64 m = 0, bs = 0, mh = 0;
    for (u64 i = threadIdx.x; i < nb; i += kPartThreads) {
      m = max(m, row[i]);
      bs += rb[i];
      mh = max(mh, rh[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      m = max(m, __shfl_down_sync(0xffffffffu, m, o));
      mh = max(mh, __shfl_down_sync(0xffffffffu, mh, o));
      bs += __shfl_down_sync(0xffffffffu, bs, o);
    }
    __shared__ u64 wm[kPartThreads / 32], wb[kPartThreads / 32], wh[kPartThreads / 32];
    if ((threadIdx.x & 31) == 0) {
      wm[threadIdx.x >> 5] = m;
      wb[threadIdx.x >> 5] = bs;
      wh[threadIdx.x >> 5] = mh;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kPartThreads / 32; ++w) {
        m = max(m, wm[w]);
        bs += wb[w];
        mh = max(mh, wh[w]);
      }
      hdr->max_tile = (i64)m;
      hdr->pair_bound = (i64)bs;
      hdr->max_huge = (i64)mh;
      hdr->sweep_min = sm;
    }
  }
  for (u64 base = 0; blockIdx.x < kNV && base < nb; base += 4 * kPartThreads) {
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
    if (blockIdx.x < kNV) row[nb] = carry;
    __threadfence();
    last = atomicAdd(&hdr->pad, 1u) == (u32)kNV;  // kNV + 1 CTAs
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
    hdr->large_r = (i64)c[L_LA];
    hdr->large_s = (i64)c[L_LB];
    hdr->nested_r = (i64)c[L_NA];
    hdr->nested_s = (i64)c[L_NB];
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
    lwin[c[L_LF]] = (u32)c[L_LW];
  }
}

struct PlanOut {
  u32 *cur_r, *cur_s;
  uint4* jrec[2];
  uint4* cdesc[2];
  uint4* lrec;
  u32* lpre;
  u32* lwin;
  u32* litem;  // [tiles]: large work item → index of its tile in lrec (k_join skips its search)
};

// the lanes k_plan_apply scans: every lane but the two totals (L_A, L_B)
constexpr int kNA = kNV - 2;
__global__ void __launch_bounds__(kPlanThreads, PBSM_PLAN_MINB) k_plan_apply(u32* __restrict__ cr,
                                                             u32* __restrict__ cs, u64 T, u64 nb,
                                                             i64 nm, i64 sm,
                                                             const u64* __restrict__ partials,
                                                             PlanOut P) {
  __shared__ u32 shs[kPlanThreads / 32][kNA];
  __shared__ u64 shp[2][kNV];  // this CTA's global prefixes, the totals
  const u64 base = (u64)blockIdx.x * kPlanTile;
  // lane-major partials: lane q of CTA b at q * (nb + 1) + b, totals at q * (nb + 1) + nb;
  // fetched first so their latency overlaps the count loads
  if (threadIdx.x < 2 * kNV) {
    const int q = threadIdx.x % kNV;
    shp[threadIdx.x / kNV][q] = partials[(u64)q * (nb + 1) + (threadIdx.x < kNV ? blockIdx.x : nb)];
  }
  // this thread's 8 consecutive tiles (plan_load8)
  const u64 t0 = base + (u64)threadIdx.x * kPlanPer;
  u32 a[kPlanPer], b[kPlanPer];
  plan_load8(cr, t0, T, a);
  plan_load8(cs, t0, T, b);
  u32 pre[kNA];  // in-CTA exclusive prefixes of lanes 2..11 (u32: a CTA's sums fit)
#pragma unroll
  for (int q = 0; q < kNA; ++q) pre[q] = 0;
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    u32 v[kNV];
    tile_vals(a[i], b[i], nm, v, sm);
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
  u32 r0v[kPlanPer], s0v[kPlanPer];  // the tiles' list starts
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    const u64 t = t0 + i;
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
      u32 v[kNV];
      tile_vals(a[i], b[i], nm, v, sm);
      if (t < T) {
        const u64 lf = g(L_LF), it0 = g(L_LI);
        P.lrec[lf] = make_uint4(r0, s0, a[i], b[i]);
        P.lpre[lf] = (u32)it0;
        P.lwin[lf] = (u32)g(L_LW);
        // item → tile, for the items the table holds (T of them)
        for (u64 it = it0; it < it0 + v[L_LI] && it < T; ++it) P.litem[it] = (u32)lf;
      }
      pre[L_LF - 2] += 1u;
      pre[L_LI - 2] += v[L_LI];
      pre[L_LA - 2] += a[i];
      pre[L_LB - 2] += b[i];
      pre[L_LW - 2] += v[L_LW];
    }
    r0v[i] = r0;
    s0v[i] = s0;
  }
  // cursors start at the list starts; the counters become the expected cursor
  // ends (for k_guard)
  plan_store8(P.cur_r, t0, T, r0v);
  plan_store8(P.cur_s, t0, T, s0v);
#pragma unroll
  for (int i = 0; i < kPlanPer; ++i) {
    r0v[i] += a[i];
    s0v[i] += b[i];
  }
  plan_store8(cr, t0, T, r0v);
  plan_store8(cs, t0, T, s0v);
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
