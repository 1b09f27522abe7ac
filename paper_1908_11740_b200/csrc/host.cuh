// host.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: host glue: launch configuration, smem attributes, join launch.
#pragma once

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

// Per-device facts, cached per device ordinal (joins may run on several
// devices, from several host threads: the caches are atomics, and a race only
// repeats an idempotent query / attribute call).
constexpr int kMaxDevices = 64;

int num_sms() {
  static std::atomic<int> n[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int v = n[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
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

// join scratch: [ticket | status[n_units] | large-tile sort area (sweep.cuh)]
inline size_t join_status_bytes(i64 n_units) {
  return 256 + align_up(8 * (size_t)(n_units + 1), 256);
}
inline size_t join_scratch(i64 n_units, i64 large_entries) {
  return join_status_bytes(n_units) + large_sort_bytes(large_entries);
}

// merge passes after the 4096-entry window sort so that a side of `max_tile`
// entries is one sorted run
inline int sort_passes(i64 max_tile) {
  int p = 0;
  while (((i64)kSortWindow << p) < max_tile) ++p;
  return p;
}

int set_smem_attrs() {
  // the dynamic shared-memory opt-in is a per-device function attribute
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & (kMaxDevices - 1));
  if (done.load(std::memory_order_acquire) & bit) return 0;
  cudaError_t e;
  e = cudaFuncSetAttribute(k_join<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(JoinSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_join<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(JoinSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_lsort_win, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSortWindow * 12);
  if (e != cudaSuccess) return (int)e;
#if PBSM_NESTED_PIPE
  {
    const int b = (int)sizeof(PipeSmemM<0>), b32 = (int)sizeof(PipeSmemM<2>);
    const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;
    if ((e = cudaFuncSetAttribute(k_join_nested_pipe<true, 0>, A, b)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<false, 0>, A, b)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<true, 1>, A, b)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<false, 1>, A, b)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<true, 2>, A, b32)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<false, 2>, A, b32)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<true, 3>, A, b32)) ||
        (e = cudaFuncSetAttribute(k_join_nested_pipe<false, 3>, A, b32)))
      return (int)e;
  }
#endif
  done.fetch_or(bit, std::memory_order_release);
  return 0;
}

// compact nested entries (SplitOut): the nested regions, their capacities,
// the exact yu columns and the id columns (null: the pairs hold rows)
struct SplitLists {
  const void* r32;
  const void* s32;
  i64 cap_r, cap_s;
  const double* r_yu;
  const double* s_yu;
  const i64* r_ids;
  const i64* s_ids;
  int few_pairs;  // occupancy hint: the join emits few pairs per entry
};

int launch_join(bool emit, bool ordered, void* ws, int kx, int ky, int row_lo, int row_hi,
                const pbsm_entry* r_list, const pbsm_entry* s_list, const pbsm_header* plan,
                void* scratch, int64_t* pairs, i64 capacity, cudaStream_t s,
                i64 max_nested = -1, i64 max_other = -1, i64 cap_r = -1, i64 cap_s = -1,
                i64 large_cap = 0, i64 max_tile = 0, int eps = 0, double eps_sq = 0.0,
                const SplitLists* split = nullptr) {
  int rc = set_smem_attrs();
  if (rc) return rc;
  const WsLayout L = ws_layout(kx, ky, row_lo, row_hi);
  Ws w = ws_bind(ws, L);
  const bool bounded = plan == nullptr;  // sizes from the device header, grids = bounds
  const i64 cn = bounded ? max_nested : plan->chunks_nested;
  const i64 rest = bounded ? max_other : plan->chunks_sorted + plan->n_items;
  const i64 n_units = cn + rest;
  // large tiles: sort buffers sized from the plan (or the caller's bounds)
  const i64 lcap = bounded ? large_cap : plan->large_r + plan->large_s;
  const i64 mtile = bounded ? max_tile : plan->max_huge;
  // the write guard (reads the cursors the scatter left behind) runs inside
  // the nested join when there is one, else as its own kernel
  // (fused only when the nested grid is large enough that its grid-stride
  // slice stays short: a small join over a large strip runs k_guard instead)
  const i64 nested_ctas =
      PBSM_NESTED_PIPE && !ordered
          ? std::min<i64>(cn, (i64)num_sms() *
                                  pipe_ctas(split ? (split->few_pairs ? 3 : 2) : eps ? 1 : 0))
          : cn;
#ifndef PBSM_GUARD_PER
#define PBSM_GUARD_PER 32  // tiles a nested-join thread may check
#endif
  const bool fused_guard = cn > 0 && (i64)L.tiles <= nested_ctas * (i64)kNT * PBSM_GUARD_PER;
  // One list passed for both inputs: a self-join partitioned once (the caller
  // copied R's counts to S's before the plan and ran one scatter, so S's
  // cursors never moved): the S side of the write guard reads R's cursors.
  const bool one_list = (const void*)r_list == (const void*)s_list &&
                        (!split || split->r32 == split->s32);
  const u32* g_cur_s = one_list ? w.cur_r : w.cur_s;
  const u32* g_end_s = one_list ? w.cnt_r : w.cnt_s;
  if (!fused_guard) {
    const unsigned gb = (unsigned)std::max<i64>(1, std::min<i64>((i64)((L.tiles + 255) / 256),
                                                                  (i64)num_sms() * 8));
    k_guard<<<gb, 256, 0, s>>>(w.cur_r, w.cnt_r, g_cur_s, g_end_s, L.tiles, w.hdr);
  }
  // (a bounded emit is the one join pass behind its plan, whose last CTA left
  // hdr->pairs at zero: no memset node between the scatter and the join —
  // ~4 µs of a graph replay, tools/timeline.py)
  if (!bounded) cudaMemsetAsync(&w.hdr->pairs, 0, sizeof(int64_t), s);
  if (n_units == 0) return launch_status();
  if (ordered) cudaMemsetAsync(scratch, 0, join_status_bytes(n_units), s);
  JoinArgs A;
  for (int q = 0; q < 2; ++q) {
    A.jrec[q] = w.jrec[q];
    A.cdesc[q] = w.cdesc[q];
  }
  A.lrec = w.lrec;
  A.lpre = w.lpre;
  A.litem = w.litem;
  A.litem_n = L.tiles;
  A.ls = large_sort_bind((char*)scratch + join_status_bytes(n_units), lcap);
  A.ls.passes = sort_passes(mtile);
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
  A.list_cap_r = cap_r;
  A.list_cap_s = cap_s;
  A.g_cur_r = w.cur_r;
  A.g_end_r = w.cnt_r;
  A.g_cur_s = g_cur_s;
  A.g_end_s = g_end_s;
  A.g_tiles = fused_guard ? L.tiles : 0;
  A.eps = eps;
  A.eps_sq = eps_sq;
  A.r32 = split ? reinterpret_cast<const Half*>(split->r32) : nullptr;
  A.s32 = split ? reinterpret_cast<const Half*>(split->s32) : nullptr;
  A.cap32_r = split ? split->cap_r : 0;
  A.cap32_s = split ? split->cap_s : 0;
  A.r_yu = split ? split->r_yu : nullptr;
  A.s_yu = split ? split->s_yu : nullptr;
  A.r_ids = split ? split->r_ids : nullptr;
  A.s_ids = split ? split->s_ids : nullptr;
#if PBSM_NESTED_PIPE
  if (cn > 0 && !ordered) {
    // persistent CTAs, two per SM, TMA-staged chunks (k_join_nested_pipe)
    const int mode = split ? (split->few_pairs ? 3 : 2) : eps ? 1 : 0;
    const unsigned g =
        (unsigned)std::max<i64>(1, std::min<i64>(cn, (i64)num_sms() * pipe_ctas(mode)));
    const size_t sm = sizeof(PipeSmemM<0>), sm32 = sizeof(PipeSmemM<2>);
    if (eps) {
      if (emit) k_join_nested_pipe<true, 1><<<g, kNT, sm, s>>>(A, cn);
      else k_join_nested_pipe<false, 1><<<g, kNT, sm, s>>>(A, cn);
    } else if (split) {
      if (mode == 3) {
        if (emit) k_join_nested_pipe<true, 3><<<g, kNT, sm32, s>>>(A, cn);
        else k_join_nested_pipe<false, 3><<<g, kNT, sm32, s>>>(A, cn);
      } else {
        if (emit) k_join_nested_pipe<true, 2><<<g, kNT, sm32, s>>>(A, cn);
        else k_join_nested_pipe<false, 2><<<g, kNT, sm32, s>>>(A, cn);
      }
    } else if (emit) {
      k_join_nested_pipe<true, 0><<<g, kNT, sm, s>>>(A, cn);
    } else {
      k_join_nested_pipe<false, 0><<<g, kNT, sm, s>>>(A, cn);
    }
  } else
#endif
  if (cn > 0) {
    // one CTA per chunk (the ordered look-back takes tickets in launch order)
    if (eps) {
      if (emit)
        k_join_nested<true, true><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
      else
        k_join_nested<false, true><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
    } else if (emit) {
      k_join_nested<true, false><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
    } else {
      k_join_nested<false, false><<<(unsigned)cn, kNT, 0, s>>>(A, cn);
    }
  }
  if (rest > 0 && lcap > 0 && mtile > 0) {
    // huge tiles: window sort, merge passes, sorted copy (sweep.cuh); a CTA
    // per sort window (grid: an upper bound, CTAs past the last window exit)
    const i64 windows = std::min<i64>((lcap + kSortWindow - 1) / kSortWindow +
                                          2 * (bounded ? max_other : plan->n_large) + 2,
                                      0x7fffffff);
    const Rec* rr = reinterpret_cast<const Rec*>(r_list);
    const Rec* sr = reinterpret_cast<const Rec*>(s_list);
    k_lsort_win<<<(unsigned)windows, kSortThreads, kSortWindow * 12, s>>>(rr, sr, w.lrec, w.lwin,
                                                                          w.hdr, A.ls);
    for (int p = 0; p < A.ls.passes; ++p)
      k_lmerge<<<(unsigned)windows, 256, 0, s>>>(w.lrec, w.lwin, w.hdr, A.ls, p);
    k_lgather<<<(unsigned)windows, 256, 0, s>>>(rr, sr, w.lrec, w.lwin, w.hdr, A.ls);
  }
  if (rest > 0) {
    // the sorted/large launch keeps its own ticket (the look-back ids follow
    // the nested chunks', whose kernel has finished by then)
    if (ordered) cudaMemsetAsync(scratch, 0, 4, s);
#if PBSM_JOIN_PDL && PBSM_NESTED_PIPE
    // right behind the persistent nested kernel (nothing between them: no
    // huge-tile sort, no ordered ticket reset): start while it drains
    if (!ordered && cn > 0 && !(lcap > 0 && mtile > 0)) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)rest);
      cfg.blockDim = dim3(kJoinThreads);
      cfg.dynamicSmemBytes = sizeof(JoinSmem);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = emit ? cudaLaunchKernelEx(&cfg, k_join<true>, A)
                                 : cudaLaunchKernelEx(&cfg, k_join<false>, A);
      return e == cudaSuccess ? launch_status() : (int)e;
    }
#endif
    if (emit)
      k_join<true><<<(unsigned)rest, kJoinThreads, sizeof(JoinSmem), s>>>(A);
    else
      k_join<false><<<(unsigned)rest, kJoinThreads, sizeof(JoinSmem), s>>>(A);
  }
  return launch_status();
}
