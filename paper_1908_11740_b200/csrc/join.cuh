// join.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: subsystems 2-4: nested / sorted (segmented sort + forward scan) / large-tile mini-joins, count -> emit.
#pragma once

// ---------------------------------------------------------------- 2-4 join
struct JoinArgs {
  const uint4* jrec[2];    // [0] nested tiles, [1] sorted tiles
  const uint4* cdesc[2];
  const uint4* lrec;
  const u32* lpre;
  const u32* litem;  // large work item → tile (items < litem_n; the plan's table)
  u64 litem_n;
  LargeSort ls;            // huge tiles: sort buffers and the sorted copies (sweep.cuh)
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
  // bounded mode: entries the tile-list buffers hold (the scatter stopped at
  // them); a plan whose lists are longer makes every unit exit (no read past
  // the buffers) with PBSM_ERR_SCATTER_OVERFLOW, and the caller re-runs
  i64 list_cap_r, list_cap_s;
  // write guard folded into the nested join (g_tiles > 0): cursor ends vs
  // the counted ends, every tile (partition.py:229-233)
  const u32 *g_cur_r, *g_end_r, *g_cur_s, *g_end_s;
  u64 g_tiles;
  // ε-distance join (engine.py:201-206 fused into the mini-joins): a pair of
  // squares is kept only if its points, carried in the entries' pad words,
  // are within sqrt(eps_sq); eps = 0: plain join
  int eps;
  double eps_sq;
  // compact nested entries (SplitOut, partition.cuh): the nested region of
  // each list as 32-byte sectors; the exact yu columns (for a y-test inside
  // yu32's float32 gap) and the id columns (ids of the hits; null: rows)
  const Half* r32;
  const Half* s32;
  i64 cap32_r, cap32_s;
  const double* r_yu;
  const double* s_yu;
  const i64* r_ids;
  const i64* s_ids;
};

// _refine_pairs (engine.py:201-206): dx*dx + dy*dy <= eps^2, every operation
// rounded on its own (numpy: no FMA contraction).  Symmetric in a, b: IEEE
// a - b = -(b - a) exactly, and squares lose the sign.
__device__ __forceinline__ bool within_eps(double2 a, double2 b, double eps_sq) {
  const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= eps_sq;
}
// the point {px, py} of an ε-join entry (pad[1], pad[2], see write_rec)
__device__ __forceinline__ double2 rec_point(const Rec& r) {
  return *reinterpret_cast<const double2*>(&r.pad[1]);
}

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

// Large work items keep their hits as one bitmap row per lead thread (bit k
// of word w = other entry 32 w + k of the item), word-major so a warp's rows
// never share a bank: the count pass sets bits without atomics and the emit
// walks them — every pair is tested exactly once, however many hits an item
// has (a 4096-entry hit list made every denser item test all its pairs twice;
// on cfg3 that was most of them).
constexpr int kLargePiece = 256;  // other-side entries staged per step
static_assert(kLargeOther % 32 == 0 && kLargePiece % 32 == 0, "bitmap words");
struct LargeSmem {
  Rec other[kLargePiece];
  u32 bits[kLargeOther / 32][kJoinThreads];
  u64 bar;
  u64 scan[kJoinThreads / 32 + 1];
  u64 base;
  int unit;
};

union JoinSmem {
  ChunkSmem c;
  LargeSmem l;
  SweepSmem w;
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

// Bounded mode: the plan's tile lists are longer than the buffers the caller
// sized from a previous plan — the scatter stopped at the capacity, so no unit
// may stage entries: flag it (the caller re-runs with the exact plan) and exit.
__device__ __forceinline__ bool lists_overflow(const JoinArgs& A) {
  const bool over = A.hdr->list_r > A.list_cap_r || A.hdr->list_s > A.list_cap_s ||
                    (A.r32 && (A.hdr->nested_r > A.cap32_r || A.hdr->nested_s > A.cap32_s));
  if (over && threadIdx.x == 0) atomicOr(&A.hdr->error, PBSM_ERR_SCATTER_OVERFLOW);
  return over;
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
__device__ __forceinline__ u32 sweep_one(const ChunkSmem& S, int p, i64* out, int eps,
                                         double eps_sq) {
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
  const double2 mpt = eps ? rec_point(S.recs[S.sidx[p]]) : make_double2(0.0, 0.0);
  for (; k < hi; ++k) {
    if (S.sxl[k] > mxu) break;
    if (myl <= S.syu[k] && S.syl[k] <= myu && (yme || S.syin[k]) &&
        (!eps || within_eps(mpt, rec_point(S.recs[S.sidx[k]]), eps_sq))) {
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
  for (int p = tid; p < N; p += kJoinThreads) cnt += sweep_one<false>(S, p, nullptr, A.eps, A.eps_sq);
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
  for (int p = tid; p < N; p += kJoinThreads)
    out += 2 * (i64)sweep_one<true>(S, p, out, A.eps, A.eps_sq);
}

// Large join tiles (|R_T|+|S_T| > kLmax): work items of kLargeLead entries of
// the larger side (one per thread) × kLargeOther entries of the other side,
// which stream through shared memory in pieces.  Every (lead, other) pair is
// tested once with the full closed-interval predicate (intersects,
// geometry.py:59-61) and the class rule (>= 1 x-in and >= 1 y-in ⇔ Eq. 1
// owner tile); a hit sets its bit in the lead thread's bitmap row.
// One piece of n (<= kLargePiece, staged in S.other) entries, the item's
// entries [k0, k0 + n): returns the lead's hits among them.
__device__ __forceinline__ u32 large_pass(LargeSmem& S, int n, bool have, const Half& me,
                                          u32 k0, double2 mpt, int eps, double eps_sq) {
  if (!have) return 0;
  u32 c = 0;
  const double mxl = key_x(me.xl_key);
  const bool mxin = !(me.xl_key & kXOut), myin = !(me.xl_key & kYOut);
  // Branch-free test on both 16-byte halves of the record: no early-outs, so
  // the loads and compares of consecutive entries are in flight together
  auto test = [&](const Rec& o) -> bool {
    const ulonglong2 ox = *reinterpret_cast<const ulonglong2*>(&o.xl_key);
    const double2 oy = *reinterpret_cast<const double2*>(&o.yl);
    const u64 ok = ox.x;
    const double oxl = key_x(ok), oxu = __longlong_as_double((long long)ox.y);
    bool hit = (mxl <= oxu) & (oxl <= me.xu) & (me.yl <= oy.y) & (oy.x <= me.yu) &
               (mxin | !(ok & kXOut)) & (myin | !(ok & kYOut));
    if (eps) hit = hit && within_eps(mpt, rec_point(o), eps_sq);
    return hit;
  };
  for (int w0 = 0; w0 < n; w0 += 32) {  // (k0 and the piece size are multiples of 32)
    const int m = min(32, n - w0);
    u32 word = 0;
    int k = 0;
    for (; k + 4 <= m; k += 4) {
      u32 h = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) h |= (u32)test(S.other[w0 + k + u]) << u;
      word |= h << k;
    }
    for (; k < m; ++k) word |= (u32)test(S.other[w0 + k]) << k;
    S.bits[(k0 + (u32)w0) >> 5][threadIdx.x] = word;
    c += __popc(word);
  }
  return c;
}

template <bool EMIT>
__device__ void join_large(LargeSmem& S, const JoinArgs& A, i64 unit, i64 item, int lj,
                           uint4 rec) {
  const int tid = threadIdx.x;
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
  double2 mpt = make_double2(0.0, 0.0);
  if (have) {
    me = *reinterpret_cast<const Half*>(L + a);
    my_id = L[a].id;
    if (A.eps) mpt = rec_point(L[a]);
  }
  if (tid == 0) mbar_init(&S.bar, 1);
  __syncthreads();
  u32 phase = 0;
  u32 cnt = 0;
  for (u32 ob = o_beg; ob < o_end; ob += kLargePiece) {
    const int n = (int)min((u32)kLargePiece, o_end - ob);
    if (ob != o_beg) __syncthreads();  // previous piece fully consumed
    if (tid == 0) {
      mbar_expect_tx(&S.bar, (u32)n * (u32)sizeof(Rec));
      bulk_g2s(&S.other[0], O + ob, (u32)n * (u32)sizeof(Rec), &S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1u;
    cnt += large_pass(S, n, have, me, ob - o_beg, mpt, A.eps, A.eps_sq);
  }
  u64 total;
  const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
  if (!EMIT) {
    if (tid == 0 && total) atomicAdd(A.total, total);
    return;
  }
  if (tid == 0) S.base = reserve(A, unit, total);
  __syncthreads();
  if ((i64)(S.base + total) > A.capacity) {
    if (tid == 0 && total) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
    return;
  }
  if (!cnt) return;
  // emit: the thread's bitmap row, in other-entry order (its own bits only:
  // no barrier needed between the passes)
  i64* out = A.pairs + 2 * (i64)(S.base + excl);
  const u32 nw = (o_end - o_beg + 31u) >> 5;
  for (u32 w = 0; w < nw; ++w) {
    u32 word = S.bits[w][tid];
    while (word) {
      const u32 k = (u32)__ffs((int)word) - 1u;
      word &= word - 1u;
      const i64 oid = O[o_beg + 32u * w + k].id;
      *reinterpret_cast<longlong2*>(out) =
          lead_r ? make_longlong2(my_id, oid) : make_longlong2(oid, my_id);
      out += 2;
    }
  }
}

// Huge join tiles (large, and |R_T|*|S_T| above the plan's sweep threshold):
// both sides were sorted by x-lower
// (sweep.cuh: k_lsort_win, k_lmerge, k_lgather); work item = 256 consecutive
// sorted entries of one side, one leader per thread, each running the
// forward scan with a binary-searched start (sweep_leader).  Items of a tile:
// its R leader blocks, then its S leader blocks.
template <bool EMIT>
__device__ void join_sweep(SweepSmem& S, const JoinArgs& A, i64 unit, i64 item, int lo,
                           uint4 rec) {
  const int tid = threadIdx.x;
  const LargeGeo g = large_geo(A.hdr);
  const bool ok = large_fits(g, A.hdr, A.ls);
  const LargeSort& L = A.ls;
  const i64 nbR = (rec.z + kSweepLeaders - 1) / kSweepLeaders;
  const i64 li = item - (i64)A.lpre[lo];
  const bool lead_r = li < nbR;
  const i64 blk = lead_r ? li : li - nbR;
  const i64 r_lo = (i64)rec.x - g.rl0, s_lo = g.LR + ((i64)rec.y - g.sl0);
  const i64 l_lo = lead_r ? r_lo : s_lo, l_n = lead_r ? rec.z : rec.w;
  const i64 p_lo = lead_r ? s_lo : r_lo, p_n = lead_r ? rec.w : rec.z;
  const i64 me = l_lo + blk * kSweepLeaders + tid;
  const bool have = ok && me < l_lo + l_n;
  if (tid == 0) {
    S.pin_n = ok ? xin_count(L, p_lo, p_lo + p_n) : 0;
    S.ulo = 0x7fffffffffffffffll;
    S.uhi = 0;
    S.nhit = 0;
    if (!ok) atomicOr(&A.hdr->error, PBSM_ERR_SCATTER_OVERFLOW);
  }
  __syncthreads();
  const i64 pn = S.pin_n;
  u64 mk = 0;
  double mxu = 0, myl = 0, myu = 0;
  i64 k0 = 0, k1 = 0;
  if (have) {
    mk = L.sk[me];
    mxu = L.sxu[me];
    myl = L.syl[me];
    myu = L.syu[me];
    sweep_range(L, mk, mxu, lead_r, p_lo, pn, k0, k1);
    if (k1 > k0) {
      atomicMin(&S.ulo, (long long)k0);
      atomicMax(&S.uhi, (long long)k1);
    }
  }
  __syncthreads();
  const i64 ulo = S.ulo, uhi = S.uhi;
  const bool myin = !(mk & kYOut);
  // one pass over the union in pieces; pass 2 only if the hit list overflowed
  u32 cnt = 0;
  i64* out = nullptr;
  bool list_ok = true;
  for (int pass = 0; pass < 2; ++pass) {
    for (i64 pb = ulo; pb < uhi; pb += kSweepPiece) {
      const int n = (int)min((i64)kSweepPiece, uhi - pb);
      __syncthreads();  // previous piece consumed
      for (int k = tid; k < n; k += kJoinThreads) {
        S.pk[k] = L.sk[pb + k];
        S.py[k] = make_double2(L.syl[pb + k], L.syu[pb + k]);
      }
      __syncthreads();
      const i64 a = max(k0, pb), b = min(k1, pb + n);
      for (i64 k = a; k < b; ++k) {
        const u64 ok_ = S.pk[k - pb];
        const double2 oy = S.py[k - pb];
        if (myl <= oy.y && oy.x <= myu && (myin || !(ok_ & kYOut))) {
          if (pass == 0) {
            if (EMIT) {
              const u32 h = atomicAdd_block(&S.nhit, 1u);
              if (h < (u32)kSweepHits) {
                S.hit_p[h] = (u32)k;
                S.hit_l[h] = (unsigned char)tid;
              }
            }
            ++cnt;
          } else {
            const i64 a_id = L.sid[me], o_id = L.sid[k];
            *reinterpret_cast<longlong2*>(out) =
                lead_r ? make_longlong2(a_id, o_id) : make_longlong2(o_id, a_id);
            out += 2;
          }
        }
      }
    }
    if (pass == 1) break;
    u64 total;
    const u64 excl = block_excl_scan<kJoinThreads>((u64)cnt, &total, S.scan);
    if (!EMIT) {
      if (tid == 0 && total) atomicAdd(A.total, total);
      return;
    }
    if (tid == 0) S.base = reserve(A, unit, total);
    __syncthreads();
    if ((i64)(S.base + total) > A.capacity) {
      if (tid == 0 && total) atomicOr(&A.hdr->error, PBSM_ERR_PAIR_OVERFLOW);
      return;
    }
    if (total <= (u64)kSweepHits) {
      // every hit is in the list: one coalesced 16-byte store per hit
      i64* o = A.pairs + 2 * (i64)S.base;
      for (u32 h = tid; h < (u32)total; h += kJoinThreads) {
        const i64 a_id = L.sid[l_lo + blk * kSweepLeaders + S.hit_l[h]];
        const i64 o_id = L.sid[S.hit_p[h]];
        *reinterpret_cast<longlong2*>(o + 2 * (i64)h) =
            lead_r ? make_longlong2(a_id, o_id) : make_longlong2(o_id, a_id);
      }
      return;
    }
    out = A.pairs + 2 * (i64)(S.base + excl);
    (void)list_ok;
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
  // row form: per lead entry pos | o0 << 9 | |other| << 18 | R-leads << 26
  // (positions < kCapN = 512; |other| <= kLmax / 2 <= 128: the smaller side
  // of a tile of <= kLmax entries)
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

// Staged-entry views for the nested tests: the cp.async-staged SoA buffer
// (k_join_nested: {xl|label, xu}, {yl, yu}, id arrays + the ε-join's points)
// or the raw 64-byte records a TMA bulk copy landed (k_join_nested_pipe).
struct SoaView {
  static constexpr bool kRZ = false;
  const NestedBuf& B;
  const double2* ap;
  __device__ __forceinline__ ulonglong2 ax(int i) const { return B.ax[i]; }
  __device__ __forceinline__ double2 ay(int i) const { return B.ay[i]; }
  __device__ __forceinline__ i64 id(int i) const { return B.aid[i]; }
  __device__ __forceinline__ double2 pt(int i) const { return ap[i]; }
  __device__ __forceinline__ uint4 jr(int t) const { return B.jr[t]; }
};
struct RecView {
  static constexpr bool kRZ = false;
  const Rec* r;
  const uint4* j;
  __device__ __forceinline__ ulonglong2 ax(int i) const {
    return *reinterpret_cast<const ulonglong2*>(&r[i].xl_key);
  }
  __device__ __forceinline__ double2 ay(int i) const {
    return *reinterpret_cast<const double2*>(&r[i].yl);
  }
  __device__ __forceinline__ i64 id(int i) const { return r[i].id; }
  __device__ __forceinline__ double2 pt(int i) const { return rec_point(r[i]); }
  __device__ __forceinline__ uint4 jr(int t) const { return j[t]; }
};
// compact nested entries: {xl | label, xu, yl, yu32 | row << 32}; ay() gives
// {yl, yu32}, yu32 <= yu < the next float32 (y-tests: rz_le)
struct RecView32 {
  static constexpr bool kRZ = true;
  const Half* r;
  const uint4* j;
  int NR;  // entries [0, NR) are R's, the rest S's
  const double* yu_r;
  const double* yu_s;
  const i64* ids_r;
  const i64* ids_s;
  __device__ __forceinline__ ulonglong2 ax(int i) const {
    return *reinterpret_cast<const ulonglong2*>(&r[i].xl_key);
  }
  __device__ __forceinline__ u64 w3(int i) const {
    return (u64)__double_as_longlong(r[i].yu);
  }
  __device__ __forceinline__ double2 ay(int i) const {
    return make_double2(r[i].yl, (double)__uint_as_float((u32)w3(i)));
  }
  __device__ __forceinline__ double yl(int i) const { return r[i].yl; }
  __device__ __forceinline__ double yu_exact(int i) const {
    return __ldg((i < NR ? yu_r : yu_s) + (w3(i) >> 32));
  }
  __device__ __forceinline__ i64 id(int i) const {
    const i64 row = (i64)(w3(i) >> 32);
    const i64* ids = i < NR ? ids_r : ids_s;
    return ids ? __ldg(ids + row) : row;
  }
  __device__ __forceinline__ double2 pt(int) const { return make_double2(0.0, 0.0); }
  __device__ __forceinline__ uint4 jr(int t) const { return j[t]; }
};

// lo <= yu for an entry known by yu32 = RZ_float(yu): decided by yu32 and the
// next float32 except inside that gap, where the exact yu is read (rare)
template <typename View>
__device__ __forceinline__ bool rz_le(double lo, double yu32, const View& B, int e) {
  if (lo <= yu32) return true;
  if (lo >= (double)__uint_as_float(__float_as_uint((float)yu32) + 1u)) return false;
  return lo <= B.yu_exact(e);
}

// the full pair test (pair_ok) on two staged entries of any view
template <typename View>
__device__ __forceinline__ bool view_pair(const View& B, int a, int b) {
  const ulonglong2 ax = B.ax(a), bx = B.ax(b);
  const double2 ay = B.ay(a), by = B.ay(b);
  if constexpr (!View::kRZ) {
    return pair_ok(ax.x, __longlong_as_double((long long)ax.y), ay.x, ay.y, bx.x,
                   __longlong_as_double((long long)bx.y), by.x, by.y);
  } else {
    const bool xy = (key_x(ax.x) <= __longlong_as_double((long long)bx.y)) &
                    (key_x(bx.x) <= __longlong_as_double((long long)ax.y)) &
                    (((ax.x & bx.x) & kLabelMask) == 0ull);
    return xy && rz_le(ay.x, by.y, B, b) && rz_le(by.x, ay.y, B, a);
  }
}

// first tile of pair q0: binary search over the boundaries (the same
// addresses in every lane: broadcast reads)
template <typename Smem>
__device__ __forceinline__ int nested_tile_of(const Smem& S, int nt, u32 q0) {
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
template <typename Smem>
__device__ __forceinline__ int nested_step_tile(const Smem& S, int nt, u32 q0, int& lt,
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
template <typename Smem>
__device__ __forceinline__ void nested_pair(const Smem& S, int t, u32 q, int& pr, int& ps) {
  const TileInfo ti = S.ti[t];
  const u32 local = q - ti.p0;
  // local / ns: local < 2^16 and |local/ns - integer| >= 0.5/ns, so the
  // float estimate of (local + 0.5) / ns truncates to the exact quotient
  const u32 r = (u32)__float2int_rz(((float)local + 0.5f) * ti.inv_ns);
  pr = (int)(ti.rs0 & 0xffffu) + (int)r;
  ps = (int)(ti.rs0 >> 16) + (int)(local - r * ti.ns);
}

template <typename View>
__device__ __forceinline__ bool nested_hit(const View& B, int pr, int ps) {
  if constexpr (View::kRZ) return view_pair(B, pr, ps);
  const ulonglong2 rx = B.ax(pr), sx = B.ax(ps);
  const double2 ry = B.ay(pr), sy = B.ay(ps);
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
template <bool EPS>
__device__ __forceinline__ void nested_stage(NestedBuf& B, double2* ap, const JoinArgs& A,
                                             const NestedChunk& k) {
  const int N = k.NR + k.NS;
  for (int e = threadIdx.x; e < N; e += kNT) {
    const Rec* src = e < k.NR ? A.rl + k.d0.y + e : A.sl + k.d0.z + (e - k.NR);
    const unsigned char* g = reinterpret_cast<const unsigned char*>(src);
    cp_async16(&B.ax[e], g);
    cp_async16(&B.ay[e], g + 16);
    cp_async8(&B.aid[e], g + 32);
    if (EPS) cp_async16(&ap[e], g + 48);  // the point (pad[1], pad[2])
  }
  for (int t = threadIdx.x; t < k.nt; t += kNT) cp_async16(&B.jr[t], A.jrec[0] + k.d0.x + t);
}

// Row form: one lane per entry of each tile's larger ("lead") side, looping
// over the tile's other side (<= 32 entries with the default cost model,
// |R_T|*|S_T| <= 1024; <= 64 for any nested tile, |R_T|+|S_T| <= 128).  No per-pair index arithmetic; a warp runs max(|other|)
// steps over its 32 lead entries.  body(hit, pr, ps, ballot) is called by
// every lane of every step.
template <bool EPS, typename Smem, typename View, typename Body>
__device__ __forceinline__ void nested_rows(const Smem& S, const View& B, double eps_sq,
                                            u32 e_beg, u32 e_end, u32 e_step, int lane,
                                            Body&& body) {
  for (u32 g = e_beg; g < e_end; g += e_step) {
    const u32 ei = g + lane;
    const bool valid = ei < e_end;
    const u32 d = valid ? S.lead[ei] : 0u;
    const u32 pos = d & 511u, o0 = (d >> 9) & 511u, nO = valid ? (d >> 18) & 255u : 0u;
    const bool lr = (d >> 26) & 1u;
    const ulonglong2 mx = B.ax(pos);
    const double2 my = B.ay(pos);
    const double mxu = __longlong_as_double((long long)mx.y);
    const double2 mp = EPS ? B.pt(pos) : make_double2(0.0, 0.0);
    // compact entries: the lead's yl bracketed by float32 (tested against the
    // partners' float32 yu), its yu32 and the next float32 as doubles (the
    // partners' yl are tested against those) — no conversion per step
    float l_dn = 0.f, l_up = 0.f;
    double l_yu = 0.0, l_yu_next = 0.0;
    if constexpr (View::kRZ) {
      l_dn = __double2float_rd(my.x);
      l_up = __double2float_ru(my.x);
      const float v = __uint_as_float((u32)B.w3(pos));
      l_yu = (double)v;
      l_yu_next = (double)__uint_as_float(__float_as_uint(v) + 1u);
    }
    const u32 steps = __reduce_max_sync(0xffffffffu, nO);
    for (u32 j = 0; j < steps; ++j) {
      bool hit = false;
      if (j < nO) {
        const ulonglong2 ox = B.ax(o0 + j);
        if constexpr (View::kRZ) {
          const double o_yl = B.yl(o0 + j);
          const float o_yu = __uint_as_float((u32)B.w3(o0 + j));
          hit = (key_x(mx.x) <= __longlong_as_double((long long)ox.y)) & (key_x(ox.x) <= mxu) &
                (((mx.x & ox.x) & kLabelMask) == 0ull);
          if (hit) {  // lead.yl <= other.yu and other.yu's float32 gap
            if (l_dn > o_yu) hit = false;
            else if (!(l_up <= o_yu)) hit = my.x <= B.yu_exact((int)(o0 + j));
          }
          if (hit) {  // other.yl <= lead.yu
            if (o_yl >= l_yu_next) hit = false;
            else if (!(o_yl <= l_yu)) hit = o_yl <= B.yu_exact((int)pos);
          }
        } else {
          const double2 oy = B.ay(o0 + j);
          hit = pair_ok(mx.x, mxu, my.x, my.y, ox.x, __longlong_as_double((long long)ox.y),
                        oy.x, oy.y);
        }
        if (EPS) hit = hit && within_eps(mp, B.pt(o0 + j), eps_sq);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      body(hit, lr ? pos : o0 + j, lr ? o0 + j : pos, m);
    }
  }
}

// Pair-flattened form (PBSM_NESTED_ROWS=0): every (r, s) pair of every tile
// gets an index (tile-major, then r, then s); lane q of a warp-step tests pair q.
template <bool EPS, typename Smem, typename View, typename Body>
__device__ __forceinline__ void nested_flat(const Smem& S, const View& B, double eps_sq,
                                            int nt, u32 q_beg, u32 q_end, int lt, int lane,
                                            Body&& body) {
  for (u32 q0 = q_beg; q0 < q_end; q0 += 32u) {
    const u32 q = q0 + lane;
    const int t = nested_step_tile(S, nt, q0, lt, lane);
    bool hit = false;
    int pr = 0, ps = 0;
    if (q < q_end) {
      nested_pair(S, t, q, pr, ps);
      hit = nested_hit(B, pr, ps);
      if (EPS) hit = hit && within_eps(B.pt(pr), B.pt(ps), eps_sq);
    }
    body(hit, (u32)pr, (u32)ps, __ballot_sync(0xffffffffu, hit));
  }
}

// One staged chunk (B landed and visible): tables, count, reserve, emit.
template <bool EMIT, bool EPS, typename Smem, typename View>
__device__ __forceinline__ void nested_chunk(Smem& S, const View& B, const JoinArgs& A,
                                             const NestedChunk& k, i64 c) {
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
    tr[h] = t < nt ? B.jr(t) : make_uint4(0, 0, 0, 0);
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
      const u32 d = (o0 << 9) | (nO << 18) | ((u32)lr << 26);
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
  if (PBSM_NESTED_ROWS) nested_rows<EPS>(S, B, A.eps_sq, w_beg, w_end, 32u * kW, lane, count);
  else nested_flat<EPS>(S, B, A.eps_sq, nt, w_beg, w_end, lt_beg, lane, count);
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
          make_longlong2(B.id(v & 0xffffu), B.id(v >> 16));
    }
    return;
  }
  auto emit = [&](bool hit, u32 pr, u32 ps, unsigned m) {
    if (hit) {
      const i64 o = __popc(m & lt_mask);
      *reinterpret_cast<longlong2*>(out + 2 * o) = make_longlong2(B.id(pr), B.id(ps));
    }
    out += 2 * (i64)__popc(m);
  };
  if (PBSM_NESTED_ROWS) nested_rows<EPS>(S, B, A.eps_sq, w_beg, w_end, 32u * kW, lane, emit);
  else nested_flat<EPS>(S, B, A.eps_sq, nt, w_beg, w_end, lt_beg, lane, emit);
}

// One CTA per chunk (chunks handed out by ticket in the ordered mode, whose
// look-back needs launch order).  Static shared memory: the compiler then
// addresses it with constant offsets.  (A persistent variant that staged chunk
// i+1 with cp.async while joining chunk i was measured slower twice: more
// resident CTAs beat the deeper pipeline.)
template <bool EMIT, bool EPS>
#ifndef PBSM_NESTED_MINB
#define PBSM_NESTED_MINB (1536 / kNT)
#endif
__global__ void __launch_bounds__(kNT, EPS ? 4 : PBSM_NESTED_MINB) k_join_nested(JoinArgs A,
                                                                          i64 n_chunks) {
  __shared__ __align__(128) NestedSmem S;
  __shared__ __align__(16) double2 s_pt[EPS ? kCapN : 1];  // ε-join: the entries' points
  if (A.g_tiles) {  // the write guard, a grid-stride slice per CTA (all CTAs)
    bool bad = false;
    for (u64 t = blockIdx.x * (u64)kNT + threadIdx.x; t < A.g_tiles; t += (u64)gridDim.x * kNT)
      bad |= !cursor_done(A.g_cur_r[t], A.g_end_r[t]) || !cursor_done(A.g_cur_s[t], A.g_end_s[t]);
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
  if (A.bounded && lists_overflow(A)) return;
  nested_check(A, k);
  nested_stage<EPS>(S.buf, s_pt, A, k);
  cp_async_wait_all();
  __syncthreads();
  nested_chunk<EMIT, EPS>(S, SoaView{S.buf, s_pt}, A, k, c);
}

// ---- nested mini-joins, persistent + TMA-staged (the default for the
// unordered emit): each CTA takes chunks blockIdx.x, + gridDim.x, ...
// (static: no ticket).  A chunk's R range, S range and tile records are three
// contiguous byte ranges (k_plan_apply), so one thread stages it with three
// cp.async.bulk copies on a stage's mbarrier — no per-entry copies through the
// load/store units (k_join_nested's 3 cp.async per entry: ~39 M lane
// operations on cfg2) and no CTA launch per chunk — and the tests read the
// 64-byte records in place (RecView).  Measured (r02z2, bench.py 10 steps):
// 1 stage x 5 CTAs per SM beats the per-chunk kernel (cfg2 join 368 -> 333 µs,
// cfg5 262 -> 231, cfg3 3.15 -> 2.93 ms); 2-3 stages at 1-2 CTAs per SM and
// smaller buckets at 6-7 CTAs per SM were slower — resident CTAs hide the
// staging latency better than a deeper pipeline.
#ifndef PBSM_NESTED_PIPE
#define PBSM_NESTED_PIPE 1
#endif
#ifndef PBSM_PIPE_STAGES
#define PBSM_PIPE_STAGES 1
#endif
#ifndef PBSM_PIPE_CTAS
#define PBSM_PIPE_CTAS 5  // resident CTAs per SM (the grid: this many per SM)
#endif
// the compact-entry instance (MODE 2: 32-byte sectors, half the staging)
#ifndef PBSM_PIPE_STAGES32
#define PBSM_PIPE_STAGES32 1
#endif
// MODE 2: 6 CTAs per SM (40 registers, no spills); MODE 3, the same kernel
// for joins with few pairs per entry: 8 CTAs per SM (32 registers) — measured
// (r02zr): cfg2 (0.17 pairs / entry) 1.124 -> 1.091 ms at 8, but cfg3 (0.37)
// and cfg5 (0.48), whose emits do more, are faster at 6
#ifndef PBSM_PIPE_CTAS32
#define PBSM_PIPE_CTAS32 6
#endif
#ifndef PBSM_PIPE_CTAS32_FEW
#define PBSM_PIPE_CTAS32_FEW 8
#endif
__host__ __device__ constexpr int pipe_stages(int mode) {
  return mode >= 2 ? PBSM_PIPE_STAGES32 : PBSM_PIPE_STAGES;
}
__host__ __device__ constexpr int pipe_ctas(int mode) {
  return mode == 3 ? PBSM_PIPE_CTAS32_FEW : mode == 2 ? PBSM_PIPE_CTAS32 : PBSM_PIPE_CTAS;
}
template <typename RecT>
struct PipeStage {
  RecT recs[kCapN];        // R range, then S range (64-byte records or compact sectors)
  uint4 jr[kMaxTilesN];    // tile records
};
template <typename RecT, int kPipeStages>
struct PipeSmem {
  PipeStage<RecT> st[kPipeStages];
  u64 bar[kPipeStages];
  NestedChunk k[kPipeStages];
  // nested_chunk's working set (the names of NestedSmem)
  u32 lead[PBSM_NESTED_ROWS ? kCapN : 1];
  TileInfo ti[PBSM_NESTED_ROWS ? 1 : kMaxTilesN];
  u32 tb[PBSM_NESTED_ROWS ? 1 : kMaxTilesN + 33];
  u64 wtot[kNT / 32 + 1];
  u32 scan32[kNT / 32 + 1];
  u32 hits[kNT / 32][kHitCap];
  u64 base;
};

// thread 0: chunk c's descriptors → stage s, its three bulk copies
template <typename RecT, int ST>
__device__ __forceinline__ void pipe_issue(PipeSmem<RecT, ST>& S, const JoinArgs& A, int s,
                                           i64 c) {
  NestedChunk k = nested_desc(A, c);
  if (!k.ok) {
    atomicOr(&A.hdr->error, PBSM_ERR_INTERNAL);
    k.nt = k.NR = k.NS = 0;
  }
  S.k[s] = k;
  const u32 rb = (u32)k.NR * (u32)sizeof(RecT), sb = (u32)k.NS * (u32)sizeof(RecT);
  const u32 tb = (u32)k.nt * 16u;
  const RecT* rsrc;
  const RecT* ssrc;
  if constexpr (sizeof(RecT) == sizeof(Rec)) {
    rsrc = A.rl + k.d0.y;
    ssrc = A.sl + k.d0.z;
  } else {
    rsrc = A.r32 + k.d0.y;
    ssrc = A.s32 + k.d0.z;
  }
  mbar_expect_tx(&S.bar[s], rb + sb + tb);
  if (rb) bulk_g2s(&S.st[s].recs[0], rsrc, rb, &S.bar[s]);
  if (sb) bulk_g2s(&S.st[s].recs[k.NR], ssrc, sb, &S.bar[s]);
  if (tb) bulk_g2s(&S.st[s].jr[0], A.jrec[0] + k.d0.x, tb, &S.bar[s]);
}

// MODE 0: 64-byte records; 1: ε-join (64-byte records carrying the point);
// 2, 3: compact nested entries (RecView32) at two occupancies
template <int MODE>
using PipeRec = std::conditional_t<MODE >= 2, Half, Rec>;
template <int MODE>
using PipeSmemM = PipeSmem<PipeRec<MODE>, pipe_stages(MODE)>;
template <bool EMIT, int MODE>
__global__ void __launch_bounds__(kNT, pipe_ctas(MODE)) k_join_nested_pipe(JoinArgs A,
                                                                           i64 n_chunks) {
  constexpr bool EPS = MODE == 1;
  constexpr int kPipeStages = pipe_stages(MODE);
  extern __shared__ __align__(128) unsigned char pipe_raw[];
  PipeSmemM<MODE>& S = *reinterpret_cast<PipeSmemM<MODE>*>(pipe_raw);
  const int tid = threadIdx.x;
#if PBSM_JOIN_PDL
  // the sorted / large units (k_join, launched with programmatic stream
  // serialization) do not read anything this kernel writes: let them start
  // as soon as SM slots free up, filling this kernel's tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const i64 n_plan = A.bounded ? (i64)A.hdr->chunks_nested : n_chunks;
  const bool over = A.bounded && lists_overflow(A);
  if (tid == 0) {
    for (int q = 0; q < kPipeStages; ++q) mbar_init(&S.bar[q], 1);
    if (!over)
      for (int q = 0; q < kPipeStages; ++q) {
        const i64 c = blockIdx.x + (i64)q * gridDim.x;
        if (c < n_plan) pipe_issue(S, A, q, c);
      }
  }
  if (A.g_tiles) {  // the write guard, a grid-stride slice per CTA (all CTAs)
    bool bad = false;
    for (u64 t = blockIdx.x * (u64)kNT + tid; t < A.g_tiles; t += (u64)gridDim.x * kNT)
      bad |= !cursor_done(A.g_cur_r[t], A.g_end_r[t]) || !cursor_done(A.g_cur_s[t], A.g_end_s[t]);
    if (bad) atomicOr(&A.hdr->error, PBSM_ERR_OFFSET_MISMATCH);
  }
  __syncthreads();
  if (over) return;
  u32 phase = 0;  // bit q: the parity stage q waits for next
  for (i64 it = 0;; ++it) {
    const i64 c = blockIdx.x + it * gridDim.x;
    if (c >= n_plan) break;
    const int q = (int)(it % kPipeStages);
    mbar_wait(&S.bar[q], (phase >> q) & 1u);
    phase ^= 1u << q;
    const NestedChunk k = S.k[q];
    if constexpr (MODE >= 2)
      nested_chunk<EMIT, false>(S, RecView32{S.st[q].recs, S.st[q].jr, k.NR, A.r_yu, A.s_yu,
                                             A.r_ids, A.s_ids}, A, k, c);
    else
      nested_chunk<EMIT, EPS>(S, RecView{S.st[q].recs, S.st[q].jr}, A, k, c);
    __syncthreads();  // stage q consumed
    if (tid == 0) {
      const i64 cn = c + (i64)kPipeStages * gridDim.x;
      if (cn < n_plan) pipe_issue(S, A, q, cn);
    }
  }
}

// 4 CTAs per SM (64 registers; 3 fit at the uncapped 67): cfg3's large work
// items 1.33 -> 1.00 ms (8.31 -> 8.08 ms per join), cfg2 neutral (r03e)
#ifndef PBSM_JOIN_MINB
#define PBSM_JOIN_MINB 4
#endif
template <bool EMIT>
__device__ __forceinline__ void k_join_body(JoinArgs& A);

// PBSM_JOIN_PDL (common.cuh): k_join may start while the nested-chunk kernel
// still runs (programmatic dependent launch); every CTA waits for that grid
// before it exits, so the work after k_join in the stream sees both done
template <bool EMIT>
__global__ void __launch_bounds__(kJoinThreads, PBSM_JOIN_MINB) k_join(JoinArgs A) {
  k_join_body<EMIT>(A);
#if PBSM_JOIN_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <bool EMIT>
__device__ __forceinline__ void k_join_body(JoinArgs& A) {
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
  if (A.bounded && lists_overflow(A)) return;
  const i64 unit = cn + local;
  if (local < cs) join_sorted<EMIT>(U.c, A, unit, local);
  else {
    // large work item → its tile: the last whose item prefix is <= item
    // (32-ary search, every warp on its own: log32 dependent loads)
    const i64 item = local - cs;
    const i64 smin = A.hdr->sweep_min;  // (in flight during the search)
    int lo = 0, hi = (int)A.hdr->n_large;  // lpre[0] = 0 <= item
    const int lane = threadIdx.x & 31;
    // (the plan's item → tile table answers in one load what the search
    // finds in log32(n_large) dependent ones; items past the table search)
    if ((u64)item < A.litem_n) {
      lo = (int)__ldg(A.litem + item);
      hi = lo + 1;
    }
    while (hi - lo > 1) {
      const int step = (hi - lo + 31) >> 5;
      const int m = lo + lane * step;
      const unsigned le = __ballot_sync(0xffffffffu, m < hi && (i64)__ldg(A.lpre + m) <= item);
      lo += (31 - __clz(le)) * step;  // prefixes are non-decreasing: le is a lane prefix
      hi = min(hi, lo + step);
    }
    const uint4 rec = A.lrec[lo];
    if (is_huge(rec.z, rec.w, smin)) {
      // (an ε-join's plan has no huge tiles: the sorted copies carry no points)
      if (A.eps) {
        if (threadIdx.x == 0) atomicOr(&A.hdr->error, PBSM_ERR_INTERNAL);
        return;
      }
      join_sweep<EMIT>(U.w, A, unit, item, lo, rec);
    } else {
      join_large<EMIT>(U.l, A, unit, item, lo, rec);
    }
  }
}
