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
//                      tiles: work items of 256 lead x 1024 other entries
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
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>

#include "../../include/pbsm.h"

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
typedef unsigned short u16;

namespace {

// The kernels and their host glue, in dependency order (one translation unit,
// so every kernel is in one fatbinary and nothing crosses a link boundary).
#include "common.cuh"
#include "partition.cuh"
#include "sweep.cuh"
#include "join.cuh"
#include "extras.cuh"
#include "host.cuh"
#include "dist.cuh"
#include "units.cuh"

}  // namespace

// ======================================================================== ABI
extern "C" {

int32_t pbsm_abi_version(void) { return PBSM_ABI_VERSION; }

#define PBSM_STR2(x) #x
#define PBSM_STR(x) PBSM_STR2(x)
const char* pbsm_build_info(void) {
  return "pbsm sm_100a abi" PBSM_STR(PBSM_ABI_VERSION) ": count+validate / plan / scatter "
         "(join tiles only; 64B records, compact 32B nested entries) / guard / mini-joins: "
         "nested (persistent, TMA-staged) | sort+forward-scan | large (TMA-staged, hit bitmaps) "
         "| huge (sort+sweep), count->emit; pair groups; B=" PBSM_STR(PBSM_CHUNK_B) " Bn=" PBSM_STR(PBSM_CHUNK_BN) " Lmax=" PBSM_STR(
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
  k_count<false><<<part_blocks(n), 256, 0, as_stream(stream)>>>(xl, xu, yl, yu, n, kx, ky,
                                                                row_lo, row_hi, w.bx, w.by,
                                                                side ? w.cnt_s : w.cnt_r, side,
                                                                w.bc[side], w.hdr, 0.0);
  return launch_status();
}

int pbsm_count_points(const double* px, const double* py, int64_t n, int32_t side, double half,
                      void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                      void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      !(half > 0.0))
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!px || !py) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  k_count<true><<<part_blocks(n), 256, 0, as_stream(stream)>>>(px, nullptr, py, nullptr, n, kx,
                                                               ky, row_lo, row_hi, w.bx, w.by,
                                                               side ? w.cnt_s : w.cnt_r, side,
                                                               w.bc[side], w.hdr, half);
  return launch_status();
}

int pbsm_plan(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
              int64_t nested_max, int64_t sweep_min, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi)) return PBSM_E_ARG;
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
  cudaStream_t s = as_stream(stream);
  const i64 nm = nested_max < 0 ? (i64)kNestedMax : (i64)nested_max;
  const i64 sm = sweep_min < 0 ? (i64)kSweepMin : (i64)sweep_min;
  k_plan_reduce<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles, nm, sm,
                                                              w.partials, w.hdr);
  k_plan_partials<<<kNV + 1, kPartThreads, 0, s>>>(w.partials, w.nblocks, w.hdr, w.cdesc[0],
                                                w.cdesc[1], w.lpre, w.lwin, sm);
  PlanOut P;
  P.cur_r = w.cur_r;
  P.cur_s = w.cur_s;
  for (int q = 0; q < 2; ++q) {
    P.jrec[q] = w.jrec[q];
    P.cdesc[q] = w.cdesc[q];
  }
  P.lrec = w.lrec;
  P.lpre = w.lpre;
  P.lwin = w.lwin;
  P.litem = w.litem;
  k_plan_apply<<<(unsigned)w.nblocks, kPlanThreads, 0, s>>>(w.cnt_r, w.cnt_s, w.tiles,
                                                             w.nblocks, nm, sm, w.partials, P);
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

int pbsm_publish_header(void* ws, pbsm_header* out, void* stream) {
  if (!ws || !out) return PBSM_E_ARG;
  k_publish_header<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<const pbsm_header*>(ws), out);
  return launch_status();
}

static int scatter_impl(const int64_t* ids, const double* xl, const double* xu,
                        const double* yl, const double* yu, const void* band, int64_t n,
                        int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                        int32_t row_hi, pbsm_entry* out, int64_t capacity, void* stream,
                        double half = 0.0, void* rec32 = nullptr, int64_t cap32 = 0) {
  Ws w = ws_bind(ws, ws_layout(kx, ky, row_lo, row_hi));
#ifndef PBSM_SCAT_GRID
#define PBSM_SCAT_GRID 32  // blocks per SM (swept 8-1000 on cfg2/cfg3: 32 best)
#endif
  const i64 blocks = std::min<i64>((n + 255) / 256, (i64)num_sms() * PBSM_SCAT_GRID);
  const SplitOut sp{reinterpret_cast<Half*>(rec32), cap32,
                    reinterpret_cast<const i64*>(side ? &w.hdr->nested_s : &w.hdr->nested_r)};
  ScatterIn in{(const i64*)ids, xl, xu, yl, yu, reinterpret_cast<const BRec*>(band), half, sp};
  u32* cur = side ? w.cur_s : w.cur_r;
  Rec* o = reinterpret_cast<Rec*>(out);
  cudaStream_t s = as_stream(stream);
  if (half > 0.0)
    k_scatter<false, true><<<(unsigned)blocks, 256, 0, s>>>(in, n, kx, ky, row_lo, row_hi, w.bx,
                                                            w.by, cur, o, capacity, w.hdr);
  else if (band)
    k_scatter<true, false><<<(unsigned)blocks, 256, 0, s>>>(in, n, kx, ky, row_lo, row_hi, w.bx,
                                                            w.by, cur, o, capacity, w.hdr);
  else
    k_scatter<false, false><<<(unsigned)blocks, 256, 0, s>>>(in, n, kx, ky, row_lo, row_hi,
                                                             w.bx, w.by, cur, o, capacity, w.hdr);
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

int pbsm_scatter_split(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                       const double* yu, int64_t n, int32_t side, void* ws, int32_t kx,
                       int32_t ky, int32_t row_lo, int32_t row_hi, pbsm_entry* out,
                       int64_t capacity, void* rec32, int64_t capacity32, void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0 || capacity32 < 0 || n > 0xffffffffll)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu || (!out && capacity > 0) || !rec32) return PBSM_E_ARG;
  return scatter_impl(ids, xl, xu, yl, yu, nullptr, n, side, ws, kx, ky, row_lo, row_hi, out,
                      capacity, stream, 0.0, rec32, capacity32);
}

int pbsm_scatter_points(const int64_t* ids, const double* px, const double* py, int64_t n,
                        int32_t side, double half, void* ws, int32_t kx, int32_t ky,
                        int32_t row_lo, int32_t row_hi, pbsm_entry* out, int64_t capacity,
                        void* stream) {
  if (!ws || !grid_ok(kx, ky, row_lo, row_hi) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0 || !(half > 0.0))
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!px || !py || (!out && capacity > 0)) return PBSM_E_ARG;
  return scatter_impl(ids, px, nullptr, py, nullptr, nullptr, n, side, ws, kx, ky, row_lo,
                      row_hi, out, capacity, stream, half);
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

int64_t pbsm_join_scratch_bytes(int64_t n_units, int64_t large_entries) {
  if (n_units < 0 || large_entries < 0) return PBSM_E_ARG;
  return (int64_t)join_scratch(n_units, large_entries);
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

int pbsm_join_emit_split(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                         const pbsm_entry* r_list, int64_t r_capacity, const void* r32,
                         int64_t r32_capacity, const double* r_yu, const int64_t* r_ids,
                         const pbsm_entry* s_list, int64_t s_capacity, const void* s32,
                         int64_t s32_capacity, const double* s_yu, const int64_t* s_ids,
                         const pbsm_header* plan, int64_t max_nested_chunks,
                         int64_t max_other_units, int64_t large_capacity, int64_t max_tile,
                         void* scratch, int64_t* pairs, int64_t capacity, int32_t few_pairs,
                         void* stream) {
#if !PBSM_NESTED_PIPE
  return PBSM_E_ARG;  // the compact nested entries are read by the persistent nested join
#endif
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || capacity < 0 ||
      (capacity > 0 && !pairs) || !r32 || !s32 || !r_yu || !s_yu || r32_capacity < 0 ||
      s32_capacity < 0 || r_capacity < 0 || s_capacity < 0 || (!r_ids) != (!s_ids))
    return PBSM_E_ARG;
  if (!plan && (max_nested_chunks < 0 || max_other_units < 0 || max_nested_chunks > 0x7fffffff ||
                max_other_units > 0x7fffffff || large_capacity < 0 || max_tile < 0))
    return PBSM_E_ARG;
  SplitLists sp{r32, s32, r32_capacity, s32_capacity, r_yu, s_yu,
                reinterpret_cast<const i64*>(r_ids), reinterpret_cast<const i64*>(s_ids),
                few_pairs != 0};
  if (plan)
    return launch_join(true, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, plan, scratch,
                       pairs, capacity, as_stream(stream), -1, -1, r_capacity, s_capacity, 0, 0,
                       0, 0.0, &sp);
  return launch_join(true, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, nullptr, scratch,
                     pairs, capacity, as_stream(stream), max_nested_chunks, max_other_units,
                     r_capacity, s_capacity, large_capacity, max_tile, 0, 0.0, &sp);
}

int pbsm_join_emit_bounded(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                           const pbsm_entry* r_list, int64_t r_capacity,
                           const pbsm_entry* s_list, int64_t s_capacity,
                           int64_t max_nested_chunks, int64_t max_other_units,
                           int64_t large_capacity, int64_t max_tile, void* scratch,
                           int64_t* pairs, int64_t capacity, void* stream) {
  if (!ws || !scratch || !grid_ok(kx, ky, row_lo, row_hi) || capacity < 0 ||
      (capacity > 0 && !pairs) || max_nested_chunks < 0 || max_other_units < 0 ||
      max_nested_chunks > 0x7fffffff || max_other_units > 0x7fffffff || r_capacity < 0 ||
      s_capacity < 0 || large_capacity < 0 || max_tile < 0)
    return PBSM_E_ARG;
  return launch_join(true, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, nullptr, scratch,
                     pairs, capacity, as_stream(stream), max_nested_chunks, max_other_units,
                     r_capacity, s_capacity, large_capacity, max_tile);
}

// ε-distance join: the plan must hold no huge (sorted + swept) tiles, whose
// sorted copies carry no points — pbsm_plan with sweep_min = INT64_MAX
static bool eps_ok(const pbsm_header* plan, double eps_sq) {
  return plan && plan->max_huge == 0 && eps_sq >= 0.0;
}

int pbsm_join_count_eps(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                        const pbsm_entry* r_list, const pbsm_entry* s_list,
                        const pbsm_header* plan, void* scratch, double eps_sq, void* stream) {
  if (!ws || !scratch || !eps_ok(plan, eps_sq) || !grid_ok(kx, ky, row_lo, row_hi))
    return PBSM_E_ARG;
  return launch_join(false, false, ws, kx, ky, row_lo, row_hi, r_list, s_list, plan, scratch,
                     nullptr, 0, as_stream(stream), -1, -1, -1, -1, 0, 0, 1, eps_sq);
}

int pbsm_join_emit_eps(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                       const pbsm_entry* r_list, const pbsm_entry* s_list,
                       const pbsm_header* plan, void* scratch, int64_t* pairs,
                       int64_t capacity, int32_t ordered, double eps_sq, void* stream) {
  if (!ws || !scratch || !eps_ok(plan, eps_sq) || !grid_ok(kx, ky, row_lo, row_hi) ||
      capacity < 0 || (capacity > 0 && !pairs))
    return PBSM_E_ARG;
  return launch_join(true, ordered != 0, ws, kx, ky, row_lo, row_hi, r_list, s_list, plan,
                     scratch, pairs, capacity, as_stream(stream), -1, -1, -1, -1, 0, 0, 1,
                     eps_sq);
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

int pbsm_group_pairs(const int64_t* pairs, int64_t n, int64_t chunk_rows, int32_t n_groups,
                     int32_t self_join, int64_t* out, int64_t* counts, void* stream) {
  if (n < 0 || chunk_rows < 1 || n_groups < 1 || n_groups > kMaxGroups || !counts)
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(counts);
  cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long) * n_groups, s);  // counts | cursors
  if (n == 0) return launch_status();
  if (!pairs || !out || pairs == out) return PBSM_E_ARG;
  // a few thousand pairs per block: the per-block group runs stay long
  const unsigned blocks = (unsigned)std::max<i64>(1, std::min<i64>((n + 2047) / 2048,
                                                                   (i64)num_sms() * 8));
  k_group_count<<<blocks, 256, 0, s>>>((const i64*)pairs, n, chunk_rows, n_groups, self_join,
                                       cnt);
  k_group_place<<<blocks, 256, 0, s>>>((const i64*)pairs, n, chunk_rows, n_groups, self_join,
                                       cnt, cnt + n_groups, (i64*)out);
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

// ------------------------------------------------------------ strip routing
int64_t pbsm_route_scratch_bytes(int64_t n, int32_t ky, int32_t world) {
  if (n < 0 || ky < 1 || ky > 65535 || world < 1 || world > kMaxRanks) return PBSM_E_ARG;
  return (int64_t)route_layout(n, ky, world).total;
}

int pbsm_route_count(const double* yl, const double* yu, int64_t n, int32_t ky,
                     const int32_t* cuts, int32_t world, void* scratch, int64_t* dest_counts,
                     void* stream) {
  if (n < 0 || ky < 1 || ky > 65535 || world < 1 || world > kMaxRanks || !cuts || !scratch ||
      !dest_counts)
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  const RouteLayout L = route_layout(n, ky, world);
  char* b = (char*)scratch;
  double* by = (double*)(b + L.by);
  u32* cnt = (u32*)(b + L.cnt);
  u64* base = (u64*)(b + L.base);
  u64* part = (u64*)(b + L.part);
  k_bounds<<<(unsigned)((ky + 256) / 256), 256, 0, s>>>(by, ky);
  if (n > 0) {
    if (!yl || !yu) return PBSM_E_ARG;
    k_route<false><<<(unsigned)L.nb, kRouteThreads, 0, s>>>(nullptr, nullptr, nullptr, yl, yu, n,
                                                            ky, by, cuts, world, cnt, nullptr,
                                                            nullptr);
  } else {
    cudaMemsetAsync(cnt, 0, 4 * L.m, s);
  }
  const u64 sb = (L.m + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<(unsigned)sb, kScanThreads, 0, s>>>(cnt, L.m, part);
  k_scan_partials<<<1, 1024, 0, s>>>(part, sb, base, L.m);
  k_scan_apply<<<(unsigned)sb, kScanThreads, 0, s>>>(cnt, L.m, part, base);
  k_route_totals<<<(unsigned)((world + 255) / 256), 256, 0, s>>>(base, L.nb, world, L.m,
                                                                 (i64*)dest_counts);
  return launch_status();
}

int pbsm_route_pack(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                    const double* yu, int64_t n, int32_t ky, const int32_t* cuts, int32_t world,
                    void* scratch, void* records, void* stream) {
  if (n < 0 || ky < 1 || ky > 65535 || world < 1 || world > kMaxRanks || !cuts || !scratch)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu || !records || ((uintptr_t)records & 7u)) return PBSM_E_ARG;
  const RouteLayout L = route_layout(n, ky, world);
  char* b = (char*)scratch;
  k_route<true><<<(unsigned)L.nb, kRouteThreads, 0, as_stream(stream)>>>(
      (const i64*)ids, xl, xu, yl, yu, n, ky, (const double*)(b + L.by), cuts, world, nullptr,
      (const u64*)(b + L.base), (u64*)records);
  return launch_status();
}

// ------------------------------------------------------------ pair sort
int64_t pbsm_sort_pairs_scratch_bytes(int64_t n) {
  if (n < 0) return PBSM_E_ARG;
  return (int64_t)pair_sort_layout(n).total;
}

int pbsm_pair_digits(const int64_t* pairs, int64_t n, uint32_t* hist, void* stream) {
  if (n < 0 || !hist) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(hist, 0, 4 * 16 * 256, s);
  if (n == 0) return launch_status();
  if (!pairs || ((uintptr_t)pairs & 15u)) return PBSM_E_ARG;
  const unsigned blocks = (unsigned)std::max<i64>(1, std::min<i64>((n + 4095) / 4096,
                                                                   (i64)num_sms() * 4));
  k_pair_digits<<<blocks, kSortT, 0, s>>>((const ulonglong2*)pairs, n, hist);
  return launch_status();
}

int pbsm_sort_pairs(int64_t* pairs, int64_t n, uint32_t pass_mask, void* tmp, void* scratch,
                    void* stream) {
  if (n < 0) return PBSM_E_ARG;
  if (n <= 1 || (pass_mask & 0xffffu) == 0) return 0;
  if (!pairs || !tmp || !scratch || ((uintptr_t)pairs & 15u) || ((uintptr_t)tmp & 15u))
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  const PairSortLayout L = pair_sort_layout(n);
  char* b = (char*)scratch;
  u32* cnt = (u32*)(b + L.cnt);
  u64* base = (u64*)(b + L.base);
  u64* part = (u64*)(b + L.part);
  const u64 sb = (L.m + kScanTile - 1) / kScanTile;
  ulonglong2* src = (ulonglong2*)pairs;
  ulonglong2* dst = (ulonglong2*)tmp;
  for (int d = 0; d < 16; ++d) {
    if (!((pass_mask >> d) & 1u)) continue;
    k_pair_count<<<(unsigned)L.nb, kSortT, 0, s>>>(src, n, d, cnt);
    k_scan_reduce<<<(unsigned)sb, kScanThreads, 0, s>>>(cnt, L.m, part);
    k_scan_partials<<<1, 1024, 0, s>>>(part, sb, base, L.m);
    k_scan_apply<<<(unsigned)sb, kScanThreads, 0, s>>>(cnt, L.m, part, base);
    k_pair_scatter<<<(unsigned)L.nb, kSortT, 0, s>>>(src, dst, n, d, base);
    std::swap(src, dst);
  }
  if (src != (ulonglong2*)pairs)
    cudaMemcpyAsync(pairs, src, 16 * (size_t)n, cudaMemcpyDeviceToDevice, s);
  return launch_status();
}

// ------------------------------------------------------------ partition()
int64_t pbsm_partition_scratch_bytes(int64_t n, int32_t kx, int32_t ky) {
  if (n < 0 || kx < 1 || ky < 1 || kx > 65535 || ky > 65535) return PBSM_E_ARG;
  return (int64_t)assign_layout(n, kx, ky).total;
}

int pbsm_partition_count(const double* xl, const double* xu, const double* yl, const double* yu,
                         int64_t n, int32_t kx, int32_t ky, void* scratch, int64_t* total,
                         void* stream) {
  if (n < 0 || kx < 1 || ky < 1 || kx > 65535 || ky > 65535 || !scratch || !total)
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  const AssignLayout L = assign_layout(n, kx, ky);
  char* b = (char*)scratch;
  double* bx = (double*)(b + L.bx);
  double* by = (double*)(b + L.by);
  u32* per = (u32*)(b + L.per);
  u64* start = (u64*)(b + L.start);
  k_bounds<<<(unsigned)((kx + 256) / 256), 256, 0, s>>>(bx, kx);
  k_bounds<<<(unsigned)((ky + 256) / 256), 256, 0, s>>>(by, ky);
  if (n == 0) {
    cudaMemsetAsync(total, 0, 8, s);
    return launch_status();
  }
  if (!xl || !xu || !yl || !yu) return PBSM_E_ARG;
  const unsigned blocks = (unsigned)std::min<i64>((n + 255) / 256, (i64)num_sms() * 8);
  k_assign_count<<<blocks, 256, 0, s>>>(xl, xu, yl, yu, n, kx, ky, bx, by, per);
  k_scan_reduce<<<(unsigned)L.nb, kScanThreads, 0, s>>>(per, (u64)n, (u64*)(b + L.part));
  k_scan_partials<<<1, 1024, 0, s>>>((u64*)(b + L.part), L.nb, start, (u64)n);
  k_scan_apply<<<(unsigned)L.nb, kScanThreads, 0, s>>>(per, (u64)n, (u64*)(b + L.part), start);
  cudaMemcpyAsync(total, start + n, 8, cudaMemcpyDeviceToDevice, s);
  return launch_status();
}

int pbsm_partition_write(const int64_t* ids, const double* xl, const double* xu,
                         const double* yl, const double* yu, int64_t n, int32_t kx, int32_t ky,
                         void* scratch, int64_t total, void* keys, void* keys_tmp,
                         void* sort_scratch, int64_t* out_ids, double* out_xl, double* out_xu,
                         double* out_yl, double* out_yu, int64_t* offsets, void* stream) {
  if (n < 0 || kx < 1 || ky < 1 || kx > 65535 || ky > 65535 || !scratch || total < 0 ||
      !offsets)
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  const AssignLayout L = assign_layout(n, kx, ky);
  char* b = (char*)scratch;
  const double* bx = (const double*)(b + L.bx);
  const double* by = (const double*)(b + L.by);
  const u64 tiles = (u64)kx * (u64)ky;
  if (total > 0) {
    if (!xl || !xu || !yl || !yu || !keys || !keys_tmp || !sort_scratch || !out_ids || !out_xl ||
        !out_xu || !out_yl || !out_yu)
      return PBSM_E_ARG;
    const unsigned blocks = (unsigned)std::min<i64>((n + 255) / 256, (i64)num_sms() * 8);
    k_assign_write<<<blocks, 256, 0, s>>>(xl, xu, yl, yu, n, kx, ky, bx, by,
                                          (const u64*)(b + L.start), (ulonglong2*)keys);
    // digits that can vary: rows < n (low word), tiles < kx*ky (high word)
    u32 mask = 0;
    for (int d = 0; d < 7; ++d) {
      if (((u64)(n - 1) >> (8 * d)) != 0) mask |= 1u << d;
      if (((tiles - 1) >> (8 * d)) != 0) mask |= 1u << (8 + d);
    }
    int rc = pbsm_sort_pairs((int64_t*)keys, total, mask, keys_tmp, sort_scratch, stream);
    if (rc) return rc;
  }
  const unsigned gb = (unsigned)std::max<i64>(1, std::min<i64>((total + 256) / 256,
                                                               (i64)num_sms() * 8));
  k_assign_gather<<<gb, 256, 0, s>>>((const ulonglong2*)keys, total, tiles, (const i64*)ids, xl,
                                     xu, yl, yu, (i64*)out_ids, out_xl, out_xu, out_yl, out_yu,
                                     (i64*)offsets);
  return launch_status();
}

// ------------------------------------------------------------ unit pipeline
static int unit_nb() { return std::min(num_sms(), 1024); }

// the dynamic shared-memory opt-in of the 128-KB kernels, per device
static int unit_smem_attrs() {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & (kMaxDevices - 1));
  if (done.load(std::memory_order_acquire) & bit) return 0;
  cudaError_t e = cudaFuncSetAttribute(k_ucount, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       4 * kUnitMaxCells);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_ubin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             4 * kUnitMaxCells);
  if (e != cudaSuccess) return (int)e;
  done.fetch_or(bit, std::memory_order_release);
  return 0;
}

int32_t pbsm_unit_supported(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi) {
  UGeo g;
  return unit_geometry(kx, ky, row_lo, row_hi, g) ? 1 : 0;
}

int64_t pbsm_unit_workspace_bytes(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi) {
  UGeo g;
  if (!unit_geometry(kx, ky, row_lo, row_hi, g)) return PBSM_E_ARG;
  return (int64_t)ulayout(g, unit_nb()).total;
}

int64_t pbsm_unit_bin_bytes(int64_t records) {
  if (records < 0) return PBSM_E_ARG;
  return (int64_t)(align_up(32 * (size_t)records, 256) + align_up(4 * (size_t)records, 256));
}

int64_t pbsm_unit_scratch_bytes(int64_t slots) {
  if (slots < 0 || slots > 0xffffffffll) return PBSM_E_ARG;
  return (int64_t)uscratch_bytes((u64)slots);
}

int pbsm_unit_init(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   void* stream) {
  UGeo g;
  if (!ws || !unit_geometry(kx, ky, row_lo, row_hi, g)) return PBSM_E_ARG;
  const ULayout L = ulayout(g, unit_nb());
  UWs w = ubind(ws, L);
  const u64 nz = (L.cls - L.cont[0]) / 4;  // cont[2]
  const unsigned blocks = (unsigned)std::max<i64>(1, std::min<i64>((i64)(nz + 255) / 256,
                                                                    (i64)num_sms() * 2));
  k_uinit<<<blocks, 256, 0, as_stream(stream)>>>(w.hdr, w.cont[0], nz, w.cls, w.bx, kx, w.by,
                                                 ky);
  return launch_status();
}

int pbsm_unit_count(const double* xl, const double* xu, const double* yl, const double* yu,
                    int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                    int32_t row_hi, void* stream) {
  UGeo g;
  if (!ws || !unit_geometry(kx, ky, row_lo, row_hi, g) || n < 0 || (side != 0 && side != 1) ||
      n > 0xffffffffll)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu) return PBSM_E_ARG;
  int rc = unit_smem_attrs();
  if (rc) return rc;
  UWs w = ubind(ws, ulayout(g, unit_nb()));
  const int nb = upart_blocks(n, w.nb);
  k_ucount<<<nb, kUCountThreads, 4 * (size_t)g.cells, as_stream(stream)>>>(
      xl, xu, yl, yu, n, g, w.bx, w.by, w.bhist[side], w.cont[side], w.hdr, side);
  return launch_status();
}

int pbsm_unit_map(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi, int64_t n_r,
                  int64_t n_s, int64_t target, void* stream) {
  UGeo g;
  if (!ws || !unit_geometry(kx, ky, row_lo, row_hi, g) || n_r < 0 || n_s < 0) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  UWs w = ubind(ws, ulayout(g, unit_nb()));
  const int nbR = n_r ? upart_blocks(n_r, w.nb) : 0, nbS = n_s ? upart_blocks(n_s, w.nb) : 0;
  const u32 t = target > 0 ? (u32)std::min<int64_t>(target, 1 << 30) : (u32)PBSM_UNIT_TARGET;
  k_ucell_sum<<<(2 * g.cells + 255) / 256, 256, 0, s>>>(w.bhist[0], nbR, w.bhist[1], nbS,
                                                         g.cells, w.first[0], w.first[1]);
  const unsigned rb = (unsigned)((g.rows + kMapRowsPerBlock - 1) / kMapRowsPerBlock);
  k_umap_rows<<<rb, 256, 0, s>>>(g, w.first[0], w.cont[0], w.first[1], w.cont[1], t,
                                 w.cell_unit, w.unR, w.unS, w.row_live, w.row_nR, w.row_nS,
                                 w.cls, w.hdr);
  k_umap_scan<<<1, kUMapThreads, 0, s>>>(g, w.row_live, w.row_nR, w.row_nS, w.cls, w.hdr);
  k_umap_write<<<rb, 256, 0, s>>>(g, w.cell_unit, w.unR, w.unS, w.row_live, w.row_nR, w.row_nS,
                                  w.cls, w.units, w.order, w.bhist[0], nbR, w.bhist[1], nbS,
                                  w.blk_base[0], w.blk_base[1], w.ccur[0], w.ccur[1]);
  return launch_status();
}

int pbsm_unit_bin(const double* xl, const double* xu, const double* yl, const double* yu,
                  int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                  int32_t row_hi, void* bin, int64_t capacity, void* stream) {
  UGeo g;
  if (!ws || !unit_geometry(kx, ky, row_lo, row_hi, g) || n < 0 || (side != 0 && side != 1) ||
      capacity < 0 || n > 0xffffffffll)
    return PBSM_E_ARG;
  if (n == 0) return 0;
  if (!xl || !xu || !yl || !yu || (!bin && capacity > 0)) return PBSM_E_ARG;
  int rc = unit_smem_attrs();
  if (rc) return rc;
  UWs w = ubind(ws, ulayout(g, unit_nb()));
  URec* b = reinterpret_cast<URec*>(bin);
  u32* bidx = reinterpret_cast<u32*>(reinterpret_cast<char*>(bin) +
                                     align_up(32 * (size_t)capacity, 256));
  const int nb = upart_blocks(n, w.nb);  // the same blocks as pbsm_unit_count
  k_ubin<<<nb, kUCountThreads, 4 * (size_t)g.cells, as_stream(stream)>>>(
      xl, xu, yl, yu, n, g, w.bx, w.by, w.cell_unit, w.blk_base[side], w.ccur[side], b, bidx,
      capacity, w.hdr);
  return launch_status();
}

int pbsm_unit_join(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const void* bin_r, int64_t bin_r_capacity, const void* bin_s,
                   int64_t bin_s_capacity, const int64_t* r_ids, const int64_t* s_ids,
                   void* scratch, int64_t scratch_slots, int64_t max_units, int64_t* pairs,
                   int64_t capacity, void* stream) {
  UGeo g;
  if (!ws || !unit_geometry(kx, ky, row_lo, row_hi, g) || bin_r_capacity < 0 ||
      bin_s_capacity < 0 || scratch_slots < 0 || scratch_slots > 0xffffffffll || capacity < 0 ||
      (capacity > 0 && !pairs) || !scratch)
    return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  UWs w = ubind(ws, ulayout(g, unit_nb()));
  // reset the join-phase block of the header (scratch_used .. pad2)
  cudaMemsetAsync(&w.hdr->scratch_used, 0,
                  offsetof(pbsm_uheader, n_def_tiles) - offsetof(pbsm_uheader, scratch_used), s);
  UJoinArgs A;
  A.g = g;
  A.bx = w.bx;
  A.by = w.by;
  A.units = w.units;
  A.order = w.order;
  A.hdr = w.hdr;
  const void* bins[2] = {bin_r, bin_s};
  const i64 caps[2] = {bin_r_capacity, bin_s_capacity};
  for (int q = 0; q < 2; ++q) {
    A.bin[q] = reinterpret_cast<const URec*>(bins[q]);
    A.bidx[q] = reinterpret_cast<const u32*>(reinterpret_cast<const char*>(bins[q]) +
                                             align_up(32 * (size_t)caps[q], 256));
    A.bcap[q] = caps[q];
  }
  A.ids[0] = (const i64*)r_ids;
  A.ids[1] = (const i64*)s_ids;
  A.sc = uscratch_bind(scratch, (u64)scratch_slots);
  A.pairs = (i64*)pairs;
  A.capacity = capacity;
  const i64 grid = max_units > 0 ? std::min<i64>(max_units, g.cells) : g.cells;
  k_ujoin<<<(unsigned)std::max<i64>(1, grid), kUJoinThreads, 0, s>>>(A);
  k_uchunks<<<(unsigned)(num_sms() * 6), kUJoinThreads, 0, s>>>(A);
  k_ularge<<<(unsigned)(num_sms() * 2), kJoinThreads, sizeof(ULargeSmem), s>>>(A);
  return launch_status();
}

int pbsm_read_uheader(void* ws, pbsm_uheader* out, void* stream) {
  if (!ws || !out) return PBSM_E_ARG;
  cudaStream_t s = as_stream(stream);
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, out);
  if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer == (void*)out) {
    k_publish_uheader<<<1, 32, 0, s>>>(reinterpret_cast<const pbsm_uheader*>(ws), out);
    e = cudaGetLastError();
  } else {
    cudaGetLastError();
    e = cudaMemcpyAsync(out, ws, sizeof(pbsm_uheader), cudaMemcpyDeviceToHost, s);
  }
  if (e != cudaSuccess) return (int)e;
  e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
