/*
 * pbsm.h — C ABI of the B200-native PBSM filter step (arXiv 1908.11740).
 *
 * This is the drop-in boundary for the reference's kernel plugin protocol
 * (`backends.get_kernels(name)` → module of six kernels,
 * /root/reference/pkg/src/sweepjoin/backends.py:41-50, kernels in
 * /root/reference/pkg/src/sweepjoin/_kernels.pyx).  The reference calls its
 * kernels once per input slice or per tile (10^4–10^7 calls); a GPU cannot
 * amortise launches at that granularity, so this ABI is *join-granular*: each
 * entry point below replaces one reference kernel for ALL tiles at once.
 *
 *   reference kernel (file:line)                      → entry point here
 *   count_tiles      _kernels.pyx:34-58               → pbsm_count
 *   compute_segment_offsets partition.py:151-164      → pbsm_plan
 *   (+ build_task_queue engine.py:84-100)
 *   write_tiles      _kernels.pyx:61-98               → pbsm_scatter
 *   (+ overflow guard partition.py:229-233)
 *   sort_segment     _kernels.pyx:188-228  ┐
 *   sweep_count      _kernels.pyx:304-315  ├─fused──→ pbsm_join_count
 *   sweep_collect    _kernels.pyx:318-341  ┘          pbsm_join_emit
 *   (+ aggregation   engine.py:293-309)
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer owned by the caller (PyTorch in the
 *     shipped host code); the library never allocates device memory.  Its
 *     only global state is a per-device cache of two idempotent facts (SM
 *     count, the shared-memory opt-in of the join kernels), kept in atomics,
 *     so calls are safe from any host thread on any device/stream; joins in
 *     flight at the same time need their own workspace, lists and scratch.
 *   - `stream` is a cudaStream_t passed as void*; every entry point only
 *     enqueues work on it (no implicit synchronisation) except
 *     pbsm_read_header, which is the one documented host sync point.
 *   - Return value: 0 = OK, >0 = cudaError_t of a failed launch, <0 = PBSM_E_*.
 *   - Coordinates are float64 in [0,1] (the reference's normalised domain,
 *     geometry.py:1-6); inputs are the reference's SoA columns
 *     (ids int64, xl, xu, yl, yu float64 — geometry.py:109-130).
 *   - Grid: kx columns × ky rows; flat tile = row*kx + col
 *     (partition.py:53-69).  2D grid: kx = ky = K.  1D stripes along x:
 *     kx = K, ky = 1; along y: kx = 1, ky = K.  A strip (multi-GPU shard)
 *     is the tile-row range [row_lo, row_hi); single GPU: [0, ky).
 */
#ifndef PBSM_H_
#define PBSM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBSM_ABI_VERSION 10

/* library error codes (negative) */
#define PBSM_E_ARG        (-1)  /* bad argument (null pointer, k out of range, ...) */
#define PBSM_E_OVERFLOW   (-2)  /* partition write overflow (partition.py:229-233)  */
#define PBSM_E_TOO_LARGE  (-3)  /* a total exceeds the 32-bit offset range           */
#define PBSM_E_PAIRS      (-4)  /* pair buffer smaller than the counted result       */

/* device-side error bits, reported in pbsm_header.error */
#define PBSM_ERR_SCATTER_OVERFLOW  1u  /* a scatter cursor left its tile range       */
#define PBSM_ERR_OFFSET_MISMATCH   2u  /* count and write passes disagree            */
#define PBSM_ERR_TOTAL_RANGE       4u  /* A_R / A_S / W exceed 2^32-1                 */
#define PBSM_ERR_PAIR_OVERFLOW     8u  /* pair buffer too small: re-run with >= pairs   */
#define PBSM_ERR_INVERTED         16u  /* R has xl > xu or yl > yu (or NaN); S: << 2    */
#define PBSM_ERR_RANGE            32u  /* R has a coordinate outside [0, 1];  S: << 2   */
#define PBSM_ERR_INTERNAL        256u  /* a work unit violated a plan invariant          */

/* one tile-list entry: a 64-byte, 64-byte-aligned record, so the random
 * scatter writes whole 32-byte sectors and a chunk of tiles is one contiguous
 * range for the TMA bulk copy.  The two top bits of `xl` (always zero for a
 * float64 in [0,1]) carry the class label of the entry in its tile: bit 63 =
 * x-out (starts left of the tile), bit 62 = y-out (starts below the tile).
 * A = neither, B = y-out, C = x-out, D = both — the class scheme of
 * PAPER.md:651-733. */
typedef struct pbsm_entry {
  uint64_t xl_key;
  double xu, yl, yu;
  int64_t id;
  uint64_t pad[3];
} pbsm_entry;

/* plan/result totals, device-resident at the start of the workspace.
 * Join tiles (both inputs non-empty, build_task_queue engine.py:97) are
 * split by a per-tile cost model into three mini-join strategies:
 *   nested — |R_T|+|S_T| <= LMAX and |R_T|*|S_T| <= NESTED_MAX: every
 *            (r, s) pair of the tile tested with the class rule (cheaper
 *            than sorting when the tile is this small);
 *   sorted — |R_T|+|S_T| <= LMAX otherwise: per-tile segmented sort by x-lower
 *            + forward-scan sweep (Alg. 1) in shared memory;
 *   large  — |R_T|+|S_T| > LMAX: each side sorted by x-lower in global
 *            memory (sort_segment), then the forward-scan sweep (Alg. 1)
 *            with one leader per thread, 256 leaders per work item.
 * Work units of one join launch: [nested chunks | sorted chunks | large items]. */
typedef struct pbsm_header {
  int64_t a_r;            /* Σ per-tile R counts = PartitionedDataset.total_assigned */
  int64_t a_s;            /* same for S                                             */
  int64_t list_r;         /* R entries written to tile lists (join tiles only)     */
  int64_t list_s;         /* same for S                                             */
  int64_t n_nested;       /* join tiles per strategy                                */
  int64_t n_sorted;
  int64_t n_large;
  int64_t w_nested;       /* entries (R+S) in nested / sorted tiles                 */
  int64_t w_sorted;
  int64_t chunks_nested;  /* CTA chunks of nested / sorted tiles                    */
  int64_t chunks_sorted;
  int64_t n_items;        /* work items of the large tiles                          */
  int64_t pairs;          /* result_count, valid after pbsm_join_count/emit         */
  int64_t pair_bound;     /* Σ |R_T|·|S_T| over join tiles (>= pairs)               */
  int64_t max_tile;       /* largest |R_T|+|S_T| over join tiles                   */
  int64_t large_r;        /* R entries in large tiles                               */
  int64_t large_s;        /* same for S                                             */
  int64_t sweep_min;      /* large tiles with |R_T|*|S_T| above this are sorted +   */
                          /* swept, the others brute-forced (pbsm_plan)             */
  int64_t max_huge;       /* largest side of a sorted + swept tile                  */
  int64_t nested_r;       /* R entries in nested tiles: the nested region of R's    */
  int64_t nested_s;       /* list is positions [0, nested_r); same for S            */
  uint32_t error;         /* PBSM_ERR_* bits                                        */
  uint32_t pad;
} pbsm_header;

/* Bytes of the grid workspace for a kx × (row_hi-row_lo) strip. */
int64_t pbsm_workspace_bytes(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi);

/* Zero counters and build the exact tile-boundary tables i/k
 * (geometry.py:82-84).  Must precede pbsm_count for each join. */
int pbsm_init(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
              void* stream);

/* count_tiles (_kernels.pyx:34-58) for ALL n rectangles of one input
 * (side 0 = R, 1 = S): per-tile assignment counts in the workspace. */
int pbsm_count(const double* xl, const double* xu, const double* yl,
               const double* yu, int64_t n, int32_t side, void* ws,
               int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
               void* stream);

/* compute_segment_offsets (partition.py:151-164) for both inputs plus the
 * join-task plan (build_task_queue, engine.py:84-100): CSR offsets, the join
 * tiles of each mini-join strategy, their CTA chunks and the large-tile work
 * items.  nested_max: cost-model threshold on |R_T|*|S_T| for the nested
 * strategy (< 0: the built-in default; 0: sort + sweep every small tile);
 * sweep_min: large tiles with |R_T|*|S_T| above it are sorted + swept, the
 * others brute-forced (< 0: the built-in default; 0: sweep every large tile). */
int pbsm_plan(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
              int64_t nested_max, int64_t sweep_min, void* stream);

/* Copy the device header to *out and synchronise the stream. */
int pbsm_read_header(void* ws, pbsm_header* out, void* stream);
/* Enqueue only: a tiny kernel stores the device header into *out, which must
 * be page-locked host memory (device-mapped); the caller synchronises later.
 * Capturable in a CUDA graph (the repeated-shape path replays init → count →
 * plan → scatter → bounded emit → this publish as one graph). */
int pbsm_publish_header(void* ws, pbsm_header* out, void* stream);

/* write_tiles (_kernels.pyx:61-98) for ALL n rectangles of one input:
 * scatter each rectangle into the list of every JOIN tile it overlaps (tiles
 * where the other input is empty can produce no pair and get no list),
 * labelled with its class there.  `out` holds `capacity` entries
 * (= header.list_r or list_s).  ids may be NULL: the entries then carry the
 * row index, and pbsm_map_ids turns the emitted pairs into ids later (the
 * host→device copy of the id columns overlaps the join). */
int pbsm_scatter(const int64_t* ids, const double* xl, const double* xu,
                 const double* yl, const double* yu, int64_t n, int32_t side,
                 void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                 pbsm_entry* out, int64_t capacity, void* stream);

/* ε-distance join (epsilon_distance_join, engine.py:326-353), fused: the
 * inputs are the POINT columns px, py (the lower corners of the caller's
 * rectangles, engine.py:333-334) and each one stands for the side-eps square
 * clip(p -/+ half, 0, 1), half = eps / 2.0 — computed inside the kernels with
 * the reference's numpy arithmetic (engine.py:342-350), never materialised.
 * pbsm_count_points / pbsm_scatter_points are pbsm_count / pbsm_scatter over
 * those squares; each entry also carries its point (pbsm_entry.pad[1..2]),
 * and pbsm_join_count_eps / pbsm_join_emit_eps keep a candidate pair only if
 * dx*dx + dy*dy <= eps_sq (every operation rounded on its own, as numpy:
 * _refine_pairs, engine.py:201-206) — in the count pass and the emit alike,
 * so no candidate list is ever written.  The plan must come from
 * pbsm_plan(..., sweep_min = INT64_MAX) (no sorted + swept tiles: their
 * sorted copies carry no points); otherwise PBSM_E_ARG.  ids may be NULL
 * (row indices, see pbsm_map_ids). */
int pbsm_count_points(const double* px, const double* py, int64_t n, int32_t side, double half,
                      void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                      void* stream);
int pbsm_scatter_points(const int64_t* ids, const double* px, const double* py, int64_t n,
                        int32_t side, double half, void* ws, int32_t kx, int32_t ky,
                        int32_t row_lo, int32_t row_hi, pbsm_entry* out, int64_t capacity,
                        void* stream);

/* Compact nested entries (the shipped driver's default where it applies):
 * the NESTED region of each tile list (positions [0, header.nested_r /
 * nested_s), every entry of a tile the nested mini-join tests) is written as
 * one 32-byte sector per entry {xl | label, xu, yl, yu32 | row << 32} into
 * rec32 — yu rounded toward zero to float32 and the entry's row index — and
 * the sorted / large regions as 64-byte entries into out (ids, or rows if ids
 * is NULL).  The scatter then stores one sector per nested entry instead of
 * two.  pbsm_join_emit_split reads the compact entries: a y-test is decided by
 * yu32 and the next float32 except inside that gap, where the exact yu is read
 * from r_yu / s_yu (the input columns, by row); hit ids come from r_ids /
 * s_ids by row (both NULL: the pairs hold row indices, map them with
 * pbsm_map_ids).  Takes the host plan (exact grids) or plan = NULL and the
 * bounds of pbsm_join_emit_bounded.  few_pairs != 0 (an occupancy hint: the
 * join is expected to emit well under one pair per 4 entries) runs the
 * nested join at 8 CTAs per SM instead of 6.  Unordered placement; not for
 * ε-joins or the binned scatter; n < 2^32. */
int pbsm_scatter_split(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                       const double* yu, int64_t n, int32_t side, void* ws, int32_t kx,
                       int32_t ky, int32_t row_lo, int32_t row_hi, pbsm_entry* out,
                       int64_t capacity, void* rec32, int64_t capacity32, void* stream);
int pbsm_join_emit_split(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                         const pbsm_entry* r_list, int64_t r_capacity, const void* r32,
                         int64_t r32_capacity, const double* r_yu, const int64_t* r_ids,
                         const pbsm_entry* s_list, int64_t s_capacity, const void* s32,
                         int64_t s32_capacity, const double* s_yu, const int64_t* s_ids,
                         const pbsm_header* plan, int64_t max_nested_chunks,
                         int64_t max_other_units, int64_t large_capacity, int64_t max_tile,
                         void* scratch, int64_t* pairs, int64_t capacity, int32_t few_pairs,
                         void* stream);

/* Binned scatter (worth it when an input's tile lists are large, e.g. > 1 GB).
 * pbsm_bin copies the input's rectangles into row-band order — 256 bands of
 * the strip's tile rows, band-major, from the band counts pbsm_count
 * gathered — as 40-byte records {id, xl, xu, yl, yu} into `band` (n records);
 * pbsm_scatter_banded then scatters from that copy.  Its random record writes
 * stay within one band's slice of the tile lists at a time (an L2-sized
 * window) instead of the whole list.  Same result; needs the pbsm_count of
 * this input with the same n. */
int pbsm_bin(const int64_t* ids, const double* xl, const double* xu, const double* yl,
             const double* yu, int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky,
             int32_t row_lo, int32_t row_hi, void* band, void* stream);
int pbsm_scatter_banded(const void* band, int64_t n, int32_t side, void* ws, int32_t kx,
                        int32_t ky, int32_t row_lo, int32_t row_hi, pbsm_entry* out,
                        int64_t capacity, void* stream);

/* Scratch bytes for one join over n_units work units
 * (n_units = chunks_nested + chunks_sorted + n_items) whose large tiles hold
 * large_entries entries (header.large_r + large_s): the output reservation
 * state plus the large tiles' sort buffers and sorted copies.  The join entry
 * points take `plan`, the host copy of the header read after pbsm_plan. */
int64_t pbsm_join_scratch_bytes(int64_t n_units, int64_t large_entries);

/* sort_segment + sweep_count (_kernels.pyx:188-228, 231-315) for every join
 * tile: the write guard (partition.py:229-233), then the mini-joins over the
 * class combinations (nested / sorted+forward-scan / large, see pbsm_header);
 * the total lands in header.pairs (= JoinReport.result_count). */
int pbsm_join_count(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                    const pbsm_entry* r_list, const pbsm_entry* s_list,
                    const pbsm_header* plan, void* scratch, void* stream);

int pbsm_join_count_eps(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                        const pbsm_entry* r_list, const pbsm_entry* s_list,
                        const pbsm_header* plan, void* scratch, double eps_sq, void* stream);

/* sweep_collect (_kernels.pyx:318-341) + aggregation (engine.py:293-309):
 * the same mini-joins; each work unit counts its pairs (pass 1 over shared
 * memory), reserves its output range, and writes its (r_id, s_id) int64
 * pairs there (pass 2): pairs[2*i], i < header.pairs.  Ranges are reserved
 * with one atomic per unit (ordered = 0: the list is a permutation of the
 * reference's, whose own order is unspecified, engine.py:61-62) or by a
 * decoupled look-back (ordered = 1: deterministic unit-major order, slower).
 * If header.pairs exceeds `capacity`, pairs past it are not written and
 * PBSM_ERR_PAIR_OVERFLOW is set: re-run with capacity >= header.pairs
 * (header.pair_bound always suffices). */
int pbsm_join_emit(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const pbsm_entry* r_list, const pbsm_entry* s_list,
                   const pbsm_header* plan, void* scratch,
                   int64_t* pairs, int64_t capacity, int32_t ordered, void* stream);
int pbsm_join_emit_eps(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                       const pbsm_entry* r_list, const pbsm_entry* s_list,
                       const pbsm_header* plan, void* scratch, int64_t* pairs,
                       int64_t capacity, int32_t ordered, double eps_sq, void* stream);

/* Self-joins (both inputs the same array) may be partitioned once: count side
 * 0 only, copy its per-tile counters over side 1's (both live in the
 * workspace; the shipped host code copies them with a device-to-device copy)
 * before pbsm_plan, scatter side 0 only, and pass the SAME list (and the same
 * compact-entry buffer) for both inputs to the join entry points — the two
 * partitions of the reference (engine.py:231-232) are identical, so the result
 * is too.  The join entry points recognise r_list == s_list and check the
 * write guard against side 0's cursors for both sides. */

/* pbsm_join_emit without the host copy of the plan: the kernels read the
 * unit counts from the device header and the grids are the caller's upper
 * bounds (e.g. the previous join's counts), so the pipeline needs no host
 * sync between pbsm_plan and the emit.  Unordered placement only, and ONE
 * bounded emit per pbsm_plan (the plan zeroes header.pairs; the bounded emit
 * does not reset it).
 * r_capacity / s_capacity are the entries the tile-list buffers hold (the
 * capacities given to pbsm_scatter): if the plan's lists are longer, no unit
 * reads them and PBSM_ERR_SCATTER_OVERFLOW is set; likewise large_capacity
 * (the large entries the scratch was sized for, pbsm_join_scratch_bytes) and
 * max_tile (an upper bound of header.max_huge: sets the sort's merge passes)
 * against the plan's.  After the final
 * pbsm_read_header the caller checks header.chunks_nested <=
 * max_nested_chunks, chunks_sorted + n_items <= max_other_units and the
 * error bits: otherwise some units were not run and the join must be
 * repeated with pbsm_join_emit. */
int pbsm_join_emit_bounded(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                           const pbsm_entry* r_list, int64_t r_capacity,
                           const pbsm_entry* s_list, int64_t s_capacity,
                           int64_t max_nested_chunks, int64_t max_other_units,
                           int64_t large_capacity, int64_t max_tile, void* scratch,
                           int64_t* pairs, int64_t capacity, void* stream);

/* pairs[2i], pairs[2i+1] (row indices, i < n) → r_ids[...], s_ids[...] in
 * place: the pair list of a join whose scatter ran without the id columns. */
int pbsm_map_ids(int64_t* pairs, int64_t n, const int64_t* r_ids, const int64_t* s_ids,
                 void* stream);

/* Row-index pairs (pairs[2i], pairs[2i+1], i < n) → out, grouped by the id
 * chunk of their last-landing id column: group g = min(s_row / chunk_rows,
 * n_groups - 1) (self_join != 0: max(r_row, s_row)), groups laid out in order,
 * order inside a group unspecified.  counts (device int64[2 * n_groups]):
 * [0, n_groups) receives the group sizes, the rest is cursor scratch.
 * 1 <= n_groups <= 32; out must not alias pairs.  Lets a join over host
 * inputs map and copy back each group as soon as its ids have landed (the
 * reference returns the pair list at once, engine.py:293-309; this only
 * changes when the bytes move). */
int pbsm_group_pairs(const int64_t* pairs, int64_t n, int64_t chunk_rows, int32_t n_groups,
                     int32_t self_join, int64_t* out, int64_t* counts, void* stream);

/* SJB1 dataset body (load_mbr_binary, io.py:113-141): n packed 40-byte
 * little-endian records {id u64, x_l, y_l, x_u, y_u f64} at an 8-byte aligned
 * device address → the RectBatch SoA columns (ids reinterpreted as int64,
 * like .astype(np.int64)).  *bad (device u32) = 1 if any record has a lower
 * bound above its upper bound (or a NaN), the check load_mbr_binary raises
 * DatasetError for. */
int pbsm_unpack_records(const void* records, int64_t n, int64_t* ids, double* xl, double* xu,
                        double* yl, double* yu, uint32_t* bad, void* stream);

/* ======================================================================
 * Unit pipeline (the default path of run_join where it applies): the grid's
 * tile rows are cut into UNITS — a tile row × a column range, sized from a
 * per-cell record histogram so every unit holds a few thousand records —
 * and each unit is partitioned AND joined by one CTA while its tile lists
 * are hot in L2:
 *
 *   pbsm_unit_count   count_tiles at cell granularity (cell = tile row ×
 *                     column group) + RectBatch.validate
 *   pbsm_unit_map     the unit map (cells merged greedily into units,
 *                     largest first)
 *   pbsm_unit_bin     every rectangle copied into each unit it overlaps
 *                     (32-byte MBR + its row index), unit-major
 *   pbsm_unit_join    per unit: count_tiles (shared-memory counters),
 *                     compute_segment_offsets, write_tiles into the unit's
 *                     slice of the scratch lists, then the nested mini-joins
 *                     of its small tiles (count -> reserve -> emit); tiles of
 *                     more than LMAX entries are queued and joined after all
 *                     units by the large-tile kernel (sort_segment by x-lower
 *                     + forward scan, _kernels.pyx:188-293)
 *
 * Same results as the tile-list pipeline above; one host sync (the header
 * after pbsm_unit_map) on the first join of a shape, none after that when
 * the caller passes the previous sizes as capacities (overflows are flagged
 * in pbsm_uheader.error and the join is repeated).
 * ====================================================================== */
typedef struct pbsm_uheader {
  int64_t a_r;            /* Σ tiles covered by R rectangles (= A_R)           */
  int64_t a_s;            /* same for S                                         */
  int64_t bin_r;          /* R records binned into live units                   */
  int64_t bin_s;
  int64_t n_units;        /* units with both inputs non-empty                   */
  int64_t max_unit;       /* largest unit (records, R + S)                      */
  int64_t cells;          /* cells of the histogram (rows × column groups)      */
  int64_t group_cols;     /* columns per column group                           */
  uint32_t error;         /* PBSM_ERR_* bits of plan and bin                    */
  uint32_t pad;
  /* join phase (reset by every pbsm_unit_join) */
  int64_t scratch_used;   /* 32-byte scratch slots the units allocated          */
  uint64_t def_packed;    /* deferred tiles << 40 | their work items            */
  int64_t work;           /* large-tile kernel's item ticket                    */
  int64_t pairs;          /* result_count                                       */
  uint32_t jerror;        /* PBSM_ERR_* bits of the join                        */
  uint32_t pad2;
  int64_t nq;             /* chunks heavy units queued for the chunk kernel      */
  int64_t qticket;        /* its ticket                                         */
  int64_t n_def_tiles;    /* tiles deferred to the large-tile kernel           */
  int64_t n_def_items;    /* their work items                                  */
} pbsm_uheader;

/* Whether the unit pipeline supports this grid strip (unit width and cell
 * count limits); 1 = yes, 0 = use the tile-list pipeline. */
int32_t pbsm_unit_supported(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi);
int64_t pbsm_unit_workspace_bytes(int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi);
/* bytes of a bin buffer holding `records` binned records (36 B each) */
int64_t pbsm_unit_bin_bytes(int64_t records);
/* bytes of the join scratch holding `slots` 32-byte list slots (+ row
 * indices and the deferred-tile table) */
int64_t pbsm_unit_scratch_bytes(int64_t slots);
/* Per join: pbsm_unit_init, pbsm_unit_count for R (side 0) and S (side 1) —
 * on two streams if wanted, both after init — then pbsm_unit_map (target =
 * records per unit, <= 0: default; n_r / n_s = the counted inputs' sizes).
 * pbsm_unit_bin of an input must get the same n as its pbsm_unit_count (the
 * bin places each record from the count pass' per-block tallies).
 * Validation errors land in the header like pbsm_count's. */
int pbsm_unit_init(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   void* stream);
int pbsm_unit_count(const double* xl, const double* xu, const double* yl, const double* yu,
                    int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                    int32_t row_hi, void* stream);
int pbsm_unit_map(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                  int64_t n_r, int64_t n_s, int64_t target, void* stream);
/* the unit-major copy of one input (side 0 = R, 1 = S) into `bin`
 * (`capacity` records; PBSM_ERR_SCATTER_OVERFLOW past it). */
int pbsm_unit_bin(const double* xl, const double* xu, const double* yl, const double* yu,
                  int64_t n, int32_t side, void* ws, int32_t kx, int32_t ky, int32_t row_lo,
                  int32_t row_hi, void* bin, int64_t capacity, void* stream);
/* per-unit partition + nested mini-joins, then the deferred large tiles.
 * r_ids / s_ids may be NULL (pairs then hold row indices, pbsm_map_ids).
 * pairs: (capacity, 2) int64; the count lands in pbsm_uheader.pairs. */
int pbsm_unit_join(void* ws, int32_t kx, int32_t ky, int32_t row_lo, int32_t row_hi,
                   const void* bin_r, int64_t bin_r_capacity, const void* bin_s,
                   int64_t bin_s_capacity, const int64_t* r_ids, const int64_t* s_ids,
                   void* scratch, int64_t scratch_slots, int64_t max_units, int64_t* pairs,
                   int64_t capacity, void* stream);
/* Copy the unit header to *out (page-locked: a tiny kernel stores it) and
 * synchronise the stream. */
int pbsm_read_uheader(void* ws, pbsm_uheader* out, void* stream);

/* ======================================================================
 * Multi-GPU plumbing
 * ====================================================================== */

/* Strip routing (the input distribution of a strip-sharded join; the
 * reference is single-process, the step is distributed PBSM's,
 * PAPER.md:492-496): every rectangle of this rank's slice goes to each strip
 * [cuts[g], cuts[g+1]) its tile rows [tile_of(yl), tile_of(yu)] meet
 * (cuts: device int32[world+1], strictly increasing, cuts[0] = 0,
 * cuts[world] = ky).  pbsm_route_count writes the rectangles per destination
 * to dest_counts (device int64[world]); pbsm_route_pack (same n, same
 * scratch, after route_count) then writes them destination-major into
 * `records` (Σ dest_counts packed 40-byte SJB1 records {id, x_l, y_l, x_u,
 * y_u}, io.py:113-141): one send buffer for one all_to_all, unpacked on the
 * receiver by pbsm_unpack_records.  ids may be NULL (row indices). */
int64_t pbsm_route_scratch_bytes(int64_t n, int32_t ky, int32_t world);
int pbsm_route_count(const double* yl, const double* yu, int64_t n, int32_t ky,
                     const int32_t* cuts, int32_t world, void* scratch, int64_t* dest_counts,
                     void* stream);
int pbsm_route_pack(const int64_t* ids, const double* xl, const double* xu, const double* yl,
                    const double* yu, int64_t n, int32_t ky, const int32_t* cuts, int32_t world,
                    void* scratch, void* records, void* stream);

/* Canonical pair order: a stable LSD radix sort of n (r_id, s_id) int64
 * pairs (16-byte aligned) into lexicographic order, in place — the parity form
 * of the reference's unordered pair list (engine.py:61-62, 293-300).
 * pbsm_pair_digits fills hist (device uint32[16*256]) with the histogram of
 * every 8-bit digit (d < 8: byte d of s_id, else byte d-8 of r_id, sign bits
 * flipped); the caller passes as pass_mask the digits that do not hold all
 * n keys in one bucket (the others cannot reorder anything).  tmp: 16*n
 * bytes; scratch: pbsm_sort_pairs_scratch_bytes(n). */
int64_t pbsm_sort_pairs_scratch_bytes(int64_t n);
int pbsm_pair_digits(const int64_t* pairs, int64_t n, uint32_t* hist, void* stream);
int pbsm_sort_pairs(int64_t* pairs, int64_t n, uint32_t pass_mask, void* tmp, void* scratch,
                    void* stream);

/* ======================================================================
 * partition() — the reference's public two-pass partitioning
 * (partition.py:243-263 → PartitionedDataset, partition.py:75-111) for the
 * kx × ky grid (1D stripes: kx × 1 or 1 × ky).  pbsm_partition_count puts
 * the total assignments A (Σ over rectangles of the tiles they overlap,
 * = PartitionedDataset.total_assigned) in *total (device int64);
 * pbsm_partition_write (same n, same scratch; keys / keys_tmp: 16*A bytes,
 * sort_scratch: pbsm_sort_pairs_scratch_bytes(A)) writes the A entries
 * tile-major, rows ascending inside a tile — the reference's order for any
 * writer count m — as SoA columns, and offsets (device int64[kx*ky+1], the
 * CSR array).  ids may be NULL (row indices). */
int64_t pbsm_partition_scratch_bytes(int64_t n, int32_t kx, int32_t ky);
int pbsm_partition_count(const double* xl, const double* xu, const double* yl, const double* yu,
                         int64_t n, int32_t kx, int32_t ky, void* scratch, int64_t* total,
                         void* stream);
int pbsm_partition_write(const int64_t* ids, const double* xl, const double* xu,
                         const double* yl, const double* yu, int64_t n, int32_t kx, int32_t ky,
                         void* scratch, int64_t total, void* keys, void* keys_tmp,
                         void* sort_scratch, int64_t* out_ids, double* out_xl, double* out_xu,
                         double* out_yl, double* out_yu, int64_t* offsets, void* stream);

/* ABI version / build identification */
int32_t pbsm_abi_version(void);
const char* pbsm_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* PBSM_H_ */
