/*
 * pbsm_oracle.c — CPU restatement of the reference PBSM join path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline ("port" kind) for the B200 implementation; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_1908_11740_b200) never links it.
 *
 * It restates, function by function, the compiled reference backend
 * (/root/reference/pkg/src/sweepjoin/_kernels.pyx) and the engine that drives
 * it (engine.py, partition.py):
 *
 *   tile_of            _kernels.pyx:20-31  (geometry.py:87-106)
 *   count_tiles        _kernels.pyx:34-58
 *   split_slices       partition.py:130-133
 *   compute_segment_offsets partition.py:151-164
 *   write_tiles        _kernels.pyx:61-98 (+ guard partition.py:229-233)
 *   sort_segment       _kernels.pyx:188-228 (stable: ties by original index)
 *   do_sweep           _kernels.pyx:231-293 (Alg. 1 + Eq. 1 reference point)
 *   _dup_params        engine.py:164-179
 *   _pipeline          engine.py:216-309 (m threads; sort tasks, then join
 *                      tasks; per-worker pair lists concatenated)
 *
 * The duplicate-avoidance rule here is the reference's own (Eq. 1), NOT the
 * class scheme of the GPU path, so the oracle is an independent check of the
 * GPU's GBDA reformulation.  Parity is pinned against the reference itself by
 * tests/golden (vectors produced by importing /root/reference's sweepjoin).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "pbsm_oracle.h"

typedef long long i64;

/* _kernels.pyx:20-31 */
long oracle_tile_of(double p, long k) {
  long i = (long)(p * k);
  if (i < 0)
    i = 0;
  else if (i > k - 1)
    i = k - 1;
  while (i > 0 && p < (double)i / (double)k) i -= 1;
  while (i < k - 1 && p >= (double)(i + 1) / (double)k) i += 1;
  return i;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

typedef struct {
  const i64* ids;
  const double *xl, *xu, *yl, *yu;
  i64 n;
} batch_t;

/* tile range of rectangle i: _ranges in _kernels_py.py:25-34 */
static void ranges(const batch_t* b, i64 i, long k, int kind, int axis, long* a0, long* a1,
                   long* r0, long* r1) {
  if (kind == 0) {
    if (axis == 0) {
      *a0 = oracle_tile_of(b->xl[i], k);
      *a1 = oracle_tile_of(b->xu[i], k);
    } else {
      *a0 = oracle_tile_of(b->yl[i], k);
      *a1 = oracle_tile_of(b->yu[i], k);
    }
    *r0 = 0;
    *r1 = 0;
  } else {
    *a0 = oracle_tile_of(b->xl[i], k);
    *a1 = oracle_tile_of(b->xu[i], k);
    *r0 = oracle_tile_of(b->yl[i], k);
    *r1 = oracle_tile_of(b->yu[i], k);
  }
}

/* count_tiles, _kernels.pyx:34-58 */
static void count_tiles(const batch_t* b, long k, int kind, int axis, i64 start, i64 stop,
                        i64* counts) {
  for (i64 i = start; i < stop; ++i) {
    long a0, a1, r0, r1;
    ranges(b, i, k, kind, axis, &a0, &a1, &r0, &r1);
    for (long row = r0; row <= r1; ++row)
      for (long col = a0; col <= a1; ++col) counts[kind == 1 ? row * k + col : col] += 1;
  }
}

int oracle_count_tiles(const double* xl, const double* xu, const double* yl, const double* yu,
                       int64_t n, int32_t kind, int32_t k, int32_t axis, int64_t* counts) {
  batch_t b = {NULL, xl, xu, yl, yu, n};
  if (k < 1) return -1;
  count_tiles(&b, k, kind, axis, 0, n, (i64*)counts);
  return 0;
}

/* partitioned dataset, partition.py:75-111 */
typedef struct {
  i64 n_tiles;
  i64* offsets; /* n_tiles + 1 */
  i64* ids;
  double *xl, *xu, *yl, *yu;
  i64 total;
} pd_t;

/* write_tiles, _kernels.pyx:61-98 */
static void write_tiles(const batch_t* b, long k, int kind, int axis, i64 start, i64 stop,
                        i64* cursors, pd_t* pd) {
  for (i64 i = start; i < stop; ++i) {
    long a0, a1, r0, r1;
    ranges(b, i, k, kind, axis, &a0, &a1, &r0, &r1);
    for (long row = r0; row <= r1; ++row)
      for (long col = a0; col <= a1; ++col) {
        long t = kind == 1 ? row * k + col : col;
        i64 pos = cursors[t]++;
        pd->ids[pos] = b->ids[i];
        pd->xl[pos] = b->xl[i];
        pd->xu[pos] = b->xu[i];
        pd->yl[pos] = b->yl[i];
        pd->yu[pos] = b->yu[i];
      }
  }
}

/* ------------------------------------------------------------------ threads */
typedef struct {
  const batch_t* b;
  long k;
  int kind, axis;
  i64 start, stop;
  i64* counts;  /* count pass */
  i64* cursors; /* write pass */
  pd_t* pd;
} slice_job;

static void* count_job(void* p) {
  slice_job* j = (slice_job*)p;
  count_tiles(j->b, j->k, j->kind, j->axis, j->start, j->stop, j->counts);
  return NULL;
}
static void* write_job(void* p) {
  slice_job* j = (slice_job*)p;
  write_tiles(j->b, j->k, j->kind, j->axis, j->start, j->stop, j->cursors, j->pd);
  return NULL;
}

static void run_jobs(int m, void* (*fn)(void*), void* jobs, size_t stride) {
  if (m == 1) {
    fn(jobs);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * m);
  for (int i = 0; i < m; ++i) pthread_create(&th[i], NULL, fn, (char*)jobs + stride * i);
  for (int i = 0; i < m; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* partition(), partition.py:243-263: split_slices → count → offsets → write */
static int partition(const batch_t* b, long k, int kind, int axis, int m, pd_t* pd) {
  i64 nt = kind == 1 ? (i64)k * k : k;
  if (m > b->n) m = b->n > 0 ? (int)b->n : 1;
  if (m < 1) m = 1;
  slice_job* jobs = (slice_job*)calloc(m, sizeof(slice_job));
  i64* per = (i64*)calloc((size_t)m * nt, sizeof(i64));
  for (int i = 0; i < m; ++i) {
    /* split_slices: np.linspace(0, n, m+1).astype(int64) */
    jobs[i].b = b;
    jobs[i].k = k;
    jobs[i].kind = kind;
    jobs[i].axis = axis;
    jobs[i].start = (i64)((double)b->n * i / m);
    jobs[i].stop = (i64)((double)b->n * (i + 1) / m);
    jobs[i].counts = per + (size_t)i * nt;
    jobs[i].pd = pd;
  }
  jobs[m - 1].stop = b->n;
  run_jobs(m, count_job, jobs, sizeof(slice_job));
  /* compute_segment_offsets, partition.py:151-164 */
  pd->n_tiles = nt;
  pd->offsets = (i64*)calloc(nt + 1, sizeof(i64));
  for (i64 t = 0; t < nt; ++t) {
    i64 tot = 0;
    for (int i = 0; i < m; ++i) tot += per[(size_t)i * nt + t];
    pd->offsets[t + 1] = pd->offsets[t] + tot;
  }
  pd->total = pd->offsets[nt];
  /* segment starts: per[i][t] becomes writer i's cursor */
  for (i64 t = 0; t < nt; ++t) {
    i64 run = pd->offsets[t];
    for (int i = 0; i < m; ++i) {
      i64 c = per[(size_t)i * nt + t];
      per[(size_t)i * nt + t] = run;
      run += c;
    }
  }
  i64 tot = pd->total > 0 ? pd->total : 1;
  pd->ids = (i64*)malloc(sizeof(i64) * tot);
  pd->xl = (double*)malloc(sizeof(double) * tot);
  pd->xu = (double*)malloc(sizeof(double) * tot);
  pd->yl = (double*)malloc(sizeof(double) * tot);
  pd->yu = (double*)malloc(sizeof(double) * tot);
  i64* starts = (i64*)malloc(sizeof(i64) * (size_t)m * nt);
  memcpy(starts, per, sizeof(i64) * (size_t)m * nt);
  for (int i = 0; i < m; ++i) jobs[i].cursors = per + (size_t)i * nt;
  run_jobs(m, write_job, jobs, sizeof(slice_job));
  /* guard, partition.py:229-233: each writer lands on the next writer's start,
   * the last one on the next tile's offset */
  int bad = 0;
  for (i64 t = 0; t < nt && !bad; ++t)
    for (int i = 0; i < m; ++i) {
      i64 expect = i + 1 < m ? starts[(size_t)(i + 1) * nt + t] : pd->offsets[t + 1];
      if (per[(size_t)i * nt + t] != expect) bad = 1;
    }
  free(starts);
  free(per);
  free(jobs);
  return bad ? -2 : 0;
}

static void pd_free(pd_t* pd) {
  free(pd->offsets);
  free(pd->ids);
  free(pd->xl);
  free(pd->xu);
  free(pd->yl);
  free(pd->yu);
  memset(pd, 0, sizeof(*pd));
}

/* ---------------------------------------------------------- sort_segment */
typedef struct {
  double key;
  i64 idx;
} kv_t;

static int kv_cmp(const void* a, const void* b) {
  const kv_t* x = (const kv_t*)a;
  const kv_t* y = (const kv_t*)b;
  if (x->key < y->key) return -1;
  if (x->key > y->key) return 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* _kernels.pyx:188-228: std::sort of (key, original index) pairs, then permute */
static void sort_segment(pd_t* pd, i64 lo, i64 hi, int axis, kv_t* order, double* tmpd,
                         i64* tmpi) {
  i64 n = hi - lo;
  if (n <= 1) return;
  for (i64 i = 0; i < n; ++i) {
    order[i].key = axis == 0 ? pd->xl[lo + i] : pd->yl[lo + i];
    order[i].idx = i;
  }
  qsort(order, n, sizeof(kv_t), kv_cmp);
  for (i64 i = 0; i < n; ++i) tmpi[i] = pd->ids[lo + order[i].idx];
  memcpy(pd->ids + lo, tmpi, n * sizeof(i64));
  double* cols[4] = {pd->xl, pd->xu, pd->yl, pd->yu};
  for (int c = 0; c < 4; ++c) {
    for (i64 i = 0; i < n; ++i) tmpd[i] = cols[c][lo + order[i].idx];
    memcpy(cols[c] + lo, tmpd, n * sizeof(double));
  }
}

/* ------------------------------------------------------------- do_sweep */
typedef struct {
  i64* r;
  i64* s;
  i64 n, cap;
} pairbuf;

static void push(pairbuf* pb, i64 r, i64 s) {
  if (pb->n == pb->cap) {
    pb->cap = pb->cap ? pb->cap * 2 : 1024;
    pb->r = (i64*)realloc(pb->r, sizeof(i64) * pb->cap);
    pb->s = (i64*)realloc(pb->s, sizeof(i64) * pb->cap);
  }
  pb->r[pb->n] = r;
  pb->s[pb->n] = s;
  pb->n++;
}

/* _kernels.pyx:231-293.  Views are (sweep lo, sweep hi, other lo, other hi). */
static i64 do_sweep(const i64* r_ids, const double* r_alo, const double* r_ahi,
                    const double* r_blo, const double* r_bhi, i64 n_r, const i64* s_ids,
                    const double* s_alo, const double* s_ahi, const double* s_blo,
                    const double* s_bhi, i64 n_s, int dup_mode, double t_alo, double t_blo,
                    pairbuf* out) {
  const int test_a = (dup_mode & 1) != 0;
  const int test_b = (dup_mode & 2) != 0;
  i64 count = 0, i = 0, j = 0, kk;
  double hi, lo_a, lo_b, hi_b, m;
  while (i < n_r && j < n_s) {
    if (r_alo[i] < s_alo[j]) {
      hi = r_ahi[i];
      lo_a = r_alo[i];
      lo_b = r_blo[i];
      hi_b = r_bhi[i];
      for (kk = j; kk < n_s && hi >= s_alo[kk]; ++kk) {
        if (lo_b <= s_bhi[kk] && s_blo[kk] <= hi_b) {
          if (test_a) {
            m = lo_a > s_alo[kk] ? lo_a : s_alo[kk];
            if (m < t_alo) continue;
          }
          if (test_b) {
            m = lo_b > s_blo[kk] ? lo_b : s_blo[kk];
            if (m < t_blo) continue;
          }
          count++;
          if (out) push(out, r_ids[i], s_ids[kk]);
        }
      }
      i++;
    } else {
      hi = s_ahi[j];
      lo_a = s_alo[j];
      lo_b = s_blo[j];
      hi_b = s_bhi[j];
      for (kk = i; kk < n_r && hi >= r_alo[kk]; ++kk) {
        if (lo_b <= r_bhi[kk] && r_blo[kk] <= hi_b) {
          if (test_a) {
            m = lo_a > r_alo[kk] ? lo_a : r_alo[kk];
            if (m < t_alo) continue;
          }
          if (test_b) {
            m = lo_b > r_blo[kk] ? lo_b : r_blo[kk];
            if (m < t_blo) continue;
          }
          count++;
          if (out) push(out, r_ids[kk], s_ids[j]);
        }
      }
      j++;
    }
  }
  return count;
}

/* --------------------------------------------------------------- engine */
typedef struct {
  pd_t *pr, *ps;
  long k;
  int kind, part_axis, sweep_axis, collect;
  /* task lists: tiles (sort: tile*2+which), claimed by an atomic cursor */
  i64* sort_tasks;
  i64 n_sort;
  i64* join_tasks;
  i64 n_join;
  i64 next_sort, next_join;
  pthread_mutex_t mu;
  /* per-worker output */
  i64 count;
  pairbuf pairs;
  i64 max_seg;
} eng_t;

typedef struct {
  eng_t* e;
  i64 count;
  pairbuf pairs;
} worker_t;

/* the reference's workers popleft() from a shared deque (engine.py:241-249,
 * 261-265); here an atomic cursor hands out the task list in order */
static i64 claim(eng_t* e, i64* cursor, i64 n) {
  (void)e;
  i64 v = __atomic_fetch_add(cursor, 1, __ATOMIC_RELAXED);
  return v < n ? v : -1;
}

static void* sort_worker(void* p) {
  worker_t* w = (worker_t*)p;
  eng_t* e = w->e;
  i64 cap = e->max_seg > 0 ? e->max_seg : 1;
  kv_t* order = (kv_t*)malloc(sizeof(kv_t) * cap);
  double* tmpd = (double*)malloc(sizeof(double) * cap);
  i64* tmpi = (i64*)malloc(sizeof(i64) * cap);
  for (;;) {
    i64 q = claim(e, &e->next_sort, e->n_sort);
    if (q < 0) break;
    i64 task = e->sort_tasks[q];
    pd_t* pd = (task & 1) ? e->ps : e->pr;
    i64 t = task >> 1;
    sort_segment(pd, pd->offsets[t], pd->offsets[t + 1], e->sweep_axis, order, tmpd, tmpi);
  }
  free(order);
  free(tmpd);
  free(tmpi);
  return NULL;
}

/* _dup_params, engine.py:164-179 */
static void dup_params(const eng_t* e, i64 tile, int* mode, double* t_alo, double* t_blo) {
  long k = e->k;
  if (k == 1) {
    *mode = 0;
    *t_alo = 0.0;
    *t_blo = 0.0;
    return;
  }
  if (e->kind == 0) {
    double lo = (double)tile / (double)k;
    if (e->part_axis == e->sweep_axis) {
      *mode = 1;
      *t_alo = lo;
      *t_blo = 0.0;
    } else {
      *mode = 2;
      *t_alo = 0.0;
      *t_blo = lo;
    }
    return;
  }
  long row = (long)(tile / k), col = (long)(tile % k);
  double x_lo = (double)col / (double)k, y_lo = (double)row / (double)k;
  *mode = 3;
  if (e->sweep_axis == 0) {
    *t_alo = x_lo;
    *t_blo = y_lo;
  } else {
    *t_alo = y_lo;
    *t_blo = x_lo;
  }
}

static void* join_worker(void* p) {
  worker_t* w = (worker_t*)p;
  eng_t* e = w->e;
  for (;;) {
    i64 q = claim(e, &e->next_join, e->n_join);
    if (q < 0) break;
    i64 t = e->join_tasks[q];
    int mode;
    double ta, tb;
    dup_params(e, t, &mode, &ta, &tb);
    pd_t *pr = e->pr, *ps = e->ps;
    i64 lr = pr->offsets[t], hr = pr->offsets[t + 1];
    i64 ls = ps->offsets[t], hs = ps->offsets[t + 1];
    /* _sweep_views, engine.py:182-186 */
    const double *ra, *rA, *rb, *rB, *sa, *sA, *sb, *sB;
    if (e->sweep_axis == 0) {
      ra = pr->xl + lr; rA = pr->xu + lr; rb = pr->yl + lr; rB = pr->yu + lr;
      sa = ps->xl + ls; sA = ps->xu + ls; sb = ps->yl + ls; sB = ps->yu + ls;
    } else {
      ra = pr->yl + lr; rA = pr->yu + lr; rb = pr->xl + lr; rB = pr->xu + lr;
      sa = ps->yl + ls; sA = ps->yu + ls; sb = ps->xl + ls; sB = ps->xu + ls;
    }
    w->count += do_sweep(pr->ids + lr, ra, rA, rb, rB, hr - lr, ps->ids + ls, sa, sA, sb, sB,
                         hs - ls, mode, ta, tb, e->collect ? &w->pairs : NULL);
  }
  return NULL;
}

static void run_workers(int m, void* (*fn)(void*), worker_t* ws) {
  run_jobs(m, fn, ws, sizeof(worker_t));
}

int oracle_join(const int64_t* r_ids, const double* r_xl, const double* r_xu,
                const double* r_yl, const double* r_yu, int64_t n_r, const int64_t* s_ids,
                const double* s_xl, const double* s_xu, const double* s_yl,
                const double* s_yu, int64_t n_s, int32_t kind, int32_t k, int32_t part_axis,
                int32_t sweep_axis, int32_t threads, int32_t collect, oracle_result* out) {
  memset(out, 0, sizeof(*out));
  if (k < 1 || threads < 1 || (kind != 0 && kind != 1)) return -1;
  double t0 = now_s();
  if (n_r == 0 || n_s == 0) {
    out->total_time = now_s() - t0;
    return 0;
  }
  batch_t br = {(const i64*)r_ids, r_xl, r_xu, r_yl, r_yu, n_r};
  batch_t bs = {(const i64*)s_ids, s_xl, s_xu, s_yl, s_yu, n_s};
  pd_t pr, ps;
  memset(&pr, 0, sizeof(pr));
  memset(&ps, 0, sizeof(ps));
  int rc = partition(&br, k, kind, part_axis, threads, &pr);
  if (rc == 0) rc = partition(&bs, k, kind, part_axis, threads, &ps);
  if (rc != 0) {
    pd_free(&pr);
    pd_free(&ps);
    return rc;
  }
  out->a_r = pr.total;
  out->a_s = ps.total;
  double t1 = now_s();
  out->partition_time = t1 - t0;

  eng_t e;
  memset(&e, 0, sizeof(e));
  e.pr = &pr;
  e.ps = &ps;
  e.k = k;
  e.kind = kind;
  e.part_axis = part_axis;
  e.sweep_axis = sweep_axis;
  e.collect = collect;
  pthread_mutex_init(&e.mu, NULL);
  i64 nt = pr.n_tiles;
  e.sort_tasks = (i64*)malloc(sizeof(i64) * 2 * nt);
  e.join_tasks = (i64*)malloc(sizeof(i64) * nt);
  /* build_task_queue, engine.py:84-100 (order does not change the result set) */
  for (i64 t = 0; t < nt; ++t) {
    i64 cr = pr.offsets[t + 1] - pr.offsets[t], cs = ps.offsets[t + 1] - ps.offsets[t];
    if (cr) e.sort_tasks[e.n_sort++] = t * 2;
    if (cs) e.sort_tasks[e.n_sort++] = t * 2 + 1;
    if (cr > e.max_seg) e.max_seg = cr;
    if (cs > e.max_seg) e.max_seg = cs;
    if (cr && cs) e.join_tasks[e.n_join++] = t;
  }
  out->n_join_tasks = e.n_join;
  worker_t* ws = (worker_t*)calloc(threads, sizeof(worker_t));
  for (int i = 0; i < threads; ++i) ws[i].e = &e;
  run_workers(threads, sort_worker, ws);
  double t2 = now_s();
  out->sort_time = t2 - t1;
  run_workers(threads, join_worker, ws);
  double t3 = now_s();
  out->join_time = t3 - t2;
  /* aggregation, engine.py:293-300 */
  i64 total = 0, np_ = 0;
  for (int i = 0; i < threads; ++i) {
    total += ws[i].count;
    np_ += ws[i].pairs.n;
  }
  out->count = total;
  if (collect) {
    out->pairs = (int64_t*)malloc(sizeof(int64_t) * 2 * (np_ > 0 ? np_ : 1));
    i64 o = 0;
    for (int i = 0; i < threads; ++i) {
      for (i64 q = 0; q < ws[i].pairs.n; ++q) {
        out->pairs[2 * o] = ws[i].pairs.r[q];
        out->pairs[2 * o + 1] = ws[i].pairs.s[q];
        ++o;
      }
      free(ws[i].pairs.r);
      free(ws[i].pairs.s);
    }
    out->n_pairs = np_;
  }
  free(ws);
  free(e.sort_tasks);
  free(e.join_tasks);
  pthread_mutex_destroy(&e.mu);
  pd_free(&pr);
  pd_free(&ps);
  out->total_time = now_s() - t0;
  return 0;
}

void oracle_free(oracle_result* r) {
  if (r && r->pairs) {
    free(r->pairs);
    r->pairs = NULL;
  }
}
