/* pbsm_oracle.h — CPU parity oracle / baseline (TEST INFRASTRUCTURE ONLY).
 * See pbsm_oracle.c for the reference file:line each function restates. */
#ifndef PBSM_ORACLE_H_
#define PBSM_ORACLE_H_
#include <stdint.h>

typedef struct oracle_result {
  int64_t count;      /* JoinReport.result_count */
  int64_t* pairs;     /* n_pairs × (r_id, s_id), unordered (engine.py:61-62) */
  int64_t n_pairs;
  int64_t a_r, a_s;   /* PartitionedDataset.total_assigned of R and S */
  int64_t n_join_tasks;
  double partition_time, sort_time, join_time, total_time;
} oracle_result;

long oracle_tile_of(double p, long k);
int oracle_count_tiles(const double* xl, const double* xu, const double* yl, const double* yu,
                       int64_t n, int32_t kind, int32_t k, int32_t axis, int64_t* counts);
int oracle_join(const int64_t* r_ids, const double* r_xl, const double* r_xu,
                const double* r_yl, const double* r_yu, int64_t n_r, const int64_t* s_ids,
                const double* s_xl, const double* s_xu, const double* s_yl,
                const double* s_yu, int64_t n_s, int32_t kind, int32_t k, int32_t part_axis,
                int32_t sweep_axis, int32_t threads, int32_t collect, oracle_result* out);
void oracle_free(oracle_result* r);

#endif
