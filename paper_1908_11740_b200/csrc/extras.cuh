// extras.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: SJB1 unpack, header publish, id map, pair groups.
#pragma once

// ---------------------------------------------------------------- input formats
// SJB1 body (io.py:113-141 in the reference): packed little-endian records
// {id u64, x_l f64, y_l f64, x_u f64, y_u f64} (40 bytes) → the SoA columns
// of RectBatch, with load_mbr_binary's check (lower <= upper on both axes;
// NaN fails it) as an error flag.
__global__ void k_unpack_records(const u64* __restrict__ rec, i64 n, i64* __restrict__ ids,
                                 double* __restrict__ xl, double* __restrict__ xu,
                                 double* __restrict__ yl, double* __restrict__ yu,
                                 u32* __restrict__ bad) {
  bool b = false;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const u64* r = rec + 5 * i;
    const double a = __longlong_as_double((long long)__ldcs(r + 1));
    const double c = __longlong_as_double((long long)__ldcs(r + 2));
    const double bb = __longlong_as_double((long long)__ldcs(r + 3));
    const double d = __longlong_as_double((long long)__ldcs(r + 4));
    ids[i] = (i64)__ldcs(r);
    xl[i] = a;
    yl[i] = c;
    xu[i] = bb;
    yu[i] = d;
    b |= !(a <= bb) || !(c <= d);
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1u);
}

// header → page-locked host memory (see pbsm_read_header)
__global__ void k_publish_header(const pbsm_header* __restrict__ hdr, pbsm_header* out) {
  static_assert(sizeof(pbsm_header) % 8 == 0, "header words");
  const int i = threadIdx.x;
  if (i < (int)(sizeof(pbsm_header) / 8))
    reinterpret_cast<volatile u64*>(out)[i] = __ldcg(reinterpret_cast<const u64*>(hdr) + i);
}

// row indices → ids in a pair list (scatter run without the id columns)
__global__ void k_map_ids(i64* __restrict__ pairs, i64 n, const i64* __restrict__ r_ids,
                          const i64* __restrict__ s_ids) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
    reinterpret_cast<longlong2*>(pairs)[i] = make_longlong2(__ldg(r_ids + p.x), __ldg(s_ids + p.y));
  }
}

// ---- pair groups for the staged return of a host-input join (engine.join):
// a row-index pair list is split into groups by the id chunk its LAST-landing
// id column needs (group = s_row / chunk_rows, or max(r_row, s_row) / chunk_rows
// for a self-join, capped at n_groups - 1), so each group can be mapped to ids
// and copied back as soon as its id chunk has crossed PCIe.  Order inside a
// group is arbitrary (the pair list is unordered, engine.py:61-62).
constexpr int kMaxGroups = 32;

__device__ __forceinline__ int pair_group(longlong2 p, i64 chunk_rows, int n_groups, int self) {
  const i64 row = self ? max(p.x, p.y) : p.y;
  return (int)min(row / chunk_rows, (i64)(n_groups - 1));
}

// the contiguous pair range of block b (both passes use the same split)
__device__ __forceinline__ void group_range(i64 n, i64& beg, i64& end) {
  const i64 per = (n + gridDim.x - 1) / gridDim.x;
  beg = min(n, (i64)blockIdx.x * per);
  end = min(n, beg + per);
}

// pass 1: per-group counts (block histogram in shared memory, one global
// atomic per group and block)
__global__ void __launch_bounds__(256) k_group_count(const i64* __restrict__ pairs, i64 n,
                                                     i64 chunk_rows, int n_groups, int self,
                                                     unsigned long long* __restrict__ counts) {
  __shared__ u32 h[kMaxGroups];
  if (threadIdx.x < kMaxGroups) h[threadIdx.x] = 0;
  __syncthreads();
  i64 beg, end;
  group_range(n, beg, end);
  for (i64 i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
    atomicAdd_block(&h[pair_group(p, chunk_rows, n_groups, self)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < n_groups && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], h[threadIdx.x]);
}

// pass 2: each block reserves its run inside every group (one atomic on the
// group cursor), then its threads place the pairs group-major into out
__global__ void __launch_bounds__(256) k_group_place(const i64* __restrict__ pairs, i64 n,
                                                     i64 chunk_rows, int n_groups, int self,
                                                     const unsigned long long* __restrict__ counts,
                                                     unsigned long long* __restrict__ cursors,
                                                     i64* __restrict__ out) {
  __shared__ u32 h[kMaxGroups];
  __shared__ unsigned long long base[kMaxGroups];
  if (threadIdx.x < kMaxGroups) h[threadIdx.x] = 0;
  __syncthreads();
  i64 beg, end;
  group_range(n, beg, end);
  for (i64 i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
    atomicAdd_block(&h[pair_group(p, chunk_rows, n_groups, self)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < n_groups) {
    unsigned long long off = 0;  // the group's start: counts of the groups before it
    for (int g = 0; g < (int)threadIdx.x; ++g) off += counts[g];
    base[threadIdx.x] = h[threadIdx.x] ? off + atomicAdd(&cursors[threadIdx.x], h[threadIdx.x]) : 0;
    h[threadIdx.x] = 0;
  }
  __syncthreads();
  for (i64 i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
    const int g = pair_group(p, chunk_rows, n_groups, self);
    const u32 o = atomicAdd_block(&h[g], 1u);
    reinterpret_cast<longlong2*>(out)[base[g] + o] = p;
  }
}
