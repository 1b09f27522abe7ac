// extras.cuh — part of pbsm.cu (one translation unit: included inside its
// anonymous namespace, after the types and includes at its top).
// Contents: epsilon refinement, SJB1 unpack, id map.
#pragma once

// ---------------------------------------------------------------- ε refinement
// _refine_pairs (engine.py:201-206): keep a candidate (row i of P, row j of Q)
// iff dx*dx + dy*dy <= eps^2 with every operation rounded on its own (numpy
// semantics: no FMA contraction), then map row indices to ids (:298-300).
__device__ __forceinline__ bool within_eps(const i64* __restrict__ cand, i64 i,
                                           const double* __restrict__ px,
                                           const double* __restrict__ py,
                                           const double* __restrict__ qx,
                                           const double* __restrict__ qy, double eps_sq) {
  const i64 a = cand[2 * i], b = cand[2 * i + 1];
  const double dx = __dsub_rn(px[a], qx[b]);
  const double dy = __dsub_rn(py[a], qy[b]);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= eps_sq;
}

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

__global__ void k_refine_flag(const i64* __restrict__ cand, i64 n, const double* __restrict__ px,
                              const double* __restrict__ py, const double* __restrict__ qx,
                              const double* __restrict__ qy, double eps_sq,
                              u32* __restrict__ flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    flag[i] = within_eps(cand, i, px, py, qx, qy, eps_sq) ? 1u : 0u;
}

__global__ void k_refine_compact(const i64* __restrict__ cand, i64 n,
                                 const u32* __restrict__ flag, const u64* __restrict__ base,
                                 const i64* __restrict__ p_ids, const i64* __restrict__ q_ids,
                                 i64* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    if (flag[i]) {
      const u64 o = base[i];
      out[2 * o] = p_ids[cand[2 * i]];
      out[2 * o + 1] = q_ids[cand[2 * i + 1]];
    }
  }
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
