// dgswe_diag.cuh -- device diagnostics and initial-condition projection
// (SURVEY.md section 8f, ranks 1 and 3), for the strip-blocked state layout
// of dgswe_kernels.cuh.
//
//   mass_rows_kernel   per-row partial sums of the conserved-mass monitor
//                      sum_elements (M_j c)_0        (diagnostics.py:92-107)
//   l2_rows_kernel     per-row partial sums of the L2 error with a p+2 rule
//                      and the cos(theta) metric      (diagnostics.py:42-80)
//   rows_total_kernel  fixed-order sum of the row partials
//
// Reductions are deterministic (fixed per-thread order, fixed shuffle tree,
// fixed row order) and carried in double-double (TwoSum), so the result is
// the correctly rounded sum of the per-element contributions up to ~1 ulp:
// repeated runs print identical digits, like the reference's sequential
// loop, and agree with it to its own rounding (~n eps relative).
#pragma once

#include <cuda_runtime.h>

#include "dgswe_params.h"

namespace dgswe {

// error-free transformations (no FMA contraction: explicit _rn intrinsics)
struct DD {
    double hi, lo;
};

__device__ __forceinline__ DD two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}

__device__ __forceinline__ DD dd_add(DD x, DD y)
{
    DD s = two_sum(x.hi, y.hi);
    const double e = __dadd_rn(s.lo, __dadd_rn(x.lo, y.lo));
    const double h = __dadd_rn(s.hi, e);
    return {h, __dsub_rn(e, __dsub_rn(h, s.hi))};
}

__device__ __forceinline__ DD dd_add(DD x, double y) { return dd_add(x, DD{y, 0.0}); }

__device__ __forceinline__ DD dd_shfl_xor(DD x, int m)
{
    return {__shfl_xor_sync(0xffffffffu, x.hi, m), __shfl_xor_sync(0xffffffffu, x.lo, m)};
}

// fixed-order block reduction of K double-doubles (blockDim = 256)
template <int K>
__device__ __forceinline__ void block_reduce(DD (&v)[K], DD (*sm)[8])
{
    for (int m = 16; m >= 1; m >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = dd_add(v[k], dd_shfl_xor(v[k], m));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sm[k][w] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            DD t = sm[k][0];
            for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = dd_add(t, sm[k][q]);
            v[k] = t;
        }
    }
}


__device__ __forceinline__ const double *elem_ptr(const double *X, const DiagLayout &L, int z, int j, int v,
                                                  int i)
{
    return X + (size_t)z * L.zstride + (size_t)j * L.rstride + (size_t)v * L.vstride +
           (size_t)(i >> 5) * L.nphi * 32 + (i & 31);
}

// grid (ny, nz), block 256: part[z][j] = sum_i sum_m m0[j][m] c_m  (dd)
__global__ void mass_rows_kernel(const double *__restrict__ X, DiagLayout L, int v,
                                 const double *__restrict__ m0, double *part)
{
    __shared__ DD sm[1][8];
    const int j = blockIdx.x, z = blockIdx.y;
    DD acc[1] = {{0.0, 0.0}};
    const double *mr = m0 + (size_t)j * L.nphi;
    for (int i = threadIdx.x; i < L.nx; i += blockDim.x) {
        const double *c = elem_ptr(X, L, z, j, v, i);
        double cell = 0.0;
        for (int m = 0; m < L.nphi; ++m) cell = fma(mr[m], c[m * 32], cell);
        acc[0] = dd_add(acc[0], cell);
    }
    block_reduce<1>(acc, sm);
    if (threadIdx.x == 0) {
        part[((size_t)z * L.ny + j) * 2] = acc[0].hi;
        part[((size_t)z * L.ny + j) * 2 + 1] = acc[0].lo;
    }
}

// grid (ny, nz), block 256: per row, sum over elements of
//   sum_q wrow[j][q] (u_q - ref_q)^2   and   sum_q wrow[j][q] ref_q^2,
// u_q = sum_m phi2[q][m] c_m at the p+2 Gauss nodes; ref is [ny][nx][nq2]
__global__ void l2_rows_kernel(const double *__restrict__ X, DiagLayout L, int v,
                               const double *__restrict__ phi2, int nq2, const double *__restrict__ wrow,
                               const double *__restrict__ ref, double *part)
{
    __shared__ DD sm[2][8];
    const int j = blockIdx.x, z = blockIdx.y;
    DD acc[2] = {{0.0, 0.0}, {0.0, 0.0}};
    const double *w = wrow + (size_t)j * nq2;
    for (int i = threadIdx.x; i < L.nx; i += blockDim.x) {
        const double *c = elem_ptr(X, L, z, j, v, i);
        const double *r = ref + ((size_t)j * L.nx + i) * nq2;
        double e2 = 0.0, r2 = 0.0;
        for (int q = 0; q < nq2; ++q) {
            double u = 0.0;
            for (int m = 0; m < L.nphi; ++m) u = fma(phi2[q * L.nphi + m], c[m * 32], u);
            const double d = u - r[q];
            e2 = fma(w[q], d * d, e2);
            r2 = fma(w[q], r[q] * r[q], r2);
        }
        acc[0] = dd_add(acc[0], e2);
        acc[1] = dd_add(acc[1], r2);
    }
    block_reduce<2>(acc, sm);
    if (threadIdx.x == 0)
        for (int k = 0; k < 2; ++k) {
            part[(((size_t)z * L.ny + j) * 2 + k) * 2] = acc[k].hi;
            part[(((size_t)z * L.ny + j) * 2 + k) * 2 + 1] = acc[k].lo;
        }
}

// one block of 256: out[k] = sum_j part[z][j][k] (dd, fixed order)
template <int K>
__global__ void rows_total_kernel(const double *__restrict__ part, int ny, int z, double *out)
{
    __shared__ DD sm[K][8];
    DD acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = {0.0, 0.0};
    for (int j = threadIdx.x; j < ny; j += blockDim.x)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double *p = part + (((size_t)z * ny + j) * K + k) * 2;
            acc[k] = dd_add(acc[k], DD{p[0], p[1]});
        }
    block_reduce<K>(acc, sm);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = __dadd_rn(acc[k].hi, acc[k].lo);
}

}  // namespace dgswe
