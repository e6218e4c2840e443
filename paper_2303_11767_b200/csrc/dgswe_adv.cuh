// dgswe_adv.cuh -- the reference's linear advection model on the doubly
// periodic plane (models.py:114-140, F = beta_x u, G = beta_y u; case
// advection_sine, cases.py:99-110) as one fused stage kernel per RK stage.
//
// A one-variable scalar model outside the shallow-water hot path, so the
// kernel is plain: one thread per element, the state in the reference's
// modal coefficients with layout [nz][ny][nphi][nx] (a warp reads 32
// consecutive elements of one mode), the element's and its four
// neighbours' tiles converted to the Gauss nodes in registers, the nodal
// form of the same operator as the shallow-water kernel (DESIGN.md
// section 3): weak derivatives with the tables of dgswe_params.h NodTab,
// Rusanov faces with alpha = |beta . n| (the model's wavespeed,
// models.py:129-135), the diagonal nodal mass, and
//   Y = a U + b X + g RHS(X)
// with the nodal RHS converted back to modes.  Each face is evaluated by
// both elements from the same operands in the same order (bit-identical).
#pragma once

#include "dgswe_kernels.cuh"

namespace dgswe {


// Rusanov flux of u across a face with normal velocity bn, scaled by the
// face Jacobian: scale (bn (in + out) / 2 - |bn| (out - in) / 2)
__device__ __forceinline__ double adv_flux(double in, double out, double bn, double scale)
{
    return scale * fma(0.5 * bn, in + out, -0.5 * fabs(bn) * (out - in));
}

template <int P>
__global__ void __launch_bounds__(128) adv_stage_kernel(AdvParams ap)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= ap.nx) return;
    const size_t zoff = (size_t)blockIdx.z * ap.zstride;
    // nodal tile of element (ii, jj), periodic in both directions
    auto tile = [&](int ii, int jj, double (&u)[N][N]) {
        ii = (ii + ap.nx) % ap.nx;
        jj = (jj + ap.ny) % ap.ny;
        const double *c = ap.X + zoff + (size_t)jj * NP * ap.nx + ii;
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) u[a][b] = c[(size_t)(a * N + b) * ap.nx];
        to_nodal<P>(u);
    };
    double u[N][N], nb[N][N];
    tile(i, j, u);
    double lt[N], rt[N], bt[N], tt[N], nr[N], nl[N], nt[N], nbt[N];
    xtrace<P, true>(u, lt);
    xtrace<P, false>(u, rt);
    ytrace<P, true>(u, bt);
    ytrace<P, false>(u, tt);
    tile(i - 1, j, nb);
    xtrace<P, false>(nb, nr);        // left neighbour's R trace
    tile(i + 1, j, nb);
    xtrace<P, true>(nb, nl);         // right neighbour's L trace
    tile(i, j - 1, nb);
    ytrace<P, false>(nb, nt);        // lower neighbour's top trace
    tile(i, j + 1, nb);
    ytrace<P, true>(nb, nbt);        // upper neighbour's bottom trace
    // volume: sum_k Dx[i][k] F[k][j] + sum_k dh[j][k] G[i][k]
    double acc[N][N];
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
#pragma unroll
        for (int jj = 0; jj < N; ++jj) {
            double e = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) e = fma(ap.cx * c_nod[P].dh[ii][k], ap.bx * u[k][jj], e);
#pragma unroll
            for (int k = 0; k < N; ++k) e = fma(c_nod[P].dh[jj][k], ap.cy * ap.by * u[ii][k], e);
            acc[ii][jj] = e;
        }
    // faces (lower / left element = "in"), lifted along xi / eta with mu
#pragma unroll
    for (int q = 0; q < N; ++q) {
        const double fl = adv_flux(nr[q], lt[q], ap.bx, ap.bdy);
        const double fr = adv_flux(rt[q], nl[q], ap.bx, ap.bdy);
        const double fb = adv_flux(nt[q], bt[q], ap.by, ap.bdx);
        const double ft = adv_flux(tt[q], nbt[q], ap.by, ap.bdx);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            acc[k][q] = fma(c_nod[P].mu[k], fl, fma(-c_nod[P].mu[N - 1 - k], fr, acc[k][q]));
            acc[q][k] = fma(c_nod[P].mu[k], fb, fma(-c_nod[P].mu[N - 1 - k], ft, acc[q][k]));
        }
    }
    // RHS at the nodes (diagonal mass), back to modes, stage combination
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
#pragma unroll
        for (int jj = 0; jj < N; ++jj) acc[ii][jj] *= ap.inv_determ;
    to_modal<P>(acc);
    const double *xm = ap.X + zoff + (size_t)j * NP * ap.nx + i;
    const double *um = ap.U ? ap.U + zoff + (size_t)j * NP * ap.nx + i : nullptr;
    double *ym = ap.Y + zoff + (size_t)j * NP * ap.nx + i;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) {
            const size_t o = (size_t)(a * N + b) * ap.nx;
            double y = fma(ap.b, xm[o], ap.g * acc[a][b]);
            if (um) y = fma(ap.a, um[o], y);
            ym[o] = y;
        }
}

}  // namespace dgswe
