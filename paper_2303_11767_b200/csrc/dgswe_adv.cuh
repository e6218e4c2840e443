// dgswe_adv.cuh -- the reference's linear advection model on the doubly
// periodic plane (models.py:114-140, F = beta_x u, G = beta_y u; case
// advection_sine, cases.py:99-110) as one fused stage kernel per RK stage.
//
// A one-variable scalar model outside the shallow-water hot path, so the
// kernel is plain: one thread per element, the state in the reference's
// modal coefficients with layout [nz][ny][nphi][nx] (a warp reads 32
// consecutive elements of one mode).  Face traces come straight from the
// modes (Legendre P_a(+-1) = (+-1)^a: a signed sum over one index, then the
// Gauss-node values of the other, the same formula for an element's own
// trace and for its neighbour's, so both sides of a face use identical
// operands and the face flux is bit-identical); each neighbour is streamed
// through two N-vectors instead of a converted tile, which keeps p <= 5
// free of spills.  Then the nodal form of the same operator as the
// shallow-water kernel: Rusanov faces with
// alpha = |beta . n| (the model's wavespeed, models.py:129-135) lifted with
// mu, weak derivatives with the tables of dgswe_params.h NodTab, the
// diagonal nodal mass, and
//   Y = a U + b X + g RHS(X)
// with the nodal RHS converted back to modes.
#pragma once

#include "dgswe_kernels.cuh"

namespace dgswe {


// Rusanov flux of u across a face with normal velocity bn and
// stabilisation alpha (|bn|, or a pinned global value), scaled by the face
// Jacobian: scale (bn (in + out) / 2 - alpha (out - in) / 2)
__device__ __forceinline__ double adv_flux(double in, double out, double bn, double alpha, double scale)
{
    return scale * fma(0.5 * bn, in + out, -0.5 * alpha * (out - in));
}

// trace of element (ii, jj) at the Gauss nodes of one side, from its
// modes c[a][b] (a: x degree, b: y degree): X side (xi = SGN) or Y side
template <int P, bool XSIDE, int SGN>
__device__ __forceinline__ void adv_trace(const double *c, long long mstride, double (&tr)[P + 1])
{
    constexpr int N = P + 1;
    double s[N];
#pragma unroll
    for (int o = 0; o < N; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int a = XSIDE ? k : o, b = XSIDE ? o : k;
            const double v = c[(size_t)(a * N + b) * mstride];
            acc = (SGN < 0 && (k & 1)) ? acc - v : acc + v;
        }
        s[o] = acc;
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        double t = 0.0;
#pragma unroll
        for (int o = 0; o < N; ++o) t = fma(c_nod[P].leg[o][q], s[o], t);
        tr[q] = t;
    }
}

template <int P>
__global__ void __launch_bounds__(128) adv_elem_kernel(AdvParams ap)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= ap.nx) return;
    const size_t zoff = (size_t)blockIdx.z * ap.zstride;
    const long long ms = ap.nx;                                  // mode stride
    auto elem = [&](int ii, int jj) {                            // periodic in both directions
        ii = ii < 0 ? ii + ap.nx : (ii >= ap.nx ? ii - ap.nx : ii);
        jj = jj < 0 ? jj + ap.ny : (jj >= ap.ny ? jj - ap.ny : jj);
        return ap.X + zoff + (size_t)jj * NP * ap.nx + ii;
    };
    const double *self = elem(i, j);
    // the four face fluxes (lower / left element = "in"), scaled by the face Jacobian
    double fl[N], fr[N], fb[N], ft[N];
    {
        double own[N], nb[N];
        adv_trace<P, true, -1>(self, ms, own);
        adv_trace<P, true, 1>(elem(i - 1, j), ms, nb);
#pragma unroll
        for (int q = 0; q < N; ++q) fl[q] = adv_flux(nb[q], own[q], ap.bx, ap.ax, ap.bdy);
        adv_trace<P, true, 1>(self, ms, own);
        adv_trace<P, true, -1>(elem(i + 1, j), ms, nb);
#pragma unroll
        for (int q = 0; q < N; ++q) fr[q] = adv_flux(own[q], nb[q], ap.bx, ap.ax, ap.bdy);
        adv_trace<P, false, -1>(self, ms, own);
        adv_trace<P, false, 1>(elem(i, j - 1), ms, nb);
#pragma unroll
        for (int q = 0; q < N; ++q) fb[q] = adv_flux(nb[q], own[q], ap.by, ap.ay, ap.bdx);
        adv_trace<P, false, 1>(self, ms, own);
        adv_trace<P, false, -1>(elem(i, j + 1), ms, nb);
#pragma unroll
        for (int q = 0; q < N; ++q) ft[q] = adv_flux(own[q], nb[q], ap.by, ap.ay, ap.bdx);
    }
    // lifts (x faces along xi, y faces along eta), then the volume:
    // sum_k Dx[ii][k] F[k][jj] + sum_k dh[jj][k] G[ii][k]
    double acc[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b)
            acc[a][b] = fma(c_nod[P].mu[a], fl[b], -c_nod[P].mu[N - 1 - a] * fr[b]) +
                        fma(c_nod[P].mu[b], fb[a], -c_nod[P].mu[N - 1 - b] * ft[a]);
    {
        double u[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) u[a][b] = self[(size_t)(a * N + b) * ms];
        to_nodal<P>(u);
#pragma unroll
        for (int ii = 0; ii < N; ++ii)
#pragma unroll
            for (int jj = 0; jj < N; ++jj) {
                double e = acc[ii][jj];
#pragma unroll
                for (int k = 0; k < N; ++k) e = fma(ap.cx * c_nod[P].dh[ii][k], ap.bx * u[k][jj], e);
#pragma unroll
                for (int k = 0; k < N; ++k) e = fma(c_nod[P].dh[jj][k], ap.cy * ap.by * u[ii][k], e);
                acc[ii][jj] = e;
            }
    }
    // RHS at the nodes (diagonal mass), back to modes, stage combination
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
#pragma unroll
        for (int jj = 0; jj < N; ++jj) acc[ii][jj] *= ap.inv_determ;
    to_modal<P>(acc);
    const double *um = ap.U ? ap.U + zoff + (size_t)j * NP * ap.nx + i : nullptr;
    double *ym = ap.Y + zoff + (size_t)j * NP * ap.nx + i;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) {
            const size_t o = (size_t)(a * N + b) * ms;
            double y = fma(ap.b, self[o], ap.g * acc[a][b]);
            if (um) y = fma(ap.a, um[o], y);
            ym[o] = y;
        }
}


// trace of a mode tile held in registers (the formula of adv_trace)
template <int P, bool XSIDE, int SGN>
__device__ __forceinline__ void adv_trace_r(const double (&c)[P + 1][P + 1], double (&tr)[P + 1])
{
    constexpr int N = P + 1;
    double s[N];
#pragma unroll
    for (int o = 0; o < N; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const double v = XSIDE ? c[k][o] : c[o][k];
            acc = (SGN < 0 && (k & 1)) ? acc - v : acc + v;
        }
        s[o] = acc;
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        double t = 0.0;
#pragma unroll
        for (int o = 0; o < N; ++o) t = fma(c_nod[P].leg[o][q], s[o], t);
        tr[q] = t;
    }
}

constexpr int kAdvOwn = kLanes - 2;   // elements a warp owns (lanes 1..30; 0 / 31: neighbours)
__host__ __device__ constexpr int adv_segments(int nx) { return (nx + kAdvOwn - 1) / kAdvOwn; }
// the row-marching kernel serves p <= 2 (4096^2, p = 2: 0.45 of the HBM
// roofline against 0.41 for the thread-per-element kernel; p = 3: 0.32
// against 0.34 -- the next row's 16 modes per variable loaded and consumed
// in one iteration; p = 4 spilled)
template <int P>
__host__ __device__ constexpr bool adv_marching() { return P <= 2; }

// Row-marching form (p <= 2): warp w of a CTA owns a 30-element segment
// (lanes 1..30; lanes 0 and 31 hold the periodic x-neighbours) and marches
// north through ap.rc rows: the x-face between lanes l and l+1 is evaluated
// once by lane l (operands of lane l+1 by shuffle), the y-face above a row
// once and carried up as the next row's bottom face; each trace is formed
// by its own element with the same formula as adv_trace, so a face is the
// same bits whichever CTA evaluates it.  The next row's modes are loaded at
// the top of the iteration and consumed at its end (the top face).
template <int P>
__global__ void __launch_bounds__(128) adv_stage_kernel(AdvParams ap)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    const int lane = threadIdx.x & 31;
    const int seg = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int nx = ap.nx, ny = ap.ny;
    if (seg >= adv_segments(nx)) return;
    const int first = seg * kAdvOwn;
    const int nvalid = min(kAdvOwn, nx - first);
    const bool owned = lane >= 1 && lane <= nvalid;
    int g = first - 1 + min(lane, nvalid + 1);
    g = g < 0 ? g + nx : (g >= nx ? g - nx : g);
    const int jb = blockIdx.y * ap.rc;
    const int je = min(jb + ap.rc, ny);
    if (jb >= je) return;
    const size_t zoff = (size_t)blockIdx.z * ap.zstride;
    const long long ms = nx;
    auto row_ptr = [&](const double *base, int r) {
        r = r < 0 ? r + ny : (r >= ny ? r - ny : r);
        return base + zoff + (size_t)r * NP * nx + g;
    };
    auto load = [&](int r, double (&c)[N][N]) {
        const double *b = row_ptr(ap.X, r);
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int k = 0; k < N; ++k) c[a][k] = b[(size_t)(a * N + k) * ms];
    };
    double cur[N][N], nxt[N][N];
    load(jb, cur);
    double fb[N];
    {
        double tT[N], tB[N];
        load(jb - 1, nxt);
        adv_trace_r<P, false, 1>(nxt, tT);
        adv_trace_r<P, false, -1>(cur, tB);
#pragma unroll
        for (int q = 0; q < N; ++q) fb[q] = adv_flux(tT[q], tB[q], ap.by, ap.ay, ap.bdx);
    }
    for (int j = jb; j < je; ++j) {
        load(j + 1, nxt);
        // x-faces
        double fr[N], fl[N];
        {
            double tR[N], tL[N];
            adv_trace_r<P, true, 1>(cur, tR);
            adv_trace_r<P, true, -1>(cur, tL);
#pragma unroll
            for (int q = 0; q < N; ++q) fr[q] = adv_flux(tR[q], __shfl_down_sync(0xffffffffu, tL[q], 1), ap.bx, ap.ax, ap.bdy);
#pragma unroll
            for (int q = 0; q < N; ++q) fl[q] = __shfl_up_sync(0xffffffffu, fr[q], 1);
        }
        double tT[N];
        adv_trace_r<P, false, 1>(cur, tT);
        // lifts of the left, right and bottom faces
        double acc[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b)
                acc[a][b] = fma(c_nod[P].mu[a], fl[b], fma(-c_nod[P].mu[N - 1 - a], fr[b], c_nod[P].mu[b] * fb[a]));
        // volume on the nodal tile (cur is converted in place; its modes are
        // re-read for the stage combination)
        to_nodal<P>(cur);
#pragma unroll
        for (int ii = 0; ii < N; ++ii)
#pragma unroll
            for (int jj = 0; jj < N; ++jj) {
                double e = acc[ii][jj];
#pragma unroll
                for (int k = 0; k < N; ++k) e = fma(ap.cx * c_nod[P].dh[ii][k], ap.bx * cur[k][jj], e);
#pragma unroll
                for (int k = 0; k < N; ++k) e = fma(c_nod[P].dh[jj][k], ap.cy * ap.by * cur[ii][k], e);
                acc[ii][jj] = e;
            }
        // the top face (row j+1's bottom trace), lifted; carried up
        {
            double tB[N];
            adv_trace_r<P, false, -1>(nxt, tB);
#pragma unroll
            for (int q = 0; q < N; ++q) fb[q] = adv_flux(tT[q], tB[q], ap.by, ap.ay, ap.bdx);
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) acc[a][b] = fma(-c_nod[P].mu[N - 1 - b], fb[a], acc[a][b]);
        }
#pragma unroll
        for (int ii = 0; ii < N; ++ii)
#pragma unroll
            for (int jj = 0; jj < N; ++jj) acc[ii][jj] *= ap.inv_determ;
        to_modal<P>(acc);
        if (owned) {
            const double *xm = row_ptr(ap.X, j);
            const double *um = ap.U ? row_ptr(ap.U, j) : nullptr;
            double *ym = ap.Y + zoff + (size_t)j * NP * nx + g;
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    const size_t o = (size_t)(a * N + b) * ms;
                    double y = fma(ap.b, xm[o], ap.g * acc[a][b]);
                    if (um) y = fma(ap.a, um[o], y);
                    ym[o] = y;
                }
        }
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) cur[a][b] = nxt[a][b];
    }
}

}  // namespace dgswe
