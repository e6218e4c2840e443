// dgswe_kernels.cuh -- fused fp64 DG shallow-water stage kernel for sm_100a.
//
// One CTA = 4 warps x 32 lanes: warp v < 3 owns variable v in {h, hu, hv};
// warp 0 (lightest physics) also evaluates the row's x-face fluxes and
// warp 3 (the face warp) the bottom traces of the row above and the y-face.
// Lane l holds longitude element i0-1+l (mod nx) of a 30-element strip:
// lanes 1..30 own their element, lanes 0 and 31 are the periodic/strip halo
// whose traces feed the strip's two border faces.  The CTA marches north
// through a chunk of latitude rows; every y-face is evaluated once per
// chunk, every x-face once per strip.
//
// Memory pipeline: each lane streams its own element's coefficients with
// cp.async (LDGSTS) into a two-row shared-memory ring, two rows ahead of
// use, and the u^n tile of the current row one phase ahead; every lane
// reads back only the words it copied, so no CTA barrier guards the ring.
//
// Per row, per variable and lane (n = p+1, all tensor contractions
// sum-factorised; constant tables in __constant__):
//   1. modal -> nodal: t[a][qj] = sum_b c[a][b] P_b(x_qj),
//      U[qi][qj] = sum_a P_a(x_qi) t[a][qj]; traces L/R from t, T/B from
//      sum_b c[a][b](+-1)^b                          (dg.py:348-357)
//   2. nodal values exchanged through shared memory; pointwise flux /
//      source physics for this warp's variable      (models.py:161-252)
//   3. face warps: Rusanov flux with local alpha    (dg.py:92-119,385-453)
//   4. volume + source projection streamed over qi, boundary lifts,
//      per-row inverse mass (Kronecker block form), fused RK stage update
//      (dg.py:455-502, timestep.py:132-167)
//
// Floating point: FMA contraction and a Newton-refined reciprocal are used;
// results agree with the reference's exact-order oracle to ~1e-15 relative
// per step (tests/test_gpu_parity.py).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgswe {

constexpr int kMaxP = 6;
constexpr int kLanes = 32;
constexpr int kOwned = 30;   // owned elements per strip (lanes 1..30)
constexpr int kVarWarps = 3; // one per conserved variable
constexpr int kWarps = 4;    // + one face warp (Rusanov fluxes)
constexpr int kThreads = kWarps * kLanes;

// [p][table][a][q]: 0 P_a(x_q), 1 P'_a(x_q), 2 w_q P_a(x_q), 3 w_q P'_a(x_q)
__constant__ double c_tab[kMaxP + 1][4][kMaxP + 1][kMaxP + 1];

struct StageParams {
    const double *X;      // stage input (level 0, buffer row 0)
    const double *U;      // u^n for the combination (may be null when a == 0)
    double *Y;            // output
    long long zstride;    // doubles per level
    long long rstride;    // doubles per buffer row (3 * nphi * nx)
    int nx, ny, row0, nrows;
    int j_begin, j_end, rc;   // local rows [j_begin, j_end), rc rows per CTA
    double a, b, g;       // Y = a U + b X + g RHS(X)
    const double *rowtab; // per global row, see RowLayout
    double inv_r;         // 1/R
    double inv_r_cx;      // (1/R) * determ/bd_det_x
    double gravity, half_g, h_floor, sqrt_g;
    double bdx, bdy;      // bd_det_x, bd_det_y
    int alpha_mode;       // 0 local, 1 pinned, 2 global (from alpha_dev)
    double alpha;
    const double *alpha_dev;
    unsigned *status;
    int *first_tag;
    int tag;
    int check_finite;
    int check_mean;
};

// per-row table layout (doubles): crc[n] srs[n] fcs[n] cr_b cos_b T[n][n]
template <int P>
struct RowLayout {
    static constexpr int N = P + 1;
    static constexpr int CRC = 0;
    static constexpr int SRS = N;
    static constexpr int FCS = 2 * N;
    static constexpr int CRB = 3 * N;
    static constexpr int COSB = 3 * N + 1;
    static constexpr int T = 3 * N + 2;
    static constexpr int STRIDE = 3 * N + 2 + N * N;
};

__host__ __device__ inline int row_stride(int p) { return 3 * (p + 1) + 2 + (p + 1) * (p + 1); }

#define LEG(a, q) c_tab[P][0][a][q]
#define WP(a, q) c_tab[P][2][a][q]
#define WD(a, q) c_tab[P][3][a][q]

// Gauss nodes are exactly antisymmetric (numpy's leggauss symmetrises them)
// and the Legendre recurrences are odd/even in x, so the tables satisfy
//   T(a, N-1-q) = (-1)^(a + PAR) T(a, q)   exactly,
// PAR = 0 for P and wP, 1 for P' and wP'.  Every 1-D contraction below
// uses this even/odd split: N adds + N*ceil(N/2) FMA instead of N*N.
// DG_ABL: timing ablations for experiments only (results are wrong):
// 1 no y-face, 2 no x-face, 4 no u^n loads, 8 no hu/hv volume, 16 no eval, 32 no finalize math
#ifndef DG_ABL
#define DG_ABL 0
#endif
#ifndef DG_MINB
#define DG_MINB 4   // resident CTAs per SM the p <= 3 build is register-capped for
#endif
#ifndef DG_VOL_COMPACT
#define DG_VOL_COMPACT 0
#endif
#ifndef DG_FOLD_CX
#define DG_FOLD_CX 1
#endif
#ifndef DG_PF_SPREAD
#define DG_PF_SPREAD 0
#endif
#if DG_FOLD_CX
#define CXF kp.inv_r_cx
#define CXN 1.0
#else
#define CXF 1.0
#define CXN kp.inv_r_cx
#endif

// DG_TIMING builds record per-role phase durations (clock cycles) of every
// row: [role][A work, barrier-1 wait, B work, barrier-2 wait, C work, rows]
#ifdef DG_TIMING
__device__ unsigned long long g_timing[4][6];
#define TSTAMP(k) unsigned tk##k = clock()
#define TACC(i, d) tacc[i] += (d)
#else
#define TSTAMP(k)
#define TACC(i, d)
#endif

template <int TAB>
struct TabPar {
    static constexpr int v = (TAB == 1 || TAB == 3) ? 1 : 0;
};

// sum over a = S, S+2, ... < N of T(a, q) in[a]
template <int P, int TAB, int S>
__device__ __forceinline__ double dot_step2(const double (&in)[P + 1], int q)
{
    double acc = c_tab[P][TAB][S][q] * in[S];
#pragma unroll
    for (int a = S + 2; a < P + 1; a += 2) acc = fma(c_tab[P][TAB][a][q], in[a], acc);
    return acc;
}

// modes -> nodes: out[q] = sum_a T(a, q) in[a]
template <int P, int TAB>
__device__ __forceinline__ void m2n(const double (&in)[P + 1], double (&out)[P + 1])
{
    constexpr int N = P + 1, H = N / 2, PAR = TabPar<TAB>::v;
#pragma unroll
    for (int q = 0; q < H; ++q) {
        const double e = dot_step2<P, TAB, 0>(in, q);
        const double o = dot_step2<P, TAB, 1>(in, q);
        out[q] = e + o;
        out[N - 1 - q] = PAR == 0 ? e - o : o - e;
    }
    if constexpr (N & 1) {   // middle node x = 0: only (a + PAR) even survives
        if constexpr (PAR == 0)
            out[H] = dot_step2<P, TAB, 0>(in, H);
        else if constexpr (N > 1)
            out[H] = dot_step2<P, TAB, 1>(in, H);
        else
            out[H] = 0.0;
    }
}

// node-pair folds of a nodal line: ip[q] = x[q] + x[N-1-q], im[q] = x[q] - x[N-1-q]
template <int P>
__device__ __forceinline__ void fold(const double (&x)[P + 1], double (&ip)[(P + 1) / 2],
                                     double (&im)[(P + 1) / 2])
{
    constexpr int N = P + 1;
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
        ip[q] = x[q] + x[N - 1 - q];
        im[q] = x[q] - x[N - 1 - q];
    }
}

// nodes -> modes: out[b] = sum_q T(b, q) x[q], from the folds of x
template <int P, int TAB>
__device__ __forceinline__ double n2m_one(const double *ip, const double *im, const double (&x)[P + 1],
                                          int b)
{
    constexpr int N = P + 1, H = N / 2, PAR = TabPar<TAB>::v;
    const bool sym = ((b + PAR) & 1) == 0;
    double acc = 0.0;
    if constexpr (H > 0) {
        acc = c_tab[P][TAB][b][0] * (sym ? ip[0] : im[0]);
#pragma unroll
        for (int q = 1; q < H; ++q) acc = fma(c_tab[P][TAB][b][q], sym ? ip[q] : im[q], acc);
        if constexpr (N & 1)
            if (sym) acc = fma(c_tab[P][TAB][b][H], x[H], acc);
    } else {
        if (sym) acc = c_tab[P][TAB][b][0] * x[0];
    }
    return acc;
}

template <int P, int TAB>
__device__ __forceinline__ void n2m(const double (&x)[P + 1], double (&out)[P + 1])
{
    constexpr int N = P + 1, H = N / 2;
    double ip[H > 0 ? H : 1], im[H > 0 ? H : 1];
    if constexpr (H > 0) fold<P>(x, ip, im);
#pragma unroll
    for (int b = 0; b < N; ++b) out[b] = n2m_one<P, TAB>(ip, im, x, b);
}

// out[b] = sum_q TA(b, q) x[q] + TB(b, q) y[q] in one accumulation chain
template <int P, int TA, int TB>
__device__ __forceinline__ void n2m2(const double (&x)[P + 1], const double (&y)[P + 1],
                                     double (&out)[P + 1])
{
    constexpr int N = P + 1, H = N / 2;
    double xp[H > 0 ? H : 1], xm[H > 0 ? H : 1], yp[H > 0 ? H : 1], ym[H > 0 ? H : 1];
    if constexpr (H > 0) {
        fold<P>(x, xp, xm);
        fold<P>(y, yp, ym);
    }
#pragma unroll
    for (int b = 0; b < N; ++b) {
        const bool sx = ((b + TabPar<TA>::v) & 1) == 0, sy = ((b + TabPar<TB>::v) & 1) == 0;
        double acc = 0.0;
        bool first = true;
#pragma unroll
        for (int q = 0; q < H; ++q) {
            acc = first ? c_tab[P][TA][b][q] * (sx ? xp[q] : xm[q])
                        : fma(c_tab[P][TA][b][q], sx ? xp[q] : xm[q], acc);
            first = false;
            acc = fma(c_tab[P][TB][b][q], sy ? yp[q] : ym[q], acc);
        }
        if constexpr (N & 1) {
            if (sx) {
                acc = first ? c_tab[P][TA][b][H] * x[H] : fma(c_tab[P][TA][b][H], x[H], acc);
                first = false;
            }
            if (sy) acc = first ? c_tab[P][TB][b][H] * y[H] : fma(c_tab[P][TB][b][H], y[H], acc);
        }
        out[b] = acc;
    }
}

template <int P>
struct Smem {
    static constexpr int N = P + 1;
    static constexpr int NP = N * N;
    static constexpr int TILE = 3 * NP * kLanes;         // one row of coefficients, all vars
    static constexpr int TR = 3 * N * kLanes;            // one trace / face-flux set
    // offsets in doubles
    static constexpr int XR0 = 0;                        // coefficient ring slot 0
    static constexpr int XR1 = XR0 + TILE;               // slot 1
    static constexpr int U = XR1 + TILE;                 // nodal values [3][NP][32]
    static constexpr int XL = U + TILE;                  // [3][N][32]
    static constexpr int XRT = XL + TR;
    static constexpr int TT = XRT + TR;                  // top traces of current row
    static constexpr int FX = TT + TR;                   // x-face flux, right face of lane
    static constexpr int FY0 = FX + TR;                  // y-face flux buffers
    static constexpr int FY1 = FY0 + TR;
    static constexpr int ROW = FY1 + TR;                 // row-table ring, 3 rows
    static constexpr int TOTAL = ROW + 3 * RowLayout<P>::STRIDE;
};

__device__ __forceinline__ double sgn(int k) { return (k & 1) ? -1.0 : 1.0; }

// max(x, y) for y > 0 on the integer pipe: the signed 64-bit order of the
// bit patterns equals the floating-point order for non-negative values and
// puts every negative x below y (fp64 fmax is a DSETP + select sequence,
// ~25 cycles of dependent latency on sm_100)
__device__ __forceinline__ double max_pos(double x, double y)
{
    const long long xb = __double_as_longlong(x), yb = __double_as_longlong(y);
    return __longlong_as_double(xb > yb ? xb : yb);
}

// max of two non-negative values (same integer trick)
__device__ __forceinline__ double max_nn(double x, double y) { return max_pos(x, y); }

// 1/x: MUFU seed (~2^-22) + one cubic correction r (1 + e + e^2), e = 1 - x r
// (error ~e^3, i.e. <= 1 ulp for normal x)
__device__ __forceinline__ double rcp64(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// 1/sqrt(x): MUFU seed + one cubic correction y (1 + e/2 + 3e^2/8),
// e = 1 - x y^2 (x > 0, normal)
__device__ __forceinline__ double rsqrt64(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y, e * fma(e, 0.375, 0.5), y);
}

// 1/hf and sqrt(g hf) with hf = max(h, floor) from one rsqrt; equals the
// reference's sqrt(g max(h, 0)) whenever h >= floor (callers fix the rest)
__device__ __forceinline__ void inv_and_celerity(double h, double h_floor, double sqrt_g, double &r,
                                                 double &c)
{
    const double hf = max_pos(h, h_floor);
    const double y = rsqrt64(hf);
    r = y * y;
    c = sqrt_g * (hf * y);
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// L2 prefetch of one variable's modes over the strip: three probes per mode
// (first, middle and last element) cover the <= 3 lines a 32-element span
// touches, spread over the lanes (2 instructions per row at p = 3).
#if !DG_PF_SPREAD
template <int P>
__device__ __forceinline__ void row_prefetch_l2(const double *src, int nx, int ifirst, int lane)
{
    constexpr int NP = (P + 1) * (P + 1);
    int i = ifirst + lane;
    if (i >= nx) i -= nx;
    if (i < 0) i += nx;
    const double *p = src + i;
#pragma unroll
    for (int m = 0; m < NP; ++m, p += nx) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
#else
template <int P>
__device__ __forceinline__ void row_prefetch_l2(const double *src, int nx, int ifirst, int lane)
{
    constexpr int NP = (P + 1) * (P + 1);
#pragma unroll
    for (int k = lane; k < 3 * NP; k += kLanes) {
        const int m = k / 3, part = k - 3 * m;
        int e = ifirst + (part == 0 ? 0 : part == 1 ? 16 : kLanes - 1);
        if (e >= nx) e -= nx;
        if (e < 0) e += nx;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (size_t)m * nx + e));
    }
}
#endif

// this lane's element, one variable: NP words, mode-major, lane-minor
template <int P>
__device__ __forceinline__ void tile_fetch(double *dst, const double *src, int nx, int i, int lane)
{
    constexpr int NP = (P + 1) * (P + 1);
#pragma unroll
    for (int m = 0; m < NP; ++m) cp_async8(dst + m * kLanes + lane, src + (size_t)m * nx + i);
}

// bottom (sign -1) or top (sign +1) trace at the n edge nodes from modes
template <int P, bool TOP>
__device__ __forceinline__ void ytrace(const double (&c)[P + 1][P + 1], double (&tr)[P + 1])
{
    constexpr int N = P + 1;
    double s[N];
#pragma unroll
    for (int a = 0; a < N; ++a) {
        double e = c[a][0], o = 0.0;
#pragma unroll
        for (int b = 2; b < N; b += 2) e += c[a][b];
        if constexpr (N > 1) {
            o = c[a][1];
#pragma unroll
            for (int b = 3; b < N; b += 2) o += c[a][b];
            s[a] = TOP ? e + o : e - o;
        } else {
            s[a] = e;
        }
    }
    m2n<P, 0>(s, tr);
}

template <int P>
__device__ __forceinline__ void tile_read(double (&c)[P + 1][P + 1], const double *s, int lane)
{
    constexpr int N = P + 1;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) c[a][b] = s[(a * N + b) * kLanes + lane];
}

// Interior nodal values and L/R/T traces of one variable -> shared memory.
template <int P>
__device__ __forceinline__ unsigned eval_row(const double (&c)[P + 1][P + 1], double *sU, double *sXL,
                                             double *sXR, double *sT, int lane, bool check)
{
    constexpr int N = P + 1;
    unsigned bad = 0;
    double t[N][N];   // t[a][qj] = sum_b c[a][b] P_b(x_qj)
#pragma unroll
    for (int a = 0; a < N; ++a) m2n<P, 0>(c[a], t[a]);
#pragma unroll
    for (int q = 0; q < N; ++q) {   // xi = -1 / +1 traces: parity of a
        double e = t[0][q], o = 0.0;
#pragma unroll
        for (int a = 2; a < N; a += 2) e += t[a][q];
        if constexpr (N > 1) {
            o = t[1][q];
#pragma unroll
            for (int a = 3; a < N; a += 2) o += t[a][q];
        }
        const double l = e - o, r = e + o;
        sXL[q * kLanes + lane] = l;
        sXR[q * kLanes + lane] = r;
        if (check) bad |= !(l > 0.0) | !(r > 0.0);
    }
    double tt[N];
    ytrace<P, true>(c, tt);
#pragma unroll
    for (int q = 0; q < N; ++q) {
        sT[q * kLanes + lane] = tt[q];
        if (check) bad |= !(tt[q] > 0.0);
    }
#pragma unroll
    for (int qj = 0; qj < N; ++qj) {
        double col[N], u[N];
#pragma unroll
        for (int a = 0; a < N; ++a) col[a] = t[a][qj];
        m2n<P, 0>(col, u);
#pragma unroll
        for (int qi = 0; qi < N; ++qi) {
            sU[(qi * N + qj) * kLanes + lane] = u[qi];
            if (check) bad |= !(u[qi] > 0.0);
        }
    }
    return bad;
}

// Rusanov flux over one face from register traces: "in" = lower/left
// element, "out" = upper/right element, [var][node].  Stored is the face's
// boundary-integral projection g[var][k'] = scale * sum_k w_k P_k'(x_k) f*[k]
// (dg.py:206-212, 465-495): both neighbours lift it with their own
// outward-normal sign and mode parity, so each face is projected once.
// DIR 0: x-face, physical flux F, alpha = (|u|+c)/R.
// DIR 1: y-face, physical flux G = cos/R * (...), alpha = cos (|v|+c)/R.
template <int P, int DIR>
__device__ __forceinline__ void face_flux(const double (&in)[3][P + 1], const double (&out)[3][P + 1],
                                          double *sF, int lane, const StageParams &kp,
                                          double cr_e, double cos_e, double alpha_glob,
                                          double scale)
{
    constexpr int N = P + 1;
    constexpr int M = DIR == 0 ? 1 : 2;   // normal momentum
    double rin[N], rout[N];
    double am[N];
    bool low = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double ci, co;
        inv_and_celerity(in[0][k], kp.h_floor, kp.sqrt_g, rin[k], ci);
        inv_and_celerity(out[0][k], kp.h_floor, kp.sqrt_g, rout[k], co);
        low |= (in[0][k] < kp.h_floor) | (out[0][k] < kp.h_floor);
        am[k] = max_nn(fabs(in[M][k] * rin[k]) + ci, fabs(out[M][k] * rout[k]) + co);
    }
#pragma unroll
    for (int w = 1; w < N; w *= 2)     // pairwise tree: log2(N) dependent maxima
#pragma unroll
        for (int k = 0; k + w < N; k += 2 * w) am[k] = max_nn(am[k], am[k + w]);
    double amax = am[0];
    if (__any_sync(0xffffffffu, low)) {      // h below the velocity floor: exact celerity
        amax = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k)
            amax = fmax(amax, fmax(fabs(in[M][k] * rin[k]) + sqrt(kp.gravity * fmax(in[0][k], 0.0)),
                                   fabs(out[M][k] * rout[k]) + sqrt(kp.gravity * fmax(out[0][k], 0.0))));
    }
    double alpha = amax * kp.inv_r;
    if (DIR == 1) alpha *= cos_e;
    if (kp.alpha_mode != 0) alpha = alpha_glob;
    // the face's lift scale (bd_det) is folded into both halves of f*
    const double ha = (0.5 * scale) * alpha;
    const double hs = (0.5 * scale) * (DIR == 0 ? kp.inv_r : cr_e);
    double fs[3][N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double hi = in[0][k], ui = in[1][k], vi = in[2][k];
        const double ho = out[0][k], uo = out[1][k], vo = out[2][k];
        const double gi = hi * hi * kp.half_g, go = ho * ho * kp.half_g;
        double fi0, fi1, fi2, fo0, fo1, fo2;
        if (DIR == 0) {
            const double ui_ = ui * rin[k], vi_ = vi * rin[k];
            const double uo_ = uo * rout[k], vo_ = vo * rout[k];
            fi0 = ui; fi1 = fma(ui, ui_, gi); fi2 = ui * vi_;
            fo0 = uo; fo1 = fma(uo, uo_, go); fo2 = uo * vo_;
        } else {
            const double vi_ = vi * rin[k], vo_ = vo * rout[k];
            fi0 = vi; fi1 = ui * vi_; fi2 = fma(vi, vi_, gi);
            fo0 = vo; fo1 = uo * vo_; fo2 = fma(vo, vo_, go);
        }
        fs[0][k] = fma(hs, fi0 + fo0, -ha * (ho - hi));
        fs[1][k] = fma(hs, fi1 + fo1, -ha * (uo - ui));
        fs[2][k] = fma(hs, fi2 + fo2, -ha * (vo - vi));
    }
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double g[N];
        n2m<P, 2>(fs[v], g);
#pragma unroll
        for (int b = 0; b < N; ++b) sF[(v * N + b) * kLanes + lane] = g[b];
    }
}

template <int P>
__device__ __forceinline__ void traces_from_smem(double (&tr)[3][P + 1], const double *s, int lane)
{
    constexpr int N = P + 1;
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int k = 0; k < N; ++k) tr[v][k] = s[(v * N + k) * kLanes + lane];
}

// Face warp: bottom traces of the row above (from the coefficient ring,
// all three variables) -> y-face flux with the current row's top traces.
template <int P>
__device__ __forceinline__ unsigned yface_from_ring(const double *ring_row, const double *sT,
                                                    double *sF, int lane, const StageParams &kp,
                                                    const double *rowtab_above, double alpha_y)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using RL = RowLayout<P>;
    double bt[3][N];
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double cv[N][N];
        tile_read<P>(cv, ring_row + v * NP * kLanes, lane);
        ytrace<P, false>(cv, bt[v]);
    }
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) bad |= !(bt[0][k] > 0.0);
    double tt[3][N];
    traces_from_smem<P>(tt, sT, lane);
    face_flux<P, 1>(tt, bt, sF, lane, kp, rowtab_above[RL::CRB], rowtab_above[RL::COSB], alpha_y,
                    kp.bdx);
    return bad;
}

// Pointwise flux / source of variable v at the N nodes (qi, qj), qj = 0..N-1
// (models.py:161-252): F = x-flux (its cx/R goes into the xi weights),
// G = y-flux * cy cos/R, S = source.
template <int P>
__device__ __forceinline__ void node_physics(int v, int qi, const double *sU, const double *row, int lane,
                                             const StageParams &kp, double (&F)[P + 1],
                                             double (&G)[P + 1], double (&S)[P + 1])
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using RL = RowLayout<P>;
#pragma unroll
    for (int qj = 0; qj < N; ++qj) {
        const int q = qi * N + qj;
        const double hu = sU[(1 * NP + q) * kLanes + lane];
        const double hv = sU[(2 * NP + q) * kLanes + lane];
        const double crc = row[RL::CRC + qj];
        if (v == 0) {
            F[qj] = hu * CXN;
            G[qj] = hv * crc;
            S[qj] = 0.0;
        } else {
            const double h = sU[(0 * NP + q) * kLanes + lane];
            const double r = rcp64(max_pos(h, kp.h_floor));
            const double gh2 = h * h * kp.half_g;
            const double u = hu * r, w = hv * r;
            const double t = fma(u, row[RL::SRS + qj], row[RL::FCS + qj]);
            if (v == 1) {
                F[qj] = fma(hu, u, gh2) * CXN;
                G[qj] = hu * w * crc;
                S[qj] = t * hv;
            } else {
                F[qj] = hu * w * CXN;
                G[qj] = fma(hv, w, gh2) * crc;
                S[qj] = -fma(gh2, row[RL::SRS + qj], t * hu);
            }
        }
    }
}

// eta projections of one xi node line: f[b] = sum_qj wP_b F, g[b] = sum_qj (wP'_b G + wP_b S)
template <int P>
__device__ __forceinline__ void line_project(int v, const double (&F)[P + 1], const double (&G)[P + 1],
                                             const double (&S)[P + 1], double (&f)[P + 1],
                                             double (&g)[P + 1])
{
    n2m<P, 2>(F, f);
    if (v == 0)
        n2m<P, 3>(G, g);
    else
        n2m2<P, 3, 2>(G, S, g);
}

// Volume + source projection of variable v at the current row, streamed
// over pairs of xi node lines (qi, N-1-qi) so that the xi contraction also
// uses the even/odd split:
// vol[a][b] = sum_q (cx dphi/dxi F + cy dphi/deta G + cs phi S)[q]
template <int P>
__device__ __forceinline__ void volume(double (&vol)[P + 1][P + 1], int v, const double *sU,
                                       const double *row, int lane, const StageParams &kp)
{
    constexpr int N = P + 1;
    constexpr int H = N / 2;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) vol[a][b] = 0.0;
#pragma unroll 1
    for (int ip = 0; ip < H; ++ip) {
        double f0[N], g0[N], f1[N], g1[N];
#if DG_VOL_COMPACT
        // one loop body for both lines of the pair (I-cache footprint)
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
            double F[N], G[N], S[N];
            node_physics<P>(v, side ? N - 1 - ip : ip, sU, row, lane, kp, F, G, S);
            line_project<P>(v, F, G, S, f1, g1);
            if (side == 0) {
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    f0[b] = f1[b];
                    g0[b] = g1[b];
                }
            }
        }
#else
        {
            double F[N], G[N], S[N];
            node_physics<P>(v, ip, sU, row, lane, kp, F, G, S);
            line_project<P>(v, F, G, S, f0, g0);
            node_physics<P>(v, N - 1 - ip, sU, row, lane, kp, F, G, S);
            line_project<P>(v, F, G, S, f1, g1);
        }
#endif
        double pd[N], pp[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            pd[a] = WD(a, ip) * CXF;   // F's 1/R * determ/bd_det_x folded in here
            pp[a] = WP(a, ip);
        }
#pragma unroll
        for (int b = 0; b < N; ++b) {
            // wP'_a(N-1-i) = -(-1)^a wP'_a(i), wP_a(N-1-i) = (-1)^a wP_a(i)
            const double fp = f0[b] + f1[b], fm = f0[b] - f1[b];
            const double gp = g0[b] + g1[b], gm = g0[b] - g1[b];
#pragma unroll
            for (int a = 0; a < N; ++a)
                vol[a][b] = fma(pd[a], (a & 1) ? fp : fm, fma(pp[a], (a & 1) ? gm : gp, vol[a][b]));
        }
    }
    if constexpr (N & 1) {   // middle line xi = 0: wP'_a vanishes for even a, wP_a for odd a
        double F[N], G[N], S[N], f[N], g[N];
        node_physics<P>(v, H, sU, row, lane, kp, F, G, S);
        line_project<P>(v, F, G, S, f, g);
#pragma unroll
        for (int b = 0; b < N; ++b)
#pragma unroll
            for (int a = 0; a < N; ++a)
                vol[a][b] = (a & 1) ? fma(WD(a, H) * CXF, f[b], vol[a][b])
                                    : fma(WP(a, H), g[b], vol[a][b]);
    }
}

// Boundary lifts, inverse mass, stage combination and store for variable v.
// The mass block is applied column by column (one row of T from shared
// memory at a time) so that vol, c and u^n are the only tiles held.
template <int P, bool HAS_U>
__device__ __forceinline__ unsigned finalize(double (&vol)[P + 1][P + 1], const double *cur,
                                             const double *Uv, int v, const double *sFX,
                                             const double *sFtop, const double *sFbot, bool has_top,
                                             bool has_bot, const double *row, int lane, bool owned,
                                             double *Yv, int nx, int i, const StageParams &kp)
{
    constexpr int N = P + 1;
    using RL = RowLayout<P>;
    double un[N][N];
    if (HAS_U && !(DG_ABL & 4)) {      // u^n: plain loads (U may alias Y)
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) un[a][b] = Uv[(size_t)(a * N + b) * nx + i];
    }
    const int ll = lane > 0 ? lane - 1 : 0;
    const int o = (v * N) * kLanes;
#pragma unroll
    for (int b = 0; b < N; ++b) {
        // projected face lifts (bdy / bdx folded in by the face warp)
        const double r = sFX[o + b * kLanes + lane];
        const double l = sFX[o + b * kLanes + ll];
        const double t = has_top ? sFtop[o + b * kLanes + lane] : 0.0;   // pole faces carry
        const double bo = has_bot ? sFbot[o + b * kLanes + lane] : 0.0;  // no flux (dg.py:483-495)
        // x lifts broadcast along a (parity of a), y lifts along b (parity of b)
        const double xe = l - r, xo = -l - r;
        const double ye = bo - t, yo = -bo - t;
#pragma unroll
        for (int a = 0; a < N; ++a) {
            vol[a][b] += (a & 1) ? xo : xe;   // x lift: column b
            vol[b][a] += (a & 1) ? yo : ye;   // y lift of row b: column a parity
        }
    }
    const double *T = row + RL::T;
    int fexp = 0;                     // max exponent field of the outputs (integer pipe)
    double mean = 1.0;
#pragma unroll
    for (int b = 0; b < N; ++b) {
        double tb[N];
#pragma unroll
        for (int bb = 0; bb < N; ++bb) tb[bb] = T[b * N + bb];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            double k = tb[0] * vol[a][0];
            if (!(DG_ABL & 32)) {
#pragma unroll
                for (int bb = 1; bb < N; ++bb) k = fma(tb[bb], vol[a][bb], k);
            } else {
                k = vol[a][b];
            }
            double y = fma(kp.b, cur[(a * N + b) * kLanes + lane], (kp.g * (double)(2 * a + 1)) * k);
            if (HAS_U && !(DG_ABL & 4)) y = fma(kp.a, un[a][b], y);
            if (owned) Yv[(a * N + b) * nx] = y;
            fexp = max(fexp, __double2hiint(y) & 0x7ff00000);
            if (a == 0 && b == 0) mean = y;
        }
    }
    unsigned bad = 0;
    if (owned) {
        bad |= (kp.check_finite && fexp == 0x7ff00000) ? 2u : 0u;   // Inf or NaN
        bad |= (v == 0 && kp.check_mean && !(mean > 0.0)) ? 4u : 0u;
    }
    return bad;
}

template <int P, bool HAS_U>
__global__ void __launch_bounds__(kThreads, (P <= 3 ? DG_MINB : 2)) stage_kernel(StageParams kp)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using SM = Smem<P>;
    using RL = RowLayout<P>;
    extern __shared__ double smem[];
    // fixed roles: warp w runs on sub-partition w of its SM, so every
    // sub-partition executes a single code path (better I-cache locality
    // than rotating roles across CTAs, measured)
    const int role = threadIdx.x >> 5;
    const int v = role < kVarWarps ? role : 0;     // face warp borrows var 0's addressing
    const bool face_warp = role == kVarWarps;
    const int lane = threadIdx.x & 31;
    const int nx = kp.nx;
    const int i0 = blockIdx.x * kOwned;
    int i = (i0 - 1 + lane) % nx;
    if (i < 0) i += nx;
    const int nown = min(kOwned, nx - i0);
    const bool owned = lane >= 1 && lane <= nown;
    const int jb = kp.j_begin + blockIdx.y * kp.rc;
    const int je = min(jb + kp.rc, kp.j_end);
    if (jb >= je) return;

    // coefficient ring: slot s holds row (jb + s) mod 2, layout [var][mode][lane]
    double *const ringS = smem + SM::XR0;
    double *const ring0 = ringS + v * NP * kLanes;   // this warp's variable
    double *sU = smem + SM::U;
    double *sXL = smem + SM::XL;
    double *sXR = smem + SM::XRT;
    double *sT = smem + SM::TT;
    double *sFX = smem + SM::FX;
    double *sFa = smem + SM::FY0;
    double *sFb = smem + SM::FY1;
    double *sRow = smem + SM::ROW;

    const double *Xz = kp.X + (size_t)blockIdx.z * kp.zstride + (size_t)v * NP * nx;
    const double *Uz = kp.U ? kp.U + (size_t)blockIdx.z * kp.zstride + (size_t)v * NP * nx : nullptr;
    double *Yz = kp.Y + (size_t)blockIdx.z * kp.zstride + (size_t)v * NP * nx;
    const bool chk = (v == 0) && !face_warp;
    unsigned bad = 0;

    // rows whose coefficients exist: local r with global row0+r in [0, ny)
    const int r_last = min(kp.nrows - 1, kp.ny - 1 - kp.row0);

    // prologue: start streaming rows jb and jb+1
    if (!face_warp) {
        tile_fetch<P>(ring0, Xz + (size_t)jb * kp.rstride, nx, i, lane);
        cp_commit();
        if (jb + 1 <= min(je, r_last))
            tile_fetch<P>(ring0 + SM::TILE, Xz + (size_t)(jb + 1) * kp.rstride, nx, i, lane);
        cp_commit();
    }

    // row-table ring: slot (r - jb) % 3 holds local row r (rows jb, jb+1 now,
    // row jl+2 staged by the face warp during iteration jl)
    const int gfirst = kp.row0 + jb;
    {
        const int nload = min(2, kp.ny - gfirst);
        for (int idx = threadIdx.x; idx < nload * RL::STRIDE; idx += kThreads)
            sRow[idx] = kp.rowtab[(size_t)gfirst * RL::STRIDE + idx];
    }

    double alpha_x = kp.alpha, alpha_y = kp.alpha;
    if (kp.alpha_mode == 2) {
        alpha_x = kp.alpha_dev[0];
        alpha_y = kp.alpha_dev[1];
    }

    // top traces of the row below the chunk (its first row's bottom face)
    const bool below = gfirst > 0;
    double c[N][N];
    if (below && !face_warp) {
        const double *src = Xz + (size_t)(jb - 1) * kp.rstride;
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) c[a][b] = __ldg(src + (size_t)(a * N + b) * nx + i);
        double tt[N];
        ytrace<P, true>(c, tt);
#pragma unroll
        for (int q = 0; q < N; ++q) sT[(v * N + q) * kLanes + lane] = tt[q];
    }
    if (!face_warp) cp_wait<1>();                    // row jb landed (own copies); jb+1 in flight
    __syncthreads();
    if (face_warp) {
        if (below)
            bad |= yface_from_ring<P>(ringS, sT, sFb, lane, kp, sRow, alpha_y);
        else
            bad |= 0u;
    }
    __syncthreads();
    if (face_warp && !below) {
        // no bottom face, but the first row's bottom traces still need the positivity check
        double cv[N][N];
        tile_read<P>(cv, ringS, lane);
        double bt[N];
        ytrace<P, false>(cv, bt);
#pragma unroll
        for (int k = 0; k < N; ++k) bad |= !(bt[k] > 0.0);
    }

#ifdef DG_TIMING
    unsigned tacc[5] = {0, 0, 0, 0, 0};
#endif
    for (int jl = jb; jl < je; ++jl) {
        TSTAMP(0);
        const int slot = (jl - jb) & 1;
        double *const cur = ring0 + slot * SM::TILE;
        const int jg = kp.row0 + jl;
        const bool has_top = jg + 1 < kp.ny;
        const bool has_bot = jg > 0;
        const double *row = sRow + ((jl - jb) % 3) * RL::STRIDE;

        if (!face_warp) {
            // warm L2 for this row's u^n and for row jl+2 (copied in after finalize)
            if (HAS_U) row_prefetch_l2<P>(Uz + (size_t)jl * kp.rstride, nx, i0 - 1, lane);
            if (jl + 2 <= min(je, r_last))
                row_prefetch_l2<P>(Xz + (size_t)(jl + 2) * kp.rstride, nx, i0 - 1, lane);
            tile_read<P>(c, cur, lane);                // X(jl)
            if (DG_ABL & 16) {
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) sU[(v * NP + a * N + b) * kLanes + lane] = c[a][b];
            } else {
                bad |= eval_row<P>(c, sU + v * NP * kLanes, sXL + v * N * kLanes, sXR + v * N * kLanes,
                                   sT + v * N * kLanes, lane, chk);
            }
            cp_wait<0>();                              // X(jl+1) landed (own copies)
        }
        TSTAMP(1);
        __syncthreads();
        TSTAMP(2);

        if (face_warp) {
            if (has_top && !(DG_ABL & 1))
                bad |= yface_from_ring<P>(ringS + (slot ^ 1) * SM::TILE, sT, sFa, lane, kp,
                                          sRow + ((jl + 1 - jb) % 3) * RL::STRIDE, alpha_y);
            // stage the table of row jl+2 (its slot held row jl-1, no longer read)
            if (jl + 2 <= je && jg + 2 < kp.ny) {
                double *dst = sRow + ((jl + 2 - jb) % 3) * RL::STRIDE;
                const double *src = kp.rowtab + (size_t)(jg + 2) * RL::STRIDE;
                for (int idx = lane; idx < RL::STRIDE; idx += kLanes) dst[idx] = src[idx];
            }
            TSTAMP(3);
            __syncthreads();
            TSTAMP(4);
            TACC(2, tk3 - tk2);
            TACC(3, tk4 - tk3);
        } else {
            if (v == 0 && !(DG_ABL & 2)) {
                // the h warp has the lightest volume work: it takes the x-faces
                double in[3][N], out[3][N];
                traces_from_smem<P>(in, sXR, lane);
                traces_from_smem<P>(out, sXL, min(lane + 1, 31));
                face_flux<P, 0>(in, out, sFX, lane, kp, 0.0, 0.0, alpha_x, kp.bdy);
            }
            double vol[N][N];
            if ((DG_ABL & 8) && v > 0) {
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) vol[a][b] = sU[(a * N + b) * kLanes + lane];
            } else {
                volume<P>(vol, v, sU, row, lane, kp);
            }
            TSTAMP(3);
            __syncthreads();
            TSTAMP(4);
            const size_t roff = (size_t)jl * kp.rstride;
            bad |= finalize<P, HAS_U>(vol, cur, HAS_U ? Uz + roff : nullptr, v, sFX, sFa, sFb,
                                      has_top, has_bot, row, lane, owned, Yz + roff + i, nx, i, kp);
            // X(jl) is consumed: stream row jl+2 into its slot (L2-warm by now)
            __syncwarp();
            if (jl + 2 <= min(je, r_last))
                tile_fetch<P>(cur, Xz + (size_t)(jl + 2) * kp.rstride, nx, i, lane);
            cp_commit();
            TSTAMP(5);
            TACC(2, tk3 - tk2);
            TACC(3, tk4 - tk3);
            TACC(4, tk5 - tk4);
        }
        TACC(0, tk1 - tk0);
        TACC(1, tk2 - tk1);
        double *tmp = sFa;
        sFa = sFb;
        sFb = tmp;
    }
    if (!face_warp) cp_wait<0>();

#ifdef DG_TIMING
    if (lane == 0) {
        for (int k = 0; k < 5; ++k) atomicAdd(&g_timing[role][k], (unsigned long long)tacc[k]);
        atomicAdd(&g_timing[role][5], (unsigned long long)(je - jb));
    }
#endif
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) {
        atomicOr(kp.status, bad);
        atomicMin(kp.first_tag, kp.tag);
    }
}

#undef LEG
#undef WP
#undef WD

}  // namespace dgswe
