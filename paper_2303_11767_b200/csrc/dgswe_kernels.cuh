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

// 1/x: MUFU seed + two Newton steps (<= 1 ulp for normal x)
__device__ __forceinline__ double rcp64(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// 1/sqrt(x): MUFU seed + two Newton steps (x > 0, normal)
__device__ __forceinline__ double rsqrt64(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double e = fma(-hx * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-hx * y, y, 0.5);
    return fma(y, e, y);
}

// 1/hf and sqrt(g hf) with hf = max(h, floor) from one rsqrt; equals the
// reference's sqrt(g max(h, 0)) whenever h >= floor (callers fix the rest)
__device__ __forceinline__ void inv_and_celerity(double h, double h_floor, double sqrt_g, double &r,
                                                 double &c)
{
    const double hf = fmax(h, h_floor);
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

// L2 prefetch of one variable's modes for elements [lo, hi) of a row
// (bulk async prefetch, one mode per lane)
template <int P>
__device__ __forceinline__ void row_prefetch_l2(const double *src, int nx, int lo, int hi, int lane)
{
    constexpr int NP = (P + 1) * (P + 1);
    for (int m = lane; m < NP; m += kLanes) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(src + (size_t)m * nx + lo) & ~(uintptr_t)15;
        const uintptr_t e = (reinterpret_cast<uintptr_t>(src + (size_t)m * nx + hi) + 15) & ~(uintptr_t)15;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a))
                     : "memory");
    }
}

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
        double acc = c[a][0];
#pragma unroll
        for (int b = 1; b < N; ++b) acc = TOP ? acc + c[a][b] : fma(sgn(b), c[a][b], acc);
        s[a] = acc;
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        double acc = LEG(0, q) * s[0];
#pragma unroll
        for (int a = 1; a < N; ++a) acc = fma(LEG(a, q), s[a], acc);
        tr[q] = acc;
    }
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
    double t[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int q = 0; q < N; ++q) {
            double acc = c[a][0] * LEG(0, q);
#pragma unroll
            for (int b = 1; b < N; ++b) acc = fma(c[a][b], LEG(b, q), acc);
            t[a][q] = acc;
        }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        double l = t[0][q], r = t[0][q];
#pragma unroll
        for (int a = 1; a < N; ++a) {
            r += t[a][q];
            l = fma(sgn(a), t[a][q], l);
        }
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
#pragma unroll 1
    for (int qi = 0; qi < N; ++qi) {
        double pa[N];
#pragma unroll
        for (int a = 0; a < N; ++a) pa[a] = LEG(a, qi);
#pragma unroll
        for (int qj = 0; qj < N; ++qj) {
            double acc = pa[0] * t[0][qj];
#pragma unroll
            for (int a = 1; a < N; ++a) acc = fma(pa[a], t[a][qj], acc);
            sU[(qi * N + qj) * kLanes + lane] = acc;
            if (check) bad |= !(acc > 0.0);
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
    double amax = 0.0;
    bool low = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double ci, co;
        inv_and_celerity(in[0][k], kp.h_floor, kp.sqrt_g, rin[k], ci);
        inv_and_celerity(out[0][k], kp.h_floor, kp.sqrt_g, rout[k], co);
        low |= (in[0][k] < kp.h_floor) | (out[0][k] < kp.h_floor);
        amax = fmax(amax, fmax(fabs(in[M][k] * rin[k]) + ci, fabs(out[M][k] * rout[k]) + co));
    }
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
    const double ha = 0.5 * alpha;
    const double hs = 0.5 * (DIR == 0 ? kp.inv_r : cr_e);
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
    for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int b = 0; b < N; ++b) {
            double g = WP(b, 0) * fs[v][0];
#pragma unroll
            for (int k = 1; k < N; ++k) g = fma(WP(b, k), fs[v][k], g);
            sF[(v * N + b) * kLanes + lane] = g * scale;
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

// Volume + source projection of variable v at the current row, streamed
// over the xi node index qi:
// vol[a][b] = sum_q (cx dphi/dxi F + cy dphi/deta G + cs phi S)[q]
template <int P>
__device__ __forceinline__ void volume(double (&vol)[P + 1][P + 1], int v, const double *sU,
                                       const double *row, int lane, const StageParams &kp)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using RL = RowLayout<P>;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) vol[a][b] = 0.0;
#pragma unroll 1
    for (int qi = 0; qi < N; ++qi) {
        double F[N], G[N], S[N];
#pragma unroll
        for (int qj = 0; qj < N; ++qj) {
            const int q = qi * N + qj;
            const double hu = sU[(1 * NP + q) * kLanes + lane];
            const double hv = sU[(2 * NP + q) * kLanes + lane];
            const double crc = row[RL::CRC + qj];
            if (v == 0) {
                F[qj] = hu * kp.inv_r_cx;
                G[qj] = hv * crc;
                S[qj] = 0.0;
            } else {
                const double h = sU[(0 * NP + q) * kLanes + lane];
                const double r = rcp64(fmax(h, kp.h_floor));
                const double gh2 = h * h * kp.half_g;
                const double u = hu * r, w = hv * r;
                const double t = fma(u, row[RL::SRS + qj], row[RL::FCS + qj]);
                if (v == 1) {
                    F[qj] = fma(hu, u, gh2) * kp.inv_r_cx;
                    G[qj] = hu * w * crc;
                    S[qj] = t * hv;
                } else {
                    F[qj] = hu * w * kp.inv_r_cx;
                    G[qj] = fma(hv, w, gh2) * crc;
                    S[qj] = -fma(gh2, row[RL::SRS + qj], t * hu);
                }
            }
        }
        double pd[N], pp[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            pd[a] = WD(a, qi);
            pp[a] = WP(a, qi);
        }
        if (v == 0) {
#pragma unroll
            for (int b = 0; b < N; ++b) {
                double f = WP(b, 0) * F[0], g = WD(b, 0) * G[0];
#pragma unroll
                for (int qj = 1; qj < N; ++qj) {
                    f = fma(WP(b, qj), F[qj], f);
                    g = fma(WD(b, qj), G[qj], g);
                }
#pragma unroll
                for (int a = 0; a < N; ++a) vol[a][b] = fma(pd[a], f, fma(pp[a], g, vol[a][b]));
            }
        } else {
#pragma unroll
            for (int b = 0; b < N; ++b) {
                double f = WP(b, 0) * F[0], g = fma(WD(b, 0), G[0], WP(b, 0) * S[0]);
#pragma unroll
                for (int qj = 1; qj < N; ++qj) {
                    f = fma(WP(b, qj), F[qj], f);
                    g = fma(WD(b, qj), G[qj], g);
                    g = fma(WP(b, qj), S[qj], g);
                }
#pragma unroll
                for (int a = 0; a < N; ++a) vol[a][b] = fma(pd[a], f, fma(pp[a], g, vol[a][b]));
            }
        }
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
    if (HAS_U) {                       // u^n: plain loads (U may alias Y)
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
    double fin = 0.0;                 // NaN iff some output is not finite
    double mean = 1.0;
#pragma unroll
    for (int b = 0; b < N; ++b) {
        double tb[N];
#pragma unroll
        for (int bb = 0; bb < N; ++bb) tb[bb] = T[b * N + bb];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            double k = tb[0] * vol[a][0];
#pragma unroll
            for (int bb = 1; bb < N; ++bb) k = fma(tb[bb], vol[a][bb], k);
            double y = fma(kp.b, cur[(a * N + b) * kLanes + lane], (kp.g * (double)(2 * a + 1)) * k);
            if (HAS_U) y = fma(kp.a, un[a][b], y);
            if (owned) Yv[(a * N + b) * nx] = y;
            fin += y - y;
            if (a == 0 && b == 0) mean = y;
        }
    }
    unsigned bad = 0;
    if (owned) {
        bad |= (kp.check_finite && !(fin == fin)) ? 2u : 0u;
        bad |= (v == 0 && kp.check_mean && !(mean > 0.0)) ? 4u : 0u;
    }
    return bad;
}

template <int P, bool HAS_U>
__global__ void __launch_bounds__(kThreads, (P <= 3 ? 4 : 2)) stage_kernel(StageParams kp)
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
    const int plo = max(i0 - 1, 0), phi = min(i0 + kLanes - 1, nx);   // prefetch range
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

    for (int jl = jb; jl < je; ++jl) {
        const int slot = (jl - jb) & 1;
        double *const cur = ring0 + slot * SM::TILE;
        const int jg = kp.row0 + jl;
        const bool has_top = jg + 1 < kp.ny;
        const bool has_bot = jg > 0;
        const double *row = sRow + ((jl - jb) % 3) * RL::STRIDE;

        if (!face_warp) {
            // warm L2 for this row's u^n and for row jl+2 (copied in after finalize)
            if (HAS_U) row_prefetch_l2<P>(Uz + (size_t)jl * kp.rstride, nx, plo, phi, lane);
            if (jl + 2 <= min(je, r_last))
                row_prefetch_l2<P>(Xz + (size_t)(jl + 2) * kp.rstride, nx, plo, phi, lane);
            tile_read<P>(c, cur, lane);                // X(jl)
            bad |= eval_row<P>(c, sU + v * NP * kLanes, sXL + v * N * kLanes, sXR + v * N * kLanes,
                               sT + v * N * kLanes, lane, chk);
            cp_wait<0>();                              // X(jl+1) landed (own copies)
        }
        __syncthreads();

        if (face_warp) {
            if (has_top)
                bad |= yface_from_ring<P>(ringS + (slot ^ 1) * SM::TILE, sT, sFa, lane, kp,
                                          sRow + ((jl + 1 - jb) % 3) * RL::STRIDE, alpha_y);
            // stage the table of row jl+2 (its slot held row jl-1, no longer read)
            if (jl + 2 <= je && jg + 2 < kp.ny) {
                double *dst = sRow + ((jl + 2 - jb) % 3) * RL::STRIDE;
                const double *src = kp.rowtab + (size_t)(jg + 2) * RL::STRIDE;
                for (int idx = lane; idx < RL::STRIDE; idx += kLanes) dst[idx] = src[idx];
            }
            __syncthreads();
        } else {
            if (v == 0) {
                // the h warp has the lightest volume work: it takes the x-faces
                double in[3][N], out[3][N];
                traces_from_smem<P>(in, sXR, lane);
                traces_from_smem<P>(out, sXL, min(lane + 1, 31));
                face_flux<P, 0>(in, out, sFX, lane, kp, 0.0, 0.0, alpha_x, kp.bdy);
            }
            double vol[N][N];
            volume<P>(vol, v, sU, row, lane, kp);
            __syncthreads();
            const size_t roff = (size_t)jl * kp.rstride;
            bad |= finalize<P, HAS_U>(vol, cur, HAS_U ? Uz + roff : nullptr, v, sFX, sFa, sFb,
                                      has_top, has_bot, row, lane, owned, Yz + roff + i, nx, i, kp);
            // X(jl) is consumed: stream row jl+2 into its slot (L2-warm by now)
            __syncwarp();
            if (jl + 2 <= min(je, r_last))
                tile_fetch<P>(cur, Xz + (size_t)(jl + 2) * kp.rstride, nx, i, lane);
            cp_commit();
        }
        double *tmp = sFa;
        sFa = sFb;
        sFb = tmp;
    }
    if (!face_warp) cp_wait<0>();

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
