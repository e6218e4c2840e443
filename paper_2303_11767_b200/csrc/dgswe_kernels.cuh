// dgswe_kernels.cuh -- fused fp64 DG shallow-water stage kernel for sm_100a.
//
// HBM layout of a state (strip-blocked structure of arrays):
//   [nz][row][var 3][strip][mode nphi][32 elements]
// A strip is 32 consecutive longitude elements (the last one zero-padded),
// so one variable's row tile of a strip is a single contiguous block of
// nphi * 256 bytes: it moves with ONE TMA bulk copy (cp.async.bulk +
// mbarrier), its L2 prefetch is one bulk-prefetch instruction, and every
// per-lane load/store inside it is an immediate offset from one base.
//
// One CTA = 4 warps x 32 lanes on one strip: warp v < 3 owns variable v in
// {h, hu, hv}; warp 0 (lightest physics) also evaluates the row's x-faces
// 1..32 and warp 3 (the face warp) the y-face above the row, the strip's
// two halo traces and its left border face 0.  Lane l owns element
// 32*strip + l.  The CTA marches north through a chunk of latitude rows.
//
// Per row, per variable and lane (n = p+1, all tensor contractions
// sum-factorised with the even/odd split; constant tables in __constant__):
//   1. modal -> nodal: t[a][qj] = sum_b c[a][b] P_b(x_qj),
//      U[qi][qj] = sum_a P_a(x_qi) t[a][qj]; traces L/R from t, T/B from
//      sum_b c[a][b](+-1)^b                          (dg.py:348-357)
//   2. nodal values exchanged through shared memory; pointwise flux /
//      source physics for this warp's variable      (models.py:161-252)
//   3. Rusanov fluxes with local alpha               (dg.py:92-119,385-453)
//   4. volume + source projection streamed over xi node pairs, boundary
//      lifts, per-row inverse mass (Kronecker block form), fused RK stage
//      update (dg.py:455-502, timestep.py:132-167)
//
// Floating point: FMA contraction, refined MUFU reciprocals and a different
// summation order than the reference; results agree with the reference's
// exact-order oracle to ~1e-15 relative per step (tests/test_gpu_parity.py).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgswe {

constexpr int kMaxP = 6;
constexpr int kLanes = 32;   // elements per strip (== DGSWE_STRIP)
constexpr int kVarWarps = 3; // one per conserved variable
constexpr int kWarps = 4;    // + one face warp (Rusanov fluxes)
constexpr int kThreads = kWarps * kLanes;

// [p][table][a][q]: 0 P_a(x_q), 1 P'_a(x_q), 2 w_q P_a(x_q), 3 w_q P'_a(x_q)
__constant__ double c_tab[kMaxP + 1][4][kMaxP + 1][kMaxP + 1];

struct StageParams {
    const double *X;      // stage input (level 0, buffer row 0)
    const double *U;      // u^n for the combination (may be null when a == 0)
    double *Y;            // output
    const double *A;      // second output's addend (HAS_Y2 kernels; may alias Y2)
    double *Y2;           // second output Y2 = A + g2 RHS(X) (classical RK4's accumulator)
    double g2;
    long long zstride;    // doubles per level
    long long rstride;    // doubles per buffer row (3 * vstride)
    long long vstride;    // doubles per variable row (nstrip * nphi * 32)
    int nx, nstrip, ny, row0, nrows;
    int j_begin, j_end, rc;   // local rows [j_begin, j_end), rc rows per CTA
    int nchunk1;              // chunks of the first range; later chunks cover [j_begin2, j_end2)
    int j_begin2, j_end2;
    double a, b, g;       // Y = a U + b X + g RHS(X)
    const double *rowtab; // per global row, see RowLayout
    double inv_r;         // 1/R
    double inv_r_cx;      // (1/R) * determ/bd_det_x
    double gravity, half_g, h_floor, inv_floor, sqrt_g;
    double bdx, bdy;      // bd_det_x, bd_det_y
    int alpha_mode;       // 0 local, 1 pinned, 2 global (from alpha_dev)
    double alpha;
    const double *alpha_dev;
    unsigned *status;
    int *first_tag;
    int tag;
    int check_finite;
    int check_mean;
    // fused halo exchange over peer memory (edge launches of a latitude
    // band, bands.py transport "fused"): [0] south, [1] north neighbour
    int edge;                           // 1: this launch computes the band's edge rows
    int band_lo, band_hi;               // the band's computed rows [band_lo, band_hi)
    double *peer_row[2];                // neighbour's halo row (level 0) our edge row is copied to
    long long peer_zstride[2];
    unsigned long long *peer_count[2];  // neighbour's receive counter for that halo
    const unsigned long long *recv_count;   // own receive counters [2] (system-scope atomics)
    unsigned long long *stage_ctr;      // own [0] completed edge launches, [1] CTA completions
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

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
#ifndef DG_SELFLOOR
#define DG_SELFLOOR 1   // 1/max(h, floor) as rcp(h) + select: the reciprocal starts at once
#endif
#ifndef DG_VOL_UNROLL
#define DG_VOL_UNROLL 0
#endif
#ifndef DG_MINB
#define DG_MINB 3   // resident CTAs per SM the p <= 3 build is register-capped for (~160 registers;
                    // 4 CTAs at 128 registers measured 7% slower at C3 once the code was compact)
#endif

// DG_TIMING builds record per-role phase durations (clock cycles) of every
// row: [role][A work, barrier-1 wait, B work, barrier-2 wait, C work, rows]
#ifdef DG_TIMING
__device__ unsigned long long g_timing[4][7];
#define TSTAMP(k)                                                                  \
    unsigned tk##k;                                                                \
    asm volatile("mov.u32 %0, %%clock;" : "=r"(tk##k)::"memory")
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
    static constexpr int XR0 = 0;                        // coefficient ring slot 0 [var][mode][lane]
    static constexpr int XR1 = XR0 + TILE;               // slot 1
    static constexpr int U = XR1 + TILE;                 // nodal values [3][NP][32]
    static constexpr int XL = U + TILE;                  // [3][N][32]
    static constexpr int XRT = XL + TR;
    static constexpr int TT = XRT + TR;                  // top traces of current row
    static constexpr int FX = TT + TR;                   // x-face fluxes [3][N][33], face f left of lane f
                                                         // (face 0 lives in F0, double-buffered)
    static constexpr int FY0 = FX + 3 * N * (kLanes + 1);   // y-face flux buffers [3][N][32]
    static constexpr int FY1 = FY0 + TR;
    static constexpr int HL = FY1 + TR;                  // left-halo R trace [3][N]
    static constexpr int HR = HL + 3 * N;                // right-halo L trace [3][N]
    static constexpr int E0 = HR + 3 * N;                // element 0's L trace [3][N] (face warp)
    static constexpr int F0 = E0 + 3 * N;                // face 0 flux [row parity][3][N]
    static constexpr int HB = F0 + 6 * N;                // next row's neighbour coefficients [2][3][NP]
    static constexpr int ROW = HB + 6 * NP;              // row-table ring, 3 rows
    static constexpr int MBAR = ROW + 3 * RowLayout<P>::STRIDE;   // 6 mbarriers [slot][var]
    static constexpr int TOTAL = MBAR + 6;
};

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

// 1/hf with hf = max(h, floor) (models.py:161-166) and the celerity
// sqrt(g max(h, 0)) (models.py:254-258) from ONE rsqrt of h: below the floor
// 1/hf is the constant 1/floor, and h <= 0 (flagged by the positivity
// check) gives c = 0 like the reference.
__device__ __forceinline__ void inv_and_celerity(double h, double h_floor, double inv_floor, double sqrt_g,
                                                 double &r, double &c)
{
    const double y = rsqrt64(max_pos(h, 2.2250738585072014e-308));
    r = h >= h_floor ? y * y : inv_floor;
    c = h > 0.0 ? sqrt_g * (h * y) : 0.0;
}

// --- TMA bulk copies and mbarriers (one elected lane per variable warp) ---
__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long *mb, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}

// one variable's row tile of the strip (bytes contiguous) -> shared memory
__device__ __forceinline__ void tma_row(double *dst, const double *src, unsigned bytes,
                                        unsigned long long *mb)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *mb, unsigned parity)
{
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mb)),
        "r"(parity)
        : "memory");
}

// shared-memory reads of the generic proxy before a TMA overwrite
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// per-lane 8-byte async copies (the face warp's small gathers)
__device__ __forceinline__ void cp_async8(double *dst, const double *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l2_bulk(const double *src, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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

// Scalars of one face-flux call, by value (no pointer to the kernel
// parameters may escape into a non-inlined function).
struct FaceArgs {
    double h_floor, inv_floor, sqrt_g, half_g, inv_r;
    int alpha_mode, dir;
    double cr_e, cos_e, alpha_glob, scale;
};

// Rusanov flux over one face per lane (dg.py:92-119, 385-453): "in" =
// lower/left element's traces, "out" = upper/right element's, [var][node];
// local alpha = max over both sides' nodes of (|normal velocity| + c)/R
// (y-faces scaled by cos of the edge latitude, models.py:254-280), or the
// global / pinned alpha.  Stored is the face's boundary-integral projection
// g[var][k'] = scale * sum_k w_k P_k'(x_k) f*[k] (dg.py:206-212, 465-495):
// both neighbours lift it with their own outward-normal sign and mode
// parity, so each face is evaluated and projected once.
// dir 0: x-face, physical flux F; dir 1: y-face, G = cos/R * (...).
//
// ONE non-inlined copy serves the h warp's x-faces, the face warp's y-faces
// and the strip's border face: traces and result are addressed as (offset,
// leading dimension, column) in the kernel's dynamic shared memory, so no
// register array crosses the call.  (Three inlined copies cost ~1k SASS
// instructions of a kernel whose speed tracks its instruction-cache
// footprint; sF may alias the "out" traces.)
template <int P>
__device__ __forceinline__ void face_flux_body(int in_off, int in_ld, int in_col, int out_off, int out_ld,
                                               int out_col, int dst_off, int dst_ld, int dst_col, FaceArgs fa)
{
    constexpr int N = P + 1;
    extern __shared__ double smem[];
    double in[3][N], out[3][N];
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int k = 0; k < N; ++k) {
            in[v][k] = smem[in_off + (v * N + k) * in_ld + in_col];
            out[v][k] = smem[out_off + (v * N + k) * out_ld + out_col];
        }
    double rin[N], rout[N], mi[N], mo[N];
    double am[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double ci, co;
        inv_and_celerity(in[0][k], fa.h_floor, fa.inv_floor, fa.sqrt_g, rin[k], ci);
        inv_and_celerity(out[0][k], fa.h_floor, fa.inv_floor, fa.sqrt_g, rout[k], co);
        mi[k] = fa.dir == 0 ? in[1][k] : in[2][k];     // normal momentum
        mo[k] = fa.dir == 0 ? out[1][k] : out[2][k];
        am[k] = max_nn(fabs(mi[k] * rin[k]) + ci, fabs(mo[k] * rout[k]) + co);
    }
#pragma unroll
    for (int w = 1; w < N; w *= 2)
#pragma unroll
        for (int k = 0; k + w < N; k += 2 * w) am[k] = max_nn(am[k], am[k + w]);
    double alpha = am[0] * fa.inv_r;
    if (fa.dir == 1) alpha *= fa.cos_e;
    if (fa.alpha_mode != 0) alpha = fa.alpha_glob;
    const double ha = (0.5 * fa.scale) * alpha;
    const double hs = (0.5 * fa.scale) * (fa.dir == 0 ? fa.inv_r : fa.cr_e);
    const double sx = fa.dir == 0 ? 1.0 : 0.0, sy = 1.0 - sx;
    double fs[3][N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double hi = in[0][k], ui = in[1][k], vi = in[2][k];
        const double ho = out[0][k], uo = out[1][k], vo = out[2][k];
        const double gi = hi * hi * fa.half_g, go = ho * ho * fa.half_g;
        const double wi = mi[k] * rin[k], wo = mo[k] * rout[k];
        const double fi1 = fma(ui, wi, sx * gi), fo1 = fma(uo, wo, sx * go);
        const double fi2 = fma(vi, wi, sy * gi), fo2 = fma(vo, wo, sy * go);
        fs[0][k] = fma(hs, mi[k] + mo[k], -ha * (ho - hi));
        fs[1][k] = fma(hs, fi1 + fo1, -ha * (uo - ui));
        fs[2][k] = fma(hs, fi2 + fo2, -ha * (vo - vi));
    }
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double g[N];
        n2m<P, 2>(fs[v], g);
#pragma unroll
        for (int b = 0; b < N; ++b) smem[dst_off + (v * N + b) * dst_ld + dst_col] = g[b];
    }
}

template <int P>
__device__ __noinline__ void face_flux_noinline(int in_off, int in_ld, int in_col, int out_off, int out_ld,
                                                int out_col, int dst_off, int dst_ld, int dst_col, FaceArgs fa)
{
    face_flux_body<P>(in_off, in_ld, in_col, out_off, out_ld, out_col, dst_off, dst_ld, dst_col, fa);
}

// p >= 2: the shared non-inlined copy; p <= 1: inlined (the face work is a
// large share of a low-order element and the call's overhead shows, measured)
template <int P>
__device__ __forceinline__ void face_flux_call(int in_off, int in_ld, int in_col, int out_off, int out_ld,
                                               int out_col, int dst_off, int dst_ld, int dst_col, FaceArgs fa)
{
    if constexpr (P <= 1)
        face_flux_body<P>(in_off, in_ld, in_col, out_off, out_ld, out_col, dst_off, dst_ld, dst_col, fa);
    else
        face_flux_noinline<P>(in_off, in_ld, in_col, out_off, out_ld, out_col, dst_off, dst_ld, dst_col, fa);
}


// Pointwise flux / source at the N nodes (qi, qj), qj = 0..N-1
// (models.py:161-252): F = x-flux (its cx/R goes into the xi weights),
// G = y-flux * cy cos/R, S = source.  MOM = false: the h equation
// (F = hu, G = hv cos/R, no source).  MOM = true: one branch-free code path
// for both momentum equations, the variable (is_v: hv) entering only
// through uniform selects, so the nodes' instructions interleave:
//   hu: F = hu u + g h^2/2,  G = hu w cos/R,             S = t hv
//   hv: F = hu w,            G = (hv w + g h^2/2) cos/R, S = -(g h^2/2 sin/R + t hu)
// with u = hu/hf, w = hv/hf, t = u sin/R + 2 Omega sin cos.
template <int P, bool MOM>
__device__ __forceinline__ void node_physics(bool is_v, int qi, const double *sU, const double *row, int lane,
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
        if constexpr (!MOM) {
            F[qj] = hu;
            G[qj] = hv * crc;
            S[qj] = 0.0;
        } else {
            const double h = sU[(0 * NP + q) * kLanes + lane];
#if DG_SELFLOOR
            const double r0 = rcp64(h);
            const double r = h >= kp.h_floor ? r0 : kp.inv_floor;
#else
            const double r = rcp64(max_pos(h, kp.h_floor));
#endif
            const double gh2 = h * h * kp.half_g;
            const double u = hu * r, w = hv * r;
            const double srs = row[RL::SRS + qj];
            const double t = fma(u, srs, row[RL::FCS + qj]);
            F[qj] = fma(hu, is_v ? w : u, is_v ? 0.0 : gh2);
            G[qj] = fma(is_v ? hv : hu, w, is_v ? gh2 : 0.0) * crc;
            S[qj] = fma(is_v ? -gh2 : 0.0, srs, t * (is_v ? -hu : hv));
        }
    }
}

// eta projections of one xi node line: f[b] = sum_qj wP_b F, g[b] = sum_qj (wP'_b G + wP_b S)
template <int P, bool MOM>
__device__ __forceinline__ void line_project(const double (&F)[P + 1], const double (&G)[P + 1],
                                             const double (&S)[P + 1], double (&f)[P + 1],
                                             double (&g)[P + 1])
{
    n2m<P, 2>(F, f);
    if constexpr (!MOM)
        n2m<P, 3>(G, g);
    else
        n2m2<P, 3, 2>(G, S, g);
}

// Volume + source projection of variable v at the current row, streamed
// over pairs of xi node lines (qi, N-1-qi) so that the xi contraction also
// uses the even/odd split:
// vol[a][b] = sum_q (cx dphi/dxi F + cy dphi/deta G + cs phi S)[q]
template <int P, bool MOM>
__device__ __forceinline__ void volume(double (&vol)[P + 1][P + 1], int v, const double *sU,
                                       const double *row, int lane, const StageParams &kp)
{
    constexpr int N = P + 1;
    constexpr int H = N / 2;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) vol[a][b] = 0.0;
#if DG_VOL_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int ip = 0; ip < H; ++ip) {
        double f0[N], g0[N], f1[N], g1[N];
        {
            double F[N], G[N], S[N];
            node_physics<P, MOM>(v == 2, ip, sU, row, lane, kp, F, G, S);
            line_project<P, MOM>(F, G, S, f0, g0);
            node_physics<P, MOM>(v == 2, N - 1 - ip, sU, row, lane, kp, F, G, S);
            line_project<P, MOM>(F, G, S, f1, g1);
        }
        double pd[N], pp[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            pd[a] = WD(a, ip) * kp.inv_r_cx;   // F's 1/R * determ/bd_det_x folded in here
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
        node_physics<P, MOM>(v == 2, H, sU, row, lane, kp, F, G, S);
        line_project<P, MOM>(F, G, S, f, g);
#pragma unroll
        for (int b = 0; b < N; ++b)
#pragma unroll
            for (int a = 0; a < N; ++a)
                vol[a][b] = (a & 1) ? fma(WD(a, H) * kp.inv_r_cx, f[b], vol[a][b])
                                    : fma(WP(a, H), g[b], vol[a][b]);
    }
}

// Boundary lifts, inverse mass, stage combination and store for variable v.
// The mass block is applied column by column (one row of T from shared
// memory at a time) so that vol, c and u^n are the only tiles held.
// Uv / Yv point at this lane's element of the variable's strip block
// (mode stride 32 doubles: immediate offsets).
template <int P, bool HAS_U, bool HAS_Y2>
__device__ __forceinline__ unsigned finalize(double (&vol)[P + 1][P + 1], const double *cur,
                                             const double *Uv, const double *Av, double *Y2v, int v,
                                             const double *sFX, const double *sF0,
                                             const double *sFtop, const double *sFbot, bool has_top,
                                             bool has_bot, const double *row, int lane, bool owned,
                                             double *Yv, const StageParams &kp, double *Ypeer = nullptr,
                                             double *Ypeer2 = nullptr)
{
    constexpr int N = P + 1;
    using RL = RowLayout<P>;
    double un[N][N];
    if (HAS_U) {                       // u^n: plain loads (U may alias Y)
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) un[a][b] = Uv[(a * N + b) * kLanes];
    }
    double an[HAS_Y2 ? N : 1][HAS_Y2 ? N : 1];
    if constexpr (HAS_Y2) {            // second output's addend (may alias Y2)
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) an[a][b] = Av[(a * N + b) * kLanes];
    }
    constexpr int LDX = kLanes + 1;    // x-face columns: face f is the left face of lane f
    const int o = (v * N) * kLanes, ox = (v * N) * LDX;
#pragma unroll
    for (int b = 0; b < N; ++b) {
        // projected face lifts (bdy / bdx folded in by the face warps)
        const double l = lane == 0 ? sF0[v * N + b] : sFX[ox + b * LDX + lane];
        const double r = sFX[ox + b * LDX + lane + 1];
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
#pragma unroll
            for (int bb = 1; bb < N; ++bb) k = fma(tb[bb], vol[a][bb], k);
            double y = fma(kp.b, cur[(a * N + b) * kLanes + lane], (kp.g * (double)(2 * a + 1)) * k);
            if (HAS_U) y = fma(kp.a, un[a][b], y);
            if (owned) Yv[(a * N + b) * kLanes] = y;
            if (owned && Ypeer) Ypeer[(a * N + b) * kLanes] = y;   // fused halo exchange (NVLink store)
            if (owned && Ypeer2) Ypeer2[(a * N + b) * kLanes] = y;
            fexp = max(fexp, __double2hiint(y) & 0x7ff00000);
            if constexpr (HAS_Y2) {
                const double y2 = fma(kp.g2 * (double)(2 * a + 1), k, an[a][b]);
                if (owned) Y2v[(a * N + b) * kLanes] = y2;
            }
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

// Face warp: the neighbour elements' coefficients of row r (left eL =
// (32 s - 1) mod nx, right eR = (32 s + nvalid) mod nx; 3 vars x nphi each)
// gathered into shared memory with per-lane async copies, one phase ahead
// of their use, so no global latency sits on the face warp's critical path.
template <int P>
__device__ __forceinline__ void fetch_neighbours(const double *Xrow, int eL, int eR, double *sHB, int lane,
                                                 long long vstride)
{
    constexpr int NP = (P + 1) * (P + 1);
    for (int t = lane; t < 6 * NP; t += kLanes) {
        const int side = t / (3 * NP), r = t - side * 3 * NP, vv = r / NP, m = r - vv * NP;
        const int e = side ? eR : eL;
        cp_async8(sHB + t, Xrow + (size_t)vv * vstride + (size_t)(e >> 5) * NP * kLanes + m * kLanes + (e & 31));
    }
}

// Face warp: the traces of the strip's left border face for one row.
// Lanes 0..5 each build one trace: (side 0) R trace of the left neighbour
// element, from the gathered coefficients; (side 1) L trace of the strip's
// element 0, from the coefficient ring.  Also the L trace of the right
// neighbour (lanes 6..8), which the h warp needs for the last lane's right face.
template <int P>
__device__ __forceinline__ void border_traces(const double *sHB, const double *ring_slot, double *sHL,
                                              double *sE0, double *sHR, int lane)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    if (lane < 9) {
        const int side = lane / 3, v = lane - 3 * side;
        double c[N][N];
        if (side == 1) {
            const double *src = ring_slot + v * NP * kLanes;   // lane 0 of the ring tile
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) c[a][b] = src[(a * N + b) * kLanes];
        } else {
            const double *src = sHB + ((side == 0 ? 0 : 3) + v) * NP;
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) c[a][b] = src[a * N + b];
        }
        double t[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a) m2n<P, 0>(c[a], t[a]);
        const double sg = side == 0 ? 1.0 : -1.0;    // R trace: sum_a t, L trace: sum_a (-1)^a t
        double *dst = side == 0 ? sHL : side == 1 ? sE0 : sHR;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            double e = t[0][q], o = 0.0;
#pragma unroll
            for (int a = 2; a < N; a += 2) e += t[a][q];
            if constexpr (N > 1) {
                o = t[1][q];
#pragma unroll
                for (int a = 3; a < N; a += 2) o += t[a][q];
            }
            dst[v * N + q] = fma(sg, o, e);
        }
    }
    __syncwarp();
}

// bottom traces (eta = -1) of one row, all three variables, from its ring tile
template <int P>
__device__ __forceinline__ void bottom_traces(const double *ring_row, int lane, double (&bt)[3][P + 1])
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double cv[N][N];
        tile_read<P>(cv, ring_row + v * NP * kLanes, lane);
        ytrace<P, false>(cv, bt[v]);
    }
}

template <int P, bool HAS_U, bool HAS_Y2, bool EDGE>
__global__ void __launch_bounds__(kThreads, (P <= 2 ? 4 : P == 3 ? DG_MINB : 2)) stage_kernel(StageParams kp)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    constexpr unsigned kTileBytes = NP * kLanes * sizeof(double);   // one variable's row tile
    using SM = Smem<P>;
    using RL = RowLayout<P>;
    extern __shared__ double smem[];
    // fixed roles: warp w runs on sub-partition w of its SM, so every
    // sub-partition executes a single code path (better I-cache locality
    // than rotating roles, measured)
    const int role = threadIdx.x >> 5;
    const int v = role < kVarWarps ? role : 0;     // face warp borrows var 0's addressing
    const bool face_warp = role == kVarWarps;
    const int lane = threadIdx.x & 31;
    const int nx = kp.nx;
    const int strip = blockIdx.x;
    const int nvalid = min(kLanes, nx - strip * kLanes);
    const bool owned = lane < nvalid;
    const bool second = (int)blockIdx.y >= kp.nchunk1;   // one launch can cover two row ranges
    const int jb = second ? kp.j_begin2 + ((int)blockIdx.y - kp.nchunk1) * kp.rc : kp.j_begin + blockIdx.y * kp.rc;
    const int je = min(jb + kp.rc, second ? kp.j_end2 : kp.j_end);
    if (jb >= je) return;
    // fused halo exchange: an edge row first waits until the neighbour has
    // delivered this stage's halo row (its previous stage's edge row):
    // nstrip deliveries per completed stage, counted in our memory
    if constexpr (EDGE) {
        if (threadIdx.x == 0) {
            const unsigned long long need =
                ld_acquire_sys(kp.stage_ctr) * (unsigned long long)kp.nstrip * gridDim.z;
            const int g = kp.row0 + jb;
            if (jb == kp.band_lo && g > 0)
                while (ld_acquire_sys(kp.recv_count) < need) __nanosleep(64);
            if (jb == kp.band_hi - 1 && g + 1 < kp.ny)
                while (ld_acquire_sys(kp.recv_count + 1) < need) __nanosleep(64);
            asm volatile("fence.proxy.async.global;" ::: "memory");   // peer stores -> TMA reads
        }
        __syncthreads();
    }

    double *const ringS = smem + SM::XR0;          // [slot][var][mode][lane]
    double *const ring0 = ringS + v * NP * kLanes;   // this warp's variable
    double *sU = smem + SM::U;
    double *sXL = smem + SM::XL;
    double *sXR = smem + SM::XRT;
    double *sT = smem + SM::TT;
    double *sFX = smem + SM::FX;
    double *sFa = smem + SM::FY0;
    double *sFb = smem + SM::FY1;
    double *sRow = smem + SM::ROW;
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem + SM::MBAR);   // [slot][var]

    // this strip's block of variable v (row 0); per-lane element pointers
    const double *Xb = kp.X + (size_t)blockIdx.z * kp.zstride + (size_t)strip * NP * kLanes;
    const double *Xz = Xb + (size_t)v * kp.vstride;
    const double *Uz = kp.U ? kp.U + (size_t)blockIdx.z * kp.zstride + (size_t)strip * NP * kLanes +
                                  (size_t)v * kp.vstride + lane
                            : nullptr;
    const size_t lane_off = (size_t)blockIdx.z * kp.zstride + (size_t)strip * NP * kLanes +
                            (size_t)v * kp.vstride + lane;
    double *Yz = kp.Y + lane_off;
    const double *Az = HAS_Y2 ? kp.A + lane_off : nullptr;
    double *Y2z = HAS_Y2 ? kp.Y2 + lane_off : nullptr;
    const bool chk = (v == 0) && !face_warp;
    unsigned bad = 0;

    // rows whose coefficients exist: local r with global row0+r in [0, ny)
    const int r_last = min(kp.nrows - 1, kp.ny - 1 - kp.row0);
    const int last_fetch = min(je, r_last);        // rows jb..last_fetch stream through the ring

    if (threadIdx.x == 0) {
        for (int k = 0; k < 6; ++k) mbar_init(mbar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // prologue: the var warps' elected lanes start streaming rows jb, jb+1
    if (!face_warp && lane == 0) {
        tma_row(ring0, Xz + (size_t)jb * kp.rstride, kTileBytes, mbar + v);
        if (jb + 1 <= last_fetch)
            tma_row(ring0 + SM::TILE, Xz + (size_t)(jb + 1) * kp.rstride, kTileBytes, mbar + 3 + v);
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
    if (below && !face_warp) {
        const double *src = Xz + (size_t)(jb - 1) * kp.rstride + lane;
        double c[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) c[a][b] = __ldg(src + (a * N + b) * kLanes);
        double tt[N];
        ytrace<P, true>(c, tt);
#pragma unroll
        for (int q = 0; q < N; ++q) sT[(v * N + q) * kLanes + lane] = tt[q];
    }
    if (!face_warp) mbar_wait(mbar + v, 0);        // row jb landed (this variable)
    // periodic neighbours of the strip's border elements
    const int eL = (strip * kLanes - 1 + nx) % nx;
    const int eR = (strip * kLanes + nvalid) % nx;
    if (face_warp) {   // the first row's neighbour coefficients (used after the pre-iteration's face)
        fetch_neighbours<P>(kp.X + (size_t)blockIdx.z * kp.zstride + (size_t)jb * kp.rstride, eL, eR,
                            smem + SM::HB, lane, kp.vstride);
        cp_commit();
    }
    __syncthreads();                               // prologue barrier A
#ifdef DG_TIMING
    unsigned tacc[6] = {0, 0, 0, 0, 0, 0};
#endif

    if (face_warp) {
        // Face warp.  Iteration `it` (from the pre-iteration jb-1): job 0 =
        // the y-face above row it (the bottom face of row jb in the
        // pre-iteration), job 1 = the strip's left border x-face of row it+1,
        // computed in the window between the rows' barriers 2 and 1.
        double *fa = sFa, *fb = sFb;
        for (int it = jb - 1; it < je; ++it) {
            const int k = it - jb;
            const bool pre = it < jb;
            TSTAMP(a);
            if (!pre) __syncthreads();                 // barrier 1 of row it
            TSTAMP(b);
            if (!pre) {
                // async gathers, consumed after barrier 2: the next row's neighbour
                // coefficients and the table of row it+2 (its slot held row it-1)
                if (it + 1 < je)
                    fetch_neighbours<P>(kp.X + (size_t)blockIdx.z * kp.zstride + (size_t)(it + 1) * kp.rstride,
                                        eL, eR, smem + SM::HB, lane, kp.vstride);
                if (it + 2 <= je && kp.row0 + it + 2 < kp.ny) {
                    double *dst = sRow + ((k + 2) % 3) * RL::STRIDE;
                    const double *src = kp.rowtab + (size_t)(kp.row0 + it + 2) * RL::STRIDE;
                    for (int idx = lane; idx < RL::STRIDE; idx += kLanes) cp_async8(dst + idx, src + idx);
                }
                cp_commit();
            }
            const double *next_tile = ringS + ((k + 1) & 1) * SM::TILE;   // X(it+1)
            if (it + 1 <= last_fetch) {
                double bt[3][N];
                bottom_traces<P>(next_tile, lane, bt);
#pragma unroll
                for (int q = 0; q < N; ++q) bad |= owned && !(bt[0][q] > 0.0);
                const bool face = pre ? below : (kp.row0 + it + 1 < kp.ny);
                if (face) {
                    // bottom traces staged in the face's output slot, read back by the call
                    const int dst = (int)((pre ? fb : fa) - smem);
#pragma unroll
                    for (int vv = 0; vv < 3; ++vv)
#pragma unroll
                        for (int q = 0; q < N; ++q) smem[dst + (vv * N + q) * kLanes + lane] = bt[vv][q];
                    const double *above = sRow + ((k + 1) % 3) * RL::STRIDE;
                    face_flux_call<P>(SM::TT, kLanes, lane, dst, kLanes, lane, dst, kLanes, lane,
                                      FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r,
                                               kp.alpha_mode, 1, above[RL::CRB], above[RL::COSB], alpha_y,
                                               kp.bdx});
                }
            }
            TSTAMP(c);
            __syncthreads();                           // barrier 2 of row it (prologue barrier B)
            TSTAMP(d);
            if (!pre) {
                double *t = fa;
                fa = fb;
                fb = t;
            }
            cp_wait_all();                             // gathers of this row's phase B (and row tables)
            __syncwarp();
            if (it + 1 < je) {
                border_traces<P>(smem + SM::HB, next_tile, smem + SM::HL, smem + SM::E0, smem + SM::HR, lane);
                // every lane computes the same face (uniform control flow, identical stores)
                face_flux_call<P>(SM::HL, 1, 0, SM::E0, 1, 0, SM::F0 + ((k + 1) & 1) * 3 * N, 1, 0,
                                  FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r,
                                           kp.alpha_mode, 0, 0.0, 0.0, alpha_x, kp.bdy});
            }
            TSTAMP(e);
            if (!pre) {
                TACC(2, tkb - tka);   // barrier 1 wait
                TACC(3, tkc - tkb);   // y-face
                TACC(4, tkd - tkc);   // barrier 2 wait
                TACC(5, tke - tkd);   // border face (next row)
            }
        }
    } else {
        __syncthreads();                           // prologue barrier B
        for (int jl = jb; jl < je; ++jl) {
            const int k = jl - jb;
            const int slot = k & 1;
            double *const cur = ring0 + slot * SM::TILE;
            const int jg = kp.row0 + jl;
            const bool has_top = jg + 1 < kp.ny;
            const bool has_bot = jg > 0;
            const double *row = sRow + (k % 3) * RL::STRIDE;
            TSTAMP(s);

            // warm L2 for this row's u^n and for row jl+2 (copied in after finalize)
            if (lane == 0) {
                if (HAS_U) prefetch_l2_bulk(Uz - lane + (size_t)jl * kp.rstride, kTileBytes);
                if (jl + 2 <= last_fetch) prefetch_l2_bulk(Xz + (size_t)(jl + 2) * kp.rstride, kTileBytes);
            }
            {
                double c[N][N];
                tile_read<P>(c, cur, lane);            // X(jl)
                bad |= owned & eval_row<P>(c, sU + v * NP * kLanes, sXL + v * N * kLanes,
                                           sXR + v * N * kLanes, sT + v * N * kLanes, lane, chk);
            }
            TSTAMP(0);
            if (jl + 1 <= last_fetch) mbar_wait(mbar + (slot ^ 1) * 3 + v, ((k + 1) >> 1) & 1);   // X(jl+1)
            TSTAMP(1);
            __syncthreads();                           // barrier 1
            TSTAMP(2);

            if (v == 0) {
                // the h warp has the lightest volume work: it takes the x-faces 1..32
                // (right face of every lane; the last valid lane's neighbour is the halo)
                const bool last = lane == nvalid - 1;
                face_flux_call<P>(SM::XRT, kLanes, lane, last ? SM::HR : SM::XL, last ? 1 : kLanes,
                                  last ? 0 : min(lane + 1, kLanes - 1), SM::FX, kLanes + 1, lane + 1,
                                  FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r,
                                           kp.alpha_mode, 0, 0.0, 0.0, alpha_x, kp.bdy});
            }
            double vol[N][N];
            if (v == 0)
                volume<P, false>(vol, v, sU, row, lane, kp);
            else
                volume<P, true>(vol, v, sU, row, lane, kp);
            TSTAMP(3);
            __syncthreads();                           // barrier 2
            TSTAMP(4);
            const size_t roff = (size_t)jl * kp.rstride;
            // fused exchange: an edge row is also stored into the neighbour's
            // halo row (south: band_lo, north: band_hi-1; a one-row band feeds both)
            double *Ypeer = nullptr, *Ypeer2 = nullptr;
            if constexpr (EDGE) {
                const size_t off = (size_t)strip * NP * kLanes + (size_t)v * kp.vstride + lane;
                if (jl == kp.band_lo && kp.peer_row[0])
                    Ypeer = kp.peer_row[0] + (size_t)blockIdx.z * kp.peer_zstride[0] + off;
                if (jl == kp.band_hi - 1 && kp.peer_row[1])
                    Ypeer2 = kp.peer_row[1] + (size_t)blockIdx.z * kp.peer_zstride[1] + off;
            }
            bad |= finalize<P, HAS_U, HAS_Y2>(vol, cur, HAS_U ? Uz + roff : nullptr,
                                              HAS_Y2 ? Az + roff : nullptr, HAS_Y2 ? Y2z + roff : nullptr, v, sFX,
                                      smem + SM::F0 + slot * 3 * N, sFa, sFb, has_top, has_bot, row, lane,
                                      owned, Yz + roff, kp, Ypeer, Ypeer2);
            // X(jl) is consumed: stream row jl+2 into its slot (L2-warm by now)
            __syncwarp();
            if (lane == 0 && jl + 2 <= last_fetch) {
                fence_proxy_async();
                tma_row(cur, Xz + (size_t)(jl + 2) * kp.rstride, kTileBytes, mbar + slot * 3 + v);
            }
            TSTAMP(5);
            TACC(0, tk0 - tks);   // phase A work (eval)
            TACC(1, tk1 - tk0);   // wait for X(jl+1)
            TACC(2, tk2 - tk1);   // barrier 1
            TACC(3, tk3 - tk2);   // phase B work
            TACC(4, tk4 - tk3);   // barrier 2
            TACC(5, tk5 - tk4);   // phase C work (finalize)
            double *tmp = sFa;
            sFa = sFb;
            sFb = tmp;
        }
    }

#ifdef DG_TIMING
    if (lane == 0) {
        for (int q = 0; q < 6; ++q) atomicAdd(&g_timing[role][q], (unsigned long long)tacc[q]);
        atomicAdd(&g_timing[role][6], (unsigned long long)(je - jb));
    }
#endif
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) {
        atomicOr(kp.status, bad);
        atomicMin(kp.first_tag, kp.tag);
    }
    if constexpr (EDGE) {
        // publish the edge rows stored into the neighbours' halos, then count
        // this CTA; the last one advances the band's stage counter
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            for (int side = 0; side < 2; ++side) {
                const int r = side == 0 ? kp.band_lo : kp.band_hi - 1;
                if (kp.peer_count[side] && jb <= r && r < je) atomicAdd_system(kp.peer_count[side], 1ull);
            }
            const unsigned total = gridDim.x * gridDim.y * gridDim.z;
            if (atomicAdd(kp.stage_ctr + 1, 1ull) == total - 1) {
                kp.stage_ctr[1] = 0;
                __threadfence();
                atomicAdd(kp.stage_ctr, 1ull);
            }
        }
    }
}

#undef LEG
#undef WP
#undef WD

}  // namespace dgswe
