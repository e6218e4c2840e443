// dgswe_kernels.cuh -- fused fp64 DG shallow-water stage kernel for sm_100a.
//
// HBM layout of a state (strip-blocked structure of arrays):
//   [nz][row][var 3][strip][mode nphi][32 elements]
// A strip is 32 consecutive longitude elements (the last one zero-padded),
// so one variable's row tile of a strip is a single contiguous block of
// nphi * 256 bytes: it moves with ONE TMA bulk copy (cp.async.bulk +
// mbarrier), its L2 prefetch is one bulk-prefetch instruction, and every
// per-lane load/store inside it is an immediate offset from one base.
// Inside a step the slot of mode (a, b) holds the value at Gauss node
// (i, j) instead (convert_kernel; DESIGN.md section 3 "Nodal form").
//
// One CTA = 4 warps x 32 lanes on one strip: warp v < 3 owns variable v in
// {h, hu, hv}; warp 0 also evaluates the row's x-faces 1..32 and warp 3
// (the face warp) the y-face above the row, the strip's two halo traces and
// its left border face 0.  Lane l owns element 32*strip + l.  The CTA
// marches north through a chunk of latitude rows.
//
// Per row, per variable and lane (n = p+1; constant tables in __constant__):
//   1. traces L/R/T (and B of the next row) of the nodal tile: one n-point
//      dot product each                               (dg.py:348-357)
//   2. pointwise flux / source physics at the nodes    (models.py:161-252)
//   3. Rusanov fluxes with local alpha                 (dg.py:92-119,385-453)
//   4. weak derivatives of the fluxes (W^-1 D^T W per direction), source,
//      face lifts, the diagonal nodal mass and the fused RK stage update
//      (dg.py:455-502, timestep.py:132-167)
//
// Kernel variants (template bitmask F, see kHasU ... kOrog): the stage
// combination's u^n term, classical RK4's second output, the band edge rows
// of the fused halo exchange, modal in/out states (the reference's own
// coefficients: every tile is converted to the Gauss nodes in shared memory
// as it lands and the output back to modes in registers -- the single-launch
// form of assemble_rhs and the modal stage entry points) and the orography
// source of Williamson TC5 (-g h grad b, not in the reference: SPEC.md:157).
// At p = 0 the plain nodal stages run on the barrier-free kernel of
// dgswe_lo.cuh instead (same arithmetic, identical bits).
//
// Floating point: FMA contraction, refined MUFU reciprocals and a different
// summation order than the reference; results agree with the reference's
// exact-order oracle to ~1e-15 relative per step (tests/test_gpu_parity.py).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "dgswe_params.h"

namespace dgswe {

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Resident CTAs per SM the stage kernels are register-capped for: p <= 3
// at 128 registers (4 CTAs), p >= 4 at 2 CTAs; a rolled volume loop (row-
// local terms through shared memory) for p >= 2.
template <int P>
__host__ __device__ constexpr int min_blocks() { return P <= 3 ? 4 : 2; }
// per variant: the plain nodal stages (the SSPRK3 path) at p = 1 / 2 fit 6 /
// 5 CTAs at 80 / 96 registers without spills (+9% / +1.8%; the modal, band
// and orography variants would spill there); at p = 3 the orography and
// RK4-accumulator variants run 3 CTAs at 168 registers (the orography
// tiles' shared memory leaves no room for a fourth; RK4's second output
// spilled at 128); p = 6 fits one CTA per SM
template <int P, int F>
__host__ __device__ constexpr int min_blocks_f()
{
    return (F & ~kHasU) == 0 && P == 1   ? 6
           : (F & ~kHasU) == 0 && P == 2 ? 5
           : P == 3 && (F & (kOrog | kHasY2)) ? 3
           : P >= 6                      ? 1
                                         : min_blocks<P>();
}
template <int P>
__host__ __device__ constexpr bool vol_rolled() { return P >= 2; }
// u^n loaded into registers before barrier 2 (in flight during the wait) up
// to p = 5 except with RK4's second output (its addend needs those
// registers: it spilled); at p = 6 the 49 doubles next to the 49
// accumulators would.  Otherwise finalize loads u^n before its first store.
template <int P, int F>
__host__ __device__ constexpr bool early_u() { return P <= 5 && (F & kHasY2) == 0; }


// DG_TIMING builds record per-role phase durations (clock cycles) of every
// row: [role][A work, barrier-1 wait, B work, barrier-2 wait, C work, rows]
#ifdef DG_TIMING
namespace {
__device__ unsigned long long g_timing[4][7];
}
#define TSTAMP(k)                                                                  \
    unsigned tk##k;                                                                \
    asm volatile("mov.u32 %0, %%clock;" : "=r"(tk##k)::"memory")
#define TACC(i, d) tacc[i] += (d)
#else
#define TSTAMP(k)
#define TACC(i, d)
#endif

// internal linkage: every degree's translation unit (deg_p*.cu) owns its
// copy, uploaded by that unit's dgswe_create path
namespace {
__constant__ NodTab c_nod[kMaxP + 1];
}

#define LEG(a, q) c_nod[P].leg[a][q]
#define WP(a, q) c_nod[P].wp[a][q]

// Modal <-> nodal change of basis of one element tile in registers, in the
// operation order of convert_kernel (so both give identical bits):
//   nodal u[i][j] = sum_a P_a(x_i) sum_b P_b(x_j) c[a][b]
//   modal c[a][b] = (2a+1)(2b+1)/4 sum_i w_i P_a(x_i) sum_j w_j P_b(x_j) u[i][j]
template <int P>
__device__ __forceinline__ void to_nodal(double (&x)[P + 1][P + 1])
{
    constexpr int N = P + 1;
    double t[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int q = 0; q < N; ++q) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(LEG(b, q), x[a][b], s);
            t[a][q] = s;
        }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
        for (int r = 0; r < N; ++r) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < N; ++a) s = fma(LEG(a, q), t[a][r], s);
            x[q][r] = s;
        }
}

template <int P>
__device__ __forceinline__ void to_modal(double (&x)[P + 1][P + 1])
{
    constexpr int N = P + 1;
    double t[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int q = 0; q < N; ++q) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(WP(q, b), x[a][b], s);
            t[a][q] = s;
        }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
        for (int r = 0; r < N; ++r) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < N; ++a) s = fma(WP(q, a), t[a][r], s);
            x[q][r] = s * (0.25 * (double)((2 * q + 1) * (2 * r + 1)));
        }
}

// value at xi = -1 (LO) or +1 of the nodal line x
template <int P, bool LO>
__device__ __forceinline__ double line_trace(const double (&x)[P + 1])
{
    constexpr int N = P + 1;
    double s = c_nod[P].lm[LO ? 0 : N - 1] * x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) s = fma(c_nod[P].lm[LO ? i : N - 1 - i], x[i], s);
    return s;
}


template <int P>
struct Smem {
    static constexpr int N = P + 1;
    static constexpr int NP = N * N;
    static constexpr int TILE = 3 * NP * kLanes;         // one row of coefficients, all vars
    static constexpr int LD = kLanes + 1;                // leading dimension of trace / flux arrays:
                                                         // columns 0..31 = lanes, column 32 = a strip-
                                                         // border value (halo traces, border face flux)
    static constexpr int TR = 3 * N * LD;                // one trace / face-flux set [3][N][LD]
    // offsets in doubles
    static constexpr int XR0 = 0;                        // coefficient ring slot 0 [var][mode][lane]
    static constexpr int XR1 = XR0 + TILE;               // slot 1
    static constexpr int E = XR1 + TILE;                 // row-local volume terms [3][NP][32] (rolled volume)
    static constexpr int XL = E + (vol_rolled<P>() ? TILE : 0);   // L traces [3][N][LD]
    static constexpr int XRT = XL + TR;                  // R traces
    static constexpr int TT = XRT + TR;                  // top traces of current row
    static constexpr int FX = TT + TR;                   // x-face fluxes, column c = LEFT face of lane c
                                                         // (column 0: the strip's border face)
    static constexpr int FY0 = FX + TR;                  // y-face flux buffers
    static constexpr int FY1 = FY0 + TR;
    // column 32 of those arrays (face warp): halo / border values
    static constexpr int HR = XL + kLanes;               // right neighbour's L trace (x-face of the last lane)
    static constexpr int HL = XRT + kLanes;              // left neighbour's R trace (border face "in")
    static constexpr int E0 = TT + kLanes;               // element 0's L trace (border face "out")
    static constexpr int F0T = FY0 + kLanes;             // next row's border face flux (copied to FX
                                                         // column 0 after that row's barrier 1)
    static constexpr int HB = FY1 + TR;                  // next row's neighbour coefficients [2][3][NP]
    static constexpr int ROW = HB + 6 * NP;              // row-table ring, 3 rows
    static constexpr int MBAR = ROW + 3 * RowLayout<P>::SSTRIDE;  // 6 mbarriers [slot][var]
    static constexpr int TOTAL = MBAR + 6;
    static constexpr int OB = (TOTAL + 1) & ~1;          // orography tiles [slot][hu, hv][NP][32] (kOrog)
    static constexpr int TOTAL_OROG = OB + 4 * NP * kLanes;
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

// x >= y for y > 0 and x > 0 on the integer pipe (signed 64-bit order of
// the bit patterns; differs from the fp64 compare only for NaN x, which the
// positivity checks flag anyway)
__device__ __forceinline__ bool ge_pos(double x, double y)
{
    return __double_as_longlong(x) >= __double_as_longlong(y);
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

// 1/hf with hf = max(h, floor) (models.py:161-166) and sqrt(max(h, 0)) --
// the celerity is sqrt(g) times it (models.py:254-258), which the face
// fuses explicitly into |w| + c -- from ONE rsqrt of h: below the floor 1/hf
// is the constant 1/floor.  h <= 0 or NaN at any trace node sets the
// positivity status bit, which discards the whole step (PositivityError,
// dg.py:359-372), so the root there only has to stay finite (it is <= 0
// instead of the reference's 0; the rsqrt argument is clamped to DBL_MIN).
__device__ __forceinline__ void inv_and_sqrt(double h, double h_floor, double inv_floor, double &r, double &sh)
{
    const double y = rsqrt64(max_pos(h, 2.2250738585072014e-308));
    r = ge_pos(h, h_floor) ? y * y : inv_floor;   // branches compared on the integer pipe
    sh = h * y;
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

__device__ __forceinline__ double *smem_base()
{
    extern __shared__ double smem[];
    return smem;
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

// bottom (eta = -1, LO) or top trace of a nodal tile u[i][j]: per xi node i
template <int P, bool LO>
__device__ __forceinline__ void ytrace(const double (&u)[P + 1][P + 1], double (&tr)[P + 1])
{
#pragma unroll
    for (int i = 0; i < P + 1; ++i) tr[i] = line_trace<P, LO>(u[i]);
}

// left (xi = -1, LO) or right trace of a nodal tile: per eta node j
template <int P, bool LO>
__device__ __forceinline__ void xtrace(const double (&u)[P + 1][P + 1], double (&tr)[P + 1])
{
    constexpr int N = P + 1;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double col[N];
#pragma unroll
        for (int i = 0; i < N; ++i) col[i] = u[i][j];
        tr[j] = line_trace<P, LO>(col);
    }
}

// L/R/T traces of one variable's nodal tile -> shared memory (+ positivity
// of the h nodes and traces when `check`)
template <int P>
__device__ __forceinline__ unsigned traces_row(const double (&u)[P + 1][P + 1], double *sXL, double *sXR,
                                               double *sT, int lane, bool check)
{
    constexpr int N = P + 1;
    unsigned bad = 0;
    double l[N], r[N], t[N];
    xtrace<P, true>(u, l);
    xtrace<P, false>(u, r);
    ytrace<P, false>(u, t);
#pragma unroll
    for (int q = 0; q < N; ++q) {
        sXL[q * Smem<P>::LD + lane] = l[q];
        sXR[q * Smem<P>::LD + lane] = r[q];
        sT[q * Smem<P>::LD + lane] = t[q];
    }
    if (check) {
#pragma unroll
        for (int q = 0; q < N; ++q) bad |= !(l[q] > 0.0) | !(r[q] > 0.0) | !(t[q] > 0.0);
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) bad |= !(u[i][j] > 0.0);
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
// The flux arithmetic of one face from register traces (h, normal and
// tangential momentum on the "in" / "out" side) into fh / fn / ft: shared
// by the shared-memory face routine below and the low-order kernel
// (dgswe_lo.cuh), so both give identical bits.
// the face arithmetic from given reciprocals rin / rout and square roots
// cin / cout of the two sides' h traces (inv_and_sqrt of hI / hO; the
// celerity is sqrt(g) times it, fused explicitly): the low-order kernel
// computes them once per element and shares them
template <int P>
__device__ __forceinline__ void face_core_rc(const double (&hI)[P + 1], const double (&nI)[P + 1],
                                             const double (&tI)[P + 1], const double (&rin)[P + 1],
                                             const double (&cin)[P + 1], const double (&hO)[P + 1],
                                             const double (&nO)[P + 1], const double (&tO)[P + 1],
                                             const double (&rout)[P + 1], const double (&cout)[P + 1],
                                             const FaceArgs &fa, double (&fh)[P + 1], double (&fn)[P + 1],
                                             double (&ft)[P + 1])
{
    constexpr int N = P + 1;
    double am[N];
#pragma unroll
    for (int k = 0; k < N; ++k)
        am[k] = max_nn(fma(fa.sqrt_g, cin[k], fabs(nI[k] * rin[k])), fma(fa.sqrt_g, cout[k], fabs(nO[k] * rout[k])));
#pragma unroll
    for (int w = 1; w < N; w *= 2)
#pragma unroll
        for (int k = 0; k + w < N; k += 2 * w) am[k] = max_nn(am[k], am[k + w]);
    double alpha = am[0] * fa.inv_r;
    if (fa.dir == 1) alpha *= fa.cos_e;
    if (fa.alpha_mode != 0) alpha = fa.alpha_glob;
    const double ha = (0.5 * fa.scale) * alpha;
    const double hs = (0.5 * fa.scale) * (fa.dir == 0 ? fa.inv_r : fa.cr_e);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double gi = hI[k] * hI[k] * fa.half_g, go = hO[k] * hO[k] * fa.half_g;
        const double wi = nI[k] * rin[k], wo = nO[k] * rout[k];
        const double fni = fma(nI[k], wi, gi), fno = fma(nO[k], wo, go);   // normal: m w + g h^2/2
        // tangential: m_t w on both sides, summed with an explicit fma (a plain
        // a*b + c*d lets the compiler pick which product it fuses, which can
        // differ between inlining contexts: one rounding apart)
        const double ft_sum = fma(tI[k], wi, tO[k] * wo);
        fh[k] = fma(hs, nI[k] + nO[k], -ha * (hO[k] - hI[k]));
        fn[k] = fma(hs, fni + fno, -ha * (nO[k] - nI[k]));
        ft[k] = fma(hs, ft_sum, -ha * (tO[k] - tI[k]));
    }
}

template <int P>
__device__ __forceinline__ void face_core(const double (&hI)[P + 1], const double (&nI)[P + 1],
                                          const double (&tI)[P + 1], const double (&hO)[P + 1],
                                          const double (&nO)[P + 1], const double (&tO)[P + 1], const FaceArgs &fa,
                                          double (&fh)[P + 1], double (&fn)[P + 1], double (&ft)[P + 1])
{
    constexpr int N = P + 1;
    double rin[N], rout[N], cin[N], cout[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        inv_and_sqrt(hI[k], fa.h_floor, fa.inv_floor, rin[k], cin[k]);
        inv_and_sqrt(hO[k], fa.h_floor, fa.inv_floor, rout[k], cout[k]);
    }
    face_core_rc<P>(hI, nI, tI, rin, cin, hO, nO, tO, rout, cout, fa, fh, fn, ft);
}

template <int P>
__device__ __forceinline__ void face_flux_body(int in, int out, int dst, FaceArgs fa)
{
    constexpr int N = P + 1;
    constexpr int LD = Smem<P>::LD;
    extern __shared__ double smem[];
    // variables by role: h, the normal momentum (hu across an x-face, hv
    // across a y-face) and the tangential one, addressed through the
    // runtime direction instead of per-node selects
    const int vn = 1 + fa.dir, vt = 2 - fa.dir;
    double hI[N], nI[N], tI[N], hO[N], nO[N], tO[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        hI[k] = smem[in + k * LD];
        nI[k] = smem[in + (vn * N + k) * LD];
        tI[k] = smem[in + (vt * N + k) * LD];
        hO[k] = smem[out + k * LD];
        nO[k] = smem[out + (vn * N + k) * LD];
        tO[k] = smem[out + (vt * N + k) * LD];
    }
    double fh[N], fn[N], ft[N];
    face_core<P>(hI, nI, tI, hO, nO, tO, fa, fh, fn, ft);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        smem[dst + k * LD] = fh[k];
        smem[dst + (vn * N + k) * LD] = fn[k];
        smem[dst + (vt * N + k) * LD] = ft[k];
    }
}

template <int P>
__device__ __noinline__ void face_flux_noinline(int in, int out, int dst, FaceArgs fa)
{
    face_flux_body<P>(in, out, dst, fa);
}

// p >= 2: the shared non-inlined copy; p <= 1: inlined (the face work is a
// large share of a low-order element and the call's overhead shows, measured)
template <int P>
__device__ __forceinline__ void face_flux_call(int in, int out, int dst, FaceArgs fa)
{
    if constexpr (P <= 1)
        face_flux_body<P>(in, out, dst, fa);
    else
        face_flux_noinline<P>(in, out, dst, fa);
}


// per-row factors of the physics, read from the staged row table or held
// in registers across a row's node loop
template <int P>
struct RowRef {
    const double *p;
    __device__ __forceinline__ double crc(int q) const { return p[RowLayout<P>::CRC + q]; }
    __device__ __forceinline__ double srs(int q) const { return p[RowLayout<P>::SRS + q]; }
    __device__ __forceinline__ double fcs(int q) const { return p[RowLayout<P>::FCS + q]; }
};
template <int P>
struct RowRegs {
    double c[P + 1], s[P + 1], f[P + 1];
    __device__ __forceinline__ RowRegs(const double *p)
    {
#pragma unroll
        for (int q = 0; q < P + 1; ++q) {
            c[q] = p[RowLayout<P>::CRC + q];
            s[q] = p[RowLayout<P>::SRS + q];
            f[q] = p[RowLayout<P>::FCS + q];
        }
    }
    __device__ __forceinline__ double crc(int q) const { return c[q]; }
    __device__ __forceinline__ double srs(int q) const { return s[q]; }
    __device__ __forceinline__ double fcs(int q) const { return f[q]; }
};

// Pointwise flux / source at the N nodes (qi, qj), qj = 0..N-1
// (models.py:161-252): F = x-flux (its cx/R goes into the xi weights),
// G = y-flux * cy cos/R, S = source, for the equation of KIND:
//   0 h:  F = hu,              G = hv cos/R,               S = 0
//   1 hu: F = hu u + g h^2/2,  G = hu w cos/R,             S = t hv
//   2 hv: F = hu w,            G = (hv w + g h^2/2) cos/R, S = -(g h^2/2 sin/R + t hu)
//   3:    hu or hv by the uniform flag is_v, one branch-free code path
//         (the unrolled volume, where a second copy would cost I-cache)
// with u = hu/hf, w = hv/hf, t = u sin/R + 2 Omega sin cos.  With OROG the
// momentum sources gain h * B (B = this equation's orography factor at the
// node, the warp's staged tile sB: -(g/R) db/dlambda resp. -(g cos/R)
// db/dtheta, determ folded in).
template <int P, int KIND, bool OROG, typename RT, int STRIDE = kLanes>
__device__ __forceinline__ void node_physics(bool is_v, int qi, const double *sU, const RT &row, int lane,
                                             const StageParams &kp, const double *sB, double (&F)[P + 1],
                                             double (&G)[P + 1], double (&S)[P + 1])
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
#pragma unroll
    for (int qj = 0; qj < N; ++qj) {
        const int q = qi * N + qj;
        const double hu = sU[(1 * NP + q) * STRIDE + lane];
        const double hv = sU[(2 * NP + q) * STRIDE + lane];
        const double crc = row.crc(qj);
        if constexpr (KIND == 0) {
            F[qj] = hu;
            G[qj] = hv * crc;
            S[qj] = 0.0;
        } else {
            const double h = sU[(0 * NP + q) * STRIDE + lane];
            // 1/max(h, floor) as rcp(h) + select: the reciprocal starts at once
            const double r = ge_pos(h, kp.h_floor) ? rcp64(h) : kp.inv_floor;
            const double gh2 = h * h * kp.half_g;
            const double u = hu * r, w = hv * r;
            const double srs = row.srs(qj);
            const double t = fma(u, srs, row.fcs(qj));
            if constexpr (KIND == 1) {
                F[qj] = fma(hu, u, gh2);
                G[qj] = (hu * w) * crc;
                S[qj] = t * hv;
            } else if constexpr (KIND == 2) {
                F[qj] = hu * w;
                G[qj] = fma(hv, w, gh2) * crc;
                S[qj] = fma(-gh2, srs, -(t * hu));
            } else {
                F[qj] = fma(hu, is_v ? w : u, is_v ? 0.0 : gh2);
                G[qj] = fma(is_v ? hv : hu, w, is_v ? gh2 : 0.0) * crc;
                S[qj] = fma(is_v ? -gh2 : 0.0, srs, t * (is_v ? -hu : hv));
            }
            if constexpr (OROG) {
                if (sB) S[qj] = fma(h, sB[q * STRIDE + lane], S[qj]);   // null: an all-zero tile
            }
        }
    }
}

// Volume + source terms of variable v at the row's nodes, nodal form:
//   acc[i][j] = sum_k Dx[i][k] F[k][j] + sum_k dh[j][k] G[i][k] + S[i][j]
// with Dx = (1/R) (determ/bd_det_x) dh (kernel parameter), G carrying its
// cos/R * determ/bd_det_y factor and S its determ factor (row table); the
// common 1/(determ cos_j) is applied in finalize.  Node row i (fixed xi
// node) is evaluated at once: its G/S terms land in acc[i][.], its F
// scatters into every acc[.][j].
template <int P, bool MOM, bool OROG, int STRIDE = kLanes>
__device__ __forceinline__ void volume(double (&acc)[P + 1][P + 1], int v, const double *sU,
                                       const double *row, int lane, const StageParams &kp, const double *sB)
{
    constexpr int N = P + 1;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double F[N], G[N], S[N];
        node_physics<P, MOM ? 3 : 0, OROG, RowRef<P>, STRIDE>(v == 2, i, sU, RowRef<P>{row}, lane, kp, sB, F, G, S);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double e = MOM ? S[j] : 0.0;
            if (i > 0) e += acc[i][j];
#pragma unroll
            for (int k = 0; k < N; ++k) e = fma(c_nod[P].dh[j][k], G[k], e);
            acc[i][j] = e;
        }
#pragma unroll
        for (int ii = 0; ii < N; ++ii)
#pragma unroll
            for (int j = 0; j < N; ++j)
                acc[ii][j] = (i == 0 && ii > 0) ? kp.dx[ii][i] * F[j] : fma(kp.dx[ii][i], F[j], acc[ii][j]);
    }
}

// Same terms with the loop over node rows kept rolled (a quarter of the
// code): the row-local G/S terms of row i go to shared memory sE (this
// warp's [NP][32] block) and are added at the end; F still scatters into
// the register tile through the i-th column of Dx.  Every variable warp
// forms its own row-local term (the h warp's: G = hv cos/R); the momentum
// warps' physics is the longest phase-B work, so nothing moves onto them.
template <int P, int KIND, bool OROG>
__device__ __forceinline__ void volume_rolled(double (&acc)[P + 1][P + 1], int v, const double *sU,
                                              const double *row, int lane, const StageParams &kp, double *sE,
                                              const double *sB)
{
    constexpr int N = P + 1;
#pragma unroll
    for (int ii = 0; ii < N; ++ii)
#pragma unroll
        for (int j = 0; j < N; ++j) acc[ii][j] = 0.0;
    // the row's physics factors in registers across the loop (p = 6: read
    // from the shared row table, their 42 registers would spill)
    using RowT = typename std::conditional<(P >= 6), RowRef<P>, RowRegs<P>>::type;
    const RowT rr{row};
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        double F[N], G[N], S[N];
        node_physics<P, KIND, OROG>(false, i, sU, rr, lane, kp, sB, F, G, S);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double e = S[j];
#pragma unroll
            for (int k = 0; k < N; ++k) e = fma(c_nod[P].dh[j][k], G[k], e);
            sE[(i * N + j) * kLanes + lane] = e;
        }
#pragma unroll
        for (int ii = 0; ii < N; ++ii) {
            const double d = kp.dx[ii][i];
#pragma unroll
            for (int j = 0; j < N; ++j) acc[ii][j] = fma(d, F[j], acc[ii][j]);
        }
    }
    // the row-local terms are this warp's own: add them now, before barrier
    // 2, so finalize starts on the faces (their shared-memory latency is
    // spent while the warp would wait at the barrier anyway; every lane
    // reads only its own column)
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) acc[i][j] += sE[(i * N + j) * kLanes + lane];
}

// Boundary lifts, diagonal mass, stage combination and store for variable v.
// Face values are scale * f* at the face's nodes (bd_det folded in by the
// face warps); x lifts run along xi with mu, y lifts along eta.
// `un` holds u^n (HAS_U); Yv points at this lane's element of the variable's strip block
// (node stride 32 doubles: immediate offsets).  MODAL: U, A, Y, Y2 hold
// modal coefficients; the nodal parts b X + g K and g2 K are converted to
// modes in registers before the u^n / accumulator terms are added.
template <int P, bool HAS_U, bool HAS_Y2, bool MODAL, bool EARLY_U>
__device__ __forceinline__ unsigned finalize(double (&acc)[P + 1][P + 1], const double *cur,
                                             const double *Av, double *Y2v, int v,
                                             const double *sFX,
                                             const double *sFtop, const double *sFbot,
                                             const double *row, int lane, bool owned,
                                             double *Yv, const StageParams &kp, double *Ypeer,
                                             double *Ypeer2, const double (&un_in)[P + 1][P + 1],
                                             const double *Uv)
{
    constexpr int N = P + 1;
    using RL = RowLayout<P>;
    // u^n: loaded by the caller before barrier 2 (early_u), else all of it
    // here, before the first store (U may alias Y)
    double unl[EARLY_U ? 1 : N][EARLY_U ? 1 : N];
    if constexpr (HAS_U && !EARLY_U) {
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) unl[a][b] = Uv[(a * N + b) * kLanes];
    }
#define UN(a, b) (EARLY_U ? un_in[a][b] : unl[EARLY_U ? 0 : (a)][EARLY_U ? 0 : (b)])
    double an[HAS_Y2 ? N : 1][HAS_Y2 ? N : 1];
    if constexpr (HAS_Y2) {            // second output's addend (may alias Y2)
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) an[a][b] = Av[(a * N + b) * kLanes];
    }
    constexpr int LD = Smem<P>::LD;
    const int o = (v * N) * LD;        // x-face column c: left face of lane c
#pragma unroll
    for (int q = 0; q < N; ++q) {
        const double l = sFX[o + q * LD + lane];
        const double r = sFX[o + q * LD + lane + 1];
        const double t = sFtop[o + q * LD + lane];     // zero at a pole (the face warp)
        const double bo = sFbot[o + q * LD + lane];
#pragma unroll
        for (int k = 0; k < N; ++k) {
            // x faces at eta node q lift along xi (column q); y faces at xi node q along eta (row q)
            acc[k][q] = fma(c_nod[P].mu[k], l, fma(-c_nod[P].mu[N - 1 - k], r, acc[k][q]));
            acc[q][k] = fma(c_nod[P].mu[k], bo, fma(-c_nod[P].mu[N - 1 - k], t, acc[q][k]));
        }
    }
    const double *rj = row + RL::RJ;
    if constexpr (MODAL) {
        // K = diag(rj) acc at the nodes; Y2 = A + g2 K and Y = a U + (b X + g K),
        // with the nodal parts converted to modes
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
            for (int i = 0; i < N; ++i) acc[i][j] *= rj[j];
        if constexpr (HAS_Y2) {
            double k2[N][N];
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) k2[i][j] = kp.g2 * acc[i][j];
            to_modal<P>(k2);
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (owned) Y2v[(i * N + j) * kLanes] = an[i][j] + k2[i][j];
        }
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) acc[i][j] = fma(kp.b, cur[(i * N + j) * kLanes + lane], kp.g * acc[i][j]);
        to_modal<P>(acc);
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double y = acc[i][j];
                if (HAS_U) y = fma(kp.a, UN(i, j), y);
                if (owned) Yv[(i * N + j) * kLanes] = y;
                acc[i][j] = y;
            }
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double gr = kp.g * rj[j];
            const double g2r = HAS_Y2 ? kp.g2 * rj[j] : 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const double k = acc[i][j];
                double y = fma(kp.b, cur[(i * N + j) * kLanes + lane], gr * k);
                if (HAS_U) y = fma(kp.a, UN(i, j), y);
                if (owned) Yv[(i * N + j) * kLanes] = y;
                if (owned && Ypeer) Ypeer[(i * N + j) * kLanes] = y;   // fused halo exchange (NVLink store)
                if (owned && Ypeer2) Ypeer2[(i * N + j) * kLanes] = y;
                if constexpr (HAS_Y2) {
                    const double y2 = fma(g2r, k, an[i][j]);
                    if (owned) Y2v[(i * N + j) * kLanes] = y2;
                }
                acc[i][j] = y;
            }
        }
    }
#undef UN
    unsigned bad = 0;
    if (owned) {
        if (kp.check_finite) {   // Inf or NaN: max exponent field of the outputs (integer pipe)
            int fexp = 0;
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) fexp = max(fexp, __double2hiint(acc[i][j]) & 0x7ff00000);
            bad |= fexp == 0x7ff00000 ? 2u : 0u;
        }
        if (v == 0 && kp.check_mean) {
            if constexpr (MODAL) {   // the reference's check: mode 0 (timestep.py:220-226)
                bad |= !(acc[0][0] > 0.0) ? 4u : 0u;
            } else {                 // cell mean = modal c_00 = sum w_i w_j u_ij / 4
                double m = 0.0;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) s = fma(c_nod[P].w[j], acc[i][j], s);
                    m = fma(c_nod[P].w[i], s, m);
                }
                bad |= !(m > 0.0) ? 4u : 0u;
            }
        }
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
// element, from its gathered values; (side 1) L trace of the strip's
// element 0, from the (nodal) ring.  Also the L trace of the right
// neighbour (lanes 6..8), which the h warp needs for the last lane's right
// face.  MODAL: the gathered neighbours hold modes, converted here.
template <int P, bool MODAL>
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
            if constexpr (MODAL) to_nodal<P>(c);
        }
        double tr[N];
        if (side == 0)
            xtrace<P, false>(c, tr);                 // R trace of the left neighbour
        else
            xtrace<P, true>(c, tr);                  // L traces of element 0 / the right neighbour
        double *dst = side == 0 ? sHL : side == 1 ? sE0 : sHR;
#pragma unroll
        for (int q = 0; q < N; ++q) dst[(v * N + q) * Smem<P>::LD] = tr[q];
    }
    __syncwarp();
}

// one variable's bottom traces of a row (its nodal ring tile) -> the
// y-face buffer the face warp evaluates in place (+ h positivity)
template <int P>
__device__ __forceinline__ unsigned stage_bottom(const double *tile, double *dst, int lane, bool check)
{
    constexpr int N = P + 1;
    double c[N][N], bt[N];
    tile_read<P>(c, tile, lane);
    ytrace<P, true>(c, bt);
    unsigned bad = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        dst[q * Smem<P>::LD + lane] = bt[q];
        if (check) bad |= !(bt[q] > 0.0);
    }
    return bad;
}

// MODAL: a landed ring tile (this lane's element of one variable) -> nodal
// values in place; every later reader of the slot sees the nodal tile
template <int P>
__device__ __forceinline__ void tile_to_nodal(double *tile, int lane)
{
    constexpr int N = P + 1;
    double c[N][N];
    tile_read<P>(c, tile, lane);
    to_nodal<P>(c);
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) tile[(a * N + b) * kLanes + lane] = c[a][b];
    __syncwarp();
}

// one variable's row tile (and, with orography, the matching tile of the
// warp's orography factor) into a ring slot, completing on one mbarrier
__device__ __forceinline__ void tma_row2(double *dst, const double *src, double *dst2, const double *src2,
                                         unsigned bytes, unsigned long long *mb)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(2 * bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst2)),
        "l"(src2), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
}

// Wait (thread 0) until a system-scope counter reaches `need`, at most
// timeout_ns; false on timeout (a neighbour that died or stalled)
__device__ __forceinline__ bool wait_counter(const unsigned long long *ctr, unsigned long long need,
                                             unsigned long long timeout_ns)
{
    if (ld_acquire_sys(ctr) >= need) return true;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(ctr) < need) {
        __nanosleep(64);
        if (globaltimer() - t0 > timeout_ns) return false;
    }
    return true;
}

// First row of chunk c when `rows` rows are split into n chunks of
// floor/ceil(rows / n) rows, the longer chunks first (lowest blockIdx.y):
// the block scheduler hands out CTAs in index order, one per SM per round,
// so the long chunks spread over distinct SMs instead of stacking on some
// (C3: +1.5% over interleaved lengths).
__device__ __forceinline__ int even_start(int c, int rows, int n)
{
    const int q = rows / n, r = rows - q * n;
    return c * q + min(c, r);
}

template <int P, int F>
__global__ void __launch_bounds__(kThreads, (min_blocks_f<P, F>())) stage_kernel(StageParams kp)
{
    constexpr bool HAS_U = (F & kHasU) != 0;
    constexpr bool HAS_Y2 = (F & kHasY2) != 0;
    constexpr bool EDGE = (F & kEdge) != 0;
    constexpr bool MODAL = (F & kModal) != 0;
    constexpr bool OROG = (F & kOrog) != 0;
    static_assert(!(EDGE && (MODAL || HAS_Y2)), "edge launches take nodal states and have one output");
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
    int jb, je;
    if constexpr (EDGE) {
        // a whole band in one launch: blockIdx.y 0 / 1 = its southern / northern
        // edge row (one row each, scheduled first), then chunks of rc interior rows
        const int nedge = min(2, kp.band_hi - kp.band_lo);
        const int y = blockIdx.y;
        if (y < nedge) {
            jb = y == 0 ? kp.band_lo : kp.band_hi - 1;
            je = jb + 1;
        } else if (kp.even > 0) {
            const int inner = kp.band_hi - kp.band_lo - 2;
            jb = kp.band_lo + 1 + even_start(y - nedge, inner, kp.even);
            je = kp.band_lo + 1 + even_start(y - nedge + 1, inner, kp.even);
        } else {
            jb = kp.band_lo + 1 + (y - nedge) * kp.rc;
            je = min(jb + kp.rc, kp.band_hi - 1);
        }
    } else {
        const bool second = (int)blockIdx.y >= kp.nchunk1;   // one launch can cover two row ranges
        if (!second && kp.even > 0) {
            const int rows = kp.j_end - kp.j_begin;
            jb = kp.j_begin + even_start(blockIdx.y, rows, kp.even);
            je = kp.j_begin + even_start(blockIdx.y + 1, rows, kp.even);
        } else {
            jb = second ? kp.j_begin2 + ((int)blockIdx.y - kp.nchunk1) * kp.rc : kp.j_begin + blockIdx.y * kp.rc;
            je = min(jb + kp.rc, second ? kp.j_end2 : kp.j_end);
        }
        if (jb >= je) return;
    }
    unsigned bad = 0;
    // fused halo exchange: an edge row first waits until the neighbour has
    // delivered this stage's halo row (its previous stage's edge row):
    // nstrip deliveries per completed stage, counted in our memory.  The
    // wait is bounded: a neighbour that never delivers raises PEER_TIMEOUT
    // (the row is then computed from a stale halo and must be discarded).
    if constexpr (EDGE) {
        if (threadIdx.x == 0) {
            const unsigned long long need =
                ld_acquire_sys(kp.stage_ctr) * (unsigned long long)kp.nstrip * gridDim.z;
            const int g = kp.row0 + jb;   // only the edge rows' CTAs wait
            bool ok = true;
            if (jb == kp.band_lo && g > 0) ok &= wait_counter(kp.recv_count, need, kp.peer_timeout_ns);
            if (jb == kp.band_hi - 1 && g + 1 < kp.ny)
                ok &= wait_counter(kp.recv_count + 1, need, kp.peer_timeout_ns);
            if (!ok) bad |= kPeerTimeout;
            asm volatile("fence.proxy.async.global;" ::: "memory");   // peer stores -> TMA reads
        }
        __syncthreads();
    }

    double *const ringS = smem + SM::XR0;          // [slot][var][mode][lane]
    double *const ring0 = ringS + v * NP * kLanes;   // this warp's variable
    double *sXL = smem + SM::XL;
    double *sXR = smem + SM::XRT;
    double *sT = smem + SM::TT;
    double *sFX = smem + SM::FX;
    double *sFa = smem + SM::FY0;
    double *sFb = smem + SM::FY1;
    double *sRow = smem + SM::ROW;
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem + SM::MBAR);   // [slot][var]
    // orography tiles of the momentum warps: [slot][hu, hv][mode][lane]
    double *const sOB = smem + SM::OB + (v > 0 ? (v - 1) * NP * kLanes : 0);
    const double *Oz = OROG && v > 0 ? kp.orog + (size_t)(v - 1) * kp.vstride + (size_t)strip * NP * kLanes : nullptr;

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

    // the row tile (and orography tile) of local row r into ring slot `slot`
    // orography: whether ring slot 0 / 1 holds a (non-zero) factor tile; the
    // mask byte of a row is read two rows ahead by every lane, so neither the
    // copy nor the volume waits on it
    bool ob_on0 = false, ob_on1 = false;
    auto ob_mask = [&](int r) {
        return OROG && v > 0 && !face_warp && kp.orog_mask[(size_t)r * kp.nstrip + strip] != 0;
    };
    // a y-periodic (planar) mesh wraps its rows: local row r is stored at
    // (r + ny) % ny (single-band contexts only; the host checks)
    const bool yper = kp.periodic_y != 0;
    auto wrap = [&](int r) { return yper ? (r + kp.ny) % kp.ny : r; };
    auto issue_row = [&](int slot, int r_, bool ob) {
        const int r = wrap(r_);
        double *dst = ring0 + slot * SM::TILE;
        if constexpr (OROG) {
            if (ob) {
                tma_row2(dst, Xz + (size_t)r * kp.rstride, sOB + slot * 2 * NP * kLanes,
                         Oz + (size_t)r * kp.orog_rstride, kTileBytes, mbar + slot * 3 + v);
                return;
            }
        }
        tma_row(dst, Xz + (size_t)r * kp.rstride, kTileBytes, mbar + slot * 3 + v);
    };

    // rows whose coefficients exist: local r with global row0+r in [0, ny)
    // (every row, wrapped, on a y-periodic mesh: no pole)
    const int r_last = yper ? je : min(kp.nrows - 1, kp.ny - 1 - kp.row0);
    const int last_fetch = min(je, r_last);        // rows jb..last_fetch stream through the ring

    // each variable warp's elected lane initialises its own two ring
    // mbarriers and starts streaming rows jb, jb+1 at once: the copies are
    // in flight while the row tables and the row below the chunk load
    if constexpr (OROG) {
        ob_on0 = ob_mask(jb);
        ob_on1 = jb + 1 <= last_fetch && ob_mask(jb + 1);
    }
    if (!face_warp && lane == 0) {
        mbar_init(mbar + v, 1);
        mbar_init(mbar + 3 + v, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue_row(0, jb, ob_on0);
        if (jb + 1 <= last_fetch) issue_row(1, jb + 1, ob_on1);
    }

    // row-table ring: slot (r - jb) % 3 holds local row r (rows jb, jb+1 now,
    // row jl+2 staged by the face warp during iteration jl)
    const int gfirst = kp.row0 + jb;
    {
        const int nload = yper ? 2 : min(2, kp.ny - gfirst);
        for (int idx = threadIdx.x; idx < nload * RL::SSTRIDE; idx += kThreads) {
            const int r = idx / RL::SSTRIDE;
            sRow[idx] = kp.rowtab[(size_t)wrap(gfirst + r) * RL::STRIDE + (idx - r * RL::SSTRIDE)];
        }
    }
    // top traces of the row below the chunk (its first row's bottom face)
    const bool below = yper || gfirst > 0;
    if (below && !face_warp) {
        const double *src = Xz + (size_t)wrap(jb - 1) * kp.rstride + lane;
        double c[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) c[a][b] = __ldg(src + (a * N + b) * kLanes);
        if constexpr (MODAL) to_nodal<P>(c);
        double tt[N];
        ytrace<P, false>(c, tt);
#pragma unroll
        for (int q = 0; q < N; ++q) sT[(v * N + q) * SM::LD + lane] = tt[q];
    }
    __syncthreads();
    double alpha_x = kp.alpha, alpha_y = kp.alpha;
    if (kp.alpha_mode == 2) {
        alpha_x = kp.alpha_dev[0];
        alpha_y = kp.alpha_dev[1];
    }
    if (!face_warp) {
        mbar_wait(mbar + v, 0);                    // row jb landed (this variable)
        if constexpr (MODAL) tile_to_nodal<P>(ring0, lane);
        // its bottom traces: the face below row jb (the face warp's pre-iteration)
        bad |= owned & stage_bottom<P>(ring0, sFb + v * N * SM::LD, lane, chk);
    }
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
                // this row's border face (formed in the last window) into FX column 0:
                // the previous row's finalize, its last reader, is done
                if (lane < 3 * N) smem[SM::FX + lane * SM::LD] = smem[SM::F0T + lane * SM::LD];
                // async gathers, consumed after barrier 2: the next row's neighbour
                // coefficients and the table of row it+2 (its slot held row it-1)
                if (it + 1 < je)
                    fetch_neighbours<P>(kp.X + (size_t)blockIdx.z * kp.zstride + (size_t)(it + 1) * kp.rstride,
                                        eL, eR, smem + SM::HB, lane, kp.vstride);
                if (it + 2 <= je && (yper || kp.row0 + it + 2 < kp.ny)) {
                    double *dst = sRow + ((k + 2) % 3) * RL::SSTRIDE;
                    const double *src = kp.rowtab + (size_t)wrap(kp.row0 + it + 2) * RL::STRIDE;
                    for (int idx = lane; idx < RL::SSTRIDE; idx += kLanes) cp_async8(dst + idx, src + idx);
                }
                cp_commit();
            }
            const double *next_tile = ringS + ((k + 1) & 1) * SM::TILE;   // X(it+1)
            // the y-face above row it, from row it's top traces and row it+1's
            // bottom traces (staged in the face's output slot by the var warps)
            if (it + 1 <= last_fetch && (!pre || below)) {
                const int dst = (int)((pre ? fb : fa) - smem);
                const double *above = sRow + ((k + 1) % 3) * RL::SSTRIDE;
                if (owned)
                face_flux_call<P>(SM::TT + lane, dst + lane, dst + lane,
                                  FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r,
                                           kp.alpha_mode, 1, above[RL::CRB], above[RL::COSB], alpha_y,
                                           kp.bdx});
            } else {
                // a pole: no face, no flux (dg.py:483-495) -- the lift reads zeros
                double *dst = pre ? fb : fa;
#pragma unroll
                for (int q = 0; q < 3 * N; ++q) dst[q * SM::LD + lane] = 0.0;
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
                border_traces<P, MODAL>(smem + SM::HB, next_tile, smem + SM::HL, smem + SM::E0, smem + SM::HR,
                                        lane);
                // one face for the whole strip: lane 0 alone (the other lanes would
                // repeat it -- ~9% of the stage's FP64 lane work, i.e. power)
                if (lane == 0)
                face_flux_call<P>(SM::HL, SM::E0, SM::F0T,
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
            const double *row = sRow + (k % 3) * RL::SSTRIDE;
            TSTAMP(s);

            const bool ob2 = OROG && jl + 2 <= last_fetch && ob_mask(jl + 2);
            // warm L2 for this row's u^n and for row jl+2 (copied in after finalize)
            if (lane == 0) {
                if (HAS_U) prefetch_l2_bulk(Uz - lane + (size_t)jl * kp.rstride, kTileBytes);
                if (jl + 2 <= last_fetch) prefetch_l2_bulk(Xz + (size_t)wrap(jl + 2) * kp.rstride, kTileBytes);
            }
            {
                double c[N][N];
                tile_read<P>(c, cur, lane);            // X(jl)
                bad |= owned & traces_row<P>(c, sXL + v * N * SM::LD, sXR + v * N * SM::LD, sT + v * N * SM::LD,
                                             lane, chk);
            }
            TSTAMP(0);
            if (jl + 1 <= last_fetch) {
                mbar_wait(mbar + (slot ^ 1) * 3 + v, ((k + 1) >> 1) & 1);   // X(jl+1)
                if constexpr (MODAL) tile_to_nodal<P>(ring0 + (slot ^ 1) * SM::TILE, lane);
                // its bottom traces for the face warp's y-face above row jl
                bad |= owned & stage_bottom<P>(ring0 + (slot ^ 1) * SM::TILE, sFa + v * N * SM::LD, lane, chk);
            }
            TSTAMP(1);
            __syncthreads();                           // barrier 1
            TSTAMP(2);

            if (v == 0) {
                // the h warp has the lightest volume work: it takes the x-faces 1..32
                // (right face of every lane; the last valid lane's neighbour is the halo)
                const bool last = lane == nvalid - 1;
                if (owned)   // padding lanes' faces are never read
                face_flux_call<P>(SM::XRT + lane, SM::XL + (last ? kLanes : min(lane + 1, kLanes - 1)), SM::FX + lane + 1,
                                  FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r,
                                           kp.alpha_mode, 0, 0.0, 0.0, alpha_x, kp.bdy});
            }
            double vol[N][N];
            const double *sB = OROG && (slot ? ob_on1 : ob_on0) ? sOB + slot * 2 * NP * kLanes : nullptr;
            if constexpr (vol_rolled<P>()) {
                double *sE = smem + SM::E + v * NP * kLanes;
                if (v == 0)
                    volume_rolled<P, 0, false>(vol, v, ringS + slot * SM::TILE, row, lane, kp, sE, sB);
                else if (v == 1)
                    volume_rolled<P, 1, OROG>(vol, v, ringS + slot * SM::TILE, row, lane, kp, sE, sB);
                else
                    volume_rolled<P, 2, OROG>(vol, v, ringS + slot * SM::TILE, row, lane, kp, sE, sB);
            } else {
                if (v == 0)
                    volume<P, false, false>(vol, v, ringS + slot * SM::TILE, row, lane, kp, sB);
                else
                    volume<P, true, OROG>(vol, v, ringS + slot * SM::TILE, row, lane, kp, sB);
            }
            TSTAMP(3);
            double unr[N][N];                          // u^n loads in flight across barrier 2
            if constexpr (HAS_U && early_u<P, F>()) {
                const double *Uv = Uz + (size_t)jl * kp.rstride;
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) unr[a][b] = Uv[(a * N + b) * kLanes];
            }
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
            bad |= finalize<P, HAS_U, HAS_Y2, MODAL, early_u<P, F>()>(vol, cur, HAS_Y2 ? Az + roff : nullptr, HAS_Y2 ? Y2z + roff : nullptr,
                                                     v, sFX, sFa, sFb, row, lane,
                                                     owned, Yz + roff, kp, Ypeer, Ypeer2, unr,
                                                     HAS_U ? Uz + roff : nullptr);
            // X(jl) is consumed: stream row jl+2 into its slot (L2-warm by now)
            __syncwarp();
            if (lane == 0 && jl + 2 <= last_fetch) {
                fence_proxy_async();
                issue_row(slot, jl + 2, ob2);
            }
            if constexpr (OROG) {
                if (slot) ob_on1 = ob2; else ob_on0 = ob2;
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
        for (int b = 0; b < kStatusBits; ++b)
            if (bad & (1u << b)) atomicMin(kp.first_tag + b, kp.tag);
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

// Modal <-> nodal change of basis of one element and variable per thread,
// grid (nstrip, rows, nz), block 96 = 3 variables x 32 lanes; in may equal
// out (every thread reads its element before writing it):
//   nodal u[i][j] = sum_ab P_a(x_i) P_b(x_j) c[a][b]                (basis.py:118-133)
//   modal c[a][b] = (2a+1)(2b+1)/4 sum_ij w_i P_a(x_i) w_j P_b(x_j) u[i][j]
// (the Gauss rule is exact for the degree-2p products, so the pair is an
// exact inverse up to rounding).
template <int P, bool TO_NODAL>
__global__ void __launch_bounds__(96) convert_kernel(const double *in, double *out, long long zstride,
                                                     long long rstride, long long vstride, int r0)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
    const size_t off = (size_t)blockIdx.z * zstride + (size_t)(r0 + (int)blockIdx.y) * rstride +
                       (size_t)v * vstride + (size_t)blockIdx.x * NP * kLanes + lane;
    double x[N][N], t[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) x[a][b] = in[off + (a * N + b) * kLanes];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int q = 0; q < N; ++q) {   // contract the second index
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b)
                s = fma(TO_NODAL ? LEG(b, q) : WP(q, b), x[a][b], s);
            t[a][q] = s;
        }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
        for (int r = 0; r < N; ++r) {   // then the first
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < N; ++a) s = fma(TO_NODAL ? LEG(a, q) : WP(q, a), t[a][r], s);
            if (!TO_NODAL) s *= 0.25 * (double)((2 * q + 1) * (2 * r + 1));
            out[off + (q * N + r) * kLanes] = s;
        }
}

// Global-mode alpha (dg.py:389-411, models.py:271-280): max over all
// traces of the rows [jlo, jhi) into out[0] (x faces) and out[1] (y faces,
// with cos of the edge latitude); MODAL converts each tile first.
template <int P, bool MODAL>
__global__ void alpha_prepass_kernel(const double *__restrict__ X, long long zstride, long long rstride,
                                     long long vstride, int nx, int row0, int jlo, int jhi,
                                     const double *__restrict__ cos_edge, double inv_r, double gravity,
                                     double h_floor, double *out)
{
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int jl = jlo + blockIdx.y;
    if (i >= nx || jl >= jhi) return;
    const double *base = X + (size_t)blockIdx.z * zstride + (size_t)jl * rstride;
    const int jg = row0 + jl;
    double tr[4][3][N];   // L R B T, from the nodal tile u[i][j]
    for (int v = 0; v < 3; ++v) {
        double u[N][N];
        for (int a = 0; a < N; ++a)
            for (int b = 0; b < N; ++b)
                u[a][b] = base[(size_t)v * vstride + (size_t)(i >> 5) * NP * 32 + (a * N + b) * 32 + (i & 31)];
        if constexpr (MODAL) to_nodal<P>(u);
        for (int q = 0; q < N; ++q) {
            double l = 0, r = 0, bo = 0, t = 0;
            for (int k = 0; k < N; ++k) {
                const double lo = c_nod[P].lm[k], hi = c_nod[P].lm[N - 1 - k];
                l = fma(lo, u[k][q], l);
                r = fma(hi, u[k][q], r);
                bo = fma(lo, u[q][k], bo);
                t = fma(hi, u[q][k], t);
            }
            tr[0][v][q] = l;
            tr[1][v][q] = r;
            tr[2][v][q] = bo;
            tr[3][v][q] = t;
        }
    }
    double ax = 0.0, ay = 0.0;
    for (int e = 0; e < 4; ++e)
        for (int q = 0; q < N; ++q) {
            const double h = tr[e][0][q];
            const double m = tr[e][e < 2 ? 1 : 2][q];
            const double a = (fabs(m / fmax(h, h_floor)) + sqrt(gravity * fmax(h, 0.0))) * inv_r;
            if (e < 2)
                ax = fmax(ax, a);
            else
                ay = fmax(ay, a * cos_edge[jg + (e == 3 ? 1 : 0)]);
        }
    atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)__double_as_longlong(ax));
    atomicMax(reinterpret_cast<unsigned long long *>(out + 1), (unsigned long long)__double_as_longlong(ay));
}

// Initial-condition projection (basis.py:206-233) of nodal values onto the
// modal basis.
// grid (ceil(nx/128), ny, 3), block 128: one thread per element and
// variable.  f: nodal values [3][ny][nx][n*n] at the (p+1)^2 Gauss nodes
// (q = qi*n + qj, qi along lambda); moments = determ sum_q w_qi w_qj
// cos(theta_qj) phi_m(q) f_q (sum-factorised), then the Kronecker inverse
// mass c[a][b] = (2a+1) sum_bb T_j[b][bb] moments[a][bb] (T_j: the a = 0
// block of the row's M^-1, from the row table); written to every level.
template <int P>
__global__ void project_kernel(const double *__restrict__ f, const double *__restrict__ cos_nodes,
                               const double *__restrict__ rowtab, int row_stride, int t_off, DiagLayout L,
                               int nz, double determ, double *Y)
{
    constexpr int N = P + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, v = blockIdx.z;
    if (i >= L.nx) return;
    const double *fv = f + (((size_t)v * L.ny + j) * L.nx + i) * (N * N);
    const double *cj = cos_nodes + (size_t)j * N;
    double g[N][N];   // g[qi][b] = sum_qj wP_b(qj) cos_qj f(qi, qj)
#pragma unroll
    for (int qi = 0; qi < N; ++qi)
#pragma unroll
        for (int b = 0; b < N; ++b) {
            double acc = 0.0;
#pragma unroll
            for (int qj = 0; qj < N; ++qj) acc = fma(c_nod[P].wp[b][qj] * cj[qj], fv[qi * N + qj], acc);
            g[qi][b] = acc;
        }
    double mom[N][N];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) {
            double acc = 0.0;
#pragma unroll
            for (int qi = 0; qi < N; ++qi) acc = fma(c_nod[P].wp[a][qi], g[qi][b], acc);
            mom[a][b] = determ * acc;
        }
    const double *T = rowtab + (size_t)j * row_stride + t_off;
    for (int z = 0; z < nz; ++z) {
        double *y = Y + (size_t)z * L.zstride + (size_t)j * L.rstride + (size_t)v * L.vstride +
                    (size_t)(i >> 5) * L.nphi * 32 + (i & 31);
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) {
                double acc = 0.0;
#pragma unroll
                for (int bb = 0; bb < N; ++bb) acc = fma(T[b * N + bb], mom[a][bb], acc);
                y[(a * N + b) * 32] = (double)(2 * a + 1) * acc;
            }
    }
}

#undef LEG
#undef WP

}  // namespace dgswe
