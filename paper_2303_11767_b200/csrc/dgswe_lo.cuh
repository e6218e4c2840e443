// dgswe_lo.cuh -- low-order (p = 0, 1) stage kernel for sm_100a.
//
// At p <= 1 an element has 1-4 nodes per variable: the warp-specialised
// kernel (dgswe_kernels.cuh) then spends its time on per-row barriers, ring
// waits and one face evaluation per 1-2 nodes, not on HBM (C5 sweep: 26% /
// 51% of the roofline).  Here ONE thread owns one element with all three variables
// in registers and there is no CTA barrier: warp w of a CTA marches north
// through a chunk of rows of segment 4 blockIdx.x + w, 30 elements wide:
// lanes 1..30 own elements 30 s .. 30 s + 29, lanes 0 and 31 hold their
// periodic neighbours (read like the owned ones, never stored).  Its loads
// go through a per-warp ring of lo_depth<P>() rows in shared memory filled by
// cp.async (LDGSTS) depth - 1 rows ahead, the row's table included
// (X and u^n are read back only by the lane that copied them; the table by
// all lanes after a __syncwarp).  C5 p = 0 (1e9 DOF): 0.29 of the roofline
// with one row loaded and consumed per iteration, 0.36 with the ring, 0.47
// with the halo lanes and shared reciprocals (below), 0.58 with the staged
// row tables at 4 CTAs per SM; p = 1: 0.65 (the main kernel 0.51).
//
// Per row j (nodal values; SAME arithmetic as the main kernel -- the traces
// of dgswe_kernels.cuh, face_core_rc, volume<> and the finalize order -- so
// both kernels give identical bits):
//   * each trace node's 1/h and sqrt(h) (inv_and_sqrt) is formed once, by
//     its own element (lo_side): the x-face takes lane l+1's L side with
//     them by shuffle, the y-face the next row's B side (the main kernel
//     forms them inside each face: identical bits, the face fuses
//     sqrt(g) sqrt(h) explicitly).  At p = 0 all four sides of an element
//     are its value (l_0 = 1): one set per element and row, the next row's
//     carried up as that row's own;
//   * row j+1 (coalesced: one 256-byte line per variable) has landed in the
//     ring while row j is computed; its traces and row j's give the y-face
//     above row j, carried in registers as the next row's bottom face (each
//     y-face evaluated once per segment);
//   * x-faces: lane l (0..30) evaluates the face between lanes l and l+1
//     (operands of lane l+1 by shuffle); an owned lane's left face is lane
//     l-1's.  No lane evaluates an extra face alone: the neighbouring
//     segments evaluate their shared border face from the same operands in
//     the same order (2 of 32 lanes are halo work instead);
//   * volume + source (models.py:161-252), lifts, diagonal mass and the
//     stage combination (timestep.py:132-167), stores of the owned lanes.
// Variants: plain nodal stages with and without the u^n term (kHasU) -- the
// SSPRK3 / RK1 / RK2 steps of dgswe_rk_steps and the nodal stage entry
// points.  Every other variant (modal, RK4's second output, band edges,
// orography) keeps the main kernel.
#pragma once

#include "dgswe_kernels.cuh"

namespace dgswe {

constexpr int kLoWarps = 4;   // strips per CTA
// rows per warp in the shared-memory ring (depth - 1 in flight) and
// resident CTAs per SM (register cap), per degree and variant, measured at
// C5 (1e9 DOF):
//   p = 0: depth 4, 4 CTAs (104 registers): 0.57-0.59 of the roofline (6
//          CTAs at 80 registers spilled: 0.45; 5: 0.49-0.51; 3: 0.57;
//          depth 3: 0.56, 6: equal);
//   p = 1: depth 3; the stage without u^n 3 CTAs (166 registers), with u^n
//          2 (212; its ring takes 75 KB): 0.65 (both at 2: 0.63, both at 3:
//          0.58; depth 4: 0.47), the main kernel 0.51.
template <int P> __host__ __device__ constexpr int lo_depth() { return P == 0 ? 4 : 3; }
template <int P, int F> __host__ __device__ constexpr int lo_min_blocks()
{
    return P == 0 ? 4 : ((F & kHasU) ? 2 : 3);
}
constexpr int kLoOwn = kLanes - 2;   // elements a warp owns: lanes 1..30 (lanes 0 / 31: neighbours)

// warp segments of kLoOwn elements covering a row
__host__ __device__ constexpr int lo_segments(int nx) { return (nx + kLoOwn - 1) / kLoOwn; }

template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// dynamic shared memory of one low-order CTA
template <int P, bool HAS_U>
constexpr int lo_smem_bytes()
{
    constexpr int NP = (P + 1) * (P + 1);
    return kLoWarps * lo_depth<P>() * ((HAS_U ? 2 : 1) * 3 * NP * kLanes + RowLayout<P>::SSTRIDE) * (int)sizeof(double);
}


// the degrees the low-order kernel serves: p = 0 (2.2x the main kernel at
// C5) and p = 1 (1.27x); p = 2 would need 255 registers and spill
template <int P>
__host__ __device__ constexpr bool lo_kernel_degree() { return P <= 1; }

// all three variables of element e of a row (row pointer: level and row
// applied), nodal slots m = i N + j
template <int P>
__device__ __forceinline__ void lo_load(const double *row, long long vstride, int e, double (&u)[3][(P + 1) * (P + 1)])
{
    constexpr int NP = (P + 1) * (P + 1);
    const double *b = row + (size_t)(e >> 5) * NP * kLanes + (e & 31);
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int m = 0; m < NP; ++m) u[v][m] = b[(size_t)v * vstride + m * kLanes];
}

template <int P>
__device__ __forceinline__ void lo_tile(const double (&u)[(P + 1) * (P + 1)], double (&t)[P + 1][P + 1])
{
#pragma unroll
    for (int i = 0; i < P + 1; ++i)
#pragma unroll
        for (int j = 0; j < P + 1; ++j) t[i][j] = u[i * (P + 1) + j];
}

// L (LO) or R traces of all three variables of an element
template <int P, bool LO>
__device__ __forceinline__ void lo_xtraces(const double (&u)[3][(P + 1) * (P + 1)], double (&tr)[3][P + 1])
{
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double t[P + 1][P + 1];
        lo_tile<P>(u[v], t);
        xtrace<P, LO>(t, tr[v]);
    }
}

// one side's traces of all three variables (SIDE 0 / 1: xi = -1 / +1,
// 2 / 3: eta = -1 / +1) with 1/h and sqrt(h) of its h nodes (inv_and_sqrt)
template <int P, int SIDE>
__device__ __forceinline__ void lo_side(const double (&u)[3][(P + 1) * (P + 1)], double (&t)[3][P + 1],
                                        double (&r)[P + 1], double (&c)[P + 1], double h_floor, double inv_floor)
{
    if constexpr (SIDE <= 1) {
        lo_xtraces<P, SIDE == 0>(u, t);
    } else {
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            double tile[P + 1][P + 1];
            lo_tile<P>(u[v], tile);
            ytrace<P, SIDE == 2>(tile, t[v]);
        }
    }
#pragma unroll
    for (int k = 0; k < P + 1; ++k) inv_and_sqrt(t[0][k], h_floor, inv_floor, r[k], c[k]);
}

template <int P>
__device__ __forceinline__ unsigned lo_positive(const double *x, int n)
{
    unsigned bad = 0;
#pragma unroll
    for (int q = 0; q < n; ++q) bad |= !(x[q] > 0.0);
    return bad;
}

template <int P, int F>
__global__ void __launch_bounds__(kLoWarps * kLanes, lo_min_blocks<P, F>()) lo_stage_kernel(StageParams kp)
{
    static_assert(P <= 1, "low-order kernel");
    static_assert((F & ~kHasU) == 0, "low-order kernel: nodal stages with or without u^n only");
    constexpr bool HAS_U = (F & kHasU) != 0;
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using RL = RowLayout<P>;
    const int lane = threadIdx.x & 31;
    const int nx = kp.nx;
    const int seg = blockIdx.x * kLoWarps + (threadIdx.x >> 5);
    if (seg >= lo_segments(nx)) return;             // whole warps: no barrier below
    // lanes 1..nvalid own elements first .. first + nvalid - 1; lane 0 and
    // lane nvalid + 1 hold the neighbours (periodic), padding lanes mirror
    // the right neighbour
    const int first = seg * kLoOwn;
    const int nvalid = min(kLoOwn, nx - first);
    const bool owned = lane >= 1 && lane <= nvalid;
    int g = first - 1 + min(lane, nvalid + 1);
    g = g < 0 ? g + nx : (g >= nx ? g - nx : g);
    const size_t eoff = (size_t)blockIdx.z * kp.zstride + (size_t)(g >> 5) * NP * kLanes + (g & 31);
    int jb, je;
    if (kp.even > 0) {
        const int rows = kp.j_end - kp.j_begin;
        jb = kp.j_begin + even_start(blockIdx.y, rows, kp.even);
        je = kp.j_begin + even_start(blockIdx.y + 1, rows, kp.even);
    } else {
        jb = kp.j_begin + blockIdx.y * kp.rc;
        je = min(jb + kp.rc, kp.j_end);
    }
    if (jb >= je) return;
    // the plane (periodic_y, one context per grid): rows wrap, no pole faces
    const bool yper = kp.periodic_y != 0;
    auto wrap = [&](int r) { return yper ? (r + kp.ny) % kp.ny : r; };
    const int r_last = yper ? je : min(kp.nrows - 1, kp.ny - 1 - kp.row0);   // local rows with coefficients
    const FaceArgs fx{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode, 0,
                      0.0, 0.0, kp.alpha_mode == 2 ? kp.alpha_dev[0] : kp.alpha, kp.bdy};
    const double alpha_y = kp.alpha_mode == 2 ? kp.alpha_dev[1] : kp.alpha;
    unsigned bad = 0;

    // per-warp ring of lo_depth<P>() rows in shared memory, filled with cp.async
    // (LDGSTS) depth - 1 rows ahead: row r's X, u^n and row table, one
    // commit group per row; X and u^n are read back only by the lane that
    // copied them, the row table by all lanes (after a __syncwarp)
    extern __shared__ __align__(16) double lo_smem[];
    constexpr int ROWW = 3 * NP * kLanes;
    constexpr int TBL = (HAS_U ? 2 : 1) * ROWW;                 // row table [RL::SSTRIDE]
    constexpr int SLOT = TBL + RL::SSTRIDE;
    static_assert(RL::SSTRIDE <= kLanes, "one row-table word per lane");
    double *ring = lo_smem + (threadIdx.x >> 5) * (lo_depth<P>() * SLOT);
    const int x_last = min(je, r_last);                         // rows whose X is read
    auto issue = [&](int r, int slot) {
        double *d = ring + slot * SLOT;
        if (r <= x_last) {
            const double *xr = kp.X + eoff + (size_t)wrap(r) * kp.rstride;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m)
                    cp_async8(d + (v * NP + m) * kLanes + lane, xr + (size_t)v * kp.vstride + m * kLanes);
            if (lane < RL::SSTRIDE) cp_async8(d + TBL + lane, kp.rowtab + (size_t)wrap(kp.row0 + r) * RL::STRIDE + lane);
            if constexpr (HAS_U) {
                if (r < je && owned) {
                    const double *ur = kp.U + eoff + (size_t)r * kp.rstride;
#pragma unroll
                    for (int v = 0; v < 3; ++v)
#pragma unroll
                        for (int m = 0; m < NP; ++m)
                            cp_async8(d + ROWW + (v * NP + m) * kLanes + lane, ur + (size_t)v * kp.vstride + m * kLanes);
                }
            }
        }
        cp_commit();
    };
#pragma unroll 1
    for (int k = 0; k < lo_depth<P>() - 1; ++k) issue(jb + k, k);

    // traces with 1/h and sqrt(h) of their h nodes, computed once per
    // element side and row: the x-face takes the right neighbour's L side
    // by shuffle, the y-face the next row's B side.  At p = 0 all four
    // sides are the element's value (l_0 = 1): one set per element, the
    // next row's carried up as that row's own (tr / rr / cc)
    double cur[3][NP], nxt[3][NP];
    lo_load<P>(kp.X + (size_t)jb * kp.rstride + (size_t)blockIdx.z * kp.zstride, kp.vstride, g, cur);
    double tr[3][N], rr[N], cc[N];                               // row jb's B side (p = 0: every side)
    lo_side<P, 2>(cur, tr, rr, cc, kp.h_floor, kp.inv_floor);
    bad |= owned & lo_positive<P>(tr[0], N);
    // the face below row jb: row jb-1's top traces against row jb's bottom ones
    double fbot[3][N];
    if (yper || kp.row0 + jb > 0) {
        double below[3][NP], tb[3][N], rb[N], cb[N];
        lo_load<P>(kp.X + (size_t)wrap(jb - 1) * kp.rstride + (size_t)blockIdx.z * kp.zstride, kp.vstride, g, below);
        lo_side<P, 3>(below, tb, rb, cb, kp.h_floor, kp.inv_floor);
        const double *rw = kp.rowtab + (size_t)(kp.row0 + jb) * RL::STRIDE;
        const FaceArgs fy{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode,
                          1, rw[RL::CRB], rw[RL::COSB], alpha_y, kp.bdx};
        double fh[N], fn[N], ft[N];
        face_core_rc<P>(tb[0], tb[2], tb[1], rb, cb, tr[0], tr[2], tr[1], rr, cc, fy, fh, fn, ft);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            fbot[0][k] = fh[k];
            fbot[2][k] = fn[k];
            fbot[1][k] = ft[k];
        }
    } else {
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int k = 0; k < N; ++k) fbot[v][k] = 0.0;   // a pole: no face (dg.py:483-495)
    }

    int slot = 0;                                                // ring slot of row j
    for (int j = jb; j < je; ++j) {
        const bool has_next = j + 1 <= r_last;
        const int slot1 = slot + 1 == lo_depth<P>() ? 0 : slot + 1;
        const int slotD = slot == 0 ? lo_depth<P>() - 1 : slot - 1;   // row j + lo_depth<P>() - 1
        __syncwarp();                                            // every lane is done with row j-1's slot
        issue(j + lo_depth<P>() - 1, slotD);
        cp_wait<lo_depth<P>() - 2>();                                 // rows <= j + 1 have landed
        __syncwarp();                                            // (the row tables: other lanes' copies)
        const double *rw = ring + slot * SLOT + TBL;             // row j's table, row j+1's next
        const double *ra = ring + slot1 * SLOT + TBL;
        if (has_next) {
            const double *d = ring + slot1 * SLOT;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m) nxt[v][m] = d[(v * NP + m) * kLanes + lane];
        }
        double un[3][NP];
        if constexpr (HAS_U) {
            const double *d = ring + slot * SLOT + ROWW;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m) un[v][m] = d[(v * NP + m) * kLanes + lane];
        }
        slot = slot1;
        bad |= owned & lo_positive<P>(cur[0], NP);
        // row j's R side (x-face in), L side (the left neighbour's out) and
        // T side (y-face in)
        double tR[3][N], rR[N], cR[N], tL[3][N], rL[N], cL[N], tT[3][N], rT[N], cT[N];
        if constexpr (P == 0) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
#pragma unroll
                for (int v = 0; v < 3; ++v) tR[v][k] = tL[v][k] = tT[v][k] = tr[v][k];
                rR[k] = rL[k] = rT[k] = rr[k];
                cR[k] = cL[k] = cT[k] = cc[k];
            }
        } else {
            lo_side<P, 1>(cur, tR, rR, cR, kp.h_floor, kp.inv_floor);
            lo_side<P, 0>(cur, tL, rL, cL, kp.h_floor, kp.inv_floor);
            lo_side<P, 3>(cur, tT, rT, cT, kp.h_floor, kp.inv_floor);
            bad |= owned & (lo_positive<P>(tR[0], N) | lo_positive<P>(tL[0], N) | lo_positive<P>(tT[0], N));
        }
        // x-faces: lane l (0..nvalid) evaluates the face between lanes l and
        // l+1 from its own traces and lane l+1's (shuffled with its
        // reciprocal and celerity); an owned lane's left face is lane l-1's
        double fr[3][N], fl[3][N];
        {
            double ho[N], no[N], to[N], ro[N], co[N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                ho[k] = __shfl_down_sync(0xffffffffu, tL[0][k], 1);
                no[k] = __shfl_down_sync(0xffffffffu, tL[1][k], 1);
                to[k] = __shfl_down_sync(0xffffffffu, tL[2][k], 1);
                ro[k] = __shfl_down_sync(0xffffffffu, rL[k], 1);
                co[k] = __shfl_down_sync(0xffffffffu, cL[k], 1);
            }
            double fh[N], fn[N], ft[N];
            face_core_rc<P>(tR[0], tR[1], tR[2], rR, cR, ho, no, to, ro, co, fx, fh, fn, ft);
#pragma unroll
            for (int k = 0; k < N; ++k) {
                fr[0][k] = fh[k];
                fr[1][k] = fn[k];
                fr[2][k] = ft[k];
            }
        }
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int k = 0; k < N; ++k) fl[v][k] = __shfl_up_sync(0xffffffffu, fr[v][k], 1);
        // the y-face above row j (zero at the pole), carried to the next row
        double ftop[3][N], trn[3][N], rn[N], cn[N];
        if (has_next) {
            lo_side<P, 2>(nxt, trn, rn, cn, kp.h_floor, kp.inv_floor);
            bad |= owned & lo_positive<P>(trn[0], N);
            const FaceArgs fy{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode,
                              1, ra[RL::CRB], ra[RL::COSB], alpha_y, kp.bdx};
            double fh[N], fn[N], ft[N];
            face_core_rc<P>(tT[0], tT[2], tT[1], rT, cT, trn[0], trn[2], trn[1], rn, cn, fy, fh, fn, ft);
#pragma unroll
            for (int k = 0; k < N; ++k) {
                ftop[0][k] = fh[k];
                ftop[2][k] = fn[k];
                ftop[1][k] = ft[k];
            }
        } else {
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int k = 0; k < N; ++k) ftop[v][k] = 0.0;
        }
        // volume, lifts, mass, stage combination per variable
        double uflat[3 * NP];
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int m = 0; m < NP; ++m) uflat[v * NP + m] = cur[v][m];
        int fexp = 0;
        double mean = 0.0;
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            double acc[N][N];
            if (v == 0)
                volume<P, false, false, 1>(acc, v, uflat, rw, 0, kp, nullptr);
            else
                volume<P, true, false, 1>(acc, v, uflat, rw, 0, kp, nullptr);
#pragma unroll
            for (int q = 0; q < N; ++q) {
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    acc[k][q] = fma(c_nod[P].mu[k], fl[v][q], fma(-c_nod[P].mu[N - 1 - k], fr[v][q], acc[k][q]));
                    acc[q][k] = fma(c_nod[P].mu[k], fbot[v][q], fma(-c_nod[P].mu[N - 1 - k], ftop[v][q], acc[q][k]));
                }
            }
            double *Yv = kp.Y + eoff + (size_t)v * kp.vstride + (size_t)j * kp.rstride;
#pragma unroll
            for (int jj = 0; jj < N; ++jj) {
                const double gr = kp.g * rw[RL::RJ + jj];
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    double y = fma(kp.b, cur[v][i * N + jj], gr * acc[i][jj]);
                    if (HAS_U) y = fma(kp.a, un[v][i * N + jj], y);
                    if (owned) Yv[(i * N + jj) * kLanes] = y;
                    fexp = max(fexp, __double2hiint(y) & 0x7ff00000);
                    acc[i][jj] = y;
                }
            }
            if (v == 0 && kp.check_mean) {   // cell mean = modal c_00 = sum w_i w_j u_ij / 4
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int jj = 0; jj < N; ++jj) s = fma(c_nod[P].w[jj], acc[i][jj], s);
                    mean = fma(c_nod[P].w[i], s, mean);
                }
            }
        }
        if (owned) {
            if (kp.check_finite) bad |= fexp == 0x7ff00000 ? 2u : 0u;
            if (kp.check_mean) bad |= !(mean > 0.0) ? 4u : 0u;
        }
        // slide the window: the next row's values, traces and bottom face
        if (has_next) {
#pragma unroll
            for (int v = 0; v < 3; ++v) {
#pragma unroll
                for (int m = 0; m < NP; ++m) cur[v][m] = nxt[v][m];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    fbot[v][k] = ftop[v][k];
                    tr[v][k] = trn[v][k];
                }
            }
#pragma unroll
            for (int k = 0; k < N; ++k) {
                rr[k] = rn[k];
                cc[k] = cn[k];
            }
        }
    }
    cp_wait_all();      // (every issued row <= je was consumed; empty groups remain)
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) {
        atomicOr(kp.status, bad);
        for (int b = 0; b < kStatusBits; ++b)
            if (bad & (1u << b)) atomicMin(kp.first_tag + b, kp.tag);
    }
}

}  // namespace dgswe
