// dgswe_lo.cuh -- low-order (p = 0) stage kernel for sm_100a.
//
// At p = 0 an element has one node per variable: the warp-specialised
// kernel (dgswe_kernels.cuh) then spends its time on per-row barriers, ring
// waits and one face evaluation per node, not on HBM (C5 sweep: 26% of the
// roofline).  Here ONE thread owns one
// element with all three variables in registers and there is no CTA
// barrier: warp w of a CTA marches north through a chunk of rows of strip
// 4 blockIdx.x + w, lane l = element 32 s + l.  Its loads go through a
// per-warp ring of kLoDepth rows in shared memory filled by cp.async
// (LDGSTS) kLoDepth - 1 rows ahead (each lane reads back only its own words:
// no warp barrier); the first version loaded row j+1 into registers and
// consumed it in the same iteration, one DRAM latency per row (C5 p = 0:
// 0.29 of the roofline -> 0.35-0.39 with the ring).
//
// Per row j (nodal values; SAME arithmetic as the main kernel -- the traces
// of dgswe_kernels.cuh, face_core, volume<> and the finalize order -- so
// both kernels give identical bits):
//   * row j+1 (coalesced: one 256-byte line per variable and node) has
//     landed in the ring while row j is computed; its bottom traces and row j's top traces give
//     the y-face above row j, which is carried in registers as the next
//     row's bottom face (each y-face evaluated once per strip);
//   * x-faces: lane l evaluates its right face from its R trace and lane
//     l+1's L trace (warp shuffles); its left face is lane l-1's (shuffle).
//     The strip's border lanes load the neighbour strip's element and form
//     its trace themselves: lane 0 of strip s+1 and the last lane of strip s
//     then evaluate the same face from the same operands, in the same order.
//   * volume + source (models.py:161-252), lifts, diagonal mass and the
//     stage combination (timestep.py:132-167), stores.
// Variants: plain nodal stages with and without the u^n term (kHasU) -- the
// SSPRK3 / RK1 / RK2 steps of dgswe_rk_steps and the nodal stage entry
// points.  Every other variant (modal, RK4's second output, band edges,
// orography) keeps the main kernel.
#pragma once

#include "dgswe_kernels.cuh"

namespace dgswe {

constexpr int kLoWarps = 4;   // strips per CTA
// rows per warp in the shared-memory ring (kLoDepth - 1 in flight) and
// resident CTAs per SM: measured at C5 p = 0 (1e9 DOF), depth 3..8 with
// 1 / 6 / 8 CTAs: 4 rows with 6 CTAs (78 registers, no spill) best, deeper
// rings slower (more open DRAM pages per SM), 8 CTAs spill
constexpr int kLoDepth = 4;
constexpr int kLoMinBlocks = 6;

template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// dynamic shared memory of one low-order CTA
template <int P, bool HAS_U>
constexpr int lo_smem_bytes()
{
    constexpr int NP = (P + 1) * (P + 1);
    return kLoWarps * kLoDepth * ((HAS_U ? 2 : 1) * 3 * NP * kLanes + 2 * 3 * NP) * (int)sizeof(double);
}


// the degrees the low-order kernel serves: p = 0 (1.7x the main kernel);
// at p = 1 the main kernel is faster (the one-thread element carries 4x the
// registers and the per-row dependency chain gets 4x longer)
template <int P>
__host__ __device__ constexpr bool lo_kernel_degree() { return P == 0; }

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

template <int P, bool LO>
__device__ __forceinline__ void lo_ytraces(const double (&u)[3][(P + 1) * (P + 1)], double (&tr)[3][P + 1])
{
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        double t[P + 1][P + 1];
        lo_tile<P>(u[v], t);
        ytrace<P, LO>(t, tr[v]);
    }
}

// Rusanov flux of one face from [var][node] traces, back into [var][node]
template <int P>
__device__ __forceinline__ void lo_face(const double (&in)[3][P + 1], const double (&out)[3][P + 1],
                                        const FaceArgs &fa, double (&f)[3][P + 1])
{
    const int vn = 1 + fa.dir, vt = 2 - fa.dir;
    double fh[P + 1], fn[P + 1], ft[P + 1];
    face_core<P>(in[0], in[vn], in[vt], out[0], out[vn], out[vt], fa, fh, fn, ft);
#pragma unroll
    for (int k = 0; k < P + 1; ++k) {
        f[0][k] = fh[k];
        f[vn][k] = fn[k];
        f[vt][k] = ft[k];
    }
}

template <int P>
__device__ __forceinline__ unsigned lo_positive(const double *x, int n)
{
    unsigned bad = 0;
#pragma unroll
    for (int q = 0; q < n; ++q) bad |= !(x[q] > 0.0);
    return bad;
}

template <int P>
__device__ __forceinline__ double lo_shfl(double x, int delta, bool down)
{
    return down ? __shfl_down_sync(0xffffffffu, x, delta) : __shfl_up_sync(0xffffffffu, x, delta);
}

template <int P, int F>
__global__ void __launch_bounds__(kLoWarps * kLanes, kLoMinBlocks) lo_stage_kernel(StageParams kp)
{
    static_assert(P <= 1, "low-order kernel");
    static_assert((F & ~kHasU) == 0, "low-order kernel: nodal stages with or without u^n only");
    constexpr bool HAS_U = (F & kHasU) != 0;
    constexpr int N = P + 1;
    constexpr int NP = N * N;
    using RL = RowLayout<P>;
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kLoWarps + (threadIdx.x >> 5);
    if (strip >= kp.nstrip) return;                 // whole warps: no barrier below
    const int nx = kp.nx;
    const int nvalid = min(kLanes, nx - strip * kLanes);
    const bool owned = lane < nvalid;
    const int e = strip * kLanes + (owned ? lane : nvalid - 1);   // padding lanes mirror a valid one
    const int eL = (strip * kLanes - 1 + nx) % nx;                 // left neighbour of lane 0
    const int eR = (strip * kLanes + nvalid) % nx;                 // right neighbour of the last lane
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
    const double *X = kp.X + (size_t)blockIdx.z * kp.zstride;
    const size_t lane_off = (size_t)blockIdx.z * kp.zstride + (size_t)strip * NP * kLanes + lane;
    const int r_last = min(kp.nrows - 1, kp.ny - 1 - kp.row0);      // local rows with coefficients
    const FaceArgs fx{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode, 0,
                      0.0, 0.0, kp.alpha_mode == 2 ? kp.alpha_dev[0] : kp.alpha, kp.bdy};
    const double alpha_y = kp.alpha_mode == 2 ? kp.alpha_dev[1] : kp.alpha;
    unsigned bad = 0;

    // per-warp ring of kLoDepth rows in shared memory, filled with
    // cp.async (LDGSTS) kLoDepth - 1 rows ahead: row j's X, u^n and border
    // neighbours, one commit group per row.  Each lane reads back only the
    // words it copied itself, so no warp barrier is needed.
    extern __shared__ __align__(16) double lo_smem[];
    constexpr int ROWW = 3 * NP * kLanes;                       // one row of one variable set
    constexpr int SLOT = (HAS_U ? 2 : 1) * ROWW + 2 * 3 * NP;   // X, u^n, left/right neighbour
    double *ring = lo_smem + (threadIdx.x >> 5) * (kLoDepth * SLOT);
    const bool lft = lane == 0, rgt = lane == nvalid - 1;
    const int x_last = min(je, r_last);                         // rows whose X is read
    auto issue = [&](int r, int slot) {
        double *d = ring + slot * SLOT;
        if (r <= x_last) {
            const double *xr = X + (size_t)r * kp.rstride + (size_t)(e >> 5) * NP * kLanes + (e & 31);
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m)
                    cp_async8(d + (v * NP + m) * kLanes + lane, xr + (size_t)v * kp.vstride + m * kLanes);
            if (r < je) {
                if constexpr (HAS_U) {
                    const double *ur = kp.U + lane_off + (size_t)r * kp.rstride;
#pragma unroll
                    for (int v = 0; v < 3; ++v)
#pragma unroll
                        for (int m = 0; m < NP; ++m)
                            cp_async8(d + ROWW + (v * NP + m) * kLanes + lane, ur + (size_t)v * kp.vstride + m * kLanes);
                }
                const double *row = X + (size_t)r * kp.rstride;
                double *nb = d + (HAS_U ? 2 : 1) * ROWW;
                if (lft) {
                    const double *b = row + (size_t)(eL >> 5) * NP * kLanes + (eL & 31);
#pragma unroll
                    for (int v = 0; v < 3; ++v)
#pragma unroll
                        for (int m = 0; m < NP; ++m) cp_async8(nb + v * NP + m, b + (size_t)v * kp.vstride + m * kLanes);
                }
                if (rgt) {
                    const double *b = row + (size_t)(eR >> 5) * NP * kLanes + (eR & 31);
#pragma unroll
                    for (int v = 0; v < 3; ++v)
#pragma unroll
                        for (int m = 0; m < NP; ++m)
                            cp_async8(nb + 3 * NP + v * NP + m, b + (size_t)v * kp.vstride + m * kLanes);
                }
            }
        }
        cp_commit();
    };
    auto xrow = [&](int slot, double (&u)[3][NP]) {
        const double *d = ring + slot * SLOT;
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int m = 0; m < NP; ++m) u[v][m] = d[(v * NP + m) * kLanes + lane];
    };
#pragma unroll 1
    for (int k = 0; k < kLoDepth - 1; ++k) issue(jb + k, k);

    double cur[3][NP], nxt[3][NP];
    lo_load<P>(X + (size_t)jb * kp.rstride, kp.vstride, e, cur);
    // the face below row jb: row jb-1's top traces against row jb's bottom ones
    double fbot[3][N];
    {
        double bt[3][N];
        lo_ytraces<P, true>(cur, bt);
        bad |= owned & lo_positive<P>(bt[0], N);
        if (kp.row0 + jb > 0) {
            double below[3][NP], tt[3][N];
            lo_load<P>(X + (size_t)(jb - 1) * kp.rstride, kp.vstride, e, below);
            lo_ytraces<P, false>(below, tt);
            const double *rw = kp.rowtab + (size_t)(kp.row0 + jb) * RL::STRIDE;
            lo_face<P>(tt, bt, FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode,
                                        1, rw[RL::CRB], rw[RL::COSB], alpha_y, kp.bdx}, fbot);
        } else {
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int k = 0; k < N; ++k) fbot[v][k] = 0.0;   // a pole: no face (dg.py:483-495)
        }
    }

    int slot = 0;                                                // ring slot of row j
    for (int j = jb; j < je; ++j) {
        const bool has_next = j + 1 <= r_last;
        const int slot1 = slot + 1 == kLoDepth ? 0 : slot + 1;
        const int slotD = slot == 0 ? kLoDepth - 1 : slot - 1;   // row j + kLoDepth - 1
        issue(j + kLoDepth - 1, slotD);
        cp_wait<kLoDepth - 2>();                                 // rows <= j + 1 have landed
        if (has_next) xrow(slot1, nxt);
        double un[3][NP];
        if constexpr (HAS_U) {
            const double *d = ring + slot * SLOT + ROWW;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m) un[v][m] = d[(v * NP + m) * kLanes + lane];
        }
        double nbl[3][NP], nbr[3][NP];   // lane 0's left / the last lane's right neighbour
        {
            const double *nb = ring + slot * SLOT + (HAS_U ? 2 : 1) * ROWW;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int m = 0; m < NP; ++m) {
                    nbl[v][m] = nb[v * NP + m];
                    nbr[v][m] = nb[3 * NP + v * NP + m];
                }
        }
        slot = slot1;
        const double *rw = kp.rowtab + (size_t)(kp.row0 + j) * RL::STRIDE;
        // traces of row j (and positivity of the h nodes and traces)
        double lt[3][N], rt[3][N], tt[3][N];
        lo_xtraces<P, true>(cur, lt);
        lo_xtraces<P, false>(cur, rt);
        lo_ytraces<P, false>(cur, tt);
        bad |= owned & (lo_positive<P>(lt[0], N) | lo_positive<P>(rt[0], N) | lo_positive<P>(tt[0], N) |
                        lo_positive<P>(cur[0], NP));
        // x-faces: the right face of every lane from lane+1's L trace; the
        // last valid lane's neighbour (and lane 0's left one) from memory
        double nl[3][N];
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int k = 0; k < N; ++k) nl[v][k] = lo_shfl<P>(lt[v][k], 1, true);
        if (rgt) lo_xtraces<P, true>(nbr, nl);
        double fr[3][N], fl[3][N];
        lo_face<P>(rt, nl, fx, fr);
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int k = 0; k < N; ++k) fl[v][k] = lo_shfl<P>(fr[v][k], 1, false);
        if (lft) {
            double nr[3][N];
            lo_xtraces<P, false>(nbl, nr);
            lo_face<P>(nr, lt, fx, fl);
        }
        // the y-face above row j (zero at the pole), carried to the next row
        double ftop[3][N];
        if (has_next) {
            double bt[3][N];
            lo_ytraces<P, true>(nxt, bt);
            bad |= owned & lo_positive<P>(bt[0], N);
            const double *ra = rw + RL::STRIDE;
            lo_face<P>(tt, bt, FaceArgs{kp.h_floor, kp.inv_floor, kp.sqrt_g, kp.half_g, kp.inv_r, kp.alpha_mode,
                                        1, ra[RL::CRB], ra[RL::COSB], alpha_y, kp.bdx}, ftop);
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
            double *Yv = kp.Y + lane_off + (size_t)v * kp.vstride + (size_t)j * kp.rstride;
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
        // slide the window: the next row's bottom face is this row's top face
        if (has_next) {
#pragma unroll
            for (int v = 0; v < 3; ++v) {
#pragma unroll
                for (int m = 0; m < NP; ++m) cur[v][m] = nxt[v][m];
#pragma unroll
                for (int k = 0; k < N; ++k) fbot[v][k] = ftop[v][k];
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
