// dgswe_params.h -- plain structs shared by the host launchers and the
// sm_100a kernels (no device symbols: every degree's translation unit owns
// its __constant__ tables, see dgswe_kernels.cuh).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgswe {

constexpr int kMaxP = 6;
constexpr int kLanes = 32;   // elements per strip (== DGSWE_STRIP)
constexpr int kVarWarps = 3; // one per conserved variable
constexpr int kWarps = 4;    // + one face warp (Rusanov fluxes)
constexpr int kThreads = kWarps * kLanes;

// stage kernel variant bits
constexpr int kHasU = 1;    // Y = a U + ...: reads u^n
constexpr int kHasY2 = 2;   // second output Y2 = A + g2 RHS(X) (classical RK4)
constexpr int kEdge = 4;    // band edge rows of the fused halo exchange (peer stores + counters)
constexpr int kModal = 8;   // modal X / U / A / Y / Y2 (converted inside the kernel)
constexpr int kOrog = 16;   // bottom-topography source -g h grad b (TC5)

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
    int even;                 // > 0: the first range (edge launches: the interior rows) is split
                              // into `even` chunks of floor/ceil(rows/even) rows instead of rc
    int j_begin2, j_end2;
    double a, b, g;       // Y = a U + b X + g RHS(X)
    double dx[kMaxP + 1][kMaxP + 1];   // (1/R)(determ/bd_det_x) dh: the xi derivative of F
    const double *rowtab; // per global row, see RowLayout
    double inv_r;         // 1/R
    double inv_r_cx;      // (1/R) * determ/bd_det_x
    double gravity, half_g, h_floor, inv_floor, sqrt_g;
    double bdx, bdy;      // bd_det_x, bd_det_y
    int alpha_mode;       // 0 local, 1 pinned, 2 global (from alpha_dev)
    double alpha;
    const double *alpha_dev;
    unsigned *status;
    int *first_tag;       // [kStatusBits]: smallest tag that raised each status bit
    int tag;
    int check_finite;
    int check_mean;
    // fused halo exchange over peer memory (edge launches of a latitude
    // band, bands.py transport "fused"): [0] south, [1] north neighbour
    int edge;                           // 1: this launch computes the band's edge rows
    int modal;                          // 1: modal states (dispatch only; the kernel variant knows)
    int band_lo, band_hi;               // the band's computed rows [band_lo, band_hi)
    double *peer_row[2];                // neighbour's halo row (level 0) our edge row is copied to
    long long peer_zstride[2];
    unsigned long long *peer_count[2];  // neighbour's receive counter for that halo
    const unsigned long long *recv_count;   // own receive counters [2] (system-scope atomics)
    unsigned long long *stage_ctr;      // own [0] completed edge launches, [1] CTA completions
    unsigned long long peer_timeout_ns; // bound on the wait for a neighbour's rows
    // orography (kOrog): per buffer row [2][nstrip][nphi][32], the nodal source
    // factors -(g/R) db/dlambda and -(g cos/R) db/dtheta with determ folded in
    const double *orog;
    long long orog_rstride;             // doubles per row of `orog` (2 * vstride / 3)
    const unsigned char *orog_mask;     // [nrows][nstrip]: 0 = the row's factor tile is all zero
    int periodic_y;                     // 1: y-periodic (planar) mesh, rows wrap, no poles
};

constexpr int kStatusBits = 4;          // POSITIVITY, NONFINITE, MEAN_NONPOS, PEER_TIMEOUT
constexpr unsigned kPeerTimeout = 8u;

// per-row table layout (doubles): crc[n] srs[n] fcs[n] cr_b cos_b rj[n] T[n][n]
template <int P>
struct RowLayout {
    static constexpr int N = P + 1;
    static constexpr int CRC = 0;
    static constexpr int SRS = N;
    static constexpr int FCS = 2 * N;
    static constexpr int CRB = 3 * N;
    static constexpr int COSB = 3 * N + 1;
    static constexpr int RJ = 3 * N + 2;     // 1 / (determ cos_j): the nodal mass
    static constexpr int SSTRIDE = RJ + N;   // the part staged in shared memory
    static constexpr int T = SSTRIDE;        // theta block of M^-1 (modal; device IC projection only)
    static constexpr int STRIDE = T + N * N;
};

__host__ __device__ inline int row_stride(int p) { return 4 * (p + 1) + 2 + (p + 1) * (p + 1); }

// Nodal (Gauss-Lagrange) tables of degree P, built on the host from the
// Legendre tables (dgswe_b200.cu, dgswe_create): with l_i the Lagrange
// polynomial of Gauss node x_i,
//   lm[i]    = l_i(-1)                (l_i(+1) = l_{N-1-i}(-1))
//   mu[i]    = l_i(-1) / w_i          (boundary lift of a face value)
//   dh[i][k] = w_k l_i'(x_k) / w_i    (weak derivative, W^-1 D^T W)
//   w[i]     = w_i
// The state is carried at the (p+1)^2 Gauss nodes inside a step: the
// reference's modal scheme with every integral on the same (p+1)-point Gauss
// rule (dg.py:186-213, basis.py:159-177) is, in the Lagrange basis of those
// nodes, the same linear operator with a diagonal mass matrix
// determ w_i w_j cos_j (exact algebra; only the rounding differs).
//   leg[a][i] = P_a(x_i)          (modal -> nodal, basis.py:118-133)
//   wp[a][i]  = w_i P_a(x_i)      (nodal -> modal moments; the (2a+1)/2
//                                  normalisation is applied after)
struct NodTab {
    double lm[kMaxP + 1];
    double mu[kMaxP + 1];
    double dh[kMaxP + 1][kMaxP + 1];
    double w[kMaxP + 1];
    double leg[kMaxP + 1][kMaxP + 1];
    double wp[kMaxP + 1][kMaxP + 1];
};
// one stage of the linear advection kernel (dgswe_adv.cuh): Y = a U + b X
// + g RHS(X), states [nz][ny][nphi][nx] of modal coefficients
struct AdvParams {
    const double *X, *U;
    double *Y;
    double a, b, g;
    int nx, ny;
    long long zstride;                 // nx * ny * nphi
    double bx, by;                     // advection velocity
    double ax, ay;                     // Rusanov alpha per direction: |bx|, |by| or a pinned value
    double bdx, bdy;                   // face Jacobians dx/2, dy/2
    double cx, cy;                     // determ / bd_det_x, determ / bd_det_y (dg.py:199-202)
    double inv_determ;                 // the nodal mass 1 / determ
    int rc;                            // rows per CTA (row-marching kernel)
};

// strided view of a state for the diagnostics / projection kernels
struct DiagLayout {
    long long zstride, rstride, vstride;
    int nx, ny, nphi;
};

}  // namespace dgswe
