// dgswe_ctx.h -- the C-ABI context (internal), shared by the ABI unit
// (dgswe_b200.cu) and the per-degree launcher units (deg_p*.cu).
//
// The context owns only what SURVEY.md section 8(b) allows: the uploaded
// constant tables (per-row table, edge cosines, orography factors), the
// status words, the global-alpha pair, fixed-size diagnostics scratch (all
// allocated in dgswe_create) and cached CUDA graphs.  Every state buffer
// belongs to the caller; no entry point allocates device memory.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <tuple>

#include "../../include/dgswe_b200.h"
#include "dgswe_params.h"

int dgswe_fail(int code, const char *fmt, ...);

#define CUDA_TRY(expr)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return dgswe_fail(DGSWE_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                              __LINE__);                                                          \
    } while (0)

struct DevStatus {
    unsigned flags;
    int first_tag[dgswe::kStatusBits];   // smallest tag that raised each bit
};

struct GraphKey {
    int order;
    double *u, *w1, *w2, *w3;
    double dt;
    int nsteps, check_mean, basis;
    bool operator<(const GraphKey &o) const
    {
        return std::tie(order, u, w1, w2, w3, dt, nsteps, check_mean, basis) <
               std::tie(o.order, o.u, o.w1, o.w2, o.w3, o.dt, o.nsteps, o.check_mean, o.basis);
    }
};

// One stage launch: Y = a U + b X + g RHS(X) [, Y2 = A + g2 RHS(X)] on local
// rows [r0, r1) (and [r2, r3) in the same launch)
struct StageCall {
    double a = 0.0, b = 0.0, g = 0.0, g2 = 0.0;
    const double *U = nullptr, *X = nullptr, *A = nullptr;
    double *Y = nullptr, *Y2 = nullptr;
    int tag = 0, r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    int check_finite = 0, check_mean = 0;
    bool modal = false;   // modal X/U/A/Y/Y2 (in-kernel conversion)
    bool edge = false;    // band edge rows of the fused halo exchange
};

// Kernels of one degree, compiled in their own translation unit (deg_pP.cu)
// with that unit's __constant__ nodal tables.
struct DegreeOps {
    int (*upload)(const dgswe::NodTab &nt);
    int (*stage)(dgswe_ctx *c, const dgswe::StageParams &kp, cudaStream_t s);
    int (*convert)(dgswe_ctx *c, const double *in, double *out, bool to_nodal, int r0, int r1, cudaStream_t s);
    int (*alpha)(dgswe_ctx *c, const double *X, bool modal, cudaStream_t s);
    int (*project)(dgswe_ctx *c, const double *f, const double *cosn, double determ, double *Y, cudaStream_t s);
    // linear advection on the periodic plane (dgswe_adv.cuh)
    int (*adv_stage)(const dgswe::AdvParams &ap, int nz, cudaStream_t s);
};
const DegreeOps *dgswe_degree_ops(int p);

struct dgswe_ctx {
    dgswe_cfg cfg;
    int n, nphi, rc;
    long long vstride, rstride, zstride;
    int nstrip;
    double *rowtab = nullptr;     // device, ny * row_stride(p)
    double *cos_edge = nullptr;   // device, ny+1
    double *alpha = nullptr;      // device, 2 doubles
    DevStatus *status = nullptr;  // device
    DevStatus *status_host = nullptr;   // pinned host [2]: last read, reset value
    double *orog = nullptr;       // device [nrows][2][nstrip][nphi][32] orography factors, or null
    unsigned char *orog_mask = nullptr;   // device [nrows][nstrip]: 1 where a strip's factor tile is non-zero
    int external_alpha = 0;
    long long launches = 0;
    int device = 0;
    int sms = 148;
    int smem_pad = 0;             // experiment knob: extra dynamic smem per CTA
    int even_chunks = 0;          // experiment knob (DGSWE_CHUNKS): fixed chunk count, even split
    int occ_lo[2] = {};           // resident CTAs per SM of the low-order kernel (without / with u^n)
    int no_lo = 0;                // experiment knob (DGSWE_NO_LO): p <= 1 on the main kernel
    int occ[32] = {};             // resident CTAs per SM of each stage-kernel variant (0: not queried)
    // fused halo exchange (bands.py transport "fused"): set by dgswe_set_exchange
    long long peer_zstride[2] = {0, 0};
    unsigned long long *peer_count[2] = {nullptr, nullptr};
    unsigned long long *recv_count = nullptr, *stage_ctr = nullptr;
    unsigned long long peer_timeout_ns = 2000000000ull;   // 2 s
    double *edge_row[2] = {nullptr, nullptr};
    std::map<GraphKey, cudaGraphExec_t> graphs;
    double *diag = nullptr;       // device scratch for diagnostics / projection (fixed size, create)
    size_t diag_doubles = 0;
    int nq2_max = 0;              // largest l2 rule the scratch holds
    // derived scalars
    double inv_r, inv_r_cx, half_g, bdx, bdy;
    double dx[dgswe::kMaxP + 1][dgswe::kMaxP + 1];   // inv_r_cx * dh (StageParams::dx)
    // state basis of the stage entry points: 0 modal (the reference's
    // coefficients; converted inside the kernel), 1 nodal (dgswe_set_basis)
    int basis = 0;
    const DegreeOps *ops = nullptr;
};
