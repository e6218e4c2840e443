// dgswe_b200.cu -- C ABI (include/dgswe_b200.h) over the sm_100a fp64 DG
// shallow-water kernels in dgswe_kernels.cuh.
//
// The context owns only constant tables (uploaded once, as the reference
// precomputes on the host, dg.py:186-219), a status word, the global-alpha
// buffer and cached CUDA graphs; all state buffers belong to the caller.

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/dgswe_b200.h"
#include "dgswe_kernels.cuh"
#include "dgswe_diag.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(DGSWE_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                         \
    } while (0)

struct DevStatus {
    unsigned flags;
    int first_tag;
};

// global-mode alpha: max over all traces (dg.py:389-411, models.py:271-280), nodal state
template <int P>
__global__ void alpha_prepass_kernel(const double *__restrict__ X, long long zstride,
                                     long long rstride, long long vstride, int nx, int ny, int row0,
                                     int jlo, int jhi,
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
        for (int q = 0; q < N; ++q) {
            double l = 0, r = 0, bo = 0, t = 0;
            for (int k = 0; k < N; ++k) {
                const double lo = dgswe::c_nod[P].lm[k], hi = dgswe::c_nod[P].lm[N - 1 - k];
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
    atomicMax(reinterpret_cast<unsigned long long *>(out + 1),
              (unsigned long long)__double_as_longlong(ay));
}

// y = y + x*coef with two roundings (timestep.py:137-141)
__global__ void axpy_kernel(const double *__restrict__ x, double *__restrict__ y, double coef,
                            long long zstride, long long off, long long count, int check,
                            DevStatus *st, int tag)
{
    const double *xz = x + (size_t)blockIdx.y * zstride + off;
    double *yz = y + (size_t)blockIdx.y * zstride + off;
    bool bad = false;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        const double t = __dmul_rn(xz[k], coef);
        const double r = __dadd_rn(yz[k], t);
        yz[k] = r;
        if (check && !isfinite(r)) bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
        atomicOr(&st->flags, DGSWE_STATUS_NONFINITE);
        atomicMin(&st->first_tag, tag);
    }
}

}  // namespace

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

struct dgswe_ctx {
    dgswe_cfg cfg;
    int n, nphi, rc;
    long long vstride, rstride, zstride;
    int nstrip;
    double *rowtab = nullptr;     // device, ny * row_stride(p)
    double *cos_edge = nullptr;   // device, ny+1
    double *alpha = nullptr;      // device, 2 doubles
    DevStatus *status = nullptr;  // device
    int external_alpha = 0;
    long long launches = 0;
    int device = 0;
    int sms = 148;
    int smem_pad = 0;             // experiment knob: extra dynamic smem per CTA
    int pdl = 0;                  // programmatic dependent launch of stages (DGSWE_PDL=1; measured -0.7% at C3)
    // fused halo exchange (bands.py transport "fused"): set by dgswe_set_exchange
    long long peer_zstride[2] = {0, 0};
    unsigned long long *peer_count[2] = {nullptr, nullptr};
    unsigned long long *recv_count = nullptr, *stage_ctr = nullptr;
    double *edge_row[2] = {nullptr, nullptr};
    int edge_pending = 0;
    std::map<GraphKey, cudaGraphExec_t> graphs;
    double *diag = nullptr;       // device scratch for diagnostics (row partials + tables)
    size_t diag_bytes = 0;
    // derived scalars
    double inv_r, inv_r_cx, half_g, bdx, bdy;
    double dx[dgswe::kMaxP + 1][dgswe::kMaxP + 1];   // inv_r_cx * dh (StageParams::dx)
    // state basis of the stage entry points: 0 modal (the reference's
    // coefficients; converted around every launch), 1 nodal (as stored
    // inside dgswe_rk_steps; dgswe_set_basis)
    int basis = 0;
    double *scr[3] = {nullptr, nullptr, nullptr};   // modal-basis staging (X, U, A)
};

namespace {

template <int P, bool HU, bool HY, bool ED>
int setup_variant(int dev, size_t smem, int (&occ)[64][6])
{
    const int var = ED ? 4 + (HU ? 1 : 0) : (HU ? 1 : 0) + (HY ? 2 : 0);
    if (!occ[dev][var]) {
        CUDA_TRY(cudaFuncSetAttribute(dgswe::stage_kernel<P, HU, HY, ED>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int o = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, dgswe::stage_kernel<P, HU, HY, ED>,
                                                               dgswe::kThreads, smem));
        occ[dev][var] = o > 0 ? o : 1;
    }
    return occ[dev][var];
}

cudaError_t launch_pdl(void (*kern)(dgswe::StageParams), dim3 grid, size_t smem, cudaStream_t s, bool pdl,
                       const dgswe::StageParams &kq)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(dgswe::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, kq);
}

template <int P>
int launch_stage_p(dgswe_ctx *c, const dgswe::StageParams &kp, int r0, int r1, cudaStream_t s)
{
    using SM = dgswe::Smem<P>;
    const int rows = (r1 - r0) > (kp.j_end2 - kp.j_begin2) ? (r1 - r0) : (kp.j_end2 - kp.j_begin2);
    if (rows <= 0) return DGSWE_OK;
    const size_t smem = (size_t)SM::TOTAL * sizeof(double) + (size_t)c->smem_pad;
    static int occ[64][6] = {};     // resident CTAs per SM, per device and variant
    static size_t occ_smem[64] = {};
    const int dev = c->device & 63;
    if (occ_smem[dev] != smem) {
        for (int k = 0; k < 6; ++k) occ[dev][k] = 0;
        occ_smem[dev] = smem;
    }
    const bool hu = kp.U != nullptr, hy = kp.Y2 != nullptr, ed = kp.edge != 0;
    if (ed && hy) return fail(DGSWE_EUNSUPPORTED, "edge launches have one output");
    int o;
    if (ed)
        o = hu ? setup_variant<P, true, false, true>(dev, smem, occ)
               : setup_variant<P, false, false, true>(dev, smem, occ);
    else if (hy)
        o = hu ? setup_variant<P, true, true, false>(dev, smem, occ)
               : setup_variant<P, false, true, false>(dev, smem, occ);
    else
        o = hu ? setup_variant<P, true, false, false>(dev, smem, occ)
               : setup_variant<P, false, false, false>(dev, smem, occ);
    if (o < 0) return o;
    // Row chunking: every (strip, level) column of rows is split into
    // contiguous chunks, one CTA each.  The chunk count minimises the
    // modelled makespan  waves * (rows per chunk + kChunkOverhead), where
    // waves = ceil(CTAs / resident slots) and the overhead (prologue and
    // first-row work, measured ~1.4 rows) favours long chunks.  Narrow grids
    // get one full wave (C3: 23 strips x 24 chunks of 15 rows); wide grids,
    // whose strips alone outnumber the slots, get several waves of short
    // chunks instead of one under-filled wave of very long ones.
    const int strips = c->nstrip;
    int rc = kp.edge ? 1 : kp.rc;
    if (rc <= 0) {
        constexpr double kChunkOverhead = 1.5;
        const long long slots = (long long)c->sms * o;
        const long long cols = (long long)strips * c->cfg.nz;
        double best = 1e300;
        long long best_chunks = 1;
        const long long max_chunks = rows < 4 * slots ? rows : 4 * slots;
        for (long long ch = 1; ch <= max_chunks; ++ch) {
            const long long per = (rows + ch - 1) / ch;
            if (ch > 1 && (rows + ch - 2) / (ch - 1) == per) continue;   // same chunk length
            const long long waves = (cols * ch + slots - 1) / slots;
            const double t = (double)waves * ((double)per + kChunkOverhead);
            if (t < best - 1e-9) {
                best = t;
                best_chunks = ch;
            }
        }
        // Second look, by the busiest SM's row work: CTAs share their SM's
        // issue and FP64 throughput, so a one-wave grid that puts o CTAs on
        // some SMs and o-1 on the others runs at the pace of the former.
        // Chunks long enough for at most o-1 CTAs per SM win when that
        // load is clearly lower (C3: 23 strips x 19 chunks of 19 rows, 3
        // per SM, instead of 24 chunks of 15, 4 on 108 SMs: +1.4%; C2 +2%).
        // Measured for p = 3 only: at p = 2 the lighter CTAs want the 4th
        // CTA's latency hiding (-3%), at p >= 4 o - 1 = 1 CTA per SM.
        if (P == 3 && o > 1) {
            auto sm_load = [&](long long ch) {
                const long long per = (rows + ch - 1) / ch;
                const long long per_sm = (cols * ch + c->sms - 1) / c->sms;
                return (double)per_sm * ((double)per + 1.0);
            };
            const double cur = sm_load(best_chunks);
            long long alt = 0;
            double alt_cost = 1e300;
            for (long long ch = 1; ch <= rows && cols * ch <= (long long)c->sms * (o - 1); ++ch) {
                if ((cols * ch + c->sms - 1) / c->sms != o - 1) continue;   // exactly o-1 on the busiest SM
                const double t = sm_load(ch);
                if (t < alt_cost - 1e-9) {
                    alt_cost = t;
                    alt = ch;
                }
            }
            if (alt > 0 && alt_cost < 0.95 * cur) best_chunks = alt;
        }
        rc = (int)((rows + best_chunks - 1) / best_chunks);
    }
    dgswe::StageParams kq = kp;
    kq.rc = rc;
    int nchunks = (rows + rc - 1) / rc;
    if (kp.j_end2 > kp.j_begin2) {   // a second row range in the same launch
        kq.nchunk1 = nchunks;
        nchunks += (kp.j_end2 - kp.j_begin2 + rc - 1) / rc;
    }
    dim3 grid(strips, nchunks, c->cfg.nz);
    // programmatic dependent launch (overlaps this stage's prologue with the
    // previous kernel's tail); edge launches keep plain stream order
    const bool pdl = c->pdl && !ed;
    cudaError_t le;
    if (ed) {
        le = hu ? launch_pdl(dgswe::stage_kernel<P, true, false, true>, grid, smem, s, false, kq)
                : launch_pdl(dgswe::stage_kernel<P, false, false, true>, grid, smem, s, false, kq);
    } else if (hy) {
        le = hu ? launch_pdl(dgswe::stage_kernel<P, true, true, false>, grid, smem, s, pdl, kq)
                : launch_pdl(dgswe::stage_kernel<P, false, true, false>, grid, smem, s, pdl, kq);
    } else {
        le = hu ? launch_pdl(dgswe::stage_kernel<P, true, false, false>, grid, smem, s, pdl, kq)
                : launch_pdl(dgswe::stage_kernel<P, false, false, false>, grid, smem, s, pdl, kq);
    }
    CUDA_TRY(le);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

int alpha_prepass_nodal(dgswe_ctx *c, const double *X, cudaStream_t s);

// Y = a U + b X + g RHS(X) [, Y2 = A + g2 RHS(X)] on local rows [r0, r1),
// every state in the nodal basis
int launch_stage(dgswe_ctx *c, double a, const double *U, double b, const double *X, double g,
                 double *Y, const double *A, double g2, double *Y2, int tag, int r0, int r1,
                 int check_finite, int check_mean, cudaStream_t s, int r2 = 0, int r3 = 0)
{
    if (!X || !Y) return fail(DGSWE_EINVAL, "null state pointer");
    if (X == Y || X == Y2) return fail(DGSWE_EINVAL, "outputs must not alias the stage input");
    if (Y2 && (Y2 == Y || !A)) return fail(DGSWE_EINVAL, "second output needs its own buffer and an addend");
    if (a != 0.0 && !U) return fail(DGSWE_EINVAL, "U is required when a != 0");
    if (r0 < c->cfg.jlo || r1 > c->cfg.jhi || r0 > r1)
        return fail(DGSWE_EINVAL, "row range [%d,%d) outside [%d,%d)", r0, r1, c->cfg.jlo, c->cfg.jhi);
    dgswe::StageParams kp = {};
    kp.X = X;
    kp.U = (a != 0.0) ? U : nullptr;
    kp.Y = Y;
    kp.A = Y2 ? A : nullptr;
    kp.Y2 = Y2;
    kp.g2 = g2;
    kp.zstride = c->zstride;
    kp.rstride = c->rstride;
    kp.vstride = c->vstride;
    kp.nstrip = c->nstrip;
    kp.nx = c->cfg.nx;
    kp.ny = c->cfg.ny;
    kp.row0 = c->cfg.row0;
    kp.nrows = c->cfg.nrows;
    kp.j_begin = r0;
    kp.j_end = r1;
    kp.nchunk1 = INT_MAX;
    kp.j_begin2 = r2;
    kp.j_end2 = r3;
    if (r3 > r2 && (r2 < c->cfg.jlo || r3 > c->cfg.jhi || r2 < r1))
        return fail(DGSWE_EINVAL, "second row range [%d,%d) invalid", r2, r3);
    kp.rc = c->rc;
    kp.a = a;
    kp.b = b;
    kp.g = g;
    memcpy(kp.dx, c->dx, sizeof kp.dx);
    kp.rowtab = c->rowtab;
    kp.inv_r = c->inv_r;
    kp.inv_r_cx = c->inv_r_cx;
    kp.gravity = c->cfg.gravity;
    kp.half_g = c->half_g;
    kp.h_floor = c->cfg.h_floor;
    kp.inv_floor = 1.0 / c->cfg.h_floor;
    kp.sqrt_g = sqrt(c->cfg.gravity);
    kp.bdx = c->bdx;
    kp.bdy = c->bdy;
    kp.alpha_mode = c->cfg.alpha_mode;
    kp.alpha = c->cfg.alpha;
    kp.alpha_dev = c->alpha;
    kp.status = &c->status->flags;
    kp.first_tag = &c->status->first_tag;
    kp.tag = tag;
    kp.check_finite = check_finite;
    kp.check_mean = check_mean;
    if (c->edge_pending) {
        kp.edge = 1;
        kp.band_lo = c->cfg.jlo;
        kp.band_hi = c->cfg.jhi;
        for (int k = 0; k < 2; ++k) {
            kp.peer_row[k] = c->edge_row[k];
            kp.peer_zstride[k] = c->peer_zstride[k];
            kp.peer_count[k] = c->edge_row[k] ? c->peer_count[k] : nullptr;
        }
        kp.recv_count = c->recv_count;
        kp.stage_ctr = c->stage_ctr;
    }
    if (c->cfg.alpha_mode == DGSWE_ALPHA_GLOBAL && !c->external_alpha) {
        int rc = alpha_prepass_nodal(c, X, s);
        if (rc) return rc;
    }
    switch (c->cfg.p) {
    case 0: return launch_stage_p<0>(c, kp, r0, r1, s);
    case 1: return launch_stage_p<1>(c, kp, r0, r1, s);
    case 2: return launch_stage_p<2>(c, kp, r0, r1, s);
    case 3: return launch_stage_p<3>(c, kp, r0, r1, s);
    case 4: return launch_stage_p<4>(c, kp, r0, r1, s);
    case 5: return launch_stage_p<5>(c, kp, r0, r1, s);
    case 6: return launch_stage_p<6>(c, kp, r0, r1, s);
    default: return fail(DGSWE_EUNSUPPORTED, "degree p=%d not supported (0..6)", c->cfg.p);
    }
}

template <int P>
int launch_alpha_p(dgswe_ctx *c, const double *X, cudaStream_t s)
{
    const int rows = c->cfg.jhi - c->cfg.jlo;
    dim3 grid((c->cfg.nx + 127) / 128, rows, c->cfg.nz);
    alpha_prepass_kernel<P><<<grid, 128, 0, s>>>(X, c->zstride, c->rstride, c->vstride, c->cfg.nx,
                                                   c->cfg.ny,
                                                   c->cfg.row0, c->cfg.jlo, c->cfg.jhi, c->cos_edge,
                                                   c->inv_r, c->cfg.gravity, c->cfg.h_floor, c->alpha);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

int alpha_prepass_nodal(dgswe_ctx *ctx, const double *X, cudaStream_t s)
{
    CUDA_TRY(cudaMemsetAsync(ctx->alpha, 0, 2 * sizeof(double), s));
    switch (ctx->cfg.p) {
    case 0: return launch_alpha_p<0>(ctx, X, s);
    case 1: return launch_alpha_p<1>(ctx, X, s);
    case 2: return launch_alpha_p<2>(ctx, X, s);
    case 3: return launch_alpha_p<3>(ctx, X, s);
    case 4: return launch_alpha_p<4>(ctx, X, s);
    case 5: return launch_alpha_p<5>(ctx, X, s);
    case 6: return launch_alpha_p<6>(ctx, X, s);
    default: return fail(DGSWE_EUNSUPPORTED, "degree not supported");
    }
}

template <int P>
int convert_p(dgswe_ctx *c, const double *in, double *out, bool to_nodal, int r0, int r1, cudaStream_t s)
{
    dim3 grid(c->nstrip, r1 - r0, c->cfg.nz);
    if (to_nodal)
        dgswe::convert_kernel<P, true><<<grid, 96, 0, s>>>(in, out, c->zstride, c->rstride, c->vstride, r0);
    else
        dgswe::convert_kernel<P, false><<<grid, 96, 0, s>>>(in, out, c->zstride, c->rstride, c->vstride, r0);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

// change of basis of local rows [r0, r1), every level (in may equal out)
int convert_rows(dgswe_ctx *c, const double *in, double *out, bool to_nodal, int r0, int r1, cudaStream_t s)
{
    if (r1 <= r0) return DGSWE_OK;
    switch (c->cfg.p) {
    case 0: return convert_p<0>(c, in, out, to_nodal, r0, r1, s);
    case 1: return convert_p<1>(c, in, out, to_nodal, r0, r1, s);
    case 2: return convert_p<2>(c, in, out, to_nodal, r0, r1, s);
    case 3: return convert_p<3>(c, in, out, to_nodal, r0, r1, s);
    case 4: return convert_p<4>(c, in, out, to_nodal, r0, r1, s);
    case 5: return convert_p<5>(c, in, out, to_nodal, r0, r1, s);
    case 6: return convert_p<6>(c, in, out, to_nodal, r0, r1, s);
    default: return fail(DGSWE_EUNSUPPORTED, "degree not supported");
    }
}

int scratch_state(dgswe_ctx *c, int k, double **out)
{
    if (!c->scr[k]) CUDA_TRY(cudaMalloc(&c->scr[k], sizeof(double) * (size_t)c->zstride * c->cfg.nz));
    *out = c->scr[k];
    return DGSWE_OK;
}

// A stage through the public entry points: in the modal basis the inputs
// are converted into staging buffers (all local rows: X's halo rows are
// read), the nodal kernel writes Y / Y2, whose computed rows are converted
// back in place.  U may alias Y and A may alias Y2, as in launch_stage.
int api_stage(dgswe_ctx *c, double a, const double *U, double b, const double *X, double g, double *Y,
              const double *A, double g2, double *Y2, int tag, int r0, int r1, cudaStream_t s, int r2 = 0,
              int r3 = 0)
{
    if (c->basis) return launch_stage(c, a, U, b, X, g, Y, A, g2, Y2, tag, r0, r1, 0, 0, s, r2, r3);
    if (!X || !Y) return fail(DGSWE_EINVAL, "null state pointer");
    if (X == Y || X == Y2) return fail(DGSWE_EINVAL, "outputs must not alias the stage input");
    if (Y2 && (Y2 == Y || !A)) return fail(DGSWE_EINVAL, "second output needs its own buffer and an addend");
    if (a != 0.0 && !U) return fail(DGSWE_EINVAL, "U is required when a != 0");
    if (r0 < c->cfg.jlo || r1 > c->cfg.jhi || r0 > r1)
        return fail(DGSWE_EINVAL, "row range [%d,%d) outside [%d,%d)", r0, r1, c->cfg.jlo, c->cfg.jhi);
    const int nr = c->cfg.nrows;
    double *xs = nullptr, *us = nullptr, *as = nullptr;
    int rc = scratch_state(c, 0, &xs);
    if (!rc) rc = convert_rows(c, X, xs, true, 0, nr, s);
    if (!rc && a != 0.0) {
        rc = scratch_state(c, 1, &us);
        if (!rc) rc = convert_rows(c, U, us, true, r0, r3 > r2 ? r3 : r1, s);
    }
    if (!rc && Y2) {
        rc = scratch_state(c, 2, &as);
        if (!rc) rc = convert_rows(c, A, as, true, r0, r3 > r2 ? r3 : r1, s);
    }
    if (!rc) rc = launch_stage(c, a, us, b, xs, g, Y, as, g2, Y2, tag, r0, r1, 0, 0, s, r2, r3);
    for (double *o : {Y, Y2}) {
        if (rc || !o) continue;
        rc = convert_rows(c, o, o, false, r0, r1, s);
        if (!rc && r3 > r2) rc = convert_rows(c, o, o, false, r2, r3, s);
    }
    return rc;
}

}  // namespace

extern "C" {

int dgswe_abi_version(void) { return DGSWE_ABI_VERSION; }

const char *dgswe_last_error(void) { return g_last_error.c_str(); }

int dgswe_create(const dgswe_cfg *cfg, const dgswe_tables *t, dgswe_ctx **out)
{
    if (!cfg || !t || !out) return fail(DGSWE_EINVAL, "null argument");
    *out = nullptr;
    const dgswe_cfg &c = *cfg;
    if (c.p < 0 || c.p > dgswe::kMaxP) return fail(DGSWE_EUNSUPPORTED, "degree p=%d not supported (0..6)", c.p);
    if (c.nx < 1 || c.ny < 1 || c.nz < 1) return fail(DGSWE_EINVAL, "element counts must be >= 1");
    if (c.nrows < 1 || c.jlo < 0 || c.jhi > c.nrows || c.jlo >= c.jhi)
        return fail(DGSWE_EINVAL, "bad local rows: nrows=%d jlo=%d jhi=%d", c.nrows, c.jlo, c.jhi);
    if (c.row0 + c.jlo < 0 || c.row0 + c.jhi > c.ny) return fail(DGSWE_EINVAL, "band outside the sphere");
    if (c.row0 + c.jlo > 0 && c.jlo < 1) return fail(DGSWE_EINVAL, "band needs a southern halo row");
    if (c.row0 + c.jhi < c.ny && c.jhi >= c.nrows) return fail(DGSWE_EINVAL, "band needs a northern halo row");
    if (c.alpha_mode < 0 || c.alpha_mode > 2) return fail(DGSWE_EINVAL, "bad alpha mode");
    if (!(c.radius > 0) || !(c.gravity > 0) || !(c.dx > 0) || !(c.dy > 0))
        return fail(DGSWE_EINVAL, "radius, gravity, dx, dy must be positive");
    if (!t->leg || !t->dleg || !t->weights || !t->cos_r_int || !t->sin_r_int || !t->fcos_int ||
        !t->cos_r_edge || !t->cos_edge || !t->minv)
        return fail(DGSWE_EINVAL, "missing table");

    dgswe_ctx *ctx = new (std::nothrow) dgswe_ctx();
    if (!ctx) return fail(DGSWE_ENOMEM, "out of host memory");
    ctx->cfg = c;
    const int n = c.p + 1;
    ctx->n = n;
    ctx->nphi = n * n;
    ctx->nstrip = (c.nx + DGSWE_STRIP - 1) / DGSWE_STRIP;
    ctx->vstride = (long long)ctx->nstrip * ctx->nphi * DGSWE_STRIP;
    ctx->rstride = 3LL * ctx->vstride;
    ctx->zstride = ctx->rstride * c.nrows;
    cudaGetDevice(&ctx->device);

    // mesh scalars exactly as the reference forms them (mesh.py:66-84)
    const double determ = c.dx * c.dy / 4.0;
    ctx->bdx = c.dx / 2.0;
    ctx->bdy = c.dy / 2.0;
    const double cx = determ / ctx->bdx;   // volx factor (dg.py:199-200)
    const double cy = determ / ctx->bdy;   // voly factor (dg.py:201-202)
    const double cs = determ;              // src factor (dg.py:213)
    ctx->inv_r = 1.0 / c.radius;
    ctx->inv_r_cx = ctx->inv_r * cx;
    ctx->half_g = 0.5 * c.gravity;

    // rows per CTA: fixed, or 0 = sized at launch so the grid is one wave
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
    ctx->rc = c.row_chunk > 0 ? c.row_chunk : 0;
    if (const char *env = getenv("DGSWE_ROW_CHUNK")) ctx->rc = atoi(env);
    if (const char *env = getenv("DGSWE_SMEM_PAD")) ctx->smem_pad = atoi(env);
    if (const char *env = getenv("DGSWE_PDL")) ctx->pdl = atoi(env);

    // constant tables for this degree
    static double tab[4][dgswe::kMaxP + 1][dgswe::kMaxP + 1];
    memset(tab, 0, sizeof tab);
    for (int a = 0; a < n; ++a)
        for (int q = 0; q < n; ++q) {
            const double P = t->leg[a * n + q], D = t->dleg[a * n + q], w = t->weights[q];
            tab[0][a][q] = P;
            tab[1][a][q] = D;
            tab[2][a][q] = w * P;
            tab[3][a][q] = w * D;
        }
    cudaError_t e = cudaMemcpyToSymbol(dgswe::c_tab, tab, sizeof tab, sizeof tab * c.p);
    // nodal tables (dgswe_kernels.cuh NodTab) from the Legendre ones, in
    // long double: l_i(x) = sum_a (2a+1)/2 w_i P_a(x_i) P_a(x) (the Gauss
    // rule projects the degree-p Lagrange polynomial exactly)
    dgswe::NodTab nt;
    memset(&nt, 0, sizeof nt);
    for (int i = 0; i < n; ++i) {
        const long double wi = t->weights[i];
        long double lm = 0.0L;
        for (int a = 0; a < n; ++a)
            lm += 0.5L * (2 * a + 1) * wi * t->leg[a * n + i] * ((a & 1) ? -1.0L : 1.0L);
        nt.lm[i] = (double)lm;
        nt.mu[i] = (double)(lm / wi);
        nt.w[i] = (double)wi;
        for (int k = 0; k < n; ++k) {
            long double d = 0.0L;   // w_k l_i'(x_k) / w_i
            for (int a = 0; a < n; ++a)
                d += 0.5L * (2 * a + 1) * (long double)t->leg[a * n + i] * t->weights[k] * t->dleg[a * n + k];
            nt.dh[i][k] = (double)d;
        }
    }
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(dgswe::c_nod, &nt, sizeof nt, sizeof nt * c.p);
    if (e != cudaSuccess) {
        delete ctx;
        return fail(DGSWE_ECUDA, "constant upload: %s", cudaGetErrorString(e));
    }

    for (int i = 0; i <= dgswe::kMaxP; ++i)
        for (int k = 0; k <= dgswe::kMaxP; ++k) ctx->dx[i][k] = ctx->inv_r_cx * nt.dh[i][k];

    // per-row tables (global rows), layout RowLayout<P>
    const int rs = dgswe::row_stride(c.p);
    std::vector<double> rt((size_t)c.ny * rs);
    for (int j = 0; j < c.ny; ++j) {
        double *r = rt.data() + (size_t)j * rs;
        for (int q = 0; q < n; ++q) {
            r[q] = t->cos_r_int[j * n + q] * cy;
            r[n + q] = t->sin_r_int[j * n + q] * cs;
            r[2 * n + q] = t->fcos_int[j * n + q] * cs;
        }
        r[3 * n] = t->cos_r_edge[j];
        r[3 * n + 1] = t->cos_edge[j];
        const double *M = t->minv + (size_t)j * ctx->nphi * ctx->nphi;
        // nodal mass 1 / (determ cos_j) (the w_i w_j factors live in dh, mu)
        for (int q = 0; q < n; ++q)
            r[3 * n + 2 + q] = 1.0 / (determ * (t->cos_r_int[j * n + q] * c.radius));
        for (int b = 0; b < n; ++b)
            for (int bb = 0; bb < n; ++bb) r[4 * n + 2 + b * n + bb] = M[(size_t)b * ctx->nphi + bb];
    }
    bool ok = cudaMalloc(&ctx->rowtab, rt.size() * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->cos_edge, (c.ny + 1) * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->alpha, 2 * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->status, sizeof(DevStatus)) == cudaSuccess;
    if (ok) {
        DevStatus st0 = {0u, INT_MAX};
        ok = cudaMemcpy(ctx->rowtab, rt.data(), rt.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(ctx->cos_edge, t->cos_edge, (c.ny + 1) * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemset(ctx->alpha, 0, 2 * sizeof(double)) == cudaSuccess &&
             cudaMemcpy(ctx->status, &st0, sizeof st0, cudaMemcpyHostToDevice) == cudaSuccess;
    }
    if (!ok) {
        cudaError_t le = cudaGetLastError();
        dgswe_destroy(ctx);
        return fail(DGSWE_ECUDA, "device allocation/upload failed: %s", cudaGetErrorString(le));
    }
    *out = ctx;
    return DGSWE_OK;
}

void dgswe_destroy(dgswe_ctx *ctx)
{
    if (!ctx) return;
    for (auto &kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    cudaFree(ctx->rowtab);
    cudaFree(ctx->cos_edge);
    cudaFree(ctx->alpha);
    cudaFree(ctx->status);
    cudaFree(ctx->diag);
    for (double *p : ctx->scr) cudaFree(p);
    delete ctx;
}

int64_t dgswe_state_elems(const dgswe_ctx *ctx)
{
    return ctx ? (int64_t)ctx->zstride * ctx->cfg.nz : 0;
}

int dgswe_rhs(dgswe_ctx *ctx, const double *X, double *K, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, 0.0, nullptr, 0.0, X, 1.0, K, nullptr, 0.0, nullptr, 0, ctx->cfg.jlo, ctx->cfg.jhi,
                     (cudaStream_t)stream);
}

int dgswe_stage(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                double *Y, int tag, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, ctx->cfg.jlo, ctx->cfg.jhi,
                     (cudaStream_t)stream);
}

int dgswe_stage_rows(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                     double *Y, int tag, int r0, int r1, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, r0, r1, (cudaStream_t)stream);
}

int dgswe_set_exchange(dgswe_ctx *ctx, long long peer_zstride_s, unsigned long long *peer_count_s,
                       long long peer_zstride_n, unsigned long long *peer_count_n,
                       unsigned long long *recv_count, unsigned long long *stage_ctr)
{
    if (!ctx || !recv_count || !stage_ctr) return fail(DGSWE_EINVAL, "null argument");
    ctx->peer_zstride[0] = peer_zstride_s;
    ctx->peer_zstride[1] = peer_zstride_n;
    ctx->peer_count[0] = peer_count_s;
    ctx->peer_count[1] = peer_count_n;
    ctx->recv_count = recv_count;
    ctx->stage_ctr = stage_ctr;
    return DGSWE_OK;
}

int dgswe_stage_edge(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                     int tag, double *peer_row_s, double *peer_row_n, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    if (!ctx->stage_ctr) return fail(DGSWE_EINVAL, "dgswe_set_exchange first");
    if (!ctx->basis) return fail(DGSWE_EINVAL, "edge launches take nodal states (dgswe_set_basis)");
    const int lo = ctx->cfg.jlo, hi = ctx->cfg.jhi;
    ctx->edge_row[0] = peer_row_s;
    ctx->edge_row[1] = peer_row_n;
    ctx->edge_pending = 1;
    const int rc = hi - lo >= 2 ? launch_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, lo, lo + 1, 0, 0,
                                               (cudaStream_t)stream, hi - 1, hi)
                                : launch_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, lo, hi, 0, 0,
                                               (cudaStream_t)stream);
    ctx->edge_pending = 0;
    return rc;
}

int dgswe_dev_alloc(size_t bytes, void **out)
{
    if (!out) return fail(DGSWE_EINVAL, "null argument");
    CUDA_TRY(cudaMalloc(out, bytes));
    CUDA_TRY(cudaMemset(*out, 0, bytes));
    return DGSWE_OK;
}

int dgswe_dev_free(void *p)
{
    CUDA_TRY(cudaFree(p));
    return DGSWE_OK;
}

int dgswe_ipc_handle(void *p, char *out64)
{
    if (!p || !out64) return fail(DGSWE_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, p));
    memcpy(out64, &h, sizeof h);
    return DGSWE_OK;
}

int dgswe_ipc_open(const char *in64, void **out)
{
    if (!in64 || !out) return fail(DGSWE_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, in64, sizeof h);
    CUDA_TRY(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return DGSWE_OK;
}

int dgswe_ipc_close(void *p)
{
    CUDA_TRY(cudaIpcCloseMemHandle(p));
    return DGSWE_OK;
}

int dgswe_stage_rows2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                      double *Y, int tag, int r0, int r1, int r2, int r3, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, r0, r1, (cudaStream_t)stream, r2, r3);
}

int dgswe_stage_rows_checked(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                             double *Y, int tag, int r0, int r1, int check_finite, int check_mean,
                             void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    if (!ctx->basis) return fail(DGSWE_EINVAL, "checked row stages take nodal states (dgswe_set_basis)");
    return launch_stage(ctx, a, U, b, X, g, Y, nullptr, 0.0, nullptr, tag, r0, r1, check_finite ? 1 : 0,
                        check_mean ? 1 : 0, (cudaStream_t)stream);
}

int dgswe_stage2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                 double *Y, const double *A, double g2, double *Y2, int tag, int r0, int r1, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, a, U, b, X, g, Y, A, g2, Y2, tag, r0, r1, (cudaStream_t)stream);
}

int dgswe_axpy(dgswe_ctx *ctx, double coef, const double *x, double *y, int check_finite, int tag,
               void *stream)
{
    if (!ctx || !x || !y) return fail(DGSWE_EINVAL, "null argument");
    const long long off = (long long)ctx->cfg.jlo * ctx->rstride;
    const long long count = (long long)(ctx->cfg.jhi - ctx->cfg.jlo) * ctx->rstride;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    dim3 grid((unsigned)blocks, ctx->cfg.nz);
    axpy_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, y, coef, ctx->zstride, off, count,
                                                       check_finite, ctx->status, tag);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 1;
    return DGSWE_OK;
}

int dgswe_alpha_prepass(dgswe_ctx *ctx, const double *X, void *stream)
{
    if (!ctx || !X) return fail(DGSWE_EINVAL, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    if (ctx->basis) return alpha_prepass_nodal(ctx, X, s);
    double *xs = nullptr;
    int rc = scratch_state(ctx, 0, &xs);
    if (!rc) rc = convert_rows(ctx, X, xs, true, 0, ctx->cfg.nrows, s);
    return rc ? rc : alpha_prepass_nodal(ctx, xs, s);
}

int dgswe_set_basis(dgswe_ctx *ctx, int nodal)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    ctx->basis = nodal ? 1 : 0;
    return DGSWE_OK;
}

int dgswe_convert(dgswe_ctx *ctx, double *X, int to_nodal, int r0, int r1, void *stream)
{
    if (!ctx || !X) return fail(DGSWE_EINVAL, "null argument");
    if (r0 < 0 || r1 > ctx->cfg.nrows || r0 > r1) return fail(DGSWE_EINVAL, "bad row range [%d,%d)", r0, r1);
    return convert_rows(ctx, X, X, to_nodal != 0, r0, r1, (cudaStream_t)stream);
}

double *dgswe_alpha_buffer(dgswe_ctx *ctx) { return ctx ? ctx->alpha : nullptr; }

int dgswe_set_external_alpha(dgswe_ctx *ctx, int external)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    ctx->external_alpha = external ? 1 : 0;
    return DGSWE_OK;
}

// K steps of the fused explicit RK method of `order` (the tableaux of
// timestep.py:57-82, evaluated in stage form; every stage is one kernel):
//   1: forward Euler, ping-pong u <-> w1 (a final copy when K is odd)
//   2: Heun == SSPRK2 Shu-Osher: w1 = u + dt L(u); u = u/2 + (w1 + dt L(w1))/2
//   3: SSPRK3 Shu-Osher (== tableau(3), timestep.py:65-70)
//   4: classical RK4 (timestep.py:71-81) with the accumulator as the stage
//      kernel's second output: acc = u + dt/6 k1 (+ dt/3 k2 + dt/3 k3),
//      stage inputs u + dt/2 k1, u + dt/2 k2, u + dt k3, u = acc + dt/6 k4
static int enqueue_rk(dgswe_ctx *ctx, int order, double *u, double *w1, double *w2, double *w3, double dt,
                      int nsteps, int check_mean, cudaStream_t s)
{
    const int lo = ctx->cfg.jlo, hi = ctx->cfg.jhi;
    if (!ctx->basis) {   // the steps run on the nodal values; u is converted in place around them
        int rc = convert_rows(ctx, u, u, true, 0, ctx->cfg.nrows, s);
        if (rc) return rc;
    }
    for (int k = 0; k < nsteps; ++k) {
        int rc = DGSWE_OK;
        switch (order) {
        case 1: {
            double *x = (k & 1) ? w1 : u, *y = (k & 1) ? u : w1;
            rc = launch_stage(ctx, 0.0, nullptr, 1.0, x, dt, y, nullptr, 0.0, nullptr, k, lo, hi, 1, check_mean, s);
            break;
        }
        case 2:
            rc = launch_stage(ctx, 0.0, nullptr, 1.0, u, dt, w1, nullptr, 0.0, nullptr, k, lo, hi, 0, 0, s);
            if (!rc)
                rc = launch_stage(ctx, 0.5, u, 0.5, w1, 0.5 * dt, u, nullptr, 0.0, nullptr, k, lo, hi, 1,
                                  check_mean, s);
            break;
        case 3:
            rc = launch_stage(ctx, 0.0, nullptr, 1.0, u, dt, w1, nullptr, 0.0, nullptr, k, lo, hi, 0, 0, s);
            if (!rc)
                rc = launch_stage(ctx, 0.75, u, 0.25, w1, 0.25 * dt, w2, nullptr, 0.0, nullptr, k, lo, hi, 0, 0,
                                  s);
            if (!rc)
                rc = launch_stage(ctx, 1.0 / 3.0, u, 2.0 / 3.0, w2, (2.0 / 3.0) * dt, u, nullptr, 0.0, nullptr,
                                  k, lo, hi, 1, check_mean, s);
            break;
        case 4:
            rc = launch_stage(ctx, 0.0, nullptr, 1.0, u, 0.5 * dt, w1, u, dt / 6.0, w3, k, lo, hi, 0, 0, s);
            if (!rc)
                rc = launch_stage(ctx, 1.0, u, 0.0, w1, 0.5 * dt, w2, w3, dt / 3.0, w3, k, lo, hi, 0, 0, s);
            if (!rc)
                rc = launch_stage(ctx, 1.0, u, 0.0, w2, dt, w1, w3, dt / 3.0, w3, k, lo, hi, 0, 0, s);
            if (!rc)
                rc = launch_stage(ctx, 1.0, w3, 0.0, w1, dt / 6.0, u, nullptr, 0.0, nullptr, k, lo, hi, 1,
                                  check_mean, s);
            break;
        default:
            return fail(DGSWE_EUNSUPPORTED, "RK order %d not supported (1..4)", order);
        }
        if (rc) return rc;
    }
    if (order == 1 && (nsteps & 1))
        CUDA_TRY(cudaMemcpyAsync(u, w1, sizeof(double) * (size_t)ctx->zstride * ctx->cfg.nz,
                                 cudaMemcpyDeviceToDevice, s));
    if (!ctx->basis) return convert_rows(ctx, u, u, false, 0, ctx->cfg.nrows, s);
    return DGSWE_OK;
}

static int stages_of(int order) { return order; }

int dgswe_rk_steps(dgswe_ctx *ctx, int order, double *u, double *w1, double *w2, double *w3, double dt,
                   int nsteps, int check_mean, void *stream)
{
    if (!ctx || !u || !w1) return fail(DGSWE_EINVAL, "null argument");
    if (order < 1 || order > 4) return fail(DGSWE_EUNSUPPORTED, "RK order %d not supported (1..4)", order);
    if ((order >= 3 && !w2) || (order == 4 && !w3)) return fail(DGSWE_EINVAL, "missing scratch buffer");
    if (nsteps < 0) return fail(DGSWE_EINVAL, "nsteps must be >= 0");
    if (nsteps == 0) return DGSWE_OK;
    if (ctx->cfg.jlo != 0 || ctx->cfg.jhi != ctx->cfg.ny || ctx->cfg.row0 != 0)
        return fail(DGSWE_EINVAL, "fused RK steps need a single-band context; use dgswe_stage per band");
    cudaStream_t s = (cudaStream_t)stream;
    if (getenv("DGSWE_NO_GRAPH")) return enqueue_rk(ctx, order, u, w1, w2, w3, dt, nsteps, check_mean, s);
    GraphKey key{order, u, w1, w2, w3, dt, nsteps, check_mean, ctx->basis};
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
        if (ctx->graphs.size() >= 8) {
            for (auto &kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
            ctx->graphs.clear();
        }
        cudaStream_t cap = s;
        bool own = false;
        if (cap == nullptr) {   // legacy stream cannot be captured
            CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            own = true;
        }
        CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        const long long before = ctx->launches;
        int rc = enqueue_rk(ctx, order, u, w1, w2, w3, dt, nsteps, check_mean, cap);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(cap, &graph);
        ctx->launches = before;   // counted at replay
        if (own) cudaStreamDestroy(cap);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return fail(DGSWE_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return fail(DGSWE_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
        it = ctx->graphs.emplace(key, exec).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, s));
    const int per_stage = 1 + (ctx->cfg.alpha_mode == DGSWE_ALPHA_GLOBAL ? 1 : 0);
    ctx->launches += (long long)stages_of(order) * nsteps * per_stage + (ctx->basis ? 0 : 2);
    return DGSWE_OK;
}

int dgswe_ssprk3(dgswe_ctx *ctx, double *u, double *w1, double *w2, double dt, int nsteps,
                 int check_mean, void *stream)
{
    return dgswe_rk_steps(ctx, 3, u, w1, w2, nullptr, dt, nsteps, check_mean, stream);
}

int dgswe_status(dgswe_ctx *ctx, uint32_t *flags, int32_t *first_tag, int reset, void *stream)
{
    if (!ctx) return fail(DGSWE_EINVAL, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    DevStatus h;
    CUDA_TRY(cudaMemcpyAsync(&h, ctx->status, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (flags) *flags = h.flags;
    if (first_tag) *first_tag = h.first_tag;
    if (reset) {
        DevStatus st0 = {0u, INT_MAX};
        CUDA_TRY(cudaMemcpyAsync(ctx->status, &st0, sizeof st0, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    return DGSWE_OK;
}

int64_t dgswe_launch_count(const dgswe_ctx *ctx) { return ctx ? ctx->launches : 0; }

// ---- device diagnostics and IC projection (dgswe_diag.cuh) ----

static int diag_scratch(dgswe_ctx *c, size_t doubles)
{
    if (c->diag_bytes < doubles * sizeof(double)) {
        cudaFree(c->diag);
        c->diag = nullptr;
        c->diag_bytes = 0;
        CUDA_TRY(cudaMalloc(&c->diag, doubles * sizeof(double)));
        c->diag_bytes = doubles * sizeof(double);
    }
    return DGSWE_OK;
}

static dgswe::DiagLayout diag_layout(const dgswe_ctx *c)
{
    return {c->zstride, c->rstride, c->vstride, c->cfg.nx, c->cfg.ny, c->nphi};
}

static int check_diag(const dgswe_ctx *c, const double *X, int var, int level)
{
    if (!c || !X) return fail(DGSWE_EINVAL, "null argument");
    if (var < 0 || var > 2 || level < 0 || level >= c->cfg.nz) return fail(DGSWE_EINVAL, "bad var/level");
    if (c->cfg.row0 != 0 || c->cfg.nrows != c->cfg.ny)
        return fail(DGSWE_EINVAL, "diagnostics need a single-band context");
    return DGSWE_OK;
}

int dgswe_mass(dgswe_ctx *ctx, const double *X, int var, int level, const double *m0_rows, double *out,
               void *stream)
{
    int rc = check_diag(ctx, X, var, level);
    if (rc) return rc;
    if (!m0_rows || !out) return fail(DGSWE_EINVAL, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, nphi = ctx->nphi;
    rc = diag_scratch(ctx, (size_t)ny * nphi + 2 * (size_t)ny + 2);
    if (rc) return rc;
    double *tab = ctx->diag, *part = tab + (size_t)ny * nphi, *res = part + 2 * (size_t)ny;
    CUDA_TRY(cudaMemcpyAsync(tab, m0_rows, sizeof(double) * ny * nphi, cudaMemcpyHostToDevice, s));
    const dgswe::DiagLayout L = diag_layout(ctx);
    dgswe::mass_rows_kernel<<<dim3(ny, 1), 256, 0, s>>>(X + (size_t)level * ctx->zstride, L, var, tab, part);
    dgswe::rows_total_kernel<1><<<1, 256, 0, s>>>(part, ny, 0, res);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 2;
    CUDA_TRY(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DGSWE_OK;
}

int dgswe_l2_sums(dgswe_ctx *ctx, const double *X, int var, int level, const double *phi2, int nq2,
                  const double *wrow, const double *ref, double *out2, void *stream)
{
    int rc = check_diag(ctx, X, var, level);
    if (rc) return rc;
    if (!phi2 || !wrow || !ref || !out2 || nq2 < 1) return fail(DGSWE_EINVAL, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, nphi = ctx->nphi;
    const size_t nt = (size_t)nq2 * nphi + (size_t)ny * nq2;
    rc = diag_scratch(ctx, nt + 4 * (size_t)ny + 2);
    if (rc) return rc;
    double *dphi = ctx->diag, *dw = dphi + (size_t)nq2 * nphi, *part = ctx->diag + nt, *res = part + 4 * (size_t)ny;
    CUDA_TRY(cudaMemcpyAsync(dphi, phi2, sizeof(double) * nq2 * nphi, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dw, wrow, sizeof(double) * ny * nq2, cudaMemcpyHostToDevice, s));
    const dgswe::DiagLayout L = diag_layout(ctx);
    dgswe::l2_rows_kernel<<<dim3(ny, 1), 256, 0, s>>>(X + (size_t)level * ctx->zstride, L, var, dphi, nq2, dw,
                                                       ref, part);
    dgswe::rows_total_kernel<2><<<1, 256, 0, s>>>(part, ny, 0, res);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 2;
    CUDA_TRY(cudaMemcpyAsync(out2, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DGSWE_OK;
}

}  // extern "C"

template <int P>
static void launch_project(dgswe_ctx *c, const double *f, const double *cosn, double determ, double *Y,
                           cudaStream_t s)
{
    dim3 grid((c->cfg.nx + 127) / 128, c->cfg.ny, 3);
    const int rs = dgswe::row_stride(P);
    dgswe::project_kernel<P><<<grid, 128, 0, s>>>(f, cosn, c->rowtab, rs, dgswe::RowLayout<P>::T,
                                                  diag_layout(c), c->cfg.nz, determ, Y);
}

extern "C" {

int dgswe_project(dgswe_ctx *ctx, const double *fvals, const double *cos_nodes, double determ, double *Y,
                  void *stream)
{
    if (!ctx || !fvals || !cos_nodes || !Y) return fail(DGSWE_EINVAL, "null argument");
    if (ctx->cfg.row0 != 0 || ctx->cfg.nrows != ctx->cfg.ny)
        return fail(DGSWE_EINVAL, "projection needs a single-band context");
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, n = ctx->n;
    int rc = diag_scratch(ctx, (size_t)ny * n);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(ctx->diag, cos_nodes, sizeof(double) * ny * n, cudaMemcpyHostToDevice, s));
    switch (ctx->cfg.p) {
    case 0: launch_project<0>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 1: launch_project<1>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 2: launch_project<2>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 3: launch_project<3>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 4: launch_project<4>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 5: launch_project<5>(ctx, fvals, ctx->diag, determ, Y, s); break;
    case 6: launch_project<6>(ctx, fvals, ctx->diag, determ, Y, s); break;
    default: return fail(DGSWE_EUNSUPPORTED, "degree not supported");
    }
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 1;
    CUDA_TRY(cudaStreamSynchronize(s));   // the host staging buffers may be reused by the caller
    return DGSWE_OK;
}

#ifdef DG_TIMING
// experiment builds only: per-role phase cycle sums since the last call
int dgswe_debug_timing(unsigned long long *out28)
{
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out28, dgswe::g_timing, sizeof(unsigned long long) * 28));
    static unsigned long long zero[28] = {};
    CUDA_TRY(cudaMemcpyToSymbol(dgswe::g_timing, zero, sizeof zero));
    return DGSWE_OK;
}
#endif

}  // extern "C"
