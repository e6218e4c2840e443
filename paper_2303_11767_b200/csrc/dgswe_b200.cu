// dgswe_b200.cu -- C ABI (include/dgswe_b200.h) over the sm_100a fp64 DG
// shallow-water kernels (dgswe_kernels.cuh, one translation unit per degree:
// deg_p*.cu).
//
// The context owns only constant tables (uploaded once, as the reference
// precomputes on the host, dg.py:186-219), the status words, the
// global-alpha pair, a fixed-size diagnostics scratch and cached CUDA
// graphs -- all allocated in dgswe_create.  Every state buffer belongs to
// the caller; no entry point allocates device memory.

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "dgswe_ctx.h"
#include "dgswe_diag.cuh"

namespace {

thread_local std::string g_last_error;

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
        atomicMin(&st->first_tag[1], tag);
    }
}

// nodal tables (dgswe_params.h NodTab) of degree n-1 from the reference's
// Legendre tables, in long double: l_i(x) = sum_a (2a+1)/2 w_i P_a(x_i) P_a(x)
// (the Gauss rule projects the degree-p Lagrange polynomial exactly)
dgswe::NodTab nodal_tables(const double *leg, const double *dleg, const double *weights, int n)
{
    dgswe::NodTab nt;
    memset(&nt, 0, sizeof nt);
    for (int i = 0; i < n; ++i) {
        const long double wi = weights[i];
        long double lm = 0.0L;
        for (int a = 0; a < n; ++a) lm += 0.5L * (2 * a + 1) * wi * leg[a * n + i] * ((a & 1) ? -1.0L : 1.0L);
        nt.lm[i] = (double)lm;
        nt.mu[i] = (double)(lm / wi);
        nt.w[i] = (double)wi;
        for (int k = 0; k < n; ++k) {
            long double d = 0.0L;   // w_k l_i'(x_k) / w_i
            for (int a = 0; a < n; ++a)
                d += 0.5L * (2 * a + 1) * (long double)leg[a * n + i] * weights[k] * dleg[a * n + k];
            nt.dh[i][k] = (double)d;
        }
        for (int a = 0; a < n; ++a) {
            nt.leg[a][i] = leg[a * n + i];
            nt.wp[a][i] = weights[i] * leg[a * n + i];
        }
    }
    return nt;
}

constexpr DevStatus kStatus0 = {0u, {INT_MAX, INT_MAX, INT_MAX, INT_MAX}};

bool misaligned(const void *p) { return ((uintptr_t)p & 15u) != 0; }

// Y = a U + b X + g RHS(X) [, Y2 = A + g2 RHS(X)]; the state basis of the
// call is c.modal (modal: the in-kernel conversion variant)
int launch_stage(dgswe_ctx *c, const StageCall &sc, cudaStream_t s)
{
    if (!sc.X || !sc.Y) return dgswe_fail(DGSWE_EINVAL, "null state pointer");
    if (sc.X == sc.Y || sc.X == sc.Y2) return dgswe_fail(DGSWE_EINVAL, "outputs must not alias the stage input");
    if (sc.Y2 && (sc.Y2 == sc.Y || !sc.A))
        return dgswe_fail(DGSWE_EINVAL, "second output needs its own buffer and an addend");
    if (sc.a != 0.0 && !sc.U) return dgswe_fail(DGSWE_EINVAL, "U is required when a != 0");
    // the kernels move row tiles with TMA bulk copies: 16-byte aligned states
    if (misaligned(sc.X) || misaligned(sc.Y) || misaligned(sc.U) || misaligned(sc.A) || misaligned(sc.Y2))
        return dgswe_fail(DGSWE_EINVAL, "state buffers must be 16-byte aligned");
    if (sc.r0 < c->cfg.jlo || sc.r1 > c->cfg.jhi || sc.r0 > sc.r1)
        return dgswe_fail(DGSWE_EINVAL, "row range [%d,%d) outside [%d,%d)", sc.r0, sc.r1, c->cfg.jlo, c->cfg.jhi);
    if (sc.r3 > sc.r2 && (sc.r2 < c->cfg.jlo || sc.r3 > c->cfg.jhi || sc.r2 < sc.r1))
        return dgswe_fail(DGSWE_EINVAL, "second row range [%d,%d) invalid", sc.r2, sc.r3);
    if (sc.edge && (sc.modal || sc.Y2))
        return dgswe_fail(DGSWE_EINVAL, "edge launches take nodal states and have one output");
    dgswe::StageParams kp = {};
    kp.X = sc.X;
    kp.U = (sc.a != 0.0) ? sc.U : nullptr;
    kp.Y = sc.Y;
    kp.A = sc.Y2 ? sc.A : nullptr;
    kp.Y2 = sc.Y2;
    kp.g2 = sc.g2;
    kp.zstride = c->zstride;
    kp.rstride = c->rstride;
    kp.vstride = c->vstride;
    kp.nstrip = c->nstrip;
    kp.nx = c->cfg.nx;
    kp.ny = c->cfg.ny;
    kp.row0 = c->cfg.row0;
    kp.nrows = c->cfg.nrows;
    kp.j_begin = sc.r0;
    kp.j_end = sc.r1;
    kp.nchunk1 = INT_MAX;
    kp.j_begin2 = sc.r2;
    kp.j_end2 = sc.r3;
    kp.rc = c->rc;
    kp.a = sc.a;
    kp.b = sc.b;
    kp.g = sc.g;
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
    kp.first_tag = c->status->first_tag;
    kp.tag = sc.tag;
    kp.check_finite = sc.check_finite;
    kp.check_mean = sc.check_mean;
    kp.modal = sc.modal ? 1 : 0;
    kp.orog = c->orog;
    kp.orog_mask = c->orog_mask;
    kp.periodic_y = c->cfg.periodic_y;
    kp.orog_rstride = 2 * c->vstride;
    if (sc.edge) {
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
        kp.peer_timeout_ns = c->peer_timeout_ns;
    }
    if (c->cfg.alpha_mode == DGSWE_ALPHA_GLOBAL && !c->external_alpha) {
        const int rc = c->ops->alpha(c, sc.X, sc.modal, s);
        if (rc) return rc;
    }
    return c->ops->stage(c, kp, s);
}

// a stage through the public entry points, in the context's state basis
int api_stage(dgswe_ctx *c, StageCall sc, cudaStream_t s)
{
    sc.modal = c->basis == 0;
    return launch_stage(c, sc, s);
}

StageCall stage_call(double a, const double *U, double b, const double *X, double g, double *Y, int tag, int r0,
                     int r1)
{
    StageCall sc;
    sc.a = a;
    sc.U = U;
    sc.b = b;
    sc.X = X;
    sc.g = g;
    sc.Y = Y;
    sc.tag = tag;
    sc.r0 = r0;
    sc.r1 = r1;
    return sc;
}

}  // namespace

int dgswe_fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

const DegreeOps *dgswe_degree_ops_0();
const DegreeOps *dgswe_degree_ops_1();
const DegreeOps *dgswe_degree_ops_2();
const DegreeOps *dgswe_degree_ops_3();
const DegreeOps *dgswe_degree_ops_4();
const DegreeOps *dgswe_degree_ops_5();
const DegreeOps *dgswe_degree_ops_6();

const DegreeOps *dgswe_degree_ops(int p)
{
    switch (p) {
    case 0: return dgswe_degree_ops_0();
    case 1: return dgswe_degree_ops_1();
    case 2: return dgswe_degree_ops_2();
    case 3: return dgswe_degree_ops_3();
    case 4: return dgswe_degree_ops_4();
    case 5: return dgswe_degree_ops_5();
    case 6: return dgswe_degree_ops_6();
    default: return nullptr;
    }
}

extern "C" {

int dgswe_abi_version(void) { return DGSWE_ABI_VERSION; }

const char *dgswe_last_error(void) { return g_last_error.c_str(); }

int dgswe_create(const dgswe_cfg *cfg, const dgswe_tables *t, dgswe_ctx **out)
{
    if (!cfg || !t || !out) return dgswe_fail(DGSWE_EINVAL, "null argument");
    *out = nullptr;
    const dgswe_cfg &c = *cfg;
    if (c.p < 0 || c.p > dgswe::kMaxP) return dgswe_fail(DGSWE_EUNSUPPORTED, "degree p=%d not supported (0..6)", c.p);
    if (c.nx < 1 || c.ny < 1 || c.nz < 1) return dgswe_fail(DGSWE_EINVAL, "element counts must be >= 1");
    if (c.nrows < 1 || c.jlo < 0 || c.jhi > c.nrows || c.jlo >= c.jhi)
        return dgswe_fail(DGSWE_EINVAL, "bad local rows: nrows=%d jlo=%d jhi=%d", c.nrows, c.jlo, c.jhi);
    if (c.row0 + c.jlo < 0 || c.row0 + c.jhi > c.ny) return dgswe_fail(DGSWE_EINVAL, "band outside the sphere");
    if (c.row0 + c.jlo > 0 && c.jlo < 1) return dgswe_fail(DGSWE_EINVAL, "band needs a southern halo row");
    if (c.row0 + c.jhi < c.ny && c.jhi >= c.nrows) return dgswe_fail(DGSWE_EINVAL, "band needs a northern halo row");
    if (c.alpha_mode < 0 || c.alpha_mode > 2) return dgswe_fail(DGSWE_EINVAL, "bad alpha mode");
    if (!(c.radius > 0) || !(c.gravity > 0) || !(c.dx > 0) || !(c.dy > 0) || !(c.h_floor > 0))
        return dgswe_fail(DGSWE_EINVAL, "radius, gravity, dx, dy, h_floor must be positive");
    if (!t->leg || !t->dleg || !t->weights || !t->cos_r_int || !t->sin_r_int || !t->fcos_int ||
        !t->cos_r_edge || !t->cos_edge || !t->minv)
        return dgswe_fail(DGSWE_EINVAL, "missing table");
    if (c.periodic_y && (c.row0 != 0 || c.nrows != c.ny || c.jlo != 0 || c.jhi != c.ny || t->orog))
        return dgswe_fail(DGSWE_EINVAL, "a y-periodic mesh runs as one band without orography");

    dgswe_ctx *ctx = new (std::nothrow) dgswe_ctx();
    if (!ctx) return dgswe_fail(DGSWE_ENOMEM, "out of host memory");
    ctx->cfg = c;
    ctx->ops = dgswe_degree_ops(c.p);
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

    // rows per CTA: fixed, or 0 = sized at launch (dgswe_degree.cuh chunk_rows)
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
    ctx->rc = c.row_chunk > 0 ? c.row_chunk : 0;
    if (const char *env = getenv("DGSWE_ROW_CHUNK")) ctx->rc = atoi(env);
    if (const char *env = getenv("DGSWE_CHUNKS")) ctx->even_chunks = atoi(env);
    if (const char *env = getenv("DGSWE_NO_LO")) ctx->no_lo = atoi(env);
    if (const char *env = getenv("DGSWE_SMEM_PAD")) ctx->smem_pad = atoi(env);

    const dgswe::NodTab nt = nodal_tables(t->leg, t->dleg, t->weights, n);
    int rc = ctx->ops->upload(nt);
    if (rc) {
        delete ctx;
        return rc;
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
        for (int q = 0; q < n; ++q) r[3 * n + 2 + q] = 1.0 / (determ * (t->cos_r_int[j * n + q] * c.radius));
        for (int b = 0; b < n; ++b)
            for (int bb = 0; bb < n; ++bb) r[4 * n + 2 + b * n + bb] = M[(size_t)b * ctx->nphi + bb];
    }

    // Orography (Williamson TC5; not in the reference): the
    // momentum sources -(g h / R) db/dlambda and -(g h cos / R) db/dtheta
    // (cos-weighted flux form of models.py:213-252), with grad b the exact
    // derivative of b's degree-p interpolant at the Gauss nodes:
    //   db/dxi (x_i, x_j) = sum_k l_k'(x_i) b[k][j],  db/dlambda = (2/dx) db/dxi.
    // Stored per buffer row as the nodal factors B (determ folded in, like
    // the row table's source factors): S_hu += h B_x, S_hv += h B_y.
    std::vector<double> ob;
    std::vector<unsigned char> om;   // per (row, strip): 1 if the orography tile is non-zero
    if (t->orog) {
        long double D[dgswe::kMaxP + 1][dgswe::kMaxP + 1];   // D[i][k] = l_k'(x_i)
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < n; ++k) {
                long double d = 0.0L;
                for (int a = 0; a < n; ++a)
                    d += 0.5L * (2 * a + 1) * (long double)t->weights[k] * t->leg[a * n + k] * t->dleg[a * n + i];
                D[i][k] = d;
            }
        const int np = ctx->nphi;
        ob.assign((size_t)c.nrows * 2 * ctx->vstride, 0.0);
        for (int r = 0; r < c.nrows; ++r) {
            const int j = c.row0 + r;
            if (j < 0 || j >= c.ny) continue;
            for (int e = 0; e < c.nx; ++e) {
                const double *b = t->orog + ((size_t)j * c.nx + e) * np;
                for (int i = 0; i < n; ++i)
                    for (int jj = 0; jj < n; ++jj) {
                        long double dxi = 0.0L, deta = 0.0L;
                        for (int k = 0; k < n; ++k) {
                            dxi += D[i][k] * b[k * n + jj];
                            deta += D[jj][k] * b[i * n + k];
                        }
                        const long double bx = -(long double)c.gravity * ctx->inv_r * dxi * ctx->bdy;
                        const long double by =
                            -(long double)c.gravity * t->cos_r_int[j * n + jj] * deta * ctx->bdx;
                        const size_t o = (size_t)r * 2 * ctx->vstride + (size_t)(e >> 5) * np * DGSWE_STRIP +
                                         (size_t)(i * n + jj) * DGSWE_STRIP + (e & 31);
                        ob[o] = (double)bx;
                        ob[o + ctx->vstride] = (double)by;
                    }
            }
        }
        // which (row, strip) tiles have a non-zero factor: the others are
        // neither copied nor used (an isolated mountain covers a few % of
        // the sphere; h * 0 adds nothing, so skipping is exact)
        om.assign((size_t)c.nrows * ctx->nstrip, 0);
        for (int r = 0; r < c.nrows; ++r)
            for (int st = 0; st < ctx->nstrip; ++st) {
                const size_t o = (size_t)r * 2 * ctx->vstride + (size_t)st * np * DGSWE_STRIP;
                for (int q = 0; q < np * DGSWE_STRIP && !om[(size_t)r * ctx->nstrip + st]; ++q)
                    if (ob[o + q] != 0.0 || ob[o + ctx->vstride + q] != 0.0) om[(size_t)r * ctx->nstrip + st] = 1;
            }
    }

    // diagnostics scratch, sized once: mass (ny*nphi + 2ny + 2), l2 with a
    // rule of up to (p+2)^2 nodes, projection (ny*n)
    ctx->nq2_max = (c.p + 2) * (c.p + 2);
    const size_t d_mass = (size_t)c.ny * ctx->nphi + 2 * (size_t)c.ny + 2;
    const size_t d_l2 = (size_t)ctx->nq2_max * ctx->nphi + (size_t)c.ny * ctx->nq2_max + 4 * (size_t)c.ny + 2;
    const size_t d_proj = (size_t)c.ny * n;
    ctx->diag_doubles = d_mass > d_l2 ? d_mass : d_l2;
    if (d_proj > ctx->diag_doubles) ctx->diag_doubles = d_proj;

    bool ok = cudaMalloc(&ctx->rowtab, rt.size() * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->cos_edge, (c.ny + 1) * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->alpha, 2 * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->status, sizeof(DevStatus)) == cudaSuccess &&
              cudaMalloc(&ctx->diag, ctx->diag_doubles * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&ctx->status_host, 2 * sizeof(DevStatus)) == cudaSuccess &&
              (ob.empty() || cudaMalloc(&ctx->orog, ob.size() * sizeof(double)) == cudaSuccess) &&
              (om.empty() || cudaMalloc(&ctx->orog_mask, om.size()) == cudaSuccess);
    if (ok) {
        ctx->status_host[1] = kStatus0;   // the reset value, copied from pinned memory
        ok = cudaMemcpy(ctx->rowtab, rt.data(), rt.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(ctx->cos_edge, t->cos_edge, (c.ny + 1) * sizeof(double), cudaMemcpyHostToDevice) ==
                 cudaSuccess &&
             cudaMemset(ctx->alpha, 0, 2 * sizeof(double)) == cudaSuccess &&
             cudaMemcpy(ctx->status, &kStatus0, sizeof kStatus0, cudaMemcpyHostToDevice) == cudaSuccess &&
             (ob.empty() ||
              cudaMemcpy(ctx->orog, ob.data(), ob.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess) &&
             (om.empty() || cudaMemcpy(ctx->orog_mask, om.data(), om.size(), cudaMemcpyHostToDevice) == cudaSuccess);
    }
    if (!ok) {
        cudaError_t le = cudaGetLastError();
        dgswe_destroy(ctx);
        return dgswe_fail(DGSWE_ECUDA, "device allocation/upload failed: %s", cudaGetErrorString(le));
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
    cudaFree(ctx->orog);
    cudaFree(ctx->orog_mask);
    if (ctx->status_host) cudaFreeHost(ctx->status_host);
    delete ctx;
}

int64_t dgswe_state_elems(const dgswe_ctx *ctx) { return ctx ? (int64_t)ctx->zstride * ctx->cfg.nz : 0; }

int dgswe_rhs(dgswe_ctx *ctx, const double *X, double *K, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, stage_call(0.0, nullptr, 0.0, X, 1.0, K, 0, ctx->cfg.jlo, ctx->cfg.jhi),
                     (cudaStream_t)stream);
}

int dgswe_stage(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                int tag, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, stage_call(a, U, b, X, g, Y, tag, ctx->cfg.jlo, ctx->cfg.jhi), (cudaStream_t)stream);
}

int dgswe_stage_rows(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                     int tag, int r0, int r1, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    return api_stage(ctx, stage_call(a, U, b, X, g, Y, tag, r0, r1), (cudaStream_t)stream);
}

int dgswe_stage_rows2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                      double *Y, int tag, int r0, int r1, int r2, int r3, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    StageCall sc = stage_call(a, U, b, X, g, Y, tag, r0, r1);
    sc.r2 = r2;
    sc.r3 = r3;
    return api_stage(ctx, sc, (cudaStream_t)stream);
}

int dgswe_stage_rows_checked(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                             double *Y, int tag, int r0, int r1, int check_finite, int check_mean,
                             void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    StageCall sc = stage_call(a, U, b, X, g, Y, tag, r0, r1);
    sc.check_finite = check_finite ? 1 : 0;
    sc.check_mean = check_mean ? 1 : 0;
    return api_stage(ctx, sc, (cudaStream_t)stream);
}

int dgswe_stage2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                 const double *A, double g2, double *Y2, int tag, int r0, int r1, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    StageCall sc = stage_call(a, U, b, X, g, Y, tag, r0, r1);
    sc.A = A;
    sc.g2 = g2;
    sc.Y2 = Y2;
    return api_stage(ctx, sc, (cudaStream_t)stream);
}

int dgswe_set_exchange(dgswe_ctx *ctx, long long peer_zstride_s, unsigned long long *peer_count_s,
                       long long peer_zstride_n, unsigned long long *peer_count_n,
                       unsigned long long *recv_count, unsigned long long *stage_ctr)
{
    if (!ctx || !recv_count || !stage_ctr) return dgswe_fail(DGSWE_EINVAL, "null argument");
    ctx->peer_zstride[0] = peer_zstride_s;
    ctx->peer_zstride[1] = peer_zstride_n;
    ctx->peer_count[0] = peer_count_s;
    ctx->peer_count[1] = peer_count_n;
    ctx->recv_count = recv_count;
    ctx->stage_ctr = stage_ctr;
    return DGSWE_OK;
}

int dgswe_set_peer_timeout(dgswe_ctx *ctx, unsigned long long timeout_ns)
{
    if (!ctx || timeout_ns == 0) return dgswe_fail(DGSWE_EINVAL, "null context or zero timeout");
    ctx->peer_timeout_ns = timeout_ns;
    return DGSWE_OK;
}

int dgswe_stage_band(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                     int tag, double *peer_row_s, double *peer_row_n, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    if (!ctx->stage_ctr) return dgswe_fail(DGSWE_EINVAL, "dgswe_set_exchange first");
    if (!ctx->basis) return dgswe_fail(DGSWE_EINVAL, "band launches take nodal states (dgswe_set_basis)");
    ctx->edge_row[0] = peer_row_s;
    ctx->edge_row[1] = peer_row_n;
    StageCall sc = stage_call(a, U, b, X, g, Y, tag, ctx->cfg.jlo, ctx->cfg.jhi);
    sc.edge = true;
    return launch_stage(ctx, sc, (cudaStream_t)stream);
}

int dgswe_dev_alloc(size_t bytes, void **out)
{
    if (!out) return dgswe_fail(DGSWE_EINVAL, "null argument");
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
    if (!p || !out64) return dgswe_fail(DGSWE_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, p));
    memcpy(out64, &h, sizeof h);
    return DGSWE_OK;
}

int dgswe_ipc_open(const char *in64, void **out)
{
    if (!in64 || !out) return dgswe_fail(DGSWE_EINVAL, "null argument");
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

int dgswe_axpy(dgswe_ctx *ctx, double coef, const double *x, double *y, int check_finite, int tag, void *stream)
{
    if (!ctx || !x || !y) return dgswe_fail(DGSWE_EINVAL, "null argument");
    const long long off = (long long)ctx->cfg.jlo * ctx->rstride;
    const long long count = (long long)(ctx->cfg.jhi - ctx->cfg.jlo) * ctx->rstride;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    dim3 grid((unsigned)blocks, ctx->cfg.nz);
    axpy_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, y, coef, ctx->zstride, off, count, check_finite,
                                                        ctx->status, tag);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 1;
    return DGSWE_OK;
}

int dgswe_alpha_prepass(dgswe_ctx *ctx, const double *X, void *stream)
{
    if (!ctx || !X) return dgswe_fail(DGSWE_EINVAL, "null argument");
    return ctx->ops->alpha(ctx, X, ctx->basis == 0, (cudaStream_t)stream);
}

int dgswe_set_basis(dgswe_ctx *ctx, int nodal)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    ctx->basis = nodal ? 1 : 0;
    return DGSWE_OK;
}

int dgswe_convert(dgswe_ctx *ctx, double *X, int to_nodal, int r0, int r1, void *stream)
{
    if (!ctx || !X) return dgswe_fail(DGSWE_EINVAL, "null argument");
    if (r0 < 0 || r1 > ctx->cfg.nrows || r0 > r1) return dgswe_fail(DGSWE_EINVAL, "bad row range [%d,%d)", r0, r1);
    return ctx->ops->convert(ctx, X, X, to_nodal != 0, r0, r1, (cudaStream_t)stream);
}

double *dgswe_alpha_buffer(dgswe_ctx *ctx) { return ctx ? ctx->alpha : nullptr; }

int dgswe_set_external_alpha(dgswe_ctx *ctx, int external)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    ctx->external_alpha = external ? 1 : 0;
    return DGSWE_OK;
}

}  // extern "C"

// K steps of the fused explicit RK method of `order` (the tableaux of
// timestep.py:57-82, evaluated in stage form; every stage is one kernel),
// on nodal values (u converted in place around the steps in the modal
// basis):
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
    if (!ctx->basis) {
        int rc = ctx->ops->convert(ctx, u, u, true, 0, ctx->cfg.nrows, s);
        if (rc) return rc;
    }
    auto st = [&](double a, const double *U, double b, const double *X, double g, double *Y, int k,
                  int last) {
        StageCall sc = stage_call(a, U, b, X, g, Y, k, lo, hi);
        sc.check_finite = last;
        sc.check_mean = last ? check_mean : 0;
        return launch_stage(ctx, sc, s);
    };
    auto st2 = [&](double a, const double *U, double b, const double *X, double g, double *Y, const double *A,
                   double g2, double *Y2, int k) {
        StageCall sc = stage_call(a, U, b, X, g, Y, k, lo, hi);
        sc.A = A;
        sc.g2 = g2;
        sc.Y2 = Y2;
        return launch_stage(ctx, sc, s);
    };
    for (int k = 0; k < nsteps; ++k) {
        int rc = DGSWE_OK;
        switch (order) {
        case 1: {
            double *x = (k & 1) ? w1 : u, *y = (k & 1) ? u : w1;
            rc = st(0.0, nullptr, 1.0, x, dt, y, k, 1);
            break;
        }
        case 2:
            rc = st(0.0, nullptr, 1.0, u, dt, w1, k, 0);
            if (!rc) rc = st(0.5, u, 0.5, w1, 0.5 * dt, u, k, 1);
            break;
        case 3:
            rc = st(0.0, nullptr, 1.0, u, dt, w1, k, 0);
            if (!rc) rc = st(0.75, u, 0.25, w1, 0.25 * dt, w2, k, 0);
            if (!rc) rc = st(1.0 / 3.0, u, 2.0 / 3.0, w2, (2.0 / 3.0) * dt, u, k, 1);
            break;
        case 4:
            rc = st2(0.0, nullptr, 1.0, u, 0.5 * dt, w1, u, dt / 6.0, w3, k);
            if (!rc) rc = st2(1.0, u, 0.0, w1, 0.5 * dt, w2, w3, dt / 3.0, w3, k);
            if (!rc) rc = st2(1.0, u, 0.0, w2, dt, w1, w3, dt / 3.0, w3, k);
            if (!rc) rc = st(1.0, w3, 0.0, w1, dt / 6.0, u, k, 1);
            break;
        default:
            return dgswe_fail(DGSWE_EUNSUPPORTED, "RK order %d not supported (1..4)", order);
        }
        if (rc) return rc;
    }
    if (order == 1 && (nsteps & 1))
        CUDA_TRY(cudaMemcpyAsync(u, w1, sizeof(double) * (size_t)ctx->zstride * ctx->cfg.nz,
                                 cudaMemcpyDeviceToDevice, s));
    if (!ctx->basis) return ctx->ops->convert(ctx, u, u, false, 0, ctx->cfg.nrows, s);
    return DGSWE_OK;
}

extern "C" {

int dgswe_rk_steps(dgswe_ctx *ctx, int order, double *u, double *w1, double *w2, double *w3, double dt, int nsteps,
                   int check_mean, void *stream)
{
    if (!ctx || !u || !w1) return dgswe_fail(DGSWE_EINVAL, "null argument");
    if (order < 1 || order > 4) return dgswe_fail(DGSWE_EUNSUPPORTED, "RK order %d not supported (1..4)", order);
    if ((order >= 3 && !w2) || (order == 4 && !w3)) return dgswe_fail(DGSWE_EINVAL, "missing scratch buffer");
    if (nsteps < 0) return dgswe_fail(DGSWE_EINVAL, "nsteps must be >= 0");
    if (nsteps == 0) return DGSWE_OK;
    if (ctx->cfg.jlo != 0 || ctx->cfg.jhi != ctx->cfg.ny || ctx->cfg.row0 != 0)
        return dgswe_fail(DGSWE_EINVAL, "fused RK steps need a single-band context; use dgswe_stage per band");
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
        if (e != cudaSuccess) return dgswe_fail(DGSWE_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return dgswe_fail(DGSWE_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
        it = ctx->graphs.emplace(key, exec).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, s));
    const int per_stage = 1 + (ctx->cfg.alpha_mode == DGSWE_ALPHA_GLOBAL ? 1 : 0);
    ctx->launches += (long long)order * nsteps * per_stage + (ctx->basis ? 0 : 2);
    return DGSWE_OK;
}

int dgswe_ssprk3(dgswe_ctx *ctx, double *u, double *w1, double *w2, double dt, int nsteps, int check_mean,
                 void *stream)
{
    return dgswe_rk_steps(ctx, 3, u, w1, w2, nullptr, dt, nsteps, check_mean, stream);
}

int dgswe_status_tags(dgswe_ctx *ctx, uint32_t *flags, int32_t *tags, int reset, void *stream)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    cudaStream_t s = (cudaStream_t)stream;
    // read (into pinned host memory) and reset in stream order, one synchronisation
    DevStatus *h = ctx->status_host;
    CUDA_TRY(cudaMemcpyAsync(h, ctx->status, sizeof *h, cudaMemcpyDeviceToHost, s));
    if (reset) CUDA_TRY(cudaMemcpyAsync(ctx->status, h + 1, sizeof *h, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (flags) *flags = h->flags;
    if (tags)
        for (int b = 0; b < dgswe::kStatusBits; ++b) tags[b] = h->first_tag[b];
    return DGSWE_OK;
}

// -- linear advection on the periodic plane (dgswe_adv.cuh) ---------------

struct dgswe_adv_ctx {
    dgswe_adv_cfg cfg;
    dgswe::AdvParams ap;
    const DegreeOps *ops;
};

int dgswe_adv_create(const dgswe_adv_cfg *cfg, const double *leg, const double *dleg, const double *weights,
                     dgswe_adv_ctx **out)
{
    if (!cfg || !leg || !dleg || !weights || !out) return dgswe_fail(DGSWE_EINVAL, "null argument");
    *out = nullptr;
    const dgswe_adv_cfg &c = *cfg;
    if (c.p < 0 || c.p > dgswe::kMaxP) return dgswe_fail(DGSWE_EUNSUPPORTED, "degree %d outside 0..%d", c.p, dgswe::kMaxP);
    if (c.nx < 1 || c.ny < 1 || c.nz < 1 || !(c.dx > 0) || !(c.dy > 0) || !std::isfinite(c.beta_x) ||
        !std::isfinite(c.beta_y))
        return dgswe_fail(DGSWE_EINVAL, "bad advection configuration");
    const int n = c.p + 1;
    const DegreeOps *ops = dgswe_degree_ops(c.p);
    const int rc = ops->upload(nodal_tables(leg, dleg, weights, n));
    if (rc) return rc;
    dgswe_adv_ctx *ctx = new (std::nothrow) dgswe_adv_ctx();
    if (!ctx) return dgswe_fail(DGSWE_ENOMEM, "out of host memory");
    ctx->cfg = c;
    ctx->ops = ops;
    dgswe::AdvParams &ap = ctx->ap;
    // mesh scalars as the reference forms them (mesh.py:66-84, dg.py:199-213)
    const double determ = c.dx * c.dy / 4.0;
    ap.nx = c.nx;
    ap.ny = c.ny;
    ap.zstride = (long long)c.nx * c.ny * n * n;
    ap.bx = c.beta_x;
    ap.by = c.beta_y;
    ap.ax = std::fabs(c.beta_x);   // the model's wavespeed (models.py:129-131), local = global
    ap.ay = std::fabs(c.beta_y);
    ap.bdx = c.dx / 2.0;
    ap.bdy = c.dy / 2.0;
    ap.cx = determ / ap.bdx;
    ap.cy = determ / ap.bdy;
    ap.inv_determ = 1.0 / determ;
    *out = ctx;
    return DGSWE_OK;
}

int dgswe_adv_set_alpha(dgswe_adv_ctx *ctx, double alpha)
{
    if (!ctx) return dgswe_fail(DGSWE_EINVAL, "null context");
    if (!(alpha >= 0.0) || !std::isfinite(alpha)) return dgswe_fail(DGSWE_EINVAL, "alpha must be finite and >= 0");
    ctx->ap.ax = alpha;
    ctx->ap.ay = alpha;
    return DGSWE_OK;
}

void dgswe_adv_destroy(dgswe_adv_ctx *ctx) { delete ctx; }

int dgswe_adv_stage(dgswe_adv_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                    void *stream)
{
    if (!ctx || !X || !Y) return dgswe_fail(DGSWE_EINVAL, "null argument");
    if (X == Y) return dgswe_fail(DGSWE_EINVAL, "the output must not alias the stage input");
    if (a != 0.0 && !U) return dgswe_fail(DGSWE_EINVAL, "U is required when a != 0");
    dgswe::AdvParams ap = ctx->ap;
    ap.X = X;
    ap.U = a != 0.0 ? U : nullptr;
    ap.Y = Y;
    ap.a = a;
    ap.b = b;
    ap.g = g;
    return ctx->ops->adv_stage(ap, ctx->cfg.nz, (cudaStream_t)stream);
}

int dgswe_status(dgswe_ctx *ctx, uint32_t *flags, int32_t *first_tag, int reset, void *stream)
{
    int32_t tags[dgswe::kStatusBits];
    const int rc = dgswe_status_tags(ctx, flags, tags, reset, stream);
    if (rc) return rc;
    if (first_tag) {
        int32_t m = INT_MAX;
        for (int b = 0; b < dgswe::kStatusBits; ++b) m = tags[b] < m ? tags[b] : m;
        *first_tag = m;
    }
    return DGSWE_OK;
}

int64_t dgswe_launch_count(const dgswe_ctx *ctx) { return ctx ? ctx->launches : 0; }

// ---- device diagnostics and IC projection (dgswe_diag.cuh) ----

static dgswe::DiagLayout diag_layout(const dgswe_ctx *c)
{
    return {c->zstride, c->rstride, c->vstride, c->cfg.nx, c->cfg.ny, c->nphi};
}

static int check_diag(const dgswe_ctx *c, const double *X, int var, int level)
{
    if (!c || !X) return dgswe_fail(DGSWE_EINVAL, "null argument");
    if (var < 0 || var > 2 || level < 0 || level >= c->cfg.nz) return dgswe_fail(DGSWE_EINVAL, "bad var/level");
    if (c->cfg.row0 != 0 || c->cfg.nrows != c->cfg.ny)
        return dgswe_fail(DGSWE_EINVAL, "diagnostics need a single-band context");
    return DGSWE_OK;
}

int dgswe_mass(dgswe_ctx *ctx, const double *X, int var, int level, const double *m0_rows, double *out,
               void *stream)
{
    int rc = check_diag(ctx, X, var, level);
    if (rc) return rc;
    if (!m0_rows || !out) return dgswe_fail(DGSWE_EINVAL, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, nphi = ctx->nphi;
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
    if (!phi2 || !wrow || !ref || !out2 || nq2 < 1) return dgswe_fail(DGSWE_EINVAL, "bad argument");
    if (nq2 > ctx->nq2_max) return dgswe_fail(DGSWE_EINVAL, "l2 rule of %d nodes > (p+2)^2", nq2);
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, nphi = ctx->nphi;
    const size_t nt = (size_t)nq2 * nphi + (size_t)ny * nq2;
    double *dphi = ctx->diag, *dw = dphi + (size_t)nq2 * nphi, *part = ctx->diag + nt, *res = part + 4 * (size_t)ny;
    CUDA_TRY(cudaMemcpyAsync(dphi, phi2, sizeof(double) * nq2 * nphi, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dw, wrow, sizeof(double) * ny * nq2, cudaMemcpyHostToDevice, s));
    const dgswe::DiagLayout L = diag_layout(ctx);
    dgswe::l2_rows_kernel<<<dim3(ny, 1), 256, 0, s>>>(X + (size_t)level * ctx->zstride, L, var, dphi, nq2, dw, ref,
                                                       part);
    dgswe::rows_total_kernel<2><<<1, 256, 0, s>>>(part, ny, 0, res);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 2;
    CUDA_TRY(cudaMemcpyAsync(out2, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DGSWE_OK;
}

int dgswe_project(dgswe_ctx *ctx, const double *fvals, const double *cos_nodes, double determ, double *Y,
                  void *stream)
{
    if (!ctx || !fvals || !cos_nodes || !Y) return dgswe_fail(DGSWE_EINVAL, "null argument");
    if (ctx->cfg.row0 != 0 || ctx->cfg.nrows != ctx->cfg.ny)
        return dgswe_fail(DGSWE_EINVAL, "projection needs a single-band context");
    cudaStream_t s = (cudaStream_t)stream;
    const int ny = ctx->cfg.ny, n = ctx->n;
    CUDA_TRY(cudaMemcpyAsync(ctx->diag, cos_nodes, sizeof(double) * ny * n, cudaMemcpyHostToDevice, s));
    const int rc = ctx->ops->project(ctx, fvals, ctx->diag, determ, Y, s);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(s));   // the host staging buffers may be reused by the caller
    return DGSWE_OK;
}

}  // extern "C"
