// dgswe_degree.cuh -- host launchers of the kernels of ONE degree P.  Each
// deg_pP.cu includes this file and instantiates DGSWE_DEGREE_UNIT(P): the
// seven degrees compile in parallel, and each unit owns its copy of the
// __constant__ nodal tables (uploaded by ops->upload in dgswe_create).
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstring>

#include "dgswe_ctx.h"
#include "dgswe_kernels.cuh"
#include "dgswe_lo.cuh"
#include "dgswe_adv.cuh"

namespace dgswe_deg {

using dgswe::StageParams;

template <int P>
int upload(const dgswe::NodTab &nt)
{
    CUDA_TRY(cudaMemcpyToSymbol(dgswe::c_nod, &nt, sizeof nt, sizeof nt * P));
    return DGSWE_OK;
}

template <int P, int F>
size_t stage_smem(const dgswe_ctx *c)
{
    using SM = dgswe::Smem<P>;
    return (size_t)((F & dgswe::kOrog) ? SM::TOTAL_OROG : SM::TOTAL) * sizeof(double) + (size_t)c->smem_pad;
}

// resident CTAs per SM of variant F (queried once per context: the context
// is bound to one device)
template <int P, int F>
int occupancy(dgswe_ctx *c)
{
    if (!c->occ[F]) {
        const size_t smem = stage_smem<P, F>(c);
        CUDA_TRY(cudaFuncSetAttribute(dgswe::stage_kernel<P, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        int o = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, dgswe::stage_kernel<P, F>, dgswe::kThreads,
                                                               smem));
        c->occ[F] = o > 0 ? o : 1;
    }
    return c->occ[F];
}

// Row chunking: every (strip, level) column of rows is split into
// contiguous chunks, one CTA each.  The chunk count minimises the modelled
// makespan  waves * (rows per chunk + kChunkOverhead), where waves =
// ceil(CTAs / resident slots) and the overhead (prologue and first-row
// work, measured ~1.4 rows) favours long chunks.  Narrow grids get one full
// wave; wide grids, whose strips alone outnumber the slots, get several
// waves of short chunks instead of one under-filled wave of very long ones.
struct ChunkPlan {
    int rc;     // rows per chunk (uniform chunks), or
    int even;   // > 0: this many chunks of floor/ceil(rows / even) rows
};

template <int P>
ChunkPlan chunk_plan(const dgswe_ctx *c, int rows, int o)
{
    constexpr double kChunkOverhead = 1.5;
    const long long slots = (long long)c->sms * o;
    const long long cols = (long long)c->nstrip * c->cfg.nz;
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
    ChunkPlan plan{(int)((rows + best_chunks - 1) / best_chunks), 0};
    // Second look (p = 3), by the busiest SM's row work: CTAs share their
    // SM's issue and FP64 throughput, so a one-wave grid runs at the pace of
    // its most loaded SMs.  Candidates: uniform chunks long enough for at
    // most o-1 CTAs per SM, and the largest one-wave grid of evenly split
    // chunks (o CTAs on most SMs; a fully occupied SM hides latency better:
    // ~5% more row work per unit time, measured at 4 vs 3 CTAs).  C3: 23
    // strips x 25 even chunks of 14-15 rows (575 CTAs, 4 on 131 SMs) beats
    // 19 x 19 rows at 3 per SM (+1.7%), which beat 24 x 15 at 4 on 108 SMs
    // (+1.4%).  At p = 2 the lighter CTAs want every slot (-3% with o-1),
    // at p >= 4 o - 1 = 1 CTA per SM.
    if (P == 3 && o > 1 && cols * best_chunks <= slots) {
        auto sm_load = [&](long long ch, bool even) {
            const double per = even ? (double)rows / (double)ch : (double)((rows + ch - 1) / ch);
            const long long per_sm = (cols * ch + c->sms - 1) / c->sms;
            return (double)per_sm * (per + 1.0) / (per_sm >= o ? 1.05 : 1.0);
        };
        double cost = sm_load(best_chunks, false);
        for (long long ch = 1; ch <= rows && cols * ch <= (long long)c->sms * (o - 1); ++ch) {
            if ((cols * ch + c->sms - 1) / c->sms != o - 1) continue;   // exactly o-1 on the busiest SM
            const double t = sm_load(ch, false);
            if (t < 0.95 * cost) {
                cost = t;
                plan = ChunkPlan{(int)((rows + ch - 1) / ch), 0};
            }
        }
        const long long ch = slots / cols < rows ? slots / cols : rows;
        if (ch >= 1 && (double)rows / (double)ch >= 4.0 && sm_load(ch, true) < cost) plan = ChunkPlan{0, (int)ch};
    }
    return plan;
}

// The low-order degree (p = 0), plain nodal stages: the barrier-free kernel of
// dgswe_lo.cuh, four strips per CTA, evenly split row chunks filling one
// wave of resident CTAs (or several waves of ~8-row chunks on wide grids).
template <int P, int F>
int launch_lo(dgswe_ctx *c, const StageParams &kp0, cudaStream_t s)
{
    int &o = c->occ_lo[F & 1];
    constexpr int smem = dgswe::lo_smem_bytes<P, (F & dgswe::kHasU) != 0>();
    if (!o) {
        CUDA_TRY(cudaFuncSetAttribute(dgswe::lo_stage_kernel<P, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int q = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, dgswe::lo_stage_kernel<P, F>,
                                                               dgswe::kLoWarps * dgswe::kLanes, smem));
        o = q > 0 ? q : 1;
    }
    StageParams kp = kp0;
    const int rows = kp.j_end - kp.j_begin;
    const int segs = dgswe::lo_segments(c->cfg.nx);
    const long long cols = (long long)((segs + dgswe::kLoWarps - 1) / dgswe::kLoWarps) * c->cfg.nz;
    const long long slots = (long long)c->sms * o;
    long long nch = slots / cols;                        // one full wave
    if (nch < 1) nch = (rows + 7) / 8;                   // wide grids: ~8-row chunks, several waves
    if (c->even_chunks > 0) nch = c->even_chunks;
    if (nch > rows) nch = rows;
    if (kp.rc > 0) {                                     // explicit rows per chunk (row_chunk)
        nch = (rows + kp.rc - 1) / kp.rc;
        kp.even = 0;
    } else {
        kp.even = (int)nch;
    }
    const dim3 grid((segs + dgswe::kLoWarps - 1) / dgswe::kLoWarps, (unsigned)nch, c->cfg.nz);
    dgswe::lo_stage_kernel<P, F><<<grid, dgswe::kLoWarps * dgswe::kLanes, smem, s>>>(kp);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

template <int P, int F>
int launch_variant(dgswe_ctx *c, const StageParams &kp0, cudaStream_t s)
{
    if constexpr (dgswe::lo_kernel_degree<P>() && (F & ~dgswe::kHasU) == 0) {
        if (!c->no_lo && kp0.j_end2 <= kp0.j_begin2) return launch_lo<P, F>(c, kp0, s);
    }
    const int o = occupancy<P, F>(c);
    if (o < 0) return o;
    StageParams kp = kp0;
    int nchunks;
    if (F & dgswe::kEdge) {
        // the whole band: its two edge rows as single-row CTAs, then the
        // interior rows [band_lo+1, band_hi-1) in chunks
        const int nedge = kp.band_hi - kp.band_lo < 2 ? kp.band_hi - kp.band_lo : 2;
        const int inner = kp.band_hi - kp.band_lo - 2 > 0 ? kp.band_hi - kp.band_lo - 2 : 0;
        ChunkPlan plan{kp.rc > 0 ? kp.rc : 1, 0};
        if (kp.rc <= 0 && inner > 0) plan = c->even_chunks > 0 ? ChunkPlan{0, c->even_chunks} : chunk_plan<P>(c, inner, o);
        if (plan.even > 0) {
            kp.even = plan.even < inner ? plan.even : inner;
            nchunks = nedge + kp.even;
        } else {
            kp.rc = plan.rc;
            nchunks = nedge + (inner + plan.rc - 1) / plan.rc;
        }
    } else {
        const int rows1 = kp.j_end - kp.j_begin, rows2 = kp.j_end2 - kp.j_begin2;
        const int rows = rows1 > rows2 ? rows1 : rows2;
        if (rows <= 0) return DGSWE_OK;
        ChunkPlan plan{kp.rc, 0};
        if (kp.rc <= 0) plan = c->even_chunks > 0 ? ChunkPlan{0, c->even_chunks} : chunk_plan<P>(c, rows, o);
        if (plan.even > 0 && rows2 > 0) plan = ChunkPlan{(rows + plan.even - 1) / plan.even, 0};
        const int rc = plan.rc;
        if (plan.even > 0) {
            kp.even = plan.even < rows1 ? plan.even : rows1;
            nchunks = kp.even;
        } else {
            kp.rc = rc;
            nchunks = (rows1 + rc - 1) / rc;
        }
        if (rows2 > 0) {   // a second row range in the same launch
            kp.nchunk1 = nchunks;
            nchunks += (rows2 + rc - 1) / rc;
        }
    }
    const dim3 grid(c->nstrip, nchunks, c->cfg.nz);
    dgswe::stage_kernel<P, F><<<grid, dgswe::kThreads, stage_smem<P, F>(c), s>>>(kp);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

// the 20 instantiated variants: every combination of U, Y2, MODAL, OROG,
// and the edge launches (nodal, one output) with or without U / OROG
#define DGSWE_VARIANTS(X)                                                                   \
    X(0) X(1) X(2) X(3) X(8) X(9) X(10) X(11) X(16) X(17) X(18) X(19) X(24) X(25) X(26) X(27) \
    X(4) X(5) X(20) X(21)

template <int P>
int stage(dgswe_ctx *c, const StageParams &kp, cudaStream_t s)
{
    const int F = (kp.U ? dgswe::kHasU : 0) | (kp.Y2 ? dgswe::kHasY2 : 0) | (kp.edge ? dgswe::kEdge : 0) |
                  (kp.modal ? dgswe::kModal : 0) | (kp.orog ? dgswe::kOrog : 0);
    switch (F) {
#define DGSWE_CASE(f) \
    case f: return launch_variant<P, f>(c, kp, s);
        DGSWE_VARIANTS(DGSWE_CASE)
#undef DGSWE_CASE
    default: return dgswe_fail(DGSWE_EUNSUPPORTED, "stage variant %d not built (edge launches are nodal, one output)", F);
    }
}

template <int P>
int adv_stage(const dgswe::AdvParams &ap, int nz, cudaStream_t s)
{
    if constexpr (dgswe::adv_marching<P>()) {
        // 16-row chunks (4096^2, p = 2: 8 / 16 / 32 rows 0.44 / 0.45 / 0.43)
        dgswe::AdvParams a2 = ap;
        const int rc = 16;
        a2.rc = rc;
        const dim3 grid((dgswe::adv_segments(ap.nx) + 3) / 4, (ap.ny + rc - 1) / rc, nz);
        dgswe::adv_stage_kernel<P><<<grid, 128, 0, s>>>(a2);
    } else {
        const dim3 grid((ap.nx + 127) / 128, ap.ny, nz);
        dgswe::adv_elem_kernel<P><<<grid, 128, 0, s>>>(ap);
    }
    CUDA_TRY(cudaGetLastError());
    return DGSWE_OK;
}

template <int P>
int convert(dgswe_ctx *c, const double *in, double *out, bool to_nodal, int r0, int r1, cudaStream_t s)
{
    if (r1 <= r0) return DGSWE_OK;
    const dim3 grid(c->nstrip, r1 - r0, c->cfg.nz);
    if (to_nodal)
        dgswe::convert_kernel<P, true><<<grid, 96, 0, s>>>(in, out, c->zstride, c->rstride, c->vstride, r0);
    else
        dgswe::convert_kernel<P, false><<<grid, 96, 0, s>>>(in, out, c->zstride, c->rstride, c->vstride, r0);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

template <int P>
int alpha(dgswe_ctx *c, const double *X, bool modal, cudaStream_t s)
{
    CUDA_TRY(cudaMemsetAsync(c->alpha, 0, 2 * sizeof(double), s));
    const int rows = c->cfg.jhi - c->cfg.jlo;
    const dim3 grid((c->cfg.nx + 127) / 128, rows, c->cfg.nz);
    if (modal)
        dgswe::alpha_prepass_kernel<P, true><<<grid, 128, 0, s>>>(
            X, c->zstride, c->rstride, c->vstride, c->cfg.nx, c->cfg.row0, c->cfg.jlo, c->cfg.jhi, c->cos_edge,
            c->inv_r, c->cfg.gravity, c->cfg.h_floor, c->alpha);
    else
        dgswe::alpha_prepass_kernel<P, false><<<grid, 128, 0, s>>>(
            X, c->zstride, c->rstride, c->vstride, c->cfg.nx, c->cfg.row0, c->cfg.jlo, c->cfg.jhi, c->cos_edge,
            c->inv_r, c->cfg.gravity, c->cfg.h_floor, c->alpha);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

template <int P>
int project(dgswe_ctx *c, const double *f, const double *cosn, double determ, double *Y, cudaStream_t s)
{
    const dim3 grid((c->cfg.nx + 127) / 128, c->cfg.ny, 3);
    const dgswe::DiagLayout L{c->zstride, c->rstride, c->vstride, c->cfg.nx, c->cfg.ny, c->nphi};
    dgswe::project_kernel<P><<<grid, 128, 0, s>>>(f, cosn, c->rowtab, dgswe::row_stride(P),
                                                  dgswe::RowLayout<P>::T, L, c->cfg.nz, determ, Y);
    CUDA_TRY(cudaGetLastError());
    c->launches += 1;
    return DGSWE_OK;
}

}  // namespace dgswe_deg

#ifdef DG_TIMING
// experiment builds only: per-role phase cycle sums of degree P since the last call
#define DGSWE_TIMING_HOOK(P)                                                                     \
    extern "C" int dgswe_debug_timing_p##P(unsigned long long *out28)                             \
    {                                                                                            \
        CUDA_TRY(cudaDeviceSynchronize());                                                       \
        CUDA_TRY(cudaMemcpyFromSymbol(out28, dgswe::g_timing, sizeof(unsigned long long) * 28)); \
        static const unsigned long long zero[28] = {};                                           \
        CUDA_TRY(cudaMemcpyToSymbol(dgswe::g_timing, zero, sizeof zero));                        \
        return DGSWE_OK;                                                                         \
    }
#else
#define DGSWE_TIMING_HOOK(P)
#endif

#define DGSWE_DEGREE_UNIT(P)                                                                     \
    DGSWE_TIMING_HOOK(P)                                                                         \
    const DegreeOps *dgswe_degree_ops_##P()                                                      \
    {                                                                                            \
        static const DegreeOps ops = {dgswe_deg::upload<P>, dgswe_deg::stage<P>,                 \
                                      dgswe_deg::convert<P>, dgswe_deg::alpha<P>,                \
                                      dgswe_deg::project<P>, dgswe_deg::adv_stage<P>};           \
        return &ops;                                                                             \
    }
