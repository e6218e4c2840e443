/*
 * dgswe_b200.h -- C ABI of the B200 (sm_100a, fp64) DG shallow-water
 * time-stepping path.  Plain pointers and sizes only; every device buffer is
 * owned by the caller (PyTorch in this repo), the context owns only the
 * uploaded constant tables, a status word and cached CUDA graphs.
 *
 * Each entry point replaces one reference interface
 * (/root/reference/pkg/src/dgswe/<file>:<line>):
 *
 *   dgswe_create / dgswe_destroy   SpatialOperator.__init__ precomputation
 *                                  (dg.py:174-219, _setup_mass 223-239,
 *                                  _setup_coords 254-283)
 *   dgswe_rhs                      SpatialOperator.assemble_rhs (dg.py:504-523)
 *                                  incl. _halo_exchange 330-346, nodal_eval
 *                                  348-357, _pointwise_physics 359-372,
 *                                  _interface_alphas 385-421,
 *                                  _interface_fluxes 423-453, _contract 455-502
 *   dgswe_stage                    one RK stage: rhs + the stage update of
 *                                  rk_step (timestep.py:149-167), fused
 *   dgswe_axpy                     timestep._axpy (timestep.py:132-141) and the
 *                                  finite check of rk_step (165-166)
 *   dgswe_stage2                   an RK4 stage with the accumulator as a
 *                                  second output (timestep.py:71-81, 163-164)
 *   dgswe_rk_steps / dgswe_ssprk3  integrate's step loop (timestep.py:210-229)
 *                                  for tableau(1..4) (timestep.py:57-82), as
 *                                  fused stages, CUDA-graph batched
 *   dgswe_alpha_prepass            global Rusanov alpha (dg.py:389-411)
 *   dgswe_status / _status_tags    PositivityError (models.py:143-146) and
 *                                  DivergenceError (timestep.py:165-166,
 *                                  220-226) as device status bits, with the
 *                                  first failing step per bit
 *   dgswe_mass / dgswe_l2_sums     diagnostics.mass_integral / l2_error
 *                                  (diagnostics.py:92-107, 42-80)
 *   dgswe_project                  basis.project_initial (basis.py:206-233)
 *   dgswe_stage_band + exchange    _halo_exchange (dg.py:330-346) across GPUs:
 *                                  latitude bands, peer-memory stores
 *
 * Layout of every state buffer (fp64), strip-blocked structure of arrays:
 *   [nz][nrows][3][nstrip][nphi][DGSWE_STRIP]
 *   variable v in {h, hu, hv}; mode m = a*(p+1)+b (a: lambda degree,
 *   b: theta degree, basis.py:5-13); longitude element i = DGSWE_STRIP*s + l
 *   at strip s, lane l; nstrip = ceil(nx / DGSWE_STRIP).  Lanes i >= nx of
 *   the last strip are padding: never written, they must hold finite values
 *   (zero them once).  One variable's row tile of a strip is contiguous
 *   (nphi * DGSWE_STRIP doubles), the unit of the kernel's TMA copies.
 *   Buffer row r holds global latitude row row0 + r.  The rows computed are
 *   [jlo, jhi) (local); a band's halo rows jlo-1 and jhi must hold the
 *   neighbour band's coefficients whenever they are inside the sphere.
 *
 * State basis.  The reference's states are modal coefficients, and so are
 * this ABI's by default.  Inside a step the kernels carry the values at the
 * (p+1)^2 Gauss nodes instead (u[i][j] in place of mode (a, b), same
 * layout): with every integral of the reference on that Gauss rule the
 * nodal form is the same linear operator with a diagonal mass matrix.
 * dgswe_rk_steps converts u in place before and after its steps; the
 * single-stage entry points (dgswe_rhs, dgswe_stage*) take modal states in
 * ONE launch: every row tile is converted to nodal values in shared memory
 * as it lands and the outputs back to modes in registers.  A caller that
 * keeps its states nodal across many stages (a band driver) calls
 * dgswe_set_basis(ctx, 1) and dgswe_convert itself: then dgswe_rhs,
 * dgswe_stage*, dgswe_alpha_prepass and dgswe_rk_steps take and return
 * nodal states unchanged.  dgswe_stage_band requires the nodal basis.
 * Diagnostics (dgswe_mass, dgswe_l2_sums) and dgswe_project always use
 * modal states.
 *
 * Ownership: the caller owns every state buffer; the
 * context owns the constant tables, status words, the global-alpha pair, a
 * fixed-size diagnostics scratch and cached CUDA graphs, all allocated by
 * dgswe_create -- no other entry point allocates device memory.  State
 * pointers must be 16-byte aligned (TMA bulk copies; DGSWE_EINVAL else).
 * A context holds no process-global mutable state: contexts on different
 * threads / devices are independent (one host thread per context).
 *
 * All calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default) except dgswe_status, which synchronises it.  Return 0 on success,
 * a negative DGSWE_E* code otherwise; dgswe_last_error() describes it.
 */
#ifndef DGSWE_B200_H
#define DGSWE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGSWE_ABI_VERSION 5
#define DGSWE_STRIP 32          /* longitude elements per strip block */

/* status bits (dgswe_status) */
#define DGSWE_STATUS_POSITIVITY 0x1u  /* h <= 0 (or NaN) at a quadrature node */
#define DGSWE_STATUS_NONFINITE 0x2u   /* non-finite coefficient after an update */
#define DGSWE_STATUS_MEAN_NONPOS 0x4u /* cell-mean h <= 0 (check_positivity) */
#define DGSWE_STATUS_PEER_TIMEOUT 0x8u /* a band neighbour's halo rows never arrived */
#define DGSWE_STATUS_BITS 4

/* error codes */
#define DGSWE_OK 0
#define DGSWE_EINVAL (-1)
#define DGSWE_ECUDA (-2)
#define DGSWE_ENOMEM (-3)
#define DGSWE_EUNSUPPORTED (-4)

/* Rusanov alpha mode (dg.py:47-57) */
#define DGSWE_ALPHA_LOCAL 0
#define DGSWE_ALPHA_GLOBAL_PINNED 1
#define DGSWE_ALPHA_GLOBAL 2

typedef struct dgswe_cfg {
    int nx, ny, nz, p;        /* global element grid, levels, degree (0..6) */
    int row0;                 /* global latitude row of buffer row 0 */
    int nrows;                /* rows in every state buffer */
    int jlo, jhi;             /* local rows computed by this context */
    double radius;            /* R (mesh.py:28) */
    double gravity;           /* g (mesh.py:30) */
    double h_floor;           /* velocity-recovery floor, 1e-8*h_ref (models.py:159) */
    double dx, dy;            /* element extents in lambda / theta (mesh.py:66-72) */
    int alpha_mode;           /* DGSWE_ALPHA_* */
    double alpha;             /* pinned alpha for DGSWE_ALPHA_GLOBAL_PINNED */
    int row_chunk;            /* latitude rows per CTA, 0 = automatic */
    int periodic_y;           /* 1: y-periodic planar mesh (mesh.py:120-132): rows wrap, no pole
                                 faces; the lat-lon tables then describe the plane (cos = 1,
                                 sin = 0, f = const, radius = 1).  Single band only. */
} dgswe_cfg;

/* Host tables; copied during dgswe_create, not retained. */
typedef struct dgswe_tables {
    const double *leg;        /* (n, n): P_a(x_q), row a      (basis.py:58-66)  */
    const double *dleg;       /* (n, n): P'_a(x_q), row a     (basis.py:69-81)  */
    const double *weights;    /* (n): Gauss weights            (basis.py:50-55)  */
    const double *cos_r_int;  /* (ny, n): cos(theta)/R at interior node latitudes  (dg.py:248,268) */
    const double *sin_r_int;  /* (ny, n): sin(theta)/R */
    const double *fcos_int;   /* (ny, n): 2 Omega sin cos */
    const double *cos_r_edge; /* (ny+1): cos/R at edge latitude y_edges[e] (dg.py:276-282) */
    const double *cos_edge;   /* (ny+1): cos(y_edges[e]) for the y-direction alpha (models.py:280) */
    const double *minv;       /* (ny, nphi, nphi): per-row inverse mass (basis.py:159-190) */
    const double *orog;       /* NULL, or (ny, nx, (p+1)^2): bottom height b at the Gauss nodes
                                 (q = qi*(p+1)+qj, qi along lambda); adds the momentum sources
                                 -(g h/R) db/dlambda, -(g h cos/R) db/dtheta (Williamson TC5;
                                 not in the reference) */
} dgswe_tables;

typedef struct dgswe_ctx dgswe_ctx;

/* Linear advection u_t + beta . grad u = 0 on the doubly periodic plane
 * (the reference's advection model and advection_sine case, models.py:114-140,
 * cases.py:99-110): one fused stage kernel, Y = a U + b X + g RHS(X), on
 * modal coefficients laid out [nz][ny][nphi][nx].  RHS(X) = stage(0, NULL,
 * 0, X, 1, Y).  Y must not alias X. */
typedef struct dgswe_adv_cfg {
    int nx, ny, nz, p;
    double dx, dy;            /* element extents (mesh.py:66-72) */
    double beta_x, beta_y;    /* advection velocity (models.py:117-121) */
} dgswe_adv_cfg;
typedef struct dgswe_adv_ctx dgswe_adv_ctx;
int dgswe_adv_create(const dgswe_adv_cfg *cfg, const double *leg, const double *dleg, const double *weights,
                     dgswe_adv_ctx **out);
int dgswe_adv_stage(dgswe_adv_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                    void *stream);
/* Pinned global Rusanov alpha for both directions (RusanovParams("global",
 * alpha), dg.py:47-57, 389-392); default: |beta_x|, |beta_y| (the model's
 * wavespeed: local and global modes coincide for constant beta). */
int dgswe_adv_set_alpha(dgswe_adv_ctx *ctx, double alpha);
void dgswe_adv_destroy(dgswe_adv_ctx *ctx);

int dgswe_abi_version(void);
const char *dgswe_last_error(void);

int dgswe_create(const dgswe_cfg *cfg, const dgswe_tables *tables, dgswe_ctx **out);
void dgswe_destroy(dgswe_ctx *ctx);

/* elements of one state buffer (nz * nrows * 3 * nstrip * nphi * DGSWE_STRIP) */
int64_t dgswe_state_elems(const dgswe_ctx *ctx);

/* 0: modal states at the stage entry points (default), 1: nodal. */
int dgswe_set_basis(dgswe_ctx *ctx, int nodal);

/* In-place change of basis (to_nodal 1: modal -> nodal, 0: back) of local
 * rows [r0, r1) of every level; padding lanes stay zero. */
int dgswe_convert(dgswe_ctx *ctx, double *X, int to_nodal, int r0, int r1, void *stream);

/* K = M^-1 (volume - boundary + source)(X) on rows [jlo, jhi). */
int dgswe_rhs(dgswe_ctx *ctx, const double *X, double *K, void *stream);

/* Y = a*U + b*X + g*RHS(X) on rows [jlo, jhi); U may be NULL when a == 0.
 * Y must not alias X; Y may alias U.  `tag` is recorded as the step index
 * of the first status flag raised (dgswe_status). */
int dgswe_stage(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                double *Y, int tag, void *stream);

/* Same, restricted to local rows [r0, r1) (for interior/boundary overlap). */
int dgswe_stage_rows(dgswe_ctx *ctx, double a, const double *U, double b, const double *X,
                     double g, double *Y, int tag, int r0, int r1, void *stream);

/* ---- fused halo exchange over peer memory (one process per GPU) ----
 * dgswe_stage_band computes the band's rows [jlo, jhi) in ONE launch: its
 * two edge rows (jlo, jhi-1) as the first, single-row CTAs, then the
 * interior rows in chunks.  An edge CTA stores its output row both locally
 * and straight into the neighbour's halo row (peer pointers from CUDA IPC:
 * dgswe_ipc_handle / dgswe_ipc_open), then counts each delivered strip
 * block in the neighbour's receive counter (system-scope atomic after a
 * system fence).  Before computing, an edge CTA waits (bounded: see
 * dgswe_set_peer_timeout) until its own receive counter shows the
 * neighbour's edge rows of the previous stage; interior CTAs need no halo
 * and run at once -- no host collective, no second stream.
 * dgswe_set_exchange registers, once per context: the neighbours' level
 * strides and receive counters (NULL at a pole), and this band's own
 * counters: recv_count[2] (south, north deliveries) and stage_ctr[2]
 * (completed band launches, CTA completion scratch), zeroed.
 * peer_row_s / peer_row_n: level-0 base of the neighbour's halo row in the
 * buffer that plays Y's role there (NULL at a pole).  Nodal states only. */
int dgswe_set_exchange(dgswe_ctx *ctx, long long peer_zstride_s, unsigned long long *peer_count_s,
                       long long peer_zstride_n, unsigned long long *peer_count_n,
                       unsigned long long *recv_count, unsigned long long *stage_ctr);
int dgswe_stage_band(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g, double *Y,
                     int tag, double *peer_row_s, double *peer_row_n, void *stream);
/* device memory the neighbours can map (zero-filled), and its IPC handles */
int dgswe_dev_alloc(size_t bytes, void **out);
int dgswe_dev_free(void *p);
int dgswe_ipc_handle(void *p, char *out64);
int dgswe_ipc_open(const char *in64, void **out);
int dgswe_ipc_close(void *p);

/* Same over two row ranges [r0, r1) and [r2, r3) (r1 <= r2) in ONE launch:
 * a band's two boundary rows after its halo exchange. */
int dgswe_stage_rows2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X,
                      double g, double *Y, int tag, int r0, int r1, int r2, int r3, void *stream);

/* Nodal basis only: Y = a*U + b*X + g*RHS(X) on local rows [r0, r1) with the
 * status checks of a step's last stage (non-finite output, optional cell
 * mean) -- the row-pipelined host-state step of the Python API
 * (SpatialOperator.ssprk3_step_host: host<->device copies overlapped with
 * the stages of row chunks). */
int dgswe_stage_rows_checked(dgswe_ctx *ctx, double a, const double *U, double b, const double *X,
                             double g, double *Y, int tag, int r0, int r1, int check_finite,
                             int check_mean, void *stream);

/* Y = a*U + b*X + g*RHS(X) and Y2 = A + g2*RHS(X) in one launch, on local
 * rows [r0, r1): the stage of classical RK4 whose second output is the
 * running accumulator u + sum_i dt b_i k_i (timestep.py:71-81, 163-164).
 * Y2 may alias A; neither output may alias X. */
int dgswe_stage2(dgswe_ctx *ctx, double a, const double *U, double b, const double *X, double g,
                 double *Y, const double *A, double g2, double *Y2, int tag, int r0, int r1,
                 void *stream);

/* y = y + x*coef on rows [jlo, jhi), two roundings (timestep.py:137-141);
 * check_finite != 0 raises DGSWE_STATUS_NONFINITE for non-finite results. */
int dgswe_axpy(dgswe_ctx *ctx, double coef, const double *x, double *y, int check_finite,
               int tag, void *stream);

/* nsteps of the explicit RK method of `order` 1..4 (tableau(order) of
 * timestep.py:57-82, fused stage form: Euler, Heun/SSPRK2 and SSPRK3 in
 * Shu-Osher form, classical RK4 with its accumulator as a second kernel
 * output) on u in place, scratch w1 (all orders), w2 (order >= 3), w3
 * (order 4); one CUDA graph per (order, buffers, dt, nsteps).  Status tags
 * are the 0-based step index within the call.  Single-band contexts only. */
int dgswe_rk_steps(dgswe_ctx *ctx, int order, double *u, double *w1, double *w2, double *w3, double dt,
                   int nsteps, int check_mean, void *stream);

/* nsteps of Shu-Osher SSPRK3 on u (in place) with scratch w1, w2, batched
 * into one CUDA graph per (buffers, dt, nsteps).  check_mean != 0 enables
 * the per-step cell-mean check on h (timestep.py:220-226).  Status tags are
 * the 0-based step index within this call.  Single-band contexts only. */
int dgswe_ssprk3(dgswe_ctx *ctx, double *u, double *w1, double *w2, double dt, int nsteps,
                 int check_mean, void *stream);

/* Global-mode alpha: device max over all traces of X into the context's
 * alpha buffer (two doubles, x then y).  dgswe_alpha_buffer exposes it so a
 * multi-GPU caller can all-reduce(MAX) it before dgswe_stage. */
int dgswe_alpha_prepass(dgswe_ctx *ctx, const double *X, void *stream);
double *dgswe_alpha_buffer(dgswe_ctx *ctx);
/* 0: dgswe_stage runs the prepass itself (single GPU); 1: caller does. */
int dgswe_set_external_alpha(dgswe_ctx *ctx, int external);

/* Reads (and optionally clears) the status word; synchronises `stream`.
 * first_tag receives the smallest tag that raised a flag (INT32_MAX if none). */
int dgswe_status(dgswe_ctx *ctx, uint32_t *flags, int32_t *first_tag, int reset, void *stream);
/* Same with the smallest tag per status bit: tags[DGSWE_STATUS_BITS], bit b
 * (POSITIVITY, NONFINITE, MEAN_NONPOS, PEER_TIMEOUT) in tags[b]. */
int dgswe_status_tags(dgswe_ctx *ctx, uint32_t *flags, int32_t *tags, int reset, void *stream);

/* Bound (ns, default 2 s) on a band launch's wait for a neighbour's halo
 * rows; on expiry the launch raises DGSWE_STATUS_PEER_TIMEOUT instead of
 * hanging the GPU (the stage's result is then invalid). */
int dgswe_set_peer_timeout(dgswe_ctx *ctx, unsigned long long timeout_ns);

/* ---- device diagnostics (single-band contexts; synchronise `stream`) ----
 * dgswe_mass: *out = sum over elements of sum_m m0_rows[j][m] c_m of variable
 *   `var`, level `level` (diagnostics.mass_integral, diagnostics.py:92-107);
 *   m0_rows is the host (ny, nphi) array of row 0 of each row's mass matrix.
 * dgswe_l2_sums: out2[0] = sum over elements and the nq2 nodes of a finer
 *   rule of wrow[j][q] (u_q - ref_q)^2, out2[1] = sum of wrow[j][q] ref_q^2,
 *   with u_q = sum_m phi2[q][m] c_m (diagnostics.l2_error, diagnostics.py:
 *   42-80, before the determ factor and sqrt); phi2 (nq2, nphi) and wrow
 *   (ny, nq2) are host arrays, ref is a DEVICE array [ny][nx][nq2].
 * Both reduce in a fixed order in double-double: deterministic run to run. */
int dgswe_mass(dgswe_ctx *ctx, const double *X, int var, int level, const double *m0_rows, double *out,
               void *stream);
int dgswe_l2_sums(dgswe_ctx *ctx, const double *X, int var, int level, const double *phi2, int nq2,
                  const double *wrow, const double *ref, double *out2, void *stream);

/* Initial-condition projection (basis.project_initial, basis.py:206-233):
 * fvals is a DEVICE array [3][ny][nx][(p+1)^2] of nodal values at the Gauss
 * nodes (q = qi*(p+1) + qj, qi along lambda), cos_nodes the host (ny, p+1)
 * cos(theta) of the node latitudes, determ = dx*dy/4; writes every level of
 * the state Y (cos-weighted moments, then the row's inverse mass). */
int dgswe_project(dgswe_ctx *ctx, const double *fvals, const double *cos_nodes, double determ, double *Y,
                  void *stream);

/* Kernel launches issued by this context since creation (instrumentation). */
int64_t dgswe_launch_count(const dgswe_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGSWE_B200_H */
