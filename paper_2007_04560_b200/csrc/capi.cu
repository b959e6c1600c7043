// C ABI entry points of libacch_b200.so (include/acch_b200.h).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include "acch_internal.cuh"

static thread_local std::string g_last_error;

void acch_set_error(const std::string &msg) { g_last_error = msg; }

acch_status acch_cuda_fail(cudaError_t e, const char *where)
{
    g_last_error = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return ACCH_ERR_CUDA;
}

static cudaEvent_t prof_event(acch_ctx *ctx)
{
    auto &p = ctx->prof;
    if (!p.pool.empty()) {
        cudaEvent_t e = p.pool.back();
        p.pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(acch_ctx *c, int category, double alg_bytes) : ctx(c), cat(category), bytes(alg_bytes)
{
    if (!ctx->prof.on) return;
    cudaEvent_t e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, ctx->stream);
    ctx->prof.ev0.push_back(e0);
}

ProfScope::~ProfScope()
{
    if (!e1) return;
    cudaEventRecord(e1, ctx->stream);
    ctx->prof.ev1.push_back(e1);
    ctx->prof.cat.push_back(cat);
    ctx->prof.nbytes.push_back(bytes);
}

acch_status acch_fetch_results(acch_ctx *ctx, int count)
{
    ACCH_CUDA(cudaMemcpyAsync(ctx->h_result, ctx->d_result, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    ACCH_CUDA(cudaStreamSynchronize(ctx->stream));
    return ACCH_OK;
}

acch_status comm_allreduce(acch_ctx *ctx, double *vals, int n, int op)
{
    if (ctx->nranks <= 1 || n <= 0) return ACCH_OK;
    if (ctx->nccl_comm) return nccl_allreduce_host(ctx, vals, n, op);
    if (!ctx->allreduce) return ACCH_OK;
    if (ctx->allreduce(ctx->comm_user, vals, n, op) != 0) {
        g_last_error = "allreduce hook failed";
        return ACCH_ERR_CUDA;
    }
    return ACCH_OK;
}

acch_status comm_halo(acch_ctx *ctx, const double *vec, int doubles_per_cell, int depth)
{
    if (ctx->g.zg == 0) return ACCH_OK;
    const long long plane = (long long)doubles_per_cell * ctx->g.nx * ctx->g.ny;
    if (ctx->nccl_comm) return nccl_halo(ctx, const_cast<double *>(vec), plane, depth);   // stream-ordered
    if (!ctx->halo) return ACCH_OK;
    ACCH_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->halo(ctx->comm_user, const_cast<double *>(vec), plane, ctx->g.nz, ctx->g.zg, depth) != 0) {
        g_last_error = "halo hook failed";
        return ACCH_ERR_CUDA;
    }
    return ACCH_OK;
}

// gap reductions: NaN (inadmissible) -> -inf before the cross-rank min
static double gap_value(double g) { return isnan(g) ? -INFINITY : g; }

// launchers defined in stencil.cu without a shared header entry
acch_status launch_chord(acch_ctx *ctx, const double *a, const double *b, long long n, int force_exact, double *val,
                         double *der);
acch_status launch_gap(acch_ctx *ctx, const double *x);
acch_status launch_gap_pairs(acch_ctx *ctx, const double *x, long long n);
acch_status launch_diagnostics(acch_ctx *ctx, const double *x);
acch_status launch_trial(acch_ctx *ctx, const double *x, const double *s, double lam, double *y);
acch_status launch_feasible_cap(acch_ctx *ctx, const double *x, const double *s, double margin);
acch_status launch_rms_diff(acch_ctx *ctx, const double *a, const double *b, long long n);
acch_status gmres_impl(acch_ctx *ctx, const double *coef, double dt, acch_precond *pc, const double *b, double *x,
                       int x0_given,
                       double rel_tol, double abs_tol, int restart, int max_it, int ortho, int *iterations,
                       int *converged, double *residual_norm);

#define CHECK_CTX(ctx)                                              \
    do {                                                            \
        if (!(ctx)) {                                               \
            acch_set_error("null context");                         \
            return ACCH_ERR_INVALID_ARG;                            \
        }                                                           \
        cudaError_t _e = cudaSetDevice((ctx)->device);              \
        if (_e != cudaSuccess) return acch_cuda_fail(_e, "cudaSetDevice"); \
    } while (0)

#define TRY(x)                        \
    do {                              \
        acch_status _s = (x);         \
        if (_s != ACCH_OK) return _s; \
    } while (0)

static constexpr double kMargin = 1e-12;   // ADMISSIBILITY_MARGIN, physics.py:26

extern "C" {

const char *acch_last_error(void) { return g_last_error.c_str(); }

int32_t acch_abi_version(void) { return 1; }

acch_status acch_ctx_create(const acch_grid_desc *grid, const acch_params *params, int32_t device, acch_ctx **out)
{
    if (!grid || !params || !out) {
        acch_set_error("acch_ctx_create: null argument");
        return ACCH_ERR_INVALID_ARG;
    }
    if (grid->dim != 2 && grid->dim != 3) {
        acch_set_error("grid must be 2D or 3D");
        return ACCH_ERR_INVALID_ARG;
    }
    for (int a = 0; a < grid->dim; ++a) {
        if (grid->counts[a] < 4 || grid->counts[a] > (1 << 20)) {
            acch_set_error("need at least 4 cells per axis");
            return ACCH_ERR_INVALID_ARG;
        }
        if (!(grid->lengths[a] > 0.0)) {
            acch_set_error("box extents must be positive");
            return ACCH_ERR_INVALID_ARG;
        }
    }
    if (!(params->alpha > 0 && params->beta > 0 && params->gamma > 0 && params->theta > 0 && params->rho > 0) ||
        params->series_order < 1 || params->series_order > ACCH_MAX_ORDER) {
        acch_set_error("invalid physical parameters");
        return ACCH_ERR_INVALID_ARG;
    }
    ACCH_CUDA(cudaSetDevice(device));
    auto *ctx = new acch_ctx();
    ctx->device = device;
    ctx->desc = *grid;
    GridDev &g = ctx->g;
    g.dim = grid->dim;
    g.periodic = grid->periodic ? 1 : 0;
    g.nx = (int)grid->counts[0];
    g.ny = (int)grid->counts[1];
    g.nz = grid->dim == 3 ? (int)grid->counts[2] : 1;
    g.n = (long long)g.nx * g.ny * g.nz;
    double vol = 1.0;
    for (int a = 0; a < 3; ++a) {
        if (a < grid->dim) {
            const double h = grid->lengths[a] / (double)grid->counts[a];
            g.ih2[a] = 1.0 / (h * h);
            g.ih[a] = 1.0 / h;
            vol *= h;
        } else {
            g.ih2[a] = 0.0;
            g.ih[a] = 0.0;
        }
    }
    g.cell_volume = vol;
    g.zg = 0;
    g.zwall_lo = g.zwall_hi = g.periodic ? 0 : 1;
    g.zoff = 0;
    g.nstore = g.n;
    g.skip = nullptr;
    ParamsDev &p = ctx->p;
    p.alpha = params->alpha;
    p.beta = params->beta;
    p.gamma = params->gamma;
    p.theta = params->theta;
    p.rho = params->rho;
    p.order = params->series_order;
    for (int s = 1; s <= ACCH_MAX_ORDER; ++s) {
        const double sd = (double)s;
        p.c1[s - 1] = 1.0 / ((2.0 * sd + 1.0) * 2.0 * sd);   // physics.py:178-182
        p.c2[s - 1] = 1.0 / (2.0 * sd + 1.0);
    }
    const size_t partial_cap = (size_t)1 << 21;
    cudaError_t e;
    if ((e = cudaMalloc(&ctx->d_partials, sizeof(double) * partial_cap)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_counter, 16 * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMemset(ctx->d_counter, 0, 16 * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_result, sizeof(double) * 64)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_h, sizeof(double) * 256)) != cudaSuccess ||
        (e = cudaMallocHost(&ctx->h_result, sizeof(double) * 128)) != cudaSuccess) {
        acch_ctx_destroy(ctx);
        return acch_cuda_fail(e, "acch_ctx_create allocation");
    }
    ctx->matvec_mode = ctx->g.dim == 3 ? 2 : 1;   // re-read per call (launch_matvec)
    *out = ctx;
    return ACCH_OK;
}

acch_status acch_ctx_destroy(acch_ctx *ctx)
{
    if (!ctx) return ACCH_OK;
    cudaSetDevice(ctx->device);
    comm_release(ctx);
    cudaFree(ctx->d_partials);
    cudaFree(ctx->d_counter);
    cudaFree(ctx->d_result);
    cudaFree(ctx->d_h);
    cudaFree(ctx->d_krylov);
    cudaFree(ctx->d_work);
    cudaFree(ctx->d_zbasis);
    cudaFree(ctx->d_mvtmp);
    cudaFree(ctx->d_gm);
    if (ctx->h_gm_status) cudaFreeHost(ctx->h_gm_status);
    if (ctx->h_result) cudaFreeHost(ctx->h_result);
    delete ctx;
    return ACCH_OK;
}

acch_status acch_set_stream(acch_ctx *ctx, void *cuda_stream)
{
    CHECK_CTX(ctx);
    ctx->stream = (cudaStream_t)cuda_stream;
    return ACCH_OK;
}

int64_t acch_launch_count(acch_ctx *ctx) { return ctx ? ctx->launches : 0; }

acch_status acch_ctx_set_slab(acch_ctx *ctx, const acch_slab_desc *slab)
{
    CHECK_CTX(ctx);
    if (!slab || slab->nranks < 1 || slab->rank < 0 || slab->rank >= slab->nranks || slab->ghost_planes < 0 ||
        slab->ghost_planes > 2 || ctx->g.dim != 3 || ctx->d_krylov) {
        acch_set_error("acch_ctx_set_slab: invalid slab (3D only, 0..2 ghost planes, before any GMRES call)");
        return ACCH_ERR_INVALID_ARG;
    }
    GridDev &g = ctx->g;
    ctx->nranks = slab->nranks;
    ctx->rank = slab->rank;
    ctx->z_offset = slab->z_offset;
    ctx->nz_global = slab->nz_global > 0 ? slab->nz_global : g.nz;
    g.zg = slab->ghost_planes;
    if (g.zg == 0) {
        g.zwall_lo = g.zwall_hi = g.periodic ? 0 : 1;
    } else {
        g.zwall_lo = slab->wall_lo ? 1 : 0;
        g.zwall_hi = slab->wall_hi ? 1 : 0;
    }
    g.zoff = (long long)g.zg * g.nx * g.ny;
    g.nstore = g.n + 2 * g.zoff;
    return ACCH_OK;
}

acch_status acch_set_comm(acch_ctx *ctx, acch_allreduce_fn allreduce, acch_halo_fn halo, void *user)
{
    CHECK_CTX(ctx);
    ctx->allreduce = (acch_allreduce_cb)allreduce;
    ctx->halo = (acch_halo_cb)halo;
    ctx->comm_user = user;
    return ACCH_OK;
}

int64_t acch_storage_cells(acch_ctx *ctx) { return ctx ? ctx->g.nstore : 0; }

acch_status acch_profile_enable(acch_ctx *ctx, int32_t on)
{
    CHECK_CTX(ctx);
    ctx->prof.on = on != 0;
    return ACCH_OK;
}

acch_status acch_profile_read(acch_ctx *ctx, double *ms, int64_t *counts, double *bytes, int32_t n)
{
    CHECK_CTX(ctx);
    ACCH_CUDA(cudaStreamSynchronize(ctx->stream));
    auto &p = ctx->prof;
    for (size_t i = 0; i < p.cat.size(); ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, p.ev0[i], p.ev1[i]);
        p.ms[p.cat[i]] += t;
        p.cnt[p.cat[i]] += 1;
        p.bytes[p.cat[i]] += p.nbytes[i];
        p.pool.push_back(p.ev0[i]);
        p.pool.push_back(p.ev1[i]);
    }
    p.cat.clear();
    p.nbytes.clear();
    p.ev0.clear();
    p.ev1.clear();
    for (int i = 0; i < n && i < PC_COUNT; ++i) {
        if (ms) ms[i] = p.ms[i];
        if (counts) counts[i] = p.cnt[i];
        if (bytes) bytes[i] = p.bytes[i];
        p.bytes[i] = 0.0;
        p.ms[i] = 0.0;
        p.cnt[i] = 0;
    }
    return ACCH_OK;
}

int32_t acch_stencil_offsets(int32_t dim, int32_t *offsets_xyz)
{
    int off[25][3];
    const int n = stencil_offsets(dim, off);
    if (offsets_xyz)
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) offsets_xyz[3 * i + a] = off[i][a];
    return n;
}

acch_status acch_entropy_chord(acch_ctx *ctx, const double *a, const double *b, int64_t n, int32_t force_exact,
                               double *val, double *der)
{
    CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!a || !b || !val))) {
        acch_set_error("acch_entropy_chord: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    return launch_chord(ctx, a, b, n, force_exact, val, der);
}

acch_status acch_admissibility_gap(acch_ctx *ctx, const double *x, double *gap)
{
    CHECK_CTX(ctx);
    TRY(launch_gap(ctx, x));
    TRY(acch_fetch_results(ctx, 1));
    double v = gap_value(ctx->h_result[0]);
    TRY(comm_allreduce(ctx, &v, 1, 1));
    if (gap) *gap = v;
    return ACCH_OK;
}

acch_status acch_gap_pairs(acch_ctx *ctx, const double *x, int64_t n, double *gap)
{
    CHECK_CTX(ctx);
    if (n < 1 || !x) {
        acch_set_error("acch_gap_pairs: need at least one (u, v) pair");
        return ACCH_ERR_INVALID_ARG;
    }
    TRY(launch_gap_pairs(ctx, x, n));
    TRY(acch_fetch_results(ctx, 1));
    if (gap) *gap = gap_value(ctx->h_result[0]);
    return ACCH_OK;
}

acch_status acch_diagnostics(acch_ctx *ctx, const double *x, double *energy, double *mass_u, double *max_abs_v)
{
    CHECK_CTX(ctx);
    TRY(comm_halo(ctx, x, 2, 1));
    TRY(launch_diagnostics(ctx, x));
    TRY(acch_fetch_results(ctx, 3));
    double sums[2] = {ctx->h_result[0], ctx->h_result[1]}, vmax = ctx->h_result[2];
    TRY(comm_allreduce(ctx, sums, 2, 0));
    TRY(comm_allreduce(ctx, &vmax, 1, 2));
    if (energy) *energy = sums[0] * ctx->g.cell_volume;
    if (mass_u) *mass_u = sums[1] * ctx->g.cell_volume;
    if (max_abs_v) *max_abs_v = vmax;
    return ACCH_OK;
}

acch_status acch_residual(acch_ctx *ctx, const double *x_old, double dt, const double *x, double *F, double *gap,
                          double *norm2)
{
    CHECK_CTX(ctx);
    if (!x_old || !x || !F || !(dt > 0.0)) {
        acch_set_error("acch_residual: invalid argument (time step must be positive)");
        return ACCH_ERR_INVALID_ARG;
    }
    TRY(comm_halo(ctx, x_old, 2, 2));
    TRY(comm_halo(ctx, x, 2, 2));
    TRY(launch_residual(ctx, x_old, dt, x, F));
    if (!gap && !norm2) return ACCH_OK;   // asynchronous form: no readback, no admissibility check
    TRY(acch_fetch_results(ctx, 2));
    double nrm = ctx->h_result[0], gp = gap_value(ctx->h_result[1]);
    TRY(comm_allreduce(ctx, &nrm, 1, 0));
    TRY(comm_allreduce(ctx, &gp, 1, 1));
    if (gap) *gap = gp;
    if (norm2) *norm2 = nrm;
    if (!(gp >= kMargin)) {
        char buf[160];
        snprintf(buf, sizeof buf, "state violates admissibility bounds (gap %.3e < margin %.1e)", gp, kMargin);
        acch_set_error(buf);
        return ACCH_ERR_INADMISSIBLE;
    }
    return ACCH_OK;
}

acch_status acch_jacobian_prepare(acch_ctx *ctx, const double *x_old, double dt, const double *x, double *coef)
{
    CHECK_CTX(ctx);
    if (!x_old || !x || !coef || !(dt > 0.0)) {
        acch_set_error("acch_jacobian_prepare: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    TRY(comm_halo(ctx, x_old, 2, 1));
    TRY(comm_halo(ctx, x, 2, 1));
    TRY(launch_jacobian_prepare(ctx, x_old, dt, x, coef));
    // the factorisation reads coefficients one plane beyond an overlapping box
    TRY(comm_halo(ctx, coef, 4, 2));
    TRY(comm_halo(ctx, coef + 4 * ctx->g.nstore, 2, 2));
    TRY(comm_halo(ctx, coef + 6 * ctx->g.nstore, 1, 2));
    return ACCH_OK;
}

acch_status acch_jacobian_matvec(acch_ctx *ctx, const double *coef, double dt, const double *w, double *y)
{
    CHECK_CTX(ctx);
    if (!coef || !w || !y || !(dt > 0.0)) {
        acch_set_error("acch_jacobian_matvec: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    TRY(comm_halo(ctx, w, 2, 2));
    return launch_matvec(ctx, coef, dt, w, y);
}

acch_status acch_jacobian_blocks(acch_ctx *ctx, const double *coef, double dt, double *out)
{
    CHECK_CTX(ctx);
    if (!coef || !out || !(dt > 0.0)) {
        acch_set_error("acch_jacobian_blocks: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    return launch_jacobian_blocks(ctx, coef, dt, out);
}

acch_status acch_dot(acch_ctx *ctx, const double *a, const double *b, int64_t n, double *out)
{
    CHECK_CTX(ctx);
    // a whole-storage state vector in slab mode: reduce over this rank's interior
    if (ctx->g.zg && n == 2 * ctx->g.nstore) {
        a += 2 * ctx->g.zoff;
        b += 2 * ctx->g.zoff;
        n = 2 * ctx->g.n;
    }
    TRY(launch_dot(ctx, a, b, n));
    TRY(acch_fetch_results(ctx, 1));
    double v = ctx->h_result[0];
    TRY(comm_allreduce(ctx, &v, 1, 0));
    if (out) *out = v;
    return ACCH_OK;
}

acch_status acch_axpby(acch_ctx *ctx, double a, const double *x, double b, double *y, int64_t n)
{
    CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!x || !y))) {
        acch_set_error("acch_axpby: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    if (n == 0) return ACCH_OK;
    return launch_axpby(ctx, a, x, b, y, n);
}

acch_status acch_rms_diff(acch_ctx *ctx, const double *a, const double *b, int64_t n, double *out)
{
    CHECK_CTX(ctx);
    if (n <= 0) {
        acch_set_error("acch_rms_diff: empty vector");
        return ACCH_ERR_INVALID_ARG;
    }
    if (ctx->g.zg && n == 2 * ctx->g.nstore) {
        a += 2 * ctx->g.zoff;
        b += 2 * ctx->g.zoff;
        n = 2 * ctx->g.n;
    }
    TRY(launch_rms_diff(ctx, a, b, n));
    TRY(acch_fetch_results(ctx, 1));
    double v[2] = {ctx->h_result[0], (double)n};
    TRY(comm_allreduce(ctx, v, 2, 0));
    if (out) *out = sqrt(v[0] / v[1]);
    return ACCH_OK;
}

acch_status acch_trial(acch_ctx *ctx, const double *x, const double *s, double lam, double *y, double *gap)
{
    CHECK_CTX(ctx);
    TRY(launch_trial(ctx, x, s, lam, y));
    TRY(acch_fetch_results(ctx, 1));
    double v = gap_value(ctx->h_result[0]);
    TRY(comm_allreduce(ctx, &v, 1, 1));
    if (gap) *gap = v;
    return ACCH_OK;
}

acch_status acch_feasible_cap(acch_ctx *ctx, const double *x, const double *s, double margin, double fraction,
                              double *cap)
{
    CHECK_CTX(ctx);
    TRY(launch_feasible_cap(ctx, x, s, margin));
    TRY(acch_fetch_results(ctx, 1));
    double c = ctx->h_result[0];
    if (isnan(c)) c = INFINITY;
    TRY(comm_allreduce(ctx, &c, 1, 1));
    double out;
    if (!isfinite(c)) out = 1.0;   // newton.py:97-98 (no bound is active, or NaN)
    else out = fmin(1.0, fraction * c);
    if (cap) *cap = out;
    return ACCH_OK;
}

acch_status acch_gmres(acch_ctx *ctx, const double *coef, double dt, acch_precond *pc, const double *b, double *x,
                       double rel_tol, double abs_tol, int32_t restart, int32_t max_iterations, int32_t ortho,
                       int32_t *iterations, int32_t *converged, double *residual_norm)
{
    return acch_gmres_x0(ctx, coef, dt, pc, b, x, 0, rel_tol, abs_tol, restart, max_iterations, ortho, iterations,
                         converged, residual_norm);
}

acch_status acch_gmres_x0(acch_ctx *ctx, const double *coef, double dt, acch_precond *pc, const double *b, double *x,
                          int32_t x0_given, double rel_tol, double abs_tol, int32_t restart, int32_t max_iterations,
                          int32_t ortho, int32_t *iterations, int32_t *converged, double *residual_norm)
{
    CHECK_CTX(ctx);
    if (!coef || !b || !x || !(dt > 0.0) || max_iterations < 0 || ortho < 0 || ortho > 2) {
        acch_set_error("acch_gmres: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    int its = 0, conv = 0;
    double rn = 0.0;
    acch_status st = gmres_impl(ctx, coef, dt, pc, b, x, x0_given != 0, rel_tol, abs_tol, restart, max_iterations,
                                ortho, &its, &conv, &rn);
    if (iterations) *iterations = its;
    if (converged) *converged = conv;
    if (residual_norm) *residual_norm = rn;
    return st;
}

}  // extern "C"
