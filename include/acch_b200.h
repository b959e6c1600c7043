/*
 * acch_b200.h -- C ABI of libacch_b200.so, the B200 (sm_100a) implementation
 * of the per-time-step Newton-Krylov-Schwarz solve of the reference package
 * `acch` (arXiv 2007.04560).  Every entry point names the reference interface
 * it replaces (paths relative to /root/reference/pkg/src/acch/).
 *
 * Conventions
 *  - All vectors are DEVICE pointers to fp64, owned by the caller (PyTorch in
 *    the Python host layer).  Solver vectors use the reference layout: (u, v)
 *    interleaved per cell, cells x-fastest, length 2N (scheme.py:58-80).
 *  - Work is enqueued on the stream set with acch_set_stream (default: the
 *    legacy default stream).  Calls that return scalars synchronise that
 *    stream; all others are asynchronous.
 *  - Nothing throws across the ABI.  Every call returns an acch_status; the
 *    message of the last failure on the calling thread is acch_last_error().
 *  - No call retains a caller pointer past its return.  Library-owned device
 *    memory (reduction scratch, Krylov basis, subdomain factors) belongs to
 *    the context / preconditioner handle and is freed by its destroy call.
 */
#ifndef ACCH_B200_H
#define ACCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ACCH_OK = 0,
    ACCH_ERR_INVALID_ARG = 1,   /* ValueError in the reference               */
    ACCH_ERR_INADMISSIBLE = 2,  /* InadmissibleStateError (physics.py:116-121) */
    ACCH_ERR_ZERO_PIVOT = 3,    /* ZeroPivotError(cell, component) (linalg.py:306-311) */
    ACCH_ERR_CUDA = 4,          /* CUDA runtime failure (message has cudaGetErrorString) */
    ACCH_ERR_NO_FACTOR = 5,     /* RuntimeError: apply before update (linalg.py:375-376) */
    ACCH_ERR_PARTITION = 6      /* PartitionError (linalg.py:161-180) */
} acch_status;

/* Grid (grid.py:29-60): dim 2 or 3, counts (Nx, Ny[, Nz]) >= 4, box extents. */
typedef struct {
    int32_t dim;
    int32_t periodic;           /* 1: BoundaryCondition.PERIODIC, 0: NEUMANN */
    int64_t counts[3];
    double lengths[3];
} acch_grid_desc;

/* Params (physics.py:35-58). */
typedef struct {
    double alpha, beta, gamma, theta, rho;
    int32_t series_order;       /* 1..32 */
} acch_params;

typedef struct acch_ctx acch_ctx;          /* grid + params + stream + scratch */
typedef struct acch_precond acch_precond;  /* SchwarzPreconditioner state     */

const char *acch_last_error(void);
int32_t acch_abi_version(void);

/* Context.  Replaces the lru-cached grid operators (scheme.py:166-188). */
acch_status acch_ctx_create(const acch_grid_desc *grid, const acch_params *params,
                            int32_t device, acch_ctx **out);
acch_status acch_ctx_destroy(acch_ctx *ctx);
acch_status acch_set_stream(acch_ctx *ctx, void *cuda_stream);

/* ---- physics (physics.py) ---------------------------------------------- */

/* entropy_chord / entropy_chord_with_deriv elementwise over n pairs
 * (physics.py:213-310).  der may be NULL.  force_exact as in the reference. */
acch_status acch_entropy_chord(acch_ctx *ctx, const double *a, const double *b, int64_t n,
                               int32_t force_exact, double *val, double *der);

/* admissibility_gap (physics.py:89-109) of the interleaved state x. */
acch_status acch_admissibility_gap(acch_ctx *ctx, const double *x, double *gap);

/* admissibility_gap(u, v) (physics.py:89-109) over n interleaved (u, v)
 * pairs of any origin (not tied to the context's grid; no halo, no
 * cross-rank reduction).  NaN anywhere gives -inf, as the reference. */
acch_status acch_gap_pairs(acch_ctx *ctx, const double *x, int64_t n, double *gap);

/* total_energy, integrate(u), max|v| of a history row (physics.py:325-331,
 * grid.py:301-303, cli/drivers.py:62-73).  Any output pointer may be NULL. */
acch_status acch_diagnostics(acch_ctx *ctx, const double *x, double *energy,
                             double *mass_u, double *max_abs_v);

/* ---- scheme (scheme.py) ------------------------------------------------- */

/* residual_vector(StepProblem(old=x_old, dt), new=x) (scheme.py:343-354).
 * Writes F (2N).  Returns ACCH_ERR_INADMISSIBLE (F undefined) when the
 * admissibility gap of x is below 1e-12 (check_admissible, scheme.py:250).
 * gap and norm2 (= ||F||_2^2, deterministic) may be NULL; when both are NULL
 * the call is asynchronous and skips the admissibility check (raw launch). */
acch_status acch_residual(acch_ctx *ctx, const double *x_old, double dt, const double *x,
                          double *F, double *gap, double *norm2);

/* assemble_jacobian (scheme.py:427-484), matrix-free form: evaluates the 7
 * per-cell coefficients that define J at x into a caller-owned buffer of 7N
 * doubles (N = stored cells), laid out as N records (S, D, c_u, c_v), then N
 * records (cbar, G_u), then N values G_v.  Only this library reads it. */
acch_status acch_jacobian_prepare(acch_ctx *ctx, const double *x_old, double dt,
                                  const double *x, double *coef);

/* StencilMatrix.matvec (linalg.py:67-68): y = J w. */
acch_status acch_jacobian_matvec(acch_ctx *ctx, const double *coef, double dt,
                                 const double *w, double *y);

/* Explicit blocks of J on the radius-2 stencil: out[N][n_offsets][2][2] with
 * the offsets of acch_stencil_offsets (13 in 2D, 25 in 3D).  Offsets that
 * leave a Neumann box hold zeros.  (The reference BSR skeleton, scheme.py:166-188.) */
acch_status acch_jacobian_blocks(acch_ctx *ctx, const double *coef, double dt, double *out);
int32_t acch_stencil_offsets(int32_t dim, int32_t *offsets_xyz /* [n][3] or NULL */);

/* ---- linalg (linalg.py) ------------------------------------------------- */

/* Deterministic reductions over device vectors. */
acch_status acch_dot(acch_ctx *ctx, const double *a, const double *b, int64_t n, double *out);
/* out = sqrt(mean((a-b)^2)) (StepController.predict_dt, timestep.py:59-60). */
acch_status acch_rms_diff(acch_ctx *ctx, const double *a, const double *b, int64_t n, double *out);
/* y = a * x + b * y elementwise over n doubles. */
acch_status acch_axpby(acch_ctx *ctx, double a, const double *x, double b, double *y, int64_t n);
/* y = x + lam * s (trial_state, scheme.py:487-498); returns the gap of y. */
acch_status acch_trial(acch_ctx *ctx, const double *x, const double *s, double lam,
                       double *y, double *gap);
/* _feasible_step_cap (newton.py:75-99). */
acch_status acch_feasible_cap(acch_ctx *ctx, const double *x, const double *s, double margin,
                              double fraction, double *cap);

/* SchwarzPreconditioner(partition(grid, n_sub, overlap), variant, subsolver)
 * (linalg.py:320-347).  owned_lo/owned_hi: [n_sub][3] owned cell ranges per
 * axis (x, y, z), in the reference's box order (z slowest; linalg.py:195).
 * variant: 0 asm, 1 ras-left, 2 ras-right.  fill_level >= 0 -> ILU(k),
 * -1 -> exact LU of the subdomain matrix. */
acch_status acch_precond_create(acch_ctx *ctx, int64_t n_sub, int32_t overlap,
                                const int64_t *owned_lo, const int64_t *owned_hi,
                                int32_t variant, int32_t fill_level, acch_precond **out);
acch_status acch_precond_destroy(acch_precond *pc);
/* update(J, reuse) (linalg.py:353-372).  refactored = 1 when factors were
 * (re)computed.  On ACCH_ERR_ZERO_PIVOT, bad_cell/bad_comp name the first
 * zero pivot in subdomain order. */
acch_status acch_precond_update(acch_precond *pc, const double *coef, double dt, int32_t reuse,
                                int32_t *refactored, int64_t *bad_cell, int32_t *bad_comp);
acch_status acch_precond_invalidate(acch_precond *pc);
acch_status acch_precond_apply(acch_precond *pc, const double *r, double *z);
/* factorization_count, n subdomains, total factor bytes */
acch_status acch_precond_info(acch_precond *pc, int64_t *factorizations, int64_t *n_classes,
                              int64_t *factor_bytes);

/* gmres(J.matvec, b, precond, rel_tol, abs_tol, restart, max_iterations)
 * (linalg.py:411-506) with J given by (coef, dt) and pc optional (NULL =
 * identity).  x is overwritten with the solution (initial guess 0).
 * ortho: 0 = modified Gram-Schmidt exactly as the reference, 1 = classical
 * Gram-Schmidt with the reference's conditional second pass (fused passes),
 * 2 = classical Gram-Schmidt with the second pass lagged by one step (one
 * multi-dot and one fused update per step; the Python default). */
acch_status acch_gmres(acch_ctx *ctx, const double *coef, double dt, acch_precond *pc,
                       const double *b, double *x, double rel_tol, double abs_tol,
                       int32_t restart, int32_t max_iterations, int32_t ortho,
                       int32_t *iterations, int32_t *converged, double *residual_norm);

/* As acch_gmres with the reference's x0 argument (linalg.py:419, 434-439):
 * x0_given != 0 starts from the x passed in (r = b - J x), else from 0.
 * With ortho = 2 on one rank the Arnoldi loop is device-resident: Hessenberg
 * column, Givens rotations, the least-squares solve and the stopping test
 * run in kernels, and the host synchronises once per restart cycle. */
acch_status acch_gmres_x0(acch_ctx *ctx, const double *coef, double dt, acch_precond *pc,
                          const double *b, double *x, int32_t x0_given, double rel_tol,
                          double abs_tol, int32_t restart, int32_t max_iterations, int32_t ortho,
                          int32_t *iterations, int32_t *converged, double *residual_norm);

/* ---- z-slab decomposition (multi-GPU; one context per rank) ------------ */

/* A 3D context whose grid is this rank's slab of nz interior planes.  With
 * ghost_planes = 2 every state / solver / coefficient vector passed to the
 * library stores 2 ghost planes below and above the interior
 * ((nz + 4) * nx * ny cells, acch_storage_cells); calls refresh the ghost
 * planes of their inputs through the halo hook before reading them, and
 * every reduction (norms, dots, gaps, caps, energies) is combined across
 * ranks through the allreduce hook.  wall_lo / wall_hi mark the slabs that
 * touch a homogeneous Neumann wall.  Left-RAS only (no reverse scatter). */
typedef struct {
    int32_t nranks, rank;
    int32_t ghost_planes;       /* 0 (whole grid) or 2 */
    int32_t wall_lo, wall_hi;
    int32_t z_offset;           /* first global plane of this slab */
    int32_t nz_global;          /* global plane count (RAS boxes keep the
                                   reference's sorted-global-id cell order) */
} acch_slab_desc;

/* op: 0 sum, 1 min, 2 max over ranks, in place on n host doubles. */
typedef int32_t (*acch_allreduce_fn)(void *user, double *values, int32_t n, int32_t op);
/* Fill the `depth` ghost planes on each side of device vector `vec`
 * (plane = plane_doubles doubles; zg ghost planes, nz interior planes) from
 * the neighbouring ranks' interior planes (wrapping for periodic z).  The
 * library synchronises its stream before the call; the hook must complete
 * the exchange before returning. */
typedef int32_t (*acch_halo_fn)(void *user, double *vec, int64_t plane_doubles, int32_t nz, int32_t zg,
                                int32_t depth);

acch_status acch_ctx_set_slab(acch_ctx *ctx, const acch_slab_desc *slab);
acch_status acch_set_comm(acch_ctx *ctx, acch_allreduce_fn allreduce, acch_halo_fn halo, void *user);

/* ---- in-library NCCL data plane (replaces the host hooks) ---------------
 * Rank 0 calls acch_nccl_unique_id and shares the acch_nccl_id_bytes()
 * bytes with every rank (torch.distributed broadcast); every rank then calls
 * acch_set_nccl on its slab context (collective, blocks until all ranks
 * joined).  From then on ghost-plane exchanges are grouped ncclSend /
 * ncclRecv and every cross-rank reduction an ncclAllReduce, all enqueued on
 * the context's stream; the GMRES Arnoldi loop stays device-resident at
 * N > 1.  nccl_path: the libnccl to dlopen (NULL: "libnccl.so.2"). */
acch_status acch_nccl_unique_id(const char *nccl_path, void *id_out);
int32_t acch_nccl_id_bytes(void);
acch_status acch_set_nccl(acch_ctx *ctx, const char *nccl_path, const void *id, int32_t nranks, int32_t rank);
/* halo bytes sent and NCCL calls made by this context so far */
acch_status acch_comm_stats(acch_ctx *ctx, double *bytes, int64_t *calls);
int64_t acch_storage_cells(acch_ctx *ctx);

/* Count of kernels this library has launched on ctx since creation (for the
 * bench's gpu_launches field). */
int64_t acch_launch_count(acch_ctx *ctx);

/* Optional per-category CUDA-event kernel timing (bench / profiling only).
 * Categories, in order: residual, jacobian_prepare, matvec, precond_factor,
 * precond_apply, precond_gather, krylov_dot, krylov_update, krylov_vector,
 * state_reductions.  acch_profile_read synchronises, returns the milliseconds,
 * launch counts and algorithmic DRAM bytes (the bytes each kernel must move
 * at minimum) accumulated since the last read (n <= 10), and resets. */
acch_status acch_profile_enable(acch_ctx *ctx, int32_t on);
acch_status acch_profile_read(acch_ctx *ctx, double *ms, int64_t *counts, double *alg_bytes,
                              int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* ACCH_B200_H */
