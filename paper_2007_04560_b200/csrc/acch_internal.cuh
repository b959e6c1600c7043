// Internal declarations shared by the libacch_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/acch_b200.h"

#define ACCH_MAX_ORDER 32

// ---------------------------------------------------------------------------
// Device-side descriptors (passed by value to kernels)
// ---------------------------------------------------------------------------

struct GridDev {
    int dim;
    int periodic;
    int nx, ny, nz;          // nz == 1 in 2D; in slab mode the local interior planes
    long long n;             // interior cells of this domain
    double ih2[3];           // 1 / h^2 per axis (x, y, z)
    double ih[3];            // 1 / h per axis
    double cell_volume;
    // z-slab decomposition (multi-GPU).  zg == 0: the whole grid, z wraps or
    // clamps like x and y.  zg > 0: vectors store zg ghost planes below and
    // above the nz interior planes (refreshed by the halo hook); z never wraps
    // locally and only the physical Neumann walls (zwall_lo/hi) clamp.
    int zg;
    int zwall_lo, zwall_hi;
    long long zoff;          // zg * nx * ny: first interior cell in storage
    long long nstore;        // (nz + 2 zg) * nx * ny stored cells
    // device-resident GMRES: the Arnoldi-step kernels (matvec, Schwarz apply)
    // return at once while *skip != 0 (the cycle ended on the device and the
    // host had already queued the next steps); NULL outside GMRES
    const int *skip;
};

#ifdef __CUDACC__
#define ACCH_SKIP_IF(g)                                   \
    do {                                                  \
        if ((g).skip != nullptr && __ldcg((g).skip)) return; \
    } while (0)
#endif

struct ParamsDev {
    double alpha, beta, gamma, theta, rho;
    int order;
    double c1[ACCH_MAX_ORDER];   // 1 / ((2s+1) 2s)   (physics.py:178-182)
    double c2[ACCH_MAX_ORDER];   // 1 / (2s+1)
};

// Coefficients of the matrix-free Jacobian: 7 doubles per stored cell in
// three cell-major arrays, so a stencil kernel fetches a cell's coefficients
// with one 32-byte and one 16-byte load:
//   A[c]  = (S, D, c_u, c_v)   double4 at coef + 4c
//   B[c]  = (cbar, G_u)        double2 at coef + 4N + 2c
//   Gv[c]                      double  at coef + 6N + c
enum { CO_S = 0, CO_D, CO_CBAR, CO_GU, CO_CU, CO_CV, CO_GV, CO_NFIELDS };
__host__ __device__ __forceinline__ long long co_index(int f, long long N, long long c)
{
    switch (f) {
    case CO_S: return 4 * c;
    case CO_D: return 4 * c + 1;
    case CO_CU: return 4 * c + 2;
    case CO_CV: return 4 * c + 3;
    case CO_CBAR: return 4 * N + 2 * c;
    case CO_GU: return 4 * N + 2 * c + 1;
    default: return 6 * N + c;
    }
}
#ifdef __CUDACC__
// one 256-bit read-only load (LDG.E.256 on sm_100); not volatile, so the
// compiler may schedule it like any other load
__device__ __forceinline__ double4 ldg256(const double4 *p)
{
    double4 v;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
#endif
__host__ __device__ __forceinline__ const double4 *co_A(const double *coef) { return reinterpret_cast<const double4 *>(coef); }
__host__ __device__ __forceinline__ const double2 *co_B(const double *coef, long long N) { return reinterpret_cast<const double2 *>(coef + 4 * N); }
__host__ __device__ __forceinline__ const double *co_Gv(const double *coef, long long N) { return coef + 6 * N; }

// ---------------------------------------------------------------------------
// Host-side context
// ---------------------------------------------------------------------------

// kernel categories for the optional CUDA-event profile (acch_profile_*)
enum ProfCat {
    PC_RESIDUAL = 0, PC_JPREP, PC_MATVEC, PC_FACTOR, PC_APPLY, PC_GATHER, PC_KDOT, PC_KUPDATE, PC_KVEC,
    PC_REDUCE, PC_COUNT
};

struct ProfState {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<int> cat;
    std::vector<cudaEvent_t> ev0, ev1;
    std::vector<double> nbytes;
    double ms[PC_COUNT] = {0};
    long long cnt[PC_COUNT] = {0};
    double bytes[PC_COUNT] = {0};
};

struct acch_ctx;
typedef int (*acch_allreduce_cb)(void *user, double *values, int n, int op);
typedef int (*acch_halo_cb)(void *user, double *vec, long long plane_doubles, int nz, int zg, int depth);

struct acch_ctx {
    GridDev g;
    ParamsDev p;
    acch_grid_desc desc;
    int device = 0;
    cudaStream_t stream = 0;
    // reduction scratch: per-block partials + a completion counter + results
    double *d_partials = nullptr;     // [kRedBlocks * kRedSlots]
    unsigned int *d_counter = nullptr;
    double *d_result = nullptr;       // [kRedSlots]
    double *h_result = nullptr;       // pinned mirror
    // Krylov workspace (lazily sized)
    double *d_krylov = nullptr;       // (restart + 1) * 2N
    int krylov_cols = 0;
    double *d_work = nullptr;         // 3 * 2N: z (precond out), r, t
    double *d_zbasis = nullptr;       // lagged CGS2 with a preconditioner: M^-1 u_j per step (restart columns)
    int zbasis_cols = 0;
    double *d_h = nullptr;            // small device array for Hessenberg column
    void *d_gm = nullptr;             // device-resident GMRES cycle state (krylov.cu GmState)
    int *h_gm_status = nullptr;       // per-Arnoldi-step status, mapped pinned host memory
    int *d_gm_status = nullptr;       // its device alias
    double *d_mvtmp = nullptr;        // two-pass matvec intermediate (dG_u, eta), 2 * nstore
    int matvec_mode = 2;              // 2 z-marching one-barrier kernel (3D default), 1 two-pass (2D), 0 older fused kernel
    long long launches = 0;
    ProfState prof;
    // slab decomposition: rank topology and the host hooks that move ghost
    // planes and combine per-rank partial reductions (acch_set_comm)
    int nranks = 1, rank = 0;
    int z_offset = 0, nz_global = 0;     // slab position in the global grid
    acch_allreduce_cb allreduce = nullptr;
    acch_halo_cb halo = nullptr;
    void *comm_user = nullptr;
    // in-library NCCL data plane (comm.cu, acch_set_nccl): replaces the hooks
    void *nccl_comm = nullptr;
    double *d_comm = nullptr;         // 64-double staging buffer for host-value allreduces
    double comm_bytes = 0.0;          // halo bytes sent (statistics)
    long long comm_calls = 0;
};

// multi-rank helpers (capi.cu): no-ops for a single domain
acch_status comm_allreduce(acch_ctx *ctx, double *vals, int n, int op);
acch_status comm_halo(acch_ctx *ctx, const double *vec, int doubles_per_cell, int depth);
// NCCL data plane (comm.cu)
bool comm_has_nccl(const acch_ctx *ctx);
acch_status nccl_halo(acch_ctx *ctx, double *vec, long long plane, int depth);
acch_status comm_allreduce_dev(acch_ctx *ctx, double *dev, int n, int op);   // in place on ctx->stream
acch_status nccl_allreduce_host(acch_ctx *ctx, double *vals, int n, int op);
void comm_release(acch_ctx *ctx);

// Records a CUDA event pair around the launches in its scope when profiling is on.
struct ProfScope {
    acch_ctx *ctx;
    int cat;
    double bytes;
    cudaEvent_t e1 = nullptr;
    // bytes: algorithmic DRAM bytes the launches in scope must move
    ProfScope(acch_ctx *c, int category, double alg_bytes);
    ~ProfScope();
};

constexpr int kRedBlocks = 296;   // 2 x 148 SMs; fixed -> deterministic reductions
constexpr int kRedSlots = 40;     // up to 40 simultaneous sums per reduction pass
constexpr int kRedThreads = 256;

// error helpers -------------------------------------------------------------
void acch_set_error(const std::string &msg);
acch_status acch_cuda_fail(cudaError_t e, const char *where);

#define ACCH_CUDA(call)                                                  \
    do {                                                                 \
        cudaError_t _e = (call);                                         \
        if (_e != cudaSuccess) return acch_cuda_fail(_e, #call);         \
    } while (0)

#define ACCH_LAUNCHED(ctx)                                               \
    do {                                                                 \
        (ctx)->launches++;                                               \
        cudaError_t _e = cudaGetLastError();                             \
        if (_e != cudaSuccess) return acch_cuda_fail(_e, "kernel launch"); \
    } while (0)

// results of a reduction pass are read back through the pinned mirror
acch_status acch_fetch_results(acch_ctx *ctx, int count);

// ---------------------------------------------------------------------------
// Launchers implemented in stencil.cu / krylov.cu (return acch_status)
// ---------------------------------------------------------------------------

acch_status launch_residual(acch_ctx *ctx, const double *x_old, double dt, const double *x,
                            double *F);   // results: [0] = ||F||^2, [1] = gap
acch_status launch_jacobian_prepare(acch_ctx *ctx, const double *x_old, double dt,
                                    const double *x, double *coef);
acch_status launch_matvec(acch_ctx *ctx, const double *coef, double dt, const double *w,
                          double *y);
acch_status launch_jacobian_blocks(acch_ctx *ctx, const double *coef, double dt, double *out);

// multi-dot: results[q] = <V_q, w> (q < m), results[m] = <w, w>; V_q = V + q * ld
acch_status launch_mdot(acch_ctx *ctx, const double *V, long long ld, int m, const double *w,
                        long long n);
// w -= sum_q h[q] V_q (h on device); results[0] = <w, w>
acch_status launch_mupdate(acch_ctx *ctx, const double *V, long long ld, int m, const double *h,
                           double *w, long long n);
// y = alpha_dev[0] * x   (alpha read on device; inv == 1 -> 1 / alpha)
acch_status launch_scale(acch_ctx *ctx, const double *alpha_dev, int inv, const double *x,
                         double *y, long long n);
// t = sum_q y[q] V_q (y on device)
acch_status launch_combine(acch_ctx *ctx, const double *V, long long ld, int m, const double *y,
                           double *t, long long n);
// y = a * x + b * y (host scalars)
acch_status launch_axpby(acch_ctx *ctx, double a, const double *x, double b, double *y, long long n);
// generic reductions: [0] = <a, b>
acch_status launch_dot(acch_ctx *ctx, const double *a, const double *b, long long n);

// Schwarz (schwarz.cu)
acch_status precond_apply_impl(acch_precond *pc, const double *r, double *z);

// stencil offsets (x, y, z) with |dx|+|dy|+|dz| <= 2, fixed order
int stencil_offsets(int dim, int (*off)[3]);
