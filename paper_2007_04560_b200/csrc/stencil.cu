// Fused fp64 stencil kernels of the implicit AC/CH step on sm_100a.
//
//   residual      F(U'; U^n)                       scheme.py:323-354
//   jac_prepare   7 coefficient planes of J(U')    scheme.py:427-470
//   matvec        y = J w, matrix-free             scheme.py:471-484, linalg.py:67-68
//   jac_blocks    explicit 2x2 stencil blocks of J (for ILU factorisation)
//
// Data layout: solver vectors are interleaved (u, v) per cell, x fastest,
// read as double2 (16 B per cell, fully coalesced).  No ghost cells are
// stored: periodic wrap / Neumann mirror are index arithmetic.
//
// The residual and matvec are radius-2 stencils by composition (a flux
// divergence of a Laplacian-containing field).  Both kernels tile the x-y
// plane (TX x TY threads, one output cell each) and march along z, keeping a
// 3-plane ring of the inputs (tile + 2 halo) and of the intermediate field
// (G_u, or dG_u; tile + 1 halo) in shared memory, so every input byte is read
// from HBM once per sweep and the expensive entropy chords are evaluated only
// on the tile + 1 halo.
#include <stdlib.h>
#include <string.h>

#include "acch_internal.cuh"
#include "physics.cuh"
#include "reduce.cuh"
#include "jacobian.cuh"

namespace {

constexpr int RTX = 32, RTY = 8;     // residual tile
constexpr int ZCHUNK = 32;           // z planes per block (3D)

__host__ __device__ constexpr int ring_depth(int dim) { return dim == 3 ? 3 : 1; }

// ---------------------------------------------------------------------------
// residual
// ---------------------------------------------------------------------------

template <int DIM, int TX, int TY>
struct ResidualSmem {
    static constexpr int HX = TX + 4, HY = TY + 4, GX = TX + 2, GY = TY + 2, R = ring_depth(DIM);
    static constexpr size_t xbytes = sizeof(double2) * R * HX * HY;
    static constexpr size_t gbytes = sizeof(double) * R * GX * GY;
    static constexpr size_t bytes = 2 * xbytes + 3 * gbytes;
};

// ring slot of plane k; k >= -3 everywhere (z chunks start at 0, at most 2 planes below)
__device__ __forceinline__ int mod3(int k) { return (int)((unsigned)(k + 3) % 3u); }

// cp.async (LDGSTS) 16-byte global -> shared copies, grouped per plane
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
// bulk L2 prefetch of [p, p + bytes) (16-byte granules)
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Chord for the residual's hot loop: same branch predicates as
// entropy_chord (physics.py:193-200, bitwise-identical choices), with the
// two logs of ln z - ln(1-z) merged into one log of z/(1-z), reciprocals
// shared between the log argument and the series ratios, and FMA Horner.
// Agrees with the reference formula to a few ulps of the O(1) terms.
// ORDER > 0: the series order as a compile-time constant (fully unrolled
// Horner on constant coefficients 1/((2s+1)2s), correctly rounded exactly as
// the host computes them); ORDER = 0: P.order at run time.
template <int ORDER>
__device__ __forceinline__ double chord_fast(double a, double b, const ParamsDev &P)
{
    const double zeta = 0.5 * (a + b);
    const double sigma = 0.5 * (a - b);
    const double w = 1.0 - zeta;
    if (sigma == 0.0) return log(zeta / w);
    if (fabs(sigma) <= 0.4 * fmin(zeta, w)) {
        const double r = 1.0 / (zeta * w);            // one reciprocal for 1/zeta and 1/w
        const double iz = w * r, iw = zeta * r;
        const double rz = sigma * iz, rw = sigma * iw;
        const double tz = rz * rz, tw = rw * rw;
        double pz, pw;
        if (ORDER > 0) {
            constexpr double cl = 1.0 / ((2.0 * ORDER + 1.0) * 2.0 * ORDER);
            pz = cl;
            pw = cl;
#pragma unroll
            for (int s = ORDER - 1; s >= 1; --s) {
                const double c = 1.0 / ((2.0 * s + 1.0) * 2.0 * s);
                pz = fma(pz, tz, c);
                pw = fma(pw, tw, c);
            }
        } else {
            pz = P.c1[P.order - 1];
            pw = P.c1[P.order - 1];
            for (int s = P.order - 2; s >= 0; --s) {
                pz = fma(pz, tz, P.c1[s]);
                pw = fma(pw, tw, P.c1[s]);
            }
        }
        return log(zeta * iw) - pz * tz + pw * tw;
    }
    return (entropy(a) - entropy(b)) / (a - b);
}

// ---------------------------------------------------------------------------
// Residual chord, warp-cooperative (res_zm_kernel).  Same branch predicates
// as entropy_chord (physics.py:193-200, 240-261).  Cost cuts:
//  * ln z - ln(1 - z) = 2 atanh(s) with s = 2 z - 1 (exact for z >= 1/4):
//    for |s| <= 0.2 an odd series in s with coefficients 1/(2k+1) from the
//    constant bank (no log call, no 64-bit immediates); libdevice log only
//    for |s| > 0.2;
//  * the chord's series P(t), t = (sigma/z)^2, is cut after 4 terms when no
//    lane of the warp has t > 6.3e-5 (the dropped tail is below 2^-60 of the
//    leading term, far under one rounding of the sum: the value is that of
//    the full series up to the last-bit rounding of its partial sums) --
//    always the case for Newton iterates near U^n -- else all S terms;
//  * one reciprocal 1/(z (1 - z)) for both ratios.
// All lanes of a warp must call it together.
// ---------------------------------------------------------------------------
__constant__ double c_atanh[12] = {1.0,        1.0 / 3.0,  1.0 / 5.0,  1.0 / 7.0,  1.0 / 9.0,  1.0 / 11.0,
                                   1.0 / 13.0, 1.0 / 15.0, 1.0 / 17.0, 1.0 / 19.0, 1.0 / 21.0, 1.0 / 23.0};

// q = sum_{k=1}^{K-1} x^{k-1} / (2k+1), Horner from the top (K compile-time)
template <int K>
__device__ __forceinline__ double atanh_tail(double x)
{
    // (Estrin's scheme -- depth 5 instead of 10 at 3 extra multiplications --
    // measured slower, 0.528 against 0.492 ms: the kernel is bound by FP64 /
    // issue throughput, not by the length of this chain)
    double q = c_atanh[K - 1];
#pragma unroll
    for (int k = K - 2; k >= 1; --k) q = fma(q, x, c_atanh[k]);
    return q;
}

// P(t)/t = sum_{s=1}^{K} t^{s-1} c1[s-1], Horner from the top
template <int K>
__device__ __forceinline__ void chord_poly2(double tz, double tw, const ParamsDev &P, double &pz, double &pw)
{
    pz = P.c1[K - 1];
    pw = P.c1[K - 1];
#pragma unroll
    for (int s = K - 2; s >= 0; --s) {
        pz = fma(pz, tz, P.c1[s]);
        pw = fma(pw, tw, P.c1[s]);
    }
}


// cell_gap with plain compare-selects (NaN in u or v -> NaN, then -inf in
// the caller's reduction, as physics.py:107-108)
__device__ __forceinline__ double cell_gap_fast(double u, double v)
{
    const double p = u + v, q = u - v;
    double g = u;
    const double c[7] = {1.0 - u, p, 1.0 - p, q, 1.0 - q, 0.5 - v, 0.5 + v};
#pragma unroll
    for (int k = 0; k < 7; ++k) g = c[k] < g ? c[k] : g;
    return (v != v) ? v : g;
}

// 1/x for 0 < x <= 1/4 (x = z (1 - z) of an admissible chord pair): the
// hardware reciprocal seed and three Newton steps, no special-case branch
// (the argument is never 0, denormal, inf or NaN on the path that uses it)
// STEPS = 2 leaves a relative error below 2^-36 even from a 9-bit seed: enough
// where the ratio enters only through t = (sigma/z)^2 <= 6.3e-5 (the short
// series: the term it scales is below 1.1e-5 of the chord)
template <int STEPS = 3>
__device__ __forceinline__ double rcp_quarter(double x)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int k = 0; k < STEPS; ++k) {
        const double e = fma(-x, y, 1.0);
        y = fma(y, e, y);
    }
    return y;
}
// one more Newton step on a reciprocal
__device__ __forceinline__ double rcp_refine(double x, double y) { return fma(y, fma(-x, y, 1.0), y); }

template <int ORDER>
__device__ __forceinline__ double chord_res(double a, double b, const ParamsDev &P)
{
    static_assert(ORDER == 10, "short series: the reference's default order");
    const double zeta = 0.5 * (a + b);
    const double sigma = 0.5 * (a - b);
    const double w = 1.0 - zeta;
    const double s = 2.0 * zeta - 1.0;
    const double s2 = s * s;
    // ln(zeta) - ln(1 - zeta) = 2 atanh(s): 12 terms for |s| <= 0.2025
    double lg;
    if (s2 <= 0.0410) lg = fma(2.0 * s * s2, atanh_tail<12>(s2), 2.0 * s);
    else lg = log(zeta) - log1p(-zeta);                 // far from 1/2: libdevice
    const bool exact = sigma == 0.0;                    // exact branch (physics.py:245-247): lg
    const double as = fabs(sigma);
    const bool near = !exact && as <= 0.4 * zeta && as <= 0.4 * w;   // 0.4 min(zeta, 1 - zeta)
    double val = lg;
    if (__any_sync(0xffffffffu, near)) {
        const double zw = zeta * w;
        double r = rcp_quarter<2>(zw);                  // 1/zeta = w r, 1/w = zeta r
        double rz = sigma * (w * r), rw = sigma * (zeta * r);
        double tz = rz * rz, tw = rw * rw;
        double pz, pw;
        // Newton iterates sit close to U^n: t = (sigma/z)^2 is tiny and 4
        // terms leave a tail below 2^-60 of the sum (t <= 6.3e-5); otherwise
        // the reciprocal gets its last Newton step and all S terms are summed
        if (!__any_sync(0xffffffffu, near && (tz > 6.3e-5 || tw > 6.3e-5))) {
            chord_poly2<4>(tz, tw, P, pz, pw);
        } else {
            r = rcp_refine(zw, r);
            rz = sigma * (w * r);
            rw = sigma * (zeta * r);
            tz = rz * rz;
            tw = rw * rw;
            chord_poly2<ORDER>(tz, tw, P, pz, pw);
        }
        if (near) val = lg - pz * tz + pw * tw;
    }
    if (!exact && !near) val = (entropy(a) - entropy(b)) / (a - b);   // direct quotient (physics.py:259-261)
    return val;
}

template <int DIM, int TX, int TY>
__global__ void __launch_bounds__(TX *TY)
residual_kernel(GridDev g, ParamsDev P, double dt, const double2 *__restrict__ xo_g,
                const double2 *__restrict__ xn_g, double2 *__restrict__ F, double *partials,
                unsigned int *counter, double *result)
{
    using L = ResidualSmem<DIM, TX, TY>;
    constexpr int HX = L::HX, HY = L::HY, GX = L::GX, GY = L::GY, R = L::R, NT = TX * TY;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sxn = reinterpret_cast<double2 *>(smem_raw);
    double2 *sxo = sxn + R * HX * HY;
    double *sGu = reinterpret_cast<double *>(sxo + R * HX * HY);
    double *sGv = sGu + R * GX * GY;
    double *sCb = sGv + R * GX * GY;

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    const int zb = (DIM == 3) ? blockIdx.z * ZCHUNK : 0;
    const int ze = (DIM == 3) ? min(zb + ZCHUNK, nz) : 1;
    const double ihx = g.ih2[0], ihy = g.ih2[1], ihz = g.ih2[2];

    // plane kk of both states (tile + 2 halo) into ring slot kk mod 3, asynchronously
    auto load_plane = [&](int kk) {
        const int slot = (DIM == 3) ? mod3(kk) : 0;
        const int gz = zplane(g, kk);
        for (int i = tid; i < HX * HY; i += NT) {
            const int hx = i % HX, hy = i / HX;
            const int gx = wrap_coord(x0 + hx - 2, nx, g.periodic);
            const int gy = wrap_coord(y0 + hy - 2, ny, g.periodic);
            const long long c = ((long long)gz * ny + gy) * nx + gx;
            cp_async16(sxn + slot * HX * HY + i, xn_g + c);
            cp_async16(sxo + slot * HX * HY + i, xo_g + c);
        }
        cp_async_commit();
    };

    // G_u, G_v (scheme.py:270-287) and cbar (scheme.py:223-232) on tile + 1 halo of plane kk
    auto compute_g = [&](int kk) {
        const int s0 = (DIM == 3) ? mod3(kk) : 0;
        const int sm = (DIM == 3) ? mod3(kk - 1) : 0;
        const int sp = (DIM == 3) ? mod3(kk + 1) : 0;
        for (int i = tid; i < GX * GY; i += NT) {
            const int gx = i % GX, gy = i / GX;
            const int c = (gy + 1) * HX + (gx + 1);
            const double2 *n = sxn + s0 * HX * HY, *o = sxo + s0 * HX * HY;
            const double2 n0 = n[c], o0 = o[c];
            const double2 nxm = n[c - 1], nxp = n[c + 1], nym = n[c - HX], nyp = n[c + HX];
            const double2 oxm = o[c - 1], oxp = o[c + 1], oym = o[c - HX], oyp = o[c + HX];
            // Laplacian, axes summed x, y, z (grid.py:263-271)
            double lun = (nxp.x - 2.0 * n0.x + nxm.x) * ihx;
            double lvn = (nxp.y - 2.0 * n0.y + nxm.y) * ihx;
            double luo = (oxp.x - 2.0 * o0.x + oxm.x) * ihx;
            double lvo = (oxp.y - 2.0 * o0.y + oxm.y) * ihx;
            lun += (nyp.x - 2.0 * n0.x + nym.x) * ihy;
            lvn += (nyp.y - 2.0 * n0.y + nym.y) * ihy;
            luo += (oyp.x - 2.0 * o0.x + oym.x) * ihy;
            lvo += (oyp.y - 2.0 * o0.y + oym.y) * ihy;
            if (DIM == 3) {
                const double2 nzm = sxn[sm * HX * HY + c], nzp = sxn[sp * HX * HY + c];
                const double2 ozm = sxo[sm * HX * HY + c], ozp = sxo[sp * HX * HY + c];
                lun += (nzp.x - 2.0 * n0.x + nzm.x) * ihz;
                lvn += (nzp.y - 2.0 * n0.y + nzm.y) * ihz;
                luo += (ozp.x - 2.0 * o0.x + ozm.x) * ihz;
                lvo += (ozp.y - 2.0 * o0.y + ozm.y) * ihz;
            }
            const double phi = chord_fast<0>(n0.x + n0.y, o0.x + o0.y, P);
            const double psi = chord_fast<0>(n0.x - n0.y, o0.x - o0.y, P);
            const int idx = s0 * GX * GY + i;
            sGu[idx] = -0.5 * P.alpha * (n0.x + o0.x - 1.0) + P.theta * (phi + psi) - 0.5 * P.gamma * (lun + luo);
            sGv[idx] = -0.5 * P.beta * (n0.y + o0.y) + P.theta * (phi - psi) - 0.5 * P.gamma * (lvn + lvo);
            sCb[idx] = 0.5 * (mobility(o0.x, o0.y) + mobility(n0.x, n0.y));
        }
    };

    double acc_norm = 0.0, acc_gap = INFINITY;
    const int x = x0 + tx, y = y0 + ty;
    const bool active = x < nx && y < ny;
    const bool per = g.periodic != 0;
    const int gc = (ty + 1) * GX + (tx + 1);
    const int xc = (ty + 2) * HX + (tx + 2);

    auto output = [&](int k, const double2 &n0, const double2 &o0) {
        const int s0 = (DIM == 3) ? mod3(k) : 0;
        const int sm = (DIM == 3) ? mod3(k - 1) : 0;
        const int sp = (DIM == 3) ? mod3(k + 1) : 0;
        const double *Gu = sGu + s0 * GX * GY, *Cb = sCb + s0 * GX * GY;
        const double G0 = Gu[gc], C0 = Cb[gc];
        // div(cbar grad G_u), flux form (grid.py:274-298); a Neumann wall face
        // carries no flux (mirrored ghost: g[ghost] - g[cell] == 0).
        double div = 0.0;
        {
            const bool lo = per || x > 0, hi = per || x < nx - 1;
            const double fp = hi ? 0.5 * (C0 + Cb[gc + 1]) * (Gu[gc + 1] - G0) : 0.0;
            const double fm = lo ? 0.5 * (C0 + Cb[gc - 1]) * (G0 - Gu[gc - 1]) : 0.0;
            div += (fp - fm) * ihx;
        }
        {
            const bool lo = per || y > 0, hi = per || y < ny - 1;
            const double fp = hi ? 0.5 * (C0 + Cb[gc + GX]) * (Gu[gc + GX] - G0) : 0.0;
            const double fm = lo ? 0.5 * (C0 + Cb[gc - GX]) * (G0 - Gu[gc - GX]) : 0.0;
            div += (fp - fm) * ihy;
        }
        if (DIM == 3) {
            const bool lo = zstep_ok(g, k, -1), hi = zstep_ok(g, k, +1);
            const double fp = hi ? 0.5 * (C0 + sCb[sp * GX * GY + gc]) * (sGu[sp * GX * GY + gc] - G0) : 0.0;
            const double fm = lo ? 0.5 * (C0 + sCb[sm * GX * GY + gc]) * (G0 - sGu[sm * GX * GY + gc]) : 0.0;
            div += (fp - fm) * ihz;
        }
        double2 f;
        f.x = (n0.x - o0.x) / dt - div;
        f.y = (n0.y - o0.y) / dt + (C0 / P.rho) * sGv[s0 * GX * GY + gc];
        F[cell_at(g, x, y, zplane(g, k))] = f;
        acc_norm += f.x * f.x + f.y * f.y;
        acc_gap = red_combine(acc_gap, cell_gap(n0.x, n0.y), RED_MIN);
    };

    if (DIM == 2) {
        load_plane(0);
        cp_async_wait_all();
        __syncthreads();
        compute_g(0);
        __syncthreads();
        if (active) output(0, sxn[xc], sxo[xc]);
    } else {
        // pipeline: x ring {k, k+1, k+2}, x(k+3) in flight; G ring {k-1, k, k+1}
        load_plane(zb - 2);
        load_plane(zb - 1);
        load_plane(zb);
        cp_async_wait_all();
        __syncthreads();
        compute_g(zb - 1);
        __syncthreads();
        load_plane(zb + 1);
        cp_async_wait_all();
        __syncthreads();
        compute_g(zb);
        __syncthreads();
        load_plane(zb + 2);
        for (int k = zb; k < ze; ++k) {
            cp_async_wait_all();
            __syncthreads();
            const double2 n0 = sxn[mod3(k) * HX * HY + xc], o0 = sxo[mod3(k) * HX * HY + xc];
            compute_g(k + 1);
            __syncthreads();
            if (k + 3 <= ze + 1) load_plane(k + 3);
            if (active) output(k, n0, o0);
        }
    }
    double v[2] = {acc_norm, acc_gap};
    const int ops[2] = {RED_SUM, RED_MIN};
    reduce_finish<2>(v, ops, partials, counter, result);
}

// ---------------------------------------------------------------------------
// z-marching residual, one barrier per plane (3D default) -- the matvec's
// pipeline (mv_zm_kernel below) with the discrete variational derivative:
//   * both states U', U^n: 4-slot smem rings of tile+2 planes, cp.async two
//     planes ahead;
//   * every tile+1 column (centre columns one per thread + the ring columns
//     of the first threads) evaluates G_u, G_v, cbar once per plane
//     (scheme.py:270-287, entropy chords included) into a 3-slot smem ring
//     B = (G_u, cbar); the centre keeps G_v and its states in registers;
//   * the z-neighbours of a column's states stay in the owning thread's
//     registers; all offsets are computed once.
// ||F||^2 and the admissibility gap are fused (deterministic grid reduction).
// ---------------------------------------------------------------------------

template <int TX, int TY>
struct RzmSmem {
    static constexpr int HX = TX + 4, HY = TY + 4, GX = TX + 2, GY = TY + 2;
    // ring columns: the tile+1 border without its 4 corners (never read by the 5-point output)
    static constexpr int NW = HX * HY, NB = GX * GY, NRING = 2 * TX + 2 * TY;
    static constexpr size_t bytes = sizeof(double2) * (2 * 4 * NW + 3 * NB);
};

template <int TX, int TY, int MINB, bool PER, bool RW, int ORDER>
__global__ void __launch_bounds__(TX *TY + (RW ? 32 * ((2 * TX + 2 * TY + 31) / 32) : 0), MINB)
res_zm_kernel(const GridDev g, const ParamsDev P, double dt, const double2 *__restrict__ xo_g,
              const double2 *__restrict__ xn_g, double2 *__restrict__ F, double *partials, unsigned int *counter,
              double *result, int nchunk)
{
    using L = RzmSmem<TX, TY>;
    constexpr int HX = L::HX, GX = L::GX, NW = L::NW, NB = L::NB, NRING = L::NRING, NT = TX * TY;
    // RW: the ring columns get their own warps (every thread owns one column,
    // the centre warps also emit the outputs), else the first NRING centre
    // threads own a ring column too
    constexpr int NTA = NT + (RW ? 32 * ((NRING + 31) / 32) : 0);
    constexpr int NWR = (NW + NTA - 1) / NTA;
    static_assert(NRING <= NT, "ring columns must fit one per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sN = reinterpret_cast<double2 *>(smem_raw);   // [4][NW]   U'
    double2 *sO = sN + 4 * NW;                               // [4][NW]   U^n
    double2 *sB = sO + 4 * NW;                               // [3][NB]   (G_u, cbar)

    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const bool centre = !RW || tid < NT;
    const int tx = tid % TX, ty = centre ? tid / TX : 0;
    const int nx = g.nx, ny = g.ny;
    const long long nxy = (long long)nx * ny;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = (int)(((long long)blockIdx.z * g.nz) / nchunk);
    const int ze = (int)(((long long)(blockIdx.z + 1) * g.nz) / nchunk);
    const double ihx = g.ih2[0], ihy = g.ih2[1], ihz = g.ih2[2];
    const double c2lap = 2.0 * (ihx + ihy + ihz);
    const double ha = -0.5 * P.alpha, hb = -0.5 * P.beta, hg = 0.5 * P.gamma;
    const double idt = 1.0 / dt, irho2 = 2.0 * (1.0 / P.rho);

    int woff[NWR];
#pragma unroll
    for (int r = 0; r < NWR; ++r) {
        const int i = tid + r * NTA;
        const int hx = i % HX, hy = i / HX;
        woff[r] = (i < NW) ? wrap_coord(y0 + hy - 2, ny, g.periodic) * nx + wrap_coord(x0 + hx - 2, nx, g.periodic) : 0;
    }
    const bool has_ring = !RW && tid < NRING;
    int cx[2], cy[2];
    cx[0] = tx;
    cy[0] = ty;
    {
        int r = has_ring ? tid : 0;
        if (RW && !centre) r = min(tid - NT, NRING - 1);   // spare lanes repeat the last ring column
        if (r < TX) { cx[1] = r; cy[1] = -1; }
        else if (r < 2 * TX) { cx[1] = r - TX; cy[1] = TY; }
        else if (r < 2 * TX + TY) { cx[1] = -1; cy[1] = r - 2 * TX; }
        else { cx[1] = TX; cy[1] = r - 2 * TX - TY; }
        if (RW && !centre) {
            cx[0] = cx[1];
            cy[0] = cy[1];
        }
    }
    int hc[2], gc[2], coff[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        hc[j] = (cy[j] + 2) * HX + (cx[j] + 2);
        gc[j] = (cy[j] + 1) * GX + (cx[j] + 1);
        coff[j] = wrap_coord(y0 + cy[j], ny, g.periodic) * nx + wrap_coord(x0 + cx[j], nx, g.periodic);
    }
    const int x = x0 + tx, y = y0 + ty;
    const bool active = centre && x < nx && y < ny;
    const bool fxl = PER || x > 0, fxh = PER || x < nx - 1, fyl = PER || y > 0, fyh = PER || y < ny - 1;
    const int jn = has_ring ? 2 : 1;

    // shared-memory addresses of this thread's copy targets in slot 0 and
    // its source pointers, computed once (per plane only the offsets move)
    const unsigned sn0 = (unsigned)__cvta_generic_to_shared(sN + tid);
    const unsigned so0 = (unsigned)__cvta_generic_to_shared(sO + tid);
    const double2 *srcn_r[NWR], *srco_r[NWR];
#pragma unroll
    for (int r = 0; r < NWR; ++r) {
        srcn_r[r] = xn_g + woff[r];
        srco_r[r] = xo_g + woff[r];
    }
    auto load_x = [&](long long poff, int slot) {
        const unsigned so = (unsigned)(slot * NW) * (unsigned)sizeof(double2);
#pragma unroll
        for (int r = 0; r < NWR; ++r)
            if (r < NWR - 1 || tid + r * NTA < NW) {
                const unsigned ro = so + (unsigned)(r * NTA) * (unsigned)sizeof(double2);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sn0 + ro), "l"(srcn_r[r] + poff));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(so0 + ro), "l"(srco_r[r] + poff));
            }
    };

    double2 nz[2], oz[2];                     // column states at the plane below the one being built
    double2 nk = make_double2(0.0, 0.0), ok_ = nk, nk1 = nk, ok1 = nk;   // centre states, planes k, k+1
    double gvk = 0.0, gvk1 = 0.0;             // centre G_v, planes k, k+1

    // B(kk) from X(kk) (slot s1) and X(kk+1) (slot s2); nz/oz = states at kk-1
    auto build = [&](int s1, int s2, int sb) {
        const double2 *N1 = sN + s1 * NW, *O1 = sO + s1 * NW, *N2 = sN + s2 * NW, *O2 = sO + s2 * NW;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (j < jn) {
                const int h = hc[j];
                const double2 n0 = N1[h], o0 = O1[h];
                const double2 nxm = N1[h - 1], nxp = N1[h + 1], nym = N1[h - HX], nyp = N1[h + HX];
                const double2 oxm = O1[h - 1], oxp = O1[h + 1], oym = O1[h - HX], oyp = O1[h + HX];
                const double2 nzp = N2[h], ozp = O2[h];
                // Laplacians of U' + U^n (the DVD needs only their sum,
                // scheme.py:277-286): neighbour pairs per axis, one centre term
                const double lu = (nxp.x + nxm.x + (oxp.x + oxm.x)) * ihx + (nyp.x + nym.x + (oyp.x + oym.x)) * ihy +
                                  (nzp.x + nz[j].x + (ozp.x + oz[j].x)) * ihz - c2lap * (n0.x + o0.x);
                const double lv = (nxp.y + nxm.y + (oxp.y + oxm.y)) * ihx + (nyp.y + nym.y + (oyp.y + oym.y)) * ihy +
                                  (nzp.y + nz[j].y + (ozp.y + oz[j].y)) * ihz - c2lap * (n0.y + o0.y);
                double phi, psi;
                if constexpr (ORDER == 10) {
                    phi = chord_res<ORDER>(n0.x + n0.y, o0.x + o0.y, P);
                    psi = chord_res<ORDER>(n0.x - n0.y, o0.x - o0.y, P);
                } else {
                    phi = chord_fast<0>(n0.x + n0.y, o0.x + o0.y, P);
                    psi = chord_fast<0>(n0.x - n0.y, o0.x - o0.y, P);
                }
                const double Gu = ha * (n0.x + o0.x - 1.0) + P.theta * (phi + psi) - hg * lu;
                // half the averaged mobility: the face value (c(a) + c(b)) / 2 is then one
                // addition, and the v row scales by 2 / rho (exact power-of-two shifts:
                // bitwise the same fluxes)
                const double cbh = 0.25 * (mobility(o0.x, o0.y) + mobility(n0.x, n0.y));
                sB[sb * NB + gc[j]] = make_double2(Gu, cbh);
                nz[j] = n0;
                oz[j] = o0;
                if (j == 0) {
                    gvk1 = hb * (n0.y + o0.y) + P.theta * (phi - psi) - hg * lv;
                    nk1 = n0;
                    ok1 = o0;
                }
            }
        }
    };

    int z0 = zplane_near(g, zb), z1 = zplane_near(g, zb + 1), z2 = zplane_near(g, zb + 2), z3 = zplane_near(g, zb + 3);
    auto poff = [&](int zs) { return (long long)zs * nxy; };
    {
        const long long pm2 = zplane_near(g, zb - 2) * nxy, pm1 = zplane_near(g, zb - 1) * nxy;
#pragma unroll
        for (int j = 0; j < 2; ++j)
            if (j < jn) {
                nz[j] = __ldg(xn_g + pm2 + coff[j]);
                oz[j] = __ldg(xo_g + pm2 + coff[j]);
            }
        load_x(pm1, 0);
        load_x(poff(z0), 1);
        cp_async_commit();
    }
    cp_async_wait_all();
    __syncthreads();
    load_x(poff(z1), 2);
    cp_async_commit();
    load_x(poff(z2), 3);
    cp_async_commit();
    build(0, 1, 0);              // B(zb-1)
    cp_async_wait_group<1>();
    __syncthreads();
    load_x(poff(z3), 0);
    cp_async_commit();
    build(1, 2, 1);              // B(zb)
    nk = nk1;
    ok_ = ok1;
    gvk = gvk1;
    double acc_norm = 0.0, acc_gap = INFINITY;
    int sw1 = 2, sw2 = 3, sw3 = 0;
    int sb0 = 0, sb1 = 1, sb2 = 2;
    int z4 = zplane_near(g, zb + 4);
    for (int k = zb; k < ze; ++k) {
        cp_async_wait_group<1>();
        __syncthreads();
        const int swf = 6 - sw1 - sw2 - sw3;
        if (k + 4 <= ze + 1) load_x(poff(z4), swf);
        cp_async_commit();
        build(sw1, sw2, sb2);    // B(k+1)
        if (active) {
            const double2 *B = sB + sb1 * NB;
            const int c0 = gc[0];
            const double2 b0 = B[c0];
            const double G0 = b0.x, C0 = b0.y;   // C0 = cbar / 2
            double div = 0.0;
            {
                const double2 bp = B[c0 + 1], bm = B[c0 - 1];
                const double fp = fxh ? (C0 + bp.y) * (bp.x - G0) : 0.0;
                const double fm = fxl ? (C0 + bm.y) * (G0 - bm.x) : 0.0;
                div += (fp - fm) * ihx;
            }
            {
                const double2 bp = B[c0 + GX], bm = B[c0 - GX];
                const double fp = fyh ? (C0 + bp.y) * (bp.x - G0) : 0.0;
                const double fm = fyl ? (C0 + bm.y) * (G0 - bm.x) : 0.0;
                div += (fp - fm) * ihy;
            }
            {
                const double2 bp = sB[sb2 * NB + c0], bm = sB[sb0 * NB + c0];
                const double fp = (PER || zstep_ok(g, k, +1)) ? (C0 + bp.y) * (bp.x - G0) : 0.0;
                const double fm = (PER || zstep_ok(g, k, -1)) ? (C0 + bm.y) * (G0 - bm.x) : 0.0;
                div += (fp - fm) * ihz;
            }
            double2 f;
            f.x = (nk.x - ok_.x) * idt - div;
            f.y = (nk.y - ok_.y) * idt + (C0 * irho2) * gvk;
            F[poff(z0) + coff[0]] = f;
            acc_norm += f.x * f.x + f.y * f.y;
            acc_gap = red_combine(acc_gap, cell_gap_fast(nk.x, nk.y), RED_MIN);
        }
        nk = nk1;
        ok_ = ok1;
        gvk = gvk1;
        sw1 = sw2;
        sw2 = sw3;
        sw3 = swf;
        const int tb = sb0;
        sb0 = sb1;
        sb1 = sb2;
        sb2 = tb;
        z0 = z1;
        z1 = z2;
        z2 = z3;
        z3 = z4;
        z4 = zplane_near(g, k + 5);
    }
    double v[2] = {acc_norm, acc_gap};
    const int ops[2] = {RED_SUM, RED_MIN};
    reduce_finish<2>(v, ops, partials, counter, result);
}

// ---------------------------------------------------------------------------
// Jacobian coefficient planes (one thread per cell)
// ---------------------------------------------------------------------------

__global__ void jac_prepare_kernel(GridDev g, ParamsDev P, const double2 *__restrict__ xo,
                                   const double2 *__restrict__ xn, double *__restrict__ coef)
{
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= g.n) return;
    const int x = (int)(q % g.nx), y = (int)((q / g.nx) % g.ny), z = (int)(q / ((long long)g.nx * g.ny));
    const long long c = cell_at(g, x, y, zplane(g, z));
    const double2 n0 = xn[c], o0 = xo[c];
    double lun = 0.0, lvn = 0.0, luo = 0.0, lvo = 0.0;
    for (int a = 0; a < g.dim; ++a) {
        long long im, ip;
        if (a == 0) {
            im = cell_at(g, wrap_coord(x - 1, g.nx, g.periodic), y, zplane(g, z));
            ip = cell_at(g, wrap_coord(x + 1, g.nx, g.periodic), y, zplane(g, z));
        } else if (a == 1) {
            im = cell_at(g, x, wrap_coord(y - 1, g.ny, g.periodic), zplane(g, z));
            ip = cell_at(g, x, wrap_coord(y + 1, g.ny, g.periodic), zplane(g, z));
        } else {
            im = cell_at(g, x, y, zplane(g, z - 1));
            ip = cell_at(g, x, y, zplane(g, z + 1));
        }
        const double2 nm = xn[im], np_ = xn[ip], om = xo[im], op = xo[ip];
        lun += (np_.x - 2.0 * n0.x + nm.x) * g.ih2[a];
        lvn += (np_.y - 2.0 * n0.y + nm.y) * g.ih2[a];
        luo += (op.x - 2.0 * o0.x + om.x) * g.ih2[a];
        lvo += (op.y - 2.0 * o0.y + om.y) * g.ih2[a];
    }
    double phi, psi, dp, dq;
    entropy_chord<true>(n0.x + n0.y, o0.x + o0.y, P, 0, phi, dp);
    entropy_chord<true>(n0.x - n0.y, o0.x - o0.y, P, 0, psi, dq);
    const long long N = g.nstore;
    double4 a;
    a.x = P.theta * (dp + dq);                                   // S
    a.y = P.theta * (dp - dq);                                   // D
    a.z = (1.0 - 2.0 * n0.x) * (0.25 - n0.y * n0.y);             // c_u  (physics.py:133-135)
    a.w = -2.0 * n0.y * n0.x * (1.0 - n0.x);                     // c_v
    reinterpret_cast<double4 *>(coef)[c] = a;
    double2 b;
    b.x = 0.5 * (mobility(o0.x, o0.y) + mobility(n0.x, n0.y));   // cbar
    b.y = -0.5 * P.alpha * (n0.x + o0.x - 1.0) + P.theta * (phi + psi) - 0.5 * P.gamma * (lun + luo);   // G_u
    reinterpret_cast<double2 *>(coef + 4 * N)[c] = b;
    coef[6 * N + c] = -0.5 * P.beta * (n0.y + o0.y) + P.theta * (phi - psi) - 0.5 * P.gamma * (lvn + lvo);   // G_v
}

// ---------------------------------------------------------------------------
// matrix-free Jacobian matvec
//   dG_u = (-alpha/2 + S) w_u + D w_v - gamma/2 lap(w_u)
//   eta  = (c_u w_u + c_v w_v) / 2            (linearised trapezoidal mobility)
//   y_u  = w_u/dt - div(cbar grad dG_u) - div(eta_face grad G_u)
//   y_v  = w_v/dt + cbar/rho (D w_u + (-beta/2 + S) w_v - gamma/2 lap(w_v)) + G_v/rho eta
// term-for-term the operator assembled at scheme.py:471-482.
// ---------------------------------------------------------------------------

template <int TX, int TY>
struct ZmSmem {
    static constexpr int HX = TX + 4, HY = TY + 4, GX = TX + 2, GY = TY + 2;
    // ring columns: the tile+1 border without its 4 corners (never read by the 5-point output)
    static constexpr int NW = HX * HY, NB = GX * GY, NRING = 2 * TX + 2 * TY;
    static constexpr size_t bytes = sizeof(double2) * (4 * NW + 2 * 3 * NB);
};

// host-computed constants of the matvec (kernel parameters, i.e. constant-bank
// operands, so they cost no registers in the plane loop)
struct MvConst {
    const double4 *A;
    const double2 *B;
    const double *Gv;
    double ihx, ihy, ihz;    // 1/h^2
    double fhx, fhy, fhz;    // 0.5/h^2 (flux weights)
    double hg, ha, hb;       // gamma/2, -alpha/2, -beta/2
    double idt, irho;        // 1/dt, 1/rho
};

template <int TX, int TY, int MINB, bool PER, bool RW>
__global__ void __launch_bounds__(TX *TY + (RW ? 32 * ((2 * TX + 2 * TY + 31) / 32) : 0), MINB)
mv_zm_kernel(const GridDev g, const MvConst mc, const double2 *__restrict__ w_g, double2 *__restrict__ yout,
             int nchunk)
{
    ACCH_SKIP_IF(g);
    using L = ZmSmem<TX, TY>;
    constexpr int HX = L::HX, GX = L::GX, NW = L::NW, NB = L::NB, NRING = L::NRING, NT = TX * TY;
    // RW: the ring columns get their own warps (every thread owns one column,
    // the centre warps also emit the outputs), else the first NRING centre
    // threads own a ring column too
    constexpr int NTA = NT + (RW ? 32 * ((NRING + 31) / 32) : 0);
    constexpr int NWR = (NW + NTA - 1) / NTA;
    static_assert(NRING <= NT, "ring columns must fit one per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sW = reinterpret_cast<double2 *>(smem_raw);      // [4][NW]   w
    double2 *sB1 = sW + 4 * NW;                                  // [3][NB]   (dG_u, cbar)
    double2 *sB2 = sB1 + 3 * NB;                                 // [3][NB]   (eta, G_u)

    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const bool centre = !RW || tid < NT;
    const int tx = tid % TX, ty = centre ? tid / TX : 0;
    const int nx = g.nx, ny = g.ny;
    const long long nxy = (long long)nx * ny;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    // z range of this chunk: chunks split nz as evenly as possible
    const int zb = (int)(((long long)blockIdx.z * g.nz) / nchunk);
    const int ze = (int)(((long long)(blockIdx.z + 1) * g.nz) / nchunk);
    const double4 *__restrict__ cA = mc.A;
    const double2 *__restrict__ cB = mc.B;
    const double *__restrict__ cGv = mc.Gv;
    const double &ihx = mc.ihx, &ihy = mc.ihy, &ihz = mc.ihz;
    // flux weights 0.5/h^2: 0.5 (C0 + Cn) (Gn - G0) / h^2 == (C0 + Cn) (Gn - G0) (0.5/h^2) bitwise
    const double &fhx = mc.fhx, &fhy = mc.fhy, &fhz = mc.fhz;
    const double &hg = mc.hg, &ha = mc.ha, &hb = mc.hb;
    const double &idt = mc.idt, &irho = mc.irho;

    // w tile+2 copy offsets (plane-relative)
    int woff[NWR];
#pragma unroll
    for (int r = 0; r < NWR; ++r) {
        const int i = tid + r * NTA;
        const int hx = i % HX, hy = i / HX;
        woff[r] = (i < NW) ? wrap_coord(y0 + hy - 2, ny, g.periodic) * nx + wrap_coord(x0 + hx - 2, nx, g.periodic) : 0;
    }
    // owned columns: j = 0 centre (tx, ty); j = 1 ring column tid (tid < NRING)
    const bool has_ring = tid < NRING;
    int cx[2], cy[2];
    cx[0] = tx;
    cy[0] = ty;
    {
        // ring of the tile+1 region in tile coordinates (-1 .. TX, -1 .. TY)
        int r = has_ring ? tid : 0;
        if (r < TX) { cx[1] = r; cy[1] = -1; }
        else if (r < 2 * TX) { cx[1] = r - TX; cy[1] = TY; }
        else if (r < 2 * TX + TY) { cx[1] = -1; cy[1] = r - 2 * TX; }
        else { cx[1] = TX; cy[1] = r - 2 * TX - TY; }
        if (RW && !centre) {
            cx[0] = cx[1];
            cy[0] = cy[1];
        }
    }
    int hc[2], gc[2], coff[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        hc[j] = (cy[j] + 2) * HX + (cx[j] + 2);
        gc[j] = (cy[j] + 1) * GX + (cx[j] + 1);
        coff[j] = wrap_coord(y0 + cy[j], ny, g.periodic) * nx + wrap_coord(x0 + cx[j], nx, g.periodic);
    }
    const int x = x0 + tx, y = y0 + ty;
    const bool active = centre && x < nx && y < ny;
    const bool fxl = PER || x > 0, fxh = PER || x < nx - 1, fyl = PER || y > 0, fyh = PER || y < ny - 1;
    const int jn = has_ring ? 2 : 1;

    // cp.async of one w plane (tile+2) into a ring slot; the caller commits
    auto load_w = [&](long long poff, int slot) {
        const double2 *src = w_g + poff;
        double2 *dst = sW + slot * NW + tid;
#pragma unroll
        for (int r = 0; r < NWR; ++r)
            if (r < NWR - 1 || tid + r * NTA < NW) cp_async16(dst + r * NTA, src + woff[r]);
    };

    double cS[2], cD[2], cU[2], cV[2], cC[2], cG[2];
    auto prefetch = [&](long long poff) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (j < jn) {
                const double4 a = ldg256(cA + poff + coff[j]);
                const double2 b = __ldg(cB + poff + coff[j]);
                cS[j] = a.x;
                cD[j] = a.y;
                cU[j] = a.z;
                cV[j] = a.w;
                cC[j] = b.x;
                cG[j] = b.y;
            }
        }
    };

    // column values carried across planes
    double wuz[2];                 // w_u of column j at the plane below the one being built
    double2 wk = make_double2(0.0, 0.0), wk1 = wk;   // centre w at planes k, k+1
    double wvm = 0.0;                                 // centre w_v at plane k-1
    double lxy_k = 0.0, lxy_k1 = 0.0;                 // centre xy-lap(w_v) at planes k, k+1
    double Sk = 0.0, Dk = 0.0, Sk1 = 0.0, Dk1 = 0.0;  // centre S, D at planes k, k+1
    // centre column's (dG_u, cbar, eta, G_u) at planes k-1, k, k+1 (registers:
    // the z-faces and the cell's own values need no shared-memory reads)
    double4 bm = make_double4(0.0, 0.0, 0.0, 0.0), b0 = bm, b1 = bm;

    // build B(kk) from W(kk) (slot s1) and W(kk+1) (slot s2); wuz = w_u(kk-1)
    auto build = [&](int s1, int s2, int sb) {
        const double2 *W1 = sW + s1 * NW, *W2 = sW + s2 * NW;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (j < jn) {
                const int h = hc[j];
                const double2 w0 = W1[h], xm = W1[h - 1], xp = W1[h + 1], ym = W1[h - HX], yp = W1[h + HX];
                const double zp = W2[h].x;
                double lap = (xp.x - 2.0 * w0.x + xm.x) * ihx;
                lap += (yp.x - 2.0 * w0.x + ym.x) * ihy;
                lap += (zp - 2.0 * w0.x + wuz[j]) * ihz;
                const double dG = (ha + cS[j]) * w0.x + cD[j] * w0.y - hg * lap;
                const double et = 0.5 * (cU[j] * w0.x + cV[j] * w0.y);
                sB1[sb * NB + gc[j]] = make_double2(dG, cC[j]);
                sB2[sb * NB + gc[j]] = make_double2(et, cG[j]);
                wuz[j] = w0.x;
                if (j == 0) {
                    wk1 = w0;
                    lxy_k1 = (xp.y - 2.0 * w0.y + xm.y) * ihx + (yp.y - 2.0 * w0.y + ym.y) * ihy;
                    Sk1 = cS[0];
                    Dk1 = cD[0];
                    b1 = make_double4(dG, cC[0], et, cG[0]);
                }
            }
        }
    };

    // storage offsets of planes k .. k+3 (rolled once per plane, no division)
    int z0 = zplane_near(g, zb), z1 = zplane_near(g, zb + 1), z2 = zplane_near(g, zb + 2), z3 = zplane_near(g, zb + 3);
    auto poff = [&](int zs) { return (long long)zs * nxy; };

    // prologue: B(zb-1) and B(zb) are built before iteration zb; W(zb-2) is
    // needed only as the z-neighbour w_u(zb-2) of each column (a register).
    // w planes are copied two iterations ahead (4-slot ring, one commit group
    // per plane).
    {
        const long long pm2 = zplane_near(g, zb - 2) * nxy, pm1 = zplane_near(g, zb - 1) * nxy;
#pragma unroll
        for (int j = 0; j < 2; ++j)
            if (j < jn) wuz[j] = __ldg(&w_g[pm2 + coff[j]].x);
        load_w(pm1, 0);
        load_w(poff(z0), 1);
        cp_async_commit();
        prefetch(pm1);
    }
    cp_async_wait_all();
    __syncthreads();
    load_w(poff(z1), 2);
    cp_async_commit();
    load_w(poff(z2), 3);
    cp_async_commit();
    build(0, 1, 0);              // B(zb-1) -> slot 0; needs W(zb) centre = slot 1
    wvm = wk1.y;
    bm = b1;
    prefetch(poff(z0));
    cp_async_wait_group<1>();    // W(zb+1) landed, W(zb+2) may still be in flight
    __syncthreads();
    // now W(zb) slot 1, W(zb+1) slot 2, W(zb+2) slot 3; slot 0 (W(zb-1)) is free
    load_w(poff(z3), 0);
    cp_async_commit();
    build(1, 2, 1);              // B(zb) -> slot 1
    b0 = b1;
    wk = wk1;
    lxy_k = lxy_k1;
    Sk = Sk1;
    Dk = Dk1;
    prefetch(poff(z1));
    double gvk = active ? __ldg(cGv + poff(z0) + coff[0]) : 0.0;
    int sw1 = 2, sw2 = 3, sw3 = 0;   // slots of W(k+1), W(k+2), W(k+3) at the top of iteration k
    int sb0 = 0, sb1 = 1, sb2 = 2;   // slots of B(k-1), B(k), B(k+1)
    int z4 = zplane_near(g, zb + 4);
    for (int k = zb; k < ze; ++k) {
        cp_async_wait_group<1>();    // W(k+2) landed (W(k+3) may be in flight)
        __syncthreads();
        // the W slot of plane k is free (W(k) lives in registers): W(k+4) into it
        const int swf = 6 - sw1 - sw2 - sw3;
        if (k + 4 <= ze + 1) load_w(poff(z4), swf);
        cp_async_commit();           // possibly empty: keeps one group per plane
        build(sw1, sw2, sb2);    // B(k+1)
        double gvn = 0.0;
        if (k + 2 <= ze) prefetch(poff(z2));
        if (active && k + 1 < ze) gvn = __ldg(cGv + poff(z1) + coff[0]);
        if (active) {
            const double2 *B1 = sB1 + sb1 * NB, *B2 = sB2 + sb1 * NB;
            const int c0 = gc[0];
            const double dG0 = b0.x, C0 = b0.y, E0 = b0.z, G0 = b0.w;
            double d1 = 0.0, d2 = 0.0;
            auto face = [&](const double2 &an, const double2 &en, double fh, bool lo_ok, bool hi_ok,
                            const double2 &am, const double2 &em) {
                if (hi_ok) {
                    d1 += (C0 + an.y) * (an.x - dG0) * fh;
                    d2 += (E0 + en.x) * (en.y - G0) * fh;
                }
                if (lo_ok) {
                    d1 -= (C0 + am.y) * (dG0 - am.x) * fh;
                    d2 -= (E0 + em.x) * (G0 - em.y) * fh;
                }
            };
            face(B1[c0 + 1], B2[c0 + 1], fhx, fxl, fxh, B1[c0 - 1], B2[c0 - 1]);
            face(B1[c0 + GX], B2[c0 + GX], fhy, fyl, fyh, B1[c0 - GX], B2[c0 - GX]);
            face(make_double2(b1.x, b1.y), make_double2(b1.z, b1.w), fhz, PER || zstep_ok(g, k, -1),
                 PER || zstep_ok(g, k, +1), make_double2(bm.x, bm.y), make_double2(bm.z, bm.w));
            const double lapv = lxy_k + (wk1.y - 2.0 * wk.y + wvm) * ihz;
            double2 out;
            out.x = wk.x * idt - d1 - d2;
            out.y = wk.y * idt + (C0 * irho) * (Dk * wk.x + (hb + Sk) * wk.y - hg * lapv) + (gvk * irho) * E0;
            yout[poff(z0) + coff[0]] = out;
        }
        // rotate
        bm = b0;
        b0 = b1;
        wvm = wk.y;
        wk = wk1;
        lxy_k = lxy_k1;
        Sk = Sk1;
        Dk = Dk1;
        gvk = gvn;
        sw1 = sw2;
        sw2 = sw3;
        sw3 = swf;
        const int tb = sb0;
        sb0 = sb1;
        sb1 = sb2;
        sb2 = tb;
        z0 = z1;
        z1 = z2;
        z2 = z3;
        z3 = z4;
        z4 = zplane_near(g, k + 5);
    }
}

// ---------------------------------------------------------------------------
// Two-pass matrix-free matvec (thread per cell, neighbours through L1/L2):
//   pass 1: T = (dG_u, eta) per cell                 reads w, S, D, c_u, c_v
//   pass 2: y from T, cbar, G_u (7-point), w, S, D, G_v
// 152 B/cell of DRAM traffic instead of 88, but both passes are plain
// coalesced streams with high occupancy and no barriers.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cell_xyz(const GridDev &g, long long q, int &x, int &y, int &z)
{
    x = (int)(q % g.nx);
    y = (int)((q / g.nx) % g.ny);
    z = (int)(q / ((long long)g.nx * g.ny));
}

// thread (x, y) of a 32 x 8 tile, blockIdx.z = plane: no index division
constexpr int PTX = 32, PTY = 8;

template <int DIM>
__global__ void __launch_bounds__(PTX * PTY)
mv_pass1_kernel(GridDev g, ParamsDev P, const double *__restrict__ coef, const double2 *__restrict__ w,
                double2 *__restrict__ T, int zlo)
{
    ACCH_SKIP_IF(g);
    // planes zlo .. : in slab mode also the first ghost plane past an
    // interior slab boundary, which pass 2 reads as a z-neighbour
    const int x = blockIdx.x * PTX + threadIdx.x, y = blockIdx.y * PTY + threadIdx.y;
    if (x >= g.nx || y >= g.ny) return;
    const int z = (int)blockIdx.z + zlo;
    const int zs = zplane(g, z);
    const long long c = cell_at(g, x, y, zs);
    const long long N = g.nstore;
    const double2 w0 = __ldg(w + c);
    double lap = (__ldg(w + cell_at(g, wrap_coord(x + 1, g.nx, g.periodic), y, zs)).x - 2.0 * w0.x +
                  __ldg(w + cell_at(g, wrap_coord(x - 1, g.nx, g.periodic), y, zs)).x) * g.ih2[0];
    lap += (__ldg(w + cell_at(g, x, wrap_coord(y + 1, g.ny, g.periodic), zs)).x - 2.0 * w0.x +
            __ldg(w + cell_at(g, x, wrap_coord(y - 1, g.ny, g.periodic), zs)).x) * g.ih2[1];
    if (DIM == 3)
        lap += (__ldg(w + cell_at(g, x, y, zplane(g, z + 1))).x - 2.0 * w0.x +
                __ldg(w + cell_at(g, x, y, zplane(g, z - 1))).x) * g.ih2[2];
    double2 t;
    const double4 a = ldg256(co_A(coef) + c);
    t.x = (-0.5 * P.alpha + a.x) * w0.x + a.y * w0.y - 0.5 * P.gamma * lap;
    t.y = 0.5 * (a.z * w0.x + a.w * w0.y);
    T[c] = t;
}

template <int DIM>
__global__ void __launch_bounds__(PTX * PTY)
mv_pass2_kernel(GridDev g, ParamsDev P, double dt, const double *__restrict__ coef, const double2 *__restrict__ w,
                const double2 *__restrict__ T, double2 *__restrict__ yout)
{
    ACCH_SKIP_IF(g);
    const int x = blockIdx.x * PTX + threadIdx.x, y = blockIdx.y * PTY + threadIdx.y;
    if (x >= g.nx || y >= g.ny) return;
    const int z = (int)blockIdx.z;
    const int zs = zplane(g, z);
    const long long c = cell_at(g, x, y, zs);
    const long long N = g.nstore;
    const double2 *__restrict__ cB = co_B(coef, N);
    const double2 t0 = __ldg(T + c), w0 = __ldg(w + c);
    const double2 b0 = __ldg(cB + c);
    const double C0 = b0.x, G0 = b0.y;
    const bool per = g.periodic != 0;
    double d1 = 0.0, d2 = 0.0, lapv = 0.0;
    auto face = [&](long long cn, double ih, bool ok, double sgn) {
        // sgn = +1 for the upper face (n - c), -1 for the lower face (c - n)
        if (!ok) return;
        const double2 tn = __ldg(T + cn);
        const double2 bn = __ldg(cB + cn);
        const double Cn = bn.x, Gn = bn.y;
        d1 += 0.5 * (C0 + Cn) * (tn.x - t0.x) * ih;
        d2 += 0.5 * (t0.y + tn.y) * (Gn - G0) * ih;
        (void)sgn;
    };
    const long long cxp = cell_at(g, wrap_coord(x + 1, g.nx, g.periodic), y, zs);
    const long long cxm = cell_at(g, wrap_coord(x - 1, g.nx, g.periodic), y, zs);
    const long long cyp = cell_at(g, x, wrap_coord(y + 1, g.ny, g.periodic), zs);
    const long long cym = cell_at(g, x, wrap_coord(y - 1, g.ny, g.periodic), zs);
    face(cxp, g.ih2[0], per || x < g.nx - 1, 1.0);
    face(cxm, g.ih2[0], per || x > 0, -1.0);
    face(cyp, g.ih2[1], per || y < g.ny - 1, 1.0);
    face(cym, g.ih2[1], per || y > 0, -1.0);
    lapv = (__ldg(w + cxp).y - 2.0 * w0.y + __ldg(w + cxm).y) * g.ih2[0];
    lapv += (__ldg(w + cyp).y - 2.0 * w0.y + __ldg(w + cym).y) * g.ih2[1];
    if (DIM == 3) {
        const long long czp = cell_at(g, x, y, zplane(g, z + 1));
        const long long czm = cell_at(g, x, y, zplane(g, z - 1));
        face(czp, g.ih2[2], zstep_ok(g, z, +1), 1.0);
        face(czm, g.ih2[2], zstep_ok(g, z, -1), -1.0);
        lapv += (__ldg(w + czp).y - 2.0 * w0.y + __ldg(w + czm).y) * g.ih2[2];
    }
    const double2 sd = __ldg(reinterpret_cast<const double2 *>(coef) + 2 * c);   // (S, D) half of A[c]
    const double S = sd.x, D = sd.y, Gv = __ldg(co_Gv(coef, N) + c);
    const double hg = 0.5 * P.gamma;
    double2 out;
    const double idt = 1.0 / dt, irho = 1.0 / P.rho;   // reciprocals (see matvec_kernel)
    out.x = w0.x * idt - d1 - d2;
    out.y = w0.y * idt + (C0 * irho) * (D * w0.x + (-0.5 * P.beta + S) * w0.y - hg * lapv) + (Gv * irho) * t0.y;
    yout[c] = out;
}

// ---------------------------------------------------------------------------
// explicit Jacobian blocks on the radius-2 stencil
// ---------------------------------------------------------------------------

template <int DIM>
__global__ void jac_blocks_kernel(GridDev g, ParamsDev P, double dt, const double *__restrict__ coef,
                                  double *__restrict__ out, int noff)
{
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= g.n) return;
    const int x = (int)(c % g.nx), y = (int)((c / g.nx) % g.ny), z = (int)(c / ((long long)g.nx * g.ny));
    double blk[25][4];
    jac_row_blocks<DIM>(g, P, dt, coef, x, y, z, blk, noff);
    for (int o = 0; o < noff; ++o)
        for (int e = 0; e < 4; ++e) out[(c * noff + o) * 4 + e] = blk[o][e];
}

// ---------------------------------------------------------------------------
// elementwise / reduction helpers on the state
// ---------------------------------------------------------------------------

__global__ void chord_kernel(ParamsDev P, const double *a, const double *b, long long n, int force_exact,
                             double *val, double *der)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v, d = 0.0;
    if (der) entropy_chord<true>(a[i], b[i], P, force_exact, v, d);
    else entropy_chord<false>(a[i], b[i], P, force_exact, v, d);
    val[i] = v;
    if (der) der[i] = d;
}

__global__ void gap_kernel(long long n, const double2 *__restrict__ x, double *partials, unsigned int *counter,
                           double *result)
{
    double gmin = INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 s = x[i];
        const double c = cell_gap(s.x, s.y);
        gmin = red_combine(gmin, c, RED_MIN);
    }
    double v[1] = {gmin};
    const int ops[1] = {RED_MIN};
    reduce_finish<1>(v, ops, partials, counter, result);
}

// energy (physics.py:313-331, grad_sq_avg grid.py:249-260), mass, max|v|
__global__ void diagnostics_kernel(GridDev g, ParamsDev P, const double2 *__restrict__ x, double *partials,
                                   unsigned int *counter, double *result)
{
    double e = 0.0, m = 0.0, vmax = -INFINITY;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n; q += (long long)gridDim.x * blockDim.x) {
        const int xi = (int)(q % g.nx), yi = (int)((q / g.nx) % g.ny), zi = (int)(q / ((long long)g.nx * g.ny));
        const int zs = zplane(g, zi);
        const double2 s = x[cell_at(g, xi, yi, zs)];
        double gsu = 0.0, gsv = 0.0;
        for (int a = 0; a < g.dim; ++a) {
            long long im, ip;
            if (a == 0) {
                im = cell_at(g, wrap_coord(xi - 1, g.nx, g.periodic), yi, zs);
                ip = cell_at(g, wrap_coord(xi + 1, g.nx, g.periodic), yi, zs);
            } else if (a == 1) {
                im = cell_at(g, xi, wrap_coord(yi - 1, g.ny, g.periodic), zs);
                ip = cell_at(g, xi, wrap_coord(yi + 1, g.ny, g.periodic), zs);
            } else {
                im = cell_at(g, xi, yi, zplane(g, zi - 1));
                ip = cell_at(g, xi, yi, zplane(g, zi + 1));
            }
            const double2 sm = x[im], sp = x[ip];
            const double fu = (sp.x - s.x) * g.ih[a], bu = (s.x - sm.x) * g.ih[a];
            const double fv = (sp.y - s.y) * g.ih[a], bv = (s.y - sm.y) * g.ih[a];
            gsu += 0.5 * (fu * fu + bu * bu);
            gsv += 0.5 * (fv * fv + bv * bv);
        }
        const double e1 = 0.5 * P.alpha * s.x * (1.0 - s.x) - 0.5 * P.beta * s.y * s.y;
        const double e2 = P.theta * (entropy(s.x + s.y) + entropy(s.x - s.y));
        e += e1 + e2 + 0.5 * P.gamma * (gsu + gsv);
        m += s.x;
        vmax = red_combine(vmax, fabs(s.y), RED_MAX);
    }
    double v[3] = {e, m, vmax};
    const int ops[3] = {RED_SUM, RED_SUM, RED_MAX};
    reduce_finish<3>(v, ops, partials, counter, result);
}

__global__ void trial_kernel(long long n, const double2 *__restrict__ x, const double2 *__restrict__ s, double lam,
                             double2 *__restrict__ y, double *partials, unsigned int *counter, double *result)
{
    double gmin = INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 a = x[i], d = s[i];
        double2 r;
        r.x = a.x + lam * d.x;
        r.y = a.y + lam * d.y;
        y[i] = r;
        gmin = red_combine(gmin, cell_gap(r.x, r.y), RED_MIN);
    }
    double v[1] = {gmin};
    const int ops[1] = {RED_MIN};
    reduce_finish<1>(v, ops, partials, counter, result);
}

// _feasible_step_cap (newton.py:75-99): min over bounds of (value - lo)/-slope and (hi - value)/slope
__global__ void feasible_cap_kernel(long long n, const double2 *__restrict__ x, const double2 *__restrict__ s,
                                    double margin, double *partials, unsigned int *counter, double *result)
{
    double cap = INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 a = x[i], d = s[i];
        const double vals[4] = {a.x, a.x + a.y, a.x - a.y, a.y};
        const double slopes[4] = {d.x, d.x + d.y, d.x - d.y, d.y};
        const double lo[4] = {margin, margin, margin, -0.5 + margin};
        const double hi[4] = {1.0 - margin, 1.0 - margin, 1.0 - margin, 0.5 - margin};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (slopes[b] < 0.0) cap = red_combine(cap, (vals[b] - lo[b]) / -slopes[b], RED_MIN);
            if (slopes[b] > 0.0) cap = red_combine(cap, (hi[b] - vals[b]) / slopes[b], RED_MIN);
        }
    }
    double v[1] = {cap};
    const int ops[1] = {RED_MIN};
    reduce_finish<1>(v, ops, partials, counter, result);
}

__global__ void rms_diff_kernel(long long n, const double *__restrict__ a, const double *__restrict__ b,
                                double *partials, unsigned int *counter, double *result)
{
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    double v[1] = {acc};
    const int ops[1] = {RED_SUM};
    reduce_finish<1>(v, ops, partials, counter, result);
}

int red_grid(long long n)
{
    long long b = (n + kRedThreads * 4 - 1) / (kRedThreads * 4);
    if (b < 1) b = 1;
    if (b > kRedBlocks) b = kRedBlocks;
    return (int)b;
}

template <typename K>
acch_status set_smem(K kernel, size_t bytes, int carveout = -1)
{
    static_assert(sizeof(K) > 0, "");
    ACCH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (carveout >= 0)
        ACCH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout));
    return ACCH_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

int stencil_offsets(int dim, int (*off)[3])
{
    int n = 0;
    const int zr = dim == 3 ? 2 : 0;
    for (int dz = -zr; dz <= zr; ++dz)
        for (int dy = -2; dy <= 2; ++dy)
            for (int dx = -2; dx <= 2; ++dx) {
                if (abs(dx) + abs(dy) + abs(dz) > 2) continue;
                if (off) {
                    off[n][0] = dx;
                    off[n][1] = dy;
                    off[n][2] = dz;
                }
                ++n;
            }
    return n;
}

// z chunks for a z-marching kernel: minimise waves x (planes per chunk + the
// pipeline start-up), given the resident CTAs per SM of the kernel
static int choose_zchunks(int tiles, int nz, int per_sm, int sms, double startup)
{
    const long long slots = (long long)per_sm * sms;
    int best = 1;
    double best_cost = 1e300;
    // chunks of at least 2 planes (the start-up reads planes up to zb + 3)
    for (int c = 1; c <= (nz >= 4 ? nz / 2 : 1); ++c) {
        const long long items = (long long)tiles * c;
        const long long waves = (items + slots - 1) / slots;
        const double cost = (double)waves * ((double)nz / c + startup);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = c;
        }
    }
    return best;
}

template <int MINB, bool PER, bool RW, int ORDER, int TY = 8>
static acch_status launch_residual_zm_t(acch_ctx *ctx, const double *x_old, double dt, const double *x, double *F)
{
    constexpr int TX = 32;
    using L = RzmSmem<TX, TY>;
    constexpr int NTA = TX * TY + (RW ? 32 * ((L::NRING + 31) / 32) : 0);
    auto kern = res_zm_kernel<TX, TY, MINB, PER, RW, ORDER>;
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        acch_status st = set_smem(kern, L::bytes);
        if (st != ACCH_OK) return st;
        ACCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTA, L::bytes));
        ACCH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        if (per_sm < 1) per_sm = 1;
    }
    const GridDev &g = ctx->g;
    const int gx = (g.nx + TX - 1) / TX, gy = (g.ny + TY - 1) / TY;
    const int nchunk = choose_zchunks(gx * gy, g.nz, per_sm, sms, 3.0);
    kern<<<dim3(gx, gy, nchunk), dim3(NTA), L::bytes, ctx->stream>>>(
        g, ctx->p, dt, (const double2 *)x_old, (const double2 *)x, (double2 *)F, ctx->d_partials, ctx->d_counter,
        ctx->d_result, nchunk);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_residual(acch_ctx *ctx, const double *x_old, double dt, const double *x, double *F)
{
    ProfScope prof_scope(ctx, PC_RESIDUAL, 48.0 * ctx->g.n);
    const GridDev &g = ctx->g;
    // ACCH_RESIDUAL=ring selects the older 2-barrier kernel (tests compare both)
    const char *mode = getenv("ACCH_RESIDUAL");
    const bool zm = g.dim == 3 && g.nz >= 3 && !(mode && strcmp(mode, "ring") == 0);
    if (zm) {
        // ring warps (every thread one column, measured fastest); the
        // reference's default series order 10 compiled in
        if (ctx->p.order == 10) {
            // 32x16 tiles (3 ring warps, no idle lanes; 608 threads, one CTA
            // per SM): 0.500 vs 0.511 ms for 32x8 at 256^3
            if (g.periodic) return launch_residual_zm_t<1, true, true, 10, 16>(ctx, x_old, dt, x, F);
            return launch_residual_zm_t<1, false, true, 10, 16>(ctx, x_old, dt, x, F);
        }
        if (g.periodic) return launch_residual_zm_t<2, true, true, 0>(ctx, x_old, dt, x, F);
        return launch_residual_zm_t<2, false, true, 0>(ctx, x_old, dt, x, F);
    }
    const dim3 block(RTX, RTY);
    if (g.dim == 3) {
        using L = ResidualSmem<3, RTX, RTY>;
        static bool configured = false;
        if (!configured) {
            acch_status st = set_smem(residual_kernel<3, RTX, RTY>, L::bytes);
            if (st != ACCH_OK) return st;
            configured = true;
        }
        const dim3 grid((g.nx + RTX - 1) / RTX, (g.ny + RTY - 1) / RTY, (g.nz + ZCHUNK - 1) / ZCHUNK);
        residual_kernel<3, RTX, RTY><<<grid, block, L::bytes, ctx->stream>>>(
            g, ctx->p, dt, (const double2 *)x_old, (const double2 *)x, (double2 *)F, ctx->d_partials,
            ctx->d_counter, ctx->d_result);
    } else {
        using L = ResidualSmem<2, RTX, RTY>;
        const dim3 grid((g.nx + RTX - 1) / RTX, (g.ny + RTY - 1) / RTY, 1);
        residual_kernel<2, RTX, RTY><<<grid, block, L::bytes, ctx->stream>>>(
            g, ctx->p, dt, (const double2 *)x_old, (const double2 *)x, (double2 *)F, ctx->d_partials,
            ctx->d_counter, ctx->d_result);
    }
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_jacobian_prepare(acch_ctx *ctx, const double *x_old, double dt, const double *x, double *coef)
{
    ProfScope prof_scope(ctx, PC_JPREP, 88.0 * ctx->g.n);
    (void)dt;
    const long long n = ctx->g.n;
    jac_prepare_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->g, ctx->p, (const double2 *)x_old,
                                                                          (const double2 *)x, coef);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

static acch_status launch_matvec_twopass(acch_ctx *ctx, const double *coef, double dt, const double *w, double *y)
{
    if (!ctx->d_mvtmp) ACCH_CUDA(cudaMalloc(&ctx->d_mvtmp, sizeof(double) * 2 * ctx->g.nstore));
    const GridDev &g = ctx->g;
    const int zlo = (g.zg && !g.zwall_lo) ? -1 : 0, zhi = g.nz + ((g.zg && !g.zwall_hi) ? 1 : 0);
    const dim3 blk(PTX, PTY);
    const dim3 g1((g.nx + PTX - 1) / PTX, (g.ny + PTY - 1) / PTY, g.dim == 3 ? zhi - zlo : 1);
    const dim3 g2((g.nx + PTX - 1) / PTX, (g.ny + PTY - 1) / PTY, g.dim == 3 ? g.nz : 1);
    if (g.dim == 3) {
        mv_pass1_kernel<3><<<g1, blk, 0, ctx->stream>>>(g, ctx->p, coef, (const double2 *)w, (double2 *)ctx->d_mvtmp,
                                                        zlo);
        mv_pass2_kernel<3><<<g2, blk, 0, ctx->stream>>>(g, ctx->p, dt, coef, (const double2 *)w,
                                                        (const double2 *)ctx->d_mvtmp, (double2 *)y);
    } else {
        mv_pass1_kernel<2><<<g1, blk, 0, ctx->stream>>>(g, ctx->p, coef, (const double2 *)w, (double2 *)ctx->d_mvtmp,
                                                        0);
        mv_pass2_kernel<2><<<g2, blk, 0, ctx->stream>>>(g, ctx->p, dt, coef, (const double2 *)w,
                                                        (const double2 *)ctx->d_mvtmp, (double2 *)y);
    }
    ctx->launches += 1;
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

template <int MINB, bool PER, bool RW, int TX = 32, int TY = 8>
static acch_status launch_matvec_zm_t(acch_ctx *ctx, const double *coef, double dt, const double *w, double *y)
{
    using L = ZmSmem<TX, TY>;
    constexpr int NTA = TX * TY + (RW ? 32 * ((L::NRING + 31) / 32) : 0);
    auto kern = mv_zm_kernel<TX, TY, MINB, PER, RW>;
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        acch_status st = set_smem(kern, L::bytes);
        if (st != ACCH_OK) return st;
        ACCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTA, L::bytes));
        ACCH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        if (per_sm < 1) per_sm = 1;
    }
    const GridDev &g = ctx->g;
    const int gx = (g.nx + TX - 1) / TX, gy = (g.ny + TY - 1) / TY;
    const int nchunk = choose_zchunks(gx * gy, g.nz, per_sm, sms, 3.0);
    MvConst mc;
    mc.A = co_A(coef);
    mc.B = co_B(coef, g.nstore);
    mc.Gv = co_Gv(coef, g.nstore);
    mc.ihx = g.ih2[0];
    mc.ihy = g.ih2[1];
    mc.ihz = g.ih2[2];
    mc.fhx = 0.5 * g.ih2[0];
    mc.fhy = 0.5 * g.ih2[1];
    mc.fhz = 0.5 * g.ih2[2];
    mc.hg = 0.5 * ctx->p.gamma;
    mc.ha = -0.5 * ctx->p.alpha;
    mc.hb = -0.5 * ctx->p.beta;
    mc.idt = 1.0 / dt;
    mc.irho = 1.0 / ctx->p.rho;
    kern<<<dim3(gx, gy, nchunk), dim3(NTA), L::bytes, ctx->stream>>>(g, mc, (const double2 *)w, (double2 *)y, nchunk);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

static acch_status launch_matvec_zm(acch_ctx *ctx, const double *coef, double dt, const double *w, double *y)
{
    return ctx->g.periodic ? launch_matvec_zm_t<2, true, false>(ctx, coef, dt, w, y)
                           : launch_matvec_zm_t<2, false, false>(ctx, coef, dt, w, y);
}

acch_status launch_matvec(acch_ctx *ctx, const double *coef, double dt, const double *w, double *y)
{
    // 3D: the z-marching one-barrier kernel (nz >= 3); 2D: the two-pass form.
    // ACCH_MATVEC = zm | twopass selects a form (read per call, so the tests
    // exercise both on one context)
    const char *mode = getenv("ACCH_MATVEC");
    int m = ctx->g.dim == 3 ? 2 : 1;
    if (mode && strcmp(mode, "twopass") == 0) m = 1;
    if (mode && strcmp(mode, "zm") == 0 && ctx->g.dim == 3) m = 2;
    if (m == 2 && ctx->g.nz < 3) m = 1;   // the z-marching kernel's plane map assumes nz >= 3
    ctx->matvec_mode = m;
    ProfScope prof_scope(ctx, PC_MATVEC, 88.0 * ctx->g.n);
    if (m == 2) return launch_matvec_zm(ctx, coef, dt, w, y);
    return launch_matvec_twopass(ctx, coef, dt, w, y);
}

acch_status launch_jacobian_blocks(acch_ctx *ctx, const double *coef, double dt, double *out)
{
    ProfScope prof_scope(ctx, PC_JPREP, (56.0 + 32.0 * stencil_offsets(ctx->g.dim, nullptr)) * ctx->g.n);
    const int noff = stencil_offsets(ctx->g.dim, nullptr);
    const long long n = ctx->g.n;
    if (ctx->g.dim == 3)
        jac_blocks_kernel<3><<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(ctx->g, ctx->p, dt, coef, out, noff);
    else
        jac_blocks_kernel<2><<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(ctx->g, ctx->p, dt, coef, out, noff);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_chord(acch_ctx *ctx, const double *a, const double *b, long long n, int force_exact, double *val,
                         double *der)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 24.0 * n);
    if (n <= 0) return ACCH_OK;
    chord_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->p, a, b, n, force_exact, val, der);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_gap(acch_ctx *ctx, const double *x)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 16.0 * ctx->g.n);
    const long long n = ctx->g.n;
    gap_kernel<<<red_grid(n), kRedThreads, 0, ctx->stream>>>(n, (const double2 *)x + ctx->g.zoff, ctx->d_partials, ctx->d_counter,
                                                            ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

// gap over n arbitrary interleaved (u, v) pairs (the reference's
// admissibility_gap(u, v) on plain arrays, physics.py:89-109)
acch_status launch_gap_pairs(acch_ctx *ctx, const double *x, long long n)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 16.0 * n);
    gap_kernel<<<red_grid(n), kRedThreads, 0, ctx->stream>>>(n, (const double2 *)x, ctx->d_partials, ctx->d_counter,
                                                            ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_diagnostics(acch_ctx *ctx, const double *x)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 16.0 * ctx->g.n);
    diagnostics_kernel<<<red_grid(ctx->g.n), kRedThreads, 0, ctx->stream>>>(ctx->g, ctx->p, (const double2 *)x,
                                                                           ctx->d_partials, ctx->d_counter,
                                                                           ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_trial(acch_ctx *ctx, const double *x, const double *s, double lam, double *y)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 48.0 * ctx->g.n);
    const long long n = ctx->g.n;
    trial_kernel<<<red_grid(n), kRedThreads, 0, ctx->stream>>>(n, (const double2 *)x + ctx->g.zoff,
                                                              (const double2 *)s + ctx->g.zoff, lam,
                                                              (double2 *)y + ctx->g.zoff, ctx->d_partials, ctx->d_counter,
                                                              ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_feasible_cap(acch_ctx *ctx, const double *x, const double *s, double margin)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 32.0 * ctx->g.n);
    const long long n = ctx->g.n;
    feasible_cap_kernel<<<red_grid(n), kRedThreads, 0, ctx->stream>>>(n, (const double2 *)x + ctx->g.zoff,
                                                                     (const double2 *)s + ctx->g.zoff, margin,
                                                                     ctx->d_partials, ctx->d_counter, ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

acch_status launch_rms_diff(acch_ctx *ctx, const double *a, const double *b, long long n)
{
    ProfScope prof_scope(ctx, PC_REDUCE, 16.0 * n);
    rms_diff_kernel<<<red_grid(n), kRedThreads, 0, ctx->stream>>>(n, a, b, ctx->d_partials, ctx->d_counter,
                                                                 ctx->d_result);
    ACCH_LAUNCHED(ctx);
    return ACCH_OK;
}

