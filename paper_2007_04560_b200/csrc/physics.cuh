// Per-cell constitutive functions (device).  Formulas and branch predicates
// follow /root/reference/pkg/src/acch/physics.py line by line so that branch
// choices agree bitwise with the reference and values agree to a few ulps.
#pragma once

#include "acch_internal.cuh"

// mobility c(u, v) = u (1 - u) (1/4 - v^2)           (physics.py:124-130)
__device__ __forceinline__ double mobility(double u, double v)
{
    return u * (1.0 - u) * (0.25 - v * v);
}

// Phi(z) = z ln z + (1 - z) ln(1 - z)                (physics.py:160-166)
__device__ __forceinline__ double entropy(double z)
{
    return z * log(z) + (1.0 - z) * log1p(-z);
}

// Divided difference (Phi(a) - Phi(b)) / (a - b) and, with DER, d/da.
// zeta = (a+b)/2, sigma = (a-b)/2 computed exactly as physics.py:240-242;
// exact branch when sigma == 0, midpoint series when
// |sigma| <= 0.4 min(zeta, 1 - zeta) (physics.py:193-200), direct quotient
// otherwise (physics.py:259-261, 303-307).  Horner as physics.py:185-190.
template <bool DER>
__device__ __forceinline__ void entropy_chord(double a, double b, const ParamsDev &P, int force_exact,
                                              double &val, double &der)
{
    const double zeta = 0.5 * (a + b);
    const double sigma = 0.5 * (a - b);
    const double w = 1.0 - zeta;
    if (sigma == 0.0) {
        val = log(zeta) - log1p(-zeta);
        if (DER) der = 0.5 * (1.0 / zeta + 1.0 / w);
        return;
    }
    if (!force_exact && fabs(sigma) <= 0.4 * fmin(zeta, w)) {
        const double rz = sigma / zeta, rw = sigma / w;
        const double tz = rz * rz, tw = rw * rw;
        double pz = 0.0, pw = 0.0;
        for (int s = P.order - 1; s >= 0; --s) {
            pz = (pz + P.c1[s]) * tz;
            pw = (pw + P.c1[s]) * tw;
        }
        val = log(zeta) - log1p(-zeta) - pz + pw;
        if (DER) {
            double qz = 0.0, qw = 0.0;
            for (int s = P.order - 1; s >= 0; --s) {
                qz = (qz + P.c2[s]) * tz;
                qw = (qw + P.c2[s]) * tw;
            }
            der = 0.5 * ((1.0 + qz) / zeta + (-qz / sigma) + (1.0 + qw) / w - (-qw / sigma));
        }
        return;
    }
    const double ch = (entropy(a) - entropy(b)) / (a - b);
    val = ch;
    if (DER) der = ((log(a) - log1p(-a)) - ch) / (a - b);
}

// smallest distance from the admissible-set boundary (physics.py:89-109)
__device__ __forceinline__ double cell_gap(double u, double v)
{
    const double p = u + v, q = u - v;
    double g = u;
    g = fmin(g, 1.0 - u);
    g = fmin(g, p);
    g = fmin(g, 1.0 - p);
    g = fmin(g, q);
    g = fmin(g, 1.0 - q);
    g = fmin(g, 0.5 - v);
    g = fmin(g, 0.5 + v);
    // any NaN input makes the state inadmissible (physics.py:107-108)
    if (isnan(u) || isnan(v)) g = NAN;
    return g;
}

__device__ __forceinline__ int wrap_coord(int i, int n, int periodic)
{
    if (periodic) {
        // stencil and box offsets stay within one period: two compares, the
        // integer division only for a (never seen) farther offset
        i = i < 0 ? i + n : (i >= n ? i - n : i);
        if ((unsigned)i >= (unsigned)n) i = ((i % n) + n) % n;
        return i;
    }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// storage plane of local z-plane z (z may reach zg planes past either end)
__device__ __forceinline__ int zplane(const GridDev &g, int z)
{
    if (g.zg == 0) return wrap_coord(z, g.nz, g.periodic);
    if (z < 0 && g.zwall_lo) z = 0;
    if (z >= g.nz && g.zwall_hi) z = g.nz - 1;
    return z + g.zg;
}

// zplane() for -nz <= z < 2 nz without integer division (z-marching kernels)
__device__ __forceinline__ int zplane_near(const GridDev &g, int z)
{
    if (g.zg == 0) {
        if (z < 0) return g.periodic ? z + g.nz : 0;
        if (z >= g.nz) return g.periodic ? z - g.nz : g.nz - 1;
        return z;
    }
    if (z < 0 && g.zwall_lo) z = 0;
    if (z >= g.nz && g.zwall_hi) z = g.nz - 1;
    return z + g.zg;
}

// can a stencil step from local plane z to z + s (no physical wall crossed)?
__device__ __forceinline__ bool zstep_ok(const GridDev &g, int z, int s)
{
    const int t = z + s;
    if (g.zg == 0) return g.periodic || (t >= 0 && t < g.nz);
    return !((t < 0 && g.zwall_lo) || (t >= g.nz && g.zwall_hi));
}

__device__ __forceinline__ long long cell_at(const GridDev &g, int x, int y, int zs)
{
    return ((long long)zs * g.ny + y) * g.nx + x;
}
