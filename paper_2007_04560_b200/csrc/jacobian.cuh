// Explicit 2x2 blocks of one row of the step Jacobian on the radius-2
// stencil, evaluated from the 7 coefficient planes.  Shared by the
// jac_blocks kernel (stencil.cu) and the subdomain factorisation (schwarz.cu).
//
// Derivation (row cell c, neighbours n of c, m in {c} U N(c)):
//   u row:  w_u/dt - sum_n K_n (dG(n) - dG(c)) - sum_n (G(n) - G(c))/h^2 (eta(c) + eta(n))/2
//     K_n = cbar_face(c, n)/h^2, dG(m) = A(m) w_u(m) + D(m) w_v(m) - gamma/2 sum_p w_u(p)/h_p^2,
//     A(m) = -alpha/2 + S(m) + gamma/2 sum_p 1/h_p^2, eta(m) = (c_u w_u + c_v w_v)(m)/2;
//   v row:  w_v/dt + cbar/rho (D w_u + (-beta/2 + S) w_v - gamma/2 lap w_v) + G_v/rho eta(c).
// This is the operator scheme.py:471-482 assembles (data[...] updates), with
// Neumann walls dropping the links divgrad_csr drops (scheme.py:112-130).
#pragma once

#include "acch_internal.cuh"
#include "physics.cuh"

// offset id of (dx, dy, dz) in the fixed order of stencil_offsets(): dz, dy, dx
// ascending over |dx|+|dy|+|dz| <= 2; -1 outside
static __constant__ int c_off3[125] = {
-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,0,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,1,-1,-1,-1,2,3,4,-1,-1,-1,5,-1,-1,-1,-1,-1,-1,-1,-1,-1,6,-1,-1,-1,7,8,9,-1,10,11,12,13,14,-1,15,16,17,-1,-1,-1,18,-1,-1,-1,-1,-1,-1,-1,-1,-1,19,-1,-1,-1,20,21,22,-1,-1,-1,23,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,24,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1};
static __constant__ int c_off2[25] = {-1,-1,0,-1,-1,-1,1,2,3,-1,4,5,6,7,8,-1,9,10,11,-1,-1,-1,12,-1,-1};

template <int DIM>
__device__ __forceinline__ int stencil_offset_id(int dx, int dy, int dz)
{
    if (DIM == 3) return c_off3[(dx + 2) + 5 * (dy + 2) + 25 * (dz + 2)];
    return c_off2[(dx + 2) + 5 * (dy + 2)];
}


// The row's contributions in a fixed order: emit(o, comp, value) adds value
// to component comp (0 uu, 1 uv, 2 vu, 3 vv) of the block at stencil offset o.
template <int DIM, typename Emit>
__device__ __forceinline__ void jac_row_emit(const GridDev &g, const ParamsDev &P, double dt, const double *__restrict__ coef,
                                             int x, int y, int z, Emit &&emit)
{
    // x, y wrap or clamp; z stays a raw local plane index (it may address a
    // slab ghost plane) and is mapped to storage by zplane()
    const long long N = g.nstore;
    const int cc[3] = {x, y, z};
    const int nn[3] = {g.nx, g.ny, g.nz};
    auto cid = [&](const int (&q)[3]) -> long long { return cell_at(g, q[0], q[1], zplane(g, q[2])); };
    auto offid = [&](int dx, int dy, int dz) { return stencil_offset_id<DIM>(dx, dy, dz); };
    // neighbour m = c + e_a s exists (periodic, inside the box, or across a slab boundary)
    auto valid = [&](const int (&q)[3], int a, int s) {
        if (a == 2) return zstep_ok(g, q[2], s);
        if (g.periodic) return true;
        const int t = q[a] + s;
        return t >= 0 && t < nn[a];
    };
    auto shifted = [&](const int (&q)[3], int a, int s, int (&r)[3]) {
        r[0] = q[0]; r[1] = q[1]; r[2] = q[2];
        r[a] = a == 2 ? q[a] + s : wrap_coord(q[a] + s, nn[a], g.periodic);
    };
    // a cell's coefficients come as two vector loads: A = (S, D, c_u, c_v), B = (cbar, G_u)
    const double4 *__restrict__ cA = co_A(coef);
    const double2 *__restrict__ cB = co_B(coef, N);
    const long long c0 = cid(cc);
    const double2 b0 = cB[c0];
    const double4 a0 = ldg256(cA + c0);
    const double cb0 = b0.x, gu0 = b0.y;
    // weights of dG_u(m) and eta(m) in row c of the u equation
    double wdg[7], weta[7];
    int mo[3 * 7];   // relative offsets of m
    int nm = 0;
    double ktot = 0.0, eta0 = 0.0;
    mo[0] = mo[1] = mo[2] = 0;
    nm = 1;
    for (int a = 0; a < g.dim; ++a) {
        for (int s = -1; s <= 1; s += 2) {
            if (!valid(cc, a, s)) continue;
            int q[3];
            shifted(cc, a, s, q);
            const long long cn = cid(q);
            const double2 bn = cB[cn];
            const double K = 0.5 * (cb0 + bn.x) * g.ih2[a];
            const double dGn = bn.y - gu0;
            ktot += K;
            wdg[nm] = -K;
            weta[nm] = -0.5 * dGn * g.ih2[a];
            eta0 += -0.5 * dGn * g.ih2[a];
            mo[3 * nm + 0] = a == 0 ? s : 0;
            mo[3 * nm + 1] = a == 1 ? s : 0;
            mo[3 * nm + 2] = a == 2 ? s : 0;
            ++nm;
        }
    }
    wdg[0] = ktot;
    weta[0] = eta0;
    const double hg = 0.5 * P.gamma;
    for (int j = 0; j < nm; ++j) {
        int q[3] = {cc[0], cc[1], cc[2]};
        for (int a = 0; a < 2; ++a)
            if (mo[3 * j + a] != 0) q[a] = wrap_coord(cc[a] + mo[3 * j + a], nn[a], g.periodic);
        q[2] = cc[2] + mo[3 * j + 2];
        const long long cm = cid(q);
        double lsum = 0.0;   // sum of 1/h^2 over valid neighbours of m
        for (int a = 0; a < g.dim; ++a) {
            for (int s = -1; s <= 1; s += 2) {
                if (!valid(q, a, s)) continue;
                lsum += g.ih2[a];
                const int o = offid(mo[3 * j] + (a == 0 ? s : 0), mo[3 * j + 1] + (a == 1 ? s : 0),
                                    mo[3 * j + 2] + (a == 2 ? s : 0));
                emit(o, 0, -wdg[j] * hg * g.ih2[a]);
            }
        }
        const int om = offid(mo[3 * j], mo[3 * j + 1], mo[3 * j + 2]);
        const double4 am = j == 0 ? a0 : ldg256(cA + cm);
        const double A = -0.5 * P.alpha + am.x + hg * lsum;
        emit(om, 0, wdg[j] * A + weta[j] * 0.5 * am.z);
        emit(om, 1, wdg[j] * am.y + weta[j] * 0.5 * am.w);
    }
    const int o0 = offid(0, 0, 0);
    emit(o0, 0, 1.0 / dt);
    // v row
    const double cr = cb0 / P.rho;
    const double S0 = a0.x, D0 = a0.y, Gv0 = co_Gv(coef, N)[c0];
    double lsum0 = 0.0;
    for (int a = 0; a < g.dim; ++a) {
        for (int s = -1; s <= 1; s += 2) {
            if (!valid(cc, a, s)) continue;
            lsum0 += g.ih2[a];
            const int o = offid(a == 0 ? s : 0, a == 1 ? s : 0, a == 2 ? s : 0);
            emit(o, 3, -hg * cr * g.ih2[a]);
        }
    }
    emit(o0, 2, cr * D0 + Gv0 * a0.z / (2.0 * P.rho));
    emit(o0, 3, 1.0 / dt + cr * (-0.5 * P.beta + S0) + hg * cr * lsum0 + Gv0 * a0.w / (2.0 * P.rho));
}

template <int DIM>
__device__ __forceinline__ void jac_row_blocks(const GridDev &g, const ParamsDev &P, double dt, const double *__restrict__ coef,
                               int x, int y, int z, double (*blk)[4], int noff)
{
    for (int o = 0; o < noff; ++o) blk[o][0] = blk[o][1] = blk[o][2] = blk[o][3] = 0.0;
    jac_row_emit<DIM>(g, P, dt, coef, x, y, z, [&](int o, int c, double v) { blk[o][c] += v; });
}

