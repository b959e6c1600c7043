// Restricted additive Schwarz preconditioner with ILU(k) / exact LU subdomain
// solves on sm_100a (linalg.py:217-396, _ilu.py).
//
// Host (native C++, once per preconditioner):
//   * every subdomain's extended box is the owned box grown by `overlap`,
//     wrapped (periodic) or clipped (Neumann) per axis (linalg.py:185-199);
//     its local cell order is the sorted global ids (linalg.py:200-206);
//   * subdomains whose per-axis relative coordinate lists coincide share one
//     "class": block pattern (the radius-2 skeleton restricted to the box,
//     scheme.py:166-188 + restrict_cells linalg.py:71-89), level-of-fill
//     pattern (_ilu.py:19-64), J-stencil -> pattern map, IKJ update lists and
//     forward/backward level schedules.  A periodic grid of equal boxes has at
//     most 3^dim classes whatever its size.
// Device:
//   * factor_kernel: one CTA per subdomain assembles its rows of J directly
//     from the 7 coefficient planes (no global Jacobian is ever stored),
//     then runs block-IKJ ILU level by level.  2x2 blocks with an inverted
//     diagonal block reproduce the reference's scalar ILU on kron(P, 1_2x2)
//     (_ilu.py:67-120) up to rounding; the zero-pivot test is the scalar one
//     (|pivot| < 1e-300, reported as the first bad scalar row).
//   * apply_kernel: one CTA per subdomain gathers r on its extended box into
//     shared memory, runs the level-scheduled forward / backward sweeps and
//     scatters (left-RAS: owned cells straight to z; ASM / right-RAS: to a
//     per-subdomain buffer that gather_kernel sums per cell in subdomain
//     order -- the reference's fixed combination order, linalg.py:389-396).
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <unordered_map>
#include <vector>

#include "acch_internal.cuh"
#include "jacobian.cuh"
#include "physics.cuh"

namespace {

constexpr int kFactorThreads = 128;
constexpr int kApplyThreads = 128;

struct ClassDev {
    int nloc, nnzb, nlev, nlevb, ell_total, max_fwidth, max_bwidth;
    int len[3];
    const int *rel[3];
    const int *rowptr, *col, *diag;
    const int *pos;         // CSR entry -> slot in the per-subdomain level-major value array
    const int *jmap;        // nloc * noff -> slot (or -1)
    const int *upd_ptr;     // nnzb + 1 (indexed by CSR entry)
    const int2 *upd;        // (src slot, dst slot)
    const int *lev_ptr, *lev_rows, *levb_ptr, *levb_rows;
    // level-major ("ELL per level") solve layout: slot(level, t, q) = base[level] + t * m + q
    const int *f_base, *f_len, *b_base, *b_len;   // f_len/b_len indexed like lev_rows/levb_rows
    const int *ecol;        // local column of every slot (-1 = padding)
    const unsigned char *owned;
    const int *f_jptr, *f_joff, *b_jptr, *b_joff;   // per-level jagged-diagonal offsets
    // compact copies for staging into shared memory by the warp solver
    const unsigned short *f_rows16, *b_rows16;
    const unsigned short *f_len8, *b_len8;   // row lengths (slots) in level order
    // the class-group solver's shared-memory image (byte offsets into meta):
    // f_ptr | f_base | b_ptr | b_base (int) | f_rows | b_rows | f_len | b_len | ecol (uint16)
    const unsigned char *meta;
    const int *lin;   // local cell -> storage offset from the box origin (boxes that do not wrap)
    const int *own_list;   // local ids of the owned cells, ascending
    int n_owned;
    // left RAS keeps only the owned rows: a backward row i < b_min_row (the
    // first owned local row) feeds no owned row (row i reads rows j > i only),
    // so its sweep is skipped, and backward levels >= nlevb_ras hold only
    // such rows
    int b_min_row, nlevb_ras;
    int meta_bytes, m_fbs, m_bptr, m_bbs, m_frows, m_brows, m_flen, m_blen, m_ecol, m_fjp, m_bjp, m_fjo, m_bjo;
    int m_lin, m_ixyz, m_own, m_rel;   // gather / scatter tables in the group image
    int jdup;   // some row has two stencil entries on one pattern position (tiny periodic axes)
    int prezero;   // some slot receives no J entry (fill) or J entries are accumulated (jdup): zero before assembly
    // column-major layout of a narrow class (apply_cols_kernel): step words
    // (forward steps, then backward), row index of every slot, first backward slot
    const unsigned *col_steps;
    const unsigned short *col_ridx;
    int col_nf, col_nb, col_nb_ras, col_bstart, col_end, col_end_ras;
};

struct ClassHost {
    std::array<std::vector<int>, 3> rel;
    int own_len[3];
    std::vector<int> rowptr, col, diag, pos, jmap, upd_ptr, lev_ptr, lev_rows, levb_ptr, levb_rows;
    std::vector<int> f_base, f_len, b_base, b_len, ecol, f_jptr, f_joff, b_jptr, b_joff;
    std::vector<unsigned short> f_rows16, b_rows16;
    std::vector<unsigned short> f_len8, b_len8;
    std::vector<int2> upd;
    std::vector<unsigned char> owned;
    std::vector<int> jmap_csr;          // jmap / upd by CSR entry (before the slot layout is applied)
    std::vector<int2> upd_csr;
    std::vector<unsigned> col_steps;
    std::vector<unsigned short> col_ridx;
    int col_nf = 0, col_nb = 0, col_nb_ras = 0, col_bstart = 0, col_end = 0, col_end_ras = 0;
    std::vector<unsigned char> meta;   // ClassDev::meta image
    std::vector<int> lin, own_list;
    int jdup = 0;
    int prezero = 1;
    int b_min_row = 0, nlevb_ras = 0;
    long long skip_blocks = 0;   // factor blocks of the backward rows below b_min_row
    int m_off[17] = {0};
    int nloc = 0, nnzb = 0, ell_total = 0, max_fwidth = 0, max_bwidth = 0;
    void *dev_mem = nullptr;
    ClassDev dev;
};

__device__ __forceinline__ void local_to_global(const GridDev &g, const ClassDev &C, const int4 &o, int l, int &gx,
                                                int &gy, int &gz)
{
    const int ix = l % C.len[0];
    const int iy = (l / C.len[0]) % C.len[1];
    const int iz = l / (C.len[0] * C.len[1]);
    gx = wrap_coord(o.x + C.rel[0][ix], g.nx, g.periodic);
    gy = wrap_coord(o.y + C.rel[1][iy], g.ny, g.periodic);
    // z: wrapped local plane for a whole-grid domain; in slab mode a raw local
    // plane that may lie in a ghost plane (overlap into the neighbour slab)
    gz = g.dim == 3 ? (g.zg ? o.z + C.rel[2][iz] : wrap_coord(o.z + C.rel[2][iz], g.nz, g.periodic)) : 0;
}

struct Blk {
    double a, b, c, d;   // [[a, b], [c, d]]
};

// a subdomain's factor slots: slot p at base[p * stride]
struct StridedBlocks {
    double4 *base;
    int stride;
    __device__ __forceinline__ double4 &operator[](long long p) const { return base[p * stride]; }
};

__device__ __forceinline__ Blk mul(const Blk &x, const Blk &y)
{
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}

#ifndef ACCH_FACTOR_MINB
#define ACCH_FACTOR_MINB 8
#endif
template <int DIM, int NT = kFactorThreads>
__global__ void __launch_bounds__(NT, ACCH_FACTOR_MINB * kFactorThreads / NT)
factor_kernel(GridDev g, ParamsDev P, double dt, const double *__restrict__ coef, const ClassDev *__restrict__ classes,
              const int *__restrict__ sub_class, const int4 *__restrict__ sub_origin,
              const long long *__restrict__ sub_off, double4 *__restrict__ vals, int *__restrict__ bad_row, int ss)
{
    // slot p of this subdomain lives at A[p * ss] (ss = 8: row-sequential batches)
    constexpr int NOFF = DIM == 3 ? 25 : 13;
    const int s = blockIdx.x;
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    StridedBlocks A{vals + sub_off[s], ss};
    const int tid = threadIdx.x, nt = blockDim.x;
    // ILU(0) without folded stencil entries: the assembly writes every slot of the
    // pattern (the padding slots were cleared at creation and are never written)
    if (C.prezero) {
        for (int t = tid; t < C.ell_total; t += nt) A[t] = make_double4(0.0, 0.0, 0.0, 0.0);
        __syncthreads();
    }
    for (int l = tid; l < C.nloc; l += nt) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double blk[NOFF][4];
        jac_row_blocks<DIM>(g, P, dt, coef, gx, gy, gz, blk, NOFF);
        // when every stencil entry of a row has its own pattern position (all
        // but tiny periodic axes, where +-2 wrap onto one cell) the blocks are
        // stored, not accumulated: no read of the zeroed slots
        for (int q = 0; q < NOFF; ++q) {
            const int p = C.jmap[l * NOFF + q];
            if (p < 0) continue;
            if (!C.jdup) {
                A[p] = make_double4(0.0 + blk[q][0], 0.0 + blk[q][1], 0.0 + blk[q][2], 0.0 + blk[q][3]);
            } else {
                double4 v = A[p];
                v.x += blk[q][0];
                v.y += blk[q][1];
                v.z += blk[q][2];
                v.w += blk[q][3];
                A[p] = v;
            }
        }
    }
    __syncthreads();
    // diagonal block of a finished row: scalar pivots as the reference's
    // factor_inplace sees them, then the inverted block
    auto finish_diag = [&](int i, int d) {
        const int pd = C.pos[d];
        const double4 D = A[pd];
        const double p0 = D.x;
        const double p1 = D.w - (D.z / D.x) * D.y;
        int bad = -1;
        if (fabs(p0) < 1e-300) bad = 2 * i;
        else if (fabs(p1) < 1e-300) bad = 2 * i + 1;
        if (bad >= 0) atomicMin(bad_row + s, bad);
        const double det = D.x * D.w - D.y * D.z;
        A[pd] = make_double4(D.w / det, -D.y / det, -D.z / det, D.x / det);
    };
    // block IKJ elimination, level by level (rows of a level are independent)
    for (int lev = 0; lev < C.nlev; ++lev) {
        // narrow level of long rows (exact LU / ILU(k>=1) fill: <= 4 rows with
        // more than 16 pivots): the whole CTA eliminates one row at a time --
        // the updates of one pivot hit distinct targets, so they are spread
        // over the threads, with a barrier between pivots.  Every target sees
        // the same updates in the same pivot order as in the one-thread-per-row
        // loop below, so the factors are bitwise the same.
        {
            const int q0 = C.lev_ptr[lev], m = C.lev_ptr[lev + 1] - q0;
            const int i0 = C.lev_rows[q0];
            if (m <= 4 && C.diag[i0] - C.rowptr[i0] > 16) {
                for (int qq = 0; qq < m; ++qq) {
                    const int i = C.lev_rows[q0 + qq];
                    const int d = C.diag[i];
                    for (int t = C.rowptr[i]; t < d; ++t) {
                        const int k = C.col[t];
                        const int pt = C.pos[t];
                        const double4 ak = A[pt], dk = A[C.pos[C.diag[k]]];
                        const Blk L = mul({ak.x, ak.y, ak.z, ak.w}, {dk.x, dk.y, dk.z, dk.w});
                        __syncthreads();   // every thread has read A[pt]
                        if (tid == 0) A[pt] = make_double4(L.a, L.b, L.c, L.d);
                        const int u1 = C.upd_ptr[t + 1];
                        for (int u = C.upd_ptr[t] + tid; u < u1; u += nt) {
                            const int2 sd = C.upd[u];
                            const double4 us = A[sd.x];
                            double4 v = A[sd.y];
                            const Blk mm = mul(L, {us.x, us.y, us.z, us.w});
                            v.x -= mm.a;
                            v.y -= mm.b;
                            v.z -= mm.c;
                            v.w -= mm.d;
                            A[sd.y] = v;
                        }
                        __syncthreads();   // the next pivot reads its updated multiplier
                    }
                    if (tid == 0) finish_diag(i, d);
                    __syncthreads();
                }
                continue;
            }
        }
        for (int q = C.lev_ptr[lev] + tid; q < C.lev_ptr[lev + 1]; q += nt) {
            const int i = C.lev_rows[q];
            const int d = C.diag[i];
            for (int t = C.rowptr[i]; t < d; ++t) {
                const int k = C.col[t];
                const int pt = C.pos[t];
                const double4 ak = A[pt], dk = A[C.pos[C.diag[k]]];
                const Blk L = mul({ak.x, ak.y, ak.z, ak.w}, {dk.x, dk.y, dk.z, dk.w});
                A[pt] = make_double4(L.a, L.b, L.c, L.d);
                // the updates of one pivot touch distinct targets and read row
                // k's finished U blocks: batches of UB sources and targets are
                // loaded together (one L2 round trip per batch, not per update)
#ifndef ACCH_FACTOR_UB
#define ACCH_FACTOR_UB 2
#endif
                constexpr int UB = ACCH_FACTOR_UB;
                const int u1 = C.upd_ptr[t + 1];
                for (int u0 = C.upd_ptr[t]; u0 < u1; u0 += UB) {
                    int2 sd[UB];
                    double4 us[UB], v[UB];
#pragma unroll
                    for (int b = 0; b < UB; ++b) sd[b] = u0 + b < u1 ? C.upd[u0 + b] : make_int2(0, 0);
#pragma unroll
                    for (int b = 0; b < UB; ++b)
                        if (u0 + b < u1) {
                            us[b] = A[sd[b].x];
                            v[b] = A[sd[b].y];
                        }
#pragma unroll
                    for (int b = 0; b < UB; ++b)
                        if (u0 + b < u1) {
                            const Blk m = mul(L, {us[b].x, us[b].y, us[b].z, us[b].w});
                            v[b].x -= m.a;
                            v[b].y -= m.b;
                            v[b].z -= m.c;
                            v[b].w -= m.d;
                            A[sd[b].y] = v[b];
                        }
                }
            }
            finish_diag(i, d);
        }
        __syncthreads();
    }
}

template <int TPS>
__device__ __forceinline__ void level_sync()
{
    if (TPS == 32) __syncwarp();
    else __syncthreads();
}

// Bulk L2 prefetch (TMA engine, no registers or shared memory): the warp
// solver asks for the factor slots of the level D ahead while it works on the
// current one, so its own loads hit L2 instead of waiting on HBM.
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes)
{
    if (bytes >= 16) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15u) : "memory");
}

// one 256-bit read-only load (LDG.256, sm_100) per 2x2 factor block
__device__ __forceinline__ double4 ldg4(const double4 *p)
{
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}

// predicated LDG.256 into an in/out register quad: v keeps its old value when
// !pred, so the last load of a batch always defines v and can anchor a data
// dependency (see sweep_level)
// Factor slots are read exactly once per apply: the loads carry an
// L2::evict_first policy (and skip L1), so the dead lines they leave behind
// go before the levels the TMA engine has prefetched but not yet consumed.
// (v is left undefined when !pred; it is only read as a dependency anchor.)
__device__ __forceinline__ uint64_t evict_first_policy()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void ldg4_pred(double4 &v, const double4 *p, bool pred, uint64_t pol)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %6;\n\t}"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p), "r"((unsigned)pred), "l"(pol));
}

// A preconditioner whose longest factor row exceeds kWideLen blocks (exact LU,
// ILU(k >= 1)) runs the WIDE kernel instances.  There, a level of at most
// kWideRows rows whose longest row has more than kWideMin blocks -- past the
// lane-per-row sweep's MAXW slots in flight, where every extra block costs
// that sweep a round trip -- is swept warp-wide (sweep_level_wide): a single
// row by all 32 lanes, 2..8 rows together by groups of 16 / 8 / 4 lanes.
constexpr int kWideRows = 8, kWideLen = 32, kWideMin = 12;

__device__ __forceinline__ int anchor_bits(const double4 &a) { return __double2hiint(a.x); }

// acc -= a y for a 2x2 block, with the rounding pinned by intrinsics
// (product, fused second product, subtraction): every solver and code path
// gives bitwise the same result, whatever contraction the compiler would pick
__device__ __forceinline__ void blk_sub(double2 &acc, const double4 &a, const double2 &y)
{
    acc.x = __dsub_rn(acc.x, __fma_rn(a.y, y.y, __dmul_rn(a.x, y.x)));
    acc.y = __dsub_rn(acc.y, __fma_rn(a.w, y.y, __dmul_rn(a.z, y.x)));
}

template <int VARIANT, int TPS, int MAXW = 12>   // VARIANT: 0 asm, 1 ras-left, 2 ras-right
__global__ void __launch_bounds__(128, 3)
apply_kernel(GridDev g, const ClassDev *__restrict__ classes, const int *__restrict__ sub_class,
             const int4 *__restrict__ sub_origin, const long long *__restrict__ sub_off,
             const long long *__restrict__ sub_ext_off, const double4 *__restrict__ vals,
             const double2 *__restrict__ r, double2 *__restrict__ z, double2 *__restrict__ ext_out, int use_smem,
             int max_nloc, long long nsub)
{
    ACCH_SKIP_IF(g);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int group = threadIdx.x / TPS;               // subdomain slot within the CTA
    const int lane = threadIdx.x % TPS;
    const long long s = (long long)blockIdx.x * (blockDim.x / TPS) + group;
    if (s >= nsub) return;                             // whole group exits together
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    const double4 *__restrict__ A = vals + sub_off[s];
    double2 *y = use_smem ? reinterpret_cast<double2 *>(smem_raw) + (size_t)group * max_nloc
                          : ext_out + sub_ext_off[s];
    const long long nx = g.nx, ny = g.ny;
    for (int l = lane; l < C.nloc; l += TPS) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double2 v = r[cell_at(g, gx, gy, zplane(g, gz))];
        if (VARIANT == 2 && !C.owned[l]) v = make_double2(0.0, 0.0);
        y[l] = v;
    }
    level_sync<TPS>();
    // Each row's slots are fetched up front (MAXW loads in flight per lane), so a
    // level costs one global round trip; the y reads are shared-memory hits.
    for (int lev = 0; lev < C.nlev; ++lev) {
        const int r0 = C.lev_ptr[lev], m = C.lev_ptr[lev + 1] - r0, base = C.f_base[lev];
        const int *joff = C.f_joff + C.f_jptr[lev];
        for (int q = lane; q < m; q += TPS) {
            const int i = C.lev_rows[r0 + q];
            const int len = C.f_len[r0 + q];
            double2 acc = y[i];
            if (len <= MAXW) {
                double4 a[MAXW];
                int c[MAXW];
#pragma unroll
                for (int t = 0; t < MAXW; ++t) {
                    if (t < len) {
                        a[t] = ldg4(A + base + joff[t] + q);
                        c[t] = __ldg(C.ecol + base + joff[t] + q);
                    }
                }
#pragma unroll
                for (int t = 0; t < MAXW; ++t)
                    if (t < len) blk_sub(acc, a[t], y[c[t]]);
            } else {
                for (int t = 0; t < len; ++t) {
                    const int e = base + joff[t] + q;
                    blk_sub(acc, ldg4(A + e), y[__ldg(C.ecol + e)]);
                }
            }
            y[i] = acc;
        }
        level_sync<TPS>();
    }
    for (int lev = 0; lev < C.nlevb; ++lev) {
        const int r0 = C.levb_ptr[lev], m = C.levb_ptr[lev + 1] - r0, base = C.b_base[lev];
        const int *joff = C.b_joff + C.b_jptr[lev];
        for (int q = lane; q < m; q += TPS) {
            const int i = C.levb_rows[r0 + q];
            const int len = C.b_len[r0 + q];     // slot 0: inverted diagonal block
            double2 acc = y[i];
            const double4 di = ldg4(A + base + joff[0] + q);
            if (len <= MAXW + 1) {
                double4 a[MAXW];
                int c[MAXW];
#pragma unroll
                for (int t = 0; t < MAXW; ++t) {
                    if (t + 1 < len) {
                        a[t] = ldg4(A + base + joff[t + 1] + q);
                        c[t] = __ldg(C.ecol + base + joff[t + 1] + q);
                    }
                }
#pragma unroll
                for (int t = 0; t < MAXW; ++t)
                    if (t + 1 < len) blk_sub(acc, a[t], y[c[t]]);
            } else {
                for (int t = 1; t < len; ++t) {
                    const int e = base + joff[t] + q;
                    blk_sub(acc, ldg4(A + e), y[__ldg(C.ecol + e)]);
                }
            }
            y[i] = make_double2(di.x * acc.x + di.y * acc.y, di.z * acc.x + di.w * acc.y);
        }
        level_sync<TPS>();
    }
    if (VARIANT == 1) {
        for (int l = lane; l < C.nloc; l += TPS) {
            if (!C.owned[l]) continue;
            int gx, gy, gz;
            local_to_global(g, C, o, l, gx, gy, gz);
            z[cell_at(g, gx, gy, zplane(g, gz))] = y[l];
        }
    } else if (use_smem) {
        for (int l = lane; l < C.nloc; l += TPS) ext_out[sub_ext_off[s] + l] = y[l];
    }
}

// Narrow level (<= kWideRows rows) with long rows (exact LU / ILU(k >= 1)
// fill): the level's rows are swept TOGETHER, each by its own group of
// G = 32 / m2 lanes (m2 = 1, 2, 4 or 8 >= the row count).  Lane j of a group
// takes blocks j, j + G, ... of its row -- every load of the level in flight
// at once -- a shuffle tree inside the group sums the partial products and
// the group's first lane finishes the row.  One memory round trip per LEVEL
// instead of one per row: ILU(2) on 10^3 boxes has 343 + 343 levels of <= 4
// rows of up to 90 blocks (128^3 apply 8.0 -> 4.7 ms), ILU(1) 163 levels of
// <= 8 rows of up to 34 blocks (8.0 -> 3.4 ms); exact LU levels are single
// rows (G = 32).  profiles/r02/wide_sweep_variants.txt.
// UB = 6 blocks in flight per lane (4 and 8 measured slower; 12 spills next
// to the lane-per-row sweep's own 12-slot arrays).
constexpr int kWideUB = 6;
// Slot addressing: TABLE = the group solver's shared-memory tables (jo[t]:
// level-relative offset of jagged diagonal t, ecol as uint16 in shared
// memory); else the warp solver's closed form (rows sorted by decreasing
// length L[0..7]: offset of diagonal t = sum_q min(L[q], t); ecol in global).
template <typename FT, bool TABLE, int UB>
__device__ __forceinline__ void sweep_level_wide(const FT *__restrict__ A, const void *__restrict__ ecol_v,
                                              const unsigned short *__restrict__ jo, int4 L4, int4 L8, int base, int first,
                                              const unsigned short *__restrict__ rows,
                                              const unsigned short *__restrict__ lens, double2 *y, int m,
                                              bool backward, int lane, int bmin, uint64_t pol)
{
    const int m2 = m <= 1 ? 1 : (m == 2 ? 2 : (m <= 4 ? 4 : 8));
    const int G = 32 / m2;
    const int q = lane / G, j = lane - q * G;
    const bool has = q < m;
    const int i = has ? rows[q] : 0;
    // left-RAS backward rows below bmin feed no owned row: neither loaded nor written
    const bool act = has && i >= bmin;
    const int len = act ? lens[q] - (backward ? 1 : 0) : 0;
    auto slot = [&](int t) {
        if (TABLE) return base + jo[t] + q;
        return base + first + min(L4.x, t) + min(L4.y, t) + min(L4.z, t) + min(L4.w, t) + min(L8.x, t) +
               min(L8.y, t) + min(L8.z, t) + min(L8.w, t) + q;
    };
    double2 acc = make_double2(0.0, 0.0);
    for (int t0 = 0; __any_sync(0xffffffffu, t0 < len); t0 += UB * G) {
        FT a[UB];
        int c[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int t = t0 + u * G + j;
            if (t < len) {
                const int e = slot(t);
                // the group solver's streaming loads skip L1 and are evicted first from L2
                if (TABLE) ldg4_pred(a[u], A + e, true, pol);
                else a[u] = ldg4(A + e);
                c[u] = TABLE ? (int)reinterpret_cast<const unsigned short *>(ecol_v)[e]
                             : __ldg(reinterpret_cast<const int *>(ecol_v) + e);
            }
        }
#pragma unroll
        for (int u = 0; u < UB; ++u)
            if (t0 + u * G + j < len) blk_sub(acc, a[u], y[c[u]]);
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (act && j == 0) {
        double2 v = y[i];
        v.x += acc.x;
        v.y += acc.y;
        if (backward) {
            FT d;
            if (TABLE) ldg4_pred(d, A + base + q, true, pol);
            else d = ldg4(A + base + q);
            v = make_double2(d.x * v.x + d.y * v.y, d.z * v.x + d.w * v.y);
        }
        y[i] = v;
    }
    __syncwarp();
}

// Warp-per-subdomain solver (boxes with <= 32767 cells and levels <= 64 wide).
// Shared memory per subdomain: y (double2 per cell) plus the class's level
// metadata (row lists as uint16, row lengths as uint8, level starts/bases), so
// a level costs one global round trip: the factor slots (level-major, lane q
// reads slot base + t*m + q) and their column ids, all issued up front.
struct WarpSmem {
    int max_nloc, max_nlev, max_nlevb;
    __host__ __device__ size_t y_bytes() const { return sizeof(double2) * (size_t)max_nloc; }
    __host__ __device__ size_t bytes() const
    {
        size_t b = y_bytes();
        b += sizeof(int) * (size_t)(2 * max_nlev + 1 + 2 * max_nlevb + 1);
        b += sizeof(unsigned short) * 4 * (size_t)max_nloc;
        return (b + 15) / 16 * 16;
    }
};

// Warp solver's narrow long-row levels: slot (t, q) = base + first +
// sum_q' min(len_q', t) + q, rows sorted by decreasing length (closed form of
// the jagged-diagonal offsets; the group solver reads them from a table).
__device__ __forceinline__ void sweep_rows_wide_warp(const double4 *__restrict__ A,
                                                     const int *__restrict__ ecol,
                                                     const unsigned short *__restrict__ rows,
                                                     const unsigned short *__restrict__ lens, double2 *y, int base,
                                                     int m, bool backward, int lane)
{
    int L[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) L[q] = q < m ? lens[q] - (backward ? 1 : 0) : 0;
    sweep_level_wide<double4, false, kWideUB>(A, ecol, nullptr, make_int4(L[0], L[1], L[2], L[3]),
                                                   make_int4(L[4], L[5], L[6], L[7]), base, backward ? m : 0, rows,
                                                   lens, y, m, backward, lane, 0, 0ull);
}

template <int VARIANT, int MAXW = 12, int PREFETCH_DEPTH = 4, bool WIDE = false>
__global__ void __launch_bounds__(32, 8)
apply_warp_kernel(GridDev g, const ClassDev *__restrict__ classes, const int *__restrict__ sub_class,
                  const int4 *__restrict__ sub_origin, const long long *__restrict__ sub_off,
                  const long long *__restrict__ sub_ext_off, const double4 *__restrict__ vals,
                  const double2 *__restrict__ r, double2 *__restrict__ z, double2 *__restrict__ ext_out,
                  WarpSmem L, long long nsub)
{
    ACCH_SKIP_IF(g);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x;
    const long long s = blockIdx.x;
    if (s >= nsub) return;
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    const double4 *__restrict__ A = vals + sub_off[s];
    double2 *y = reinterpret_cast<double2 *>(smem_raw);
    int *f_ptr = reinterpret_cast<int *>(smem_raw + L.y_bytes());
    int *f_bs = f_ptr + (C.nlev + 1);
    int *b_ptr = f_bs + C.nlev;
    int *b_bs = b_ptr + (C.nlevb + 1);
    unsigned short *f_rows = reinterpret_cast<unsigned short *>(b_bs + C.nlevb);
    unsigned short *b_rows = f_rows + C.nloc;
    unsigned short *f_len = b_rows + C.nloc;
    unsigned short *b_len = f_len + C.nloc;
    for (int i = lane; i <= C.nlev; i += 32) f_ptr[i] = C.lev_ptr[i];
    for (int i = lane; i < C.nlev; i += 32) f_bs[i] = C.f_base[i];
    for (int i = lane; i <= C.nlevb; i += 32) b_ptr[i] = C.levb_ptr[i];
    for (int i = lane; i < C.nlevb; i += 32) b_bs[i] = C.b_base[i];
    for (int i = lane; i < C.nloc; i += 32) {
        f_rows[i] = C.f_rows16[i];
        b_rows[i] = C.b_rows16[i];
        f_len[i] = C.f_len8[i];
        b_len[i] = C.b_len8[i];
    }
    // slot range of "global level" k: forward levels 0..nlev-1 then backward 0..nlevb-1
    // (reads the shared-memory copies of the level bases: no global round trip)
    auto level_range = [&](int k, int &lo, int &hi) {
        if (k < C.nlev) {
            lo = f_bs[k];
            hi = k + 1 < C.nlev ? f_bs[k + 1] : (C.nlevb > 0 ? b_bs[0] : C.ell_total);
        } else {
            const int kb = k - C.nlev;
            lo = b_bs[kb];
            hi = kb + 1 < C.nlevb ? b_bs[kb + 1] : C.ell_total;
        }
    };
    __syncwarp();
    const int nlev_all = C.nlev + C.nlevb;
    auto prefetch_level = [&](int k) {
        if (k >= nlev_all) return;
        int lo, hi;
        level_range(k, lo, hi);
        prefetch_l2(A + lo, (unsigned)(hi - lo) * 32u);
    };
    if (lane < PREFETCH_DEPTH) prefetch_level(lane);
    const long long nx = g.nx, ny = g.ny;
    for (int l = lane; l < C.nloc; l += 32) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double2 v = r[cell_at(g, gx, gy, zplane(g, gz))];
        if (VARIANT == 2 && !C.owned[l]) v = make_double2(0.0, 0.0);
        y[l] = v;
    }
    __syncwarp();
    // Levels are at most 64 rows wide here.  Lane q owns rows q and q + 32 of
    // a level; the jagged-diagonal offsets come from ballots (rows sorted by
    // length).  The first MAXW slots of a row are loaded up front (one global
    // round trip per level); longer rows (wrapped boxes, fill-in) finish in a
    // tail loop.  Rows of a level are independent, so results are written
    // after all of the level's loads.
    for (int lev = 0; lev < C.nlev; ++lev) {
        if (lane == 0) prefetch_level(lev + PREFETCH_DEPTH);
        const int r0 = f_ptr[lev], m = f_ptr[lev + 1] - r0, base = f_bs[lev];
        if (WIDE && m <= kWideRows && f_len[r0] > kWideMin) {
            sweep_rows_wide_warp(A, C.ecol, f_rows + r0, f_len + r0, y, base, m, false, lane);
            continue;
        }
        const int len0 = lane < m ? f_len[r0 + lane] : 0;
        const int len1 = lane + 32 < m ? f_len[r0 + lane + 32] : 0;
        const int i0 = lane < m ? f_rows[r0 + lane] : 0;
        const int i1 = lane + 32 < m ? f_rows[r0 + lane + 32] : 0;
        int offs[MAXW];
        double4 a[MAXW];
        int c[MAXW];
        int off = 0;
#pragma unroll
        for (int t = 0; t < MAXW; ++t) {
            offs[t] = off;
            if (t < len0) {
                a[t] = ldg4(A + base + off + lane);
                c[t] = __ldg(C.ecol + base + off + lane);
            }
            off += __popc(__ballot_sync(0xffffffffu, len0 > t)) + __popc(__ballot_sync(0xffffffffu, len1 > t));
        }
        double2 acc0 = y[i0], acc1 = y[i1];
#pragma unroll
        for (int t = 0; t < MAXW; ++t)
            if (t < len0) blk_sub(acc0, a[t], y[c[t]]);
        if (len1 > 0) {
#pragma unroll
            for (int t = 0; t < MAXW; ++t)
                if (t < len1) {
                    a[t] = ldg4(A + base + offs[t] + lane + 32);
                    c[t] = __ldg(C.ecol + base + offs[t] + lane + 32);
                }
#pragma unroll
            for (int t = 0; t < MAXW; ++t)
                if (t < len1) blk_sub(acc1, a[t], y[c[t]]);
        }
        for (int t = MAXW;; ++t) {
            const unsigned b0 = __ballot_sync(0xffffffffu, len0 > t), b1 = __ballot_sync(0xffffffffu, len1 > t);
            if (!(b0 | b1)) break;
            if (t < len0) blk_sub(acc0, ldg4(A + base + off + lane), y[__ldg(C.ecol + base + off + lane)]);
            if (t < len1) blk_sub(acc1, ldg4(A + base + off + lane + 32), y[__ldg(C.ecol + base + off + lane + 32)]);
            off += __popc(b0) + __popc(b1);
        }
        if (lane < m) y[i0] = acc0;
        if (lane + 32 < m) y[i1] = acc1;
        __syncwarp();
    }
    for (int lev = 0; lev < C.nlevb; ++lev) {
        if (lane == 0) prefetch_level(C.nlev + lev + PREFETCH_DEPTH);
        const int r0 = b_ptr[lev], m = b_ptr[lev + 1] - r0, base = b_bs[lev];
        if (WIDE && m <= kWideRows && b_len[r0] > kWideMin + 1) {
            sweep_rows_wide_warp(A, C.ecol, b_rows + r0, b_len + r0, y, base, m, true, lane);
            continue;
        }
        // slot 0 of every row: the inverted diagonal block; U slots follow
        const int len0 = lane < m ? b_len[r0 + lane] - 1 : 0;
        const int len1 = lane + 32 < m ? b_len[r0 + lane + 32] - 1 : 0;
        const int i0 = lane < m ? b_rows[r0 + lane] : 0;
        const int i1 = lane + 32 < m ? b_rows[r0 + lane + 32] : 0;
        int offs[MAXW];
        double4 a[MAXW];
        int c[MAXW];
        int off = m;
#pragma unroll
        for (int t = 0; t < MAXW; ++t) {
            offs[t] = off;
            if (t < len0) {
                a[t] = ldg4(A + base + off + lane);
                c[t] = __ldg(C.ecol + base + off + lane);
            }
            off += __popc(__ballot_sync(0xffffffffu, len0 > t)) + __popc(__ballot_sync(0xffffffffu, len1 > t));
        }
        double2 acc0 = y[i0], acc1 = y[i1];
#pragma unroll
        for (int t = 0; t < MAXW; ++t)
            if (t < len0) blk_sub(acc0, a[t], y[c[t]]);
        if (len1 > 0) {
#pragma unroll
            for (int t = 0; t < MAXW; ++t)
                if (t < len1) {
                    a[t] = ldg4(A + base + offs[t] + lane + 32);
                    c[t] = __ldg(C.ecol + base + offs[t] + lane + 32);
                }
#pragma unroll
            for (int t = 0; t < MAXW; ++t)
                if (t < len1) blk_sub(acc1, a[t], y[c[t]]);
        }
        for (int t = MAXW;; ++t) {
            const unsigned b0 = __ballot_sync(0xffffffffu, len0 > t), b1 = __ballot_sync(0xffffffffu, len1 > t);
            if (!(b0 | b1)) break;
            if (t < len0) blk_sub(acc0, ldg4(A + base + off + lane), y[__ldg(C.ecol + base + off + lane)]);
            if (t < len1) blk_sub(acc1, ldg4(A + base + off + lane + 32), y[__ldg(C.ecol + base + off + lane + 32)]);
            off += __popc(b0) + __popc(b1);
        }
        if (lane < m) {
            const double4 di = ldg4(A + base + lane);
            y[i0] = make_double2(di.x * acc0.x + di.y * acc0.y, di.z * acc0.x + di.w * acc0.y);
        }
        if (lane + 32 < m) {
            const double4 di = ldg4(A + base + lane + 32);
            y[i1] = make_double2(di.x * acc1.x + di.y * acc1.y, di.z * acc1.x + di.w * acc1.y);
        }
        __syncwarp();
    }
    if (VARIANT == 1) {
        for (int l = lane; l < C.nloc; l += 32) {
            if (!C.owned[l]) continue;
            int gx, gy, gz;
            local_to_global(g, C, o, l, gx, gy, gz);
            z[cell_at(g, gx, gy, zplane(g, gz))] = y[l];
        }
    } else {
        for (int l = lane; l < C.nloc; l += 32) ext_out[sub_ext_off[s] + l] = y[l];
    }
}

// ---------------------------------------------------------------------------
// Column-sweep solver for narrow classes: every level of every class has at
// most kWideRows rows (exact LU: single rows; ILU(1) / ILU(2) on 10^3 boxes:
// <= 8 / <= 4 rows), so the solve is latency-bound on its dependency chain.
// A row-oriented sweep ends every row with a warp-wide reduction tree; the
// column-oriented one has none: once x_j is final, lane l subtracts
// L_ij x_j from y_i for its entry (i, j) of column j -- distinct rows, so
// distinct shared-memory words -- and the chain per column is one
// shared-memory broadcast of x_j, one 2x2 block product and one store.
// The factors of these classes are stored COLUMN-major (relayout_columns):
// the forward sweep streams the L columns 0..n-1, the backward sweep the U
// columns n-1..0 (inverted diagonal block first): ONE contiguous stream of
// slots, which the TMA engine copies tile by tile (cp.async.bulk + mbarrier)
// into a shared-memory ring kColRing tiles ahead of the sweep -- register
// prefetching cannot run that deep (six scoreboards per warp: waiting for
// the oldest of many loads in flight waits for the newest too; measured).
// A step is a column, or a 64-entry piece of a longer one:
// word = column | entries << 16 | tiles to wait for << 23 | tiles to hand back << 25 | first << 31.
// Row i accumulates its terms in column order, which is the reference's own
// order (_ilu.py:123-137).
// ---------------------------------------------------------------------------
constexpr int kColChunk = 64;   // entries per step (two per lane)
// 2 tiles of 256 slots (8 KB of blocks + 512 B of row ids each) measured best
// against 8 x 64, 4 x 128, 4 x 256 and 2 x 512: the ring competes with
// resident CTAs for shared memory (profiles/r02/wide_sweep_variants.txt)
constexpr int kColTile = 256;   // factor slots per TMA tile
constexpr int kColRing = 2;     // tiles in the shared-memory ring

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct ColSmem {
    int max_nloc, max_steps, steps_smem;
    // y: one scratch row past the box; steps: one spare word past the last step
    __host__ __device__ size_t y_bytes() const { return (sizeof(double2) * (size_t)(max_nloc + 1) + 127) / 128 * 128; }
    // steps_smem: the step table staged in shared memory (when that costs no resident CTA), else read from global
    __host__ __device__ size_t steps_bytes() const
    {
        return steps_smem ? (sizeof(unsigned) * (size_t)(max_steps + 1) + 127) / 128 * 128 : 0;
    }
    __host__ __device__ size_t bytes() const
    {
        return y_bytes() + steps_bytes() + (size_t)kColRing * kColTile * (sizeof(double4) + sizeof(unsigned short)) +
               sizeof(uint64_t) * kColRing;
    }
};

template <int VARIANT, bool SSTEPS>
__global__ void __launch_bounds__(32, 8)
apply_cols_kernel(GridDev g, const ClassDev *__restrict__ classes, const int *__restrict__ sub_class,
                  const int4 *__restrict__ sub_origin, const long long *__restrict__ sub_off,
                  const long long *__restrict__ sub_ext_off, const double4 *__restrict__ vals,
                  const double2 *__restrict__ r, double2 *__restrict__ z, double2 *__restrict__ ext_out, ColSmem L,
                  long long nsub)
{
    ACCH_SKIP_IF(g);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x;
    const long long s = blockIdx.x;
    if (s >= nsub) return;
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    const double4 *__restrict__ A = vals + sub_off[s];
    double2 *y = reinterpret_cast<double2 *>(smem_raw);
    // (two spare words past the last step: the sweep reads one step ahead)
    unsigned *ssteps = reinterpret_cast<unsigned *>(smem_raw + L.y_bytes());
    const unsigned *steps = SSTEPS ? ssteps : C.col_steps;
    double4 *ringA = reinterpret_cast<double4 *>(smem_raw + L.y_bytes() + L.steps_bytes());
    unsigned short *ringI = reinterpret_cast<unsigned short *>(ringA + kColRing * kColTile);
    uint64_t *bars = reinterpret_cast<uint64_t *>(ringI + kColRing * kColTile);
    // left RAS: the backward columns below the first owned row update only
    // rows that are never scattered
    const int nf = C.col_nf, nb = VARIANT == 1 ? C.col_nb_ras : C.col_nb;
    const int end_slot = VARIANT == 1 ? C.col_end_ras : C.col_end;
    const int ntiles = (end_slot + kColTile - 1) / kColTile;
    if (lane == 0) {
        for (int i = 0; i < kColRing; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // tile c of the factor stream (blocks + row ids) into ring slot c % kColRing
    auto issue = [&](int c) {
        if (c >= ntiles || lane != 0) return;
        const int k = c % kColRing;
        // (the ring slot was last READ through the generic proxy, before the
        // step's __syncwarp: write-after-read needs no proxy fence)
        mbar_expect_tx(bars + k, kColTile * (unsigned)(sizeof(double4) + sizeof(unsigned short)));
        bulk_g2s(ringA + k * kColTile, A + (size_t)c * kColTile, kColTile * (unsigned)sizeof(double4), bars + k);
        bulk_g2s(ringI + k * kColTile, C.col_ridx + (size_t)c * kColTile, kColTile * (unsigned)sizeof(unsigned short),
                 bars + k);
        // (a bulk L2 prefetch further ahead measured no gain at 4 tiles and a loss at 8-12)
    };
#pragma unroll
    for (int c = 0; c < kColRing; ++c) issue(c);
    if (SSTEPS)
        for (int i = lane; i <= nf + nb; i += 32) ssteps[i] = i < nf + nb ? C.col_steps[i] : 0u;
    for (int l = lane; l < C.nloc; l += 32) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double2 v = r[cell_at(g, gx, gy, zplane(g, gz))];
        if (VARIANT == 2 && !C.owned[l]) v = make_double2(0.0, 0.0);
        y[l] = v;
    }
    __syncwarp();

    constexpr int RM = kColRing * kColTile - 1;   // ring index mask
    int e = 0;        // next slot of the stream (warp-uniform)
    int ready = 0;    // tiles waited for
    int freed = 0;    // tiles handed back (and refilled)
    // the step word says how many new tiles the step reads (0 for most steps) ...
    auto acquire = [&](unsigned w) {
        for (int k = (int)((w >> 23) & 3u); k > 0; --k) {
            mbar_wait(bars + (ready % kColRing), (unsigned)(ready / kColRing) & 1u);
            ++ready;
        }
    };
    // ... and how many the stream has left behind once it is done (after its __syncwarp)
    auto release = [&](unsigned w) {
        for (int k = (int)((w >> 25) & 3u); k > 0; --k) {
            issue(freed + kColRing);
            ++freed;
        }
    };
    // A lane without an entry in this step works on the scratch row y[nloc]
    // (no divergent branch in the chain; whatever the ring holds at its
    // slot is subtracted from a row nobody reads).
    const int scratch = C.nloc;
    auto entries = [&](int n, const double2 x) {
        {
            const int q = (e + lane) & RM;
            const int i = lane < n ? (int)ringI[q] : scratch;
#ifdef ACCH_COL_CHECK
            if (i < 0 || i > C.nloc || e + n > end_slot || (e + lane) / kColTile >= ready + 0 && lane < n) __trap();
#endif
            double2 acc = y[i];
            blk_sub(acc, ringA[q], x);
            y[i] = acc;
        }
        if (n > 32) {   // warp-uniform
            const int q = (e + lane + 32) & RM;
            const int i = lane + 32 < n ? (int)ringI[q] : scratch;
#ifdef ACCH_COL_CHECK
            if (i < 0 || i > C.nloc || ((e + lane + 32) / kColTile >= ready && lane + 32 < n)) __trap();
#endif
            double2 acc = y[i];
            blk_sub(acc, ringA[q], x);
            y[i] = acc;
        }
        __syncwarp();
        e += n;
    };
    // forward: x_j = y_j is final when its column comes up; the next step's
    // word is read a step ahead (it does not depend on the sweep)
    unsigned wn = nf + nb > 0 ? steps[0] : 0u;
    for (int st = 0; st < nf; ++st) {
        const unsigned w = wn;
        wn = steps[st + 1];   // the table has one spare word past the last step
        acquire(w);
        entries((int)((w >> 16) & 0x7fu), y[w & 0xffffu]);
        release(w);
    }
    // backward: x_j = inv(D_j) y_j opens the column; it is stored one step late
    // (the lanes of this step still read the old y_j)
    {
        double2 x = make_double2(0.0, 0.0), pend_x = x;
        int pend_j = scratch;
        for (int st = nf; st < nf + nb; ++st) {
            const unsigned w = wn;
            wn = steps[st + 1];
            acquire(w);
            if (lane == 0) y[pend_j] = pend_x;
            if (w >> 31) {
                const int j = (int)(w & 0xffffu);
                const double4 d = ringA[e & RM];
                const double2 yj = y[j];
                x = make_double2(d.x * yj.x + d.y * yj.y, d.z * yj.x + d.w * yj.y);
                pend_j = j;
                pend_x = x;
                ++e;
            }
            entries((int)((w >> 16) & 0x7fu), x);
            release(w);
        }
        if (lane == 0) y[pend_j] = pend_x;
        __syncwarp();
    }
#ifdef ACCH_COL_CHECK
    // the whole stream was consumed, every issued tile was waited for, no tile is still in flight
    if (e != end_slot || ready != ntiles || freed + kColRing < ntiles) __trap();
#endif
    if (VARIANT == 1) {
        for (int l = lane; l < C.nloc; l += 32) {
            if (!C.owned[l]) continue;
            int gx, gy, gz;
            local_to_global(g, C, o, l, gx, gy, gz);
            z[cell_at(g, gx, gy, zplane(g, gz))] = y[l];
        }
    } else {
        for (int l = lane; l < C.nloc; l += 32) ext_out[sub_ext_off[s] + l] = y[l];
    }
}

// ---------------------------------------------------------------------------
// Class-group solver (default).  One CTA = NW warps = up to NW subdomains of
// the SAME class: the class's symbolic data (level tables, row lists, row
// lengths, slot column ids as uint16) is copied once into shared memory and
// shared by the NW warps, each of which keeps its own y (double2 per cell).
// A level then costs one global round trip -- the factor slots, L2-prefetched
// PD levels ahead by the TMA engine -- because every index it needs (rows,
// lengths, jagged offsets by ballot, column ids) is on-chip.
// ---------------------------------------------------------------------------

// one level of a triangular sweep for the rows owned by this lane (q, q + 32)
//   first = 0: forward (L) rows, y_i -= sum L_ij y_j
//   first = m: backward (U) rows, slot 0..m-1 hold inv(D_i); y_i = inv(D_i)(y_i - sum U_ij y_j)
//
// All of the lane's factor loads are issued before the first FMA: the
// accumulator's initial shared-memory read takes its address through the last
// load's result (masked by `zero`, a runtime 0 the compiler cannot fold), so
// ptxas cannot start consuming loads 0..5 before it has issued loads 6..11 --
// the interleaving that otherwise costs a second memory round trip per level.
template <int MAXW, typename FT = double4>
__device__ __forceinline__ void sweep_level(const FT *__restrict__ A, const unsigned short *__restrict__ ecol,
                                            const unsigned short *__restrict__ jo, double2 *y, int base, int m,
                                            int len0, int len1, int i0, int i1, bool backward, int lane, int zero,
                                            uint64_t pol, int bmin = 0)
{
    // rows below bmin (left-RAS backward sweep: they feed no owned row) are
    // neither loaded nor written
    const bool act0 = lane < m && i0 >= bmin, act1 = lane + 32 < m && i1 >= bmin;
    if (!act0) len0 = 0;
    if (!act1) len1 = 0;
    // jo[t]: level-relative slot offset of diagonal t (jagged layout; shared
    // memory, warp-uniform), so lane q's slot t is base + jo[t] + q
    FT a[MAXW];
    int c[MAXW];
    FT d0, d1;
    if (backward) {
        ldg4_pred(d0, A + base + lane, act0, pol);
        ldg4_pred(d1, A + base + lane + 32, act1, pol);
    }
#pragma unroll
    for (int t = 0; t < MAXW; ++t) {
        const int e = base + jo[t] + lane;
        ldg4_pred(a[t], A + e, t < len0, pol);
        c[t] = t < len0 ? ecol[e] : 0;
    }
    const int dep = anchor_bits(a[MAXW - 1]) & zero;
    double2 acc0 = y[i0 + dep], acc1 = y[i1];
    // (an all-products-first ordering -- bitwise the same result -- measured
    // 17% slower: it gathers y for inactive slots and lengthens the schedule)
#pragma unroll
    for (int t = 0; t < MAXW; ++t)
        if (t < len0) blk_sub(acc0, a[t], y[c[t]]);
    if (len1 > 0) {
#pragma unroll
        for (int t = 0; t < MAXW; ++t)
            if (t < len1) {
                const int e = base + jo[t] + lane + 32;
                a[t] = ldg4(A + e);
                c[t] = ecol[e];
            }
#pragma unroll
        for (int t = 0; t < MAXW; ++t)
            if (t < len1) blk_sub(acc1, a[t], y[c[t]]);
    }
    // rows longer than MAXW slots (U rows of a wrapped periodic box, <= 21):
    // the extra slots of the first row in batches of XB loads through a[],
    // one round trip per batch instead of one per slot
    constexpr int XB = 4;
    for (int t0 = MAXW; __any_sync(0xffffffffu, len0 > t0 || len1 > t0); t0 += XB) {
#pragma unroll
        for (int u = 0; u < XB; ++u) {
            const int t = t0 + u;
            const int e = base + jo[t] + lane;
            ldg4_pred(a[u], A + e, t < len0, pol);
            c[u] = t < len0 ? ecol[e] : 0;
        }
#pragma unroll
        for (int u = 0; u < XB; ++u)
            if (t0 + u < len0) blk_sub(acc0, a[u], y[c[u]]);
        for (int t = t0; t < t0 + XB; ++t)
            if (t < len1) {
                const int e = base + jo[t] + lane + 32;
                blk_sub(acc1, ldg4(A + e), y[ecol[e]]);
            }
    }
    if (backward) {
        acc0 = make_double2(d0.x * acc0.x + d0.y * acc0.y, d0.z * acc0.x + d0.w * acc0.y);
        acc1 = make_double2(d1.x * acc1.x + d1.y * acc1.y, d1.z * acc1.x + d1.w * acc1.y);
    }
    if (act0) y[i0] = acc0;
    if (act1) y[i1] = acc1;
    __syncwarp();
}

template <typename FT>
__device__ __forceinline__ void sweep_rows_wide(const FT *__restrict__ A, const unsigned short *__restrict__ ecol,
                                                const unsigned short *__restrict__ jo,
                                                const unsigned short *__restrict__ rows,
                                                const unsigned short *__restrict__ lens, double2 *y, int base,
                                                int m, bool backward, int lane, uint64_t pol, int bmin = 0)
{
    // jo[t]: level-relative offset of jagged diagonal t (for backward levels
    // the caller passes jo + 1: diagonal 0 holds the inverted diagonal blocks)
    sweep_level_wide<FT, true, kWideUB>(A, ecol, jo, make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0), base, 0, rows, lens, y, m, backward, lane, bmin, pol);
}

// one subdomain of a class group: gather, forward and backward sweeps, scatter
template <int VARIANT, int MAXW, typename FT = double4, bool WIDE = false>
__device__ __forceinline__ void group_solve_one(const GridDev &g, const ClassDev &C, const unsigned char *smem_meta,
                                             double2 *y, int s, const int4 *__restrict__ sub_origin,
                                             const long long *__restrict__ sub_off,
                                             const long long *__restrict__ sub_ext_off,
                                             const FT *__restrict__ vals, const double2 *__restrict__ r,
                                             double2 *__restrict__ z, double2 *__restrict__ ext_out, int zero, int pd)
{
    const int lane = threadIdx.x & 31;
    const int nlev = C.nlev, nlevb = C.nlevb, nloc = C.nloc, ell_total = C.ell_total;
    const int *f_ptr = reinterpret_cast<const int *>(smem_meta);
    const int *f_bs = reinterpret_cast<const int *>(smem_meta + C.m_fbs);
    const int *b_ptr = reinterpret_cast<const int *>(smem_meta + C.m_bptr);
    const int *b_bs = reinterpret_cast<const int *>(smem_meta + C.m_bbs);
    const unsigned short *f_rows = reinterpret_cast<const unsigned short *>(smem_meta + C.m_frows);
    const unsigned short *b_rows = reinterpret_cast<const unsigned short *>(smem_meta + C.m_brows);
    const unsigned short *f_len = reinterpret_cast<const unsigned short *>(smem_meta + C.m_flen);
    const unsigned short *b_len = reinterpret_cast<const unsigned short *>(smem_meta + C.m_blen);
    const unsigned short *ecol = reinterpret_cast<const unsigned short *>(smem_meta + C.m_ecol);
    const int *f_jp = reinterpret_cast<const int *>(smem_meta + C.m_fjp);
    const int *b_jp = reinterpret_cast<const int *>(smem_meta + C.m_bjp);
    const unsigned short *f_jo = reinterpret_cast<const unsigned short *>(smem_meta + C.m_fjo);
    const unsigned short *b_jo = reinterpret_cast<const unsigned short *>(smem_meta + C.m_bjo);
    const uint64_t pol = evict_first_policy();
    const int4 o = sub_origin[s];
    const long long obase = cell_at(g, o.x, o.y, zplane(g, o.z));   // used when o.w (no wrap)
    const FT *__restrict__ A = vals + sub_off[s];
    // left RAS: the backward levels past nlevb_ras and the rows below
    // b_min_row feed no owned row (see ClassDev) -- skipped
    const int nlevb_run = VARIANT == 1 ? C.nlevb_ras : nlevb;
    const int bmin = VARIANT == 1 ? C.b_min_row : 0;
    const int nall = nlev + nlevb_run;
    auto prefetch_level = [&](int k) {
        if (k >= nall) return;
        int lo, hi;
        if (k < nlev) {
            lo = f_bs[k];
            hi = k + 1 < nlev ? f_bs[k + 1] : (nlevb > 0 ? b_bs[0] : ell_total);
        } else {
            const int kb = k - nlev;
            lo = b_bs[kb];
            hi = kb + 1 < nlevb ? b_bs[kb + 1] : ell_total;
        }
        prefetch_l2(A + lo, (unsigned)((hi - lo) * sizeof(FT)));
    };
    if (lane < pd) prefetch_level(lane);
    // gather r into y with many independent loads in flight per lane; the
    // offset tables come from the class image in shared memory
    const int *s_lin = reinterpret_cast<const int *>(smem_meta + C.m_lin);
    const unsigned *s_ixyz = reinterpret_cast<const unsigned *>(smem_meta + C.m_ixyz);
    const int *s_relx = reinterpret_cast<const int *>(smem_meta + C.m_rel);
    const int *s_rely = s_relx + C.len[0], *s_relz = s_rely + C.len[1];
    // storage index of local cell l of a box that wraps (rel stored mod n)
    auto wrapped_cell = [&](int l) -> long long {
        const unsigned p = s_ixyz[l];
        int gx = o.x + s_relx[p & 1023u];
        gx = gx >= g.nx ? gx - g.nx : gx;
        int gy = o.y + s_rely[(p >> 10) & 1023u];
        gy = gy >= g.ny ? gy - g.ny : gy;
        int gz = 0;
        if (g.dim == 3) {
            gz = o.z + s_relz[p >> 20];
            gz = g.zg ? gz + g.zg : (gz >= g.nz ? gz - g.nz : gz);
        }
        return ((long long)gz * g.ny + gy) * g.nx + gx;
    };
    {
        constexpr int GB = 16;
        for (int l0 = 0; l0 < nloc; l0 += 32 * GB) {
            double2 v[GB];
#pragma unroll
            for (int j = 0; j < GB; ++j) {
                const int l = l0 + j * 32 + lane;
                if (l < nloc) v[j] = r[o.w ? obase + s_lin[l] : wrapped_cell(l)];
            }
#pragma unroll
            for (int j = 0; j < GB; ++j) {
                const int l = l0 + j * 32 + lane;
                if (l < nloc) y[l] = (VARIANT == 2 && !C.owned[l]) ? make_double2(0.0, 0.0) : v[j];
            }
        }
    }
    __syncwarp();
    // (software-pipelining level k+1's shared-memory index reads under level
    // k's loads measured 1% slower: profiles/r01_apply_sweeps_group.txt)
    for (int lev = 0; lev < nlev; ++lev) {
        if (lane == 0) prefetch_level(lev + pd);
        const int r0 = f_ptr[lev], m = f_ptr[lev + 1] - r0;
        if (WIDE && m <= kWideRows && f_len[r0] > kWideMin) {
            sweep_rows_wide<FT>(A, ecol, f_jo + f_jp[lev], f_rows + r0, f_len + r0, y, f_bs[lev], m, false, lane,
                                pol);
            continue;
        }
        const int len0 = lane < m ? f_len[r0 + lane] : 0;
        const int len1 = lane + 32 < m ? f_len[r0 + lane + 32] : 0;
        const int i0 = lane < m ? f_rows[r0 + lane] : 0;
        const int i1 = lane + 32 < m ? f_rows[r0 + lane + 32] : 0;
        sweep_level<MAXW, FT>(A, ecol, f_jo + f_jp[lev], y, f_bs[lev], m, len0, len1, i0, i1, false, lane, zero, pol);
    }
    for (int lev = 0; lev < nlevb_run; ++lev) {
        if (lane == 0) prefetch_level(nlev + lev + pd);
        const int r0 = b_ptr[lev], m = b_ptr[lev + 1] - r0;
        if (WIDE && m <= kWideRows && b_len[r0] > kWideMin + 1) {
            sweep_rows_wide<FT>(A, ecol, b_jo + b_jp[lev] + 1, b_rows + r0, b_len + r0, y, b_bs[lev], m, true, lane,
                                pol, bmin);
            continue;
        }
        // slot 0 of every backward row is its inverted diagonal block; U slots follow
        const int len0 = lane < m ? b_len[r0 + lane] - 1 : 0;
        const int len1 = lane + 32 < m ? b_len[r0 + lane + 32] - 1 : 0;
        const int i0 = lane < m ? b_rows[r0 + lane] : 0;
        const int i1 = lane + 32 < m ? b_rows[r0 + lane + 32] : 0;
        sweep_level<MAXW, FT>(A, ecol, b_jo + b_jp[lev] + 1, y, b_bs[lev], m, len0, len1, i0, i1, true, lane, zero,
                          pol, bmin);
    }
    if (VARIANT == 1) {
        // owned cells only (left RAS), from the class's owned-cell list
        const unsigned short *s_own = reinterpret_cast<const unsigned short *>(smem_meta + C.m_own);
        for (int k = lane; k < C.n_owned; k += 32) {
            const int l = s_own[k];
            z[o.w ? obase + s_lin[l] : wrapped_cell(l)] = y[l];
        }
    } else {
        for (int l = lane; l < nloc; l += 32) ext_out[sub_ext_off[s] + l] = y[l];
    }
    __syncwarp();   // y is reused by the warp's next subdomain
}

template <int VARIANT, int NW, int MAXW = 12, typename FT = double4, bool WIDE = false>
__global__ void __launch_bounds__(NW * 32, 1)
apply_group_kernel(GridDev g, const ClassDev *__restrict__ classes, const int4 *__restrict__ groups,
                   const int *__restrict__ grp_sub, const int4 *__restrict__ sub_origin,
                   const long long *__restrict__ sub_off, const long long *__restrict__ sub_ext_off,
                   const FT *__restrict__ vals, const double2 *__restrict__ r, double2 *__restrict__ z,
                   double2 *__restrict__ ext_out, int meta_max, int y_stride, int zero, int pd)
{
    ACCH_SKIP_IF(g);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int4 G = groups[blockIdx.x];   // (class, first entry of grp_sub, count, -)
    const ClassDev &C = classes[G.x];
    {
        const uint4 *__restrict__ src = reinterpret_cast<const uint4 *>(C.meta);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_raw);
        const int nb = C.meta_bytes / 16;
        for (int i = threadIdx.x; i < nb; i += NW * 32) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    double2 *y = reinterpret_cast<double2 *>(smem_raw + meta_max + (size_t)warp * y_stride);
    // one subdomain per warp (a loop over several per warp measured slower:
    // it pushes the sweep past 255 registers into spills)
    if (warp < G.z)
        group_solve_one<VARIANT, MAXW, FT, WIDE>(g, C, smem_raw, y, grp_sub[G.y + warp], sub_origin, sub_off,
                                           sub_ext_off, vals, r, z, ext_out, zero, pd);
}

__global__ void gather_kernel(long long n, const long long *__restrict__ cell_ptr, const long long *__restrict__ cell_src,
                              const double2 *__restrict__ ext_out, double2 *__restrict__ z, const int *skip)
{
    if (skip != nullptr && __ldcg(skip)) return;
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= n) return;
    double2 acc = make_double2(0.0, 0.0);
    for (long long e = cell_ptr[c]; e < cell_ptr[c + 1]; ++e) {
        const double2 v = ext_out[cell_src[e]];
        acc.x += v.x;
        acc.y += v.y;
    }
    z[c] = acc;
}

// ---------------------------------------------------------------------------
// host-side symbolic analysis
// ---------------------------------------------------------------------------

// ILU(level) fill on a block CSR pattern with sorted columns (_ilu.py:19-64);
// level < 0 means complete fill (exact LU without pivoting).
void symbolic_fill(int n, const std::vector<int> &rp, const std::vector<int> &ci, int level, std::vector<int> &orp,
                   std::vector<int> &oci)
{
    const long long lim = level < 0 ? LLONG_MAX / 4 : level;
    std::vector<std::vector<std::pair<int, long long>>> rows(n);
    orp.assign(n + 1, 0);
    oci.clear();
    for (int i = 0; i < n; ++i) {
        std::map<int, long long> lev;
        for (int t = rp[i]; t < rp[i + 1]; ++t) lev[ci[t]] = 0;
        if (level != 0) {
            for (auto it = lev.begin(); it != lev.end() && it->first < i; ++it) {
                const int k = it->first;
                const long long lik = it->second;
                if (lik >= lim) continue;
                for (const auto &e : rows[k]) {
                    if (e.first <= k) continue;
                    const long long cand = lik + e.second + 1;
                    if (cand > lim) continue;
                    auto f = lev.find(e.first);
                    if (f == lev.end()) lev.emplace(e.first, cand);
                    else if (cand < f->second) f->second = cand;
                }
            }
        }
        rows[i].assign(lev.begin(), lev.end());
        for (const auto &e : rows[i]) oci.push_back(e.first);
        orp[i + 1] = (int)oci.size();
    }
}

// a periodic box's relative coordinates are stored mod n (n - 1 for the cell
// left of the origin); the signed representative makes origin + rel linear
// for every box that does not actually wrap
int signed_rel(const GridDev &g, int axis, int r)
{
    const int n = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
    if (axis == 2 && g.zg > 0) return r;   // slab z offsets are raw local planes
    return (g.periodic && r > n / 2) ? r - n : r;
}

bool build_class(const GridDev &g, const std::array<std::vector<int>, 3> &rel, const int own_len[3], int fill,
                 ClassHost &C, std::string &err)
{
    const int dim = g.dim;
    const int nn[3] = {g.nx, g.ny, g.nz};
    C.rel = rel;
    for (int a = 0; a < 3; ++a) C.own_len[a] = own_len[a];
    const int lx = (int)rel[0].size(), ly = (int)rel[1].size(), lz = dim == 3 ? (int)rel[2].size() : 1;
    const int nloc = lx * ly * lz;
    C.nloc = nloc;
    // per-axis lookup: relative coordinate (mod n when periodic) -> index
    std::array<std::unordered_map<int, int>, 3> look;
    for (int a = 0; a < dim; ++a)
        for (int i = 0; i < (int)rel[a].size(); ++i) look[a][rel[a][i]] = i;
    int off[25][3];
    const int noff = stencil_offsets(dim, off);
    std::vector<int> tgt((size_t)nloc * noff, -1);
    std::vector<int> rp(nloc + 1, 0), ci;
    for (int l = 0; l < nloc; ++l) {
        const int ix[3] = {l % lx, (l / lx) % ly, l / (lx * ly)};
        std::vector<int> cols;
        for (int q = 0; q < noff; ++q) {
            int jl[3] = {0, 0, 0};
            bool ok = true;
            for (int a = 0; a < dim && ok; ++a) {
                int t = rel[a][ix[a]] + off[q][a];
                if (g.periodic && !(a == 2 && g.zg > 0)) t = ((t % nn[a]) + nn[a]) % nn[a];
                auto f = look[a].find(t);
                if (f == look[a].end()) ok = false;
                else jl[a] = f->second;
            }
            if (!ok) continue;
            const int lt = jl[0] + lx * (jl[1] + ly * jl[2]);
            tgt[(size_t)l * noff + q] = lt;
            cols.push_back(lt);
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        ci.insert(ci.end(), cols.begin(), cols.end());
        rp[l + 1] = (int)ci.size();
    }
    symbolic_fill(nloc, rp, ci, fill, C.rowptr, C.col);
    C.nnzb = (int)C.col.size();
    C.diag.assign(nloc, -1);
    for (int i = 0; i < nloc; ++i)
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t)
            if (C.col[t] == i) C.diag[i] = t;
    for (int i = 0; i < nloc; ++i)
        if (C.diag[i] < 0) {
            err = "subdomain pattern is missing a diagonal entry";
            return false;
        }
    // J stencil -> pattern positions
    C.jmap.assign((size_t)nloc * noff, -1);
    for (int l = 0; l < nloc; ++l)
        for (int q = 0; q < noff; ++q) {
            const int lt = tgt[(size_t)l * noff + q];
            if (lt < 0) continue;
            const int *b = C.col.data() + C.rowptr[l], *e = C.col.data() + C.rowptr[l + 1];
            const int *f = std::lower_bound(b, e, lt);
            C.jmap[(size_t)l * noff + q] = (int)(f - C.col.data());
        }
    C.jdup = 0;
    for (int l = 0; l < nloc && !C.jdup; ++l)
        for (int q = 0; q < noff; ++q)
            for (int q2 = 0; q2 < q; ++q2) {
                const int a = C.jmap[(size_t)l * noff + q], b = C.jmap[(size_t)l * noff + q2];
                if (a >= 0 && a == b) C.jdup = 1;
            }
    // IKJ update lists: for lower entry t=(i,k), pairs (U entry (k,j), entry (i,j))
    C.upd_ptr.assign(C.nnzb + 1, 0);
    C.upd.clear();
    std::vector<int> where(nloc, -1);
    for (int i = 0; i < nloc; ++i) {
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t) where[C.col[t]] = t;
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t) {
            const int k = C.col[t];
            if (k < i) {
                for (int u = C.diag[k] + 1; u < C.rowptr[k + 1]; ++u) {
                    const int w = where[C.col[u]];
                    if (w >= 0) C.upd.push_back(make_int2(u, w));
                }
            }
            C.upd_ptr[t + 1] = (int)C.upd.size();
        }
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t) where[C.col[t]] = -1;
    }
    // level schedules from the factor DAG
    std::vector<int> lev(nloc, 0), levb(nloc, 0);
    int nlev = 0, nlevb = 0;
    for (int i = 0; i < nloc; ++i) {
        int m = 0;
        for (int t = C.rowptr[i]; t < C.diag[i]; ++t) m = std::max(m, lev[C.col[t]] + 1);
        lev[i] = m;
        nlev = std::max(nlev, m + 1);
    }
    for (int i = nloc - 1; i >= 0; --i) {
        int m = 0;
        for (int t = C.diag[i] + 1; t < C.rowptr[i + 1]; ++t) m = std::max(m, levb[C.col[t]] + 1);
        levb[i] = m;
        nlevb = std::max(nlevb, m + 1);
    }
    // Width-capped list schedules: a level wider than a warp costs the warp
    // solvers a second round trip for its extra rows, so levels are refilled
    // to <= 32 rows (Kahn's algorithm, ready rows taken in order of their
    // latest feasible level).  Any topological schedule gives the same sweep
    // results bitwise: every row is still computed from finished rows only, in
    // its own slot order.  At 8^3 boxes: 55 levels of up to 34 rows -> 56 of
    // up to 32.
    {
        constexpr int kCap = 32;
        auto capped = [&](bool forward, std::vector<int> &lv, int &nl) {
            // deps(i): L columns (forward) / U columns (backward); users: the reverse
            std::vector<std::vector<int>> users(nloc);
            std::vector<int> indeg(nloc, 0);
            for (int i = 0; i < nloc; ++i) {
                const int t0 = forward ? C.rowptr[i] : C.diag[i] + 1, t1 = forward ? C.diag[i] : C.rowptr[i + 1];
                indeg[i] = t1 - t0;
                for (int t = t0; t < t1; ++t) users[C.col[t]].push_back(i);
            }
            // latest level of each row in the uncapped schedule (longest path to a sink)
            std::vector<int> tail(nloc, 0);
            for (int k = 0; k < nloc; ++k) {
                const int i = forward ? nloc - 1 - k : k;   // users come after i in the sweep order
                for (int u : users[i]) tail[i] = std::max(tail[i], tail[u] + 1);
            }
            std::vector<std::pair<int, int>> ready;   // (-tail, row): min-heap on -tail, i.e. longest tail first
            auto cmp = [](const std::pair<int, int> &a, const std::pair<int, int> &b) { return a > b; };
            for (int i = 0; i < nloc; ++i)
                if (indeg[i] == 0) ready.emplace_back(-tail[i], i);
            std::make_heap(ready.begin(), ready.end(), cmp);
            nl = 0;
            std::vector<int> take, fresh;
            while (!ready.empty()) {
                take.clear();
                while (!ready.empty() && (int)take.size() < kCap) {
                    std::pop_heap(ready.begin(), ready.end(), cmp);
                    take.push_back(ready.back().second);
                    ready.pop_back();
                }
                fresh.clear();
                for (int i : take) {
                    lv[i] = nl;
                    for (int u : users[i])
                        if (--indeg[u] == 0) fresh.push_back(u);
                }
                for (int u : fresh) {
                    ready.emplace_back(-tail[u], u);
                    std::push_heap(ready.begin(), ready.end(), cmp);
                }
                ++nl;
            }
        };
        auto width = [&](const std::vector<int> &lv, int nl) {
            std::vector<int> w(nl, 0);
            int m = 0;
            for (int i = 0; i < nloc; ++i) m = std::max(m, ++w[lv[i]]);
            return m;
        };
        if (width(lev, nlev) > kCap) capped(true, lev, nlev);
        if (width(levb, nlevb) > kCap) capped(false, levb, nlevb);
    }
    auto bucket = [&](const std::vector<int> &lv, int nl, std::vector<int> &ptr, std::vector<int> &rows) {
        ptr.assign(nl + 1, 0);
        for (int i = 0; i < nloc; ++i) ptr[lv[i] + 1]++;
        for (int k = 0; k < nl; ++k) ptr[k + 1] += ptr[k];
        rows.assign(nloc, 0);
        std::vector<int> fillp(ptr.begin(), ptr.end() - 1);
        for (int i = 0; i < nloc; ++i) rows[fillp[lv[i]]++] = i;
    };
    bucket(lev, nlev, C.lev_ptr, C.lev_rows);
    bucket(levb, nlevb, C.levb_ptr, C.levb_rows);
    // Jagged-diagonal slot layout per level (see apply_kernel): rows of a
    // level sorted by decreasing length, slot(t, q) = base + off_t + q with
    // off_t = sum_{t'<t} m_t' and m_t = #rows longer than t.  No padding, and
    // lane q of a warp reads slot base + off_t + q: consecutive 32-byte
    // blocks.  The factorisation addresses the same slots through pos[].
    C.pos.assign(C.nnzb, -1);
    int slot = 0;
    auto layout = [&](std::vector<int> &ptr, std::vector<int> &rows, bool lower, std::vector<int> &base,
                      std::vector<int> &lens, std::vector<int> &jptr, std::vector<int> &joff, int &maxw) {
        const int nl = (int)ptr.size() - 1;
        base.assign(nl, 0);
        lens.assign(nloc, 0);
        jptr.assign(nl + 1, 0);
        joff.clear();
        maxw = 0;
        auto rlen = [&](int i) { return lower ? C.diag[i] - C.rowptr[i] : C.rowptr[i + 1] - C.diag[i]; };
        for (int lv = 0; lv < nl; ++lv) {
            const int r0 = ptr[lv], m = ptr[lv + 1] - r0;
            std::stable_sort(rows.begin() + r0, rows.begin() + r0 + m, [&](int a, int b) { return rlen(a) > rlen(b); });
            const int w = m > 0 ? rlen(rows[r0]) : 0;
            slot = (slot + 3) & ~3;     // 16-byte aligned column-id range for the bulk copies
            base[lv] = slot;
            std::vector<int> off(w + 1, 0);
            for (int t = 0; t < w; ++t) {
                int mt = 0;
                while (mt < m && rlen(rows[r0 + mt]) > t) ++mt;
                off[t + 1] = off[t] + mt;
            }
            for (int q = 0; q < m; ++q) {
                const int i = rows[r0 + q];
                const int len = rlen(i);
                lens[r0 + q] = len;
                const int first = lower ? C.rowptr[i] : C.diag[i];
                for (int t = 0; t < len; ++t) C.pos[first + t] = slot + off[t] + q;
            }
            joff.insert(joff.end(), off.begin(), off.end());
            jptr[lv + 1] = (int)joff.size();
            slot += off[w];
            maxw = std::max(maxw, m);
        }
    };
    layout(C.lev_ptr, C.lev_rows, true, C.f_base, C.f_len, C.f_jptr, C.f_joff, C.max_fwidth);
    layout(C.levb_ptr, C.levb_rows, false, C.b_base, C.b_len, C.b_jptr, C.b_joff, C.max_bwidth);
    C.ell_total = ((slot + 3) & ~3) + 4;   // tail padding: bulk copies round up to 4 slots
    C.f_rows16.assign(C.lev_rows.begin(), C.lev_rows.end());
    C.b_rows16.assign(C.levb_rows.begin(), C.levb_rows.end());
    C.f_len8.assign(C.f_len.begin(), C.f_len.end());
    C.b_len8.assign(C.b_len.begin(), C.b_len.end());
    C.ecol.assign(C.ell_total, -1);
    for (int t = 0; t < C.nnzb; ++t) C.ecol[C.pos[t]] = C.col[t];
    C.jmap_csr = C.jmap;
    C.upd_csr = C.upd;
    {
        // every pattern entry written by the assembly?  (then the slots need no zero-fill pass)
        std::vector<char> hit(C.nnzb, 0);
        for (int j : C.jmap_csr)
            if (j >= 0) hit[j] = 1;
        bool all = true;
        for (int t = 0; t < C.nnzb; ++t) all = all && hit[t];
        C.prezero = (C.jdup || !all) ? 1 : 0;
    }
    for (auto &j : C.jmap)
        if (j >= 0) j = C.pos[j];
    for (auto &u : C.upd) {
        u.x = C.pos[u.x];
        u.y = C.pos[u.y];
    }
    C.lin.assign(nloc, 0);
    for (int l = 0; l < nloc; ++l) {
        const int ix = l % lx, iy = (l / lx) % ly, iz = l / (lx * ly);
        const long long rz = dim == 3 ? signed_rel(g, 2, rel[2][iz]) : 0;
        C.lin[l] = (int)((rz * g.ny + signed_rel(g, 1, rel[1][iy])) * g.nx + signed_rel(g, 0, rel[0][ix]));
    }
    C.owned.assign(nloc, 0);
    for (int l = 0; l < nloc; ++l) {
        const int ix[3] = {l % lx, (l / lx) % ly, l / (lx * ly)};
        bool own = true;
        for (int a = 0; a < dim; ++a) own = own && rel[a][ix[a]] >= 0 && rel[a][ix[a]] < own_len[a];
        C.owned[l] = own ? 1 : 0;
        if (own) C.own_list.push_back(l);
    }
    C.b_min_row = C.own_list.empty() ? 0 : C.own_list.front();
    C.nlevb_ras = 0;
    for (int k = 0; k + 1 < (int)C.levb_ptr.size(); ++k)
        for (int q = C.levb_ptr[k]; q < C.levb_ptr[k + 1]; ++q)
            if (C.levb_rows[q] >= C.b_min_row) C.nlevb_ras = k + 1;
    C.skip_blocks = 0;
    for (size_t q = 0; q < C.levb_rows.size(); ++q)
        if (C.levb_rows[q] < C.b_min_row) C.skip_blocks += C.b_len[q];
    return true;
}

// Column-major slot layout for apply_cols_kernel (narrow classes): L columns
// 0..n-1 (entries by ascending row), then U columns n-1..0, each led by the
// column's inverted diagonal block.  Replaces the level-major layout: pos[],
// the factorisation's slot tables and ell_total are rebuilt; the level
// schedules stay (the factorisation still runs level by level).
void relayout_columns(ClassHost &C)
{
    const int n = C.nloc;
    std::vector<std::vector<int>> lcol(n), ucol(n);
    for (int i = 0; i < n; ++i)
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t) {
            const int j = C.col[t];
            if (j < i) lcol[j].push_back(t);
            else if (j > i) ucol[j].push_back(t);
        }
    std::vector<int> row_of(C.nnzb);
    for (int i = 0; i < n; ++i)
        for (int t = C.rowptr[i]; t < C.rowptr[i + 1]; ++t) row_of[t] = i;
    C.pos.assign(C.nnzb, -1);
    C.col_steps.clear();
    C.col_ridx.clear();
    int slot = 0;
    auto place = [&](int t, int i) {
        C.pos[t] = slot++;
        C.col_ridx.push_back((unsigned short)i);
    };
    // the ring bookkeeping of apply_cols_kernel is a function of the class
    // only, so every step word carries it: how many new tiles the step must
    // wait for, how many it hands back to the TMA engine when it is done
    int ready = 0, freed = 0;
    auto push_step = [&](int j, int cnt, bool first, int slot_before) {
        const int total = cnt + (first ? 1 : 0);
        int nwait = 0;
        if (total > 0) {
            const int cl = (slot_before + total - 1) / kColTile;
            nwait = std::max(0, cl + 1 - ready);
            ready += nwait;
        }
        const int cf = (slot_before + total) / kColTile;
        const int nrel = cf - freed;
        freed = cf;
        C.col_steps.push_back((unsigned)j | ((unsigned)cnt << 16) | ((unsigned)nwait << 23) | ((unsigned)nrel << 25) |
                              (first ? 0x80000000u : 0u));
    };
    for (int j = 0; j < n; ++j) {
        const auto &e = lcol[j];
        for (size_t k = 0; k < e.size(); k += kColChunk) {
            const int cnt = (int)std::min<size_t>(kColChunk, e.size() - k);
            push_step(j, cnt, false, slot);
            for (int q = 0; q < cnt; ++q) place(e[k + q], row_of[e[k + q]]);
        }
    }
    C.col_nf = (int)C.col_steps.size();
    C.col_bstart = slot;
    C.col_nb_ras = 0;
    for (int j = n - 1; j >= 0; --j) {
        const auto &e = ucol[j];
        size_t k = 0;
        do {
            const int cnt = (int)std::min<size_t>(kColChunk, e.size() - k);
            push_step(j, cnt, k == 0, slot);
            if (k == 0) place(C.diag[j], j);
            for (int q = 0; q < cnt; ++q) place(e[k + q], row_of[e[k + q]]);
            k += cnt;
        } while (k < e.size());
        // left RAS stops after the first owned row's column (its entries update unowned rows only)
        if (j >= C.b_min_row) {
            C.col_nb_ras = (int)C.col_steps.size() - C.col_nf;
            C.col_end_ras = slot;
        }
    }
    C.col_nb = (int)C.col_steps.size() - C.col_nf;
    C.col_end = slot;
    C.col_steps.push_back(0u);   // spare words: the sweep reads one step ahead
    C.col_steps.push_back(0u);
    // whole TMA tiles: the last tile of the stream is read to its end
    C.ell_total = (slot + kColTile - 1) / kColTile * kColTile;
    C.col_ridx.resize(C.ell_total, 0);
    C.ecol.assign(C.ell_total, -1);
    for (int t = 0; t < C.nnzb; ++t) C.ecol[C.pos[t]] = C.col[t];
    C.jmap = C.jmap_csr;
    C.upd = C.upd_csr;
    for (auto &j : C.jmap)
        if (j >= 0) j = C.pos[j];
    for (auto &u : C.upd) {
        u.x = C.pos[u.x];
        u.y = C.pos[u.y];
    }
    C.skip_blocks = 0;
}

template <typename T>
size_t padded(size_t n) { return ((n * sizeof(T) + 255) / 256) * 256; }

// shared-memory image of a class for apply_group_kernel (ClassDev::meta)
void build_meta(ClassHost &C)
{
    size_t at = 0;
    auto seg = [&](size_t bytes) { size_t o = at; at += (bytes + 15) / 16 * 16; return (int)o; };
    const int nlev = (int)C.lev_ptr.size() - 1, nlevb = (int)C.levb_ptr.size() - 1;
    int *m = C.m_off;
    m[0] = seg(sizeof(int) * (nlev + 1));
    m[1] = seg(sizeof(int) * nlev);
    m[2] = seg(sizeof(int) * (nlevb + 1));
    m[3] = seg(sizeof(int) * nlevb);
    m[4] = seg(2 * (size_t)C.nloc);
    m[5] = seg(2 * (size_t)C.nloc);
    m[6] = seg(2 * (size_t)C.nloc);
    m[7] = seg(2 * (size_t)C.nloc);
    // jagged offsets (+ kJoPad zero entries so a sweep may read MAXW past the last level)
    constexpr size_t kJoPad = 64;
    m[9] = seg(sizeof(int) * C.f_jptr.size());
    m[10] = seg(sizeof(int) * C.b_jptr.size());
    m[11] = seg(2 * (C.f_joff.size() + kJoPad));
    m[12] = seg(2 * (C.b_joff.size() + kJoPad));
    // gather / scatter: linear offsets (boxes that do not wrap), packed local
    // coordinates + per-axis relative coordinates (boxes that wrap), owned list
    const int lx = (int)C.rel[0].size(), ly = (int)C.rel[1].size(), lz = C.rel[2].empty() ? 1 : (int)C.rel[2].size();
    m[13] = seg(sizeof(int) * (size_t)C.nloc);
    m[14] = seg(sizeof(unsigned) * (size_t)C.nloc);
    m[15] = seg(2 * std::max<size_t>(1, C.own_list.size()));
    m[16] = seg(sizeof(int) * (size_t)(lx + ly + lz));
    m[8] = seg(2 * (size_t)C.ell_total);   // slot column ids
    C.meta.assign(at, 0);
    auto put = [&](int o, const void *src, size_t bytes) { if (bytes) memcpy(C.meta.data() + o, src, bytes); };
    put(m[0], C.lev_ptr.data(), sizeof(int) * (nlev + 1));
    put(m[1], C.f_base.data(), sizeof(int) * nlev);
    put(m[2], C.levb_ptr.data(), sizeof(int) * (nlevb + 1));
    put(m[3], C.b_base.data(), sizeof(int) * nlevb);
    put(m[4], C.f_rows16.data(), 2 * (size_t)C.nloc);
    put(m[5], C.b_rows16.data(), 2 * (size_t)C.nloc);
    put(m[6], C.f_len8.data(), 2 * (size_t)C.nloc);
    put(m[7], C.b_len8.data(), 2 * (size_t)C.nloc);
    std::vector<unsigned short> e16(C.ell_total);
    for (int t = 0; t < C.ell_total; ++t) e16[t] = C.ecol[t] < 0 ? 0 : (unsigned short)C.ecol[t];
    put(m[8], e16.data(), 2 * (size_t)C.ell_total);
    put(m[9], C.f_jptr.data(), sizeof(int) * C.f_jptr.size());
    put(m[10], C.b_jptr.data(), sizeof(int) * C.b_jptr.size());
    std::vector<unsigned short> j16(C.f_joff.begin(), C.f_joff.end());
    put(m[11], j16.data(), 2 * j16.size());
    j16.assign(C.b_joff.begin(), C.b_joff.end());
    put(m[12], j16.data(), 2 * j16.size());
    put(m[13], C.lin.data(), sizeof(int) * C.lin.size());
    std::vector<unsigned> ixyz(C.nloc);
    for (int l = 0; l < C.nloc; ++l)
        ixyz[l] = (unsigned)(l % lx) | ((unsigned)((l / lx) % ly) << 10) | ((unsigned)(l / (lx * ly)) << 20);
    put(m[14], ixyz.data(), sizeof(unsigned) * ixyz.size());
    std::vector<unsigned short> o16(C.own_list.begin(), C.own_list.end());
    put(m[15], o16.data(), 2 * o16.size());
    std::vector<int> rl;
    for (int a = 0; a < 3; ++a) {
        const int la = a == 0 ? lx : (a == 1 ? ly : lz);
        for (int i = 0; i < la; ++i) rl.push_back(C.rel[a].empty() ? 0 : C.rel[a][i]);
    }
    put(m[16], rl.data(), sizeof(int) * rl.size());
}

acch_status upload_class(ClassHost &C)
{
    build_meta(C);
    size_t total = 0;
    auto add = [&](size_t bytes) { size_t o = total; total += ((bytes + 255) / 256) * 256; return o; };
    size_t o_rel[3];
    for (int a = 0; a < 3; ++a) o_rel[a] = add(sizeof(int) * std::max<size_t>(1, C.rel[a].size()));
    const size_t o_rp = add(sizeof(int) * C.rowptr.size()), o_ci = add(sizeof(int) * C.col.size());
    const size_t o_dg = add(sizeof(int) * C.diag.size()), o_jm = add(sizeof(int) * C.jmap.size());
    const size_t o_up = add(sizeof(int) * C.upd_ptr.size()), o_ud = add(sizeof(int2) * std::max<size_t>(1, C.upd.size()));
    const size_t o_lp = add(sizeof(int) * C.lev_ptr.size()), o_lr = add(sizeof(int) * C.lev_rows.size());
    const size_t o_bp = add(sizeof(int) * C.levb_ptr.size()), o_br = add(sizeof(int) * C.levb_rows.size());
    const size_t o_ow = add(C.owned.size());
    const size_t o_ps = add(sizeof(int) * C.pos.size()), o_fb = add(sizeof(int) * C.f_base.size());
    const size_t o_fl = add(sizeof(int) * C.f_len.size()), o_bb = add(sizeof(int) * C.b_base.size());
    const size_t o_bl = add(sizeof(int) * C.b_len.size()), o_ec = add(sizeof(int) * C.ecol.size());
    const size_t o_fr16 = add(2 * C.f_rows16.size()), o_br16 = add(2 * C.b_rows16.size());
    const size_t o_fl8 = add(2 * C.f_len8.size()), o_bl8 = add(2 * C.b_len8.size());
    const size_t o_fjp = add(sizeof(int) * C.f_jptr.size()), o_fjo = add(sizeof(int) * std::max<size_t>(1, C.f_joff.size()));
    const size_t o_bjp = add(sizeof(int) * C.b_jptr.size()), o_bjo = add(sizeof(int) * std::max<size_t>(1, C.b_joff.size()));
    const size_t o_meta = add(C.meta.size());
    const size_t o_lin = add(sizeof(int) * C.lin.size());
    const size_t o_own = add(sizeof(int) * std::max<size_t>(1, C.own_list.size()));
    const size_t o_cs = add(sizeof(unsigned) * std::max<size_t>(1, C.col_steps.size()));
    const size_t o_cr = add(2 * std::max<size_t>(1, C.col_ridx.size()));
    ACCH_CUDA(cudaMalloc(&C.dev_mem, total));
    std::vector<unsigned char> h(total, 0);
    auto put = [&](size_t o, const void *src, size_t bytes) { if (bytes) memcpy(h.data() + o, src, bytes); };
    for (int a = 0; a < 3; ++a) put(o_rel[a], C.rel[a].data(), sizeof(int) * C.rel[a].size());
    put(o_rp, C.rowptr.data(), sizeof(int) * C.rowptr.size());
    put(o_ci, C.col.data(), sizeof(int) * C.col.size());
    put(o_dg, C.diag.data(), sizeof(int) * C.diag.size());
    put(o_jm, C.jmap.data(), sizeof(int) * C.jmap.size());
    put(o_up, C.upd_ptr.data(), sizeof(int) * C.upd_ptr.size());
    put(o_ud, C.upd.data(), sizeof(int2) * C.upd.size());
    put(o_lp, C.lev_ptr.data(), sizeof(int) * C.lev_ptr.size());
    put(o_lr, C.lev_rows.data(), sizeof(int) * C.lev_rows.size());
    put(o_bp, C.levb_ptr.data(), sizeof(int) * C.levb_ptr.size());
    put(o_br, C.levb_rows.data(), sizeof(int) * C.levb_rows.size());
    put(o_ow, C.owned.data(), C.owned.size());
    put(o_ps, C.pos.data(), sizeof(int) * C.pos.size());
    put(o_fb, C.f_base.data(), sizeof(int) * C.f_base.size());
    put(o_fl, C.f_len.data(), sizeof(int) * C.f_len.size());
    put(o_bb, C.b_base.data(), sizeof(int) * C.b_base.size());
    put(o_bl, C.b_len.data(), sizeof(int) * C.b_len.size());
    put(o_ec, C.ecol.data(), sizeof(int) * C.ecol.size());
    put(o_fr16, C.f_rows16.data(), 2 * C.f_rows16.size());
    put(o_br16, C.b_rows16.data(), 2 * C.b_rows16.size());
    put(o_fl8, C.f_len8.data(), 2 * C.f_len8.size());
    put(o_bl8, C.b_len8.data(), 2 * C.b_len8.size());
    put(o_fjp, C.f_jptr.data(), sizeof(int) * C.f_jptr.size());
    put(o_fjo, C.f_joff.data(), sizeof(int) * C.f_joff.size());
    put(o_bjp, C.b_jptr.data(), sizeof(int) * C.b_jptr.size());
    put(o_bjo, C.b_joff.data(), sizeof(int) * C.b_joff.size());
    put(o_meta, C.meta.data(), C.meta.size());
    put(o_lin, C.lin.data(), sizeof(int) * C.lin.size());
    put(o_own, C.own_list.data(), sizeof(int) * C.own_list.size());
    put(o_cs, C.col_steps.data(), sizeof(unsigned) * C.col_steps.size());
    put(o_cr, C.col_ridx.data(), 2 * C.col_ridx.size());
    ACCH_CUDA(cudaMemcpy(C.dev_mem, h.data(), total, cudaMemcpyHostToDevice));
    unsigned char *b = (unsigned char *)C.dev_mem;
    ClassDev &d = C.dev;
    d.nloc = C.nloc;
    d.nnzb = C.nnzb;
    d.nlev = (int)C.lev_ptr.size() - 1;
    d.nlevb = (int)C.levb_ptr.size() - 1;
    for (int a = 0; a < 3; ++a) {
        d.len[a] = C.rel[a].empty() ? 1 : (int)C.rel[a].size();
        d.rel[a] = (const int *)(b + o_rel[a]);
    }
    d.rowptr = (const int *)(b + o_rp);
    d.col = (const int *)(b + o_ci);
    d.diag = (const int *)(b + o_dg);
    d.jmap = (const int *)(b + o_jm);
    d.upd_ptr = (const int *)(b + o_up);
    d.upd = (const int2 *)(b + o_ud);
    d.lev_ptr = (const int *)(b + o_lp);
    d.lev_rows = (const int *)(b + o_lr);
    d.levb_ptr = (const int *)(b + o_bp);
    d.levb_rows = (const int *)(b + o_br);
    d.owned = (const unsigned char *)(b + o_ow);
    d.pos = (const int *)(b + o_ps);
    d.f_base = (const int *)(b + o_fb);
    d.f_len = (const int *)(b + o_fl);
    d.b_base = (const int *)(b + o_bb);
    d.b_len = (const int *)(b + o_bl);
    d.ecol = (const int *)(b + o_ec);
    d.f_rows16 = (const unsigned short *)(b + o_fr16);
    d.b_rows16 = (const unsigned short *)(b + o_br16);
    d.f_len8 = (const unsigned short *)(b + o_fl8);
    d.b_len8 = (const unsigned short *)(b + o_bl8);
    d.f_jptr = (const int *)(b + o_fjp);
    d.f_joff = (const int *)(b + o_fjo);
    d.b_jptr = (const int *)(b + o_bjp);
    d.b_joff = (const int *)(b + o_bjo);
    d.meta = b + o_meta;
    d.lin = (const int *)(b + o_lin);
    d.own_list = (const int *)(b + o_own);
    d.n_owned = (int)C.own_list.size();
    d.b_min_row = C.b_min_row;
    d.nlevb_ras = C.nlevb_ras;
    d.jdup = C.jdup;
    d.prezero = C.prezero;
    d.col_steps = (const unsigned *)(b + o_cs);
    d.col_ridx = (const unsigned short *)(b + o_cr);
    d.col_nf = C.col_nf;
    d.col_nb = C.col_nb;
    d.col_nb_ras = C.col_nb_ras;
    d.col_bstart = C.col_bstart;
    d.col_end = C.col_end;
    d.col_end_ras = C.col_end_ras;
    d.meta_bytes = (int)C.meta.size();
    d.m_fbs = C.m_off[1];
    d.m_bptr = C.m_off[2];
    d.m_bbs = C.m_off[3];
    d.m_frows = C.m_off[4];
    d.m_brows = C.m_off[5];
    d.m_flen = C.m_off[6];
    d.m_blen = C.m_off[7];
    d.m_ecol = C.m_off[8];
    d.m_fjp = C.m_off[9];
    d.m_bjp = C.m_off[10];
    d.m_fjo = C.m_off[11];
    d.m_bjo = C.m_off[12];
    d.m_lin = C.m_off[13];
    d.m_ixyz = C.m_off[14];
    d.m_own = C.m_off[15];
    d.m_rel = C.m_off[16];
    d.ell_total = C.ell_total;
    d.max_fwidth = C.max_fwidth;
    d.max_bwidth = C.max_bwidth;
    return ACCH_OK;
}

}  // namespace

struct acch_precond {
    acch_ctx *ctx = nullptr;
    int variant = 1, fill = 0, dim = 2;
    long long nsub = 0;
    std::vector<ClassHost> classes;
    std::vector<int> sub_class;
    std::vector<int4> sub_origin;
    std::vector<long long> sub_off, sub_ext_off;
    ClassDev *d_classes = nullptr;
    int *d_sub_class = nullptr;
    int4 *d_sub_origin = nullptr;
    long long *d_sub_off = nullptr, *d_sub_ext_off = nullptr;
    double4 *d_vals = nullptr;
    int wide = 0;                 // some factor row exceeds kWideLen blocks (LU / high fill): warp-wide rows
    long long total_blocks = 0, total_ext = 0, total_nnzb = 0;
    long long total_skip = 0;   // left-RAS backward blocks the class-group solver never reads
    int *d_bad = nullptr;
    double2 *d_ext_out = nullptr;
    long long *d_cell_ptr = nullptr, *d_cell_src = nullptr;
    bool have_factors = false;
    long long factorizations = 0;
    size_t apply_smem = 0;
    int use_smem = 1;
    int tps = 32;          // threads per subdomain in the solves
    int max_nloc = 0;
    int warp_mode = 0;     // apply_warp_kernel usable
    int col_mode = 0;      // apply_cols_kernel: narrow classes (every level <= kWideRows rows, long rows), column-major factors
    ColSmem cl{0, 0, 0};
    // class-group solver (apply_group_kernel): groups of <= group_nw subdomains of one class
    int group_mode = 0, group_nw = 8, group_per_warp = 1, meta_max = 0, y_stride = 0;
    int factor_threads = 0;   // threads per subdomain CTA of factor_kernel (32 / 64 / 128)
    size_t group_smem = 0;
    std::vector<int4> groups;
    int4 *d_groups = nullptr;
    int *d_grp_sub = nullptr;
    int pf_depth = 3;      // levels prefetched ahead into L2 (ACCH_PREFETCH_DEPTH overrides; 3 measured best for the group solver with capped levels)
    WarpSmem wl{0, 0, 0};
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per kernel, so
// every preconditioner raises it to the device's opt-in maximum (a smaller
// value set by a later preconditioner would break launches of an earlier one)
static int smem_optin()
{
    int dev = 0, v = 48 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

static void free_precond(acch_precond *pc)
{
    for (auto &C : pc->classes)
        if (C.dev_mem) cudaFree(C.dev_mem);
    cudaFree(pc->d_classes);
    cudaFree(pc->d_sub_class);
    cudaFree(pc->d_sub_origin);
    cudaFree(pc->d_sub_off);
    cudaFree(pc->d_sub_ext_off);
    cudaFree(pc->d_vals);
    cudaFree(pc->d_bad);
    cudaFree(pc->d_ext_out);
    cudaFree(pc->d_cell_ptr);
    cudaFree(pc->d_cell_src);
    cudaFree(pc->d_groups);
    cudaFree(pc->d_grp_sub);
}

extern "C" acch_status acch_precond_create(acch_ctx *ctx, int64_t n_sub, int32_t overlap, const int64_t *owned_lo,
                                           const int64_t *owned_hi, int32_t variant, int32_t fill_level,
                                           acch_precond **out)
{
    if (!ctx || !out || n_sub < 1 || overlap < 0 || !owned_lo || !owned_hi || variant < 0 || variant > 2) {
        acch_set_error("acch_precond_create: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    if (ctx->g.zg > 0 && (variant != 1 || overlap > ctx->g.zg)) {
        acch_set_error("acch_precond_create: slab mode supports left-RAS with overlap <= ghost planes");
        return ACCH_ERR_INVALID_ARG;
    }
    const GridDev &g = ctx->g;
    const int dim = g.dim;
    const int nn[3] = {g.nx, g.ny, g.nz};
    auto *pc = new acch_precond();
    pc->ctx = ctx;
    pc->variant = variant;
    pc->fill = fill_level;
    pc->dim = dim;
    pc->nsub = n_sub;
    std::map<std::vector<int>, int> sig2class;
    for (long long s = 0; s < n_sub; ++s) {
        std::array<std::vector<int>, 3> rel;
        int own_len[3] = {1, 1, 1};
        int lo3[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) {
            const long long lo = owned_lo[3 * s + a], hi = owned_hi[3 * s + a];
            if (lo < 0 || hi > nn[a] || hi <= lo) {
                delete pc;
                acch_set_error("acch_precond_create: owned box out of range");
                return ACCH_ERR_PARTITION;
            }
            lo3[a] = (int)lo;
            own_len[a] = (int)(hi - lo);
            std::vector<int> ext;
            if (a == 2 && g.zg > 0) {
                // slab mode: z never wraps locally; an overlap past an interior
                // slab boundary lands in the ghost planes, a physical wall clips
                const long long zlo = g.zwall_lo ? 0 : -(long long)g.zg, zhi = g.zwall_hi ? nn[a] : nn[a] + g.zg;
                std::vector<long long> cs;
                for (long long c = std::max<long long>(lo - overlap, zlo); c < std::min<long long>(hi + overlap, zhi); ++c)
                    cs.push_back(c);
                // the reference orders a box's cells by sorted GLOBAL id: a ghost
                // plane that wraps around the periodic z axis sorts to the other end
                const long long ng = ctx->nz_global, z0 = ctx->z_offset;
                std::stable_sort(cs.begin(), cs.end(), [&](long long a, long long b) {
                    return ((z0 + a) % ng + ng) % ng < ((z0 + b) % ng + ng) % ng;
                });
                for (long long c : cs) ext.push_back((int)(c - lo));
            } else if (g.periodic) {
                std::vector<int> all;
                for (long long c = lo - overlap; c < hi + overlap; ++c) all.push_back((int)(((c % nn[a]) + nn[a]) % nn[a]));
                std::sort(all.begin(), all.end());
                all.erase(std::unique(all.begin(), all.end()), all.end());
                for (int c : all) ext.push_back(((c - (int)lo) % nn[a] + nn[a]) % nn[a]);
            } else {
                for (long long c = std::max<long long>(lo - overlap, 0); c < std::min<long long>(hi + overlap, nn[a]); ++c)
                    ext.push_back((int)(c - lo));
            }
            rel[a] = ext;
        }
        std::vector<int> sig;
        for (int a = 0; a < dim; ++a) {
            sig.push_back((int)rel[a].size());
            sig.push_back(own_len[a]);
            sig.insert(sig.end(), rel[a].begin(), rel[a].end());
        }
        auto f = sig2class.find(sig);
        int cls;
        if (f == sig2class.end()) {
            cls = (int)pc->classes.size();
            sig2class.emplace(sig, cls);
            pc->classes.emplace_back();
            std::string err;
            if (!build_class(g, rel, own_len, fill_level, pc->classes.back(), err)) {
                free_precond(pc);
                delete pc;
                acch_set_error("acch_precond_create: " + err);
                return ACCH_ERR_INVALID_ARG;
            }
        } else {
            cls = f->second;
        }
        pc->sub_class.push_back(cls);
        // w = 1: every cell of the box sits at origin + rel without wrapping
        // (slab z: ghost planes are stored), so its storage index is linear
        int nowrap = 1;
        for (int a = 0; a < dim; ++a) {
            if (a == 2 && g.zg > 0) continue;
            for (int r : rel[a]) {
                const int d = signed_rel(g, a, r);
                if (lo3[a] + d < 0 || lo3[a] + d >= nn[a]) nowrap = 0;
            }
        }
        pc->sub_origin.push_back(make_int4(lo3[0], lo3[1], lo3[2], nowrap));
    }
    int max_width = 0, max_nloc = 0, max_len = 0;
    for (const auto &C : pc->classes) {
        max_width = std::max(max_width, std::max(C.max_fwidth, C.max_bwidth));
        max_nloc = std::max(max_nloc, C.nloc);
        for (int v : C.f_len) max_len = std::max(max_len, v);
        for (int v : C.b_len) max_len = std::max(max_len, v - 1);
    }
    // Narrow classes (every level <= kWideRows rows) with long rows -- exact
    // LU, ILU(k >= 1) -- are solved by column sweeps on column-major factors
    // (apply_cols_kernel); ACCH_NARROW=0 keeps the level-major solvers.
    pc->col_mode = max_width <= kWideRows && max_len > kWideLen && max_nloc <= 65535;
    if (const char *e = getenv("ACCH_NARROW")) pc->col_mode = pc->col_mode && atoi(e) != 0;
    if (const char *e = getenv("ACCH_WIDE_ROWS")) pc->col_mode = pc->col_mode && atoi(e) != 0;
    if (pc->col_mode) {
        int max_steps = 0;
        for (auto &C : pc->classes) {
            relayout_columns(C);
            max_steps = std::max(max_steps, C.col_nf + C.col_nb);
        }
        // the step table goes to shared memory when every subdomain is resident anyway
        pc->cl = ColSmem{max_nloc, max_steps, 1};
        {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
            const long long fit = (long long)sms * std::min<long long>(8, (227 * 1024) / (long long)(pc->cl.bytes() + 1024));
            if (n_sub > fit) pc->cl.steps_smem = 0;
        }
        if (pc->cl.bytes() > 200 * 1024) {
            free_precond(pc);
            delete pc;
            acch_set_error("acch_precond_create: subdomain too large for the column solver (set ACCH_NARROW=0)");
            return ACCH_ERR_INVALID_ARG;
        }
    }
    // offsets
    long long vo = 0, eo = 0;
    pc->sub_off.assign(n_sub, 0);
    for (long long s = 0; s < n_sub; ++s) {
        const ClassHost &C = pc->classes[pc->sub_class[s]];
        pc->sub_off[s] = vo;
        vo += C.ell_total;
        pc->sub_ext_off.push_back(eo);
        eo += C.nloc;
        pc->total_nnzb += C.nnzb;
        pc->total_skip += C.skip_blocks;
    }
    pc->total_blocks = vo;
    pc->total_ext = eo;
    pc->max_nloc = max_nloc;
    pc->tps = max_width <= 64 ? 32 : 128;
    {
        int mnl = 0, mnb = 0;
        for (const auto &C : pc->classes) {
            mnl = std::max(mnl, (int)C.lev_ptr.size() - 1);
            mnb = std::max(mnb, (int)C.levb_ptr.size() - 1);
        }
        pc->wl = WarpSmem{max_nloc, mnl, mnb};
        pc->wide = max_len > kWideLen;   // exact LU / high fill: warp-wide sweeps of narrow levels
        if (const char *e = getenv("ACCH_WIDE_ROWS")) pc->wide = pc->wide && atoi(e) != 0;
        pc->warp_mode = (max_width <= 64 && max_nloc <= 65535 && pc->wl.bytes() <= 200 * 1024) ? 1 : 0;
        if (const char *e = getenv("ACCH_PREFETCH_DEPTH")) pc->pf_depth = atoi(e);
        if (const char *e = getenv("ACCH_SCHWARZ_BLOCK_SOLVER"))   // testing: force the CTA-wide solver
            if (atoi(e)) pc->warp_mode = 0, pc->tps = 128;
        if (getenv("ACCH_DEBUG"))
            fprintf(stderr, "[acch] precond: %lld subdomains, %zu classes, max_nloc %d, max level width %d, "
                            "max row %d, warp smem %zu B -> %s solver\n",
                    (long long)n_sub, pc->classes.size(), max_nloc, max_width, max_len, pc->wl.bytes(),
                    pc->col_mode ? "column-sweep" : (pc->warp_mode ? "warp" : "CTA"));
    }
    const int groups = 128 / pc->tps;
    pc->apply_smem = sizeof(double2) * (size_t)max_nloc * groups;
    pc->use_smem = pc->apply_smem <= 200 * 1024 ? 1 : 0;
    if (!pc->use_smem) pc->apply_smem = 0;

#define PC_CUDA(call)                                        \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) {                             \
            free_precond(pc);                                \
            delete pc;                                       \
            return acch_cuda_fail(_e, #call);                \
        }                                                    \
    } while (0)
    for (auto &C : pc->classes) {
        acch_status st = upload_class(C);
        if (st != ACCH_OK) {
            free_precond(pc);
            delete pc;
            return st;
        }
    }
    std::vector<ClassDev> cd;
    for (auto &C : pc->classes) cd.push_back(C.dev);
    PC_CUDA(cudaMalloc(&pc->d_classes, sizeof(ClassDev) * cd.size()));
    PC_CUDA(cudaMemcpy(pc->d_classes, cd.data(), sizeof(ClassDev) * cd.size(), cudaMemcpyHostToDevice));
    PC_CUDA(cudaMalloc(&pc->d_sub_class, sizeof(int) * n_sub));
    PC_CUDA(cudaMemcpy(pc->d_sub_class, pc->sub_class.data(), sizeof(int) * n_sub, cudaMemcpyHostToDevice));
    PC_CUDA(cudaMalloc(&pc->d_sub_origin, sizeof(int4) * n_sub));
    PC_CUDA(cudaMemcpy(pc->d_sub_origin, pc->sub_origin.data(), sizeof(int4) * n_sub, cudaMemcpyHostToDevice));
    PC_CUDA(cudaMalloc(&pc->d_sub_off, sizeof(long long) * n_sub));
    PC_CUDA(cudaMemcpy(pc->d_sub_off, pc->sub_off.data(), sizeof(long long) * n_sub, cudaMemcpyHostToDevice));
    PC_CUDA(cudaMalloc(&pc->d_sub_ext_off, sizeof(long long) * n_sub));
    PC_CUDA(cudaMemcpy(pc->d_sub_ext_off, pc->sub_ext_off.data(), sizeof(long long) * n_sub, cudaMemcpyHostToDevice));
    PC_CUDA(cudaMalloc(&pc->d_vals, sizeof(double4) * std::max<long long>(1, pc->total_blocks)));
    // padding slots (level alignment, tile tails) are prefetched or copied but never used in arithmetic
    PC_CUDA(cudaMemset(pc->d_vals, 0, sizeof(double4) * std::max<long long>(1, pc->total_blocks)));
    PC_CUDA(cudaMalloc(&pc->d_bad, sizeof(int) * n_sub));
    const bool need_ext = variant != 1 || !pc->use_smem;
    if (need_ext) PC_CUDA(cudaMalloc(&pc->d_ext_out, sizeof(double2) * std::max<long long>(1, pc->total_ext)));
    if (variant != 1) {
        // per-cell contributor lists in subdomain order
        const long long N = g.n;
        std::vector<long long> cnt(N + 1, 0);
        std::vector<std::pair<long long, long long>> ent;   // (cell, ext index)
        ent.reserve(pc->total_ext);
        for (long long s = 0; s < n_sub; ++s) {
            const ClassHost &C = pc->classes[pc->sub_class[s]];
            const int lx = (int)C.rel[0].size(), ly = (int)C.rel[1].size();
            for (int l = 0; l < C.nloc; ++l) {
                const int ix = l % lx, iy = (l / lx) % ly, iz = l / (lx * ly);
                long long gc[3] = {0, 0, 0};
                const int o3[3] = {pc->sub_origin[s].x, pc->sub_origin[s].y, pc->sub_origin[s].z};
                const int id3[3] = {ix, iy, iz};
                for (int a = 0; a < dim; ++a) {
                    int c = o3[a] + C.rel[a][id3[a]];
                    if (g.periodic) c = ((c % nn[a]) + nn[a]) % nn[a];
                    gc[a] = c;
                }
                const long long cell = (gc[2] * g.ny + gc[1]) * g.nx + gc[0];
                ent.emplace_back(cell, pc->sub_ext_off[s] + l);
                cnt[cell + 1]++;
            }
        }
        for (long long c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
        std::vector<long long> src(ent.size());
        std::vector<long long> fillp(cnt.begin(), cnt.end() - 1);
        for (const auto &e : ent) src[fillp[e.first]++] = e.second;   // ent is in subdomain order
        PC_CUDA(cudaMalloc(&pc->d_cell_ptr, sizeof(long long) * (N + 1)));
        PC_CUDA(cudaMemcpy(pc->d_cell_ptr, cnt.data(), sizeof(long long) * (N + 1), cudaMemcpyHostToDevice));
        PC_CUDA(cudaMalloc(&pc->d_cell_src, sizeof(long long) * std::max<size_t>(1, src.size())));
        PC_CUDA(cudaMemcpy(pc->d_cell_src, src.data(), sizeof(long long) * src.size(), cudaMemcpyHostToDevice));
    }
    if (pc->use_smem && pc->apply_smem > 48 * 1024) {
        const int b = smem_optin();   // per-function state: never lower it under another live preconditioner
        const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<0, 32>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<1, 32>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<2, 32>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<0, 128>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<1, 128>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<2, 128>, attr, b));
    }
    {
        // the solvers live on shared memory: ask for the full L1/shared carveout
        const auto co = cudaFuncAttributePreferredSharedMemoryCarveout;
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<0, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<1, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<2, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<0, false>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<1, false>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<2, false>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 4>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 4, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 4>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 4, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 4>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 4, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 8>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 8, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 8>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 8, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 8>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 8, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 16>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 16, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 16>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 16, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 16>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 16, true>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<0, 32>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<1, 32>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<2, 32>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<0, 128>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<1, 128>, co, 100));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<2, 128>, co, 100));
    }
    if (pc->col_mode) {
        const cudaFuncAttribute attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
        const int b = smem_optin();
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<0, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<1, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<2, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<0, false>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<1, false>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_cols_kernel<2, false>, attr, b));
    }
    if (pc->warp_mode && pc->wl.bytes() > 48 * 1024) {
        const int b = smem_optin();   // per-function state: never lower it under another live preconditioner
        const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 4>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 4, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 4>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 4, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 4>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 4, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 8>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 8, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 8>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 8, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 8>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 8, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 16>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<0, 12, 16, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 16>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<1, 12, 16, true>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 16>, attr, b));
        PC_CUDA(cudaFuncSetAttribute(apply_warp_kernel<2, 12, 16, true>, attr, b));
    }
    {
        // class-group solver: NW subdomains of one class per CTA sharing the
        // class's symbolic data in shared memory (ACCH_GROUP=0 disables,
        // ACCH_GROUP_WARPS=4|8 picks the group size)
        int meta_max = 0;
        for (const auto &C : pc->classes) meta_max = std::max(meta_max, (int)C.meta.size());
        pc->meta_max = (meta_max + 15) / 16 * 16;
        pc->y_stride = (int)((sizeof(double2) * (size_t)max_nloc + 15) / 16 * 16);
        int enable = pc->warp_mode && !pc->col_mode;   // column-major factors: apply_cols_kernel only
        if (const char *e = getenv("ACCH_GROUP")) enable = enable && atoi(e) != 0;
        int nw = 8;
        if (const char *e = getenv("ACCH_GROUP_WARPS")) nw = atoi(e) <= 4 ? 4 : 8;
        const size_t limit = 227 * 1024;
        while (nw >= 4 && (size_t)pc->meta_max + (size_t)nw * pc->y_stride > limit) nw /= 2;
        // (a class image too large for a group -- ILU(2) / LU on 10^3-cell
        // boxes, 349 KB -- stays on the warp solver: staging the image
        // without its slot column ids, read from global memory instead, fits
        // 4 warps per SM and measured 11.2 vs 8.0 ms per apply at 128^3)
        if (enable && nw >= 4) {
            pc->group_mode = 1;
            pc->group_nw = nw;
            pc->group_smem = (size_t)pc->meta_max + (size_t)nw * pc->y_stride;
            std::vector<std::vector<int>> members(pc->classes.size());
            for (long long s = 0; s < n_sub; ++s) members[pc->sub_class[s]].push_back((int)s);
            const long long per = 1;
            pc->group_per_warp = (int)per;
            const size_t gsize = (size_t)nw * per;
            std::vector<int> order;
            for (size_t c = 0; c < members.size(); ++c)
                for (size_t i = 0; i < members[c].size(); i += gsize) {
                    const int cnt = (int)std::min<size_t>(gsize, members[c].size() - i);
                    pc->groups.push_back(make_int4((int)c, (int)order.size(), cnt, 0));
                    for (int q = 0; q < cnt; ++q) order.push_back(members[c][i + q]);
                }
            PC_CUDA(cudaMalloc(&pc->d_groups, sizeof(int4) * pc->groups.size()));
            PC_CUDA(cudaMalloc(&pc->d_grp_sub, sizeof(int) * order.size()));
            PC_CUDA(cudaMemcpy(pc->d_groups, pc->groups.data(), sizeof(int4) * pc->groups.size(),
                               cudaMemcpyHostToDevice));
            PC_CUDA(cudaMemcpy(pc->d_grp_sub, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
            const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
            const int b = smem_optin();   // per-function state: never lower it under another live preconditioner
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<0, 8>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<1, 8>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<2, 8>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<0, 4>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<1, 4>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<2, 4>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<0, 8, 12, double4, true>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<1, 8, 12, double4, true>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<2, 8, 12, double4, true>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<0, 4, 12, double4, true>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<1, 4, 12, double4, true>, attr, b));
            PC_CUDA(cudaFuncSetAttribute(apply_group_kernel<2, 4, 12, double4, true>, attr, b));
        }
        if (getenv("ACCH_DEBUG"))
        {
            int occ = 0;
            if (pc->group_mode)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apply_group_kernel<1, 8>, pc->group_nw * 32,
                                                              pc->group_smem);
            fprintf(stderr, "[acch] group solver %s: %d warps/CTA, %d subdomains/warp, %zu groups, meta %d B, "
                            "smem %zu B, CTAs/SM %d\n",
                    pc->group_mode ? "on" : "off", pc->group_nw, pc->group_per_warp, pc->groups.size(),
                    pc->meta_max, pc->group_smem, occ);
        }
    }
    {
        // threads per subdomain CTA of factor_kernel, fixed at creation: a 3D
        // ILU level is at most 32 rows wide, so one warp per subdomain keeps
        // every lane busy and fits 4x the subdomains per SM (128^3 ILU(2)
        // 455 -> 262 ms, 256^3 ILU(0) 101.7 -> 86.6 ms, profiles/r01_factor_threads.txt);
        // in 2D (LU) 128 measured faster.  ACCH_FACTOR_THREADS = 32 | 64 | 128
        // overrides (the factors are bitwise the same for every choice -- the
        // per-row update order does not depend on it; tested).
        int nt = dim == 3 ? 32 : kFactorThreads;
        if (const char *e = getenv("ACCH_FACTOR_THREADS")) {
            nt = atoi(e);
            if (nt != 32 && nt != 64 && nt != 128) {
                free_precond(pc);
                delete pc;
                acch_set_error("ACCH_FACTOR_THREADS must be 32, 64 or 128");
                return ACCH_ERR_INVALID_ARG;
            }
        }
        pc->factor_threads = nt;
    }
#undef PC_CUDA
    *out = pc;
    return ACCH_OK;
}

extern "C" acch_status acch_precond_destroy(acch_precond *pc)
{
    if (!pc) return ACCH_OK;
    free_precond(pc);
    delete pc;
    return ACCH_OK;
}

extern "C" acch_status acch_precond_invalidate(acch_precond *pc)
{
    if (!pc) {
        acch_set_error("acch_precond_invalidate: null handle");
        return ACCH_ERR_INVALID_ARG;
    }
    pc->have_factors = false;
    return ACCH_OK;
}

extern "C" acch_status acch_precond_update(acch_precond *pc, const double *coef, double dt, int32_t reuse,
                                           int32_t *refactored, int64_t *bad_cell, int32_t *bad_comp)
{
    if (!pc || !coef) {
        acch_set_error("acch_precond_update: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    if (refactored) *refactored = 0;
    if (reuse && pc->have_factors) return ACCH_OK;
    acch_ctx *ctx = pc->ctx;
    ACCH_CUDA(cudaMemsetAsync(pc->d_bad, 0x7f, sizeof(int) * pc->nsub, ctx->stream));
    ProfScope prof_scope(ctx, PC_FACTOR, 32.0 * pc->total_nnzb + 56.0 * pc->total_ext);
    {
        const int nt = pc->factor_threads;
#define FK(D, NT) factor_kernel<D, NT><<<(unsigned)pc->nsub, NT, 0, ctx->stream>>>( \
            ctx->g, ctx->p, dt, coef, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_vals, \
            pc->d_bad, 1)
        if (pc->dim == 3) {
            if (nt == 32) FK(3, 32);
            else if (nt == 64) FK(3, 64);
            else FK(3, kFactorThreads);
        } else {
            if (nt == 32) FK(2, 32);
            else if (nt == 64) FK(2, 64);
            else FK(2, kFactorThreads);
        }
#undef FK
    }
    ACCH_LAUNCHED(ctx);
    std::vector<int> bad(pc->nsub);
    ACCH_CUDA(cudaMemcpyAsync(bad.data(), pc->d_bad, sizeof(int) * pc->nsub, cudaMemcpyDeviceToHost, ctx->stream));
    ACCH_CUDA(cudaStreamSynchronize(ctx->stream));
    pc->factorizations += 1;
    for (long long s = 0; s < pc->nsub; ++s) {
        if (bad[s] != 0x7f7f7f7f) {
            const ClassHost &C = pc->classes[pc->sub_class[s]];
            const int row = bad[s] / 2;
            const int lx = (int)C.rel[0].size(), ly = (int)C.rel[1].size();
            const int id3[3] = {row % lx, (row / lx) % ly, row / (lx * ly)};
            const int o3[3] = {pc->sub_origin[s].x, pc->sub_origin[s].y, pc->sub_origin[s].z};
            const int nn[3] = {ctx->g.nx, ctx->g.ny, ctx->g.nz};
            long long gc[3] = {0, 0, 0};
            for (int a = 0; a < pc->dim; ++a) {
                int c = o3[a] + C.rel[a][id3[a]];
                if (ctx->g.periodic) c = ((c % nn[a]) + nn[a]) % nn[a];
                gc[a] = c;
            }
            if (bad_cell) *bad_cell = (gc[2] * ctx->g.ny + gc[1]) * ctx->g.nx + gc[0];
            if (bad_comp) *bad_comp = bad[s] % 2;
            pc->have_factors = false;
            acch_set_error("zero pivot during incomplete factorization");
            return ACCH_ERR_ZERO_PIVOT;
        }
    }
    pc->have_factors = true;
    if (refactored) *refactored = 1;
    return ACCH_OK;
}

acch_status precond_apply_impl(acch_precond *pc, const double *r, double *z)
{
    if (!pc->have_factors) {
        acch_set_error("preconditioner has no factorization; call update() first");
        return ACCH_ERR_NO_FACTOR;
    }
    acch_ctx *ctx = pc->ctx;
    const int groups = 128 / pc->tps;
    const unsigned nb = (unsigned)((pc->nsub + groups - 1) / groups);
    const size_t sm = pc->apply_smem;
    // algorithmic bytes: every factor block the sweeps need (left RAS in the
    // class-group solver skips the backward rows that feed no owned cell),
    // the gather of r over the extended boxes, the write of z
    const long long blocks = pc->total_nnzb - (pc->group_mode && pc->variant == 1 ? pc->total_skip : 0);
    ProfScope prof_scope(ctx, PC_APPLY, 32.0 * blocks + 16.0 * pc->total_ext + 16.0 * ctx->g.n);
#define APPLY(V, T)                                                                                    \
    apply_kernel<V, T><<<nb, 128, sm, ctx->stream>>>(ctx->g, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, \
        pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals, (const double2 *)r, (double2 *)z, pc->d_ext_out,      \
        pc->use_smem, pc->max_nloc, pc->nsub)
#define WAPPLY_D(V, D)                                                                                        \
    do { if (pc->wide) apply_warp_kernel<V, 12, D, true><<<(unsigned)pc->nsub, 32, pc->wl.bytes(), ctx->stream>>>(ctx->g, \
        pc->d_classes, pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals,            \
        (const double2 *)r, (double2 *)z, pc->d_ext_out, pc->wl, pc->nsub);                                     \
    else apply_warp_kernel<V, 12, D><<<(unsigned)pc->nsub, 32, pc->wl.bytes(), ctx->stream>>>(ctx->g, pc->d_classes,    \
        pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals, (const double2 *)r,       \
        (double2 *)z, pc->d_ext_out, pc->wl, pc->nsub); } while (0)
#define GAPPLY_W(V, NW)                                                                                       \
    do { if (pc->wide) apply_group_kernel<V, NW, 12, double4, true><<<(unsigned)pc->groups.size(),                \
        NW * 32, pc->group_smem, ctx->stream>>>(ctx->g, pc->d_classes, pc->d_groups, pc->d_grp_sub, pc->d_sub_origin, \
        pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals, (const double2 *)r, (double2 *)z, pc->d_ext_out, pc->meta_max,  \
        pc->y_stride, 0, pc->pf_depth);                                                                           \
    else apply_group_kernel<V, NW><<<(unsigned)pc->groups.size(), NW * 32, pc->group_smem, ctx->stream>>>(ctx->g,         \
        pc->d_classes, pc->d_groups, pc->d_grp_sub, pc->d_sub_origin, pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals, \
        (const double2 *)r, (double2 *)z, pc->d_ext_out, pc->meta_max, pc->y_stride, 0, pc->pf_depth); } while (0)
#define GAPPLY(V)                                                            \
    do {                                                                     \
        if (pc->group_nw == 8) GAPPLY_W(V, 8);                               \
        else GAPPLY_W(V, 4);                                                 \
    } while (0)
#define WAPPLY(V)                                            \
    do {                                                     \
        if (pc->pf_depth <= 4) WAPPLY_D(V, 4);               \
        else if (pc->pf_depth <= 8) WAPPLY_D(V, 8);          \
        else WAPPLY_D(V, 16);                                \
    } while (0)
    // class-group solver (default), else one warp per subdomain (class image
    // too large for a group), else one CTA-wide solver per subdomain
#define NAPPLY_S(V, S)                                                                                        \
    apply_cols_kernel<V, S><<<(unsigned)pc->nsub, 32, pc->cl.bytes(), ctx->stream>>>(                             \
        ctx->g, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals,   \
        (const double2 *)r, (double2 *)z, pc->d_ext_out, pc->cl, pc->nsub)
#define NAPPLY(V)                                \
    do {                                         \
        if (pc->cl.steps_smem) NAPPLY_S(V, true); \
        else NAPPLY_S(V, false);                 \
    } while (0)
    if (pc->col_mode) {
        if (pc->variant == 1) NAPPLY(1);
        else if (pc->variant == 0) NAPPLY(0);
        else NAPPLY(2);
    } else if (pc->group_mode) {
        if (pc->variant == 1) GAPPLY(1);
        else if (pc->variant == 0) GAPPLY(0);
        else GAPPLY(2);
    } else if (pc->warp_mode) {
        if (pc->variant == 1) WAPPLY(1);
        else if (pc->variant == 0) WAPPLY(0);
        else WAPPLY(2);
    } else if (pc->tps == 32) {
        if (pc->variant == 1) APPLY(1, 32);
        else if (pc->variant == 0) APPLY(0, 32);
        else APPLY(2, 32);
    } else {
        if (pc->variant == 1) APPLY(1, 128);
        else if (pc->variant == 0) APPLY(0, 128);
        else APPLY(2, 128);
    }
#undef NAPPLY
#undef NAPPLY_S
#undef APPLY
#undef WAPPLY
#undef WAPPLY_D
#undef GAPPLY
#undef GAPPLY_W
    ACCH_LAUNCHED(ctx);
    if (pc->variant != 1) {
        const long long n = ctx->g.n;
        gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(n, pc->d_cell_ptr, pc->d_cell_src,
                                                                          pc->d_ext_out, (double2 *)z, ctx->g.skip);
        ACCH_LAUNCHED(ctx);
    }
    return ACCH_OK;
}

extern "C" acch_status acch_precond_apply(acch_precond *pc, const double *r, double *z)
{
    if (!pc || !r || !z) {
        acch_set_error("acch_precond_apply: invalid argument");
        return ACCH_ERR_INVALID_ARG;
    }
    const acch_status st = comm_halo(pc->ctx, r, 2, 1);
    if (st != ACCH_OK) return st;
    return precond_apply_impl(pc, r, z);
}

extern "C" acch_status acch_precond_info(acch_precond *pc, int64_t *factorizations, int64_t *n_classes,
                                         int64_t *factor_bytes)
{
    if (!pc) {
        acch_set_error("acch_precond_info: null handle");
        return ACCH_ERR_INVALID_ARG;
    }
    if (factorizations) *factorizations = pc->factorizations;
    if (n_classes) *n_classes = (int64_t)pc->classes.size();
    if (factor_bytes) *factor_bytes = pc->total_blocks * (int64_t)sizeof(double4);
    return ACCH_OK;
}
