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
    int nloc, nnzb, nlev, nlevb;
    int len[3];
    const int *rel[3];
    const int *rowptr, *col, *diag;
    const int *jmap;        // nloc * noff
    const int *upd_ptr;     // nnzb + 1
    const int2 *upd;        // (src, dst)
    const int *lev_ptr, *lev_rows, *levb_ptr, *levb_rows;
    const unsigned char *owned;
};

struct ClassHost {
    std::array<std::vector<int>, 3> rel;
    int own_len[3];
    std::vector<int> rowptr, col, diag, jmap, upd_ptr, lev_ptr, lev_rows, levb_ptr, levb_rows;
    std::vector<int2> upd;
    std::vector<unsigned char> owned;
    int nloc = 0, nnzb = 0;
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
    gz = g.dim == 3 ? wrap_coord(o.z + C.rel[2][iz], g.nz, g.periodic) : 0;
}

struct Blk {
    double a, b, c, d;   // [[a, b], [c, d]]
};

__device__ __forceinline__ Blk mul(const Blk &x, const Blk &y)
{
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}

template <int DIM>
__global__ void __launch_bounds__(kFactorThreads)
factor_kernel(GridDev g, ParamsDev P, double dt, const double *__restrict__ coef, const ClassDev *__restrict__ classes,
              const int *__restrict__ sub_class, const int4 *__restrict__ sub_origin,
              const long long *__restrict__ sub_off, double4 *__restrict__ vals, int *__restrict__ bad_row)
{
    constexpr int NOFF = DIM == 3 ? 25 : 13;
    const int s = blockIdx.x;
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    double4 *A = vals + sub_off[s];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < C.nnzb; t += nt) A[t] = make_double4(0.0, 0.0, 0.0, 0.0);
    __syncthreads();
    for (int l = tid; l < C.nloc; l += nt) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double blk[NOFF][4];
        jac_row_blocks<DIM>(g, P, dt, coef, gx, gy, gz, blk, NOFF);
        for (int q = 0; q < NOFF; ++q) {
            const int p = C.jmap[l * NOFF + q];
            if (p < 0) continue;
            double4 v = A[p];
            v.x += blk[q][0];
            v.y += blk[q][1];
            v.z += blk[q][2];
            v.w += blk[q][3];
            A[p] = v;
        }
    }
    __syncthreads();
    for (int lev = 0; lev < C.nlev; ++lev) {
        for (int q = C.lev_ptr[lev] + tid; q < C.lev_ptr[lev + 1]; q += nt) {
            const int i = C.lev_rows[q];
            const int d = C.diag[i];
            for (int t = C.rowptr[i]; t < d; ++t) {
                const int k = C.col[t];
                const double4 ak = A[t], dk = A[C.diag[k]];
                const Blk L = mul({ak.x, ak.y, ak.z, ak.w}, {dk.x, dk.y, dk.z, dk.w});
                A[t] = make_double4(L.a, L.b, L.c, L.d);
                for (int u = C.upd_ptr[t]; u < C.upd_ptr[t + 1]; ++u) {
                    const int2 sd = C.upd[u];
                    const double4 us = A[sd.x];
                    const Blk m = mul(L, {us.x, us.y, us.z, us.w});
                    double4 v = A[sd.y];
                    v.x -= m.a;
                    v.y -= m.b;
                    v.z -= m.c;
                    v.w -= m.d;
                    A[sd.y] = v;
                }
            }
            // diagonal block: scalar pivots as the reference's factor_inplace sees them
            const double4 D = A[d];
            const double p0 = D.x;
            const double p1 = D.w - (D.z / D.x) * D.y;
            int bad = -1;
            if (fabs(p0) < 1e-300) bad = 2 * i;
            else if (fabs(p1) < 1e-300) bad = 2 * i + 1;
            if (bad >= 0) atomicMin(bad_row + s, bad);
            const double det = D.x * D.w - D.y * D.z;
            A[d] = make_double4(D.w / det, -D.y / det, -D.z / det, D.x / det);
        }
        __syncthreads();
    }
}

template <int VARIANT>   // 0 asm, 1 ras-left, 2 ras-right
__global__ void __launch_bounds__(kApplyThreads)
apply_kernel(GridDev g, const ClassDev *__restrict__ classes, const int *__restrict__ sub_class,
             const int4 *__restrict__ sub_origin, const long long *__restrict__ sub_off,
             const long long *__restrict__ sub_ext_off, const double4 *__restrict__ vals,
             const double2 *__restrict__ r, double2 *__restrict__ z, double2 *__restrict__ ext_out, int use_smem)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int s = blockIdx.x;
    const ClassDev C = classes[sub_class[s]];
    const int4 o = sub_origin[s];
    const double4 *A = vals + sub_off[s];
    double2 *y = use_smem ? reinterpret_cast<double2 *>(smem_raw) : ext_out + sub_ext_off[s];
    const int tid = threadIdx.x, nt = blockDim.x;
    const long long nx = g.nx, ny = g.ny;
    for (int l = tid; l < C.nloc; l += nt) {
        int gx, gy, gz;
        local_to_global(g, C, o, l, gx, gy, gz);
        double2 v = r[(gz * ny + gy) * nx + gx];
        if (VARIANT == 2 && !C.owned[l]) v = make_double2(0.0, 0.0);
        y[l] = v;
    }
    __syncthreads();
    for (int lev = 0; lev < C.nlev; ++lev) {
        for (int q = C.lev_ptr[lev] + tid; q < C.lev_ptr[lev + 1]; q += nt) {
            const int i = C.lev_rows[q];
            double2 acc = y[i];
            for (int t = C.rowptr[i]; t < C.diag[i]; ++t) {
                const double4 a = A[t];
                const double2 yk = y[C.col[t]];
                acc.x -= a.x * yk.x + a.y * yk.y;
                acc.y -= a.z * yk.x + a.w * yk.y;
            }
            y[i] = acc;
        }
        __syncthreads();
    }
    for (int lev = 0; lev < C.nlevb; ++lev) {
        for (int q = C.levb_ptr[lev] + tid; q < C.levb_ptr[lev + 1]; q += nt) {
            const int i = C.levb_rows[q];
            double2 acc = y[i];
            const int d = C.diag[i];
            for (int t = d + 1; t < C.rowptr[i + 1]; ++t) {
                const double4 a = A[t];
                const double2 xk = y[C.col[t]];
                acc.x -= a.x * xk.x + a.y * xk.y;
                acc.y -= a.z * xk.x + a.w * xk.y;
            }
            const double4 di = A[d];
            y[i] = make_double2(di.x * acc.x + di.y * acc.y, di.z * acc.x + di.w * acc.y);
        }
        __syncthreads();
    }
    if (VARIANT == 1) {
        for (int l = tid; l < C.nloc; l += nt) {
            if (!C.owned[l]) continue;
            int gx, gy, gz;
            local_to_global(g, C, o, l, gx, gy, gz);
            z[(gz * ny + gy) * nx + gx] = y[l];
        }
    } else if (use_smem) {
        for (int l = tid; l < C.nloc; l += nt) ext_out[sub_ext_off[s] + l] = y[l];
    }
}

// z[c] = sum over subdomains containing c, in subdomain order, of their local solution
__global__ void gather_kernel(long long n, const long long *__restrict__ cell_ptr, const long long *__restrict__ cell_src,
                              const double2 *__restrict__ ext_out, double2 *__restrict__ z)
{
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
                if (g.periodic) t = ((t % nn[a]) + nn[a]) % nn[a];
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
    C.owned.assign(nloc, 0);
    for (int l = 0; l < nloc; ++l) {
        const int ix[3] = {l % lx, (l / lx) % ly, l / (lx * ly)};
        bool own = true;
        for (int a = 0; a < dim; ++a) own = own && rel[a][ix[a]] >= 0 && rel[a][ix[a]] < own_len[a];
        C.owned[l] = own ? 1 : 0;
    }
    return true;
}

template <typename T>
size_t padded(size_t n) { return ((n * sizeof(T) + 255) / 256) * 256; }

acch_status upload_class(ClassHost &C)
{
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
    long long total_blocks = 0, total_ext = 0;
    int *d_bad = nullptr;
    double2 *d_ext_out = nullptr;
    long long *d_cell_ptr = nullptr, *d_cell_src = nullptr;
    bool have_factors = false;
    long long factorizations = 0;
    size_t apply_smem = 0;
    int use_smem = 1;
};

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
}

extern "C" acch_status acch_precond_create(acch_ctx *ctx, int64_t n_sub, int32_t overlap, const int64_t *owned_lo,
                                           const int64_t *owned_hi, int32_t variant, int32_t fill_level,
                                           acch_precond **out)
{
    if (!ctx || !out || n_sub < 1 || overlap < 0 || !owned_lo || !owned_hi || variant < 0 || variant > 2) {
        acch_set_error("acch_precond_create: invalid argument");
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
            if (g.periodic) {
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
        pc->sub_origin.push_back(make_int4(lo3[0], lo3[1], lo3[2], 0));
    }
    // offsets
    long long vo = 0, eo = 0;
    int max_nloc = 0;
    for (long long s = 0; s < n_sub; ++s) {
        const ClassHost &C = pc->classes[pc->sub_class[s]];
        pc->sub_off.push_back(vo);
        pc->sub_ext_off.push_back(eo);
        vo += C.nnzb;
        eo += C.nloc;
        max_nloc = std::max(max_nloc, C.nloc);
    }
    pc->total_blocks = vo;
    pc->total_ext = eo;
    pc->apply_smem = sizeof(double2) * (size_t)max_nloc;
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
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc->apply_smem));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc->apply_smem));
        PC_CUDA(cudaFuncSetAttribute(apply_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc->apply_smem));
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
    ProfScope prof_scope(ctx, PC_FACTOR, 32.0 * pc->total_blocks + 56.0 * pc->total_ext);
    if (pc->dim == 3)
        factor_kernel<3><<<(unsigned)pc->nsub, kFactorThreads, 0, ctx->stream>>>(
            ctx->g, ctx->p, dt, coef, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_vals,
            pc->d_bad);
    else
        factor_kernel<2><<<(unsigned)pc->nsub, kFactorThreads, 0, ctx->stream>>>(
            ctx->g, ctx->p, dt, coef, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, pc->d_sub_off, pc->d_vals,
            pc->d_bad);
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
    const unsigned nb = (unsigned)pc->nsub;
    const size_t sm = pc->apply_smem;
    ProfScope prof_scope(ctx, PC_APPLY, 32.0 * pc->total_blocks + 16.0 * pc->total_ext + 16.0 * ctx->g.n);
#define APPLY(V) \
    apply_kernel<V><<<nb, kApplyThreads, sm, ctx->stream>>>(ctx->g, pc->d_classes, pc->d_sub_class, pc->d_sub_origin, \
        pc->d_sub_off, pc->d_sub_ext_off, pc->d_vals, (const double2 *)r, (double2 *)z, pc->d_ext_out, pc->use_smem)
    if (pc->variant == 1) APPLY(1);
    else if (pc->variant == 0) APPLY(0);
    else APPLY(2);
#undef APPLY
    ACCH_LAUNCHED(ctx);
    if (pc->variant != 1) {
        const long long n = ctx->g.n;
        gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(n, pc->d_cell_ptr, pc->d_cell_src,
                                                                          pc->d_ext_out, (double2 *)z);
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
