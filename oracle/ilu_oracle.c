/* CPU oracle kernels for the pattern-restricted incomplete LU.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/acch_oracle.py).  Restates the
 * numerics of /root/reference/pkg/src/acch/_ilu.py:90-137: row-wise (IKJ)
 * elimination restricted to a fixed CSR pattern with a unit-diagonal L stored
 * left of the diagonal and U on/right of it, zero pivot reported when
 * |pivot| < 1e-300 (_ilu.py:118-119), then forward/backward substitution.
 * Built by oracle/Makefile (or acch_oracle.build_c) with plain gcc.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

int64_t oracle_ilu_factor(int64_t n, const int64_t *rowptr, const int64_t *col,
                          double *val, const int64_t *dpos)
{
    int64_t *where = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t bad = -1;
    for (int64_t c = 0; c < n; ++c) where[c] = -1;
    for (int64_t i = 0; i < n && bad < 0; ++i) {
        const int64_t b = rowptr[i], e = rowptr[i + 1];
        for (int64_t t = b; t < e; ++t) where[col[t]] = t;
        for (int64_t t = b; t < e && col[t] < i; ++t) {
            const int64_t k = col[t];
            const double l = val[t] / val[dpos[k]];
            val[t] = l;
            for (int64_t u = dpos[k] + 1; u < rowptr[k + 1]; ++u) {
                const int64_t hit = where[col[u]];
                if (hit >= 0) val[hit] -= l * val[u];
            }
        }
        const int64_t d = where[i];
        for (int64_t t = b; t < e; ++t) where[col[t]] = -1;
        if (d < 0 || fabs(val[d]) < 1e-300) bad = i;
    }
    free(where);
    return bad;
}

void oracle_ilu_solve(int64_t n, const int64_t *rowptr, const int64_t *col,
                      const double *val, const int64_t *dpos,
                      const double *rhs, double *x)
{
    for (int64_t i = 0; i < n; ++i) {
        double s = rhs[i];
        for (int64_t t = rowptr[i]; t < dpos[i]; ++t) s -= val[t] * x[col[t]];
        x[i] = s;
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t t = dpos[i] + 1; t < rowptr[i + 1]; ++t) s -= val[t] * x[col[t]];
        x[i] = s / val[dpos[i]];
    }
}
