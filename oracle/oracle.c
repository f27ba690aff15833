/*
 * oracle.c -- CPU restatement of the reference's compiled kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline timed by bench.py.  Nothing in the product
 * package (paper_2009_08875_b200/) may link or call it.
 *
 * Every kernel restates one numba kernel of the reference
 * (/root/reference/pkg/src/heatwave/_kernels.py) with the same arithmetic
 * order: CSR rows accumulate strictly left-to-right in column order, Gauss-
 * Seidel is lexicographic forward on the way down and backward on the way
 * up.  Row loops are OpenMP-parallel; since every output row is computed by
 * the same instruction sequence, results do not depend on the thread count
 * (the reference's own worker-count determinism, solver.py:1-11).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* _kernels.py:25-34 csr_rows_matvec: out[r] = A @ X[r], r in [r0, r1) */
/* OpenMP only pays off above this many scalar updates per call */
#define OR_PAR_MIN 65536

void or_csr_rows_matvec(const i64 *ip, const i64 *ix, const double *v, i64 n,
                        const double *X, double *out, i64 ldx, i64 r0, i64 r1)
{
#pragma omp parallel for schedule(static) if ((r1 - r0) * ldx > OR_PAR_MIN)
    for (i64 r = r0; r < r1; ++r) {
        const double *x = X + r * ldx;
        double *o = out + r * ldx;
        for (i64 i = 0; i < n; ++i) {
            double acc = 0.0;
            for (i64 k = ip[i]; k < ip[i + 1]; ++k) acc += v[k] * x[ix[k]];
            o[i] = acc;
        }
    }
}

/* _kernels.py:37-52 temporal_apply: out[c] = sum_k B[c,k] X[k] */
void or_temporal_apply(const i64 *ip, const i64 *ix, const double *v,
                       const double *X, double *out, i64 nx, i64 c0, i64 c1)
{
#pragma omp parallel for schedule(static) if ((c1 - c0) * nx > OR_PAR_MIN)
    for (i64 c = c0; c < c1; ++c) {
        double *o = out + c * nx;
        for (i64 i = 0; i < nx; ++i) o[i] = 0.0;
        for (i64 k = ip[c]; k < ip[c + 1]; ++k) {
            const double a = v[k];
            const double *x = X + ix[k] * nx;
            for (i64 i = 0; i < nx; ++i) o[i] += a * x[i];
        }
    }
}

/* _kernels.py:55-61 col_dots: per-row partial, left to right */
void or_col_dots(const double *X, const double *Y, double *out, i64 nx,
                 i64 r0, i64 r1)
{
#pragma omp parallel for schedule(static) if ((r1 - r0) * nx > OR_PAR_MIN)
    for (i64 c = r0; c < r1; ++c) {
        double acc = 0.0;
        const double *x = X + c * nx, *y = Y + c * nx;
        for (i64 i = 0; i < nx; ++i) acc += x[i] * y[i];
        out[c] = acc;
    }
}

/* solver.py:111-119 tree_reduce: fixed pairwise order over the partials */
double or_tree_reduce(const double *vals, i64 n, double *scratch)
{
    if (n <= 0) return 0.0;
    memcpy(scratch, vals, (size_t)n * sizeof(double));
    while (n > 1) {
        i64 half = n / 2;
        for (i64 i = 0; i < half; ++i) scratch[i] = scratch[2 * i] + scratch[2 * i + 1];
        if (n % 2) scratch[half] = scratch[n - 1];
        n = half + (n % 2);
    }
    return scratch[0];
}

/* _kernels.py:64-68 axpy_rows (Y += aX) and :71-76 xpay_rows (Y = X + aY) */
void or_axpy(double a, const double *X, double *Y, i64 n)
{
#pragma omp parallel for schedule(static) if (n > OR_PAR_MIN)
    for (i64 i = 0; i < n; ++i) Y[i] += a * X[i];
}

void or_xpay(double a, const double *X, double *Y, i64 n)
{
#pragma omp parallel for schedule(static) if (n > OR_PAR_MIN)
    for (i64 i = 0; i < n; ++i) Y[i] = X[i] + a * Y[i];
}

/* Flattened multigrid hierarchy, the same tuple make_solver builds
 * (multigrid.py:77-131): per-level CSR of alpha*A + mu*M, P_k, R_k = P_k^T
 * (level 0 padded with 1x1 dummies) and the dense coarse inverse. */
typedef struct {
    i64 nlev;
    const i64 *nk, *xoff;
    const i64 *ip_off, *nnz_off, *A_ip, *A_ix;
    const double *A_v, *diag;
    const i64 *pip_off, *pnnz_off, *P_ip, *P_ix;
    const double *P_v;
    const i64 *rip_off, *rnnz_off, *R_ip, *R_ix;
    const double *R_v;
    const double *coarse_inv;
} or_mg;

/* _kernels.py:110-199 _mg_core: n_vcycles V-cycles from a zero start */
static void mg_core(const or_mg *h, const double *b, double *x, int nv, int ns,
                    double *xw, double *bw, double *rw)
{
    const i64 top = h->nlev - 1, n0 = h->nk[0];
    if (h->nlev == 1) {
        for (i64 i = 0; i < n0; ++i) {
            double acc = 0.0;
            for (i64 j = 0; j < n0; ++j) acc += h->coarse_inv[i * n0 + j] * b[j];
            x[i] = acc;
        }
        return;
    }
    for (i64 i = 0; i < h->nk[top]; ++i) {
        bw[h->xoff[top] + i] = b[i];
        xw[h->xoff[top] + i] = 0.0;
    }
    for (int cyc = 0; cyc < nv; ++cyc) {
        for (i64 k = top; k > 0; --k) {
            const i64 o = h->xoff[k], n = h->nk[k];
            const i64 *ip = h->A_ip + h->ip_off[k];
            const i64 *ix = h->A_ix + h->nnz_off[k];
            const double *av = h->A_v + h->nnz_off[k];
            double *xl = xw + o, *bl = bw + o, *rl = rw + o;
            for (int s = 0; s < ns; ++s)            /* forward GS */
                for (i64 i = 0; i < n; ++i) {
                    double acc = bl[i];
                    for (i64 t = ip[i]; t < ip[i + 1]; ++t)
                        if (ix[t] != i) acc -= av[t] * xl[ix[t]];
                    xl[i] = acc / h->diag[o + i];
                }
            for (i64 i = 0; i < n; ++i) {             /* residual */
                double acc = bl[i];
                for (i64 t = ip[i]; t < ip[i + 1]; ++t) acc -= av[t] * xl[ix[t]];
                rl[i] = acc;
            }
            const i64 oc = h->xoff[k - 1];             /* restrict */
            const i64 *rip = h->R_ip + h->rip_off[k];
            const i64 *rix = h->R_ix + h->rnnz_off[k];
            const double *rv = h->R_v + h->rnnz_off[k];
            for (i64 i = 0; i < h->nk[k - 1]; ++i) {
                double acc = 0.0;
                for (i64 t = rip[i]; t < rip[i + 1]; ++t) acc += rv[t] * rl[rix[t]];
                bw[oc + i] = acc;
                xw[oc + i] = 0.0;
            }
        }
        for (i64 i = 0; i < n0; ++i) {                  /* coarse solve */
            double acc = 0.0;
            for (i64 j = 0; j < n0; ++j) acc += h->coarse_inv[i * n0 + j] * bw[j];
            xw[i] = acc;
        }
        for (i64 k = 1; k <= top; ++k) {
            const i64 o = h->xoff[k], oc = h->xoff[k - 1], n = h->nk[k];
            const i64 *ip = h->A_ip + h->ip_off[k];
            const i64 *ix = h->A_ix + h->nnz_off[k];
            const double *av = h->A_v + h->nnz_off[k];
            const i64 *pip = h->P_ip + h->pip_off[k];
            const i64 *pix = h->P_ix + h->pnnz_off[k];
            const double *pv = h->P_v + h->pnnz_off[k];
            double *xl = xw + o, *bl = bw + o;
            for (i64 i = 0; i < n; ++i) {               /* prolongate */
                double acc = 0.0;
                for (i64 t = pip[i]; t < pip[i + 1]; ++t) acc += pv[t] * xw[oc + pix[t]];
                xl[i] += acc;
            }
            for (int s = 0; s < ns; ++s)                /* backward GS */
                for (i64 i = n - 1; i >= 0; --i) {
                    double acc = bl[i];
                    for (i64 t = ip[i]; t < ip[i + 1]; ++t)
                        if (ix[t] != i) acc -= av[t] * xl[ix[t]];
                    xl[i] = acc / h->diag[o + i];
                }
        }
    }
    for (i64 i = 0; i < h->nk[top]; ++i) x[i] = xw[h->xoff[top] + i];
}

/* _kernels.py:217-249 mg_solve_rows / mg_solve_indexed.  rows == NULL means
 * rows [0, nrows); otherwise the listed rows.  Workspaces are per thread. */
int or_mg_rows(const or_mg *h, const double *B, double *X, i64 ld,
               const i64 *rows, i64 nrows, int nv, int ns)
{
    const i64 ntot = h->xoff[h->nlev];
    int err = 0;
#pragma omp parallel if (nrows > 1 && nrows * ntot > 4096)
    {
        double *ws = (double *)malloc(3 * (size_t)ntot * sizeof(double));
        if (!ws) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (i64 k = 0; k < nrows; ++k) {
                const i64 r = rows ? rows[k] : k;
                mg_core(h, B + r * ld, X + r * ld, nv, ns, ws, ws + ntot, ws + 2 * ntot);
            }
            free(ws);
        }
    }
    return err;
}

int or_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
