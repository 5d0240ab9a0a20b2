/* TEST INFRASTRUCTURE ONLY — C restatement of the reference's single native
 * kernel, numba `_kernels.sequential_corrected_sweep`
 * (/root/reference/pkg/src/mgrit_advect/_kernels.py:104-131) with its inlined
 * GMRES (`_gmres_imsd`, _kernels.py:34-101) and stencil apply (`_apply_imsd`,
 * _kernels.py:18-31).
 *
 * Same sequential loop orders as the numba code (which is compiled without
 * fastmath); build with -ffp-contract=off so no FMA contraction changes the
 * rounding.  Used by oracle/mgrit_oracle.py:solve_sequential under the same
 * condition as mgrit.py:304-305 (1D, corrected, >= 64 steps).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* out_i = v_i - sig_i * sum_{k=-rad..rad} st[rad+k] * v_{(i+k) mod n} */
static void imsd_apply(const double *sig, const double *st, int nst,
                       const double *v, double *out, long n) {
    int rad = (nst - 1) / 2;
    for (long i = 0; i < n; i++) {
        double acc = 0.0;
        for (int k = -rad; k <= rad; k++) {
            long j = i + k;
            if (j < 0) j += n;
            else if (j >= n) j -= n;
            acc += st[rad + k] * v[j];
        }
        out[i] = v[i] - sig[i] * acc;
    }
}

/* GMRES on (I - diag(sig) D) x = rhs; tol < 0 runs all iterations.
 * Returns the number of Arnoldi steps performed. */
static int gmres_imsd(const double *sig, const double *st, int nst,
                      const double *rhs, long n, int max_iters, double tol,
                      double *x, double *work) {
    double beta = 0.0;
    for (long i = 0; i < n; i++) beta += rhs[i] * rhs[i];
    beta = sqrt(beta);
    if (beta == 0.0) {
        for (long i = 0; i < n; i++) x[i] = 0.0;
        return 0;
    }
    int K = max_iters;
    double *basis = work;                    /* (K+1) x n */
    double *w = basis + (size_t)(K + 1) * n; /* n */
    double *hess = (double *)calloc((size_t)(K + 1) * K, sizeof(double));
    double *cs = (double *)calloc(K, sizeof(double));
    double *sn = (double *)calloc(K, sizeof(double));
    double *g = (double *)calloc(K + 1, sizeof(double));
    double *y = (double *)calloc(K + 1, sizeof(double));
#define H(a, b) hess[(size_t)(a) * K + (b)]
    g[0] = beta;
    for (long i = 0; i < n; i++) basis[i] = rhs[i] / beta;
    int done = 0;
    for (int k = 0; k < K; k++) {
        imsd_apply(sig, st, nst, basis + (size_t)k * n, w, n);
        for (int j = 0; j <= k; j++) {
            const double *bj = basis + (size_t)j * n;
            double h = 0.0;
            for (long i = 0; i < n; i++) h += bj[i] * w[i];
            H(j, k) = h;
            for (long i = 0; i < n; i++) w[i] -= h * bj[i];
        }
        double nrm = 0.0;
        for (long i = 0; i < n; i++) nrm += w[i] * w[i];
        nrm = sqrt(nrm);
        H(k + 1, k) = nrm;
        int brk = nrm <= 1e-14 * beta;
        if (!brk) {
            double *bk1 = basis + (size_t)(k + 1) * n;
            for (long i = 0; i < n; i++) bk1[i] = w[i] / nrm;
        }
        for (int j = 0; j < k; j++) {
            double t = cs[j] * H(j, k) + sn[j] * H(j + 1, k);
            H(j + 1, k) = -sn[j] * H(j, k) + cs[j] * H(j + 1, k);
            H(j, k) = t;
        }
        double den = hypot(H(k, k), H(k + 1, k));
        cs[k] = H(k, k) / den;
        sn[k] = H(k + 1, k) / den;
        H(k, k) = den;
        H(k + 1, k) = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
        done = k + 1;
        if (brk) break;
        if (tol >= 0.0 && fabs(g[k + 1]) <= tol * beta) break;
    }
    for (int j = done - 1; j >= 0; j--) {
        double acc = g[j];
        for (int jj = j + 1; jj < done; jj++) acc -= H(j, jj) * y[jj];
        y[j] = acc / H(j, j);
    }
    for (long i = 0; i < n; i++) {
        double acc = 0.0;
        for (int j = 0; j < done; j++) acc += basis[(size_t)j * n + i] * y[j];
        x[i] = acc;
    }
#undef H
    free(hess); free(cs); free(sn); free(g); free(y);
    return done;
}

/* In-place U[s+1] = GMRES(I - diag(sig_k) D, sum_j w U[s, idx]) + G[s+1].
 * idx int32 [S][n][q], w f64 [S][n][q], sig f64 [S][n], U/G f64 [n_steps+1][n].
 * counts (nullable) receives the per-step Arnoldi step count (-1 on NaN row). */
void oracle_sequential_corrected_sweep(const int *idx, const double *w,
                                       const double *sig, const double *st, int nst,
                                       double *U, const double *G, long n_steps, long n,
                                       int q, double tol, int max_iters, int shared,
                                       int *counts) {
    double *rhs = (double *)malloc(sizeof(double) * n);
    double *work = (double *)malloc(sizeof(double) * (size_t)(max_iters + 2) * n);
    for (long step = 0; step < n_steps; step++) {
        long k = shared ? 0 : step;
        int ok = 1;
        const double *Us = U + (size_t)step * n;
        for (long i = 0; i < n; i++) {
            double acc = 0.0;
            const int *ix = idx + ((size_t)k * n + i) * q;
            const double *wx = w + ((size_t)k * n + i) * q;
            for (int j = 0; j < q; j++) acc += wx[j] * Us[ix[j]];
            rhs[i] = acc;
            if (!isfinite(acc)) ok = 0;
        }
        double *out = U + (size_t)(step + 1) * n;
        if (!ok) {
            for (long i = 0; i < n; i++) out[i] = NAN;
            if (counts) counts[step] = -1;
            continue;
        }
        int c = gmres_imsd(sig + (size_t)k * n, st, nst, rhs, n, max_iters, tol, out, work);
        if (counts) counts[step] = c;
        const double *Gs = G + (size_t)(step + 1) * n;
        for (long i = 0; i < n; i++) out[i] += Gs[i];
    }
    free(rhs);
    free(work);
}
