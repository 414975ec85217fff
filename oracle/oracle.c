/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of the power-method truncated SVD of
 * arXiv 2208.08410 ("Distributed Out-of-Memory SVD on CPU/GPU Architectures").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this file's library.  The product path
 * (paper_2208_08410_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * Citations are PAPER.md line numbers (P:nnn) of /root/reference/PAPER.md.
 *
 *   Alg. 1 SVD(A, eps, k)           P:63-100  -> oracle_tsvd
 *   Alg. 2 SVD_1D(X, eps)           P:102-129 -> inner loop of oracle_tsvd
 *   Eq. 2 (m > n Gram-vector)       P:202-211 -> oracle_gram_apply (modes below)
 *   Eq. 3 (m < n mirror)            P:212-219 -> oracle_gram_apply_wide
 *
 * Gram-vector modes (reading R7):
 *   ORACLE_F2      exact factored form of B v0 with B = X'^T X', X' = A - U S V^T:
 *                    c = S (V^T v); t = A v - U c; w = S (U^T t); y = A^T t - V w
 *                  (X' never formed; no U^T U = I assumption).  Default reference.
 *   ORACLE_LITERAL Alg. 1 line 8 + Alg. 2 line 7 as written: X' explicit (m x n),
 *                  B = X'^T X' explicit (n x n), y = B v.  Tiny inputs only.
 *   ORACLE_EQ2     the paper's four-term Eq. 2 right to left:
 *                  y = A^T(A v) - V S (U^T (A v)) - A^T (U (S (V^T v))) + V S^2 V^T v.
 *                  Exact only when U^T U = I; kept to document that reading.
 *
 * Every sum runs in index order.  OpenMP only splits independent outputs (rows of
 * t, columns of y) across threads; each output's sum keeps the same sequential
 * order, so results are bitwise independent of the thread count.
 *
 * A is fp32 (the same bits the GPU sees), promoted to fp64 on read.  U (m x ldu),
 * V (n x ldv) are fp64 row-major, S is fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_F2 0
#define ORACLE_LITERAL 1
#define ORACLE_EQ2 2

/* status codes (mirror the meaning, not the header, of the product ABI) */
#define OR_OK 0
#define OR_NOT_CONVERGED 1
#define OR_RANK_EXHAUSTED 2
#define OR_ERR_ARG -1
#define OR_ERR_NOMEM -4
#define OR_ERR_NUMERIC -7

static inline double a_at(const float *A, int64_t lda, int64_t r, int64_t j) {
    return (double)A[r * lda + j];
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- plain products ---------------------------------------------------------- */

/* out[r] = sum_j A[r,j] x[j]  (Alg. 1 line 12 "A @ V_l") */
void oracle_matvec(const float *A, int64_t m, int64_t n, int64_t lda, const double *x, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += a_at(A, lda, r, j) * x[j];
        out[r] = s;
    }
}

/* out[j] = sum_r A[r,j] x[r]  (A^T x; Alg. 4 line 5).  Sum over r in order. */
void oracle_matvec_t(const float *A, int64_t m, int64_t n, int64_t lda, const double *x, double *out) {
#pragma omp parallel
    {
        int64_t j0 = 0, j1 = n;
#ifdef _OPENMP
        int nt = omp_get_num_threads(), id = omp_get_thread_num();
        int64_t chunk = (n + nt - 1) / nt;
        j0 = (int64_t)id * chunk;
        j1 = j0 + chunk < n ? j0 + chunk : n;
#endif
        for (int64_t j = j0; j < j1; ++j) out[j] = 0.0;
        for (int64_t r = 0; r < m; ++r) {
            const double xr = x[r];
            for (int64_t j = j0; j < j1; ++j) out[j] += a_at(A, lda, r, j) * xr;
        }
    }
}

static double dot(const double *a, const double *b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static double nrm2(const double *a, int64_t n) { return sqrt(dot(a, a, n)); }

/* ---- CSR products (sparse A: "stored in a sparse Compressed Sparse Row (CSR) format") */

/* out[r] = sum_k val[k] x[col[k]], k over row r in stored order */
void oracle_csr_matvec(const int64_t *rp, const int32_t *ci, const float *va, int64_t m, const double *x,
                       double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
        double s = 0.0;
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += (double)va[k] * x[ci[k]];
        out[r] = s;
    }
}

/* out[j] = sum_r A[r,j] x[r]: rows in order (sequential, so each out[j] sums in row order) */
void oracle_csr_matvec_t(const int64_t *rp, const int32_t *ci, const float *va, int64_t m, int64_t n,
                         const double *x, double *out) {
    for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
    for (int64_t r = 0; r < m; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) out[ci[k]] += (double)va[k] * x[r];
}

/* The operator A of one problem: dense (A != NULL) or CSR. */
typedef struct {
    const float *A;
    int64_t lda;
    const int64_t *rp;
    const int32_t *ci;
    const float *va;
} op_t;

static void op_mv(const op_t *o, int64_t m, int64_t n, const double *x, double *out) {
    if (o->A) oracle_matvec(o->A, m, n, o->lda, x, out);
    else oracle_csr_matvec(o->rp, o->ci, o->va, m, x, out);
}

static void op_mvt(const op_t *o, int64_t m, int64_t n, const double *x, double *out) {
    if (o->A) oracle_matvec_t(o->A, m, n, o->lda, x, out);
    else oracle_csr_matvec_t(o->rp, o->ci, o->va, m, n, x, out);
}

/* ---- Gram-vector products ---------------------------------------------------- */

/* ORACLE_F2: y = X'^T X' v with X' = A - U diag(S) V^T, never formed.
 * Right-to-left as Eq. 2 asks, but grouped as X'^T (X' v). */
static int gram_f2(const op_t *op, int64_t m, int64_t n, const double *U, int64_t ldu,
                   const double *S, const double *V, int64_t ldv, int l, const double *v, double *y) {
    double *c = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    double *w = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    double *t = (double *)malloc((size_t)m * sizeof(double));
    if (!c || !w || !t) { free(c); free(w); free(t); return OR_ERR_NOMEM; }
    /* c_i = S_i * sum_j V[j,i] v_j          (Sigma V^T v) */
    for (int i = 0; i < l; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += V[j * ldv + i] * v[j];
        c[i] = S[i] * s;
    }
    /* t_r = sum_j A[r,j] v_j - sum_i U[r,i] c_i     (X' v) */
    op_mv(op, m, n, v, t);
    for (int64_t r = 0; r < m; ++r) {
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += U[r * ldu + i] * c[i];
        t[r] -= s;
    }
    /* w_i = S_i * sum_r U[r,i] t_r           (Sigma U^T X' v) */
    for (int i = 0; i < l; ++i) {
        double s = 0.0;
        for (int64_t r = 0; r < m; ++r) s += U[r * ldu + i] * t[r];
        w[i] = S[i] * s;
    }
    /* y_j = sum_r A[r,j] t_r - sum_i V[j,i] w_i   (X'^T X' v) */
    op_mvt(op, m, n, t, y);
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += V[j * ldv + i] * w[i];
        y[j] -= s;
    }
    free(c); free(w); free(t);
    return OR_OK;
}

/* ORACLE_LITERAL: X' = A - U[:l] diag(S[:l]) V[:l]^T explicitly (Alg. 1 line 8),
 * B = X'^T X' explicitly (Alg. 2 line 7), y = B v (Alg. 2 line 11). */
static int gram_literal(const float *A, int64_t m, int64_t n, int64_t lda, const double *U, int64_t ldu,
                        const double *S, const double *V, int64_t ldv, int l, const double *v, double *y) {
    double *X = (double *)malloc((size_t)m * (size_t)n * sizeof(double));
    double *B = (double *)malloc((size_t)n * (size_t)n * sizeof(double));
    if (!X || !B) { free(X); free(B); return OR_ERR_NOMEM; }
    for (int64_t r = 0; r < m; ++r)
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < l; ++i) s += U[r * ldu + i] * S[i] * V[j * ldv + i];
            X[r * n + j] = a_at(A, lda, r, j) - s;
        }
    for (int64_t p = 0; p < n; ++p)
        for (int64_t q = 0; q < n; ++q) {
            double s = 0.0;
            for (int64_t r = 0; r < m; ++r) s += X[r * n + p] * X[r * n + q];
            B[p * n + q] = s;
        }
    for (int64_t p = 0; p < n; ++p) {
        double s = 0.0;
        for (int64_t q = 0; q < n; ++q) s += B[p * n + q] * v[q];
        y[p] = s;
    }
    free(X); free(B);
    return OR_OK;
}

/* ORACLE_EQ2: Eq. 2, each product right to left, X = A:
 *   y = A^T A v  -  V S U^T A v  -  A^T U S V^T v  +  V S^2 V^T v                     */
static int gram_eq2(const float *A, int64_t m, int64_t n, int64_t lda, const double *U, int64_t ldu,
                    const double *S, const double *V, int64_t ldv, int l, const double *v, double *y) {
    double *Av = (double *)malloc((size_t)m * sizeof(double));
    double *t1 = (double *)malloc((size_t)n * sizeof(double));
    double *Uc = (double *)malloc((size_t)m * sizeof(double));
    double *t3 = (double *)malloc((size_t)n * sizeof(double));
    double *Vtv = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    double *UtAv = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    if (!Av || !t1 || !Uc || !t3 || !Vtv || !UtAv) {
        free(Av); free(t1); free(Uc); free(t3); free(Vtv); free(UtAv);
        return OR_ERR_NOMEM;
    }
    oracle_matvec(A, m, n, lda, v, Av);            /* X v0            */
    oracle_matvec_t(A, m, n, lda, Av, t1);         /* X^T X v0        */
    for (int i = 0; i < l; ++i) {                  /* U^T X v0, V^T v0 */
        double s = 0.0, q = 0.0;
        for (int64_t r = 0; r < m; ++r) s += U[r * ldu + i] * Av[r];
        for (int64_t j = 0; j < n; ++j) q += V[j * ldv + i] * v[j];
        UtAv[i] = s;
        Vtv[i] = q;
    }
    for (int64_t r = 0; r < m; ++r) {              /* U S V^T v0      */
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += U[r * ldu + i] * (S[i] * Vtv[i]);
        Uc[r] = s;
    }
    oracle_matvec_t(A, m, n, lda, Uc, t3);         /* X^T U S V^T v0  */
    for (int64_t j = 0; j < n; ++j) {
        double t2 = 0.0, t4 = 0.0;
        for (int i = 0; i < l; ++i) {
            t2 += V[j * ldv + i] * (S[i] * UtAv[i]);          /* V S^T U^T X v0 */
            t4 += V[j * ldv + i] * (S[i] * (S[i] * Vtv[i]));  /* V S^2 V^T v0   */
        }
        y[j] = t1[j] - t2 - t3[j] + t4;
    }
    free(Av); free(t1); free(Uc); free(t3); free(Vtv); free(UtAv);
    return OR_OK;
}

/* One Gram-vector product y = B v for the current deflation state (l found components). */
int oracle_gram_apply(int mode, const float *A, int64_t m, int64_t n, int64_t lda, const double *U, int64_t ldu,
                      const double *S, const double *V, int64_t ldv, int l, const double *v, double *y) {
    if (m <= 0 || n <= 0 || lda < n || l < 0) return OR_ERR_ARG;
    const op_t op = {A, lda, NULL, NULL, NULL};
    switch (mode) {
    case ORACLE_F2: return gram_f2(&op, m, n, U, ldu, S, V, ldv, l, v, y);
    case ORACLE_LITERAL: return gram_literal(A, m, n, lda, U, ldu, S, V, ldv, l, v, y);
    case ORACLE_EQ2: return gram_eq2(A, m, n, lda, U, ldu, S, V, ldv, l, v, y);
    default: return OR_ERR_ARG;
    }
}

/* Same product for a CSR A (F2 only: the literal / Eq. 2 modes are dense cross-checks). */
int oracle_gram_apply_csr(const int64_t *rp, const int32_t *ci, const float *va, int64_t m, int64_t n,
                          const double *U, int64_t ldu, const double *S, const double *V, int64_t ldv, int l,
                          const double *v, double *y) {
    if (m <= 0 || n <= 0 || l < 0) return OR_ERR_ARG;
    const op_t op = {NULL, 0, rp, ci, va};
    return gram_f2(&op, m, n, U, ldu, S, V, ldv, l, v, y);
}

/* Mirror for m < n (Eq. 3), exact factored form: y = X' X'^T u,
 *   c = S (U^T u); t = A^T u - V c; w = S (V^T t); y = A t - U w.                       */
int oracle_gram_apply_wide(const float *A, int64_t m, int64_t n, int64_t lda, const double *U, int64_t ldu,
                           const double *S, const double *V, int64_t ldv, int l, const double *u, double *y) {
    double *c = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    double *w = (double *)calloc((size_t)(l > 0 ? l : 1), sizeof(double));
    double *t = (double *)malloc((size_t)n * sizeof(double));
    if (!c || !w || !t) { free(c); free(w); free(t); return OR_ERR_NOMEM; }
    for (int i = 0; i < l; ++i) {
        double s = 0.0;
        for (int64_t r = 0; r < m; ++r) s += U[r * ldu + i] * u[r];
        c[i] = S[i] * s;
    }
    oracle_matvec_t(A, m, n, lda, u, t);
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += V[j * ldv + i] * c[i];
        t[j] -= s;
    }
    for (int i = 0; i < l; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += V[j * ldv + i] * t[j];
        w[i] = S[i] * s;
    }
    oracle_matvec(A, m, n, lda, t, y);
    for (int64_t r = 0; r < m; ++r) {
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += U[r * ldu + i] * w[i];
        y[r] -= s;
    }
    free(c); free(w); free(t);
    return OR_OK;
}

/* ---- Alg. 1 + Alg. 2 ---------------------------------------------------------- */

/*
 * oracle_tsvd — Alg. 1 with SVD_1D = Alg. 2.
 *
 *   A       m x n fp32 row-major (lda), promoted to fp64.
 *   k       number of components (k == -1 -> min(m, n)).
 *   eps     stop when |v0 . v1| >= 1 - eps.
 *   V0      k x len fp64, row l = the N(0,1) sample x of component l; len = n if
 *           m >= n else m.  Normalised here.
 *   max_iter  cap on iterations per component (P:119 has none; reading R5); <= 0 -> 10000.
 *   fixed_T   > 0: run exactly fixed_T iterations, convergence test disabled.
 *   mode    ORACLE_F2 / ORACLE_LITERAL / ORACLE_EQ2 (m >= n only; wide inputs use F2 mirror).
 *
 * Outputs (caller-owned): U m x k row-major, S k, V n x k row-major (fp64),
 *   iters[k] iterations per component, dots[k] final |v0 . v1|.
 * Returns the number of components found in *k_found and a status:
 *   OR_OK, OR_NOT_CONVERGED (some component hit max_iter), OR_RANK_EXHAUSTED (||B v0|| == 0
 *   or sigma == 0 before k components), OR_ERR_ARG, OR_ERR_NUMERIC (non-finite), OR_ERR_NOMEM.
 */
static int tsvd_core(const op_t *op, int64_t m, int64_t n, int k, double eps, const double *V0, int max_iter,
                     int fixed_T, int mode, double *U, double *S, double *V, int *iters, double *dots, int *k_found);

int oracle_tsvd(const float *A, int64_t m, int64_t n, int64_t lda, int k, double eps, const double *V0,
                int max_iter, int fixed_T, int mode, double *U, double *S, double *V, int *iters, double *dots,
                int *k_found) {
    *k_found = 0;
    if (lda < n) return OR_ERR_ARG;
    const op_t op = {A, lda, NULL, NULL, NULL};
    return tsvd_core(&op, m, n, k, eps, V0, max_iter, fixed_T, mode, U, S, V, iters, dots, k_found);
}

/* oracle_tsvd for a CSR A (m >= n, F2): same algorithm, sparse products. */
int oracle_tsvd_csr(const int64_t *rp, const int32_t *ci, const float *va, int64_t m, int64_t n, int k, double eps,
                    const double *V0, int max_iter, int fixed_T, double *U, double *S, double *V, int *iters,
                    double *dots, int *k_found) {
    *k_found = 0;
    if (m < n) return OR_ERR_ARG;
    const op_t op = {NULL, 0, rp, ci, va};
    return tsvd_core(&op, m, n, k, eps, V0, max_iter, fixed_T, ORACLE_F2, U, S, V, iters, dots, k_found);
}

static int tsvd_core(const op_t *op, int64_t m, int64_t n, int k, double eps, const double *V0, int max_iter,
                     int fixed_T, int mode, double *U, double *S, double *V, int *iters, double *dots, int *k_found) {
    const int tall = (m >= n); /* reading R2: square -> V first (P:83 vs P:264) */
    const int64_t len = tall ? n : m;     /* SVD_1D vector length */
    const int64_t other = tall ? m : n;
    if (k == -1) k = (int)(m < n ? m : n);
    *k_found = 0;
    if (m <= 0 || n <= 0 || k <= 0 || k > (m < n ? m : n) || !(eps > 0.0 && eps < 1.0))
        return OR_ERR_ARG;
    if ((!tall || !op->A) && mode != ORACLE_F2) return OR_ERR_ARG;
    if (max_iter <= 0) max_iter = 10000;
    double *v0 = (double *)malloc((size_t)len * sizeof(double));
    double *v1 = (double *)malloc((size_t)len * sizeof(double));
    double *p = (double *)malloc((size_t)other * sizeof(double));
    if (!v0 || !v1 || !p) { free(v0); free(v1); free(p); return OR_ERR_NOMEM; }
    int status = OR_OK;
    for (int l = 0; l < k; ++l) {           /* P:75, 0-based: l components already found */
        const double *x = V0 + (size_t)l * (size_t)len;
        double nx = nrm2(x, len);
        if (!(nx > 0.0) || !isfinite(nx)) { status = OR_ERR_NUMERIC; goto done; }
        for (int64_t j = 0; j < len; ++j) v0[j] = x[j] / nx;
        int it = 0;
        double d = 0.0;
        for (;;) {                           /* P:119 while true */
            int rc;
            if (!tall) rc = oracle_gram_apply_wide(op->A, m, n, op->lda, U, k, S, V, k, l, v0, v1);
            else if (op->A) rc = oracle_gram_apply(mode, op->A, m, n, op->lda, U, k, S, V, k, l, v0, v1);
            else rc = gram_f2(op, m, n, U, k, S, V, k, l, v0, v1);
            if (rc != OR_OK) { status = rc; goto done; }
            double ny = nrm2(v1, len);
            if (!isfinite(ny)) { status = OR_ERR_NUMERIC; goto done; }
            if (ny == 0.0) { status = OR_RANK_EXHAUSTED; goto done; }   /* reading R14 */
            for (int64_t j = 0; j < len; ++j) v1[j] /= ny;
            ++it;
            d = fabs(dot(v0, v1, len));
            if (fixed_T > 0) {
                if (it >= fixed_T) break;
            } else if (d >= 1.0 - eps) {
                break;
            } else if (it >= max_iter) {
                status = OR_NOT_CONVERGED;
                break;
            }
            memcpy(v0, v1, (size_t)len * sizeof(double));
        }
        /* Extraction with the ORIGINAL A (P:85-87 / P:90-92) */
        if (tall) op_mv(op, m, n, v1, p);
        else op_mvt(op, m, n, v1, p);
        double sigma = nrm2(p, other);
        if (!isfinite(sigma)) { status = OR_ERR_NUMERIC; goto done; }
        if (sigma == 0.0) { status = OR_RANK_EXHAUSTED; goto done; }
        for (int64_t r = 0; r < other; ++r) p[r] /= sigma;
        double *Uo = tall ? U : V, *Vo = tall ? V : U;  /* tall: p = u, v1 = v */
        for (int64_t r = 0; r < other; ++r) Uo[r * k + l] = p[r];
        for (int64_t j = 0; j < len; ++j) Vo[j * k + l] = v1[j];
        S[l] = sigma;
        iters[l] = it;
        dots[l] = d;
        *k_found = l + 1;
    }
done:
    free(v0); free(v1); free(p);
    return status;
}

/* ---- independent check: one-sided Jacobi SVD (Hestenes), fp64 -------------------
 * Textbook algorithm (Golub & Van Loan §8.6.3 / Demmel–Veselic); used only to pin
 * oracle_tsvd on tiny matrices.  A (m x n, m >= n) fp64 row-major is overwritten.
 * On return sig[n] (descending), Vj (n x n row-major, columns = right vectors),
 * A's columns hold sigma_j u_j (unsorted order recorded in perm[n]).  Returns sweeps. */
int oracle_jacobi_svd(double *A, int64_t m, int64_t n, double *sig, double *Vj, int *perm, double tol, int max_sweeps) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) Vj[i * n + j] = (i == j) ? 1.0 : 0.0;
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        int rotated = 0;
        for (int64_t p = 0; p < n - 1; ++p)
            for (int64_t q = p + 1; q < n; ++q) {
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (int64_t r = 0; r < m; ++r) {
                    alpha += A[r * n + p] * A[r * n + p];
                    beta += A[r * n + q] * A[r * n + q];
                    gamma += A[r * n + p] * A[r * n + q];
                }
                if (fabs(gamma) <= tol * sqrt(alpha * beta) || gamma == 0.0) continue;
                rotated = 1;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int64_t r = 0; r < m; ++r) {
                    double ap = A[r * n + p], aq = A[r * n + q];
                    A[r * n + p] = c * ap - s * aq;
                    A[r * n + q] = s * ap + c * aq;
                }
                for (int64_t r = 0; r < n; ++r) {
                    double vp = Vj[r * n + p], vq = Vj[r * n + q];
                    Vj[r * n + p] = c * vp - s * vq;
                    Vj[r * n + q] = s * vp + c * vq;
                }
            }
        if (!rotated) break;
    }
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t r = 0; r < m; ++r) s += A[r * n + j] * A[r * n + j];
        sig[j] = sqrt(s);
        perm[j] = (int)j;
    }
    /* selection sort of indices by descending sigma */
    for (int64_t i = 0; i < n; ++i) {
        int64_t best = i;
        for (int64_t j = i + 1; j < n; ++j)
            if (sig[perm[j]] > sig[perm[best]]) best = j;
        int tmp = perm[i]; perm[i] = perm[best]; perm[best] = tmp;
    }
    double *ss = (double *)malloc((size_t)n * sizeof(double));
    if (ss) {
        for (int64_t i = 0; i < n; ++i) ss[i] = sig[perm[i]];
        memcpy(sig, ss, (size_t)n * sizeof(double));
        free(ss);
    }
    return sweep;
}
