/*
 * oracle/lora_oracle.c -- CPU fp64 oracle for the JORA LoRA-linear hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2403_11366_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   PAPER.md:109 (Sec. 3, "JORA Framework"): W0 in R^{m x n}, A in R^{r x n},
 *     B in R^{m x r}; the computation W0 x + b0 is tuned to W0 x + b0 + B A x.
 *   PAPER.md:115-120 (Eq. 1):  Output = W0 x + b0 + B A x = (W0 + B A) x + b0.
 *   "B and A are the trainable weights" -> gradients for A, B
 *     (and for the input x, which the previous layer needs); none for W0, b0.
 *   PAPER.md:80-81 (Listing 3): LORA_R, LORA_ALPHA -> scale s = alpha / r
 *     (reading R2; at the paper defaults 16/16, s = 1 and Eq. 1
 *     holds verbatim).
 *
 * Orientation (reading R1): the paper writes column vectors; we
 * store tokens as rows, so for token t (row t of x):
 *   h[t,j]  = sum_k x[t,k] A[j,k]                       ("A x")
 *   y[t,i]  = sum_k x[t,k] W0[i,k] + s sum_j h[t,j] B[i,j] + b0[i]
 * Backward of L with upstream G = dL/dy (plain chain rule of the bilinear
 * map above; no approximation):
 *   gh[t,j] = s sum_i G[t,i] B[i,j]                     (dL/dh)
 *   dX[t,k] = sum_i G[t,i] W0[i,k] + sum_j gh[t,j] A[j,k]
 *   dA[j,k] = sum_t gh[t,j] x[t,k]
 *   dB[i,j] = s sum_t G[t,i] h[t,j]
 * Merge (Eq. 1, second line; PAPER.md:92-106 export script):
 *   W'[i,k] = W0[i,k] + s sum_j B[i,j] A[j,k]
 *
 * Arithmetic: every input is a bf16 bit pattern ("brain
 * floating point"), widened exactly to double; every sum is accumulated in
 * double in ascending index order, exactly as written above.  OpenMP only
 * splits independent output elements across threads, so results are bitwise
 * independent of the thread count.  Loops are interchanged for cache
 * friendliness where that leaves each element's summation order unchanged.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* bf16 bit pattern -> double.  bf16 is the upper half of an IEEE binary32. */
static double bf(uint16_t bits) {
    uint32_t u = (uint32_t)bits << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int nt) {
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}

/* s = alpha / r  (reading R2). */
double oracle_scale(int r, double alpha) { return alpha / (double)r; }

static int bad_dims(int64_t T, int64_t n, int64_t m, int r) {
    return T < 0 || n <= 0 || m <= 0 || r <= 0;
}

/* Row t's index in the full [T, .] tensors: rows[q] if a row subset is
 * given, else q itself. */
static int64_t row_of(const int64_t* rows, int64_t q) { return rows ? rows[q] : q; }

/*
 * Forward, Eq. 1 line 1.  Computes the n_rows selected tokens
 * (rows == NULL: all T tokens, n_rows must equal T).
 *   y_out : [n_rows, m] double     h_out : [n_rows, r] double (nullable)
 * bias may be NULL (Llama-2 projections have none).  Returns 0, or -1 on bad
 * arguments.
 */
int oracle_lora_fwd(int64_t T, int64_t n, int64_t m, int r, double alpha,
                    const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                    const uint16_t* b, const uint16_t* bias,
                    const int64_t* rows, int64_t n_rows,
                    double* y_out, double* h_out) {
    if (bad_dims(T, n, m, r) || !x || !w0 || !a || !b || !y_out) return -1;
    if (!rows && n_rows != T) return -1;
    const double s = oracle_scale(r, alpha);
    int64_t q;
#pragma omp parallel for schedule(dynamic, 1)
    for (q = 0; q < n_rows; ++q) {
        const int64_t t = row_of(rows, q);
        const uint16_t* xt = x + t * n;
        double* h = (double*)malloc(sizeof(double) * (size_t)r);
        /* h[t,j] = sum_k x[t,k] A[j,k]  -- "A x" of Eq. 1 */
        for (int j = 0; j < r; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < n; ++k) acc += bf(xt[k]) * bf(a[(int64_t)j * n + k]);
            h[j] = acc;
            if (h_out) h_out[q * r + j] = acc;
        }
        for (int64_t i = 0; i < m; ++i) {
            /* base term W0 x */
            double base = 0.0;
            const uint16_t* wi = w0 + i * n;
            for (int64_t k = 0; k < n; ++k) base += bf(xt[k]) * bf(wi[k]);
            /* low-rank term B (A x), scaled by s */
            double lora = 0.0;
            for (int j = 0; j < r; ++j) lora += h[j] * bf(b[i * r + j]);
            double v = base + s * lora;
            if (bias) v += bf(bias[i]);
            y_out[q * m + i] = v;
        }
        free(h);
    }
    return 0;
}

/*
 * Backward of Eq. 1 w.r.t. x, A, B for upstream gradient G = dy [T, m]
 * (A, B trainable; W0, b0 frozen -> no dW0, no db0).
 *   dx_out : [n_rows, n] for the selected rows (nullable)
 *   gh_out : [T, r]   dL/dh for every token (nullable)
 *   da_out : [r, n]   (nullable)        db_out : [m, r] (nullable)
 * dA and dB are reductions over all T tokens, so they always use every row.
 */
int oracle_lora_bwd(int64_t T, int64_t n, int64_t m, int r, double alpha,
                    const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                    const uint16_t* b, const uint16_t* dy,
                    const int64_t* rows, int64_t n_rows,
                    double* dx_out, double* gh_out, double* da_out, double* db_out) {
    if (bad_dims(T, n, m, r) || !x || !w0 || !a || !b || !dy) return -1;
    if (dx_out && !rows && n_rows != T) return -1;
    const double s = oracle_scale(r, alpha);
    double* h = (double*)malloc(sizeof(double) * (size_t)(T * r + 1));
    double* gh = (double*)malloc(sizeof(double) * (size_t)(T * r + 1));
    if (!h || !gh) { free(h); free(gh); return -2; }
    int64_t t;
    /* h[t,j] = sum_k x[t,k] A[j,k];  gh[t,j] = s * sum_i G[t,i] B[i,j] */
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        for (int j = 0; j < r; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < n; ++k) acc += bf(x[t * n + k]) * bf(a[(int64_t)j * n + k]);
            h[t * r + j] = acc;
            double g = 0.0;
            for (int64_t i = 0; i < m; ++i) g += bf(dy[t * m + i]) * bf(b[i * r + j]);
            gh[t * r + j] = s * g;
        }
    }
    if (gh_out) memcpy(gh_out, gh, sizeof(double) * (size_t)(T * r));

    /* dX[t,k] = sum_i G[t,i] W0[i,k] + sum_j gh[t,j] A[j,k]
     * (i-loop outside the k-loop: each dX[t,k] still sums i = 0..m-1 in order) */
    if (dx_out) {
        int64_t q;
#pragma omp parallel for schedule(dynamic, 1)
        for (q = 0; q < n_rows; ++q) {
            const int64_t tt = row_of(rows, q);
            double* base = (double*)calloc((size_t)n, sizeof(double));
            for (int64_t i = 0; i < m; ++i) {
                const double g = bf(dy[tt * m + i]);
                const uint16_t* wi = w0 + i * n;
                for (int64_t k = 0; k < n; ++k) base[k] += g * bf(wi[k]);
            }
            for (int64_t k = 0; k < n; ++k) {
                double lora = 0.0;
                for (int j = 0; j < r; ++j) lora += gh[tt * r + j] * bf(a[(int64_t)j * n + k]);
                dx_out[q * n + k] = base[k] + lora;
            }
            free(base);
        }
    }
    /* dA[j,k] = sum_t gh[t,j] x[t,k]   (t ascending) */
    if (da_out) {
        int64_t k;
#pragma omp parallel for schedule(static)
        for (k = 0; k < n; ++k) {
            for (int j = 0; j < r; ++j) {
                double acc = 0.0;
                for (int64_t tt = 0; tt < T; ++tt) acc += gh[tt * r + j] * bf(x[tt * n + k]);
                da_out[(int64_t)j * n + k] = acc;
            }
        }
    }
    /* dB[i,j] = s * sum_t G[t,i] h[t,j]   (t ascending) */
    if (db_out) {
        int64_t i;
#pragma omp parallel for schedule(static)
        for (i = 0; i < m; ++i) {
            for (int j = 0; j < r; ++j) {
                double acc = 0.0;
                for (int64_t tt = 0; tt < T; ++tt) acc += bf(dy[tt * m + i]) * h[tt * r + j];
                db_out[i * r + j] = s * acc;
            }
        }
    }
    free(h);
    free(gh);
    return 0;
}

/*
 * Merge, Eq. 1 line 2 and the export script:
 *   W'[i,k] = W0[i,k] + s * sum_j B[i,j] A[j,k]      w_out : [m, n] double
 */
int oracle_lora_merge(int64_t n, int64_t m, int r, double alpha,
                      const uint16_t* w0, const uint16_t* a, const uint16_t* b,
                      double* w_out) {
    if (bad_dims(0, n, m, r) || !w0 || !a || !b || !w_out) return -1;
    const double s = oracle_scale(r, alpha);
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < m; ++i) {
        for (int64_t k = 0; k < n; ++k) {
            double ba = 0.0;
            for (int j = 0; j < r; ++j) ba += bf(b[i * r + j]) * bf(a[(int64_t)j * n + k]);
            w_out[i * n + k] = bf(w0[i * n + k]) + s * ba;
        }
    }
    return 0;
}
