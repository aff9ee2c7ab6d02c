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
 * LoRA dropout (Listing 3, LORA_DROPOUT = 0.05; placement per
 * DESIGN.md reading R7: inverted dropout on the adapter input only, the
 * frozen path never sees it): with keep mask M[t,k] in {0,1} and
 * q = 1/(1-p),  xd[t,k] = q M[t,k] x[t,k]  replaces x in "A x":
 *   h[t,j]  = sum_k xd[t,k] A[j,k]
 *   dX[t,k] = sum_i G[t,i] W0[i,k] + q M[t,k] sum_j gh[t,j] A[j,k]
 *   dA[j,k] = sum_t gh[t,j] xd[t,k]          (y, gh, dB unchanged given h)
 * M is a pure function of (t, k, seed, offset, p) through Philox4x32-10
 * (Salmon et al., SC'11), so the backward regenerates it; each 32-bit output
 * word gives two 16-bit draws (R7, round 2: one Philox block per 8
 * columns, p resolved to 2^-16):
 *   (w0..w3) = Philox4x32-10(counter = (k/8, t, offset_lo, offset_hi),
 *                            key = (seed_lo, seed_hi));
 *   u[t,k]   = (w_{(k mod 8) / 2} >> (16 ((k mod 8) mod 2))) & 0xFFFF;
 *   M[t,k]   = (u[t,k] >= floor(p 2^16)).
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
#include <math.h>
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
/* adapter input xd[t,k] of the dropout reading (mask == NULL: x itself) */
static double xin(const uint16_t* x, const uint8_t* mask, double q, int64_t idx) {
    if (!mask) return bf(x[idx]);
    return mask[idx] ? q * bf(x[idx]) : 0.0;
}

static int lora_fwd_impl(int64_t T, int64_t n, int64_t m, int r, double alpha,
                         const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                         const uint16_t* b, const uint16_t* bias,
                         const uint8_t* mask, double q,
                         const int64_t* rows, int64_t n_rows,
                         double* y_out, double* h_out) {
    if (bad_dims(T, n, m, r) || !x || !w0 || !a || !b || !y_out) return -1;
    if (!rows && n_rows != T) return -1;
    const double s = oracle_scale(r, alpha);
    int64_t qq;
#pragma omp parallel for schedule(dynamic, 1)
    for (qq = 0; qq < n_rows; ++qq) {
        const int64_t t = row_of(rows, qq);
        const uint16_t* xt = x + t * n;
        double* h = (double*)malloc(sizeof(double) * (size_t)r);
        /* h[t,j] = sum_k x[t,k] A[j,k]  -- "A x" of Eq. 1 (xd under dropout) */
        for (int j = 0; j < r; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < n; ++k) acc += xin(x, mask, q, t * n + k) * bf(a[(int64_t)j * n + k]);
            h[j] = acc;
            if (h_out) h_out[qq * r + j] = acc;
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
            y_out[qq * m + i] = v;
        }
        free(h);
    }
    return 0;
}

int oracle_lora_fwd(int64_t T, int64_t n, int64_t m, int r, double alpha,
                    const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                    const uint16_t* b, const uint16_t* bias,
                    const int64_t* rows, int64_t n_rows,
                    double* y_out, double* h_out) {
    return lora_fwd_impl(T, n, m, r, alpha, x, w0, a, b, bias, NULL, 1.0, rows, n_rows, y_out, h_out);
}

/* Forward with LoRA dropout: mask [T, n] of 0/1, q = 1 / (1 - p). */
int oracle_lora_fwd_dropout(int64_t T, int64_t n, int64_t m, int r, double alpha,
                            const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                            const uint16_t* b, const uint16_t* bias,
                            const uint8_t* mask, double q,
                            const int64_t* rows, int64_t n_rows,
                            double* y_out, double* h_out) {
    if (!mask) return -1;
    return lora_fwd_impl(T, n, m, r, alpha, x, w0, a, b, bias, mask, q, rows, n_rows, y_out, h_out);
}

/*
 * Backward of Eq. 1 w.r.t. x, A, B for upstream gradient G = dy [T, m]
 * (A, B trainable; W0, b0 frozen -> no dW0, no db0).
 *   dx_out : [n_rows, n] for the selected rows (nullable)
 *   gh_out : [T, r]   dL/dh for every token (nullable)
 *   da_out : [r, n]   (nullable)        db_out : [m, r] (nullable)
 * dA and dB are reductions over all T tokens, so they always use every row.
 */
static int lora_bwd_impl(int64_t T, int64_t n, int64_t m, int r, double alpha,
                         const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                         const uint16_t* b, const uint16_t* dy,
                         const uint8_t* mask, double q,
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
            for (int64_t k = 0; k < n; ++k) acc += xin(x, mask, q, t * n + k) * bf(a[(int64_t)j * n + k]);
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
        int64_t qq;
#pragma omp parallel for schedule(dynamic, 1)
        for (qq = 0; qq < n_rows; ++qq) {
            const int64_t tt = row_of(rows, qq);
            double* base = (double*)calloc((size_t)n, sizeof(double));
            for (int64_t i = 0; i < m; ++i) {
                const double g = bf(dy[tt * m + i]);
                const uint16_t* wi = w0 + i * n;
                for (int64_t k = 0; k < n; ++k) base[k] += g * bf(wi[k]);
            }
            for (int64_t k = 0; k < n; ++k) {
                double lora = 0.0;
                for (int j = 0; j < r; ++j) lora += gh[tt * r + j] * bf(a[(int64_t)j * n + k]);
                if (mask) lora = mask[tt * n + k] ? q * lora : 0.0;   /* through the dropout */
                dx_out[qq * n + k] = base[k] + lora;
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
                for (int64_t tt = 0; tt < T; ++tt) acc += gh[tt * r + j] * xin(x, mask, q, tt * n + k);
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

int oracle_lora_bwd(int64_t T, int64_t n, int64_t m, int r, double alpha,
                    const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                    const uint16_t* b, const uint16_t* dy,
                    const int64_t* rows, int64_t n_rows,
                    double* dx_out, double* gh_out, double* da_out, double* db_out) {
    return lora_bwd_impl(T, n, m, r, alpha, x, w0, a, b, dy, NULL, 1.0, rows, n_rows, dx_out, gh_out, da_out,
                         db_out);
}

/* Backward with LoRA dropout (same mask and q as the forward). */
int oracle_lora_bwd_dropout(int64_t T, int64_t n, int64_t m, int r, double alpha,
                            const uint16_t* x, const uint16_t* w0, const uint16_t* a,
                            const uint16_t* b, const uint16_t* dy,
                            const uint8_t* mask, double q,
                            const int64_t* rows, int64_t n_rows,
                            double* dx_out, double* gh_out, double* da_out, double* db_out) {
    if (!mask) return -1;
    return lora_bwd_impl(T, n, m, r, alpha, x, w0, a, b, dy, mask, q, rows, n_rows, dx_out, gh_out, da_out,
                         db_out);
}

/*
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 * easy as 1, 2, 3", SC'11): 10 rounds of
 *   (c0, c1, c2, c3) <- (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0))
 * with the key bumped by (W0, W1) between rounds.
 */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += W0; k1 += W1; }
        const uint64_t p0 = (uint64_t)M0 * c[0];
        const uint64_t p1 = (uint64_t)M1 * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* keep threshold: floor(p 2^16) for the fp32 dropout probability p in [0, 1) */
uint32_t oracle_dropout_threshold(float p) {
    const double v = (double)p * 65536.0;
    return (uint32_t)v;   /* truncation == floor for v >= 0 */
}

/* M[t,k] in {0,1} for a [T, n] activation (header comment above). */
int oracle_dropout_mask(int64_t T, int64_t n, float p, uint64_t seed, uint64_t offset, uint8_t* mask) {
    if (T < 0 || n <= 0 || !(p >= 0.0f && p < 1.0f) || !mask) return -1;
    const uint32_t thr = oracle_dropout_threshold(p);
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        for (int64_t k = 0; k < n; ++k) {
            const uint32_t ctr[4] = {(uint32_t)(k / 8), (uint32_t)t, (uint32_t)offset, (uint32_t)(offset >> 32)};
            uint32_t w[4];
            oracle_philox4x32_10(ctr, key, w);
            const uint32_t u = (w[(k % 8) / 2] >> (16 * ((k % 8) % 2))) & 0xFFFFu;
            mask[t * n + k] = u >= thr ? 1 : 0;
        }
    }
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

/*
 * Adapter update ("standard bias-corrected
 * Adam"; the paper names no optimizer): Adam, Kingma & Ba, ICLR
 * 2015, Algorithm 1, one step t >= 1 for `count` independent elements:
 *   m <- b1 m + (1 - b1) g;   v <- b2 v + (1 - b2) g^2
 *   m_hat = m / (1 - b1^t);   v_hat = v / (1 - b2^t)
 *   theta <- theta - lr m_hat / (sqrt(v_hat) + eps)
 * All in fp64, in place.
 */
int oracle_adam_step(int64_t count, double* theta, const double* grad, double* m, double* v, int64_t t,
                     double lr, double b1, double b2, double eps) {
    if (count < 0 || t < 1 || !theta || !grad || !m || !v) return -1;
    const double bc1 = 1.0 - pow(b1, (double)t);
    const double bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < count; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * grad[i];
        v[i] = b2 * v[i] + (1.0 - b2) * grad[i] * grad[i];
        const double m_hat = m[i] / bc1;
        const double v_hat = v[i] / bc2;
        theta[i] = theta[i] - lr * m_hat / (sqrt(v_hat) + eps);
    }
    return 0;
}
