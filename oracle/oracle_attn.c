/*
 * oracle_attn.c -- plain, slow, fp64 CPU attention oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2511_02132_b200/csrc, include/).
 *
 * What it computes is the plain definition of attention, NOT the tiled
 * FlashAttention algorithm:
 *
 *   PAPER.md:149-155 (eq:fa)   S = Q K^T,  P = softmax(S / sqrt(d)),  O = P V
 *   PAPER.md:167               MHA / GQA: K,V shared by groups of query heads
 *   PAPER.md:172               FA "ensures numerical correctness": the tiled
 *                              algorithm reaches exactly this result up to
 *                              rounding, so the oracle is the definition.
 *   PAPER.md:187 (fig:attn-grid) tensors are Z x H x N_CTX x HEAD_DIM.
 *
 * Readings of points the paper leaves open:
 *   R1  scale is an explicit argument (eq:fa fixes 1/sqrt(d); callers pass it).
 *   R2  causal: key j is visible to query i iff j <= i (N_q == N_k).
 *   R3  GQA grouping g = h / (Hq / Hkv).
 *   R5  layout [B][H][N][d] contiguous, row-major.
 *
 * Per query row (b, h, i), with g = h / (Hq/Hkv) and J the visible keys:
 *   s_j = scale * sum_{c<d} q[b,h,i,c] * k[b,g,j,c]      (fp64, c ascending)
 *   m   = max_{j in J} s_j
 *   w_j = exp(s_j - m)                                     (libm exp, fp64)
 *   l   = sum_{j in J} w_j                                 (j ascending)
 *   o_c = (sum_{j in J} w_j * v[b,g,j,c]) / l
 * Two passes over the keys; no online softmax, no blocking, no reordering.
 *
 * Input element types (dtype argument):
 *   0 = bf16 given as raw uint16 bit patterns, widened EXACTLY
 *       ((uint32)bits << 16 reinterpreted as float, then to double);
 *   1 = float32;   2 = float64.
 * Output is always float64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double oracle_widen(const void *base, int dtype, int64_t idx) {
    if (dtype == 0) {
        uint32_t u = ((uint32_t)((const uint16_t *)base)[idx]) << 16;
        float f;
        memcpy(&f, &u, sizeof f);
        return (double)f;
    }
    if (dtype == 1) return (double)((const float *)base)[idx];
    return ((const double *)base)[idx];
}

static int oracle_check(int dtype, int B, int Hq, int Hkv, int N, int d) {
    if (dtype < 0 || dtype > 2) return 1;
    if (B <= 0 || Hq <= 0 || Hkv <= 0 || N <= 0 || d <= 0) return 1;
    if (Hq % Hkv != 0) return 1;
    return 0;
}

/* One query row: fills out[0..d) and, if w != NULL, the normalised weights
 * w[0..N) (zero for masked keys).  s is caller scratch of N doubles. */
static void oracle_row(const void *q, const void *k, const void *v, int dtype,
                       int Hq, int Hkv, int N, int d, int causal, double scale,
                       int64_t b, int64_t h, int64_t i,
                       double *s, double *out, double *w) {
    const int64_t g = h / (Hq / Hkv);
    const int64_t qrow = ((b * Hq + h) * (int64_t)N + i) * d;
    const int64_t kvbase = (b * Hkv + g) * (int64_t)N;
    const int64_t nvis = causal ? i + 1 : N; /* keys 0..nvis-1 visible */

    double m = -INFINITY;
    for (int64_t j = 0; j < nvis; ++j) {
        double acc = 0.0;
        const int64_t krow = (kvbase + j) * d;
        for (int c = 0; c < d; ++c)
            acc += oracle_widen(q, dtype, qrow + c) * oracle_widen(k, dtype, krow + c);
        s[j] = scale * acc;
        if (s[j] > m) m = s[j];
    }
    double l = 0.0;
    for (int64_t j = 0; j < nvis; ++j) {
        s[j] = exp(s[j] - m); /* s now holds the unnormalised weights w_j */
        l += s[j];
    }
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int64_t j = 0; j < nvis; ++j) {
        const int64_t vrow = (kvbase + j) * d;
        for (int c = 0; c < d; ++c) out[c] += s[j] * oracle_widen(v, dtype, vrow + c);
    }
    for (int c = 0; c < d; ++c) out[c] /= l;
    if (w) {
        for (int64_t j = 0; j < N; ++j) w[j] = (j < nvis) ? s[j] / l : 0.0;
    }
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Row-sampled oracle: rows[3*r + {0,1,2}] = (b, h, i); out is nrows x d. */
int oracle_attn_rows(const void *q, const void *k, const void *v, int dtype,
                     int B, int Hq, int Hkv, int N, int d, int causal, double scale,
                     const int64_t *rows, int64_t nrows, double *out) {
    if (oracle_check(dtype, B, Hq, Hkv, N, d)) return 1;
    for (int64_t r = 0; r < nrows; ++r) {
        if (rows[3 * r] < 0 || rows[3 * r] >= B || rows[3 * r + 1] < 0 ||
            rows[3 * r + 1] >= Hq || rows[3 * r + 2] < 0 || rows[3 * r + 2] >= N)
            return 1;
    }
    int err = 0;
#pragma omp parallel
    {
        double *s = (double *)malloc(sizeof(double) * (size_t)N);
        if (!s) {
#pragma omp atomic write
            err = 2;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t r = 0; r < nrows; ++r)
                oracle_row(q, k, v, dtype, Hq, Hkv, N, d, causal, scale, rows[3 * r],
                           rows[3 * r + 1], rows[3 * r + 2], s, out + r * d, NULL);
            free(s);
        }
    }
    return err;
}

/* Full oracle: out is B x Hq x N x d (float64). */
int oracle_attn_full(const void *q, const void *k, const void *v, int dtype,
                     int B, int Hq, int Hkv, int N, int d, int causal, double scale,
                     double *out) {
    if (oracle_check(dtype, B, Hq, Hkv, N, d)) return 1;
    const int64_t total = (int64_t)B * Hq * N;
    int err = 0;
#pragma omp parallel
    {
        double *s = (double *)malloc(sizeof(double) * (size_t)N);
        if (!s) {
#pragma omp atomic write
            err = 2;
        } else {
#pragma omp for schedule(dynamic, 16)
            for (int64_t r = 0; r < total; ++r) {
                const int64_t i = r % N, h = (r / N) % Hq, b = r / ((int64_t)N * Hq);
                oracle_row(q, k, v, dtype, Hq, Hkv, N, d, causal, scale, b, h, i, s,
                           out + r * d, NULL);
            }
            free(s);
        }
    }
    return err;
}

/* Debug hook for the softmax pins: normalised weights P[b,h,i,:] (N doubles,
 * zero where masked) and the output row (d doubles). */
int oracle_attn_weights(const void *q, const void *k, const void *v, int dtype,
                        int B, int Hq, int Hkv, int N, int d, int causal, double scale,
                        int64_t b, int64_t h, int64_t i, double *w, double *out) {
    if (oracle_check(dtype, B, Hq, Hkv, N, d)) return 1;
    if (b < 0 || b >= B || h < 0 || h >= Hq || i < 0 || i >= N) return 1;
    double *s = (double *)malloc(sizeof(double) * (size_t)N);
    if (!s) return 2;
    oracle_row(q, k, v, dtype, Hq, Hkv, N, d, causal, scale, b, h, i, s, out, w);
    free(s);
    return 0;
}

/* ------------------------------------------------------------------ backward
 * PAPER.md:157-165 (eq:ba), for P = softmax(scale * Q K^T) (masked as in the
 * forward) and an upstream gradient dO:
 *   dV = P^T dO,   dP = dO V^T,   dS = dsoftmax(dP) = P o (dP - rowsum(P o dP)),
 *   dQ = scale * dS K,   dK = scale * dS^T Q.
 * GQA: dK, dV of a KV group sum over the query heads of the group.
 * Plain definition: per (b, h) the full N x N matrices P and dP in fp64; no
 * tiling, no recomputation tricks.  Outputs are fp64, zero-initialised here.
 * Also returns lse[b,h,i] = log sum_j exp(scale * s_ij) (natural log) when lse
 * is non-NULL. */
int oracle_attn_bwd(const void *q, const void *k, const void *v, const void *dout, int dtype,
                    int B, int Hq, int Hkv, int N, int d, int causal, double scale,
                    double *dq, double *dk, double *dv, double *lse) {
    if (oracle_check(dtype, B, Hq, Hkv, N, d)) return 1;
    const int G = Hq / Hkv;
    const int64_t hsz = (int64_t)N * d;
    for (int64_t x = 0; x < (int64_t)B * Hq * hsz; ++x) dq[x] = 0.0;
    for (int64_t x = 0; x < (int64_t)B * Hkv * hsz; ++x) { dk[x] = 0.0; dv[x] = 0.0; }
    double *P = (double *)malloc(sizeof(double) * (size_t)N * N);
    double *dP = (double *)malloc(sizeof(double) * (size_t)N * N);
    if (!P || !dP) { free(P); free(dP); return 2; }
    for (int b = 0; b < B; ++b) {
        for (int h = 0; h < Hq; ++h) {
            const int g = h / G;
            const int64_t qo = ((int64_t)b * Hq + h) * hsz, ko = ((int64_t)b * Hkv + g) * hsz;
            /* P: row-wise two-pass softmax (same definition as the forward) */
#pragma omp parallel for schedule(dynamic, 8)
            for (int i = 0; i < N; ++i) {
                const int nvis = causal ? i + 1 : N;
                double m = -INFINITY;
                for (int j = 0; j < nvis; ++j) {
                    double acc = 0.0;
                    for (int c = 0; c < d; ++c)
                        acc += oracle_widen(q, dtype, qo + (int64_t)i * d + c) *
                               oracle_widen(k, dtype, ko + (int64_t)j * d + c);
                    P[(int64_t)i * N + j] = scale * acc;
                    if (P[(int64_t)i * N + j] > m) m = P[(int64_t)i * N + j];
                }
                double l = 0.0;
                for (int j = 0; j < nvis; ++j) {
                    P[(int64_t)i * N + j] = exp(P[(int64_t)i * N + j] - m);
                    l += P[(int64_t)i * N + j];
                }
                for (int j = 0; j < N; ++j) P[(int64_t)i * N + j] = (j < nvis) ? P[(int64_t)i * N + j] / l : 0.0;
                if (lse) lse[((int64_t)b * Hq + h) * N + i] = m + log(l);
                /* dP = dO V^T, then dS = P o (dP - rowsum(P o dP)) in place */
                double dot = 0.0;
                for (int j = 0; j < N; ++j) {
                    double acc = 0.0;
                    if (j < nvis)
                        for (int c = 0; c < d; ++c)
                            acc += oracle_widen(dout, dtype, qo + (int64_t)i * d + c) *
                                   oracle_widen(v, dtype, ko + (int64_t)j * d + c);
                    dP[(int64_t)i * N + j] = acc;
                    dot += P[(int64_t)i * N + j] * acc;
                }
                for (int j = 0; j < N; ++j) dP[(int64_t)i * N + j] = P[(int64_t)i * N + j] * (dP[(int64_t)i * N + j] - dot);
                /* dQ_i = scale * sum_j dS_ij K_j */
                for (int j = 0; j < nvis; ++j)
                    for (int c = 0; c < d; ++c)
                        dq[qo + (int64_t)i * d + c] += scale * dP[(int64_t)i * N + j] * oracle_widen(k, dtype, ko + (int64_t)j * d + c);
            }
            /* dV_j += sum_i P_ij dO_i ;  dK_j += scale * sum_i dS_ij Q_i */
#pragma omp parallel for schedule(dynamic, 8)
            for (int j = 0; j < N; ++j) {
                for (int i = 0; i < N; ++i) {
                    const double p = P[(int64_t)i * N + j], ds = dP[(int64_t)i * N + j];
                    if (p == 0.0 && ds == 0.0) continue;
                    for (int c = 0; c < d; ++c) {
                        dv[ko + (int64_t)j * d + c] += p * oracle_widen(dout, dtype, qo + (int64_t)i * d + c);
                        dk[ko + (int64_t)j * d + c] += scale * ds * oracle_widen(q, dtype, qo + (int64_t)i * d + c);
                    }
                }
            }
        }
    }
    free(P);
    free(dP);
    return 0;
}
