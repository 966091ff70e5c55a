/*
 * sigattn_oracle.c -- fp64 CPU oracle for padding-aware bidirectional sigmoid attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (libsigattn.so and the
 * paper_2604_27124_b200 package) never calls, links or imports anything under oracle/.
 * It shares no code, headers or constants with the CUDA path.
 *
 * What it computes is the plain definition, not the tiled algorithm (tiling is an exact
 * re-association of the same sums, PAPER.md P:130 and Alg. 1), written out in fp64:
 *
 *   x_ij  = alpha * <q_i, k_j> + b_z                               Eq. 2; b per sequence P:582
 *   P_ij  = sigma(x_ij) if (i < n_q[z] and j < n_k[z]) else 0     mask-then-sigma, Alg. 1
 *   O_i   = sum_j P_ij v_j ;   O_i = 0 for i >= n_q[z]             Alg. 1
 *   dP_ij = <dO_i, v_j>                                            Alg. 2
 *   dS_ij = P_ij (1 - P_ij) dP_ij                                  Alg. 2 P:663 / Alg. 3
 *   dV_j  = sum_i P_ij dO_i                                        Alg. 3
 *   dQ_i  = alpha * sum_j dS_ij k_j                                Alg. 2
 *   dK_j  = alpha * sum_i dS_ij q_i                                Alg. 3
 *   padded rows of dQ, dK, dV are 0                                Alg. 2, Alg. 3
 *   db_z  = sum_h sum_(i,j valid) dS_ij   (learnable bias)  x_ij = ... + b_z, chain rule
 *
 * Mask reading (reading R2): "S + (-inf)(1 - mask)" is read as a select,
 * sigma(-inf) := 0 exactly; no -inf arithmetic is performed.
 *
 * Layout: every tensor is [B, H, N, d] contiguous (N = Nq for q/o/dout/dq, Nk for k/v/dk/dv).
 * Bias: one value per sequence, b[z] (the caller expands a scalar).
 * Per-row functions evaluate one output row from the definition; the full-tensor functions
 * loop the per-row functions over every row (OpenMP over rows only -- each row's sum is a
 * plain sequential loop over j (or i) in index order).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Numerically stable logistic function sigma(x) = 1 / (1 + e^{-x}). */
static double sigma_fp64(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

static double dot(const double* a, const double* b, int d) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) s += a[t] * b[t];
    return s;
}

/* P_ij for one (b,h) slice; 0 when i or j is padded (Alg. 1). */
static double p_entry(const double* qs, const double* ks, int d, int nq, int nk,
                      double alpha, double bias, int i, int j) {
    if (i >= nq || j >= nk) return 0.0;
    double x = alpha * dot(qs + (size_t)i * d, ks + (size_t)j * d, d) + bias;
    return sigma_fp64(x);
}

static size_t slice(int b, int h, int H, int N, int d) {
    return ((size_t)b * H + h) * (size_t)N * d;
}

static int clampn(int n, int N) { return n < 0 ? 0 : (n > N ? N : n); }

/* ---------------- per-row evaluations ---------------- */

/* O row i of (b,h):  O_i = sum_{j} P_ij v_j  (Eq. 2); zero if i >= n_q. */
void sigattn_oracle_o_row(int H, int Nq, int Nk, int d, const double* q, const double* k,
                          const double* v, const int32_t* nq, const int32_t* nk, double alpha,
                          const double* bias, int b, int h, int i, double* out) {
    const double* qs = q + slice(b, h, H, Nq, d);
    const double* ks = k + slice(b, h, H, Nk, d);
    const double* vs = v + slice(b, h, H, Nk, d);
    int nqb = clampn(nq[b], Nq), nkb = clampn(nk[b], Nk);
    for (int t = 0; t < d; ++t) out[t] = 0.0;
    if (i >= nqb) return;
    for (int j = 0; j < nkb; ++j) {
        double p = p_entry(qs, ks, d, nqb, nkb, alpha, bias[b], i, j);
        for (int t = 0; t < d; ++t) out[t] += p * vs[(size_t)j * d + t];
    }
}

/* dQ row i: alpha * sum_j P_ij(1-P_ij)<dO_i,v_j> k_j  (Alg. 2); zero if i >= n_q. */
void sigattn_oracle_dq_row(int H, int Nq, int Nk, int d, const double* q, const double* k,
                           const double* v, const double* dout, const int32_t* nq,
                           const int32_t* nk, double alpha, const double* bias, int b, int h,
                           int i, double* out) {
    const double* qs = q + slice(b, h, H, Nq, d);
    const double* ks = k + slice(b, h, H, Nk, d);
    const double* vs = v + slice(b, h, H, Nk, d);
    const double* dos = dout + slice(b, h, H, Nq, d);
    int nqb = clampn(nq[b], Nq), nkb = clampn(nk[b], Nk);
    for (int t = 0; t < d; ++t) out[t] = 0.0;
    if (i >= nqb) return;
    for (int j = 0; j < nkb; ++j) {
        double p = p_entry(qs, ks, d, nqb, nkb, alpha, bias[b], i, j);
        double dp = dot(dos + (size_t)i * d, vs + (size_t)j * d, d);
        double ds = p * (1.0 - p) * dp;
        for (int t = 0; t < d; ++t) out[t] += ds * ks[(size_t)j * d + t];
    }
    for (int t = 0; t < d; ++t) out[t] *= alpha;
}

/* dK row j and dV row j (Alg. 3); zero if j >= n_k. */
void sigattn_oracle_dkdv_row(int H, int Nq, int Nk, int d, const double* q, const double* k,
                             const double* v, const double* dout, const int32_t* nq,
                             const int32_t* nk, double alpha, const double* bias, int b, int h,
                             int j, double* dk_out, double* dv_out) {
    const double* qs = q + slice(b, h, H, Nq, d);
    const double* ks = k + slice(b, h, H, Nk, d);
    const double* vs = v + slice(b, h, H, Nk, d);
    const double* dos = dout + slice(b, h, H, Nq, d);
    int nqb = clampn(nq[b], Nq), nkb = clampn(nk[b], Nk);
    for (int t = 0; t < d; ++t) { dk_out[t] = 0.0; dv_out[t] = 0.0; }
    if (j >= nkb) return;
    for (int i = 0; i < nqb; ++i) {
        double p = p_entry(qs, ks, d, nqb, nkb, alpha, bias[b], i, j);
        double dp = dot(dos + (size_t)i * d, vs + (size_t)j * d, d);
        double ds = p * (1.0 - p) * dp;
        for (int t = 0; t < d; ++t) {
            dv_out[t] += p * dos[(size_t)i * d + t];
            dk_out[t] += ds * qs[(size_t)i * d + t];
        }
    }
    for (int t = 0; t < d; ++t) dk_out[t] *= alpha;
}

/* ---------------- full tensors ---------------- */

void sigattn_oracle_fwd(int B, int H, int Nq, int Nk, int d, const double* q, const double* k,
                        const double* v, const int32_t* nq, const int32_t* nk, double alpha,
                        const double* bias, double* o) {
    long long rows = (long long)B * H * Nq;
#pragma omp parallel for schedule(dynamic, 16)
    for (long long r = 0; r < rows; ++r) {
        int i = (int)(r % Nq);
        int bh = (int)(r / Nq);
        int b = bh / H, h = bh % H;
        sigattn_oracle_o_row(H, Nq, Nk, d, q, k, v, nq, nk, alpha, bias, b, h, i,
                             o + (size_t)r * d);
    }
}

void sigattn_oracle_bwd(int B, int H, int Nq, int Nk, int d, const double* q, const double* k,
                        const double* v, const double* dout, const int32_t* nq,
                        const int32_t* nk, double alpha, const double* bias, double* dq,
                        double* dk, double* dv) {
    long long qrows = (long long)B * H * Nq;
#pragma omp parallel for schedule(dynamic, 16)
    for (long long r = 0; r < qrows; ++r) {
        int i = (int)(r % Nq);
        int bh = (int)(r / Nq);
        sigattn_oracle_dq_row(H, Nq, Nk, d, q, k, v, dout, nq, nk, alpha, bias, bh / H, bh % H,
                              i, dq + (size_t)r * d);
    }
    long long krows = (long long)B * H * Nk;
#pragma omp parallel for schedule(dynamic, 16)
    for (long long r = 0; r < krows; ++r) {
        int j = (int)(r % Nk);
        int bh = (int)(r / Nk);
        sigattn_oracle_dkdv_row(H, Nq, Nk, d, q, k, v, dout, nq, nk, alpha, bias, bh / H,
                                bh % H, j, dk + (size_t)r * d, dv + (size_t)r * d);
    }
}

/* Row-sampled evaluation: rows[] are query rows (fwd / dq) or key rows (dkdv) of one (b,h).
 * Exact: O_i and dQ_i depend only on (q_i, dO_i, all K, V); dK_j, dV_j only on (k_j, v_j, all
 * Q, dO).  out arrays are [nrows, d]. */
void sigattn_oracle_fwd_rows(int H, int Nq, int Nk, int d, const double* q, const double* k,
                             const double* v, const int32_t* nq, const int32_t* nk,
                             double alpha, const double* bias, int b, int h,
                             const int32_t* rows, int nrows, double* o_rows) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int r = 0; r < nrows; ++r)
        sigattn_oracle_o_row(H, Nq, Nk, d, q, k, v, nq, nk, alpha, bias, b, h, rows[r],
                             o_rows + (size_t)r * d);
}

void sigattn_oracle_dq_rows(int H, int Nq, int Nk, int d, const double* q, const double* k,
                            const double* v, const double* dout, const int32_t* nq,
                            const int32_t* nk, double alpha, const double* bias, int b, int h,
                            const int32_t* rows, int nrows, double* dq_rows) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int r = 0; r < nrows; ++r)
        sigattn_oracle_dq_row(H, Nq, Nk, d, q, k, v, dout, nq, nk, alpha, bias, b, h, rows[r],
                              dq_rows + (size_t)r * d);
}

void sigattn_oracle_dkdv_rows(int H, int Nq, int Nk, int d, const double* q, const double* k,
                              const double* v, const double* dout, const int32_t* nq,
                              const int32_t* nk, double alpha, const double* bias, int b, int h,
                              const int32_t* rows, int nrows, double* dk_rows,
                              double* dv_rows) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int r = 0; r < nrows; ++r)
        sigattn_oracle_dkdv_row(H, Nq, Nk, d, q, k, v, dout, nq, nk, alpha, bias, b, h,
                                rows[r], dk_rows + (size_t)r * d, dv_rows + (size_t)r * d);
}

/* Intermediates of one (b,h) for the invariant pins: P, dP and dS as [Nq, Nk] matrices
 * (padded entries 0).  dS_ij = P_ij (1 - P_ij) dP_ij. */
void sigattn_oracle_p_ds(int H, int Nq, int Nk, int d, const double* q, const double* k,
                         const double* v, const double* dout, const int32_t* nq,
                         const int32_t* nk, double alpha, const double* bias, int b, int h,
                         double* P, double* dP, double* dS) {
    const double* qs = q + slice(b, h, H, Nq, d);
    const double* ks = k + slice(b, h, H, Nk, d);
    const double* vs = v + slice(b, h, H, Nk, d);
    const double* dos = dout + slice(b, h, H, Nq, d);
    int nqb = clampn(nq[b], Nq), nkb = clampn(nk[b], Nk);
    for (int i = 0; i < Nq; ++i)
        for (int j = 0; j < Nk; ++j) {
            size_t e = (size_t)i * Nk + j;
            if (i >= nqb || j >= nkb) { P[e] = 0.0; dP[e] = 0.0; dS[e] = 0.0; continue; }
            double p = p_entry(qs, ks, d, nqb, nkb, alpha, bias[b], i, j);
            double dp = dot(dos + (size_t)i * d, vs + (size_t)j * d, d);
            P[e] = p;
            dP[e] = dp;
            dS[e] = p * (1.0 - p) * dp;
        }
}

/* Gradient of sum(dout * O) w.r.t. the per-sequence bias b_z ("fixed or learnable"; x =
 * alpha s + b_z enters every valid logit of sequence z, so dL/db_z = sum over heads h and valid
 * (i, j) of dS_ij, dS = P (1 - P) dP as in Alg. 2 line P:663).  db is [B]. */
void sigattn_oracle_dbias(int B, int H, int Nq, int Nk, int d, const double* q, const double* k,
                          const double* v, const double* dout, const int32_t* nq, const int32_t* nk,
                          double alpha, const double* bias, double* db) {
    for (int b = 0; b < B; ++b) {
        int nqb = clampn(nq[b], Nq), nkb = clampn(nk[b], Nk);
        double acc = 0.0;
#pragma omp parallel for reduction(+ : acc) schedule(dynamic, 4)
        for (long long r = 0; r < (long long)H * nqb; ++r) {
            int h = (int)(r / (nqb > 0 ? nqb : 1)), i = (int)(r % (nqb > 0 ? nqb : 1));
            const double* qs = q + slice(b, h, H, Nq, d);
            const double* ks = k + slice(b, h, H, Nk, d);
            const double* vs = v + slice(b, h, H, Nk, d);
            const double* dos = dout + slice(b, h, H, Nq, d);
            for (int j = 0; j < nkb; ++j) {
                double p = p_entry(qs, ks, d, nqb, nkb, alpha, bias[b], i, j);
                double dp = dot(dos + (size_t)i * d, vs + (size_t)j * d, d);
                acc += p * (1.0 - p) * dp;
            }
        }
        db[b] = acc;
    }
}

int sigattn_oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
