/*
 * starsd_ref.c -- CPU ORACLE for the StarSD speculative-sampling verify step.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs, never by the product path.  Shares no code
 * with paper_2601_21622_b200/ or include/ (see DESIGN.md "Oracle").
 *
 * What it computes (Appendix D, Algorithm 2), per request:
 *   p_1..p_{d+1}  = target next-token distributions along the drafted chain
 *   r_i ~ U(0,1), l = min({i-1 : test i fails} U {d})
 *   if l < d: t ~ norm(max(0, p_{l+1} - q_{l+1}))
 * read with SURVEY.md 8(c):
 *   C-1  the acceptance test is the ratio rule: accept x_j iff u < min(1, p_j(x_j)/q_j(x_j))
 *   C-2  u on the 2^-24 grid; accept iff u < a; a >= 1 accepts without consulting u
 *   C-3  bonus token t ~ p_k at full acceptance (l = d)
 *   C-4  p_j = softmax(z_p,j / T), q_j = softmax(z_q,j / T), same T
 *   C-5  T == 0: greedy, argmax matching, lowest index on ties, q unused
 *   C-6  zero residual -> sample from p_L (informational status bit)
 *   C-7  q_j(x_j) = 0 -> rejection (informational status bit)
 *   C-8  Philox4x32-10, key = seed, ctr = (j, round_lo, rid_lo, rid_hi); u_acc = u24(w0), u_smp = u24(w1)
 *   C-9  inverse CDF in ascending token id, strict C(x) > theta; clamp to last positive-mass token
 *   C-10 0-based: p rows j = 0..k, q rows j = 0..k-1; residual at L uses (p_L, q_L)
 *   C-11 fp64 throughout
 *   C-12 -inf logits allowed; NaN, +inf, an all -inf row, or a draft id outside [0,V) are faults
 * It is lazy: rows after the first rejection are never read (the method's data dependency).
 */
#include "starsd_ref.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10.  Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
 * SC'11; constants as in Random123 (multipliers 0xD2511F53, 0xCD9E8D57, Weyl key increments
 * 0x9E3779B9, 0xBB67AE85).  Pinned by the Random123 known-answer vectors in tests/golden/.
 * ---------------------------------------------------------------------------------------- */
void sd_ref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {            /* key schedule: bump between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* C-8: 24-bit uniform on the grid {0, 2^-24, ..., 1 - 2^-24}; exact in fp64. */
double sd_ref_u24(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }

void sd_ref_uniforms(uint64_t seed, uint32_t j, uint64_t round, uint64_t rid,
                     double* u_acc, double* u_smp) {
    uint32_t ctr[4] = {j, (uint32_t)round, (uint32_t)rid, (uint32_t)(rid >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    sd_ref_philox4x32_10(ctr, key, w);
    if (u_acc) *u_acc = sd_ref_u24(w[0]);
    if (u_smp) *u_smp = sd_ref_u24(w[1]);
}

/* ------------------------------------------------------------------------------------------
 * Row access: inputs are fp32 or bf16 logits; both widen exactly to fp64.
 * ---------------------------------------------------------------------------------------- */
static double logit_at(const void* base, int32_t dtype, int64_t idx) {
    if (dtype == 0) return (double)((const float*)base)[idx];
    uint32_t bits = (uint32_t)((const uint16_t*)base)[idx] << 16;   /* bf16 -> fp32 bit pattern */
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
}

typedef struct {
    const void* base;   /* start of the row */
    int32_t dtype;
    int32_t V;
} row_t;

static double z_of(row_t r, int32_t x) { return logit_at(r.base, r.dtype, x); }

/* C-12: NaN or +inf anywhere, or an all -inf row, is a fault. */
static int row_fault(row_t r) {
    int any_finite = 0;
    for (int32_t x = 0; x < r.V; ++x) {
        double z = z_of(r, x);
        if (isnan(z) || z == INFINITY) return SD_REF_FAULT_NONFINITE;
        if (z != -INFINITY) any_finite = 1;
    }
    return any_finite ? 0 : SD_REF_FAULT_EMPTY_ROW;
}

/* C-4: lambda = log sum_x exp(z(x)/T), computed as max, then sum of exp, then log (fp64). */
static double row_logsumexp(row_t r, double T) {
    double m = -INFINITY;
    for (int32_t x = 0; x < r.V; ++x) {
        double z = z_of(r, x);
        if (z > m) m = z;
    }
    double s = 0.0;
    for (int32_t x = 0; x < r.V; ++x) s += exp((z_of(r, x) - m) / T);
    return m / T + log(s);
}

/* softmax probability of token x: exp(z(x)/T - lambda) */
static double prob_of(row_t r, int32_t x, double T, double lam) {
    return exp(z_of(r, x) / T - lam);
}

/* C-5: lowest index achieving the maximum logit. */
static int32_t row_argmax(row_t r) {
    int32_t g = 0;
    double best = z_of(r, 0);
    for (int32_t x = 1; x < r.V; ++x) {
        double z = z_of(r, x);
        if (z > best) { best = z; g = x; }
    }
    return g;
}

/* ------------------------------------------------------------------------------------------
 * Sampling distribution at the stop position L (C-3, C-6, C-9):
 *   L < k : r(y) = max(0, p_L(y) - q_L(y)), R = sum r; if R == 0 fall back to r = p_L
 *   L = k : r(y) = p_k(y), R = sum p_k (computed, not assumed to be 1)
 * writes r into buf[V]; returns R and sets *zero_res when the C-6 fallback fired.
 * ---------------------------------------------------------------------------------------- */
static double sampling_dist(row_t pr, double lam_p, const row_t* qr, double lam_q, double T,
                            double* buf, int* zero_res) {
    double R = 0.0;
    *zero_res = 0;
    if (qr) {
        for (int32_t y = 0; y < pr.V; ++y) {
            double d = prob_of(pr, y, T, lam_p) - prob_of(*qr, y, T, lam_q);
            buf[y] = d > 0.0 ? d : 0.0;
            R += buf[y];
        }
        if (R > 0.0) return R;
        *zero_res = 1;
    }
    R = 0.0;
    for (int32_t y = 0; y < pr.V; ++y) {
        buf[y] = prob_of(pr, y, T, lam_p);
        R += buf[y];
    }
    return R;
}

/* C-9: t = smallest y with C(y) = sum_{y' <= y} r(y') > theta; if none (rounding), the largest
 * y with r(y) > 0.  Also reports C(t-1) and C(t). */
static int32_t inverse_cdf(const double* r, int32_t V, double theta, double* C_prev, double* C_tok) {
    double C = 0.0;
    for (int32_t y = 0; y < V; ++y) {
        double Cn = C + r[y];
        if (Cn > theta) {
            *C_prev = C;
            *C_tok = Cn;
            return y;
        }
        C = Cn;
    }
    int32_t t = V - 1;
    while (t > 0 && !(r[t] > 0.0)) --t;
    double Cp = 0.0;
    for (int32_t y = 0; y < t; ++y) Cp += r[y];
    *C_prev = Cp;
    *C_tok = Cp + r[t];
    return t;
}

/* ------------------------------------------------------------------------------------------
 * One request.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    const void* p; const void* q; const int32_t* ids;
    int32_t B, k, V; int64_t ld_p, ld_q; int32_t dtype;
    double T; uint64_t seed, round, rid_base;
    int32_t* out_L; int32_t* out_tokens; int32_t* out_status; sd_ref_trace* trace;
} batch_t;

static row_t p_row(const batch_t* a, int32_t b, int32_t j) {
    size_t esz = a->dtype == 0 ? 4 : 2;
    row_t r = {(const char*)a->p + ((size_t)b * (a->k + 1) + j) * a->ld_p * esz, a->dtype, a->V};
    return r;
}
static row_t q_row(const batch_t* a, int32_t b, int32_t j) {
    size_t esz = a->dtype == 0 ? 4 : 2;
    row_t r = {(const char*)a->q + ((size_t)b * a->k + j) * a->ld_q * esz, a->dtype, a->V};
    return r;
}

static void emit(const batch_t* a, int32_t b, int32_t L, int32_t t, int32_t status) {
    int32_t k = a->k;
    int32_t* tok = a->out_tokens + (size_t)b * (k + 1);
    int hard = (status & SD_REF_HARD_FAULTS) != 0;
    if (hard) L = 0;
    for (int32_t i = 0; i <= k; ++i) {
        if (hard) tok[i] = -1;
        else if (i < L) tok[i] = a->ids[(size_t)b * k + i];   /* accepted draft tokens */
        else if (i == L) tok[i] = t;                          /* correction or bonus         */
        else tok[i] = -1;
    }
    a->out_L[b] = L;
    if (a->out_status) a->out_status[b] = status;
}

static void verify_greedy_one(const batch_t* a, int32_t b, double* buf) {
    (void)buf;
    int32_t k = a->k, V = a->V, L = k, status = 0;
    sd_ref_trace* tr = a->trace ? &a->trace[b] : NULL;
    if (tr) { memset(tr, 0, sizeof *tr); tr->mu_a = 1.0; tr->mu_s = 1.0; }
    int32_t g = -1;
    for (int32_t j = 0; j < k; ++j) {
        int32_t x = a->ids[(size_t)b * k + j];
        if (x < 0 || x >= V) { status = SD_REF_FAULT_BAD_DRAFT_ID; break; }
        row_t pr = p_row(a, b, j);
        int f = row_fault(pr);
        if (f) { status = f; break; }
        g = row_argmax(pr);
        if (tr) tr->n_tested = j + 1;
        if (x != g) { L = j; break; }                         /* first mismatch */
    }
    if (!(status & SD_REF_HARD_FAULTS) && L == k) {
        row_t pr = p_row(a, b, k);
        int f = row_fault(pr);
        if (f) status = f;
        else g = row_argmax(pr);                              /* bonus = argmax p_k */
    }
    int32_t t = (status & SD_REF_HARD_FAULTS) ? -1 : g;
    if (tr) { tr->L = (status & SD_REF_HARD_FAULTS) ? 0 : L; tr->token = t; tr->status = status; }
    emit(a, b, L, t, status);
}

static void verify_sampled_one(const batch_t* a, int32_t b, double* buf) {
    int32_t k = a->k, V = a->V, L = k, status = 0;
    double T = a->T;
    uint64_t rid = a->rid_base + (uint64_t)b;
    sd_ref_trace* tr = a->trace ? &a->trace[b] : NULL;
    if (tr) { memset(tr, 0, sizeof *tr); tr->mu_a = 1.0; tr->mu_s = 1.0; }
    double lam_p = 0.0, lam_q = 0.0;
    int stopped = 0;
    /* Acceptance tests in chain order (P:729-731 with C-1, C-2). */
    for (int32_t j = 0; j < k; ++j) {
        int32_t x = a->ids[(size_t)b * k + j];
        if (x < 0 || x >= V) { status = SD_REF_FAULT_BAD_DRAFT_ID; stopped = 1; break; }
        row_t pr = p_row(a, b, j), qr = q_row(a, b, j);
        int f = row_fault(pr);
        if (!f) f = row_fault(qr);
        if (f) { status = f; stopped = 1; break; }
        lam_p = row_logsumexp(pr, T);
        lam_q = row_logsumexp(qr, T);
        double zp = z_of(pr, x), zq = z_of(qr, x);
        double u_acc;
        sd_ref_uniforms(a->seed, (uint32_t)j, a->round, rid, &u_acc, NULL);
        if (tr) {
            tr->n_tested = j + 1;
            tr->lam_p[j] = lam_p; tr->lam_q[j] = lam_q; tr->u_acc[j] = u_acc;
        }
        if (zq == -INFINITY) {                                 /* C-7: q_j(x_j) = 0 */
            status |= SD_REF_FAULT_ZERO_Q;
            if (tr) { tr->ell[j] = -INFINITY; tr->a[j] = 0.0; }
            L = j; stopped = 1; break;
        }
        double ell = (zp / T - lam_p) - (zq / T - lam_q);     /* log p_j(x_j) - log q_j(x_j) */
        double acc = ell >= 0.0 ? 1.0 : exp(ell);              /* min(1, p/q) */
        if (tr) {
            tr->ell[j] = ell; tr->a[j] = acc;
            if (ell < 0.0) {
                double mu = fabs(u_acc - acc);
                if (mu < tr->mu_a) tr->mu_a = mu;
            }
        }
        if (ell < 0.0 && u_acc >= acc) { L = j; stopped = 1; break; }   /* rejection */
    }
    (void)stopped;
    if (status & SD_REF_HARD_FAULTS) {
        if (tr) { tr->L = 0; tr->token = -1; tr->status = status; }
        emit(a, b, 0, -1, status);
        return;
    }
    /* Correction (L < k) or bonus (L == k) (C-3, C-6, C-9). */
    int zero_res = 0;
    double R;
    row_t pr = p_row(a, b, L);
    if (L < k) {
        row_t qr = q_row(a, b, L);
        R = sampling_dist(pr, lam_p, &qr, lam_q, T, buf, &zero_res);
    } else {
        int f = row_fault(pr);
        if (f) {
            status |= f;
            if (tr) { tr->L = 0; tr->token = -1; tr->status = status; }
            emit(a, b, 0, -1, status);
            return;
        }
        double lam_k = row_logsumexp(pr, T);
        if (tr) tr->lam_p[k] = lam_k;
        R = sampling_dist(pr, lam_k, NULL, 0.0, T, buf, &zero_res);
    }
    if (zero_res) status |= SD_REF_FAULT_ZERO_RESIDUAL;
    double u_smp;
    sd_ref_uniforms(a->seed, (uint32_t)L, a->round, rid, NULL, &u_smp);
    double theta = u_smp * R;
    double Cp, Ct;
    int32_t t = inverse_cdf(buf, V, theta, &Cp, &Ct);
    if (tr) {
        tr->L = L; tr->token = t; tr->status = status;
        tr->R = R; tr->u_smp = u_smp; tr->theta = theta; tr->C_prev = Cp; tr->C_tok = Ct;
        double m1 = theta - Cp, m2 = Ct - theta;
        tr->mu_s = (m1 < m2 ? m1 : m2) / R;
    }
    emit(a, b, L, t, status);
}

typedef struct { const batch_t* a; int32_t b0, b1; } span_t;

static void* run_span(void* arg) {
    span_t* s = (span_t*)arg;
    double* buf = (double*)malloc(sizeof(double) * (size_t)s->a->V);
    for (int32_t b = s->b0; b < s->b1; ++b) {
        if (s->a->T == 0.0) verify_greedy_one(s->a, b, buf);
        else verify_sampled_one(s->a, b, buf);
    }
    free(buf);
    return NULL;
}

int sd_ref_verify(const void* p, const void* q, const int32_t* ids,
                  int32_t B, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                  double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                  int32_t* out_L, int32_t* out_tokens, int32_t* out_status,
                  sd_ref_trace* trace, int32_t n_threads) {
    if (!p || !ids || !out_L || !out_tokens || B < 0 || k < 1 || k > SD_REF_KMAX || V < 2 ||
        (dtype != 0 && dtype != 1) || !(T >= 0.0) || isinf(T) || (T > 0.0 && !q))
        return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    if (ld_p < V || ld_q < V) return 1;
    batch_t a = {p, q, ids, B, k, V, ld_p, ld_q, dtype, T, seed, round, rid_base,
                 out_L, out_tokens, out_status, trace};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > B) n_threads = B > 0 ? B : 1;
    if (n_threads == 1) {
        span_t s = {&a, 0, B};
        run_span(&s);
        return 0;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    span_t* sp = (span_t*)malloc(sizeof(span_t) * (size_t)n_threads);
    for (int32_t i = 0; i < n_threads; ++i) {
        sp[i].a = &a;
        sp[i].b0 = (int32_t)((int64_t)B * i / n_threads);
        sp[i].b1 = (int32_t)((int64_t)B * (i + 1) / n_threads);
        pthread_create(&th[i], NULL, run_span, &sp[i]);
    }
    for (int32_t i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
    free(sp);
    return 0;
}

int sd_ref_sample_check(const void* p, const void* q, const int32_t* ids,
                        int32_t b, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        int32_t L, int32_t t, double* C_prev, double* C_tok, double* R, double* theta) {
    if (!p || !q || L < 0 || L > k || t < 0 || t >= V || !(T > 0.0)) return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    batch_t a = {p, q, ids, b + 1, k, V, ld_p, ld_q, dtype, T, seed, round, rid_base,
                 NULL, NULL, NULL, NULL};
    double* buf = (double*)malloc(sizeof(double) * (size_t)V);
    row_t pr = p_row(&a, b, L);
    double lam_p = row_logsumexp(pr, T);
    int zero_res;
    double Rv;
    if (L < k) {
        row_t qr = q_row(&a, b, L);
        Rv = sampling_dist(pr, lam_p, &qr, row_logsumexp(qr, T), T, buf, &zero_res);
    } else {
        Rv = sampling_dist(pr, lam_p, NULL, 0.0, T, buf, &zero_res);
    }
    double u_smp;
    sd_ref_uniforms(seed, (uint32_t)L, round, rid_base + (uint64_t)b, NULL, &u_smp);
    double C = 0.0;
    for (int32_t y = 0; y < t; ++y) C += buf[y];
    *C_prev = C;
    *C_tok = C + buf[t];
    *R = Rv;
    *theta = u_smp * Rv;
    free(buf);
    return 0;
}

int sd_ref_accept_probs(const void* p, const void* q, const int32_t* ids,
                        int32_t b, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        double* a_out, double* u_out) {
    if (!p || !q || !ids || !(T > 0.0) || k < 1 || k > SD_REF_KMAX) return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    batch_t a = {p, q, ids, b + 1, k, V, ld_p, ld_q, dtype, T, seed, round, rid_base,
                 NULL, NULL, NULL, NULL};
    for (int32_t j = 0; j < k; ++j) {
        int32_t x = ids[(size_t)b * k + j];
        row_t pr = p_row(&a, b, j), qr = q_row(&a, b, j);
        double lam_p = row_logsumexp(pr, T), lam_q = row_logsumexp(qr, T);
        double zq = z_of(qr, x);
        if (zq == -INFINITY) a_out[j] = 0.0;
        else {
            double ell = (z_of(pr, x) / T - lam_p) - (zq / T - lam_q);
            a_out[j] = ell >= 0.0 ? 1.0 : exp(ell);
        }
        sd_ref_uniforms(seed, (uint32_t)j, round, rid_base + (uint64_t)b, &u_out[j], NULL);
    }
    return 0;
}

/* Exact distribution of (L, emitted token) for fixed draft paths, with the continuous
 * uniforms of P:730 integrated out:
 *   Pr(L = j, t = y) = (prod_{i<j} a_i) (1 - a_j) r_j(y) / R_j      (j < k)
 *   Pr(L = k, t = y) = (prod_{i<k} a_i) p_k(y)                       (bonus, C-3)
 * Greedy (T == 0) is deterministic: a point mass at the oracle's (L, t). */
int sd_ref_outcome_dist(const void* p, const void* q, const int32_t* ids,
                        int32_t B, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, double* out) {
    if (!p || !ids || !out || k < 1 || k > SD_REF_KMAX || V < 2 || !(T >= 0.0)) return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    memset(out, 0, sizeof(double) * (size_t)B * (k + 1) * V);
    batch_t a = {p, q, ids, B, k, V, ld_p, ld_q, dtype, T, 0, 0, 0, NULL, NULL, NULL, NULL};
    double* buf = (double*)malloc(sizeof(double) * (size_t)V);
    for (int32_t b = 0; b < B; ++b) {
        double* ob = out + (size_t)b * (k + 1) * V;
        if (T == 0.0) {
            int32_t L, tok, st;
            int32_t* tk = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k + 1));
            batch_t g = a;
            g.ids = ids + (size_t)b * k;
            g.p = (const char*)p + (size_t)b * (k + 1) * ld_p * (dtype == 0 ? 4 : 2);
            g.B = 1; g.out_L = &L; g.out_tokens = tk; g.out_status = &st;
            verify_greedy_one(&g, 0, buf);
            tok = tk[L];
            if (tok >= 0) ob[(size_t)L * V + tok] = 1.0;
            free(tk);
            continue;
        }
        double reach = 1.0;
        for (int32_t j = 0; j < k; ++j) {
            int32_t x = ids[(size_t)b * k + j];
            row_t pr = p_row(&a, b, j), qr = q_row(&a, b, j);
            double lam_p = row_logsumexp(pr, T), lam_q = row_logsumexp(qr, T);
            double zq = z_of(qr, x), acc;
            if (zq == -INFINITY) acc = 0.0;
            else {
                double ell = (z_of(pr, x) / T - lam_p) - (zq / T - lam_q);
                acc = ell >= 0.0 ? 1.0 : exp(ell);
            }
            if (acc < 1.0) {
                int zr;
                double R = sampling_dist(pr, lam_p, &qr, lam_q, T, buf, &zr);
                for (int32_t y = 0; y < V; ++y) ob[(size_t)j * V + y] = reach * (1.0 - acc) * buf[y] / R;
            }
            reach *= acc;
        }
        row_t pk = p_row(&a, b, k);
        double lam_k = row_logsumexp(pk, T);
        for (int32_t y = 0; y < V; ++y) ob[(size_t)k * V + y] = reach * prob_of(pk, y, T, lam_k);
    }
    free(buf);
    return 0;
}

/* Eq. (1): beta = sum_x min{p(x), q(x)}. */
double sd_ref_beta(const float* zp, const float* zq, int32_t V, double T) {
    row_t pr = {zp, 0, V}, qr = {zq, 0, V};
    double lp = row_logsumexp(pr, T), lq = row_logsumexp(qr, T), s = 0.0;
    for (int32_t x = 0; x < V; ++x) {
        double a = prob_of(pr, x, T, lp), b = prob_of(qr, x, T, lq);
        s += a < b ? a : b;
    }
    return s;
}

void sd_ref_softmax(const float* z, int32_t V, double T, double* out) {
    row_t r = {z, 0, V};
    double l = row_logsumexp(r, T);
    for (int32_t x = 0; x < V; ++x) out[x] = prob_of(r, x, T, l);
}

/* ------------------------------------------------------------------------------------------
 * Draft-side sampler: the step before the verify path.  PAPER.md Alg. 2
 * ExpandLayer draws the draft tokens from M_q, and "the draft probabilities q_t(.) needed
 * by the correction step are stored in the tree metadata".  Chain form, per request b and
 * position j (reading D-1 of DESIGN.md):
 *   q_j = softmax(z_q,j / T);  x_j = the smallest token y (ascending id) with C(y) > theta,
 *   C(y) = sum_{y' <= y} q_j(y'),  theta = u * sum_y q_j(y),  u = u24(w1) of Philox4x32-10 with
 *   key = seed and counter (0, round, rid_d lo, rid_d hi), rid_d = 2^63 + (rid_base + b) k + j
 *   (a counter domain disjoint from the verify step's, whose request ids stay below 2^63);
 *   clamp to the last positive-mass token as in C-9.  T == 0: x_j = argmax (lowest index, C-5).
 * out_logq[b][j] = log q_j(x_j) = z(x_j)/T - lambda_j (0 at T == 0); out_mu[b][j] (nullable) =
 * min(theta - C(x-1), C(x) - theta) / sum q: the CDF-cell margin (tie rule).  Rows with NaN / +inf
 * or no finite logit are faults (C-12): id -1, status bit set.
 * ---------------------------------------------------------------------------------------- */
int sd_ref_draft_sample(const void* q, int32_t B, int32_t k, int32_t V, int64_t ld_q,
                        int32_t dtype, double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        int32_t* out_ids, double* out_logq, double* out_mu, int32_t* out_status) {
    if (!q || !out_ids || B < 0 || k < 1 || V < 2 || (dtype != 0 && dtype != 1) || !(T >= 0.0) ||
        isinf(T))
        return 1;
    if (ld_q == 0) ld_q = V;
    if (ld_q < V) return 1;
    size_t esz = dtype == 0 ? 4 : 2;
    double* buf = (double*)malloc(sizeof(double) * (size_t)V);
    for (int32_t b = 0; b < B; ++b)
        for (int32_t j = 0; j < k; ++j) {
            size_t r = (size_t)b * k + j;
            row_t qr = {(const char*)q + r * ld_q * esz, dtype, V};
            int f = row_fault(qr);
            if (out_status) out_status[r] = f;
            if (out_mu) out_mu[r] = 1.0;
            if (f) {
                out_ids[r] = -1;
                if (out_logq) out_logq[r] = 0.0;
                continue;
            }
            if (T == 0.0) {
                out_ids[r] = row_argmax(qr);
                if (out_logq) out_logq[r] = 0.0;
                continue;
            }
            double lam = row_logsumexp(qr, T);
            int zr;
            double S = sampling_dist(qr, lam, NULL, 0.0, T, buf, &zr);
            uint64_t rid = ((uint64_t)1 << 63) + (rid_base + (uint64_t)b) * (uint64_t)k + (uint64_t)j;
            double u;
            sd_ref_uniforms(seed, 0u, round, rid, NULL, &u);
            double theta = u * S, Cp, Ct;
            int32_t x = inverse_cdf(buf, V, theta, &Cp, &Ct);
            out_ids[r] = x;
            if (out_logq) out_logq[r] = z_of(qr, x) / T - lam;
            if (out_mu) {
                double m1 = theta - Cp, m2 = Ct - theta;
                out_mu[r] = (m1 < m2 ? m1 : m2) / S;
            }
        }
    free(buf);
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * Lossless tree verification.  The paper drafts a depth-d tree with
 * branching factor k (Alg. 2) and verifies its k^d paths independently,
 * keeping the longest accepted one -- a rule that is not lossless (SPEC S:176,
 * SURVEY C-14).  The replacement (reading D-2 of DESIGN.md) is recursive rejection sampling over
 * the children of each node (SpecInfer's multi-candidate speculative sampling, the paper's ref.
 * [miao2024specinfer]): the children c_1..c_m of a node are i.i.d. draws from the node's
 * draft distribution q; with d_0 = p (the node's target distribution):
 *   for i = 1..m: accept c_i iff u_i < min(1, d_{i-1}(x_i) / q(x_i)) (x_i = token of c_i) ->
 *                 descend into c_i;
 *                 else d_i = norm(max(0, d_{i-1} - q))   (the residual of P:736, applied again)
 *   all m rejected: emit t ~ d_m and stop;  a leaf reached (depth d): emit the bonus t ~ p_leaf.
 * m = 1 is exactly the chain of sd_ref_verify (same counters).  Layout: a full m-ary tree of
 * depth d per request, level order: node 0 = root, children of n are m n + 1 .. m n + m;
 * N = sum_{t<=d} m^t nodes, N_int = sum_{t<d} m^t internal ones.
 *   p: [B][N][ld_p] target logits at every node; q: [B][N_int][ld_q] draft logits at internal
 *   nodes; tok: [B][N] int32 token of each node (root entry unused).
 * Uniforms (C-8 counters, key = seed): candidate i (0-based) at depth t: u_acc = u24(w0) of
 * counter (t + 32 i, round, rid); the final sample at depth t: u_smp = u24(w1) of (t, round, rid).
 * Outputs: out_L[b] = depth reached (accepted tokens), out_tokens[b][0..d] = the accepted path's
 * tokens, then the emitted token, then -1; out_node[b] (nullable) = the node the walk stopped at;
 * out_mu[b] (nullable) = the smallest decision margin (|u - a| over the tests decided with a
 * uniform, and the CDF-cell margin of the final sample relative to its mass), for the tie rule.
 * T == 0: greedy -- descend into the first child whose token is argmax p_node, else emit argmax.
 * Hard faults (C-12) on a reached row: L = 0, tokens -1, status bit set.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    const void* p; const void* q; const int32_t* tok;
    int32_t m, d, V, N, Nint; int64_t ld_p, ld_q; int32_t dtype; double T;
    uint64_t seed, round, rid_base;
} tree_t;

static row_t tree_p(const tree_t* a, int32_t b, int32_t n) {
    size_t esz = a->dtype == 0 ? 4 : 2;
    row_t r = {(const char*)a->p + ((size_t)b * a->N + n) * a->ld_p * esz, a->dtype, a->V};
    return r;
}
static row_t tree_q(const tree_t* a, int32_t b, int32_t n) {
    size_t esz = a->dtype == 0 ? 4 : 2;
    row_t r = {(const char*)a->q + ((size_t)b * a->Nint + n) * a->ld_q * esz, a->dtype, a->V};
    return r;
}

/* d_i of the node into buf (normalised), from d_{i-1} in buf and q (probabilities in qb):
 * returns the mass R_i = sum max(0, d_{i-1} - q) before normalising (0: keep d_{i-1}, C-6). */
static double residual_step(double* buf, const double* qb, int32_t V) {
    double R = 0.0;
    for (int32_t y = 0; y < V; ++y) {
        double dd = buf[y] - qb[y];
        R += dd > 0.0 ? dd : 0.0;
    }
    if (!(R > 0.0)) return 0.0;
    for (int32_t y = 0; y < V; ++y) {
        double dd = buf[y] - qb[y];
        buf[y] = (dd > 0.0 ? dd : 0.0) / R;
    }
    return R;
}

static int tree_one(const tree_t* a, int32_t b, int32_t* out_L, int32_t* tokens, int32_t* node_out,
                    double* mu_out, double* pb, double* qb, double* outc) {
    const int32_t m = a->m, d = a->d, V = a->V;
    uint64_t rid = a->rid_base + (uint64_t)b;
    double mu = 1.0;
    int32_t n = 0, depth = 0, status = 0;
    for (int32_t i = 0; i <= d; ++i) tokens[i] = -1;
    while (1) {
        row_t pr = tree_p(a, b, n);
        int f = row_fault(pr);
        if (f) { status = f; break; }
        if (depth == d) {                                   /* leaf: bonus t ~ p_leaf (C-3) */
            if (a->T == 0.0) { tokens[depth] = row_argmax(pr); break; }
            double lam = row_logsumexp(pr, a->T), R = 0.0;
            for (int32_t y = 0; y < V; ++y) { pb[y] = prob_of(pr, y, a->T, lam); R += pb[y]; }
            double us, Cp, Ct;
            sd_ref_uniforms(a->seed, (uint32_t)depth, a->round, rid, NULL, &us);
            double th = us * R;
            tokens[depth] = inverse_cdf(pb, V, th, &Cp, &Ct);
            double m1 = th - Cp, m2 = Ct - th, ms = (m1 < m2 ? m1 : m2) / R;
            if (ms < mu) mu = ms;
            break;
        }
        if (a->T == 0.0) {                                  /* greedy tree */
            int32_t g = row_argmax(pr), next = -1;
            for (int32_t i = 0; i < m; ++i) {
                int32_t c = m * n + 1 + i, x = a->tok[(size_t)b * a->N + c];
                if (x < 0 || x >= V) { status = SD_REF_FAULT_BAD_DRAFT_ID; break; }
                if (x == g) { next = c; break; }
            }
            if (status) break;
            if (next < 0) { tokens[depth] = g; break; }
            tokens[depth] = g;
            n = next;
            ++depth;
            continue;
        }
        row_t qr = tree_q(a, b, n);
        f = row_fault(qr);
        if (f) { status = f; break; }
        double lp = row_logsumexp(pr, a->T), lq = row_logsumexp(qr, a->T);
        for (int32_t y = 0; y < V; ++y) { pb[y] = prob_of(pr, y, a->T, lp); qb[y] = prob_of(qr, y, a->T, lq); }
        int32_t next = -1;
        for (int32_t i = 0; i < m; ++i) {
            int32_t c = m * n + 1 + i, x = a->tok[(size_t)b * a->N + c];
            if (x < 0 || x >= V) { status = SD_REF_FAULT_BAD_DRAFT_ID; break; }
            if (i > 0 && residual_step(pb, qb, V) == 0.0) status |= SD_REF_FAULT_ZERO_RESIDUAL;
            double u, acc;
            if (z_of(qr, x) == -INFINITY) {                  /* C-7: q(x) = 0 rejects */
                acc = 0.0;
                status |= SD_REF_FAULT_ZERO_Q;
            } else if (!(qb[x] > 0.0)) {
                acc = pb[x] > 0.0 ? 1.0 : 0.0;               /* (underflowed q: the limit) */
            } else {
                acc = pb[x] >= qb[x] ? 1.0 : pb[x] / qb[x];
            }
            sd_ref_uniforms(a->seed, (uint32_t)(depth + 32 * i), a->round, rid, &u, NULL);
            if (acc < 1.0) {
                double mm = fabs(u - acc);
                if (mm < mu) mu = mm;
                if (u >= acc) continue;                     /* reject: next candidate */
            }
            next = c;
            break;
        }
        if (status & SD_REF_HARD_FAULTS) break;
        if (next >= 0) {
            tokens[depth] = a->tok[(size_t)b * a->N + next];
            n = next;
            ++depth;
            continue;
        }
        /* every candidate rejected: t ~ d_m */
        if (residual_step(pb, qb, V) == 0.0) status |= SD_REF_FAULT_ZERO_RESIDUAL;
        double R = 0.0;
        for (int32_t y = 0; y < V; ++y) R += pb[y];
        double us, Cp, Ct;
        sd_ref_uniforms(a->seed, (uint32_t)depth, a->round, rid, NULL, &us);
        double th = us * R;
        tokens[depth] = inverse_cdf(pb, V, th, &Cp, &Ct);
        double m1 = th - Cp, m2 = Ct - th, ms = (m1 < m2 ? m1 : m2) / R;
        if (ms < mu) mu = ms;
        break;
    }
    (void)outc;
    if (status & SD_REF_HARD_FAULTS) {
        for (int32_t i = 0; i <= d; ++i) tokens[i] = -1;
        depth = 0;
    }
    *out_L = depth;
    if (node_out) *node_out = n;
    if (mu_out) *mu_out = mu;
    return status;
}

int sd_ref_tree_verify(const void* p, const void* q, const int32_t* tok, int32_t B, int32_t m,
                       int32_t d, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype, double T,
                       uint64_t seed, uint64_t round, uint64_t rid_base, int32_t* out_L,
                       int32_t* out_tokens, int32_t* out_status, int32_t* out_node,
                       double* out_mu) {
    if (!p || !tok || !out_L || !out_tokens || B < 0 || m < 1 || m > 8 || d < 1 || d > SD_REF_KMAX ||
        V < 2 || (dtype != 0 && dtype != 1) || !(T >= 0.0) || isinf(T) || (T > 0.0 && !q))
        return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    int64_t N = 0, Nint = 0, w = 1;
    for (int32_t t = 0; t <= d; ++t) { N += w; if (t < d) Nint += w; w *= m; if (N > (1 << 24)) return 1; }
    tree_t a = {p, q, tok, m, d, V, (int32_t)N, (int32_t)Nint, ld_p, ld_q, dtype, T, seed, round, rid_base};
    double* pb = (double*)malloc(sizeof(double) * (size_t)V);
    double* qb = (double*)malloc(sizeof(double) * (size_t)V);
    for (int32_t b = 0; b < B; ++b) {
        int st = tree_one(&a, b, &out_L[b], out_tokens + (size_t)b * (d + 1),
                          out_node ? &out_node[b] : NULL, out_mu ? &out_mu[b] : NULL, pb, qb, NULL);
        if (out_status) out_status[b] = st;
    }
    free(pb);
    free(qb);
    return 0;
}

/* Exact outcome distribution of one tree verify with the uniforms integrated out:
 * out[b][n][y] = Pr(the walk stops at node n and emits token y), fixed tree (T > 0). */
int sd_ref_tree_outcome_dist(const void* p, const void* q, const int32_t* tok, int32_t B,
                             int32_t m, int32_t d, int32_t V, int64_t ld_p, int64_t ld_q,
                             int32_t dtype, double T, double* out) {
    if (!p || !q || !tok || !out || m < 1 || d < 1 || V < 2 || !(T > 0.0)) return 1;
    if (ld_p == 0) ld_p = V;
    if (ld_q == 0) ld_q = V;
    int64_t N = 0, Nint = 0, w = 1;
    for (int32_t t = 0; t <= d; ++t) { N += w; if (t < d) Nint += w; w *= m; if (N > (1 << 20)) return 1; }
    tree_t a = {p, q, tok, m, d, V, (int32_t)N, (int32_t)Nint, ld_p, ld_q, dtype, T, 0, 0, 0};
    memset(out, 0, sizeof(double) * (size_t)B * N * V);
    double* pb = (double*)malloc(sizeof(double) * (size_t)V);
    double* qb = (double*)malloc(sizeof(double) * (size_t)V);
    double* reach = (double*)malloc(sizeof(double) * (size_t)N);
    int32_t* depth_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
    for (int32_t b = 0; b < B; ++b) {
        double* ob = out + (size_t)b * N * V;
        for (int64_t n = 0; n < N; ++n) reach[n] = 0.0;
        reach[0] = 1.0;
        depth_of[0] = 0;
        for (int64_t n = 0; n < N; ++n) {                   /* level order: parents first */
            if (n > 0) depth_of[n] = depth_of[(n - 1) / m] + 1;
            if (reach[n] == 0.0) continue;
            row_t pr = tree_p(&a, b, (int32_t)n);
            double lp = row_logsumexp(pr, T);
            for (int32_t y = 0; y < V; ++y) pb[y] = prob_of(pr, y, T, lp);
            if (depth_of[n] == d) {                         /* leaf: bonus */
                for (int32_t y = 0; y < V; ++y) ob[(size_t)n * V + y] += reach[n] * pb[y];
                continue;
            }
            row_t qr = tree_q(&a, b, (int32_t)n);
            double lq = row_logsumexp(qr, T);
            for (int32_t y = 0; y < V; ++y) qb[y] = prob_of(qr, y, T, lq);
            double stay = reach[n];                         /* Pr(at n, all earlier candidates rejected) */
            for (int32_t i = 0; i < m; ++i) {
                int32_t c = (int32_t)(m * n + 1 + i), x = tok[(size_t)b * N + c];
                if (i > 0) residual_step(pb, qb, V);
                double acc = qb[x] > 0.0 ? (pb[x] >= qb[x] ? 1.0 : pb[x] / qb[x]) : 0.0;
                reach[c] += stay * acc;
                stay *= 1.0 - acc;
            }
            residual_step(pb, qb, V);
            for (int32_t y = 0; y < V; ++y) ob[(size_t)n * V + y] += stay * pb[y];
        }
    }
    free(pb); free(qb); free(reach); free(depth_of);
    return 0;
}
