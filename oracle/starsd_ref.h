/*
 * starsd_ref.h -- CPU ORACLE for the StarSD speculative-sampling verify step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or link this.
 * The product path (paper_2601_21622_b200/, include/starsd.h) never does, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Everything is plain C99 in fp64 on host pointers.  Citations are to
 * /root/reference/PAPER.md lines ("P:nnn") and to the readings C-1..C-17 of
 * SURVEY.md section 8(c), which DESIGN.md lists.
 */
#ifndef STARSD_REF_H
#define STARSD_REF_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SD_REF_KMAX 31

/* same numeric values as the product's status / fault codes (restated, not shared) */
#define SD_REF_FAULT_BAD_DRAFT_ID   1
#define SD_REF_FAULT_NONFINITE      2
#define SD_REF_FAULT_EMPTY_ROW      4
#define SD_REF_FAULT_ZERO_Q         8   /* informational: q_j(x_j)=0 -> rejection (C-7) */
#define SD_REF_FAULT_ZERO_RESIDUAL 16   /* informational: R==0 -> sample from p_L (C-6) */
#define SD_REF_HARD_FAULTS (SD_REF_FAULT_BAD_DRAFT_ID | SD_REF_FAULT_NONFINITE | SD_REF_FAULT_EMPTY_ROW)

/* Per-request record of every fp64 quantity the oracle decided on (parity rule C-13). */
typedef struct {
    int32_t L;            /* accept length l, 0..k                               */
    int32_t token;        /* correction (L<k) or bonus (L==k) token; -1 on a hard fault  */
    int32_t status;       /* fault bitmask                                                */
    int32_t n_tested;     /* number of positions j whose acceptance test was evaluated    */
    double lam_p[SD_REF_KMAX + 1]; /* logsumexp_x z_p,j(x)/T, j = 0..n_tested(-1 or L)    */
    double lam_q[SD_REF_KMAX];     /* logsumexp_x z_q,j(x)/T                              */
    double ell[SD_REF_KMAX];       /* log p_j(x_j) - log q_j(x_j)                          */
    double a[SD_REF_KMAX];         /* min(1, p_j(x_j)/q_j(x_j))                            */
    double u_acc[SD_REF_KMAX];     /* r_{j+1} of P:730 on the 2^-24 grid                   */
    double R;             /* mass of the sampling distribution (residual, or sum p_k)     */
    double u_smp;         /* sampling uniform                                             */
    double theta;         /* u_smp * R                                                    */
    double C_prev;        /* C(t-1): inclusive prefix mass before the emitted token       */
    double C_tok;         /* C(t)                                                         */
    double mu_a;          /* min_j |u_acc(j) - a_j| over tested j with ell<0 (1 if none)  */
    double mu_s;          /* min(theta - C(t-1), C(t) - theta) / R                        */
} sd_ref_trace;

/* Philox4x32-10 (Salmon et al. 2011, Random123), restated. */
void sd_ref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* u24(w) = (w >> 8) * 2^-24   (C-8) */
double sd_ref_u24(uint32_t w);
/* the two uniforms of position j for one request: u_acc = u24(w0), u_smp = u24(w1) (C-8) */
void sd_ref_uniforms(uint64_t seed, uint32_t j, uint64_t round, uint64_t rid,
                     double* u_acc, double* u_smp);

/* Lazy, step-by-step verify of a batch (P:727-742 with readings C-1..C-12).
 *   p: [B][k+1][ld_p], q: [B][k][ld_q] (may be NULL iff T == 0), dtype 0 = fp32, 1 = bf16 (raw u16)
 *   ids: [B][k] int32.  T == 0 -> greedy (C-5).
 *   out_L: [B], out_tokens: [B][k+1] (-1 padded), out_status: [B] (nullable), trace: [B] (nullable)
 *   n_threads: requests are independent and are split across this many threads (>=1).
 * Returns 0, or 1 on an invalid argument. */
int sd_ref_verify(const void* p, const void* q, const int32_t* ids,
                  int32_t B, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                  double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                  int32_t* out_L, int32_t* out_tokens, int32_t* out_status,
                  sd_ref_trace* trace, int32_t n_threads);

/* For a FORCED accept length L of request b (0<=L<=k), the fp64 sampling distribution the
 * algorithm would use there (residual at L<k, p_k at L==k; C-6 fallback) and its CDF at
 * token t: C(t-1), C(t), R and theta = u_smp(L)*R.  Used by the C-13 tie check. */
int sd_ref_sample_check(const void* p, const void* q, const int32_t* ids,
                        int32_t b, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        int32_t L, int32_t t, double* C_prev, double* C_tok, double* R, double* theta);

/* a_j = min(1, p_j(x_j)/q_j(x_j)) and u_acc(j) at EVERY position j = 0..k-1 of request b
 * (no early stop; rows assumed fault-free).  Used by the C-13 tie rule when a GPU result
 * stops at a different position than the oracle. */
int sd_ref_accept_probs(const void* p, const void* q, const int32_t* ids,
                        int32_t b, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        double* a_out, double* u_out);

/* Exact outcome distribution of one verify call, integrating the uniforms analytically
 * (continuous U(0,1) of P:730):  out[b][j][y] = Pr(L = j, emitted token = y | draft path).
 * Shape [B][k+1][V], fp64.  Used by the exact-enumeration losslessness pins. */
int sd_ref_outcome_dist(const void* p, const void* q, const int32_t* ids,
                        int32_t B, int32_t k, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype,
                        double T, double* out);

/* Draft-side sampler (NEXT-2): x_j ~ softmax(z_q,j / T) by inverse CDF on the
 * Philox counter (0, round, 2^63 + (rid_base + b) k + j), word w1; T == 0 -> argmax.  See the .c
 * file for the exact definition.  out_logq / out_mu / out_status are nullable. */
int sd_ref_draft_sample(const void* q, int32_t B, int32_t k, int32_t V, int64_t ld_q,
                        int32_t dtype, double T, uint64_t seed, uint64_t round, uint64_t rid_base,
                        int32_t* out_ids, double* out_logq, double* out_mu, int32_t* out_status);

/* Lossless tree verification (NEXT-3, reading D-2): recursive rejection sampling over the m
 * i.i.d. children of each node of a full m-ary depth-d tree (level order).  See the .c file. */
int sd_ref_tree_verify(const void* p, const void* q, const int32_t* tok, int32_t B, int32_t m,
                       int32_t d, int32_t V, int64_t ld_p, int64_t ld_q, int32_t dtype, double T,
                       uint64_t seed, uint64_t round, uint64_t rid_base, int32_t* out_L,
                       int32_t* out_tokens, int32_t* out_status, int32_t* out_node,
                       double* out_mu);
/* Exact Pr(stop at node n, emit y) of one tree verify, uniforms integrated out (T > 0). */
int sd_ref_tree_outcome_dist(const void* p, const void* q, const int32_t* tok, int32_t B,
                             int32_t m, int32_t d, int32_t V, int64_t ld_p, int64_t ld_q,
                             int32_t dtype, double T, double* out);

/* Eq. (1): beta = sum_x min{p(x), q(x)} for p = softmax(zp/T), q = softmax(zq/T) (fp32 logits). */
double sd_ref_beta(const float* zp, const float* zq, int32_t V, double T);
/* softmax at temperature T of one fp32 logit row, fp64 out. */
void sd_ref_softmax(const float* z, int32_t V, double T, double* out);

#ifdef __cplusplus
}
#endif
#endif
