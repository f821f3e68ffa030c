/*
 * starsd.h -- C ABI of the B200-native StarSD verify path (libstarsd.so).
 *
 * StarSD (arXiv 2601.21622) serves N target instances from one draft instance (PAPER.md
 * Alg. 1).  Every target ("verifier") runs, each round, the speculative-sampling
 * verify step of Alg. 2 on a chain of k draft tokens per request.  This header is
 * the boundary of that hot path:
 *
 *   sd_verify                 the batched verify step on one GPU                 (a1-a10)
 *   sd_verify_workspace_size  scratch it needs
 *   sd_star_*                 1 draft -> N verifier exchange + round scheduler  (a11-a12)
 *   sd_philox_uniforms        the counter-based uniforms the verify step draws  (a4)
 *
 * Conventions
 *   - Plain C: no C++ types or exceptions cross this boundary.  All functions return sd_status.
 *   - Device pointers are caller-owned CUDA device memory (e.g. torch tensors on the current
 *     device).  The library never allocates on the hot path; sd_star_create allocates its
 *     staging slots and communicators once.
 *   - Calls are asynchronous and stream-ordered on the cudaStream_t argument (0 = legacy
 *     default stream).  Results are valid once the stream reaches the call.
 *   - Host-checkable problems return SD_ERR_INVALID_ARGUMENT synchronously and launch nothing;
 *     sd_last_error() then names the offending argument.
 *
 * Symbols follow the paper: p = target distributions, q = draft distributions, k = the chain
 * length (the paper's depth d), L = accept length (the paper's l).
 */
#ifndef STARSD_H
#define STARSD_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SD_OK = 0,
    SD_ERR_INVALID_ARGUMENT = 1,  /* host-checkable argument error, nothing launched          */
    SD_ERR_UNSUPPORTED = 2,       /* valid request this build cannot serve                    */
    SD_ERR_CUDA = 3,              /* a CUDA runtime call or kernel launch failed              */
    SD_ERR_NCCL = 4,              /* an NCCL call failed or the communicator reported an error */
    SD_ERR_TIMEOUT = 5,           /* sd_star_poll: nothing completed within the timeout        */
    SD_ERR_NOT_READY = 6,         /* sd_star_poll with timeout 0: nothing completed yet        */
    SD_ERR_INTERNAL = 7
} sd_status;

typedef enum { SD_DTYPE_F32 = 0, SD_DTYPE_BF16 = 1 } sd_dtype;

/* Per-request fault bits written to out_status (reading C-12 of DESIGN.md).
 * Hard faults force L = 0 and all tokens = -1; the call still returns SD_OK.
 * Faults are only detected on rows the method actually reaches (positions <= L): the step is
 * lazy (P:731 stops at the first failed test), so a bad row after the first rejection is not
 * an error. */
enum {
    SD_FAULT_BAD_DRAFT_ID = 1,     /* hard: draft id outside [0, V)                          */
    SD_FAULT_NONFINITE = 2,        /* hard: NaN or +inf logit in a reached row               */
    SD_FAULT_EMPTY_ROW = 4,        /* hard: reached row is all -inf                           */
    SD_FAULT_ZERO_Q = 8,           /* info: q_j(x_j) = 0, treated as a rejection at j (C-7)   */
    SD_FAULT_ZERO_RESIDUAL = 16,   /* info: residual mass R == 0, sampled from p_L (C-6)      */
    SD_FAULT_PROTOCOL = 32         /* hard: an internal wait of the kernels gave up (200 ms):
                                      the workspace was used concurrently or corrupted; the
                                      request's result is void (never set in a correct run)     */
};

#define SD_MAX_K 31

typedef struct {
    int32_t batch;    /* B >= 0 requests                                              */
    int32_t k;        /* 1 <= k <= 31 draft tokens per request (chain depth d) */
    int32_t vocab;    /* V >= 2                                                        */
    int64_t ld_p;     /* row stride of p_logits in elements; 0 => V; >= V              */
    int64_t ld_q;     /* row stride of q_logits in elements; 0 => V; >= V              */
    sd_dtype dtype;   /* element type of both p_logits and q_logits                    */
} sd_shape;

/*
 * sd_verify -- one batched speculative-sampling verify step (Alg. 2, P:727-742;
 * Leviathan et al.'s ratio rule, cited at P:33 and P:121; readings C-1..C-12 in DESIGN.md).
 *
 * For each request b (independently; the batch is data-parallel):
 *   p_j = softmax(p_logits[b][j] / T), j = 0..k        (target rows; p_{j+1} of P:727)
 *   q_j = softmax(q_logits[b][j] / T), j = 0..k-1      (draft rows;  q_{j+1} of P:679)
 *   x_j = draft_ids[b][j]                              (assumed drawn from q_j)
 *   L   = first j with u_acc(j) >= min(1, p_j(x_j)/q_j(x_j)), else k        (C-1, C-2)
 *   t   = inverse-CDF sample from norm(max(0, p_L - q_L)) if L < k           (C-9)
 *         from p_k if L == k (bonus token, C-3); from p_L if the residual mass is 0 (C-6)
 *   u_acc(j), u_smp(j) = uniforms of Philox4x32-10 with key = seed and counter
 *         (j, round mod 2^32, rid mod 2^32, rid >> 32), rid = request_id_base + b     (C-8)
 * Greedy (temperature == 0): L = first j with x_j != argmax p_logits[b][j] (lowest index on
 * ties), t = argmax p_logits[b][L]; q_logits is not read and may be NULL (C-5).
 *
 * Arguments
 *   p_logits      device, [B][k+1][ld_p] elements of shape->dtype, rows 16-byte aligned; or
 *                 pinned host memory mapped into the device's address space (cudaHostAlloc /
 *                 cudaHostRegister under unified addressing): the kernels then read it in place
 *                 over PCIe, and the lazy path moves only the rows it needs (zero copy)
 *   q_logits      device (or mapped pinned host), [B][k][ld_q], rows 16-byte aligned; may be NULL
 *                 iff temperature == 0
 *   draft_ids     device, [B][k] int32
 *   shape         host pointer, read during the call only
 *   temperature   0 (greedy) or finite and >= 1e-3 (else SD_ERR_INVALID_ARGUMENT)
 *   seed, round, request_id_base   Philox stream selectors (see above)
 *   out_accept_len device, [B] int32: L in [0, k]
 *   out_tokens    device, [B][k+1] int32: x_0..x_{L-1}, then t, then -1 padding
 *   out_status    device, [B] int32 fault bitmask, or NULL
 *   workspace     device, >= sd_verify_workspace_size() bytes, 16-byte aligned, zero-filled
 *                 once before its first use.  Every call leaves the zero region of its shape
 *                 zeroed again (word 0 excepted: a 32-bit counter of calls the kernels keep, it
 *                 wraps); the library
 *                 remembers, per workspace pointer in this process, the layout of the last call
 *                 it enqueued there, and a call of another shape (batch, k, vocab, dtype, T == 0
 *                 or not) first zero-fills the union of both zero regions on `stream` (a
 *                 stream-ordered memset).  So one workspace serves any sequence of shapes as long
 *                 as it is large enough.  One workspace must not be used by two calls that may
 *                 run concurrently (e.g. on two streams); such misuse is detected by bounded
 *                 waits inside the kernels and reported as SD_FAULT_PROTOCOL, never as a hang.
 *   stream        CUDA stream the work is ordered on
 * Returns SD_OK (work enqueued), SD_ERR_INVALID_ARGUMENT, or SD_ERR_CUDA (launch failure).
 * The input and output buffers must stay valid until the stream has reached the call.
 */
sd_status sd_verify(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                    const sd_shape* shape, float temperature, uint64_t seed,
                    uint64_t round, uint64_t request_id_base,
                    int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                    void* workspace, size_t workspace_bytes, cudaStream_t stream);

/*
 * sd_verify_staged -- sd_verify for logits that live in mapped pinned HOST memory (zero copy,
 * see p_logits above): the statistics pass reads each row it needs over PCIe once and also writes
 * it to a device stage; the sampling pass then reads its stop row (p_L, q_L -- or p_k) from the
 * stage instead of crossing PCIe a second time.  Same arguments and results as sd_verify, plus
 *   p_stage, q_stage  device, [B][k+1][ld_p] and [B][k][ld_q] elements of shape->dtype, 16-byte
 *                     aligned, caller-owned; only the rows the call reads are written (contents
 *                     are scratch).  Ignored at T = 0 (greedy has no sampling pass).
 * The sampler then starts after the statistics kernel completes (no early launch).  Returns
 * SD_ERR_INVALID_ARGUMENT for a NULL / misaligned stage at T > 0.
 */
sd_status sd_verify_staged(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                           const sd_shape* shape, float temperature, uint64_t seed,
                           uint64_t round, uint64_t request_id_base,
                           int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                           void* workspace, size_t workspace_bytes, void* p_stage, void* q_stage,
                           cudaStream_t stream);

/* Bytes of workspace sd_verify needs for this shape/temperature (host only, no GPU work). */
sd_status sd_verify_workspace_size(const sd_shape* shape, float temperature, size_t* bytes);

/*
 * sd_verify_plan -- how sd_verify will run this shape (host only; launches nothing).
 *   variant      SD_VARIANT_TWO_LAUNCH: k_row_stats (grid = chunk x request x position,
 *                position-major; row statistics, decisions and most sampling chunk tasks) +
 *                k_sample_tail / k_finalize_greedy, PDL-chained
 *   launches     kernel launches per sd_verify call
 *   cluster      k_row_stats cluster size (0: none); slice = logits per CTA chunk
 *   ctas         CTAs of k_row_stats; tail_ctas: CTAs of the second kernel
 *   tagged       rows publish tagged partials to a start-ticket decider (2..64 chunks per row)
 *   options      SD_PLAN_* bits of the scheduling options in effect (environment knobs read once
 *                per process): EARLY = k_sample_req launched during the last
 *                position wave (tail_ctas includes its completion probe).  Bits 1 and 4 (PIPE,
 *                FUSED) are retired: those opt-in variants measured slower and were removed.
 */
enum { SD_PLAN_PIPE = 1, SD_PLAN_EARLY = 2, SD_PLAN_FUSED = 4 };
enum { SD_VARIANT_TWO_LAUNCH = 1 };
typedef struct {
    int32_t variant, launches, cluster, slice;
    int64_t ctas;
    int64_t tail_ctas;
    int32_t tagged;
    int32_t options;
} sd_plan;
sd_status sd_verify_plan(const sd_shape* shape, float temperature, sd_plan* out);

/*
 * sd_philox_uniforms -- the uniforms sd_verify draws (reading C-8), for tests and tooling.
 * For i in [0, n): counter = (pos[i], round mod 2^32, rid[i] mod 2^32, rid[i] >> 32), key = seed;
 * out_words[4 i .. 4 i + 3] = the four Philox4x32-10 output words (device, uint32).
 * pos (uint32) and rid (uint64) are device arrays of length n.
 */
sd_status sd_philox_uniforms(uint64_t seed, uint64_t round, const uint32_t* pos,
                             const uint64_t* rid, int32_t n, uint32_t* out_words,
                             cudaStream_t stream);

/*
 * sd_profile_events -- tracing hook for benchmarks.  After this call, the next n_pairs
 * sd_verify calls on this thread record events[2 i] immediately before and events[2 i + 1]
 * immediately after their dominant kernel (k_row_stats, the HBM-streaming kernel), on the call's
 * stream (graph capture records them as event nodes).  events: host array of 2 * n_pairs
 * caller-created cudaEvent_t handles; n_pairs = 0 disables.  The caller reads the durations
 * with cudaEventElapsedTime.
 */
sd_status sd_profile_events(cudaEvent_t* events, int32_t n_pairs);

/*
 * sd_profile_timestamps -- device-clock span of the dominant kernel without event nodes (an event
 * node between two kernels of a captured graph costs microseconds and inflates what it brackets).
 * After this call, the next n_calls two-launch sd_verify calls on this thread fold %globaltimer
 * (ns) into device_buf with atomic min: word 2 i = the earliest start of a k_row_stats CTA of call
 * i (after its dependency wait; the first row's CTAs, which the hardware dispatches first, report),
 * word 2 i + 1 = the earliest moment one of the first CTAs of the call's second kernel saw
 * k_row_stats complete (griddepcontrol.wait returned).  device_buf: device, 2 * n_calls
 * uint64 the caller fills with all-ones before the calls it profiles; NULL / 0 disables.
 */
sd_status sd_profile_timestamps(unsigned long long* device_buf, int32_t n_calls);

/*
 * sd_verify_trace -- test/debug hook: the fp64 statistics the most recent sd_verify call on
 * `workspace` (same shape and temperature > 0, already reached by `stream`) decided with, for the
 * tolerance checks of north_star ("probabilities and residual masses within 1e-5 relative").
 * Copied out by a small kernel on `stream` (device pointers):
 *   accept_len  [B] int32  the out_accept_len that call produced (selects the rows it reached)
 *   lam_p [B][k+1], lam_q [B][k]   natural-log log-normalisers logsumexp_x z(x)/T of the reached
 *               rows (j <= L); NaN for rows after L
 *   a     [B][k]   p_j(x_j)/q_j(x_j) as the acceptance test used it (not clamped to 1; 0 when
 *               q_j(x_j) = 0); NaN for rows after L or rows with a hard fault
 *   R     [B]      mass of the distribution the token was sampled from: residual 1 - beta_L
 *               (P:736), sum p_k at the bonus, sum p_L after the C-6 fallback; NaN if hard
 * Must be called before the workspace is used again.  Greedy calls have no such statistics
 * (SD_ERR_INVALID_ARGUMENT).
 */
sd_status sd_verify_trace(const sd_shape* shape, float temperature, const void* workspace,
                          const int32_t* accept_len, double* lam_p, double* lam_q, double* a,
                          double* R, cudaStream_t stream);

/* ======================================================================================
 * Draft side and exchange-minimal verify
 *
 * PAPER.md Alg. 2 ExpandLayer draws the draft tokens, and "the draft probabilities q_t(.)
 * needed by the correction step are stored in the tree metadata".  The verify step needs
 * of q_j only q_j(x_j) at every tested position, and the whole row only at the stop position L
 * (the residual).  sd_qmeta carries the first part in the kernels' own arithmetic, so
 * sd_verify_qmeta reads q rows only at L (a peer / remote pointer is fine) and takes decisions
 * bit-identical to sd_verify on the same rows ("minimal-transfer design").
 * log q_j(x_j) = ln 2 (zx c2 - D - log2 S), c2 = fl32(log2(e) / T).
 * ====================================================================================== */
typedef struct sd_qmeta_s {
    double S;          /* sum_x 2^(z(x) c2 - D) over the q row (fp64 across threads)           */
    float D;           /* the row's scaled maximum: max_x fl32(z(x) c2) (T = 0: the raw max)    */
    float zx;          /* z(x_j): the draft token's logit (NaN if x_j is outside [0, V))        */
    int32_t status;    /* SD_FAULT_NONFINITE / SD_FAULT_EMPTY_ROW of the q row, else 0         */
    int32_t reserved;
} sd_qmeta;            /* 24 bytes, 8-byte aligned */

/* Bytes of workspace sd_draft_sample / sd_draft_qmeta need (host only). */
sd_status sd_draft_workspace_size(const sd_shape* shape, float temperature, size_t* bytes);

/*
 * sd_draft_sample -- the draft-side sampler of the chain: x_j ~ softmax(q_logits[b][j] / T) for
 * every (b, j), by inverse CDF in ascending token id (C-9) at theta = u * sum_y q_j(y),
 * u = u24(w1) of Philox4x32-10 with key = seed and counter (0, round, rid_d lo, rid_d hi),
 * rid_d = 2^63 + (request_id_base + b) k + j -- a counter domain disjoint from sd_verify's (whose
 * request ids stay below 2^63), reading D-1 of DESIGN.md.  T = 0: argmax, lowest index.
 *   q_logits  device [B][k][ld_q] (shape->ld_q; shape->ld_p is ignored), rows 16-byte aligned
 *   out_ids   device [B][k] int32 (-1 for a row with NaN / +inf or no finite logit)
 *   out_qmeta device [B][k] sd_qmeta of the sampled tokens, or NULL
 *   out_status device [B][k] int32 fault bits of the q rows, or NULL
 *   workspace >= sd_draft_workspace_size() bytes, zero-filled once (same contract as sd_verify's)
 * Two passes over q (row statistics, then the sample) through the verify kernels themselves.
 */
sd_status sd_draft_sample(const void* q_logits, const sd_shape* shape, float temperature,
                          uint64_t seed, uint64_t round, uint64_t request_id_base,
                          int32_t* out_ids, sd_qmeta* out_qmeta, int32_t* out_status,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* sd_draft_qmeta -- the metadata of GIVEN draft tokens draft_ids [B][k] (T > 0): one pass of row
 * statistics over q_logits.  Same arguments as sd_draft_sample. */
sd_status sd_draft_qmeta(const void* q_logits, const int32_t* draft_ids, const sd_shape* shape,
                         float temperature, sd_qmeta* out_qmeta, void* workspace,
                         size_t workspace_bytes, cudaStream_t stream);

/*
 * sd_verify_qmeta -- sd_verify with the draft rows given as metadata: q_meta [B][k] (device)
 * replaces the statistics of q rows 0..k-1, and q_logits [B][k][ld_q] is read only at each
 * request's stop position L < k (one row per rejecting request; it may point to a peer GPU's
 * memory).  Same results as sd_verify on the same rows (bit-identical decisions and tokens when
 * q_meta comes from sd_draft_sample / sd_draft_qmeta on those rows); same workspace (size and
 * contract) as sd_verify.  T = 0 ignores q_meta and q_logits (greedy).
 */
sd_status sd_verify_qmeta(const void* p_logits, const void* q_logits, const sd_qmeta* q_meta,
                          const int32_t* draft_ids, const sd_shape* shape, float temperature,
                          uint64_t seed, uint64_t round, uint64_t request_id_base,
                          int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/*
 * sd_tree_verify -- lossless verification of a draft TREE.  The paper drafts
 * a depth-d tree with branching k (Alg. 2) and keeps the best of its
 * independently verified paths, which is not lossless; this call instead
 * walks the tree by recursive rejection sampling over the children of each node (reading D-2,
 * SpecInfer's multi-candidate rule, ref. [miao2024specinfer] at P:80): the `branching` children of
 * a node are i.i.d. draws from the node's draft distribution q; with d_0 = p,
 *   accept child i iff u_i < min(1, d_{i-1}(x_i) / q(x_i)) -> descend;
 *   else d_i = norm(max(0, d_{i-1} - q)) (the residual of P:736, applied again);
 *   all children rejected: emit t ~ d_m;  a leaf (depth d) reached: the bonus t ~ p_leaf.
 * branching = 1 is exactly sd_verify's chain (same Philox counters).  T = 0: descend into the first
 * child whose token is argmax p_node, else emit argmax p_node.
 * Layout: full m-ary trees (m = branching), level order: node 0 = root, children of n are
 * m n + 1 .. m n + m; N = sum_{t <= d} m^t nodes, N_int = sum_{t < d} m^t internal nodes.
 *   p_logits    device [B][N][ld_p]: target logits at every node (after the node's prefix)
 *   q_logits    device [B][N_int][ld_q]: draft logits at internal nodes (NULL iff T == 0)
 *   tree_tokens device [B][N] int32: each node's token (the root's entry is unused)
 *   shape       batch = B, k = depth d (1..31), vocab, ld_p, ld_q, dtype
 *   uniforms    child i at depth t: u24(w0) of counter (t + 32 i, round, rid); the emitted token
 *               at depth t: u24(w1) of (t, round, rid); rid = request_id_base + b (C-8)
 *   out_accept_len [B] = depth reached; out_tokens [B][d+1] = the accepted path's tokens, the
 *   emitted token, then -1; out_status [B] (nullable) fault bits; out_node [B] (nullable) = the
 *   node the walk stopped at.  One CTA per request; no workspace.
 */
sd_status sd_tree_verify(const void* p_logits, const void* q_logits, const int32_t* tree_tokens,
                         const sd_shape* shape, int32_t branching, float temperature,
                         uint64_t seed, uint64_t round, uint64_t request_id_base,
                         int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                         int32_t* out_node, cudaStream_t stream);

/*
 * sd_debug_trace -- development instrumentation (library built with STARSD_BUILD_DEBUG=1;
 * otherwise ignored).  When device_buf != NULL, subsequent sd_verify calls on this thread write
 * eight uint64 per k_row_stats CTA: %globaltimer at phase points 0..6 and word 7 = smid << 32 |
 * flags (tools/trace_rowstats.py).  NULL disables.
 */
sd_status sd_debug_trace(unsigned long long* device_buf);

/* ======================================================================================
 * Star exchange + round scheduler (Alg. 1, Sec. 4.1, App. E)
 *
 * One process per GPU.  Rank 0 is the draft instance M_q; ranks 1..world-1 are verifiers
 * M_p^(v).  Each (0, v) pair owns a dedicated 2-rank NCCL communicator -- the paper's
 * "unique tag and dedicated port" of the one-time handshake.
 *
 * Per round and verifier the draft sends the draft ids [B_v][k] (int32) and q logits
 * [B_v][k][V], and receives accept lengths [B_v] and tokens [B_v][k+1] (int32): the
 * verified prefix of P:806.  Each verifier has n_slots >= 2 in-flight slots (double
 * buffering), so the draft drafts for slot s' while slot s is being verified.
 * ====================================================================================== */

typedef struct sd_star sd_star;

typedef struct {
    int32_t rank;        /* 0 = draft, 1..world-1 = verifier                                 */
    int32_t world;       /* 2..8 on one node                                                 */
    int32_t n_slots;     /* >= 2 outstanding rounds per verifier                             */
    sd_shape max_shape;  /* upper bound of the per-round shape (B_v, k, V, dtype); rows are
                            exchanged dense: ld_p = ld_q = 0 or V, and V * element size must
                            be a multiple of 16 bytes (else SD_ERR_UNSUPPORTED /
                            SD_ERR_INVALID_ARGUMENT)                                         */
    float temperature;   /* verify temperature (0 = greedy)                                  */
    uint64_t seed;       /* Philox key used by the verifiers                                 */
    int32_t timeout_ms;  /* per-round completion timeout before SD_ERR_TIMEOUT (0 = none)    */
    int32_t device;      /* CUDA device ordinal of this rank                                 */
    int32_t transport;   /* SD_STAR_NCCL, or SD_STAR_LOOPBACK: one process plays the draft and
                            all world-1 verifiers on one device; the exchange is a D2D copy on
                            the pair's stream and the draft's round desc carries p_logits.
                            Same scheduler, poll and stats code as the NCCL transport.       */
    float target_ms;     /* verifier-side stand-in for the target model's forward (t_v of Eq.
                            6): a device-side spin of this many ms on the verifier's
                            stream before each verify (0 = none); used by tools/star_bench.py  */
    int32_t payload;     /* SD_STAR_PAYLOAD_FULL: ids + q rows [B_v][k][V] go out each round;
                            SD_STAR_PAYLOAD_QMETA (NEXT-1, "minimal-transfer design"): ids +
                            sd_qmeta [B_v][k] go out (24 bytes per draft token) and the verifier
                            reads only its requests' stop rows q_L from the draft GPU's memory
                            (NCCL transport: CUDA IPC peer mapping of per-(verifier, slot) staging
                            buffers exchanged at create; loopback: the draft's q_logits directly),
                            running sd_verify_qmeta                                            */
} sd_star_config;

enum { SD_STAR_PAYLOAD_FULL = 0, SD_STAR_PAYLOAD_QMETA = 1 };

enum { SD_STAR_NCCL = 0, SD_STAR_LOOPBACK = 1 };

/* One round for one (verifier, slot). */
typedef struct {
    int32_t verifier;            /* 1..world-1 (the peer, on the draft; own rank on a verifier) */
    int32_t slot;                /* 0..n_slots-1                                                 */
    uint64_t round;              /* Philox round selector                                        */
    int32_t batch;               /* B_v <= max_shape.batch                                       */
    uint64_t request_id_base;    /* Philox request-id base of this cohort                        */
    const void* p_logits;        /* verifier: [B_v][k+1][V] target logits; draft: NULL (NCCL) or
                                    the virtual verifier's target logits (SD_STAR_LOOPBACK)      */
    const int32_t* draft_ids;    /* draft: send source [B_v][k]; verifier: NULL -> receive       */
    const void* q_logits;        /* draft: send source [B_v][k][V]; verifier: NULL -> receive    */
    int32_t* out_accept_len;     /* draft: receive dst [B_v]; verifier: local result [B_v]       */
    int32_t* out_tokens;         /* draft: receive dst [B_v][k+1]; verifier: local result        */
    const struct sd_qmeta_s* q_meta; /* draft, QMETA payload: [B_v][k] metadata of draft_ids (from
                                    sd_draft_sample / sd_draft_qmeta); q_logits must then stay
                                    valid until the round returns (stop rows are read from it)  */
} sd_round_desc;

typedef struct {
    double busy_fraction;   /* union of draft-busy intervals / window (M_q load)          */
    double mean_idle_ms;    /* total draft idle / number of consecutive-service pairs; with N
                               verifiers served round-robin, N * mean_idle_ms = T_idle (Eq. 9)   */
    double mean_wait_ms;    /* mean time a completed return waited in Q_in before service        */
    double window_ms;       /* measurement window                                                */
    uint64_t rounds;        /* completed (verifier, slot) rounds                                 */
} sd_star_stats_t;

/* Size of the opaque communicator id the caller must broadcast (ncclUniqueId). */
#define SD_STAR_ID_BYTES 128

/* Draft rank only: generate the communicator ids, two per (0, v) pair -- id 2 (v-1) for the
 * draft -> verifier direction (ids, q rows), id 2 (v-1) + 1 for the verifier -> draft direction
 * (accept lengths, tokens) -- into ids_out [2 * (world-1) * SD_STAR_ID_BYTES] host bytes.  The
 * caller broadcasts them (e.g. through the torch.distributed store) before every rank calls
 * sd_star_create. */
sd_status sd_star_unique_ids(int32_t world, void* ids_out);

/* Create the handle: per-pair communicators (blocking, collective over each pair; one per
 * direction, each on its own stream, so a slot's payload ships while another slot's result is in
 * flight -- the decoupling of P:815-819), staging slots sized for max_shape, streams and events
 * (including a ring of 1024 pre-created busy-interval event pairs). */
sd_status sd_star_create(sd_star** out, const sd_star_config* cfg, const void* ids);

/* Draft: enqueue send(ids, q) on the pair's down stream and recv(results) on its up stream for
 *        (verifier, slot), ordered after `stream` (where the draft produced ids/q); returns at
 *        once.  The out buffers belong to the library until sd_star_poll returns that slot.
 * Verifier: recv(ids, q) into the slot's staging (down stream) -> sd_verify(p_logits, ...) on
 *        `stream` -> send(results) (up stream); results also land in out_accept_len / out_tokens,
 *        which must stay untouched until sd_star_poll returns the round.  A batch change between
 *        rounds of a slot is handled (the verify workspace re-zeroes itself). */
sd_status sd_star_round(sd_star* h, const sd_round_desc* d, cudaStream_t stream);

/* Draft: pop the next completed return in completion (FIFO) order -- the global request
 * buffer Q_in of Alg. 1.  Verifier: the oldest round whose results have been sent.
 * Waits up to timeout_us (0 = do not wait).  Returns SD_ERR_NOT_READY / SD_ERR_TIMEOUT when
 * nothing completed.  If a round has been in flight for longer than cfg.timeout_ms (> 0), or a
 * communicator reports an asynchronous error, every communicator of the handle is aborted
 * (ncclCommAbort) and SD_ERR_TIMEOUT / SD_ERR_NCCL is returned; the handle then only accepts
 * sd_star_destroy. */
sd_status sd_star_poll(sd_star* h, int32_t* verifier, int32_t* slot, uint64_t* round,
                       int32_t timeout_us);

/* Draft only: mark the start / end of draft work on `stream` (recorded as CUDA events from a
 * pre-created ring); the busy fraction is the union of these intervals over the window.
 * _v tags the interval with the verifier it serves (S(d) per verifier for the analytics). */
sd_status sd_star_draft_begin(sd_star* h, cudaStream_t stream);
sd_status sd_star_draft_begin_v(sd_star* h, int32_t verifier, cudaStream_t stream);
sd_status sd_star_draft_end(sd_star* h, cudaStream_t stream);

sd_status sd_star_stats(sd_star* h, sd_star_stats_t* out);
sd_status sd_star_destroy(sd_star* h);

/*
 * sd_star_simulate -- host-only run of the SAME work-conserving FIFO scheduler the draft rank
 * uses, driven by a deterministic fake transport (no GPU, no NCCL): n_verifiers targets, each
 * with n_slots independent closed-loop request streams (a stream issues its next request
 * only after its previous one was verified); every draft service takes service_ms (S(d), Eq. 5)
 * and every return takes return_ms (Z(d) = t_c + t_v, Eq. 6).  Runs `rounds` services and
 * reports busy fraction, mean idle gap (T_idle, Eq. 9) and mean queueing wait (T_wait).
 * For n_slots = 1 the busy fraction equals N S / (N S + T_idle) with
 * T_idle = max(0, Z - (N - 1) S)  (Eqs. 8-10); the smallest N with no idle gap is ceil(Z/S)+1.
 * sd_star_simulate_ex: per-verifier service_ms[v-1] / return_ms[v-1] (heterogeneous star, C4);
 * rounds_out[v-1] (nullable) = services of verifier v counted in the window.
 */
sd_status sd_star_simulate(int32_t n_verifiers, int32_t n_slots, double service_ms,
                           double return_ms, int32_t rounds, sd_star_stats_t* out);
sd_status sd_star_simulate_ex(int32_t n_verifiers, int32_t n_slots, const double* service_ms,
                              const double* return_ms, int32_t rounds, uint64_t* rounds_out,
                              sd_star_stats_t* out);

/* ======================================================================================
 * Star analytics and admission (Sec. 4, Eqs. 3-11; N_full / N_max)
 * ====================================================================================== */
typedef struct {
    double expected_accepted;      /* E[l]_gamma = sum_i beta_i (1 - beta_i^d) / (1 - beta_i)   (Eqs. 3-4) */
    double t_idle_ms;              /* max(0, Z - (N - 1) S)                                      (Eq. 9)    */
    double t_gamma_ms;             /* N S + T_idle                                               (Eq. 10)   */
    double throughput_per_ms;      /* O_gamma = E[l]_gamma / T_gamma (accepted tokens per ms)   (Eq. 11)   */
    double per_target_min_per_ms;  /* min_i E[l_i] / T_gamma                                               */
    double busy_fraction;          /* N S / T_gamma (the draft's load)                                     */
    int32_t n_full;                /* ceil(Z / S) + 1: the full-load onset */
    int32_t n_max;                 /* largest N whose per-target throughput E[l_i]/T_gamma(N) (mean beta)
                                      stays >= o_alone: the admission bound of P:343-345 (0: none)    */
    double service_ms, return_ms;  /* the S(d), Z(d) used (online estimates for sd_*_predict)           */
} sd_star_prediction;

/* Closed forms for n targets with acceptance rates beta[0..n-1], depth d, S(d) = service_ms,
 * Z(d) = return_ms and a standalone target speed o_alone (tokens per ms). */
sd_status sd_star_analytics(int32_t n, const double* beta, int32_t d, double service_ms,
                            double return_ms, double o_alone_per_ms, sd_star_prediction* out);

/* Draft only: feed the accept lengths of a returned round (host copy, n requests) into the online
 * estimate of verifier v's beta (MLE over the tests evaluated: accepted / (accepted + rejections));
 * sd_star_predict evaluates the closed forms on the online S(d) (draft busy intervals), Z(d)
 * (submit -> return, host clock) and betas, and the admission bound N_max. */
sd_status sd_star_observe(sd_star* h, int32_t verifier, const int32_t* accept_len_host, int32_t n);
sd_status sd_star_predict(sd_star* h, double o_alone_per_ms, sd_star_prediction* out);

/* Host-only scheduler handle: the star's FIFO scheduler and online estimators for callers that
 * bring their own transport (e.g. a gloo cross-process star in the tests).  Times are caller ms. */
typedef struct sd_sched sd_sched;
sd_status sd_sched_create(sd_sched** out, int32_t n_verifiers, int32_t k);
sd_status sd_sched_push(sd_sched* h, int32_t verifier, int32_t slot, uint64_t round, double t_ms);
sd_status sd_sched_pop(sd_sched* h, double now_ms, int32_t* verifier, int32_t* slot, uint64_t* round);
sd_status sd_sched_service(sd_sched* h, int32_t verifier, double t0_ms, double t1_ms);
sd_status sd_sched_observe(sd_sched* h, int32_t verifier, double return_ms,
                           const int32_t* accept_len, int32_t n);
sd_status sd_sched_stats(sd_sched* h, sd_star_stats_t* out);
sd_status sd_sched_predict(sd_sched* h, double o_alone_per_ms, sd_star_prediction* out);
sd_status sd_sched_destroy(sd_sched* h);

/* Static description of a status code. */
const char* sd_status_string(sd_status s);
/* Thread-local detail of the last error on this thread (CUDA/NCCL message, argument name). */
const char* sd_last_error(void);
/* Library version string. */
const char* sd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STARSD_H */
