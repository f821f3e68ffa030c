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
    SD_FAULT_ZERO_RESIDUAL = 16    /* info: residual mass R == 0, sampled from p_L (C-6)      */
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
 *   p_logits      device, [B][k+1][ld_p] elements of shape->dtype, rows 16-byte aligned
 *   q_logits      device, [B][k][ld_q], rows 16-byte aligned; may be NULL iff temperature == 0
 *   draft_ids     device, [B][k] int32
 *   shape         host pointer, read during the call only
 *   temperature   0 (greedy) or finite and >= 1e-3 (else SD_ERR_INVALID_ARGUMENT)
 *   seed, round, request_id_base   Philox stream selectors (see above)
 *   out_accept_len device, [B] int32: L in [0, k]
 *   out_tokens    device, [B][k+1] int32: x_0..x_{L-1}, then t, then -1 padding
 *   out_status    device, [B] int32 fault bitmask, or NULL
 *   workspace     device, >= sd_verify_workspace_size() bytes, 16-byte aligned, zero-filled
 *                 once before first use.  Every call leaves the zero region of its shape
 *                 zeroed again (word 0 excepted: a call counter the kernels keep, any value is
 *                 valid), so calls of one shape (batch, k, vocab, dtype, T == 0 or not) reuse it
 *                 as is; before a call of another shape it must be zero-filled again.  One
 *                 workspace must not be used by two calls that may run concurrently.
 *   stream        CUDA stream the work is ordered on
 * Returns SD_OK (work enqueued), SD_ERR_INVALID_ARGUMENT, or SD_ERR_CUDA (launch failure).
 * The input and output buffers must stay valid until the stream has reached the call.
 */
sd_status sd_verify(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                    const sd_shape* shape, float temperature, uint64_t seed,
                    uint64_t round, uint64_t request_id_base,
                    int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                    void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Bytes of workspace sd_verify needs for this shape/temperature (host only, no GPU work). */
sd_status sd_verify_workspace_size(const sd_shape* shape, float temperature, size_t* bytes);

/*
 * sd_verify_plan -- how sd_verify will run this shape on the current device (host only; it
 * may query the device's occupancy limits, but launches nothing).
 *   variant      SD_VARIANT_TWO_LAUNCH (default): k_row_stats (grid = chunk x request x position,
 *                position-major) + k_sample / k_finalize_greedy, PDL-chained;
 *                SD_VARIANT_STREAM (STARSD_KERNEL=stream, when the shape fits): one launch of `ctas`
 *                persistent CTAs in clusters of `cluster`, each streaming a `slice`-logit slice of
 *                every row pair its cluster owns through a TMA ring
 *   launches     kernel launches per sd_verify call
 *   cluster, slice, ctas   cluster size (0: none), logits per CTA slice / chunk, CTAs in the first
 *                launch
 *   max_active_clusters, smem_bytes   occupancy of the stream variant (0 otherwise)
 */
enum { SD_VARIANT_TWO_LAUNCH = 1, SD_VARIANT_STREAM = 3 };
typedef struct {
    int32_t variant, launches, cluster, slice;
    int64_t ctas;
    int32_t max_active_clusters;   /* stream variant: clusters the device keeps resident */
    int32_t smem_bytes;            /* stream variant: dynamic shared memory per CTA       */
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
 * immediately after their dominant kernel (k_row_stats, the HBM-streaming kernel, or the stream
 * variant's single kernel), on the call's
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
 * sd_debug_trace -- development instrumentation of the stream variant (library built with
 * STARSD_BUILD_DEBUG=1; otherwise ignored).  When device_buf != NULL, subsequent stream-variant
 * sd_verify calls on this thread write, per CTA, a record log of kSTraceN = 8192 uint64 words:
 * word 0 = record count, then event records (type << 56 | arg << 40 | %globaltimer), and the
 * last 16 words = clock64 accounting counters (tools/trace_stream.py, tools/analyze_strace.py).
 * NULL disables.
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
} sd_star_config;

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

/* Draft rank only: generate (world-1) ids, one per (0, v) pair, into ids_out
 * [(world-1) * SD_STAR_ID_BYTES] host bytes.  The caller broadcasts them (e.g. through the
 * torch.distributed store) before every rank calls sd_star_create. */
sd_status sd_star_unique_ids(int32_t world, void* ids_out);

/* Create the handle: per-pair communicators (blocking, collective over each pair), staging
 * slots sized for max_shape, streams and events. */
sd_status sd_star_create(sd_star** out, const sd_star_config* cfg, const void* ids);

/* Draft: enqueue send(ids, q) -> recv(results) for (verifier, slot) on the pair's stream,
 *        ordered after `stream` (where the draft produced ids/q); returns immediately.
 * Verifier: recv(ids, q) into the slot -> sd_verify(p_logits, ...) -> send(results), all
 *        ordered on `stream`; results also land in out_accept_len / out_tokens. */
sd_status sd_star_round(sd_star* h, const sd_round_desc* d, cudaStream_t stream);

/* Draft only: pop the next completed return in completion (FIFO) order -- the global request
 * buffer Q_in of Alg. 1.  Waits up to timeout_us (0 = do not wait).  Returns
 * SD_ERR_NOT_READY / SD_ERR_TIMEOUT when nothing completed. */
sd_status sd_star_poll(sd_star* h, int32_t* verifier, int32_t* slot, uint64_t* round,
                       int32_t timeout_us);

/* Draft only: mark the start / end of draft work on `stream` (recorded as CUDA events); the
 * busy fraction is the union of these intervals over the window. */
sd_status sd_star_draft_begin(sd_star* h, cudaStream_t stream);
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
 */
sd_status sd_star_simulate(int32_t n_verifiers, int32_t n_slots, double service_ms,
                           double return_ms, int32_t rounds, sd_star_stats_t* out);

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
