// abi.cu -- the extern "C" boundary of libstarsd.so (include/starsd.h): argument validation,
// workspace layout and bookkeeping, dispatch to the sm_100a kernels, status strings.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/starsd.h"
#include "abi_internal.h"
#include "verify.cuh"

namespace sd {
cudaError_t launch_verify(const Params& P, bool greedy, bool bf16, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1);
cudaError_t launch_philox(uint64_t seed, uint64_t round, const uint32_t* pos, const uint64_t* rid,
                          int n, uint32_t* out, cudaStream_t st);
cudaError_t launch_trace(const Params& P, const int32_t* accept_len, double* lam_p, double* lam_q,
                         double* a, double* R, cudaStream_t st);
cudaError_t launch_qmeta(const Params& P, bool bf16, const int32_t* ids, QMeta* out,
                         cudaStream_t st);
struct TreeParams {
    const void* p;
    const void* q;
    const int32_t* tok;
    int32_t B, m, d, V, N, Nint;
    int64_t ld_p, ld_q;
    float c2;
    uint64_t seed, round, rid_base;
    int32_t* out_L;
    int32_t* out_tok;
    int32_t* out_status;
    int32_t* out_node;
};
cudaError_t launch_tree(const TreeParams& P, bool bf16, cudaStream_t st);
cudaError_t qmeta_gather(const Params& P, bool bf16, const int32_t* ids, QMeta* out,
                         cudaStream_t st);

static thread_local char g_err[512] = "";
static thread_local cudaEvent_t* g_prof_ev = nullptr;
static thread_local int32_t g_prof_n = 0, g_prof_i = 0;
static thread_local unsigned long long* g_ts = nullptr;
static thread_local int32_t g_ts_n = 0, g_ts_i = 0;
static thread_local unsigned long long* g_trace = nullptr;

sd_status fail(sd_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}
void clear_error() { g_err[0] = '\0'; }
const char* last_error() { return g_err; }

static int env_flag(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

constexpr int32_t kMaxVocab = 1 << 24;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Validate a shape + temperature; fills the element size.
sd_status check_shape(const sd_shape* s, float T, int* esz) {
    if (!s) return fail(SD_ERR_INVALID_ARGUMENT, "shape is NULL");
    if (s->batch < 0) return fail(SD_ERR_INVALID_ARGUMENT, "shape.batch=%d < 0", s->batch);
    if (s->k < 1 || s->k > SD_MAX_K)
        return fail(SD_ERR_INVALID_ARGUMENT, "shape.k=%d outside [1, %d]", s->k, SD_MAX_K);
    if (s->vocab < 2) return fail(SD_ERR_INVALID_ARGUMENT, "shape.vocab=%d < 2", s->vocab);
    if (s->dtype != SD_DTYPE_F32 && s->dtype != SD_DTYPE_BF16)
        return fail(SD_ERR_INVALID_ARGUMENT, "shape.dtype=%d unknown", (int)s->dtype);
    *esz = s->dtype == SD_DTYPE_F32 ? 4 : 2;
    const int64_t ldp = s->ld_p ? s->ld_p : s->vocab;
    const int64_t ldq = T == 0.0f ? ldp : (s->ld_q ? s->ld_q : s->vocab);   // q unused at T=0
    if (ldp < s->vocab || ldq < s->vocab)
        return fail(SD_ERR_INVALID_ARGUMENT, "row stride smaller than vocab");
    if ((ldp * *esz) % 16 != 0 || (ldq * *esz) % 16 != 0)
        return fail(SD_ERR_INVALID_ARGUMENT,
                    "row strides must be multiples of 16 bytes (ld_p=%lld, ld_q=%lld)",
                    (long long)ldp, (long long)ldq);
    if (!(T == 0.0f || (std::isfinite(T) && T >= 1e-3f)))
        return fail(SD_ERR_INVALID_ARGUMENT, "temperature=%g must be 0 or finite >= 1e-3",
                    (double)T);
    if (s->vocab > kMaxVocab)
        return fail(SD_ERR_UNSUPPORTED, "vocab=%d too large for this build (max %d)", s->vocab,
                    kMaxVocab);
    const int64_t rows = (int64_t)(s->k + 1) * s->batch;
    if (rows >= (1LL << 31)) return fail(SD_ERR_UNSUPPORTED, "batch=%d too large", s->batch);
    return SD_OK;
}

// ---- workspace bookkeeping --------------------------------------------------------------------
// Every call leaves the zero region of ITS layout zeroed.  The library remembers, per workspace
// pointer, the layout of the last call it enqueued there; a call whose layout differs first
// zero-fills (stream-ordered memset) the union of both zero regions -- past word 0, the call
// counter the tagged partials derive their tags from, which must keep increasing.  So one
// workspace serves any sequence of shapes (include/starsd.h).
struct WsSig {
    int32_t B, k, V, esz;
    bool greedy;
    size_t zero_bytes;
    bool operator==(const WsSig& o) const {
        return B == o.B && k == o.k && V == o.V && esz == o.esz && greedy == o.greedy;
    }
};
static std::mutex g_ws_mu;
static std::unordered_map<uintptr_t, WsSig> g_ws;

static sd_status ws_prepare(void* ws, const WsSig& sig, cudaStream_t st) {
    size_t clear = 0;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        auto it = g_ws.find(reinterpret_cast<uintptr_t>(ws));
        if (it == g_ws.end()) {
            g_ws.emplace(reinterpret_cast<uintptr_t>(ws), sig);   // zero-filled by the caller
        } else if (!(it->second == sig)) {
            clear = it->second.zero_bytes > sig.zero_bytes ? it->second.zero_bytes : sig.zero_bytes;
            it->second = sig;
        }
    }
    if (clear > 16) {
        const cudaError_t e = cudaMemsetAsync(static_cast<char*>(ws) + 16, 0, clear - 16, st);
        if (e != cudaSuccess)
            return fail(SD_ERR_CUDA, "workspace reset: %s", cudaGetErrorString(e));
    }
    return SD_OK;
}

// Shared by sd_verify and sd_verify_trace: the kernels' view of a call.
static void fill_params(Params& P, const sd_shape* shape, int esz, float temperature,
                        void* workspace) {
    const bool greedy = temperature == 0.0f;
    const WsLayout w = ws_layout(shape->batch, shape->k, shape->vocab, esz);
    char* ws = static_cast<char*>(workspace);
    P.B = shape->batch;
    P.k = shape->k;
    P.V = shape->vocab;
    P.ld_p = shape->ld_p ? shape->ld_p : shape->vocab;
    P.ld_q = shape->ld_q ? shape->ld_q : shape->vocab;
    chunking(P.V, esz, &P.nch, &P.CH, rs_chunk_bytes(greedy, esz));
    P.CL = row_cluster(P.nch);
    P.G = (P.nch + P.CL - 1) / P.CL;
    P.nseg = P.CH / (32 * (kVecBytes / esz));
    // c2 = log2(e) / T rounded to fp32; every exponent in the kernels uses this one constant
    P.c2 = greedy ? 0.0f : static_cast<float>(1.4426950408889634 / static_cast<double>(temperature));
    P.c2d = static_cast<double>(P.c2);
    P.epoch = reinterpret_cast<uint32_t*>(ws + w.epoch);
    P.state = reinterpret_cast<unsigned long long*>(ws + w.state);
    P.ticketA = reinterpret_cast<uint32_t*>(ws + w.ticketA);
    P.ticketB = reinterpret_cast<uint32_t*>(ws + w.ticketB);
    P.tailT = reinterpret_cast<uint32_t*>(ws + w.tailT);
    P.rowstat = reinterpret_cast<RowStat*>(ws + w.rowstat);
    P.partA = reinterpret_cast<PartA*>(ws + w.partA);
    P.partB = reinterpret_cast<PartB*>(ws + w.partB);
    P.segtab = reinterpret_cast<double2*>(ws + w.segtab);
    P.rres = reinterpret_cast<double*>(ws + w.rres);
    P.partT = reinterpret_cast<unsigned long long*>(ws + w.partT);
    static const int tag = env_flag("STARSD_PUBLISH_TICKET", 0) ? 0 : 1;   // A/B knob
    P.tagpub = (tag && P.CL == 1 && P.nch >= 2 && P.nch <= kMaxTagNch) ? 1 : 0;
    static const int chain = env_flag("STARSD_CHAIN", 1);   // 0: plain stream order
    P.chain = chain ? 1 : 0;
    P.esz = esz;
    static const int early = env_flag("STARSD_EARLY", 1);       // A/B knob
    const int64_t nseg_row = (static_cast<int64_t>(P.V) + 32 * (16 / esz) - 1) / (32 * (16 / esz));
    P.early = (early && !greedy && P.chain &&
               nseg_row <= 2048) ? 1 : 0;   // (k_sample_req's on-chip table: kSMaxSeg)
    static const int rg = env_flag("STARSD_RGROUP", 0);          // A/B knob
    P.rgroup = rg > 0 ? rg : 0;
}

}  // namespace sd

using namespace sd;

extern "C" {

sd_status sd_verify_workspace_size(const sd_shape* shape, float temperature, size_t* bytes) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (!bytes) return fail(SD_ERR_INVALID_ARGUMENT, "bytes is NULL");
    *bytes = ws_layout(shape->batch, shape->k, shape->vocab, esz).total;
    return SD_OK;
}

static sd_status verify_impl(const void* p_logits, const void* q_logits, const QMeta* qmeta,
                             const int32_t* draft_ids, const sd_shape* shape, float temperature,
                             uint64_t seed, uint64_t round, uint64_t request_id_base,
                             int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream,
                             void* p_stage = nullptr, void* q_stage = nullptr) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (shape->batch == 0) return SD_OK;
    const bool greedy = temperature == 0.0f;
    if (!p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "p_logits is NULL");
    if (!greedy && !q_logits) return fail(SD_ERR_INVALID_ARGUMENT, "q_logits is NULL (T > 0)");
    if (!greedy && qmeta && (reinterpret_cast<uintptr_t>(qmeta) & 7u))
        return fail(SD_ERR_INVALID_ARGUMENT, "q_meta not 8-byte aligned");
    if (!draft_ids) return fail(SD_ERR_INVALID_ARGUMENT, "draft_ids is NULL");
    if (!out_accept_len || !out_tokens)
        return fail(SD_ERR_INVALID_ARGUMENT, "out_accept_len / out_tokens is NULL");
    if (!workspace) return fail(SD_ERR_INVALID_ARGUMENT, "workspace is NULL");
    if (!aligned16(p_logits) || (!greedy && !aligned16(q_logits)) || !aligned16(workspace))
        return fail(SD_ERR_INVALID_ARGUMENT, "p_logits / q_logits / workspace not 16-byte aligned");
    const WsLayout w = ws_layout(shape->batch, shape->k, shape->vocab, esz);
    if (workspace_bytes < w.total)
        return fail(SD_ERR_INVALID_ARGUMENT, "workspace_bytes=%zu < required %zu",
                    workspace_bytes, w.total);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (g_prof_ev && g_prof_i < g_prof_n) {
        ev0 = g_prof_ev[2 * g_prof_i];
        ev1 = g_prof_ev[2 * g_prof_i + 1];
        ++g_prof_i;
    }
    s = ws_prepare(workspace, WsSig{shape->batch, shape->k, shape->vocab, esz, greedy, w.zero_bytes},
                   stream);
    if (s != SD_OK) return s;
    Params P{};
    fill_params(P, shape, esz, temperature, workspace);
    P.p = p_logits;
    P.q = greedy ? nullptr : q_logits;
    P.qmeta = greedy ? nullptr : qmeta;
    P.ids = draft_ids;
    if (!greedy && p_stage) {
        // staged rows: the sampler reads them after k_row_stats is complete (no early launch,
        // no in-kernel sampling, the grid form of k_row_stats)
        P.p_stage = p_stage;
        P.q_stage = q_stage;
        P.early = 0;
    }
    P.seed = seed;
    P.round = round;
    P.rid_base = request_id_base;
    P.out_L = out_accept_len;
    P.out_tok = out_tokens;
    P.out_status = out_status;
    P.trace = g_trace;
    P.prof_ts = nullptr;
    if (g_ts && g_ts_i < g_ts_n) P.prof_ts = g_ts + 2 * static_cast<size_t>(g_ts_i++);
    cudaError_t e = launch_verify(P, greedy, shape->dtype == SD_DTYPE_BF16, stream, ev0, ev1);
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_verify(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                    const sd_shape* shape, float temperature, uint64_t seed, uint64_t round,
                    uint64_t request_id_base, int32_t* out_accept_len, int32_t* out_tokens,
                    int32_t* out_status, void* workspace, size_t workspace_bytes,
                    cudaStream_t stream) {
    return verify_impl(p_logits, q_logits, nullptr, draft_ids, shape, temperature, seed, round,
                       request_id_base, out_accept_len, out_tokens, out_status, workspace,
                       workspace_bytes, stream);
}

sd_status sd_verify_staged(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                           const sd_shape* shape, float temperature, uint64_t seed, uint64_t round,
                           uint64_t request_id_base, int32_t* out_accept_len, int32_t* out_tokens,
                           int32_t* out_status, void* workspace, size_t workspace_bytes,
                           void* p_stage, void* q_stage, cudaStream_t stream) {
    if (temperature != 0.0f && (!p_stage || !q_stage || !aligned16(p_stage) || !aligned16(q_stage))) {
        clear_error();
        return fail(SD_ERR_INVALID_ARGUMENT, "p_stage / q_stage NULL or not 16-byte aligned (T > 0)");
    }
    return verify_impl(p_logits, q_logits, nullptr, draft_ids, shape, temperature, seed, round,
                       request_id_base, out_accept_len, out_tokens, out_status, workspace,
                       workspace_bytes, stream, temperature != 0.0f ? p_stage : nullptr,
                       temperature != 0.0f ? q_stage : nullptr);
}

sd_status sd_verify_qmeta(const void* p_logits, const void* q_logits, const sd_qmeta* q_meta,
                          const int32_t* draft_ids, const sd_shape* shape, float temperature,
                          uint64_t seed, uint64_t round, uint64_t request_id_base,
                          int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream) {
    static_assert(sizeof(sd_qmeta) == sizeof(QMeta), "sd_qmeta layout");
    if (temperature != 0.0f && !q_meta) {
        clear_error();
        return fail(SD_ERR_INVALID_ARGUMENT, "q_meta is NULL (T > 0)");
    }
    return verify_impl(p_logits, q_logits, reinterpret_cast<const QMeta*>(q_meta), draft_ids,
                       shape, temperature, seed, round, request_id_base, out_accept_len,
                       out_tokens, out_status, workspace, workspace_bytes, stream);
}

// ---- draft side (NEXT-2): the q rows as k = 0 "requests" of the verify kernels ----------------
// Row r = b k + j of q_logits is request r of an internal call with k = 0: k_row_stats computes its
// statistics exactly as it does for a verify's q rows (so the metadata is bit-identical to what a
// full verify computes), and k_sample_req's bonus path samples it by inverse CDF with the counter
// (0, round, 2^63 + request_id_base k + r) (reading D-1) -- or k_finalize_greedy takes its argmax.
static WsLayout draft_layout(const sd_shape* shape, int esz, size_t* total) {
    const int32_t R = shape->batch * shape->k;
    const WsLayout w = ws_layout(R, 0, shape->vocab, esz);
    *total = w.total + align16(sizeof(int32_t) * (size_t)R);
    return w;
}

sd_status sd_draft_workspace_size(const sd_shape* shape, float temperature, size_t* bytes) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (!bytes) return fail(SD_ERR_INVALID_ARGUMENT, "bytes is NULL");
    if ((int64_t)shape->batch * shape->k >= (1LL << 31))
        return fail(SD_ERR_UNSUPPORTED, "batch * k too large");
    draft_layout(shape, esz, bytes);
    return SD_OK;
}

static sd_status draft_call(const void* q_logits, const int32_t* ids_in, const sd_shape* shape,
                            float temperature, uint64_t seed, uint64_t round,
                            uint64_t request_id_base, int32_t* out_ids, sd_qmeta* out_qmeta,
                            int32_t* out_status, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream) {
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (shape->batch == 0) return SD_OK;
    if (!q_logits || !workspace) return fail(SD_ERR_INVALID_ARGUMENT, "q_logits / workspace NULL");
    if (!aligned16(q_logits) || !aligned16(workspace) ||
        (out_qmeta && (reinterpret_cast<uintptr_t>(out_qmeta) & 7u)))
        return fail(SD_ERR_INVALID_ARGUMENT, "q_logits / workspace / out_qmeta misaligned");
    size_t need;
    const WsLayout w = draft_layout(shape, esz, &need);
    if (workspace_bytes < need)
        return fail(SD_ERR_INVALID_ARGUMENT, "workspace_bytes=%zu < required %zu", workspace_bytes, need);
    const bool greedy = temperature == 0.0f;
    sd_shape in = *shape;                     // internal: R rows, k = 0, the q stride as p stride
    in.batch = shape->batch * shape->k;
    in.k = 0;
    in.ld_p = shape->ld_q ? shape->ld_q : shape->vocab;
    in.ld_q = in.ld_p;
    s = ws_prepare(workspace, WsSig{in.batch, 0, in.vocab, esz, greedy, w.zero_bytes}, stream);
    if (s != SD_OK) return s;
    Params P{};
    fill_params(P, &in, esz, temperature, workspace);
    P.p = q_logits;
    P.q = nullptr;
    P.ids = nullptr;
    P.seed = seed;
    P.round = round;
    P.rid_base = (1ull << 63) + request_id_base * static_cast<uint64_t>(shape->k);
    P.out_L = reinterpret_cast<int32_t*>(static_cast<char*>(workspace) + w.total);
    P.out_status = out_status;
    const bool bf16 = shape->dtype == SD_DTYPE_BF16;
    cudaError_t e;
    if (ids_in) {                              // metadata of given tokens (no sampling)
        e = launch_qmeta(P, bf16, ids_in, reinterpret_cast<QMeta*>(out_qmeta), stream);
    } else {
        P.out_tok = out_ids;
        e = launch_verify(P, greedy, bf16, stream, nullptr, nullptr);
        if (e == cudaSuccess && out_qmeta)
            e = qmeta_gather(P, bf16, out_ids, reinterpret_cast<QMeta*>(out_qmeta), stream);
    }
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_draft_sample(const void* q_logits, const sd_shape* shape, float temperature,
                          uint64_t seed, uint64_t round, uint64_t request_id_base,
                          int32_t* out_ids, sd_qmeta* out_qmeta, int32_t* out_status,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream) {
    clear_error();
    if (!out_ids) return fail(SD_ERR_INVALID_ARGUMENT, "out_ids is NULL");
    return draft_call(q_logits, nullptr, shape, temperature, seed, round, request_id_base, out_ids,
                      out_qmeta, out_status, workspace, workspace_bytes, stream);
}

sd_status sd_draft_qmeta(const void* q_logits, const int32_t* draft_ids, const sd_shape* shape,
                         float temperature, sd_qmeta* out_qmeta, void* workspace,
                         size_t workspace_bytes, cudaStream_t stream) {
    clear_error();
    if (!draft_ids || !out_qmeta) return fail(SD_ERR_INVALID_ARGUMENT, "draft_ids / out_qmeta NULL");
    if (temperature == 0.0f) return fail(SD_ERR_INVALID_ARGUMENT, "sd_draft_qmeta: T > 0 only");
    return draft_call(q_logits, draft_ids, shape, temperature, 0, 0, 0, nullptr, out_qmeta,
                      nullptr, workspace, workspace_bytes, stream);
}

sd_status sd_tree_verify(const void* p_logits, const void* q_logits, const int32_t* tree_tokens,
                         const sd_shape* shape, int32_t branching, float temperature,
                         uint64_t seed, uint64_t round, uint64_t request_id_base,
                         int32_t* out_accept_len, int32_t* out_tokens, int32_t* out_status,
                         int32_t* out_node, cudaStream_t stream) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (branching < 1 || branching > 8)
        return fail(SD_ERR_INVALID_ARGUMENT, "branching=%d outside [1, 8]", branching);
    int64_t N = 0, Nint = 0, w = 1;
    for (int t = 0; t <= shape->k; ++t) {
        N += w;
        if (t < shape->k) Nint += w;
        w *= branching;
        if (N > (1 << 20)) return fail(SD_ERR_UNSUPPORTED, "tree of more than 2^20 nodes");
    }
    if (shape->batch == 0) return SD_OK;
    const bool greedy = temperature == 0.0f;
    if (!p_logits || (!greedy && !q_logits) || !tree_tokens || !out_accept_len || !out_tokens)
        return fail(SD_ERR_INVALID_ARGUMENT, "NULL pointer");
    if (!aligned16(p_logits) || (!greedy && !aligned16(q_logits)))
        return fail(SD_ERR_INVALID_ARGUMENT, "p_logits / q_logits not 16-byte aligned");
    TreeParams P{};
    P.p = p_logits;
    P.q = greedy ? nullptr : q_logits;
    P.tok = tree_tokens;
    P.B = shape->batch;
    P.m = branching;
    P.d = shape->k;
    P.V = shape->vocab;
    P.N = static_cast<int32_t>(N);
    P.Nint = static_cast<int32_t>(Nint);
    P.ld_p = shape->ld_p ? shape->ld_p : shape->vocab;
    P.ld_q = shape->ld_q ? shape->ld_q : shape->vocab;
    P.c2 = greedy ? 0.0f : static_cast<float>(1.4426950408889634 / static_cast<double>(temperature));
    P.seed = seed;
    P.round = round;
    P.rid_base = request_id_base;
    P.out_L = out_accept_len;
    P.out_tok = out_tokens;
    P.out_status = out_status;
    P.out_node = out_node;
    cudaError_t e = launch_tree(P, shape->dtype == SD_DTYPE_BF16, stream);
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_verify_trace(const sd_shape* shape, float temperature, const void* workspace,
                          const int32_t* accept_len, double* lam_p, double* lam_q, double* a,
                          double* R, cudaStream_t stream) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (temperature == 0.0f)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_verify_trace: sampled calls only (T > 0)");
    if (shape->batch == 0) return SD_OK;
    if (!workspace || !accept_len || !lam_p || !lam_q || !a || !R)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_verify_trace: NULL argument");
    Params P{};
    fill_params(P, shape, esz, temperature, const_cast<void*>(workspace));
    cudaError_t e = launch_trace(P, accept_len, lam_p, lam_q, a, R, stream);
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_verify_plan(const sd_shape* shape, float temperature, sd_plan* out) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (!out) return fail(SD_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = sd_plan{};
    int32_t nch, CH;
    chunking(shape->vocab, esz, &nch, &CH, rs_chunk_bytes(temperature == 0.0f, esz));
    out->variant = SD_VARIANT_TWO_LAUNCH;
    out->launches = 2;
    out->slice = CH;
    const int32_t CL = row_cluster(nch), G = (nch + CL - 1) / CL;
    out->cluster = CL > 1 ? CL : 0;
    out->ctas = (int64_t)(shape->k + 1) * shape->batch * (CL > 1 ? G * CL : nch);
    const int32_t nseg_row = (shape->vocab + 32 * (16 / esz) - 1) / (32 * (16 / esz));
    out->tail_ctas = temperature == 0.0f ? (shape->batch + 127) / 128
                     : nseg_row <= 2048   ? shape->batch                       /* k_sample_req */
                                          : (int64_t)nch * shape->batch;       /* k_sample_chunked */
    out->tagged = (CL == 1 && nch >= 2 && nch <= kMaxTagNch && !env_flag("STARSD_PUBLISH_TICKET", 0));
    // the options fill_params takes for this shape (no workspace is touched: pointers only)
    Params P{};
    alignas(16) static char dummy[16];
    fill_params(P, shape, esz, temperature, dummy);
    out->options = P.early ? SD_PLAN_EARLY : 0;
    if (P.early) out->tail_ctas += 1;
    return SD_OK;
}

sd_status sd_philox_uniforms(uint64_t seed, uint64_t round, const uint32_t* pos,
                             const uint64_t* rid, int32_t n, uint32_t* out_words,
                             cudaStream_t stream) {
    clear_error();
    if (n < 0) return fail(SD_ERR_INVALID_ARGUMENT, "n < 0");
    if (n > 0 && (!pos || !rid || !out_words))
        return fail(SD_ERR_INVALID_ARGUMENT, "NULL pointer");
    if (!aligned16(out_words)) return fail(SD_ERR_INVALID_ARGUMENT, "out_words not 16-byte aligned");
    cudaError_t e = launch_philox(seed, round, pos, rid, n, out_words, stream);
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_profile_events(cudaEvent_t* events, int32_t n_pairs) {
    clear_error();
    if (n_pairs < 0 || (n_pairs > 0 && !events))
        return fail(SD_ERR_INVALID_ARGUMENT, "events / n_pairs");
    g_prof_ev = n_pairs ? events : nullptr;
    g_prof_n = n_pairs;
    g_prof_i = 0;
    return SD_OK;
}

sd_status sd_profile_timestamps(unsigned long long* device_buf, int32_t n_calls) {
    clear_error();
    if (n_calls < 0 || (n_calls > 0 && !device_buf))
        return fail(SD_ERR_INVALID_ARGUMENT, "device_buf / n_calls");
    g_ts = n_calls ? device_buf : nullptr;
    g_ts_n = n_calls;
    g_ts_i = 0;
    return SD_OK;
}

sd_status sd_debug_trace(unsigned long long* device_buf) {
    g_trace = device_buf;
    return SD_OK;
}

const char* sd_status_string(sd_status s) {
    switch (s) {
        case SD_OK: return "SD_OK";
        case SD_ERR_INVALID_ARGUMENT: return "SD_ERR_INVALID_ARGUMENT";
        case SD_ERR_UNSUPPORTED: return "SD_ERR_UNSUPPORTED";
        case SD_ERR_CUDA: return "SD_ERR_CUDA";
        case SD_ERR_NCCL: return "SD_ERR_NCCL";
        case SD_ERR_TIMEOUT: return "SD_ERR_TIMEOUT";
        case SD_ERR_NOT_READY: return "SD_ERR_NOT_READY";
        case SD_ERR_INTERNAL: return "SD_ERR_INTERNAL";
    }
    return "SD_ERR_UNKNOWN";
}

const char* sd_last_error(void) { return last_error(); }

const char* sd_version(void) { return "starsd-b200 0.2 (sm_100a)"; }

}  // extern "C"
