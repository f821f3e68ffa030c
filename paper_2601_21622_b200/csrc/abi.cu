// abi.cu -- the extern "C" boundary of libstarsd.so (include/starsd.h): argument validation,
// workspace layout, dispatch to the sm_100a kernels, status strings.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/starsd.h"
#include "abi_internal.h"
#include "verify.cuh"

namespace sd {
cudaError_t launch_verify(const Params& P, bool greedy, bool bf16, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1);
cudaError_t launch_philox(uint64_t seed, uint64_t round, const uint32_t* pos, const uint64_t* rid,
                          int n, uint32_t* out, cudaStream_t st);

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

// Kernel variant.  Default: the two-launch path (verify_kernels.cu: k_row_stats + k_sample /
// k_finalize_greedy, PDL-chained), measured fastest on B200 for every BASELINE config.
// STARSD_KERNEL=stream selects the persistent warp-specialized cluster kernel (verify_stream.cu)
// when the shape fits it: a cross-variant parity check and design study.
enum Variant { kTwoLaunch = 1, kStream = 3 };
static Variant variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("STARSD_KERNEL");
        v = (e && strcmp(e, "stream") == 0) ? kStream : kTwoLaunch;
    }
    return static_cast<Variant>(v);
}

bool stream_config(int32_t V, int esz, bool greedy, StreamPlan* out);
cudaError_t launch_stream(const SParams& P, bool greedy, bool bf16, size_t smem, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1);

void record_event(cudaEvent_t ev, cudaStream_t st);

// The stream kernel uses a prefix of the two-launch layout (rej_mask, ticketB, rowstat).
static size_t ws_bytes(int32_t B, int32_t k, int32_t V, int32_t esz) {
    return ws_layout(B, k, V, esz).total;
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

}  // namespace sd

using namespace sd;

extern "C" {

sd_status sd_verify_workspace_size(const sd_shape* shape, float temperature, size_t* bytes) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (!bytes) return fail(SD_ERR_INVALID_ARGUMENT, "bytes is NULL");
    *bytes = ws_bytes(shape->batch, shape->k, shape->vocab, esz);
    return SD_OK;
}

sd_status sd_verify(const void* p_logits, const void* q_logits, const int32_t* draft_ids,
                    const sd_shape* shape, float temperature, uint64_t seed, uint64_t round,
                    uint64_t request_id_base, int32_t* out_accept_len, int32_t* out_tokens,
                    int32_t* out_status, void* workspace, size_t workspace_bytes,
                    cudaStream_t stream) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (shape->batch == 0) return SD_OK;
    const bool greedy = temperature == 0.0f;
    if (!p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "p_logits is NULL");
    if (!greedy && !q_logits) return fail(SD_ERR_INVALID_ARGUMENT, "q_logits is NULL (T > 0)");
    if (!draft_ids) return fail(SD_ERR_INVALID_ARGUMENT, "draft_ids is NULL");
    if (!out_accept_len || !out_tokens)
        return fail(SD_ERR_INVALID_ARGUMENT, "out_accept_len / out_tokens is NULL");
    if (!workspace) return fail(SD_ERR_INVALID_ARGUMENT, "workspace is NULL");
    if (!aligned16(p_logits) || (!greedy && !aligned16(q_logits)) || !aligned16(workspace))
        return fail(SD_ERR_INVALID_ARGUMENT, "p_logits / q_logits / workspace not 16-byte aligned");
    const size_t need = ws_bytes(shape->batch, shape->k, shape->vocab, esz);
    if (workspace_bytes < need)
        return fail(SD_ERR_INVALID_ARGUMENT, "workspace_bytes=%zu < required %zu",
                    workspace_bytes, need);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (g_prof_ev && g_prof_i < g_prof_n) {
        ev0 = g_prof_ev[2 * g_prof_i];
        ev1 = g_prof_ev[2 * g_prof_i + 1];
        ++g_prof_i;
    }
    // c2 = log2(e) / T rounded to fp32; every exponent in the kernels uses this one constant
    const float c2 =
        greedy ? 0.0f : static_cast<float>(1.4426950408889634 / static_cast<double>(temperature));
    const WsLayout w = ws_layout(shape->batch, shape->k, shape->vocab, esz);
    char* ws = static_cast<char*>(workspace);
    StreamPlan sp;
    if (variant() == kStream && stream_config(shape->vocab, esz, greedy, &sp)) {
        SParams S{};
        S.p = p_logits;
        S.q = greedy ? nullptr : q_logits;
        S.ids = draft_ids;
        S.B = shape->batch;
        S.k = shape->k;
        S.V = shape->vocab;
        S.ld_p = shape->ld_p ? shape->ld_p : shape->vocab;
        S.ld_q = shape->ld_q ? shape->ld_q : shape->vocab;
        S.C = sp.C;
        S.G = sp.G;
        S.W = sp.W;
        S.segmax = sp.segmax;
        S.nslot = sp.nslot;
        S.c2 = c2;
        S.seed = seed;
        S.round = round;
        S.rid_base = request_id_base;
        S.out_L = out_accept_len;
        S.out_tok = out_tokens;
        S.out_status = out_status;
        S.rej_mask = reinterpret_cast<uint32_t*>(ws + w.rej_mask);
        S.ticket = reinterpret_cast<uint32_t*>(ws + w.ticketB);
        S.rowres = reinterpret_cast<int2*>(ws + w.rowstat);
        S.trace = g_trace;
        {
            static int dbg = -1;
            if (dbg < 0) {
                const char* e = getenv("STARSD_DEBUG");
                dbg = e ? atoi(e) : 0;
            }
            S.debug = dbg;
        }
        cudaError_t e = launch_stream(S, greedy, shape->dtype == SD_DTYPE_BF16, sp.smem, stream, ev0, ev1);
        if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
        return SD_OK;
    }
    Params P{};
    P.p = p_logits;
    P.q = greedy ? nullptr : q_logits;
    P.ids = draft_ids;
    P.B = shape->batch;
    P.k = shape->k;
    P.V = shape->vocab;
    P.ld_p = shape->ld_p ? shape->ld_p : shape->vocab;
    P.ld_q = shape->ld_q ? shape->ld_q : shape->vocab;
    chunking(P.V, esz, &P.nch, &P.CH);
    P.CL = row_cluster(P.nch);
    P.G = (P.nch + P.CL - 1) / P.CL;
    P.nseg = P.CH / (32 * (kVecBytes / esz));
    P.c2 = c2;
    P.c2d = static_cast<double>(P.c2);
    P.seed = seed;
    P.round = round;
    P.rid_base = request_id_base;
    P.out_L = out_accept_len;
    P.trace = g_trace;
    P.prof_ts = nullptr;
    P.epoch = reinterpret_cast<uint32_t*>(ws + w.epoch);
    P.partT = reinterpret_cast<unsigned long long*>(ws + w.partT);
    {
        static int tag = -1;   // STARSD_PUBLISH=ticket: release-ordered partials + row ticket
        if (tag < 0) {
            const char* e = getenv("STARSD_PUBLISH");
            tag = (e && strcmp(e, "ticket") == 0) ? 0 : 1;
        }
        P.tagpub = (tag && P.CL == 1 && P.nch >= 2 && P.nch <= kMaxTagNch) ? 1 : 0;
    }
    if (g_ts && g_ts_i < g_ts_n) P.prof_ts = g_ts + 2 * static_cast<size_t>(g_ts_i++);
    {
        static int chain = -1;   // STARSD_CHAIN=0: plain stream order before k_row_stats
        if (chain < 0) {
            const char* e = getenv("STARSD_CHAIN");
            chain = (e && strcmp(e, "0") == 0) ? 0 : 1;
        }
        P.chain = chain;
    }
    P.out_tok = out_tokens;
    P.out_status = out_status;
    P.rej_mask = reinterpret_cast<uint32_t*>(ws + w.rej_mask);
    P.ticketA = reinterpret_cast<uint32_t*>(ws + w.ticketA);
    P.ticketB = reinterpret_cast<uint32_t*>(ws + w.ticketB);
    P.rowstat = reinterpret_cast<RowStat*>(ws + w.rowstat);
    P.partA = reinterpret_cast<PartA*>(ws + w.partA);
    P.partB = reinterpret_cast<PartB*>(ws + w.partB);
    P.segtab = reinterpret_cast<double2*>(ws + w.segtab);

    cudaError_t e = launch_verify(P, greedy, shape->dtype == SD_DTYPE_BF16, stream, ev0, ev1);
    if (e != cudaSuccess) return fail(SD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SD_OK;
}

sd_status sd_verify_plan(const sd_shape* shape, float temperature, sd_plan* out) {
    clear_error();
    int esz;
    sd_status s = check_shape(shape, temperature, &esz);
    if (s != SD_OK) return s;
    if (!out) return fail(SD_ERR_INVALID_ARGUMENT, "out is NULL");
    const bool greedy = temperature == 0.0f;
    *out = sd_plan{};
    StreamPlan sp;
    if (variant() == kStream && stream_config(shape->vocab, esz, greedy, &sp)) {
        out->variant = SD_VARIANT_STREAM;
        out->launches = 1;
        out->cluster = sp.C;
        out->slice = sp.W;
        out->ctas = (int64_t)sp.G * sp.C;
        out->max_active_clusters = sp.G;
        out->smem_bytes = (int32_t)sp.smem;
        return SD_OK;
    }
    int32_t nch, CH;
    chunking(shape->vocab, esz, &nch, &CH);
    out->variant = SD_VARIANT_TWO_LAUNCH;
    out->launches = 2;
    out->slice = CH;
    const int32_t CL = row_cluster(nch), G = (nch + CL - 1) / CL;
    out->cluster = CL > 1 ? CL : 0;
    out->ctas = (int64_t)(shape->k + 1) * shape->batch * (CL > 1 ? G * CL : nch);
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

const char* sd_version(void) { return "starsd-b200 0.1 (sm_100a)"; }

}  // extern "C"
