// star.cpp -- StarSD's one-draft -> N-verifier exchange and round scheduler (a11, a12).
//
// PAPER.md Alg. 1 on one B200 node: rank 0 = draft M_q, ranks 1..N = verifiers
// M_p^(v).  The one-time handshake "unique tag + dedicated port" is one
// 2-rank NCCL communicator per (0, v) pair on its own CUDA stream; per round the draft sends the
// drafted ids + q rows and receives (accept length, tokens) -- the verified prefix of P:806.
// The draft's receiver / Q_in / draft-inference / sender loop is the scheduler below:
// completed returns are queued in completion order and served FIFO, work-conserving (P:189,
// P:296-297); busy intervals are CUDA events on the draft's compute stream (M_q load).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <queue>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "abi_internal.h"

#ifdef SD_WITH_NCCL
#include <nccl.h>
#endif

namespace sd {
cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t st);   // verify_kernels.cu

// ---- the scheduler: transport-agnostic, host-only ---------------------------------------
struct Ret {
    int32_t v, slot;
    uint64_t round;
    double t_ready;   // ms, when the return completed (entered Q_in)
};

class StarScheduler {
   public:
    void push_return(const Ret& r) { q_in_.push_back(r); }
    bool empty() const { return q_in_.empty(); }
    // FIFO pop (= "pop Q_in"); the queueing wait is recorded at service start
    bool pop(Ret* r, double now) {
        if (q_in_.empty()) return false;
        *r = q_in_.front();
        q_in_.pop_front();
        if (count_) waits_.push_back(now - r->t_ready);
        return true;
    }
    void busy(double t0, double t1) {
        if (count_) busy_.emplace_back(t0, t1);
    }
    void set_counting(bool on) { count_ = on; }
    // busy fraction = union of busy intervals / window; idle gaps between consecutive services
    sd_star_stats_t stats(uint64_t rounds) const {
        sd_star_stats_t s{};
        s.rounds = rounds;
        if (busy_.empty()) return s;
        std::vector<std::pair<double, double>> iv = busy_;
        std::sort(iv.begin(), iv.end());
        double total = 0.0, cur0 = iv[0].first, cur1 = iv[0].second, idle = 0.0;
        int gaps = 0;
        for (size_t i = 1; i < iv.size(); ++i) {
            if (iv[i].first > cur1) {
                total += cur1 - cur0;
                idle += iv[i].first - cur1;
                cur0 = iv[i].first;
            }
            ++gaps;
            cur1 = std::max(cur1, iv[i].second);
        }
        total += cur1 - cur0;
        s.window_ms = cur1 - iv[0].first;
        s.busy_fraction = s.window_ms > 0.0 ? total / s.window_ms : 1.0;
        s.mean_idle_ms = gaps ? idle / gaps : 0.0;
        double w = 0.0;
        for (double x : waits_) w += x;
        s.mean_wait_ms = waits_.empty() ? 0.0 : w / waits_.size();
        return s;
    }

   private:
    std::deque<Ret> q_in_;
    std::vector<double> waits_;
    std::vector<std::pair<double, double>> busy_;
    bool count_ = true;
};

static double host_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace sd

using namespace sd;

extern "C" {

// Deterministic fake transport driving the same scheduler (see include/starsd.h).
sd_status sd_star_simulate(int32_t n_verifiers, int32_t n_slots, double service_ms,
                           double return_ms, int32_t rounds, sd_star_stats_t* out) {
    clear_error();
    if (n_verifiers < 1 || n_slots < 1 || !(service_ms > 0.0) || !(return_ms >= 0.0) ||
        rounds < 1 || !out)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_simulate: bad argument");
    StarScheduler sched;
    // pending returns: (ready time, issue sequence) min-heap keeps FIFO order among ties
    using P = std::pair<std::pair<double, uint64_t>, Ret>;
    auto cmp = [](const P& a, const P& b) { return a.first > b.first; };
    std::priority_queue<P, std::vector<P>, decltype(cmp)> pending(cmp);
    uint64_t seq = 0;
    for (int32_t s = 0; s < n_slots; ++s)
        for (int32_t v = 1; v <= n_verifiers; ++v) sched.push_return(Ret{v, s, 0, 0.0});
    const int32_t warm = 2 * n_verifiers * n_slots;   // exclude the start-up transient
    double t = 0.0;
    sched.set_counting(false);
    for (int32_t i = 0; i < rounds + warm; ++i) {
        if (i == warm) sched.set_counting(true);
        while (!pending.empty() && pending.top().first.first <= t) {
            sched.push_return(pending.top().second);
            pending.pop();
        }
        if (sched.empty()) {                 // draft idles until the earliest return (T_idle)
            t = pending.top().first.first;
            while (!pending.empty() && pending.top().first.first <= t) {
                sched.push_return(pending.top().second);
                pending.pop();
            }
        }
        Ret r;
        sched.pop(&r, t);
        const double t0 = t;
        t += service_ms;                     // S(d) = d t_s
        sched.busy(t0, t);
        Ret nx{r.v, r.slot, r.round + 1, t + return_ms};   // Z(d) = t_c + t_v later
        pending.push(P{{nx.t_ready, seq++}, nx});
    }
    *out = sched.stats(static_cast<uint64_t>(rounds));
    return SD_OK;
}

}  // extern "C"

// ---- NCCL transport -------------------------------------------------------------------------
#ifdef SD_WITH_NCCL

struct sd_star {
    sd_star_config cfg{};
    int esz = 4;
    bool loop = false;                      // SD_STAR_LOOPBACK
    std::vector<ncclComm_t> comms;          // draft: index v (1..world-1); verifier: [0]
    std::vector<cudaStream_t> cstreams;     // draft: per-verifier pair streams
    struct Slot {
        cudaEvent_t ev_ret = nullptr;
        bool busy = false;
        uint64_t round = 0;
        uint64_t seq = 0;
    };
    std::vector<Slot> slots;                // draft: [world * n_slots]
    uint64_t seq = 0;
    cudaEvent_t ev_ready = nullptr;
    cudaEvent_t ev_origin = nullptr;
    // verifier staging (receive targets), results and verify workspace, one set per slot
    // (NCCL verifier: index slot; loopback: index v * n_slots + slot)
    std::vector<void*> q_buf;
    std::vector<int32_t*> ids_buf, L_buf, tok_buf;
    std::vector<void*> ws;
    size_t ws_bytes = 0;
    // draft busy accounting
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> busy;
    cudaEvent_t open_begin = nullptr;
    StarScheduler sched;
    uint64_t served = 0;
};

static sd_status cuda_fail(cudaError_t e, const char* what) {
    return fail(SD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
static sd_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(SD_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}
#define SD_CUDA(x)                                       \
    do {                                                 \
        cudaError_t e_ = (x);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
    } while (0)
#define SD_NCCL(x)                                       \
    do {                                                 \
        ncclResult_t r_ = (x);                           \
        if (r_ != ncclSuccess) return nccl_fail(r_, #x); \
    } while (0)

static sd_status alloc_staging(sd_star* h, int n) {
    const sd_shape& ms = h->cfg.max_shape;
    const size_t B = ms.batch, k = ms.k, V = ms.vocab;
    sd_status st = sd_verify_workspace_size(&ms, h->cfg.temperature, &h->ws_bytes);
    if (st != SD_OK) return st;
    for (int i = 0; i < n; ++i) {
        void *q = nullptr, *w = nullptr;
        int32_t *idb = nullptr, *lb = nullptr, *tb = nullptr;
        SD_CUDA(cudaMalloc(&q, B * k * V * h->esz));
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&idb), B * k * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&lb), B * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&tb), B * (k + 1) * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(&w, h->ws_bytes));
        SD_CUDA(cudaMemset(w, 0, h->ws_bytes));
        h->q_buf.push_back(q);
        h->ids_buf.push_back(idb);
        h->L_buf.push_back(lb);
        h->tok_buf.push_back(tb);
        h->ws.push_back(w);
    }
    return SD_OK;
}

static sd_status star_init(sd_star* h, const void* ids);

static ncclDataType_t nccl_dtype(sd_dtype d) { return d == SD_DTYPE_F32 ? ncclFloat32 : ncclBfloat16; }

extern "C" {

sd_status sd_star_unique_ids(int32_t world, void* ids_out) {
    clear_error();
    if (world < 2 || !ids_out) return fail(SD_ERR_INVALID_ARGUMENT, "world < 2 or ids_out NULL");
    static_assert(sizeof(ncclUniqueId) == SD_STAR_ID_BYTES, "ncclUniqueId size");
    for (int32_t v = 1; v < world; ++v) {
        ncclUniqueId id;
        SD_NCCL(ncclGetUniqueId(&id));
        memcpy(static_cast<char*>(ids_out) + (v - 1) * SD_STAR_ID_BYTES, &id, SD_STAR_ID_BYTES);
    }
    return SD_OK;
}

sd_status sd_star_create(sd_star** out, const sd_star_config* cfg, const void* ids) {
    clear_error();
    if (!out || !cfg || (!ids && cfg->transport == SD_STAR_NCCL))
        return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    if (cfg->world < 2 || cfg->rank < 0 || cfg->rank >= cfg->world || cfg->n_slots < 1)
        return fail(SD_ERR_INVALID_ARGUMENT, "rank/world/n_slots");
    int esz;
    sd_status st = check_shape(&cfg->max_shape, cfg->temperature, &esz);
    if (st != SD_OK) return st;
    if ((cfg->max_shape.ld_p && cfg->max_shape.ld_p != cfg->max_shape.vocab) ||
        (cfg->max_shape.ld_q && cfg->max_shape.ld_q != cfg->max_shape.vocab))
        return fail(SD_ERR_UNSUPPORTED, "the star exchanges dense rows (ld == vocab)");
    if (cfg->transport != SD_STAR_NCCL && cfg->transport != SD_STAR_LOOPBACK)
        return fail(SD_ERR_INVALID_ARGUMENT, "transport");
    if (cfg->transport == SD_STAR_LOOPBACK && cfg->rank != 0)
        return fail(SD_ERR_INVALID_ARGUMENT, "loopback: one process, rank 0");
    SD_CUDA(cudaSetDevice(cfg->device));
    sd_star* h = new sd_star();
    h->cfg = *cfg;
    h->esz = esz;
    h->loop = cfg->transport == SD_STAR_LOOPBACK;
    st = star_init(h, ids);
    if (st != SD_OK) {
        const std::string msg = sd_last_error();
        sd_star_destroy(h);
        return fail(st, "%s", msg.c_str());
    }
    *out = h;
    return SD_OK;
}

}  // extern "C"

static sd_status star_init(sd_star* h, const void* ids) {
    const sd_star_config* cfg = &h->cfg;
    sd_status st;
    const ncclUniqueId* uid = static_cast<const ncclUniqueId*>(ids);
    if (cfg->rank == 0) {
        h->comms.assign(cfg->world, nullptr);
        h->cstreams.assign(cfg->world, nullptr);
        if (!h->loop) {
            SD_NCCL(ncclGroupStart());
            for (int v = 1; v < cfg->world; ++v)
                SD_NCCL(ncclCommInitRank(&h->comms[v], 2, uid[v - 1], 0));
            SD_NCCL(ncclGroupEnd());
        } else {
            st = alloc_staging(h, cfg->world * cfg->n_slots);
            if (st != SD_OK) return st;
        }
        for (int v = 1; v < cfg->world; ++v)
            SD_CUDA(cudaStreamCreateWithFlags(&h->cstreams[v], cudaStreamNonBlocking));
        h->slots.resize(static_cast<size_t>(cfg->world) * cfg->n_slots);
        for (auto& s : h->slots) SD_CUDA(cudaEventCreateWithFlags(&s.ev_ret, cudaEventDisableTiming));
    } else {
        h->comms.assign(1, nullptr);
        SD_NCCL(ncclCommInitRank(&h->comms[0], 2, uid[cfg->rank - 1], 1));
        st = alloc_staging(h, cfg->n_slots);
        if (st != SD_OK) return st;
    }
    SD_CUDA(cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
    SD_CUDA(cudaEventCreate(&h->ev_origin));
    SD_CUDA(cudaEventRecord(h->ev_origin, 0));
    return SD_OK;
}

extern "C" {

sd_status sd_star_round(sd_star* h, const sd_round_desc* d, cudaStream_t stream) {
    clear_error();
    if (!h || !d) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    const sd_shape& ms = h->cfg.max_shape;
    if (d->batch < 1 || d->batch > ms.batch || d->slot < 0 || d->slot >= h->cfg.n_slots)
        return fail(SD_ERR_INVALID_ARGUMENT, "batch / slot out of range");
    if (!d->out_accept_len || !d->out_tokens)
        return fail(SD_ERR_INVALID_ARGUMENT, "out_accept_len / out_tokens NULL");
    const size_t B = d->batch, k = ms.k, V = ms.vocab;
    const ncclDataType_t dt = nccl_dtype(ms.dtype);
    const bool greedy = h->cfg.temperature == 0.0f;
    if (h->cfg.rank == 0) {
        // draft: ship ids + q (sender), post the receive of the verified prefix
        const int v = d->verifier;
        if (v < 1 || v >= h->cfg.world) return fail(SD_ERR_INVALID_ARGUMENT, "verifier");
        if (!d->draft_ids || (!greedy && !d->q_logits))
            return fail(SD_ERR_INVALID_ARGUMENT, "draft_ids / q_logits NULL");
        sd_star::Slot& s = h->slots[static_cast<size_t>(v) * h->cfg.n_slots + d->slot];
        if (s.busy) return fail(SD_ERR_INVALID_ARGUMENT, "slot still in flight");
        cudaStream_t cs = h->cstreams[v];
        SD_CUDA(cudaEventRecord(h->ev_ready, stream));
        SD_CUDA(cudaStreamWaitEvent(cs, h->ev_ready, 0));
        if (h->loop) {
            // the same exchange as a D2D copy on the pair stream; the virtual verifier's
            // recv -> verify -> send runs on that stream too
            if (!d->p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "loopback: p_logits NULL");
            const size_t i = static_cast<size_t>(v) * h->cfg.n_slots + d->slot;
            SD_CUDA(cudaMemcpyAsync(h->ids_buf[i], d->draft_ids, B * k * 4, cudaMemcpyDeviceToDevice, cs));
            if (!greedy)
                SD_CUDA(cudaMemcpyAsync(h->q_buf[i], d->q_logits, B * k * V * h->esz,
                                        cudaMemcpyDeviceToDevice, cs));
            if (h->cfg.target_ms > 0.0f) SD_CUDA(launch_spin_ns(static_cast<uint64_t>(h->cfg.target_ms * 1e6), cs));
            sd_shape sh = ms;
            sh.batch = d->batch;
            sd_status st = sd_verify(d->p_logits, greedy ? nullptr : h->q_buf[i], h->ids_buf[i], &sh,
                                     h->cfg.temperature, h->cfg.seed, d->round, d->request_id_base,
                                     h->L_buf[i], h->tok_buf[i], nullptr, h->ws[i], h->ws_bytes, cs);
            if (st != SD_OK) return st;
            SD_CUDA(cudaMemcpyAsync(d->out_accept_len, h->L_buf[i], B * 4, cudaMemcpyDeviceToDevice, cs));
            SD_CUDA(cudaMemcpyAsync(d->out_tokens, h->tok_buf[i], B * (k + 1) * 4,
                                    cudaMemcpyDeviceToDevice, cs));
            SD_CUDA(cudaEventRecord(s.ev_ret, cs));
            s.busy = true;
            s.round = d->round;
            s.seq = h->seq++;
            return SD_OK;
        }
        SD_NCCL(ncclGroupStart());
        SD_NCCL(ncclSend(d->draft_ids, B * k, ncclInt32, 1, h->comms[v], cs));
        if (!greedy) SD_NCCL(ncclSend(d->q_logits, B * k * V, dt, 1, h->comms[v], cs));
        SD_NCCL(ncclRecv(d->out_accept_len, B, ncclInt32, 1, h->comms[v], cs));
        SD_NCCL(ncclRecv(d->out_tokens, B * (k + 1), ncclInt32, 1, h->comms[v], cs));
        SD_NCCL(ncclGroupEnd());
        SD_CUDA(cudaEventRecord(s.ev_ret, cs));
        s.busy = true;
        s.round = d->round;
        s.seq = h->seq++;
        return SD_OK;
    }
    // verifier: recv -> verify -> send, all ordered on `stream`
    if (!d->p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "p_logits NULL");
    void* q = h->q_buf[d->slot];
    int32_t* ids = h->ids_buf[d->slot];
    SD_NCCL(ncclGroupStart());
    SD_NCCL(ncclRecv(ids, B * k, ncclInt32, 0, h->comms[0], stream));
    if (!greedy) SD_NCCL(ncclRecv(q, B * k * V, dt, 0, h->comms[0], stream));
    SD_NCCL(ncclGroupEnd());
    if (h->cfg.target_ms > 0.0f) SD_CUDA(launch_spin_ns(static_cast<uint64_t>(h->cfg.target_ms * 1e6), stream));
    sd_shape sh = ms;
    sh.batch = d->batch;
    sd_status st = sd_verify(d->p_logits, greedy ? nullptr : q, ids, &sh, h->cfg.temperature,
                             h->cfg.seed, d->round, d->request_id_base, d->out_accept_len,
                             d->out_tokens, nullptr, h->ws[d->slot], h->ws_bytes, stream);
    if (st != SD_OK) return st;
    SD_NCCL(ncclGroupStart());
    SD_NCCL(ncclSend(d->out_accept_len, B, ncclInt32, 0, h->comms[0], stream));
    SD_NCCL(ncclSend(d->out_tokens, B * (k + 1), ncclInt32, 0, h->comms[0], stream));
    SD_NCCL(ncclGroupEnd());
    return SD_OK;
}

sd_status sd_star_poll(sd_star* h, int32_t* verifier, int32_t* slot, uint64_t* round,
                       int32_t timeout_us) {
    clear_error();
    if (!h || !verifier || !slot || !round) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    if (h->cfg.rank != 0) return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_poll is draft-only");
    const double t_end = host_ms() + timeout_us / 1000.0;
    while (true) {
        // receiver: move completed returns into Q_in in issue order
        std::vector<std::pair<uint64_t, size_t>> done;
        for (size_t i = 0; i < h->slots.size(); ++i) {
            sd_star::Slot& s = h->slots[i];
            if (!s.busy) continue;
            const cudaError_t e = cudaEventQuery(s.ev_ret);
            if (e == cudaSuccess) done.emplace_back(s.seq, i);
            else if (e != cudaErrorNotReady) return cuda_fail(e, "cudaEventQuery");
        }
        std::sort(done.begin(), done.end());
        const double now = host_ms();
        for (auto& p : done) {
            sd_star::Slot& s = h->slots[p.second];
            s.busy = false;
            h->sched.push_return(Ret{static_cast<int32_t>(p.second / h->cfg.n_slots),
                                     static_cast<int32_t>(p.second % h->cfg.n_slots), s.round, now});
        }
        Ret r;
        if (h->sched.pop(&r, now)) {
            *verifier = r.v;
            *slot = r.slot;
            *round = r.round;
            ++h->served;
            return SD_OK;
        }
        for (int v = 1; v < h->cfg.world && !h->loop; ++v) {
            ncclResult_t ae = ncclSuccess;
            if (ncclCommGetAsyncError(h->comms[v], &ae) == ncclSuccess && ae != ncclSuccess &&
                ae != ncclInProgress)
                return nccl_fail(ae, "async NCCL error");
        }
        if (timeout_us <= 0) return SD_ERR_NOT_READY;
        if (host_ms() >= t_end) return fail(SD_ERR_TIMEOUT, "no return within %d us", timeout_us);
        std::this_thread::yield();
    }
}

sd_status sd_star_draft_begin(sd_star* h, cudaStream_t stream) {
    clear_error();
    if (!h || h->cfg.rank != 0) return fail(SD_ERR_INVALID_ARGUMENT, "draft-only");
    if (h->open_begin) return fail(SD_ERR_INVALID_ARGUMENT, "draft_begin without draft_end");
    SD_CUDA(cudaEventCreate(&h->open_begin));
    SD_CUDA(cudaEventRecord(h->open_begin, stream));
    return SD_OK;
}

sd_status sd_star_draft_end(sd_star* h, cudaStream_t stream) {
    clear_error();
    if (!h || h->cfg.rank != 0 || !h->open_begin)
        return fail(SD_ERR_INVALID_ARGUMENT, "draft_end without draft_begin");
    cudaEvent_t e;
    SD_CUDA(cudaEventCreate(&e));
    SD_CUDA(cudaEventRecord(e, stream));
    h->busy.emplace_back(h->open_begin, e);
    h->open_begin = nullptr;
    return SD_OK;
}

sd_status sd_star_stats(sd_star* h, sd_star_stats_t* out) {
    clear_error();
    if (!h || !out) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    StarScheduler s;          // busy timeline from the CUDA events (device clock)
    for (auto& p : h->busy) {
        SD_CUDA(cudaEventSynchronize(p.second));
        float a = 0.f, b = 0.f;
        SD_CUDA(cudaEventElapsedTime(&a, h->ev_origin, p.first));
        SD_CUDA(cudaEventElapsedTime(&b, h->ev_origin, p.second));
        s.busy(a, b);
    }
    *out = s.stats(h->served);
    const sd_star_stats_t q = h->sched.stats(h->served);
    out->mean_wait_ms = q.mean_wait_ms;      // queueing wait is measured on the host clock
    return SD_OK;
}

sd_status sd_star_destroy(sd_star* h) {
    clear_error();
    if (!h) return SD_OK;
    for (auto c : h->comms)
        if (c) ncclCommDestroy(c);
    for (auto s : h->cstreams)
        if (s) cudaStreamDestroy(s);
    for (auto& s : h->slots)
        if (s.ev_ret) cudaEventDestroy(s.ev_ret);
    for (auto& p : h->busy) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    for (auto q : h->q_buf) cudaFree(q);
    for (auto i : h->ids_buf) cudaFree(i);
    for (auto i : h->L_buf) cudaFree(i);
    for (auto i : h->tok_buf) cudaFree(i);
    for (auto w : h->ws) cudaFree(w);
    if (h->ev_ready) cudaEventDestroy(h->ev_ready);
    if (h->ev_origin) cudaEventDestroy(h->ev_origin);
    delete h;
    return SD_OK;
}

}  // extern "C"

#else  // !SD_WITH_NCCL

extern "C" {
sd_status sd_star_unique_ids(int32_t, void*) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_create(sd_star**, const sd_star_config*, const void*) {
    return fail(SD_ERR_UNSUPPORTED, "built without NCCL");
}
sd_status sd_star_round(sd_star*, const sd_round_desc*, cudaStream_t) {
    return fail(SD_ERR_UNSUPPORTED, "built without NCCL");
}
sd_status sd_star_poll(sd_star*, int32_t*, int32_t*, uint64_t*, int32_t) {
    return fail(SD_ERR_UNSUPPORTED, "built without NCCL");
}
sd_status sd_star_draft_begin(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_draft_end(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_stats(sd_star*, sd_star_stats_t*) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_destroy(sd_star*) { return SD_OK; }
}

#endif
