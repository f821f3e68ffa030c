// star.cpp -- StarSD's one-draft -> N-verifier exchange, round scheduler and analytics
// (8(f) NEXT-4).
//
// PAPER.md Alg. 1 on one B200 node: rank 0 = draft M_q, ranks 1..N = verifiers
// M_p^(v).  The one-time handshake "unique tag + dedicated port" is, per
// (0, v) pair, two 2-rank NCCL communicators -- one per direction, each on its own CUDA stream --
// so the draft ships slot s' (ids + q rows) while the verified prefix of slot s is still on its
// way back (the decoupling of P:815-819).  The draft's receiver / Q_in / draft-inference /
// sender loop is the scheduler below: completed returns are queued in completion
// order and served FIFO, work-conserving; busy intervals are CUDA events on the
// draft's compute stream (M_q load).  The analytics restate Sec. 4 (Eqs. 3-11)
// and the admission rule of P:343-345 over online estimates of S(d), Z(d) and beta.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
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
    explicit StarScheduler(int32_t n_verifiers = 0, int32_t k = 0)
        : k_(k), s_(n_verifiers + 1), z_(n_verifiers + 1), acc_(n_verifiers + 1), tests_(n_verifiers + 1) {}
    void push_return(const Ret& r) { q_in_.push_back(r); }
    bool empty() const { return q_in_.empty(); }
    size_t pending() const { return q_in_.size(); }
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
    // online estimates (NEXT-4): S(d) per service, Z(d) per return, accept lengths per verifier
    void observe_service(int32_t v, double ms) {
        if (v >= 0 && v < static_cast<int32_t>(s_.size())) s_[v].add(ms);
        s_all_.add(ms);
    }
    void observe_return(int32_t v, double z_ms) {
        if (v >= 0 && v < static_cast<int32_t>(z_.size())) z_[v].add(z_ms);
        z_all_.add(z_ms);
    }
    // beta-hat (MLE for i.i.d. acceptance truncated at k): accepted tests / tests evaluated;
    // a request with accept length L evaluated L tests that passed and one that failed (L < k)
    void observe_accepts(int32_t v, const int32_t* L, int32_t n) {
        if (v < 0 || v >= static_cast<int32_t>(acc_.size())) return;
        for (int32_t i = 0; i < n; ++i) {
            const int32_t l = std::max(0, std::min(L[i], k_));
            acc_[v] += l;
            tests_[v] += l + (l < k_ ? 1 : 0);
        }
    }
    double mean_S(int32_t v) const { return v > 0 && s_[v].n ? s_[v].mean() : s_all_.mean(); }
    double mean_Z(int32_t v) const { return v > 0 && z_[v].n ? z_[v].mean() : z_all_.mean(); }
    double beta_hat(int32_t v) const { return tests_[v] > 0 ? static_cast<double>(acc_[v]) / tests_[v] : NAN; }
    int32_t k() const { return k_; }
    int32_t n_verifiers() const { return static_cast<int32_t>(s_.size()) - 1; }

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
    struct Mean {
        double sum = 0.0;
        uint64_t n = 0;
        void add(double x) { sum += x, ++n; }
        double mean() const { return n ? sum / n : NAN; }
    };
    int32_t k_;
    std::deque<Ret> q_in_;
    std::vector<double> waits_;
    std::vector<std::pair<double, double>> busy_;
    std::vector<Mean> s_, z_;
    Mean s_all_, z_all_;
    std::vector<int64_t> acc_, tests_;
    bool count_ = true;
};

static double host_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ---- Sec. 4 analytics (NEXT-4) ------------------------------------------------------------
// E[l_i] = beta_i (1 - beta_i^d) / (1 - beta_i)       Eq. (3), P:156-160 (d at beta = 1)
// E[l]_gamma = sum_i E[l_i]                             Eq. (4)
// T_idle = max(0, Z - (N - 1) S)                         Eq. (9)
// T_gamma = N S + T_idle                                 Eq. (10)
// O_gamma = E[l]_gamma / T_gamma, O^(i) = E[l_i] / T_gamma     Eq. (11)
// N_full = ceil(Z / S) + 1
// N_max = the largest N with O^(i)(N) >= o_alone, the standalone speed of a target
static double expected_accept(double beta, int32_t d) {
    if (!(beta < 1.0)) return d;
    if (!(beta > 0.0)) return 0.0;
    return beta * (1.0 - std::pow(beta, d)) / (1.0 - beta);
}

static void predict(int32_t n, const double* beta, int32_t d, double S, double Z, double o_alone,
                    sd_star_prediction* out) {
    *out = sd_star_prediction{};
    double el = 0.0, el_min = INFINITY;
    for (int32_t i = 0; i < n; ++i) {
        const double e = expected_accept(beta[i], d);
        el += e;
        el_min = std::min(el_min, e);
    }
    out->expected_accepted = el;
    out->t_idle_ms = std::max(0.0, Z - (n - 1) * S);
    out->t_gamma_ms = n * S + out->t_idle_ms;
    out->throughput_per_ms = out->t_gamma_ms > 0 ? el / out->t_gamma_ms : 0.0;
    out->per_target_min_per_ms = n > 0 && out->t_gamma_ms > 0 ? el_min / out->t_gamma_ms : 0.0;
    out->busy_fraction = out->t_gamma_ms > 0 ? n * S / out->t_gamma_ms : 0.0;
    out->n_full = S > 0 ? static_cast<int32_t>(std::ceil(Z / S)) + 1 : 1;
    // N_max with the mean per-target progress (homogeneous view of the active set)
    const double e_mean = n > 0 ? el / n : 0.0;
    int32_t nmax = 0;
    for (int32_t m = 1; m <= 4096; ++m) {
        const double tg = m * S + std::max(0.0, Z - (m - 1) * S);
        if (tg > 0 && e_mean / tg >= o_alone) nmax = m;
        else if (m * S >= Z + S) break;   // fully loaded: O^(i) only decreases from here on
    }
    out->n_max = nmax;
}

}  // namespace sd

using namespace sd;

struct sd_sched {
    StarScheduler s;
    uint64_t served = 0;
};

extern "C" {

sd_status sd_star_analytics(int32_t n, const double* beta, int32_t d, double service_ms,
                            double return_ms, double o_alone_per_ms, sd_star_prediction* out) {
    clear_error();
    if (n < 1 || !beta || d < 1 || !(service_ms > 0.0) || !(return_ms >= 0.0) ||
        !(o_alone_per_ms >= 0.0) || !out)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_analytics: bad argument");
    predict(n, beta, d, service_ms, return_ms, o_alone_per_ms, out);
    return SD_OK;
}

// Host-only scheduler handle: the same StarScheduler the NCCL star runs, for callers that bring
// their own transport (tests: a gloo cross-process star).
sd_status sd_sched_create(sd_sched** out, int32_t n_verifiers, int32_t k) {
    clear_error();
    if (!out || n_verifiers < 1 || k < 1 || k > SD_MAX_K)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_sched_create: bad argument");
    *out = new sd_sched{StarScheduler(n_verifiers, k), 0};
    return SD_OK;
}
sd_status sd_sched_push(sd_sched* h, int32_t verifier, int32_t slot, uint64_t round, double t_ms) {
    clear_error();
    if (!h || verifier < 1 || verifier > h->s.n_verifiers() || slot < 0)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_sched_push: bad argument");
    h->s.push_return(Ret{verifier, slot, round, t_ms});
    return SD_OK;
}
sd_status sd_sched_pop(sd_sched* h, double now_ms, int32_t* verifier, int32_t* slot,
                       uint64_t* round) {
    clear_error();
    if (!h || !verifier || !slot || !round) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    Ret r;
    if (!h->s.pop(&r, now_ms)) return SD_ERR_NOT_READY;
    *verifier = r.v;
    *slot = r.slot;
    *round = r.round;
    ++h->served;
    return SD_OK;
}
sd_status sd_sched_service(sd_sched* h, int32_t verifier, double t0_ms, double t1_ms) {
    clear_error();
    if (!h || !(t1_ms >= t0_ms)) return fail(SD_ERR_INVALID_ARGUMENT, "sd_sched_service");
    h->s.busy(t0_ms, t1_ms);
    h->s.observe_service(verifier, t1_ms - t0_ms);
    return SD_OK;
}
sd_status sd_sched_observe(sd_sched* h, int32_t verifier, double return_ms,
                           const int32_t* accept_len, int32_t n) {
    clear_error();
    if (!h || verifier < 1 || verifier > h->s.n_verifiers() || (n > 0 && !accept_len))
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_sched_observe");
    if (return_ms >= 0.0) h->s.observe_return(verifier, return_ms);
    if (n > 0) h->s.observe_accepts(verifier, accept_len, n);
    return SD_OK;
}
sd_status sd_sched_stats(sd_sched* h, sd_star_stats_t* out) {
    clear_error();
    if (!h || !out) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    *out = h->s.stats(h->served);
    return SD_OK;
}
sd_status sd_sched_predict(sd_sched* h, double o_alone_per_ms, sd_star_prediction* out) {
    clear_error();
    if (!h || !out) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    const int32_t n = h->s.n_verifiers();
    std::vector<double> beta(n);
    double S = 0.0, Z = 0.0;
    int32_t ns = 0;
    for (int32_t v = 1; v <= n; ++v) {
        beta[v - 1] = h->s.beta_hat(v);
        if (std::isnan(beta[v - 1])) return fail(SD_ERR_NOT_READY, "no accept lengths observed for verifier %d", v);
    }
    S = h->s.mean_S(0);
    Z = h->s.mean_Z(0);
    (void)ns;
    if (!(S > 0.0) || !(Z >= 0.0)) return fail(SD_ERR_NOT_READY, "no service / return observed yet");
    predict(n, beta.data(), h->s.k(), S, Z, o_alone_per_ms, out);
    out->service_ms = S;
    out->return_ms = Z;
    return SD_OK;
}
sd_status sd_sched_destroy(sd_sched* h) {
    delete h;
    return SD_OK;
}

// Deterministic fake transport driving the same scheduler (see include/starsd.h).
sd_status sd_star_simulate(int32_t n_verifiers, int32_t n_slots, double service_ms,
                           double return_ms, int32_t rounds, sd_star_stats_t* out) {
    clear_error();
    if (n_verifiers < 1 || n_slots < 1 || !(service_ms > 0.0) || !(return_ms >= 0.0) ||
        rounds < 1 || !out)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_simulate: bad argument");
    std::vector<double> S(n_verifiers, service_ms), Z(n_verifiers, return_ms);
    return sd_star_simulate_ex(n_verifiers, n_slots, S.data(), Z.data(), rounds, nullptr, out);
}

// Heterogeneous version: per-verifier service S_v and return Z_v; per-verifier completed rounds
// (the per-target progress rate of Eq. 11) in rounds_out[v-1] if non-NULL.
sd_status sd_star_simulate_ex(int32_t n_verifiers, int32_t n_slots, const double* service_ms,
                              const double* return_ms, int32_t rounds, uint64_t* rounds_out,
                              sd_star_stats_t* out) {
    clear_error();
    if (n_verifiers < 1 || n_slots < 1 || !service_ms || !return_ms || rounds < 1 || !out)
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_simulate_ex: bad argument");
    for (int32_t v = 0; v < n_verifiers; ++v)
        if (!(service_ms[v] > 0.0) || !(return_ms[v] >= 0.0))
            return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_simulate_ex: service/return of %d", v + 1);
    StarScheduler sched(n_verifiers, 1);
    // pending returns: (ready time, issue sequence) min-heap keeps FIFO order among ties
    using P = std::pair<std::pair<double, uint64_t>, Ret>;
    auto cmp = [](const P& a, const P& b) { return a.first > b.first; };
    std::priority_queue<P, std::vector<P>, decltype(cmp)> pending(cmp);
    uint64_t seq = 0;
    std::vector<uint64_t> per(n_verifiers, 0);
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
        t += service_ms[r.v - 1];            // S(d) = d t_s
        sched.busy(t0, t);
        if (i >= warm) ++per[r.v - 1];
        Ret nx{r.v, r.slot, r.round + 1, t + return_ms[r.v - 1]};   // Z(d) = t_c + t_v later
        pending.push(P{{nx.t_ready, seq++}, nx});
    }
    *out = sched.stats(static_cast<uint64_t>(rounds));
    if (rounds_out)
        for (int32_t v = 0; v < n_verifiers; ++v) rounds_out[v] = per[v];
    return SD_OK;
}

}  // extern "C"

// ---- NCCL transport -------------------------------------------------------------------------
#ifdef SD_WITH_NCCL

struct sd_star {
    sd_star_config cfg{};
    int esz = 4;
    bool loop = false;                       // SD_STAR_LOOPBACK
    bool dead = false;                       // communicators aborted (timeout / NCCL error)
    bool qm = false;                         // SD_STAR_PAYLOAD_QMETA
    std::vector<void*> qstage;               // draft, NCCL + QMETA: per (v, slot) q rows, IPC-exported
    std::vector<void*> qpeer;                // verifier, QMETA: the draft's staging, IPC-mapped
    std::vector<void*> qmeta_buf;            // verifier, QMETA: received sd_qmeta [B][k] per slot
    // draft: index v (1..world-1); verifier: index 0.  down = draft -> verifier, up = back.
    std::vector<ncclComm_t> down, up;
    std::vector<cudaStream_t> sdown, sup;
    struct Slot {                            // draft: one per (verifier, slot)
        cudaEvent_t ev_ret = nullptr;
        bool busy = false;
        uint64_t round = 0, seq = 0;
        double t_issue = 0.0;
    };
    std::vector<Slot> slots;                 // [world * n_slots]
    uint64_t seq = 0;
    cudaEvent_t ev_ready = nullptr;
    cudaEvent_t ev_origin = nullptr;
    // verifier staging (receive targets) and verify workspace, one set per slot
    // (NCCL verifier: index slot; loopback: index v * n_slots + slot)
    std::vector<void*> q_buf;
    std::vector<int32_t*> ids_buf, L_buf, tok_buf;
    std::vector<void*> ws;
    std::vector<cudaEvent_t> ev_recv, ev_used, ev_sent;
    struct Pending {                         // verifier: rounds whose results are on the way back
        int32_t slot;
        uint64_t round;
        double t_issue;
    };
    std::deque<Pending> vpending;
    size_t ws_bytes = 0;
    // draft busy accounting: a ring of pre-created event pairs (no event creation on the draft's
    // hot loop); completed intervals are harvested into busy_ms
    std::vector<cudaEvent_t> ring_b, ring_e;
    std::vector<int32_t> ring_v;
    size_t ring_head = 0, ring_n = 0;
    bool open = false;
    int32_t open_v = 0;
    std::vector<std::pair<double, double>> busy_ms;
    StarScheduler sched;
    uint64_t served = 0;
};

static constexpr size_t kRing = 1024;

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

// Abort every communicator of the handle (a stuck peer must not hang the caller; P:486 is the
// paper's only fault analogue, delay injection).  The handle is unusable afterwards.
static void star_abort(sd_star* h) {
    if (h->dead) return;
    h->dead = true;
    for (auto c : h->down)
        if (c) ncclCommAbort(c);
    for (auto c : h->up)
        if (c) ncclCommAbort(c);
    std::fill(h->down.begin(), h->down.end(), nullptr);
    std::fill(h->up.begin(), h->up.end(), nullptr);
}

static sd_status check_async(sd_star* h) {
    for (auto* vec : {&h->down, &h->up})
        for (auto c : *vec) {
            if (!c) continue;
            ncclResult_t ae = ncclSuccess;
            if (ncclCommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess &&
                ae != ncclInProgress) {
                star_abort(h);
                return nccl_fail(ae, "async NCCL error (communicators aborted)");
            }
        }
    return SD_OK;
}

static sd_status alloc_staging(sd_star* h, int n) {
    const sd_shape& ms = h->cfg.max_shape;
    const size_t B = ms.batch, k = ms.k, V = ms.vocab;
    sd_status st = sd_verify_workspace_size(&ms, h->cfg.temperature, &h->ws_bytes);
    if (st != SD_OK) return st;
    for (int i = 0; i < n; ++i) {
        void *q = nullptr, *w = nullptr;
        int32_t *idb = nullptr, *lb = nullptr, *tb = nullptr;
        cudaEvent_t e0, e1, e2;
        if (!h->qm) SD_CUDA(cudaMalloc(&q, B * k * V * h->esz));   // (QMETA: no q rows arrive)
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&idb), B * k * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&lb), B * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&tb), B * (k + 1) * sizeof(int32_t)));
        SD_CUDA(cudaMalloc(&w, h->ws_bytes));
        SD_CUDA(cudaMemset(w, 0, h->ws_bytes));
        if (h->qm) {
            void* m = nullptr;
            SD_CUDA(cudaMalloc(&m, B * k * sizeof(sd_qmeta)));
            h->qmeta_buf.push_back(m);
        }
        SD_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
        SD_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        SD_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        h->q_buf.push_back(q);
        h->ids_buf.push_back(idb);
        h->L_buf.push_back(lb);
        h->tok_buf.push_back(tb);
        h->ws.push_back(w);
        h->ev_recv.push_back(e0);
        h->ev_used.push_back(e1);
        h->ev_sent.push_back(e2);
    }
    return SD_OK;
}

static sd_status star_init(sd_star* h, const void* ids);
static sd_status exchange_qstage(sd_star* h);

static ncclDataType_t nccl_dtype(sd_dtype d) { return d == SD_DTYPE_F32 ? ncclFloat32 : ncclBfloat16; }

extern "C" {

sd_status sd_star_unique_ids(int32_t world, void* ids_out) {
    clear_error();
    if (world < 2 || !ids_out) return fail(SD_ERR_INVALID_ARGUMENT, "world < 2 or ids_out NULL");
    static_assert(sizeof(ncclUniqueId) == SD_STAR_ID_BYTES, "ncclUniqueId size");
    for (int32_t i = 0; i < 2 * (world - 1); ++i) {   // (down, up) per pair
        ncclUniqueId id;
        SD_NCCL(ncclGetUniqueId(&id));
        memcpy(static_cast<char*>(ids_out) + i * SD_STAR_ID_BYTES, &id, SD_STAR_ID_BYTES);
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
    h->qm = cfg->payload == SD_STAR_PAYLOAD_QMETA;
    if (cfg->payload != SD_STAR_PAYLOAD_FULL && cfg->payload != SD_STAR_PAYLOAD_QMETA) {
        delete h;
        return fail(SD_ERR_INVALID_ARGUMENT, "payload");
    }
    h->sched = StarScheduler(cfg->world - 1, cfg->max_shape.k);
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
        h->down.assign(cfg->world, nullptr);
        h->up.assign(cfg->world, nullptr);
        h->sdown.assign(cfg->world, nullptr);
        h->sup.assign(cfg->world, nullptr);
        if (!h->loop) {
            SD_NCCL(ncclGroupStart());
            for (int v = 1; v < cfg->world; ++v) {
                SD_NCCL(ncclCommInitRank(&h->down[v], 2, uid[2 * (v - 1)], 0));
                SD_NCCL(ncclCommInitRank(&h->up[v], 2, uid[2 * (v - 1) + 1], 0));
            }
            SD_NCCL(ncclGroupEnd());
        } else {
            st = alloc_staging(h, cfg->world * cfg->n_slots);
            if (st != SD_OK) return st;
        }
        for (int v = 1; v < cfg->world; ++v) {
            SD_CUDA(cudaStreamCreateWithFlags(&h->sdown[v], cudaStreamNonBlocking));
            SD_CUDA(cudaStreamCreateWithFlags(&h->sup[v], cudaStreamNonBlocking));
        }
        h->slots.resize(static_cast<size_t>(cfg->world) * cfg->n_slots);
        for (auto& s : h->slots) SD_CUDA(cudaEventCreateWithFlags(&s.ev_ret, cudaEventDisableTiming));
        h->ring_b.resize(kRing);
        h->ring_e.resize(kRing);
        h->ring_v.resize(kRing);
        for (size_t i = 0; i < kRing; ++i) {
            SD_CUDA(cudaEventCreate(&h->ring_b[i]));
            SD_CUDA(cudaEventCreate(&h->ring_e[i]));
        }
    } else {
        h->down.assign(1, nullptr);
        h->up.assign(1, nullptr);
        h->sdown.assign(1, nullptr);
        h->sup.assign(1, nullptr);
        SD_NCCL(ncclGroupStart());
        SD_NCCL(ncclCommInitRank(&h->down[0], 2, uid[2 * (cfg->rank - 1)], 1));
        SD_NCCL(ncclCommInitRank(&h->up[0], 2, uid[2 * (cfg->rank - 1) + 1], 1));
        SD_NCCL(ncclGroupEnd());
        SD_CUDA(cudaStreamCreateWithFlags(&h->sdown[0], cudaStreamNonBlocking));
        SD_CUDA(cudaStreamCreateWithFlags(&h->sup[0], cudaStreamNonBlocking));
        st = alloc_staging(h, cfg->n_slots);
        if (st != SD_OK) return st;
    }
    if (h->qm && !h->loop) {
        st = exchange_qstage(h);
        if (st != SD_OK) return st;
    }
    SD_CUDA(cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
    SD_CUDA(cudaEventCreate(&h->ev_origin));
    SD_CUDA(cudaEventRecord(h->ev_origin, 0));
    return SD_OK;
}

// QMETA payload over NCCL: the draft allocates one q staging buffer per (verifier, slot) and sends
// its CUDA IPC handle to the verifier once (the one-time handshake of P:262-263); the verifier maps
// it and its sd_verify_qmeta reads the stop rows q_L over NVLink.  Per round only ids + metadata
// travel through NCCL.
static sd_status exchange_qstage(sd_star* h) {
    const sd_star_config* cfg = &h->cfg;
    const sd_shape& ms = cfg->max_shape;
    const size_t qbytes = (size_t)ms.batch * ms.k * ms.vocab * h->esz;
    const size_t hb = sizeof(cudaIpcMemHandle_t) * cfg->n_slots;
    void* dbuf = nullptr;
    SD_CUDA(cudaMalloc(&dbuf, hb));
    std::vector<cudaIpcMemHandle_t> hs(cfg->n_slots);
    if (cfg->rank == 0) {
        h->qstage.assign(static_cast<size_t>(cfg->world) * cfg->n_slots, nullptr);
        for (int v = 1; v < cfg->world; ++v) {
            for (int s = 0; s < cfg->n_slots; ++s) {
                void*& q = h->qstage[static_cast<size_t>(v) * cfg->n_slots + s];
                SD_CUDA(cudaMalloc(&q, qbytes));
                SD_CUDA(cudaIpcGetMemHandle(&hs[s], q));
            }
            SD_CUDA(cudaMemcpy(dbuf, hs.data(), hb, cudaMemcpyHostToDevice));
            SD_NCCL(ncclSend(dbuf, hb, ncclInt8, 1, h->down[v], h->sdown[v]));
            SD_CUDA(cudaStreamSynchronize(h->sdown[v]));
        }
    } else {
        SD_NCCL(ncclRecv(dbuf, hb, ncclInt8, 0, h->down[0], h->sdown[0]));
        SD_CUDA(cudaStreamSynchronize(h->sdown[0]));
        SD_CUDA(cudaMemcpy(hs.data(), dbuf, hb, cudaMemcpyDeviceToHost));
        h->qpeer.assign(cfg->n_slots, nullptr);
        for (int s = 0; s < cfg->n_slots; ++s)
            SD_CUDA(cudaIpcOpenMemHandle(&h->qpeer[s], hs[s], cudaIpcMemLazyEnablePeerAccess));
    }
    SD_CUDA(cudaFree(dbuf));
    return SD_OK;
}

// busy ring: move completed intervals (or, with wait, the oldest one) into busy_ms
static sd_status harvest(sd_star* h, bool wait_oldest, bool all) {
    while (h->ring_n > 0) {
        const size_t tail = (h->ring_head + kRing - h->ring_n) % kRing;
        if (wait_oldest || all) {
            SD_CUDA(cudaEventSynchronize(h->ring_e[tail]));
            wait_oldest = false;
        } else {
            const cudaError_t e = cudaEventQuery(h->ring_e[tail]);
            if (e == cudaErrorNotReady) break;
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventQuery");
        }
        float a = 0.f, b = 0.f;
        SD_CUDA(cudaEventElapsedTime(&a, h->ev_origin, h->ring_b[tail]));
        SD_CUDA(cudaEventElapsedTime(&b, h->ev_origin, h->ring_e[tail]));
        h->busy_ms.emplace_back(a, b);
        h->sched.observe_service(h->ring_v[tail], static_cast<double>(b) - a);
        --h->ring_n;
    }
    return SD_OK;
}

extern "C" {

sd_status sd_star_round(sd_star* h, const sd_round_desc* d, cudaStream_t stream) {
    clear_error();
    if (!h || !d) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    if (h->dead) return fail(SD_ERR_NCCL, "star handle aborted (timeout or NCCL error)");
    const sd_shape& ms = h->cfg.max_shape;
    if (d->batch < 1 || d->batch > ms.batch || d->slot < 0 || d->slot >= h->cfg.n_slots)
        return fail(SD_ERR_INVALID_ARGUMENT, "batch / slot out of range");
    if (!d->out_accept_len || !d->out_tokens)
        return fail(SD_ERR_INVALID_ARGUMENT, "out_accept_len / out_tokens NULL");
    const size_t B = d->batch, k = ms.k, V = ms.vocab;
    const ncclDataType_t dt = nccl_dtype(ms.dtype);
    const bool greedy = h->cfg.temperature == 0.0f;
    sd_shape sh = ms;
    sh.batch = d->batch;   // (the verify workspace of a slot re-zeroes itself on a batch change)
    if (h->cfg.rank == 0) {
        // draft: ship ids + q (sender), post the receive of the verified prefix
        const int v = d->verifier;
        if (v < 1 || v >= h->cfg.world) return fail(SD_ERR_INVALID_ARGUMENT, "verifier");
        if (!d->draft_ids || (!greedy && !d->q_logits))
            return fail(SD_ERR_INVALID_ARGUMENT, "draft_ids / q_logits NULL");
        if (h->qm && !greedy && !d->q_meta)
            return fail(SD_ERR_INVALID_ARGUMENT, "QMETA payload: q_meta NULL");
        sd_star::Slot& s = h->slots[static_cast<size_t>(v) * h->cfg.n_slots + d->slot];
        if (s.busy) return fail(SD_ERR_INVALID_ARGUMENT, "slot still in flight");
        SD_CUDA(cudaEventRecord(h->ev_ready, stream));
        SD_CUDA(cudaStreamWaitEvent(h->sdown[v], h->ev_ready, 0));
        if (h->loop) {
            // the same exchange as D2D copies on the pair's streams; the virtual verifier's
            // recv -> verify -> send runs there too
            if (!d->p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "loopback: p_logits NULL");
            const size_t i = static_cast<size_t>(v) * h->cfg.n_slots + d->slot;
            cudaStream_t cs = h->sdown[v];
            SD_CUDA(cudaMemcpyAsync(h->ids_buf[i], d->draft_ids, B * k * 4, cudaMemcpyDeviceToDevice, cs));
            if (!greedy && h->qm)
                SD_CUDA(cudaMemcpyAsync(h->qmeta_buf[i], d->q_meta, B * k * sizeof(sd_qmeta),
                                        cudaMemcpyDeviceToDevice, cs));
            else if (!greedy)
                SD_CUDA(cudaMemcpyAsync(h->q_buf[i], d->q_logits, B * k * V * h->esz,
                                        cudaMemcpyDeviceToDevice, cs));
            if (h->cfg.target_ms > 0.0f) SD_CUDA(launch_spin_ns(static_cast<uint64_t>(h->cfg.target_ms * 1e6), cs));
            // QMETA: the virtual verifier reads its stop rows straight from the draft's q_logits
            sd_status st = h->qm && !greedy
                ? sd_verify_qmeta(d->p_logits, d->q_logits, static_cast<const sd_qmeta*>(h->qmeta_buf[i]),
                                  h->ids_buf[i], &sh, h->cfg.temperature, h->cfg.seed, d->round,
                                  d->request_id_base, h->L_buf[i], h->tok_buf[i], nullptr, h->ws[i],
                                  h->ws_bytes, cs)
                : sd_verify(d->p_logits, greedy ? nullptr : h->q_buf[i], h->ids_buf[i], &sh,
                            h->cfg.temperature, h->cfg.seed, d->round, d->request_id_base,
                            h->L_buf[i], h->tok_buf[i], nullptr, h->ws[i], h->ws_bytes, cs);
            if (st != SD_OK) return st;
            SD_CUDA(cudaEventRecord(h->ev_used[i], cs));
            SD_CUDA(cudaStreamWaitEvent(h->sup[v], h->ev_used[i], 0));
            SD_CUDA(cudaMemcpyAsync(d->out_accept_len, h->L_buf[i], B * 4, cudaMemcpyDeviceToDevice, h->sup[v]));
            SD_CUDA(cudaMemcpyAsync(d->out_tokens, h->tok_buf[i], B * (k + 1) * 4,
                                    cudaMemcpyDeviceToDevice, h->sup[v]));
        } else {
            const size_t i = static_cast<size_t>(v) * h->cfg.n_slots + d->slot;
            if (h->qm && !greedy && d->q_logits != h->qstage[i])   // stop rows are read from here
                SD_CUDA(cudaMemcpyAsync(h->qstage[i], d->q_logits, B * k * V * h->esz,
                                        cudaMemcpyDeviceToDevice, h->sdown[v]));
            SD_NCCL(ncclGroupStart());
            SD_NCCL(ncclSend(d->draft_ids, B * k, ncclInt32, 1, h->down[v], h->sdown[v]));
            if (!greedy && h->qm)
                SD_NCCL(ncclSend(d->q_meta, B * k * sizeof(sd_qmeta), ncclInt8, 1, h->down[v], h->sdown[v]));
            else if (!greedy)
                SD_NCCL(ncclSend(d->q_logits, B * k * V, dt, 1, h->down[v], h->sdown[v]));
            SD_NCCL(ncclGroupEnd());
            SD_NCCL(ncclGroupStart());
            SD_NCCL(ncclRecv(d->out_accept_len, B, ncclInt32, 1, h->up[v], h->sup[v]));
            SD_NCCL(ncclRecv(d->out_tokens, B * (k + 1), ncclInt32, 1, h->up[v], h->sup[v]));
            SD_NCCL(ncclGroupEnd());
        }
        SD_CUDA(cudaEventRecord(s.ev_ret, h->sup[v]));
        s.busy = true;
        s.round = d->round;
        s.seq = h->seq++;
        s.t_issue = host_ms();
        return SD_OK;
    }
    // verifier: recv (down stream) -> verify (`stream`) -> send (up stream)
    if (!d->p_logits) return fail(SD_ERR_INVALID_ARGUMENT, "p_logits NULL");
    const int sl = d->slot;
    void* q = h->q_buf[sl];
    int32_t* ids = h->ids_buf[sl];
    // the slot's staging is free once its previous verify has read it
    SD_CUDA(cudaStreamWaitEvent(h->sdown[0], h->ev_used[sl], 0));
    SD_NCCL(ncclGroupStart());
    SD_NCCL(ncclRecv(ids, B * k, ncclInt32, 0, h->down[0], h->sdown[0]));
    if (!greedy && h->qm)
        SD_NCCL(ncclRecv(h->qmeta_buf[sl], B * k * sizeof(sd_qmeta), ncclInt8, 0, h->down[0], h->sdown[0]));
    else if (!greedy)
        SD_NCCL(ncclRecv(q, B * k * V, dt, 0, h->down[0], h->sdown[0]));
    SD_NCCL(ncclGroupEnd());
    SD_CUDA(cudaEventRecord(h->ev_recv[sl], h->sdown[0]));
    SD_CUDA(cudaStreamWaitEvent(stream, h->ev_recv[sl], 0));
    if (h->cfg.target_ms > 0.0f) SD_CUDA(launch_spin_ns(static_cast<uint64_t>(h->cfg.target_ms * 1e6), stream));
    sd_status st = h->qm && !greedy
        ? sd_verify_qmeta(d->p_logits, h->qpeer[sl], static_cast<const sd_qmeta*>(h->qmeta_buf[sl]),
                          ids, &sh, h->cfg.temperature, h->cfg.seed, d->round, d->request_id_base,
                          d->out_accept_len, d->out_tokens, nullptr, h->ws[sl], h->ws_bytes, stream)
        : sd_verify(d->p_logits, greedy ? nullptr : q, ids, &sh, h->cfg.temperature, h->cfg.seed,
                    d->round, d->request_id_base, d->out_accept_len, d->out_tokens, nullptr,
                    h->ws[sl], h->ws_bytes, stream);
    if (st != SD_OK) return st;
    SD_CUDA(cudaEventRecord(h->ev_used[sl], stream));
    SD_CUDA(cudaStreamWaitEvent(h->sup[0], h->ev_used[sl], 0));
    SD_NCCL(ncclGroupStart());
    SD_NCCL(ncclSend(d->out_accept_len, B, ncclInt32, 0, h->up[0], h->sup[0]));
    SD_NCCL(ncclSend(d->out_tokens, B * (k + 1), ncclInt32, 0, h->up[0], h->sup[0]));
    SD_NCCL(ncclGroupEnd());
    SD_CUDA(cudaEventRecord(h->ev_sent[sl], h->sup[0]));
    h->vpending.push_back(sd_star::Pending{sl, d->round, host_ms()});
    return SD_OK;
}

sd_status sd_star_poll(sd_star* h, int32_t* verifier, int32_t* slot, uint64_t* round,
                       int32_t timeout_us) {
    clear_error();
    if (!h || !verifier || !slot || !round) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    if (h->dead) return fail(SD_ERR_NCCL, "star handle aborted (timeout or NCCL error)");
    const double t_end = host_ms() + timeout_us / 1000.0;
    const double tmo = h->cfg.timeout_ms;
    while (true) {
        const double now = host_ms();
        if (h->cfg.rank != 0) {
            // verifier: the oldest round whose results have left (its send completed)
            if (!h->vpending.empty()) {
                const sd_star::Pending p = h->vpending.front();
                const cudaError_t e = cudaEventQuery(h->ev_sent[p.slot]);
                if (e == cudaSuccess) {
                    h->vpending.pop_front();
                    *verifier = h->cfg.rank;
                    *slot = p.slot;
                    *round = p.round;
                    return SD_OK;
                }
                if (e != cudaErrorNotReady) return cuda_fail(e, "cudaEventQuery");
                if (tmo > 0 && now - p.t_issue > tmo) {
                    star_abort(h);
                    return fail(SD_ERR_TIMEOUT, "verifier round %llu (slot %d) not done in %d ms: "
                                "communicators aborted", (unsigned long long)p.round, p.slot,
                                h->cfg.timeout_ms);
                }
            }
        } else {
            // receiver: move completed returns into Q_in in issue order
            std::vector<std::pair<uint64_t, size_t>> done;
            for (size_t i = 0; i < h->slots.size(); ++i) {
                sd_star::Slot& s = h->slots[i];
                if (!s.busy) continue;
                const cudaError_t e = cudaEventQuery(s.ev_ret);
                if (e == cudaSuccess) done.emplace_back(s.seq, i);
                else if (e != cudaErrorNotReady) return cuda_fail(e, "cudaEventQuery");
                else if (tmo > 0 && now - s.t_issue > tmo) {
                    star_abort(h);
                    return fail(SD_ERR_TIMEOUT, "verifier %d slot %d round %llu not back in %d ms: "
                                "communicators aborted", static_cast<int>(i / h->cfg.n_slots),
                                static_cast<int>(i % h->cfg.n_slots),
                                (unsigned long long)s.round, h->cfg.timeout_ms);
                }
            }
            std::sort(done.begin(), done.end());
            for (auto& p : done) {
                sd_star::Slot& s = h->slots[p.second];
                s.busy = false;
                const int32_t v = static_cast<int32_t>(p.second / h->cfg.n_slots);
                h->sched.push_return(Ret{v, static_cast<int32_t>(p.second % h->cfg.n_slots), s.round, now});
                h->sched.observe_return(v, now - s.t_issue);   // Z(d) = t_c + t_v (Eq. 6)
            }
            Ret r;
            if (h->sched.pop(&r, now)) {
                *verifier = r.v;
                *slot = r.slot;
                *round = r.round;
                ++h->served;
                return SD_OK;
            }
        }
        if (!h->loop) {
            const sd_status a = check_async(h);
            if (a != SD_OK) return a;
        }
        if (timeout_us <= 0) return SD_ERR_NOT_READY;
        if (host_ms() >= t_end) return fail(SD_ERR_TIMEOUT, "no return within %d us", timeout_us);
        std::this_thread::yield();
    }
}

sd_status sd_star_observe(sd_star* h, int32_t verifier, const int32_t* accept_len_host, int32_t n) {
    clear_error();
    if (!h || h->cfg.rank != 0 || verifier < 1 || verifier >= h->cfg.world || (n > 0 && !accept_len_host))
        return fail(SD_ERR_INVALID_ARGUMENT, "sd_star_observe: draft only, host accept lengths");
    h->sched.observe_accepts(verifier, accept_len_host, n);
    return SD_OK;
}

sd_status sd_star_predict(sd_star* h, double o_alone_per_ms, sd_star_prediction* out) {
    clear_error();
    if (!h || !out || h->cfg.rank != 0) return fail(SD_ERR_INVALID_ARGUMENT, "draft only");
    sd_status s = harvest(h, false, true);
    if (s != SD_OK) return s;
    sd_sched tmp{h->sched, h->served};
    return sd_sched_predict(&tmp, o_alone_per_ms, out);
}

sd_status sd_star_draft_begin(sd_star* h, cudaStream_t stream) {
    return sd_star_draft_begin_v(h, 0, stream);
}

sd_status sd_star_draft_begin_v(sd_star* h, int32_t verifier, cudaStream_t stream) {
    clear_error();
    if (!h || h->cfg.rank != 0) return fail(SD_ERR_INVALID_ARGUMENT, "draft-only");
    if (h->open) return fail(SD_ERR_INVALID_ARGUMENT, "draft_begin without draft_end");
    sd_status s = harvest(h, h->ring_n == kRing, false);   // ring full: wait for the oldest
    if (s != SD_OK) return s;
    SD_CUDA(cudaEventRecord(h->ring_b[h->ring_head], stream));
    h->open = true;
    h->open_v = verifier;
    return SD_OK;
}

sd_status sd_star_draft_end(sd_star* h, cudaStream_t stream) {
    clear_error();
    if (!h || h->cfg.rank != 0 || !h->open)
        return fail(SD_ERR_INVALID_ARGUMENT, "draft_end without draft_begin");
    SD_CUDA(cudaEventRecord(h->ring_e[h->ring_head], stream));
    h->ring_v[h->ring_head] = h->open_v;
    h->ring_head = (h->ring_head + 1) % kRing;
    ++h->ring_n;
    h->open = false;
    return harvest(h, false, false);
}

sd_status sd_star_stats(sd_star* h, sd_star_stats_t* out) {
    clear_error();
    if (!h || !out) return fail(SD_ERR_INVALID_ARGUMENT, "NULL argument");
    if (h->cfg.rank == 0) {
        sd_status s = harvest(h, false, true);
        if (s != SD_OK) return s;
    }
    StarScheduler s;          // busy timeline from the CUDA events (device clock)
    for (auto& p : h->busy_ms) s.busy(p.first, p.second);
    *out = s.stats(h->served);
    const sd_star_stats_t q = h->sched.stats(h->served);
    out->mean_wait_ms = q.mean_wait_ms;      // queueing wait is measured on the host clock
    return SD_OK;
}

sd_status sd_star_destroy(sd_star* h) {
    clear_error();
    if (!h) return SD_OK;
    for (auto* vec : {&h->down, &h->up})
        for (auto c : *vec)
            if (c) ncclCommDestroy(c);
    for (auto* vec : {&h->sdown, &h->sup})
        for (auto s : *vec)
            if (s) cudaStreamDestroy(s);
    for (auto& s : h->slots)
        if (s.ev_ret) cudaEventDestroy(s.ev_ret);
    for (auto e : h->ring_b) cudaEventDestroy(e);
    for (auto e : h->ring_e) cudaEventDestroy(e);
    for (auto* vec : {&h->ev_recv, &h->ev_used, &h->ev_sent})
        for (auto e : *vec) cudaEventDestroy(e);
    for (auto q : h->q_buf) cudaFree(q);
    for (auto i : h->ids_buf) cudaFree(i);
    for (auto i : h->L_buf) cudaFree(i);
    for (auto i : h->tok_buf) cudaFree(i);
    for (auto w : h->ws) cudaFree(w);
    for (auto p : h->qpeer)
        if (p) cudaIpcCloseMemHandle(p);
    for (auto p : h->qstage)
        if (p) cudaFree(p);
    for (auto p : h->qmeta_buf) cudaFree(p);
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
sd_status sd_star_observe(sd_star*, int32_t, const int32_t*, int32_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_predict(sd_star*, double, sd_star_prediction*) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_draft_begin(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_draft_begin_v(sd_star*, int32_t, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_draft_end(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_stats(sd_star*, sd_star_stats_t*) { return fail(SD_ERR_UNSUPPORTED, "built without NCCL"); }
sd_status sd_star_destroy(sd_star*) { return SD_OK; }
}

#endif
