// verify_fused.cu -- alternative sm_100a verify kernel: ONE persistent launch per call
// (selected with STARSD_KERNEL=fused; the default two-launch path in verify_kernels.cu measured
// faster on every BASELINE config -- see DESIGN.md "Kernel variants").
//
// Method (Alg. 2, readings C-1..C-12 of DESIGN.md), per request b:
//   accept x_j iff u_acc(j) < min(1, p_j(x_j)/q_j(x_j)); L = first rejection (else k);
//   emit x_0..x_{L-1}, then t ~ norm(max(0, p_L - q_L)) (L < k) or t ~ p_k (L == k).
//
// Structure:
//   * grid = one CTA per SM (cooperative launch: all CTAs co-resident), 9 warps per CTA:
//     warp 8 = producer (TMA bulk copies into a 12-stage shared-memory ring, mbarriers),
//     warps 0-7 = consumers, each owning whole items (item n is consumed by warp n % 8).
//   * phase 1 items = (position j, request b, vocab chunk c) in POSITION-MAJOR order, dealt
//     round-robin to CTAs.  A consumer warp computes the chunk's max and sum of
//     2^((z - m) log2e / T) for p_j and q_j (one MUFU.EX2 per element, fp64 sums), publishes
//     them, and takes a per-row ticket; the warp that completes a row combines the chunks
//     (fp64), draws u_acc from Philox and decides the acceptance test.  The producer skips
//     the loads of rows after a known stop (laziness: rows after L are never needed).
//   * phase 2 items = the residual / bonus inverse-CDF pass over the stop row (re-read from
//     L2), pulled from a device work queue filled by the deciding warps.  The last chunk of a
//     pass searches chunk -> 128-token segment -> token.
//   * per-request event counters tell the last piece of work for a request to write its
//     outputs and leave the workspace zeroed; the last CTA to exit resets the queue.
// No tensor cores: the step is a streaming reduction, not a contraction.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "philox.cuh"
#include "ptx.cuh"
#include "verify.cuh"

namespace sd {
namespace fused {

constexpr int kConsumers = 12;                   // consumer warps
constexpr int kGroups = 3;                       // consumer groups; stage n belongs to group n % 3
constexpr int kGW = kConsumers / kGroups;        // warps per group (all work on each group stage)
constexpr int kProducerWarp = kConsumers;        // TMA producer
constexpr int kMonitorWarp = kConsumers + 1;     // mirrors global state into shared memory
constexpr int kEpilogueWarp = kConsumers + 2;    // publishes finished stages, takes tickets
constexpr int kDeciderWarp = kConsumers + 3;     // decides completed rows, searches passes
constexpr int kThreadsF = 32 * (kConsumers + 4);   // 512 threads: 128 registers each
constexpr int kEq = 64;                          // epilogue -> decider event queue
constexpr int kTraceWarps = kConsumers + 4;
constexpr int kMaxB = 4096;                      // stop-mask mirror capacity (max batch)
constexpr int kR = 16;                           // result ring between consumers and epilogue
constexpr int kMq = 256;                         // shared-memory queue of ready mailbox entries
constexpr int kStages = 6;                       // ring depth; a multiple of kGroups, so a slot
                                                 // always belongs to the same group (no mbarrier
                                                 // parity aliasing across groups)
constexpr int kRowChunkBytes = 16384;            // one row's slice per item: 16 KB bulk copies
                                                 // (8 KB copies cap at ~3.8 TB/s on B200,
                                                 // 16 KB reach ~7.3 TB/s: tools/stream_bench)
constexpr int kStageBytes = 2 * kRowChunkBytes;  // p slice + q slice
constexpr int kSegs = 32;                        // 32-lane-vector segments per chunk
constexpr uint32_t kValid = 0x80000000u;        // mailbox entry: valid
constexpr uint32_t kMsg = 0x40000000u;          // mailbox entry: message for the decider
constexpr uint32_t kMsgDecide = 1u, kMsgSearch = 2u;
constexpr uint32_t kSkipArrive = 1u | (1u << 16);

// status bits (values of include/starsd.h SD_FAULT_*)
constexpr int32_t kBadId = 1, kNonfinite = 2, kEmptyRow = 4, kZeroQ = 8, kZeroResidual = 16;
constexpr int32_t kHard = kBadId | kNonfinite | kEmptyRow;

static_assert(kRowChunkBytes == kRowChunkBytesH && kSegs == kSegsH, "verify.cuh out of sync");
static_assert(kStages % kGroups == 0 && kConsumers % kGroups == 0, "group geometry");


enum : int32_t { kItemStats = 1, kItemSkip = 2, kItemResid = 3, kItemStop = 4 };

struct Meta {
    int32_t type, b, j, c;
};

// ---- element types ----------------------------------------------------------------------
template <typename E>
struct Vec;
template <>
struct Vec<float> {
    static constexpr int N = 4;
    __device__ static void unpack(const uint4 u, float (&v)[4]) {
        v[0] = __uint_as_float(u.x);
        v[1] = __uint_as_float(u.y);
        v[2] = __uint_as_float(u.z);
        v[3] = __uint_as_float(u.w);
    }
    __device__ static float one(const void* base, int64_t i) {
        return static_cast<const float*>(base)[i];
    }
};
template <>
struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ static void unpack(const uint4 u, float (&v)[8]) {
        v[0] = __uint_as_float(u.x << 16);
        v[1] = __uint_as_float(u.x & 0xFFFF0000u);
        v[2] = __uint_as_float(u.y << 16);
        v[3] = __uint_as_float(u.y & 0xFFFF0000u);
        v[4] = __uint_as_float(u.z << 16);
        v[5] = __uint_as_float(u.z & 0xFFFF0000u);
        v[6] = __uint_as_float(u.w << 16);
        v[7] = __uint_as_float(u.w & 0xFFFF0000u);
    }
    __device__ static float one(const void* base, int64_t i) {
        return __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(base)[i]) << 16);
    }
};

// ---- small helpers ----------------------------------------------------------------------
// NaN-propagating max: a NaN anywhere in a row makes its max NaN (fault detection for free)
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float warp_max_nan(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, i, o);
        if (ov > v || (ov == v && oi < i)) {
            v = ov;
            i = oi;
        }
    }
}
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, n);
    }
    return v;
}
// 16 values per lane -> lane l holds the warp total of value (l >> 1) & 15 in v[0]
__device__ __forceinline__ void reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
    for (int K = 16, off = 16; K >= 2; K >>= 1, off >>= 1) {
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < K / 2; ++i) {
            const double send = hi ? v[i] : v[K / 2 + i];
            const double keep = hi ? v[K / 2 + i] : v[i];
            v[i] = __dadd_rn(keep, __shfl_xor_sync(0xFFFFFFFFu, send, off));
        }
    }
    v[0] = __dadd_rn(v[0], __shfl_xor_sync(0xFFFFFFFFu, v[0], 1));
}
template <typename T>
__device__ __forceinline__ T load_cg(const T* p) {
    static_assert(sizeof(T) % 8 == 0, "record must be a multiple of 8 bytes");
    T out;
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(p);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(&out);
#pragma unroll
    for (size_t i = 0; i < sizeof(T) / 8; ++i) d[i] = __ldcg(s + i);
    return out;
}
// acq_rel atomic add at gpu scope: orders this thread's earlier writes before the add and the
// caller's later reads after it (no separate __threadfence, which also invalidates L1)
__device__ __forceinline__ uint32_t atomic_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
                 : "memory");
    return old;
}
// release-only atomic add: orders this thread's earlier writes before the add without the
// L1 invalidation an acquire implies (readers use L2-coherent loads and fence themselves)
__device__ __forceinline__ uint32_t atomic_add_release(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
                 : "memory");
    return old;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// one probability term of the sampling pass: 2^((z - M) c2) / S in fp64 after the exp
__device__ __forceinline__ double prob_term(float z, float M, float c2, double invS) {
    return __dmul_rn(static_cast<double>(ex2_approx(__fmul_rn(__fsub_rn(z, M), c2))), invS);
}

__device__ __forceinline__ const void* row_p(const FParams& P, int b, int j, size_t esz) {
    return static_cast<const char*>(P.p) + ((int64_t)b * (P.k + 1) + j) * P.ld_p * esz;
}
__device__ __forceinline__ const void* row_q(const FParams& P, int b, int j, size_t esz) {
    return static_cast<const char*>(P.q) + ((int64_t)b * P.k + j) * P.ld_q * esz;
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace layout: [4 x grid] CTA start / producer phase-1 end / producer end / CTA exit,
// then [rows] decision time, [rows] sampling-pass end, [B] request completion
__device__ __forceinline__ void trace_at(const FParams& P, size_t i) {
    if (P.trace) P.trace[i] = gtime();
}
// per-warp cycle counters: [wait, work, items, extra] after the timeline
__device__ __forceinline__ void trace_warp(const FParams& P, int warp, const unsigned long long (&c)[4]) {
    if (!P.trace) return;
    const size_t base = 4 * gridDim.x + 2 * static_cast<size_t>(P.B) * (P.k + 1) + P.B;
    unsigned long long* o = P.trace + base + (static_cast<size_t>(blockIdx.x) * kTraceWarps + warp) * 4;
    for (int i = 0; i < 4; ++i) o[i] = c[i];
}

// ---- request completion ------------------------------------------------------------------
// Called by one lane after its work on request b is published.  The event that completes the
// request (all k+1 rows done and every spawned sampling pass done) writes the outputs.
__device__ void request_event(const FParams& P, int b, uint32_t delta) {
    const uint32_t old = atomic_add_acq_rel(P.evt + b, delta);
    const uint32_t nw = old + delta;
    const uint32_t rows = nw & 0xFFu, spawned = (nw >> 8) & 0xFFu, rdone = (nw >> 16) & 0xFFu;
    if (rows != static_cast<uint32_t>(P.k + 1) || rdone != spawned) return;
    const int kk = P.k;
    const uint32_t s = __ldcg(P.stop + b);
    const int L = s ? __ffs(static_cast<int>(s)) - 1 : kk;
    const size_t r = static_cast<size_t>(b) * (kk + 1) + L;
    const RowStat rs = load_cg(P.rowstat + r);
    const bool hard = (rs.status & kHard) != 0;
    int32_t status = rs.status;
    int32_t tok = -1;
    if (!hard) {
        const int2 cd = __ldcg(P.cand + r);
        tok = cd.x;
        status |= cd.y;
    }
    P.out_L[b] = hard ? 0 : L;
    int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
    for (int i = 0; i <= kk; ++i) {
        int32_t v = -1;
        if (!hard) v = i < L ? P.ids[static_cast<size_t>(b) * kk + i] : (i == L ? tok : -1);
        ot[i] = v;
    }
    if (P.out_status) P.out_status[b] = status;
    trace_at(P, 4 * gridDim.x + 2 * static_cast<size_t>(P.B) * (kk + 1) + b);
    P.evt[b] = 0u;
    P.stop[b] = 0u;
    atomic_add_acq_rel(P.glob + 2, 1u);
}

// ---- phase 1: per-chunk statistics -----------------------------------------------------
// lane partial over the chunk held in shared memory: NaN-propagating max, then
// sum 2^((z - m) c2) with the lane max m (fp32 per vector, fp64 across vectors).  Four
// vectors per iteration with independent accumulators (the warp is latency-bound otherwise).
template <typename E>
__device__ __forceinline__ void lane_stats(const E* s, int len, int lane, float c2, float& m,
                                           double& S) {
    using V = Vec<E>;
    constexpr int N = V::N;
    const int nfull = len / N;                   // fully valid vectors
    const bool ragged = nfull * N < len && lane == (nfull & 31);
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int g = lane;
    for (; g + 96 < nfull; g += 128) {
        float v[4][N];
#pragma unroll
        for (int t = 0; t < 4; ++t) V::unpack(*reinterpret_cast<const uint4*>(s + (g + 32 * t) * N), v[t]);
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int u = 0; u < N; u += 2) mx[t] = fmax_nan(mx[t], fmax_nan(v[t][u], v[t][u + 1]));
    }
    for (; g < nfull; g += 32) {
        float v[N];
        V::unpack(*reinterpret_cast<const uint4*>(s + g * N), v);
#pragma unroll
        for (int u = 0; u < N; u += 2) mx[0] = fmax_nan(mx[0], fmax_nan(v[u], v[u + 1]));
    }
    if (ragged) {
        float v[N];
        V::unpack(*reinterpret_cast<const uint4*>(s + nfull * N), v);
        for (int u = 0; u < N; ++u)
            if (nfull * N + u < len) mx[1] = fmax_nan(mx[1], v[u]);
    }
    const float mxl = fmax_nan(fmax_nan(mx[0], mx[1]), fmax_nan(mx[2], mx[3]));
    const float me = fmaxf(mxl, -FLT_MAX);   // all -inf so far: terms are exactly 0
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    g = lane;
    for (; g + 96 < nfull; g += 128) {
        float v[4][N];
#pragma unroll
        for (int t = 0; t < 4; ++t) V::unpack(*reinterpret_cast<const uint4*>(s + (g + 32 * t) * N), v[t]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int u = 0; u < N; u += 2) {
                a0 += ex2_approx(__fmul_rn(__fsub_rn(v[t][u], me), c2));
                a1 += ex2_approx(__fmul_rn(__fsub_rn(v[t][u + 1], me), c2));
            }
            acc[t] += static_cast<double>(a0 + a1);
        }
    }
    for (; g < nfull; g += 32) {
        float v[N];
        V::unpack(*reinterpret_cast<const uint4*>(s + g * N), v);
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int u = 0; u < N; u += 2) {
            a0 += ex2_approx(__fmul_rn(__fsub_rn(v[u], me), c2));
            a1 += ex2_approx(__fmul_rn(__fsub_rn(v[u + 1], me), c2));
        }
        acc[0] += static_cast<double>(a0 + a1);
    }
    if (ragged) {
        float v[N];
        V::unpack(*reinterpret_cast<const uint4*>(s + nfull * N), v);
        float t = 0.0f;
        for (int u = 0; u < N; ++u)
            if (nfull * N + u < len) t += ex2_approx(__fmul_rn(__fsub_rn(v[u], me), c2));
        acc[1] += static_cast<double>(t);
    }
    m = mxl;
    S = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// combine lane partials of a warp: M = max, S = sum S_l 2^((m_l - M) c2)   (fp64)
__device__ __forceinline__ void warp_combine(float m, double S, double c2d, float& M, double& SW) {
    M = warp_max_nan(m);
    double t = 0.0;
    if (S > 0.0 && M < INFINITY) t = S * exp2((static_cast<double>(m) - M) * c2d);
    SW = warp_sum_d(t);
}

template <typename E>
__device__ __forceinline__ void lane_argmax(const E* s, int len, int lane, int base, float& m,
                                            int& idx, float& mn) {
    using V = Vec<E>;
    constexpr int N = V::N;
    const int ng = (len + N - 1) / N;
    float best = -INFINITY, nanmax = -INFINITY;
    int bi = INT_MAX;
    for (int g = lane; g < ng; g += 32) {
        float v[N];
        V::unpack(*reinterpret_cast<const uint4*>(s + g * N), v);
#pragma unroll
        for (int u = 0; u < N; ++u) {
            if (g * N + u < len) {
                nanmax = fmax_nan(nanmax, v[u]);
                if (v[u] > best) {
                    best = v[u];
                    bi = base + g * N + u;
                }
            }
        }
    }
    m = best;
    idx = bi;
    mn = nanmax;
}

// ---- decision of one row pair (last-arriving warp) --------------------------------------
template <bool GREEDY, typename E>
__device__ void decide_row(const FParams& P, int b, int j, int lane) {
    const int kk = P.k, nch = P.nch;
    const size_t r = static_cast<size_t>(b) * (kk + 1) + j;
    const PartA* parts = P.partA + r * nch;
    // the draft token and its logits, read here (once per row, L2-hot) rather than gathered
    // on the streaming path
    const int x = j < kk ? P.ids[static_cast<size_t>(b) * kk + j] : -1;
    float zxp = 0.0f, zxq = 0.0f;
    if (!GREEDY && x >= 0 && x < P.V) {
        zxp = Vec<E>::one(row_p(P, b, j, sizeof(E)), x);
        zxq = Vec<E>::one(row_q(P, b, j, sizeof(E)), x);
    }
    __syncwarp();
    float Mp = -INFINITY, Mq = -INFINITY;
    int G = INT_MAX, nf = 0;
    for (int cc = lane; cc < nch; cc += 32) {
        const PartA a = load_cg(parts + cc);
        nf |= a.flags;
        if (GREEDY) {
            if (a.M_p > Mp || (a.M_p == Mp && a.argmax < G)) {
                Mp = a.M_p;
                G = a.argmax;
            }
        } else {
            Mp = fmax_nan(Mp, a.M_p);
            Mq = fmax_nan(Mq, a.M_q);
        }
    }
    if (GREEDY) {
        warp_argmax(Mp, G);
    } else {
        Mp = warp_max_nan(Mp);
        Mq = warp_max_nan(Mq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nf |= __shfl_xor_sync(0xFFFFFFFFu, nf, o);
    double Sp = 0.0, Sq = 0.0;
    if (!GREEDY) {
        const bool okp = Mp > -INFINITY && Mp < INFINITY, okq = Mq > -INFINITY && Mq < INFINITY;
        for (int cc = lane; cc < nch; cc += 32) {
            const PartA a = load_cg(parts + cc);
            if (okp && a.S_p > 0.0) Sp += a.S_p * exp2((static_cast<double>(a.M_p) - Mp) * P.c2d);
            if (okq && a.S_q > 0.0) Sq += a.S_q * exp2((static_cast<double>(a.M_q) - Mq) * P.c2d);
        }
        Sp = warp_sum_d(Sp);
        Sq = warp_sum_d(Sq);
    }
    const bool has_q = !GREEDY && j < kk;
    int32_t st = 0;
    bool stop = false, pass = false;
    if (j < kk && (x < 0 || x >= P.V)) st = kBadId;
    if (!st) {
        if ((nf & kPartNonfiniteP) || !(Mp < INFINITY)) st = kNonfinite;  // NaN or +inf
        else if (Mp == -INFINITY) st = kEmptyRow;
    }
    if (!st && has_q) {
        if ((nf & kPartNonfiniteQ) || !(Mq < INFINITY)) st = kNonfinite;
        else if (Mq == -INFINITY) st = kEmptyRow;
    }
    if (st) {
        stop = true;
    } else if (j < kk) {
        if (GREEDY) {
            stop = (x != G);                                          // argmax matching (C-5)
        } else if (zxq == -INFINITY) {
            st = kZeroQ;                                              // q_j(x_j) = 0 (C-7)
            stop = true;
        } else {
            // log2 p_j(x_j) - log2 q_j(x_j), fp64, on the kernel's softmax scale
            const double ell = (static_cast<double>(zxp) - Mp) * P.c2d - log2(Sp) -
                               ((static_cast<double>(zxq) - Mq) * P.c2d - log2(Sq));
            if (ell < 0.0) {
                const double a = exp2(ell);
                const uint4 w = verify_words(P.seed, static_cast<uint32_t>(j), P.round,
                                             P.rid_base + static_cast<uint64_t>(b));
                stop = unit24(w.x) >= a;                              // reject iff u >= a (C-2)
            }
        }
    }
    if (!GREEDY && !(st & kHard) && (stop || j == kk)) {
        // the sampling pass over this row is needed unless an earlier stop is already known
        const uint32_t cur = ld_relaxed_u32(P.stop + b);
        pass = (cur & ((1u << j) - 1u)) == 0u;
    }
    if (lane == 0) {
        trace_at(P, 4 * gridDim.x + r);
        RowStat rs;
        rs.S_p = Sp;
        rs.S_q = Sq;
        rs.M_p = Mp;
        rs.M_q = Mq;
        rs.status = st;
        rs.argmax = G;
        P.rowstat[r] = rs;
        if (GREEDY) P.cand[r] = make_int2(G, 0);
        if (stop) atomicOr(P.stop + b, 1u << j);
    }
    if (pass) {
        // deal the pass's chunks to nch consecutive CTAs' mailboxes (rowstat published first)
        __syncwarp();
        __threadfence();
        const uint32_t base = static_cast<uint32_t>(r * 2654435761ull >> 7) % gridDim.x;
        for (int cc = lane; cc < nch; cc += 32) {
            const uint32_t cta = (base + cc) % gridDim.x;
            const uint32_t at = atomicAdd(P.mbox_tail + cta, 1u);
            st_relaxed_u32(P.mbox + static_cast<size_t>(cta) * P.mcap + at,
                           kValid | (static_cast<uint32_t>(r) << 8) | cc);
        }
    }
    __syncwarp();
    if (lane == 0) request_event(P, b, 1u + (pass ? (1u << 8) : 0u));
}

// ---- phase 1: one warp's share of a chunk ----------------------------------------------
// Warp w owns vectors [w VPW, (w + 1) VPW) of the 16 KB slice (4 per lane for fp32), read
// once into registers; elements past the row end are masked to -inf (contribute nothing).
struct SPart {
    double S_p, S_q;
    float M_p, M_q;
    int32_t argmax, nf;
};
static_assert(sizeof(SPart) % 16 == 0, "keeps the result ring 16-byte aligned");
// One finished stage, handed from the consumer warps to the epilogue warp.
struct Res {
    int32_t type, b, j, c;
    PartA pa;                        // phase 1: the chunk's combined partial (ready to publish)
    PartB pb;                        // phase 2: the chunk's residual / p mass
    union {
        SPart part[kGW];             // phase 1: per-warp partials (combined by the last warp)
        double2 seg[kSegs];          // phase 2: segment totals (r mass, p mass)
    } u;
    uint32_t ready;                  // stage number + 1 once complete
    uint32_t pad2[3];
};
// dynamic shared memory: ring | full, empty barriers | meta | stop mirror | mail queue |
// control words [4] + stage counters | (16-aligned) result ring
constexpr size_t kScratchOff =
    (static_cast<size_t>(kStages) * kStageBytes + 2 * kStages * sizeof(uint64_t) +
     kStages * sizeof(Meta) + sizeof(uint32_t) * (kMaxB + kMq + 8 + 2 * kStages) + 15) & ~size_t(15);

template <typename E, bool GREEDY>
__device__ __forceinline__ void stats_share(const E* s, int len, int warp, int lane, float c2,
                                            int c0, float& m, double& S, int& arg, float& nanmax) {
    using V = Vec<E>;
    constexpr int N = V::N;
    constexpr int VPW = kRowChunkBytes / 16 / kGW;          // vectors per warp
    constexpr int PL = VPW / 32;                            // vectors per lane
    static_assert(PL * 32 * kGW * 16 == kRowChunkBytes, "chunk must split evenly");
    float v[PL][N];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        const int g = warp * VPW + i * 32 + lane;
        V::unpack(*reinterpret_cast<const uint4*>(s + g * N), v[i]);
        if ((g + 1) * N > len) {
#pragma unroll
            for (int u = 0; u < N; ++u)
                if (g * N + u >= len) v[i][u] = -INFINITY;
        }
    }
    if (GREEDY) {
        float best = -INFINITY, nm = -INFINITY;
        int bi = INT_MAX;
#pragma unroll
        for (int i = 0; i < PL; ++i) {
            const int g = warp * VPW + i * 32 + lane;
#pragma unroll
            for (int u = 0; u < N; ++u) {
                nm = fmax_nan(nm, v[i][u]);
                if (v[i][u] > best) {
                    best = v[i][u];
                    bi = c0 + g * N + u;
                }
            }
        }
        m = best;
        arg = bi;
        nanmax = nm;
        S = 0.0;
        return;
    }
    // warp max first, so every lane sums against the same reference (no rescaling)
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < PL; ++i)
#pragma unroll
        for (int u = 0; u < N; u += 2) mx = fmax_nan(mx, fmax_nan(v[i][u], v[i][u + 1]));
    mx = warp_max_nan(mx);
    const float me = fmaxf(mx, -FLT_MAX);     // all -inf so far: terms are exactly 0
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int u = 0; u < N; u += 2) {
            a0 += ex2_approx(__fmul_rn(__fsub_rn(v[i][u], me), c2));
            a1 += ex2_approx(__fmul_rn(__fsub_rn(v[i][u + 1], me), c2));
        }
        acc += static_cast<double>(a0 + a1);
    }
    m = mx;                                   // warp max (identical in all lanes)
    S = warp_sum_d(acc);                      // warp sum relative to m
    arg = 0;
    nanmax = mx;
}

// p and q slices of the same stage together (interleaved chains, joint reductions)
template <typename E>
__device__ __forceinline__ void stats_share_pq(const E* sp, const E* sq, bool with_q, int len,
                                               int warp, int lane, float c2, float& mp, double& Sp,
                                               float& mq, double& Sq, volatile float2* s_mx,
                                               int grp) {
    // Two passes over shared memory (max, then sum) keep the register footprint small.
    using V = Vec<E>;
    constexpr int N = V::N;
    constexpr int VPW = kRowChunkBytes / 16 / kGW;
    constexpr int PL = VPW / 32;
    const bool ragged = (warp + 1) * VPW * N > len;    // only the row's last chunk
    auto load = [&](const E* s, int i, float (&v)[N]) {
        const int g = warp * VPW + i * 32 + lane;
        V::unpack(*reinterpret_cast<const uint4*>(s + g * N), v);
        if (ragged) {
#pragma unroll
            for (int u = 0; u < N; ++u)
                if (g * N + u >= len) v[u] = -INFINITY;
        }
    };
    float xp = -INFINITY, xq = -INFINITY;
#pragma unroll 4
    for (int i = 0; i < PL; ++i) {
        float v[N], w[N];
        load(sp, i, v);
#pragma unroll
        for (int u = 0; u < N; u += 2) xp = fmax_nan(xp, fmax_nan(v[u], v[u + 1]));
        if (with_q) {
            load(sq, i, w);
#pragma unroll
            for (int u = 0; u < N; u += 2) xq = fmax_nan(xq, fmax_nan(w[u], w[u + 1]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        xp = fmax_nan(xp, __shfl_xor_sync(0xFFFFFFFFu, xp, o));
        xq = fmax_nan(xq, __shfl_xor_sync(0xFFFFFFFFu, xq, o));
    }
    // the stage max: every warp of the group publishes its max, then all sum against the same
    // reference, so the warp sums combine by plain addition (no exp rescaling anywhere)
    if (lane == 0) {
        s_mx[warp].x = xp;
        s_mx[warp].y = xq;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(kGW * 32) : "memory");
#pragma unroll
    for (int w = 0; w < kGW; ++w) {
        xp = fmax_nan(xp, s_mx[w].x);
        xq = fmax_nan(xq, s_mx[w].y);
    }
    const float ep = fmaxf(xp, -FLT_MAX), eq = fmaxf(xq, -FLT_MAX);
    double ap = 0.0, aq = 0.0;
#pragma unroll 4
    for (int i = 0; i < PL; ++i) {
        float v[N], w[N];
        load(sp, i, v);
        float p0 = 0.0f, p1 = 0.0f, q0 = 0.0f, q1 = 0.0f;
#pragma unroll
        for (int u = 0; u < N; u += 2) {
            p0 += ex2_approx(__fmul_rn(__fsub_rn(v[u], ep), c2));
            p1 += ex2_approx(__fmul_rn(__fsub_rn(v[u + 1], ep), c2));
        }
        ap += static_cast<double>(p0 + p1);
        if (with_q) {
            load(sq, i, w);
#pragma unroll
            for (int u = 0; u < N; u += 2) {
                q0 += ex2_approx(__fmul_rn(__fsub_rn(w[u], eq), c2));
                q1 += ex2_approx(__fmul_rn(__fsub_rn(w[u + 1], eq), c2));
            }
            aq += static_cast<double>(q0 + q1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ap += __shfl_xor_sync(0xFFFFFFFFu, ap, o);
        aq += __shfl_xor_sync(0xFFFFFFFFu, aq, o);
    }
    mp = xp;                                   // stage max (identical in every warp)
    Sp = ap;                                   // this warp's sum relative to it
    mq = with_q ? xq : -INFINITY;
    Sq = with_q ? aq : 0.0;
}

// ---- phase 2: sampling pass over one chunk ---------------------------------------------
// Each consumer warp computes 4 of the chunk's 32 token segments (p(x), and
// r(x) = max(0, p(x) - q(x)) in fp64 after the exp); segment totals are the last lane of an
// inclusive warp scan -- the same routine the final search re-runs on one segment.
template <typename E>
__device__ __forceinline__ void sample_share(const FParams& P, const E* sp, const E* sq,
                                             const RowStat& rs, bool use_q, int len, int warp,
                                             int lane, double2* s_seg) {
    using V = Vec<E>;
    constexpr int N = V::N;
    constexpr int SEG = 32 * N;
    constexpr int PER = kSegs / kGW;
    const float c2 = P.c2;
    const double invSp = 1.0 / rs.S_p, invSq = use_q ? 1.0 / rs.S_q : 0.0;
    double vr[PER], vpm[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e0 = (warp * PER + i) * SEG + lane * N;
        double r4 = 0.0, p4 = 0.0;
        if (e0 < len) {
            float vp[N], vq[N];
            V::unpack(*reinterpret_cast<const uint4*>(sp + e0), vp);
            if (use_q) V::unpack(*reinterpret_cast<const uint4*>(sq + e0), vq);
#pragma unroll
            for (int u = 0; u < N; ++u) {
                if (e0 + u < len) {
                    const double pd = prob_term(vp[u], rs.M_p, c2, invSp);
                    double rd = pd;
                    if (use_q) {
                        const double qd = prob_term(vq[u], rs.M_q, c2, invSq);
                        rd = pd > qd ? __dsub_rn(pd, qd) : 0.0;
                    }
                    r4 = __dadd_rn(r4, rd);
                    p4 = __dadd_rn(p4, pd);
                }
            }
        }
        vr[i] = r4;
        vpm[i] = p4;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {              // PER interleaved Kogge-Stone scans
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const double nr = __shfl_up_sync(0xFFFFFFFFu, vr[i], o);
            const double np = __shfl_up_sync(0xFFFFFFFFu, vpm[i], o);
            if (lane >= o) {
                vr[i] = __dadd_rn(vr[i], nr);
                vpm[i] = __dadd_rn(vpm[i], np);
            }
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < PER; ++i) s_seg[warp * PER + i] = make_double2(vr[i], vpm[i]);
    }
}

template <typename E>
__device__ void pass_search(const FParams& P, int b, int j, const RowStat& rs, int lane);

// last warp of a sampling-pass stage: chunk totals, publish, ticket; the last chunk searches
template <typename E>
__device__ void sample_epilogue(const FParams& P, int b, int j, int c, const RowStat& rs,
                                const double2 mine, int lane) {
    static_assert(kSegs == 32, "one segment per lane");
    const int kk = P.k, nch = P.nch;
    const size_t r = static_cast<size_t>(b) * (kk + 1) + j;
    double2* gseg = P.segtab + (r * nch + c) * kSegs;
    gseg[lane] = mine;
    double R = 0.0, Pm = 0.0;
    for (int s = 0; s < kSegs; ++s) {                // chunk totals in segment order
        R = __dadd_rn(R, __shfl_sync(0xFFFFFFFFu, mine.x, s));
        Pm = __dadd_rn(Pm, __shfl_sync(0xFFFFFFFFu, mine.y, s));
    }
    __threadfence();                                 // segment sums visible before the ticket
    __syncwarp();
    uint32_t t = 0;
    if (lane == 0) {
        P.partB[r * nch + c] = PartB{R, Pm};
        t = atomic_add_acq_rel(P.ticketB + r, 1u);
    }
    t = __shfl_sync(0xFFFFFFFFu, t, 0);
    if (t != static_cast<uint32_t>(nch - 1)) return;
    if (lane == 0) P.ticketB[r] = 0u;
    __syncwarp();
    pass_search<E>(P, b, j, rs, lane);
}

// inverse CDF over the whole pass: chunk -> 32 * N-token segment -> token (C-9)
template <typename E>
__device__ void pass_search(const FParams& P, int b, int j, const RowStat& rs, int lane) {
    using V = Vec<E>;
    constexpr int N = V::N;
    constexpr int SEG = 32 * N;
    const int kk = P.k, nch = P.nch;
    const size_t r = static_cast<size_t>(b) * (kk + 1) + j;
    const bool use_q = j < kk;
    const float c2 = P.c2;
    const double invSp = 1.0 / rs.S_p, invSq = use_q ? 1.0 / rs.S_q : 0.0;
    // lanes fetch the chunk masses in parallel (<= 8 per lane), then lane-order scans
    const PartB* pb = P.partB + r * nch;
    constexpr int kMaxPer = 8;                          // nch <= 255
    double vR[kMaxPer], vP[kMaxPer];
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
        const int cc = lane + 32 * t;
        vR[t] = 0.0;
        vP[t] = 0.0;
        if (cc < nch) {
            const PartB v = load_cg(pb + cc);
            vR[t] = v.R;
            vP[t] = v.P;
        }
    }
    // (register arrays indexed only by unrolled loop counters: no local memory)
    double Rt = 0.0, Pt = 0.0;
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
        for (int l = 0; l < 32 && 32 * t + l < nch; ++l) {
            Rt = __dadd_rn(Rt, __shfl_sync(0xFFFFFFFFu, vR[t], l));
            Pt = __dadd_rn(Pt, __shfl_sync(0xFFFFFFFFu, vP[t], l));
        }
    }
    const bool zero_res = use_q && !(Rt > 0.0);        // C-6: fall back to p_L
    const double tot = zero_res ? Pt : Rt;
    const uint4 w = verify_words(P.seed, static_cast<uint32_t>(j), P.round,
                                 P.rid_base + static_cast<uint64_t>(b));
    const double theta = unit24(w.y) * tot;
    int cstar = -1, lastpos = 0;
    double run = 0.0;
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
        const double mv = zero_res ? vP[t] : vR[t];
        for (int l = 0; l < 32 && 32 * t + l < nch; ++l) {
            const int cc = 32 * t + l;
            const double m = __shfl_sync(0xFFFFFFFFu, mv, l);
            if (m > 0.0) lastpos = cc;
            const double nr = __dadd_rn(run, m);
            if (cstar < 0 && nr > theta) cstar = cc;
            if (cstar < 0) run = nr;
        }
    }
    double th1 = theta - run;
    if (cstar < 0) {                                  // rounding: last chunk with mass (C-9)
        cstar = lastpos;
        th1 = INFINITY;
    }
    const double2* cseg = P.segtab + (r * nch + cstar) * kSegs;
    const double2 mine = lane < kSegs ? __ldcg(cseg + lane) : make_double2(0.0, 0.0);
    int sstar = -1;
    lastpos = 0;
    run = 0.0;
    for (int s = 0; s < kSegs; ++s) {
        const double m = __shfl_sync(0xFFFFFFFFu, zero_res ? mine.y : mine.x, s);
        if (m > 0.0) lastpos = s;
        const double nr = __dadd_rn(run, m);
        if (sstar < 0 && nr > th1) sstar = s;
        if (sstar < 0) run = nr;
    }
    double th2 = th1 - run;
    if (sstar < 0) {
        sstar = lastpos;
        th2 = INFINITY;
    }
    // re-read the segment's tokens from global memory (L2) and scan them as the pass did
    const int base = cstar * P.CHI + sstar * SEG;
    const int my0 = base + lane * N;
    const int cend = min(cstar * P.CHI + P.CHI, P.V);
    const void* gp = row_p(P, b, j, sizeof(E));
    const void* gq = use_q ? row_q(P, b, j, sizeof(E)) : nullptr;
    double rv[N];
    double r4 = 0.0;
#pragma unroll
    for (int u = 0; u < N; ++u) {
        rv[u] = 0.0;
        const int xx = my0 + u;
        if (xx < cend) {
            const double pd = prob_term(V::one(gp, xx), rs.M_p, c2, invSp);
            double rd = pd;
            if (use_q && !zero_res) {
                const double qd = prob_term(V::one(gq, xx), rs.M_q, c2, invSq);
                rd = pd > qd ? __dsub_rn(pd, qd) : 0.0;
            }
            rv[u] = rd;
        }
        r4 = __dadd_rn(r4, rv[u]);
    }
    const double incl = warp_incl_scan(r4, lane);
    double excl = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
    if (lane == 0) excl = 0.0;
    const unsigned hit = __ballot_sync(0xFFFFFFFFu, incl > th2);
    int fl, fu = -1;
    if (hit) {
        fl = __ffs(hit) - 1;
        if (lane == fl) {
            double rr = excl;
            int lp = -1;
#pragma unroll
            for (int u = 0; u < N; ++u) {
                if (rv[u] > 0.0) lp = u;
                rr = __dadd_rn(rr, rv[u]);
                if (fu < 0 && rr > th2) fu = u;
            }
            if (fu < 0) fu = lp;
        }
    } else {
        int lp = -1;
#pragma unroll
        for (int u = 0; u < N; ++u)
            if (rv[u] > 0.0) lp = u;
        const unsigned pos = __ballot_sync(0xFFFFFFFFu, lp >= 0);
        fl = pos ? 31 - __clz(pos) : 0;
        if (lane == fl) fu = lp >= 0 ? lp : 0;
    }
    fu = __shfl_sync(0xFFFFFFFFu, fu, fl);
    if (lane == 0) {
        trace_at(P, 4 * gridDim.x + static_cast<size_t>(P.B) * (kk + 1) + r);
        P.cand[r] = make_int2(base + fl * N + fu, zero_res ? kZeroResidual : 0);
        request_event(P, b, 1u << 16);
    }
}

// ---- the kernel -----------------------------------------------------------------------------
template <typename E, bool GREEDY>
__global__ void __launch_bounds__(kThreadsF, 1) k_verify_fused(const FParams P) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    Meta* meta = reinterpret_cast<Meta*>(empty + kStages);
    volatile uint32_t* s_stop = reinterpret_cast<volatile uint32_t*>(meta + kStages);
    volatile uint32_t* s_mq = s_stop + kMaxB;
    // s_ctl: [0] mail-queue tail, [1] all requests finished, [2] stop stage + 1,
    //        [3] result-ring entries consumed by the epilogue warp
    volatile uint32_t* s_ctl = s_mq + kMq;
    // [4] decider event tail, [5] epilogue finished
    volatile uint32_t* s_cnt = s_ctl + 8;           // [kStages] stage arrival counters
    Res* res = reinterpret_cast<Res*>(smem + kScratchOff);
    volatile float2* s_mx = reinterpret_cast<volatile float2*>(res + kR);   // stage maxima
    // decider messages (mailbox entries with kMsg), forwarded by the monitor
    volatile int* s_ev = reinterpret_cast<volatile int*>(s_mx + kStages * kGW);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = P.nch, kk = P.k, B = P.B;
    constexpr size_t ESZ = sizeof(E);
    constexpr int CH_ELEMS = kRowChunkBytes / sizeof(E);

    for (int i = threadIdx.x; i < B; i += blockDim.x) s_stop[i] = 0u;
    if (threadIdx.x < kStages) s_cnt[threadIdx.x] = 0u;
    for (int i = threadIdx.x; i < kR; i += blockDim.x) res[i].ready = 0u;
    if (threadIdx.x == 0) {
        s_ctl[0] = 0u;
        s_ctl[1] = 0u;
        s_ctl[2] = 0u;
        s_ctl[3] = 0u;
        s_ctl[4] = 0u;
        s_ctl[5] = 0u;
        s_ctl[6] = 0u;
        s_ctl[7] = 0u;
        trace_at(P, blockIdx.x);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kMonitorWarp) {
        // ================================ monitor warp ================================
        // Keeps the producer free of global-memory latency: mirrors the per-request stop
        // masks into shared memory and forwards ready entries of this CTA's mailbox (phase-2
        // work) into a shared-memory queue, in order.  One round trip per sweep.
        {
            uint32_t* mbox = P.mbox + static_cast<size_t>(blockIdx.x) * P.mcap;
            uint32_t mhead = 0, qtail = 0, evtail = 0;
            while (true) {
                for (int t0 = 0; t0 < B; t0 += 32 * 8) {       // 8 independent loads per lane
                    uint32_t v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int bb = t0 + lane + 32 * t;
                        v[t] = bb < B ? ld_relaxed_u32(P.stop + bb) : 0u;
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int bb = t0 + lane + 32 * t;
                        if (bb < B) s_stop[bb] = v[t];
                    }
                }
                uint32_t e = 0u;
                if (mhead + lane < static_cast<uint32_t>(P.mcap)) e = ld_relaxed_u32(mbox + mhead + lane);
                const uint32_t fin = ld_relaxed_u32(P.glob + 2);
                {
                    // contiguous ready prefix, split into phase-2 work (-> producer queue) and
                    // decider messages (-> decider queue), bounded by the room in both queues
                    const unsigned ready = __ballot_sync(0xFFFFFFFFu, (e & kValid) != 0u);
                    const int cnt = __ffs(~ready) - 1;
                    const int pre = cnt < 0 ? 32 : cnt;
                    const bool msg = (e & kMsg) != 0u;
                    const unsigned mm = __ballot_sync(0xFFFFFFFFu, msg) & (pre == 32 ? ~0u : ((1u << pre) - 1u));
                    const unsigned lt = (1u << lane) - 1u;
                    const uint32_t mroom = kEq - (evtail - s_ctl[6]);
                    const uint32_t wroom = kMq - (qtail - s_ctl[7]);
                    const uint32_t mpos = __popc(mm & lt), wpos = lane - mpos;
                    const bool fits = lane < pre && (msg ? mpos < mroom : wpos < wroom);
                    const unsigned ok = __ballot_sync(0xFFFFFFFFu, fits);
                    const int c2 = __ffs(~ok) - 1;
                    const int take = c2 < 0 ? 32 : c2;
                    if (take > 0) {
                        if (lane < take) {
                            if (msg) s_ev[(evtail + mpos) % kEq] = static_cast<int>(e);
                            else s_mq[(qtail + wpos) % kMq] = e;
                            mbox[mhead + lane] = 0u;
                        }
                        const unsigned tk = take == 32 ? ~0u : ((1u << take) - 1u);
                        const int nmsg = __popc(mm & tk);
                        __syncwarp();
                        __threadfence_block();
                        evtail += nmsg;
                        qtail += take - nmsg;
                        mhead += take;
                        if (lane == 0) {
                            s_ctl[0] = qtail;
                            s_ctl[4] = evtail;
                        }
                    }
                }
                if (fin == static_cast<uint32_t>(B) || ((P.debug & 1) && s_ctl[2] != 0u)) {
                    if (lane == 0) s_ctl[1] = 1u;
                    break;
                }
                __nanosleep(20);
            }
        }
    } else if (warp == kProducerWarp) {
        // ================================ producer warp ================================
        uint32_t n = 0;   // ring sequence number
        unsigned long long cnt[4] = {0, 0, 0, 0};
        auto acquire_slot = [&](uint32_t seq) -> int {
            const int slot = static_cast<int>(seq % kStages);
            const unsigned long long t0 = clock64();
            if (seq >= static_cast<uint32_t>(kStages))
                mbar_wait(empty + slot, ((seq / kStages) - 1u) & 1u);
            cnt[0] += clock64() - t0;
            cnt[2] += 1;
            return slot;
        };
        auto issue_load = [&](int slot, int b, int j, int c, int type, bool with_q) {
            char* dst = reinterpret_cast<char*>(smem) + static_cast<size_t>(slot) * kStageBytes;
            const int c0 = c * CH_ELEMS;
            const int len = min(CH_ELEMS, P.V - c0);
            const uint32_t bytes = static_cast<uint32_t>(len) * ESZ;
            const uint32_t bulk = bytes & ~15u;
            const char* gp = static_cast<const char*>(row_p(P, b, j, ESZ)) + c0 * ESZ;
            const char* gq = with_q ? static_cast<const char*>(row_q(P, b, j, ESZ)) + c0 * ESZ
                                    : nullptr;
            meta[slot] = Meta{type, b, j, c};
            for (uint32_t o = bulk; o < bytes; o += ESZ) {       // < 16-byte ragged tail
                *reinterpret_cast<E*>(dst + o) = *reinterpret_cast<const E*>(gp + o);
                if (with_q)
                    *reinterpret_cast<E*>(dst + kRowChunkBytes + o) =
                        *reinterpret_cast<const E*>(gq + o);
            }
            mbar_arrive_expect_tx(full + slot, with_q ? 2u * bulk : bulk);
            if (bulk) {
                bulk_g2s(dst, gp, bulk, full + slot);
                if (with_q) bulk_g2s(dst + kRowChunkBytes, gq, bulk, full + slot);
            }
        };
        // Lane 0 issues everything from shared-memory state only: phase-2 chunks waiting in
        // the monitor's queue first, then the next position-major phase-1 item (skipped when
        // its request is known to have stopped before its position: laziness).
        if (lane == 0) {
            uint32_t qhead = 0;
            auto try_mail = [&]() -> bool {
                if (GREEDY) return false;
                if (qhead == s_ctl[0]) return false;
                __threadfence_block();
                const uint32_t e = s_mq[qhead % kMq];
                ++qhead;
                s_ctl[7] = qhead;
                const int c = static_cast<int>(e & 0xFFu);
                const int rr = static_cast<int>((e & 0x3FFFFFFFu) >> 8);
                const int b = rr / (kk + 1), j = rr % (kk + 1);
                issue_load(acquire_slot(n), b, j, c, kItemResid, j < kk);
                ++n;
                return true;
            };
            const int G = gridDim.x;
            for (int w = blockIdx.x; w < P.n_items; w += G) {
                try_mail();
                const int c = w % nch, rr = w / nch, b = rr % B, j = rr / B;
                const int slot = acquire_slot(n);
                if (!(P.debug & 8) && (s_stop[b] & ((1u << j) - 1u))) {  // stopped before j
                    meta[slot] = Meta{kItemSkip, b, j, c};
                    mbar_arrive(full + slot);
                } else {
                    issue_load(slot, b, j, c, kItemStats, !GREEDY && j < kk);
                }
                ++n;
            }
            trace_at(P, gridDim.x + blockIdx.x);
            if (!GREEDY && !(P.debug & 1)) {
                while (true) {                          // phase 2 only
                    if (try_mail()) continue;
                    if (s_ctl[1] && qhead == s_ctl[0]) break;
                    __nanosleep(20);
                }
            }
            trace_at(P, 2 * gridDim.x + blockIdx.x);
            trace_warp(P, kConsumers, cnt);
            s_ctl[2] = n + 1;                           // epilogue: entries end before stage n
            for (int g = 0; g < kGroups; ++g) {         // one stop stage per consumer group
                const int slot = acquire_slot(n);
                meta[slot] = Meta{kItemStop, 0, 0, 0};
                mbar_arrive(full + slot);
                ++n;
            }
        }
        __syncwarp();
    } else if (warp < kConsumers) {
        // ================================ consumer warps ================================
        // Every consumer warp computes its share of every stage into the result-ring entry of
        // that stage; a shared-memory arrival counter elects the last warp, which gathers
        // z(x_j), releases the ring slot and hands the entry to the epilogue warp.  No global
        // traffic here, so the ring turns over at the speed of the arithmetic.
        unsigned long long cnt[4] = {0, 0, 0, 0};
        const unsigned long long tstart = clock64();
        const int grp = warp / kGW, wg = warp % kGW;
        for (uint32_t n = grp;; n += kGroups) {
            const int slot = static_cast<int>(n % kStages);
            const unsigned long long tw0 = clock64();
            mbar_wait(full + slot, (n / kStages) & 1u);
            const Meta m = meta[slot];
            cnt[0] += clock64() - tw0;
            cnt[2] += 1;
            if (m.type == kItemStop) break;
            Res* re = res + (n % kR);
            if (n >= static_cast<uint32_t>(kR)) {      // the epilogue must have freed this entry
                while (s_ctl[3] < n - kR + 1) __nanosleep(20);
            }
            const E* sp = reinterpret_cast<const E*>(smem + static_cast<size_t>(slot) * kStageBytes);
            const E* sq = reinterpret_cast<const E*>(smem + static_cast<size_t>(slot) * kStageBytes +
                                                     kRowChunkBytes);
            const int c0 = m.c * CH_ELEMS;
            const int len = min(CH_ELEMS, P.V - c0);
            const bool with_q = !GREEDY && m.j < kk;
            if (m.type == kItemStats && !(P.debug & 2)) {
                float mp, mq = -INFINITY, nmp = -INFINITY;
                double Sp = 0.0, Sq = 0.0;
                int ap = 0;
                if (GREEDY) stats_share<E, GREEDY>(sp, len, wg, lane, P.c2, c0, mp, Sp, ap, nmp);
                else stats_share_pq<E>(sp, sq, with_q, len, wg, lane, P.c2, mp, Sp, mq, Sq,
                                       s_mx + slot * kGW, grp);
                SPart sp_{};
                if (GREEDY) {
                    warp_argmax(mp, ap);
                    nmp = warp_max_nan(nmp);
                    sp_.M_p = mp;
                    sp_.M_q = -INFINITY;
                    sp_.argmax = ap;
                    sp_.nf = (nmp != nmp || nmp == INFINITY) ? kPartNonfiniteP : 0;
                } else {
                    sp_.M_p = mp;                   // already warp-reduced by stats_share
                    sp_.M_q = mq;
                    sp_.S_p = Sp;
                    sp_.S_q = Sq;
                }
                if (lane == 0) re->u.part[wg] = sp_;
            } else if (m.type == kItemResid) {
                if (!GREEDY) {
                    const size_t r = static_cast<size_t>(m.b) * (kk + 1) + m.j;
                    const RowStat rs = load_cg(P.rowstat + r);
                    sample_share<E>(P, sp, sq, rs, m.j < kk, len, wg, lane, re->u.seg);
                }
            }
            __syncwarp();
            __threadfence_block();
            uint32_t old = 0;
            if (lane == 0) old = atomicAdd(const_cast<uint32_t*>(s_cnt) + slot, 1u);
            old = __shfl_sync(0xFFFFFFFFu, old, 0);
            if (old != static_cast<uint32_t>(kGW - 1)) continue;
            // ---- last warp: z(x_j) gather, release the slot, then combine and hand over ----
            __threadfence_block();
            if (lane == 0) s_cnt[slot] = 0u;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);    // ring slot free: results are in smem
            if (m.type == kItemStats && !(P.debug & 2)) {
                SPart q{};
                q.M_p = -INFINITY;
                q.M_q = -INFINITY;
                q.argmax = INT_MAX;
                if (lane < kGW) q = re->u.part[lane];
                PartA pa{};
                if (GREEDY) {
                    float mv = q.M_p;
                    int idx2 = q.argmax, nf = q.nf;
                    warp_argmax(mv, idx2);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) nf |= __shfl_xor_sync(0xFFFFFFFFu, nf, o);
                    pa.M_p = mv;
                    pa.argmax = idx2;
                    pa.flags = nf;
                } else {
                    // every warp summed against the same stage max: plain sums in warp order
                    double Sp = 0.0, Sq = 0.0;
                    for (int w = 0; w < kGW; ++w) {
                        Sp += __shfl_sync(0xFFFFFFFFu, q.S_p, w);
                        Sq += __shfl_sync(0xFFFFFFFFu, q.S_q, w);
                    }
                    const float Mp = __shfl_sync(0xFFFFFFFFu, q.M_p, 0);
                    const float Mq = __shfl_sync(0xFFFFFFFFu, q.M_q, 0);
                    pa.M_p = Mp;
                    pa.M_q = Mq;
                    pa.S_p = Sp;
                    pa.S_q = Sq;
                    pa.flags = ((Mp != Mp || Mp == INFINITY) ? kPartNonfiniteP : 0) |
                               ((Mq != Mq || Mq == INFINITY) ? kPartNonfiniteQ : 0);
                }
                if (lane == 0) re->pa = pa;
            }
            if (lane == 0) {
                re->type = m.type;
                re->b = m.b;
                re->j = m.j;
                re->c = m.c;
                __threadfence_block();
                *reinterpret_cast<volatile uint32_t*>(&re->ready) = n + 1;
            }
            __syncwarp();
        }
        cnt[1] = clock64() - tstart;
        if (lane == 0) trace_warp(P, warp, cnt);
    } else if (warp == kEpilogueWarp) {
        // ================================ epilogue warp ================================
        // Lane i publishes the i-th ready result entry and fires its ticket atomic; the
        // tickets are examined one iteration later (their round trip overlaps the next batch),
        // and the rows / sampling passes they complete are decided / searched by the warp.
        uint32_t e0 = 0;
        unsigned long long ecnt[4] = {0, 0, 0, 0};
        const unsigned long long et0 = clock64();
        int ptype = 0, pbq = 0, pjq = 0;
        uint32_t pt = 0;
        bool pvalid = false;
        auto complete = [&]() {                          // tickets of the previous batch
            const bool resid = ptype == kItemResid;
            const bool last = pvalid && (resid ? pt == static_cast<uint32_t>(nch - 1)
                                               : (pt & 0xFFFFu) == static_cast<uint32_t>(nch - 1));
            const unsigned lm = __ballot_sync(0xFFFFFFFFu, last);
            pvalid = false;
            if (!lm) return;
            __threadfence();      // acquire side of the tickets that completed rows / passes
            if (last) {
                const size_t r = static_cast<size_t>(pbq) * (kk + 1) + pjq;
                uint32_t kind = 0u;
                if (resid) {
                    P.ticketB[r] = 0u;
                    kind = kMsgSearch;
                } else {
                    P.ticketA[r] = 0u;
                    if (ptype == kItemStats && (pt >> 16) == 0u) kind = kMsgDecide;
                    else request_event(P, pbq, 1u);          // row done without a decision
                }
                if (kind) {
                    // the decision / search of row r runs on CTA hash(r): balanced load
                    const uint32_t cta =
                        static_cast<uint32_t>((r * 0x9E3779B97F4A7C15ull) >> 40) % gridDim.x;
                    const uint32_t at = atomicAdd(P.mbox_tail + cta, 1u);
                    st_relaxed_u32(P.mbox + static_cast<size_t>(cta) * P.mcap + at,
                                   kValid | kMsg | (static_cast<uint32_t>(r) << 8) | kind);
                }
            }
            __syncwarp();
        };
        while (true) {
            const uint32_t idx = e0 + lane;
            const bool rdy = lane < kR &&
                             *reinterpret_cast<volatile uint32_t*>(&res[idx % kR].ready) == idx + 1;
            const unsigned rm = __ballot_sync(0xFFFFFFFFu, rdy);
            const int cntr = (~rm) ? __ffs(~rm) - 1 : 32;
            if (cntr == 0) {
                complete();                              // nothing new: settle old tickets
                const uint32_t stopn = s_ctl[2];
                if (stopn != 0u && e0 + 1 == stopn) break;
                __nanosleep(32);
                continue;
            }
            __threadfence_block();
            const unsigned long long tp0 = clock64();
            ecnt[2] += cntr;
            ecnt[3] += 1;
            int type = 0, b = 0, j = 0;
            uint32_t t = 0;
            if (lane < cntr && !(P.debug & 4)) {
                const Res* re = res + (idx % kR);
                type = re->type;
                b = re->b;
                j = re->j;
                const int c = re->c;
                const size_t r = static_cast<size_t>(b) * (kk + 1) + j;
                if (type == kItemStats) {
                    P.partA[r * nch + c] = re->pa;
                    t = atomic_add_release(P.ticketA + r, 1u);
                } else if (type == kItemSkip) {
                    t = atomic_add_release(P.ticketA + r, kSkipArrive);
                } else if (!GREEDY) {                     // kItemResid
                    double2* gseg = P.segtab + (r * nch + c) * kSegs;
                    double R = 0.0, Pm = 0.0;
                    for (int s2 = 0; s2 < kSegs; ++s2) {    // chunk totals in segment order
                        const double2 v = re->u.seg[s2];
                        gseg[s2] = v;
                        R = __dadd_rn(R, v.x);
                        Pm = __dadd_rn(Pm, v.y);
                    }
                    P.partB[r * nch + c] = PartB{R, Pm};
                    t = atomic_add_release(P.ticketB + r, 1u);
                }
            }
            __syncwarp();
            if (lane == 0) {                              // entries copied out: free them
                __threadfence_block();
                s_ctl[3] = e0 + cntr;
            }
            complete();                                   // previous batch (round trip done)
            ecnt[0] += clock64() - tp0;
            ptype = type;
            pbq = b;
            pjq = j;
            pt = t;
            pvalid = lane < cntr;
            e0 += cntr;
        }
        complete();
        if (lane == 0) s_ctl[5] = 1u;
        ecnt[1] = clock64() - et0;
        if (lane == 0) trace_warp(P, kEpilogueWarp, ecnt);
    } else if (warp == kDeciderWarp) {
        // ================================ decider warp ================================
        // Decides the rows and searches the sampling passes whose last chunk this CTA's
        // epilogue published, off the streaming path.
        uint32_t ehead = 0;
        unsigned long long dcnt[4] = {0, 0, 0, 0};
        while (true) {
            if (ehead == s_ctl[4]) {
                if (s_ctl[1] != 0u && ehead == s_ctl[4]) break;   // every request finished
                __nanosleep(32);
                continue;
            }
            __threadfence_block();
            const uint32_t e = static_cast<uint32_t>(s_ev[ehead % kEq]);
            ++ehead;
            __syncwarp();
            if (lane == 0) s_ctl[6] = ehead;             // message slot free
            const int r = static_cast<int>((e & 0x3FFFFFFFu) >> 8);
            const uint32_t kind = e & 0xFFu;
            const int bl = r / (kk + 1), jl = r % (kk + 1);
            const unsigned long long td0 = clock64();
            __threadfence();                             // acquire: the sender's data is visible
            if (kind == kMsgSearch) {
                if (!GREEDY) {
                    const RowStat rs = load_cg(P.rowstat + r);
                    pass_search<E>(P, bl, jl, rs, lane);
                }
            } else {
                decide_row<GREEDY, E>(P, bl, jl, lane);
            }
            __syncwarp();
            const unsigned long long dd = clock64() - td0;
            if (kind == kMsgSearch) { dcnt[1] += dd; dcnt[3] += 1; } else { dcnt[0] += dd; dcnt[2] += 1; }
        }
        if (lane == 0) trace_warp(P, kDeciderWarp, dcnt);
    }

    // ---- exit: the last CTA resets the queue counters ---------------------------------------
    __syncthreads();
    if (threadIdx.x == 0) {
        P.mbox_tail[blockIdx.x] = 0u;        // every push to this CTA happened before finish
        trace_at(P, 3 * gridDim.x + blockIdx.x);
        __threadfence();
        const uint32_t e = atomicAdd(P.glob + 3, 1u);
        if (e == gridDim.x - 1) {
            P.glob[2] = 0u;
            P.glob[3] = 0u;
        }
    }
}

}  // namespace fused

// ---- launch (used by abi.cu) ---------------------------------------------------------------
constexpr int kMaxGrid = kFusedMaxGrid;


template <typename E, bool GREEDY>
static cudaError_t launch_fused_t(const fused::FParams& P, cudaStream_t st) {
    using namespace fused;
    const size_t smem = kScratchOff + sizeof(Res) * kR + sizeof(float2) * kStages * kGW +
                        sizeof(int) * kEq;
    static int grid = 0;
    if (grid == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_verify_fused<E, GREEDY>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_verify_fused<E, GREEDY>,
                                                          kThreadsF, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        grid = sms * occ;
        if (grid > kMaxGrid) grid = kMaxGrid;
        if (grid < kFusedMinGrid) return cudaErrorInvalidConfiguration;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsF);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (device-side queue)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_verify_fused<E, GREEDY>, P);
}

cudaError_t launch_fused(const fused::FParams& P, bool greedy, bool bf16, cudaStream_t st) {
    if (greedy)
        return bf16 ? launch_fused_t<__nv_bfloat16, true>(P, st) : launch_fused_t<float, true>(P, st);
    return bf16 ? launch_fused_t<__nv_bfloat16, false>(P, st) : launch_fused_t<float, false>(P, st);
}

}  // namespace sd
