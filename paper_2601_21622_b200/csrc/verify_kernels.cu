// verify_kernels.cu -- sm_100a kernels of the batched speculative-sampling verify step.
//
// The method (Alg. 2; readings C-1..C-12 of DESIGN.md), per request b:
//   accept x_j iff u_acc(j) < min(1, p_j(x_j) / q_j(x_j)),  L = first rejection (else k),
//   emit x_0..x_{L-1} and t ~ norm(max(0, p_L - q_L)) (L < k) or t ~ p_k (L == k).
//
// Data flow (two launches, stream ordered, PDL-chained):
//   k_row_stats   grid = (chunk c, request b, position j), POSITION-MAJOR (all requests' position
//                 0 first).  CTA (c, b, j) TMA-bulk-loads its 16 KB slice of p_j (and q_j), computes
//                 the slice max and sum of 2^((z - M) log2e / T) (one MUFU.EX2 per element, fp64
//                 across threads) and gathers z(x_j).  The row's partials meet in one CTA (cluster
//                 leader / start-order decider / last ticket), which draws u_acc from Philox,
//                 decides the acceptance test and ORs "decided" (and "stopped") bits into the
//                 request's 64-bit state word.
//                 A CTA whose request already stopped below j skips its load (laziness, SURVEY
//                 8(d)).
//   k_sample_req  one CTA per request streams its stop row pair (p_L, q_L) -- or p_k for the
//                 bonus -- through a TMA ring, computes the residual segment masses on chip and
//                 runs the inverse-CDF search (k_sample_chunked for vocabularies beyond its
//                 on-chip table).
//   greedy (T = 0) replaces the sum by an (max, lowest index) reduction and the tail by a tiny
//                 finalize kernel.
// No tensor cores: the step is a streaming reduction, not a contraction.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <atomic>
#include <cstdio>

#include "philox.cuh"
#include "ptx.cuh"
#include "verify.cuh"

namespace sd {

constexpr int kGridY = 32768;   // requests per grid.y span (gridDim.y <= 65535)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Bounded spin-wait.  Every wait of the protocol is on a CTA that has already started (cluster
// peers are co-scheduled; a tagged-row decider waits only on CTAs that took a start ticket before
// it), so a legitimate wait lasts microseconds.  A breach of the workspace contract must not hang
// the GPU: after kSpinNs the wait gives up and the caller marks the request SD_FAULT_PROTOCOL.
// Debug builds (SD_STREAM_DEBUG) also print the site.
constexpr unsigned long long kSpinNs = 200ull * 1000 * 1000;   // 200 ms
template <typename F>
__device__ __forceinline__ bool spin_until(F cond, int site) {
    if (cond()) return true;
    const unsigned long long t0 = gtimer();
    for (uint32_t n = 1;; ++n) {
        if (cond()) return true;
        if ((n & 255u) == 0u && gtimer() - t0 > kSpinNs) {
#if SD_STREAM_DEBUG
            printf("spin_until timeout: site %d block (%d,%d,%d) thread %d\n", site, blockIdx.x,
                   blockIdx.y, blockIdx.z, threadIdx.x);
#else
            (void)site;
#endif
            return false;
        }
    }
}

// The accept length of a settled request, else -1: positions 0..L decided and L the lowest stop
// bit (L = k with no stop).  state: bits 0..31 decided, bits 32..63 stopped.
__device__ __forceinline__ int settled_L(unsigned long long s, int k) {
    const uint32_t stop = static_cast<uint32_t>(s >> 32), dec = static_cast<uint32_t>(s);
    const int L = stop ? __ffs(stop) - 1 : k;
    const uint32_t need = (2u << L) - 1u;   // bits 0..L (L = 31: all ones)
    return (dec & need) == need ? L : -1;
}

// ------------------------------------------------------------------------------------------
// element types: one 16-byte vector holds 4 fp32 or 8 bf16 logits
template <typename E>
struct Elt;
template <>
struct Elt<float> {
    static constexpr int VEC = 4;
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
struct Elt<__nv_bfloat16> {
    static constexpr int VEC = 8;
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

__device__ __forceinline__ bool nonfinite_or_nan(float z) { return !(z < INFINITY); }

// L2-coherent (L1-bypassing) load of a record another CTA published in this launch
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
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
// (value, index) max with lowest index on ties
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
// inclusive Kogge-Stone scan over the 32 lanes (fixed association: deterministic)
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, n);
    }
    return v;
}

// ---- lean arithmetic of the stats pass (FMNMX3, FFMA2, MUFU.EX2, FADD2) ----------------------
__device__ __forceinline__ float max3nan(float a, float b, float c) {
    float d;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long ex2x2(unsigned long long a) {
    float lo, hi;
    upk2(a, lo, hi);
    return pk2(ex2_approx(lo), ex2_approx(hi));
}

// One thread's (d, s) over its NV x VEC register-resident logits (-inf padded): d = fl(max * c2),
// s = sum of 2^(z c2 - d).  A NaN or +inf sets the fault flag (the max propagates it).
template <int NV, int VEC>
__device__ __forceinline__ void thread_stats(const float (&v)[NV][VEC], float c2, int flag, float& d,
                                             float& s, int& nf) {
    float mv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        float t = max3nan(v[i][0], v[i][1], v[i][2]);
#pragma unroll
        for (int e = 3; e < VEC; e += 2) t = max3nan(t, v[i][e], v[i][e + 1 < VEC ? e + 1 : e]);
        mv[i] = t;
    }
    float m = mv[0];
#pragma unroll
    for (int i = 1; i < NV; i += 2) m = max3nan(m, mv[i], mv[i + 1 < NV ? i + 1 : i]);
    d = -INFINITY;
    s = 0.0f;
    if (!(m < INFINITY)) {
        nf |= flag;                 // NaN or +inf
        return;
    }
    if (!(m > -INFINITY)) return;   // nothing finite here
    d = m * c2;
    const unsigned long long cc = pk2(c2, c2), nd = pk2(-d, -d);
    unsigned long long a[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int e = 0; e < VEC; e += 2) {
            const int k = (i * (VEC / 2) + e / 2) & 3;
            a[k] = fadd2(a[k], ex2x2(ffma2(pk2(v[i][e], v[i][e + 1]), cc, nd)));
        }
    const unsigned long long t = fadd2(fadd2(a[0], a[1]), fadd2(a[2], a[3]));
    float x0, x1;
    upk2(t, x0, x1);
    s = x0 + x1;
}

// ---- sd_profile_timestamps: fold %globaltimer into a span word (atomic min, no return) -------
__device__ __forceinline__ void prof_min(unsigned long long* w) {
    const unsigned long long t = gtimer();
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(w), "l"(t) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void state_or_release(unsigned long long* p, unsigned long long bits) {
    asm volatile("red.release.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(bits) : "memory");
}
__device__ __forceinline__ uint32_t ticket_relaxed(uint32_t* p) {
    uint32_t t;
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(p) : "memory");
    return t;
}

// ---- outputs --------------------------------------------------------------------------------
// out_accept_len / out_tokens / out_status of request b (one thread)
__device__ __forceinline__ void write_outputs(const Params& P, int b, int L, int32_t tok,
                                              int32_t status, bool hard) {
    const int kk = P.k;
    P.out_L[b] = hard ? 0 : L;
    int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
    for (int i = 0; i <= kk; ++i) {
        int32_t v = -1;
        if (!hard) v = i < L ? P.ids[static_cast<size_t>(b) * kk + i] : (i == L ? tok : -1);
        ot[i] = v;
    }
    if (P.out_status) P.out_status[b] = status;
}

// Leave request b's words of the workspace's zero region zeroed for the next call (one thread,
// after every CTA of k_row_stats is complete).
__device__ __forceinline__ void reset_request(const Params& P, int b) {
    P.state[b] = 0ull;
    for (int i = 0; i <= P.k; ++i) P.ticketA[static_cast<size_t>(b) * (P.k + 1) + i] = 0u;
}

// Combination of n slice partials (fp64, exact 2^(D_c - D) rescales); warp-collective, the
// result is valid in every lane.  SHARED: the partials sit in this CTA's shared memory (cluster
// leader, tagged decider), else in global memory written by other CTAs of this launch.
struct Comb {
    float RMp, RMq, zxp, zxq;
    double RSp, RSq;
    int flags, RG;
};
constexpr int32_t kPartProtocol = 16;   // a wait for this row's partials timed out

template <bool GREEDY, bool SHARED>
__device__ __forceinline__ Comb combine_parts(const PartA* parts, int n, int lane) {
    float RMp = -INFINITY, RMq = -INFINITY, zxp = 0.0f, zxq = 0.0f;
    int flags = 0, RG = INT_MAX, hasx_lane = 0;
    for (int cc = lane; cc < n; cc += 32) {
        const PartA a = SHARED ? parts[cc] : load_cg(parts + cc);
        flags |= a.flags;
        if (a.flags & kPartHasX) {
            zxp = a.zx_p;
            zxq = a.zx_q;
            hasx_lane = 1;
        }
        if (GREEDY) {
            if (a.M_p > RMp || (a.M_p == RMp && a.argmax < RG)) {
                RMp = a.M_p;
                RG = a.argmax;
            }
        } else {
            RMp = fmaxf(RMp, a.M_p);
            RMq = fmaxf(RMq, a.M_q);
        }
    }
    if (GREEDY) {
        warp_argmax(RMp, RG);
    } else {
        RMp = warp_max(RMp);
        RMq = warp_max(RMq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) flags |= __shfl_xor_sync(0xFFFFFFFFu, flags, o);
    const unsigned hx = __ballot_sync(0xFFFFFFFFu, hasx_lane);
    if (hx) {
        const int src = __ffs(hx) - 1;
        zxp = __shfl_sync(0xFFFFFFFFu, zxp, src);
        zxq = __shfl_sync(0xFFFFFFFFu, zxq, src);
    }
    double RSp = 0.0, RSq = 0.0;
    if (!GREEDY) {
        // rescale each slice sum from its own scaled max to the row's: S_c * 2^(D_c - D)
        for (int cc = lane; cc < n; cc += 32) {
            const PartA a = SHARED ? parts[cc] : load_cg(parts + cc);
            if (a.S_p > 0.0) RSp += a.S_p * exp2(static_cast<double>(a.M_p) - static_cast<double>(RMp));
            if (a.S_q > 0.0) RSq += a.S_q * exp2(static_cast<double>(a.M_q) - static_cast<double>(RMq));
        }
        RSp = warp_sum(RSp);
        RSq = warp_sum(RSq);
    }
    Comb C;
    C.RMp = RMp;
    C.RMq = RMq;
    C.zxp = zxp;
    C.zxq = zxq;
    C.RSp = RSp;
    C.RSq = RSq;
    C.flags = flags;
    C.RG = RG;
    return C;
}

// The combined statistics of a group of slices, as one partial of the next level.
__device__ __forceinline__ PartA comb_as_part(const Comb& C) {
    PartA a;
    a.S_p = C.RSp;
    a.S_q = C.RSq;
    a.M_p = C.RMp;
    a.M_q = C.RMq;
    a.zx_p = C.zxp;
    a.zx_q = C.zxq;
    a.flags = C.flags;
    a.argmax = C.RG;
    return a;
}

// The acceptance decision of row pair (b, j) from its whole-row statistics (one thread): the
// row statistics go to rowstat, then "decided" (and "stopped") bits are ORed into the request's
// state with release semantics, so a CTA that sees the request settled also sees its rowstat.
template <bool GREEDY>
__device__ __forceinline__ void decide(const Params& P, int b, int j, int x, const Comb& Cin) {
    const int kk = P.k;
    const size_t pos = static_cast<size_t>(b) * (kk + 1) + j;
    const bool load_q = !GREEDY && j < kk;
    Comb C = Cin;
    int32_t qst = 0;
    if (load_q && P.qmeta) {   // lazy q (NEXT-1): the draft's row statistics replace q's partials
        const QMeta m = P.qmeta[static_cast<size_t>(b) * kk + j];
        C.RMq = m.D;
        C.RSq = m.S;
        C.zxq = m.zx;
        qst = m.status & (kNonfinite | kEmptyRow);
    }
    int32_t st = 0;
    bool stop = false;
    double a = NAN;
    if (C.flags & kPartProtocol) st = kProtocol;
    if (!st && j < kk && (x < 0 || x >= P.V)) st = kBadId;
    if (!st) {
        if (C.flags & kPartNonfiniteP) st = kNonfinite;
        else if (C.RMp == -INFINITY) st = kEmptyRow;
    }
    if (!st && load_q) {
        if ((C.flags & kPartNonfiniteQ) || (qst & kNonfinite)) st = kNonfinite;
        else if (C.RMq == -INFINITY) st = kEmptyRow;
    }
    if (st) {
        stop = true;
    } else if (j < kk) {
        if (GREEDY) {
            stop = (x != C.RG);                                     // argmax matching (C-5)
        } else if (C.zxq == -INFINITY) {
            st = kZeroQ;                                            // q_j(x_j) = 0 (C-7)
            stop = true;
            a = 0.0;
        } else {
            // a = p(x)/q(x) = 2^((z_p(x) c2 - D_p) - (z_q(x) c2 - D_q)) * S_q / S_p
            const double l = (static_cast<double>(C.zxp) * P.c2d - static_cast<double>(C.RMp)) -
                             (static_cast<double>(C.zxq) * P.c2d - static_cast<double>(C.RMq));
            a = exp2(l) * (C.RSq / C.RSp);
            if (!(a >= 1.0)) {                                      // a = min(1, p/q) < 1
                const uint4 w = verify_words(P.seed, static_cast<uint32_t>(j), P.round,
                                             P.rid_base + static_cast<uint64_t>(b));
                stop = unit24(w.x) >= a;                            // reject iff u >= a (C-2)
            }
        }
    }
    RowStat rs;
    rs.S_p = C.RSp;
    rs.S_q = C.RSq;
    rs.a = a;
    rs.M_p = C.RMp;
    rs.M_q = C.RMq;
    rs.status = st;
    rs.argmax = C.RG;
    P.rowstat[pos] = rs;
    unsigned long long bits = 1ull << j;
    if (stop) bits |= 1ull << (32 + j);
    state_or_release(P.state + b, bits);
}

// The last publisher of a row pair combines the row's G published partials (fp64) and takes the
// decision (warp 0 of the caller).
template <bool GREEDY>
__device__ __forceinline__ void row_decide(const Params& P, int b, int j, int x, int lane) {
    const size_t pos = static_cast<size_t>(b) * (P.k + 1) + j;
    __threadfence();
    const Comb C = combine_parts<GREEDY, false>(P.partA + pos * P.nch, P.G, lane);
    if (lane == 0) decide<GREEDY>(P, b, j, x, C);
}

// Development timeline (debug builds, sd_debug_trace): slot i of the CTA's 8-word record gets
// %globaltimer; word 7 = smid << 32 | flags (1 skipped, 2 decider, 4 sampling task, 8 search).
#if SD_STREAM_DEBUG
#define SD_TR(P, i)                                                                          \
    do {                                                                                     \
        if ((P).trace)                                                                       \
            (P).trace[((static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + \
                       blockIdx.x) * 8 + (i)] = gtimer();                                    \
    } while (0)
#define SD_TRF(P, f)                                                                         \
    do {                                                                                     \
        if ((P).trace) {                                                                     \
            uint32_t smid;                                                                   \
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                                \
            (P).trace[((static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + \
                       blockIdx.x) * 8 + 7] |= (static_cast<unsigned long long>(smid) << 32) | (f); \
        }                                                                                    \
    } while (0)
#else
#define SD_TR(P, i) do {} while (0)
#define SD_TRF(P, f) do {} while (0)
#endif

// ---- tagged partials (k_row_stats with P.tagpub) --------------------------------------------
// A chunk partial is ten 32-bit words, each stored as one 8-byte word tag << 32 | data (single-copy
// atomic), so a reader that sees the call's tag in all ten has the whole partial without any
// fence on the writer's side.
__device__ __forceinline__ void write_tagged(const Params& P, size_t pos, int c, const PartA& a,
                                             uint32_t tag) {
    static_assert(sizeof(PartA) == 40, "PartA is ten 32-bit words");
    unsigned long long* w = P.partT + (pos * P.nch + c) * 10;
    const uint32_t* d = reinterpret_cast<const uint32_t*>(&a);
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const unsigned long long v = (static_cast<unsigned long long>(tag) << 32) | d[i];
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(w + i), "l"(v) : "memory");
    }
}
__device__ __forceinline__ bool read_tagged(const Params& P, size_t pos, int c, uint32_t tag,
                                            PartA& a) {
    const unsigned long long* w = P.partT + (pos * P.nch + c) * 10;
    uint32_t* d = reinterpret_cast<uint32_t*>(&a);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w + i) : "memory");
        ok = ok && static_cast<uint32_t>(v >> 32) == tag;
        d[i] = static_cast<uint32_t>(v);
    }
    return ok;
}

// ---- cluster publish (k_row_stats with CL > 1) --------------------------------------------
// A peer's partial goes into the leader's slot with five asynchronous 8-byte stores that complete
// transaction bytes on the leader's s_pbar (armed for (CL-1) * 40 bytes): no release fence.
__device__ __forceinline__ void cl_send_part(uint32_t raddr, const PartA& a, uint32_t rbar) {
    static_assert(sizeof(PartA) == 40, "PartA is five 8-byte words");
    const uint2* w = reinterpret_cast<const uint2*>(&a);
#pragma unroll
    for (int i = 0; i < 5; ++i) cl_st_async_v2(raddr + 8 * i, w[i], rbar);
}

// Warp 0 of a CTA of cluster g of row pair (b, j); `pa` is valid in lane 0.
template <bool GREEDY, int CL>
__device__ __forceinline__ void cluster_publish(const Params& P, const PartA& pa, PartA* s_parts,
                                                uint64_t* s_pbar, int rank, int g, int b, int j,
                                                int x, int lane) {
    if (rank != 0) {
        if (lane == 0) {
            cl_send_part(cl_map(&s_parts[rank], 0), pa, cl_map(s_pbar, 0));
            SD_TR(P, 5);
            SD_TR(P, 6);
        }
        return;
    }
    if (lane == 0) s_parts[0] = pa;
    const bool ok = spin_until([&] { return mbar_try_wait_cluster(s_pbar, 0); }, 1);
    __syncwarp();
    Comb C = combine_parts<GREEDY, true>(s_parts, CL, lane);
    if (!ok) C.flags |= kPartProtocol;
    if (C.flags & kPartSkipped) return;   // a peer saw a stop below j: the row is not needed
    if (P.G == 1) {                       // the cluster covers the row: decide at once
        if (lane == 0) {
            SD_TR(P, 5);
            decide<GREEDY>(P, b, j, x, C);
            SD_TR(P, 6);
            SD_TRF(P, 2);
        }
        return;
    }
    const size_t pos = static_cast<size_t>(b) * (P.k + 1) + j;
    uint32_t t = 0;
    if (lane == 0) {
        P.partA[pos * P.nch + g] = comb_as_part(C);
        // release: the partial is visible before the ticket
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(P.ticketA + pos) : "memory");
        SD_TR(P, 5);
    }
    t = __shfl_sync(0xFFFFFFFFu, t, 0);
    if (t != static_cast<uint32_t>(P.G - 1)) {
        if (lane == 0) SD_TR(P, 6);
        return;
    }
    row_decide<GREEDY>(P, b, j, x, lane);
    if (lane == 0) { SD_TR(P, 6); SD_TRF(P, 2); }
}

// ------------------------------------------------------------------------------------------
// Sampling (a6-a8): residual (or bonus) terms of one 16-byte vector (raw bits of p and q),
// ascending token order:
//   p(x) = 2^(z_p c2 - D_p) / S_p,  r(x) = max(0, p(x) - q(x)); r = p if !use_q.
// Elements at or past `valid` are 0.  Returns the sequential fp32 sums of r and p (the order the
// token search re-uses, so its partial sums are bit-identical).
struct ResidParams {
    float nDp, nDq, ip, iq;
    int use_q;
};
template <typename E>
__device__ __forceinline__ void resid_terms(uint4 up, uint4 uq, int valid, const ResidParams& rp,
                                            float c2, float (&r)[Elt<E>::VEC],
                                            float (&pv)[Elt<E>::VEC], float& sr, float& spv) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    float v[VEC];
    EL::unpack(up, v);
    const unsigned long long cc = pk2(c2, c2), np = pk2(rp.nDp, rp.nDp);
#pragma unroll
    for (int u = 0; u < VEC; u += 2) {
        float e0, e1;
        upk2(ex2x2(ffma2(pk2(v[u], v[u + 1]), cc, np)), e0, e1);
        pv[u] = __fmul_rn(e0, rp.ip);
        pv[u + 1] = __fmul_rn(e1, rp.ip);
    }
    if (rp.use_q) {
        float w[VEC];
        EL::unpack(uq, w);
        const unsigned long long nq = pk2(rp.nDq, rp.nDq);
#pragma unroll
        for (int u = 0; u < VEC; u += 2) {
            float e0, e1;
            upk2(ex2x2(ffma2(pk2(w[u], w[u + 1]), cc, nq)), e0, e1);
            r[u] = fmaxf(__fsub_rn(pv[u], __fmul_rn(e0, rp.iq)), 0.0f);
            r[u + 1] = fmaxf(__fsub_rn(pv[u + 1], __fmul_rn(e1, rp.iq)), 0.0f);
        }
    } else {
#pragma unroll
        for (int u = 0; u < VEC; ++u) r[u] = pv[u];
    }
#pragma unroll
    for (int u = 0; u < VEC; ++u)
        if (u >= valid) {
            r[u] = 0.0f;
            pv[u] = 0.0f;
        }
    sr = r[0];
    spv = pv[0];
#pragma unroll
    for (int u = 1; u < VEC; ++u) {
        sr = __fadd_rn(sr, r[u]);
        spv = __fadd_rn(spv, pv[u]);
    }
}
// Scaled residual terms for the per-request sampler: with e_p = 2^(z_p c2 - D_p) and
// e_q = 2^(z_q c2 - D_q), r(x) * S_p = max(0, e_p - rho * e_q), rho = S_p / S_q, or e_p
// (bonus row / zero-residual fallback, rho < 0 means "no q").  The common factor 1/S_p cancels
// in the inverse CDF, so the sampler works with these scaled terms throughout.  Past-the-end
// lanes (>= valid) are 0.  Returns the sequential fp32 sum (the order the search re-uses).
template <typename E>
__device__ __forceinline__ float resid_scaled(uint4 up, uint4 uq, int valid, float c2, float nDp,
                                              float nDq, float rho, float (&r)[Elt<E>::VEC]) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    float v[VEC];
    EL::unpack(up, v);
    const unsigned long long cc = pk2(c2, c2), np = pk2(nDp, nDp);
#pragma unroll
    for (int u = 0; u < VEC; u += 2) upk2(ex2x2(ffma2(pk2(v[u], v[u + 1]), cc, np)), r[u], r[u + 1]);
    if (rho >= 0.0f) {
        float w[VEC];
        EL::unpack(uq, w);
        const unsigned long long nq = pk2(nDq, nDq), nr = pk2(-rho, -rho);
#pragma unroll
        for (int u = 0; u < VEC; u += 2) {
            float t0, t1;
            upk2(ffma2(ex2x2(ffma2(pk2(w[u], w[u + 1]), cc, nq)), nr, pk2(r[u], r[u + 1])), t0, t1);
            r[u] = fmaxf(t0, 0.0f);
            r[u + 1] = fmaxf(t1, 0.0f);
        }
    }
    if (valid < VEC) {
#pragma unroll
        for (int u = 0; u < VEC; ++u)
            if (u >= valid) r[u] = 0.0f;
    }
    float sr = r[0];
#pragma unroll
    for (int u = 1; u < VEC; ++u) sr = __fadd_rn(sr, r[u]);
    return sr;
}
// ---- inverse CDF over on-chip / published masses (k_sample_req and the fused chunk tasks share
// these, so both take bit-identical decisions) -------------------------------------------------
// Levels 1 and 2 (one warp): blocks of 32 segments -> segment, first x with C(x) > theta (C-9),
// theta = u24(w_y) * total.  blk(i): mass of block i < nblk; seg(i): mass of segment i < nseg (a
// block's mass is the warp tree sum of its 32 segment masses).  Returns the total (every lane);
// when it is > 0, *sgsel and *th2 (every lane) are the segment found and theta's remainder in it.
template <typename FB, typename FS>
__device__ __forceinline__ double cdf_search_blocks(FB blk, FS seg, int nblk, int nseg, uint32_t w_y,
                                                    int lane, int* sgsel, double* th2) {
    double carry = 0.0;   // level 1: blocks -- warp scans with a carry
    for (int base = 0; base < nblk; base += 32) {
        double v = base + lane < nblk ? blk(base + lane) : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double a = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v = __dadd_rn(v, a);
        }
        carry = __dadd_rn(carry, __shfl_sync(0xFFFFFFFFu, v, 31));
    }
    const double tot = carry;
    if (!(tot > 0.0)) return tot;
    const double theta = unit24(w_y) * tot;
    int bsel = -1, blast = 0;
    double run = 0.0, th = INFINITY;
    for (int base = 0; base < nblk && bsel < 0; base += 32) {
        const double m = base + lane < nblk ? blk(base + lane) : 0.0;
        double v = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double a = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v = __dadd_rn(v, a);
        }
        v = __dadd_rn(run, v);
        const unsigned h = __ballot_sync(0xFFFFFFFFu, base + lane < nblk && v > theta);
        const unsigned pm = __ballot_sync(0xFFFFFFFFu, base + lane < nblk && m > 0.0);
        if (pm) blast = base + 31 - __clz(pm);
        if (h) {
            const int l = __ffs(h) - 1;
            double e = __shfl_up_sync(0xFFFFFFFFu, v, 1);
            if (lane == 0) e = run;
            bsel = base + l;
            th = theta - __shfl_sync(0xFFFFFFFFu, e, l);
        }
        run = __shfl_sync(0xFFFFFFFFu, v, 31);
    }
    if (bsel < 0) bsel = blast;                  // rounding: last block with mass
    // level 2: the block's 32 segments
    const int sgi = bsel * 32 + lane;
    const double m = sgi < nseg ? seg(sgi) : 0.0;
    double v = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, a);
    }
    const unsigned h = __ballot_sync(0xFFFFFFFFu, sgi < nseg && v > th);
    const unsigned pm = __ballot_sync(0xFFFFFFFFu, sgi < nseg && m > 0.0);
    const int ls = h ? __ffs(h) - 1 : (pm ? 31 - __clz(pm) : 0);
    double e = __shfl_up_sync(0xFFFFFFFFu, v, 1);
    if (lane == 0) e = 0.0;
    *th2 = h ? th - __shfl_sync(0xFFFFFFFFu, e, ls) : INFINITY;
    *sgsel = bsel * 32 + ls;
    return tot;
}

// Level 3 (one warp): re-read segment sgsel of the row (p, and q when rho >= 0) from global
// memory, recompute its scaled terms exactly as the mass pass did, scan, find the lane and the
// token (clamps: C-9).  The token in every lane.
template <typename E>
__device__ __forceinline__ int32_t cdf_search_segment(const E* gp, const E* gq, int sgsel, double th2,
                                                      int V, int nvv, float c2, float nDp, float nDq,
                                                      float rho, int lane) {
    constexpr int VEC = Elt<E>::VEC;
    constexpr int SEGV = 32;
    const int g = sgsel * SEGV + lane;
    const int valid = min(VEC, max(0, V - g * VEC));
    uint4 up = make_uint4(0u, 0u, 0u, 0u), uq = up;
    if (g < nvv) {
        up = __ldcg(reinterpret_cast<const uint4*>(gp) + g);
        if (rho >= 0.0f) uq = __ldcg(reinterpret_cast<const uint4*>(gq) + g);
    }
    float r[VEC];
    const float sr = resid_scaled<E>(up, uq, g < nvv - 1 ? VEC : valid, c2, nDp, nDq, rho, r);
    double v = static_cast<double>(sr);
    const float mine = sr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, a);
    }
    const unsigned hit = __ballot_sync(0xFFFFFFFFu, v > th2);
    const unsigned posm = __ballot_sync(0xFFFFFFFFu, mine > 0.0f);
    const int ls = hit ? __ffs(hit) - 1 : (posm ? 31 - __clz(posm) : 0);
    double ex = __shfl_up_sync(0xFFFFFFFFu, v, 1);
    if (lane == 0) ex = 0.0;
    int fe = -1;
    if (lane == ls) {
        const double th3 = hit ? th2 - ex : INFINITY;
        int lastpos = -1;
        float cum = 0.0f;
#pragma unroll
        for (int e2 = 0; e2 < VEC; ++e2) {
            const float te = r[e2];
            if (te > 0.0f) lastpos = e2;
            cum = e2 == 0 ? te : __fadd_rn(cum, te);
            if (fe < 0 && static_cast<double>(cum) > th3) fe = e2;
        }
        if (fe < 0) fe = lastpos >= 0 ? lastpos : 0;   // rounding: clamp (C-9)
    }
    fe = __shfl_sync(0xFFFFFFFFu, fe, ls);
    return (sgsel * SEGV + ls) * VEC + fe;
}

// inclusive Kogge-Stone scan of (R, P) pairs over the lanes (fixed association)
__device__ __forceinline__ double2 warp_scan2(double2 v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xFFFFFFFFu, v.x, o);
        const double b = __shfl_up_sync(0xFFFFFFFFu, v.y, o);
        if (lane >= o) {
            v.x = __dadd_rn(v.x, a);
            v.y = __dadd_rn(v.y, b);
        }
    }
    return v;
}

__device__ __forceinline__ ResidParams resid_params(const RowStat& rs, bool use_q) {
    ResidParams rp;
    rp.nDp = -rs.M_p;
    rp.nDq = use_q ? -rs.M_q : 0.0f;
    rp.ip = static_cast<float>(1.0 / rs.S_p);
    rp.iq = use_q ? static_cast<float>(1.0 / rs.S_q) : 0.0f;
    rp.use_q = use_q ? 1 : 0;
    return rp;
}

// Sampling chunk task c of request b at its stop position L (whole CTA): stage chunk c of
// (p_L, q_L) (L2 when recent), compute r and p per 32-vector segment (warp scans, fp64 segment
// masses) and the chunk's masses (a warp scan over segment pairs: the search's association),
// publish them and take the request's sampling ticket.  Returns (in every thread) whether this
// CTA finished the request's last chunk task.  The mbarrier parities ph0 (p) / ph1 (q) advance
// with each use.
template <typename E>
__device__ __forceinline__ bool sample_chunk(const Params& P, unsigned char* smem, uint64_t* bar,
                                             uint32_t& ph0, uint32_t& ph1, double2* s_seg,
                                             int* s_last, int b, int L, int c, const RowStat& rs) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int SEGV = 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = P.nch, kk = P.k;
    const bool use_q = L < kk;
    const float c2 = P.c2;
    const ResidParams rp = resid_params(rs, use_q);
    const E* gp = static_cast<const E*>(P.p_stage ? P.p_stage : P.p) + (static_cast<int64_t>(b) * (kk + 1) + L) * P.ld_p;
    const E* gq = use_q ? static_cast<const E*>(P.q_stage ? P.q_stage : P.q) + (static_cast<int64_t>(b) * kk + L) * P.ld_q
                        : nullptr;
    const int c0 = c * P.CH;
    const int len = min(P.CH, P.V - c0);
    const int nvv = (len + VEC - 1) / VEC;            // vectors incl. a ragged last one
    const int nsg = (nvv + SEGV - 1) / SEGV;          // segments in this chunk
    E* sp = reinterpret_cast<E*>(smem);
    E* sq = sp + P.CH;
    const uint32_t bytes = static_cast<uint32_t>(len) * sizeof(E);
    const uint32_t bulk = bytes & ~15u;
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar[0], bulk);
        if (bulk) bulk_g2s(sp, gp + c0, bulk, &bar[0]);
    } else if (tid == 32 && use_q) {
        mbar_arrive_expect_tx(&bar[1], bulk);
        if (bulk) bulk_g2s(sq, gq + c0, bulk, &bar[1]);
    }
    for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += kThreads) {
        sp[i] = gp[c0 + i];
        if (use_q) sq[i] = gq[c0 + i];
    }
    __syncthreads();
    mbar_wait(&bar[0], ph0);   // (the copies are in flight: they complete)
    ph0 ^= 1u;
    if (use_q) {
        mbar_wait(&bar[1], ph1);
        ph1 ^= 1u;
    }
    for (int sg = warp; sg < nsg; sg += kWarps) {
        const int g = sg * SEGV + lane;
        const int valid = min(VEC, max(0, len - g * VEC));
        uint4 up = make_uint4(0u, 0u, 0u, 0u), uq = up;
        if (g < nvv) {
            up = *reinterpret_cast<const uint4*>(sp + g * VEC);
            if (use_q) uq = *reinterpret_cast<const uint4*>(sq + g * VEC);
        }
        float r[VEC], pv[VEC], sr, spv;
        resid_terms<E>(up, uq, valid, rp, c2, r, pv, sr, spv);
        const double2 inc = warp_scan2(make_double2(sr, spv), lane);
        if (lane == 31) s_seg[sg] = inc;
    }
    __syncthreads();
    double2* gseg = P.segtab + (static_cast<size_t>(b) * nch + c) * P.nseg;
    for (int sg = tid; sg < nsg; sg += kThreads) gseg[sg] = s_seg[sg];
    if (warp == 0) {   // chunk masses: segment pairs, then a warp scan (the search's association)
        const double2 a0 = 2 * lane < nsg ? s_seg[2 * lane] : make_double2(0.0, 0.0);
        const double2 a1 = 2 * lane + 1 < nsg ? s_seg[2 * lane + 1] : make_double2(0.0, 0.0);
        const double2 inc = warp_scan2(make_double2(__dadd_rn(a0.x, a1.x), __dadd_rn(a0.y, a1.y)), lane);
        if (lane == 31) P.partB[static_cast<size_t>(b) * nch + c] = PartB{inc.x, inc.y};
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const uint32_t t = atomicAdd(P.ticketB + b, 1u);
        *s_last = t == static_cast<uint32_t>(nch - 1);
    }
    __syncthreads();
    return *s_last != 0;
}

// The inverse CDF of request b over its published chunk and segment masses, chunk -> segment ->
// token (warp 0 of the request's last chunk task; the result is valid in every lane).  The one
// found segment is recomputed with the identical routine, so the search sees exactly the masses
// the chunk tasks produced; clamps implement C-9, a zero residual falls back to p_L (C-6).
// *Rout = the mass of the distribution sampled (residual, or p at the bonus / C-6 fallback).
template <typename E>
__device__ __forceinline__ int32_t sample_search(const Params& P, int b, int L, const RowStat& rs,
                                                 int32_t& status, int lane, double* Rout) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int SEGV = 32;
    const int nch = P.nch, kk = P.k;
    const bool use_q = L < kk;
    const float c2 = P.c2;
    const ResidParams rp = resid_params(rs, use_q);
    const E* gp = static_cast<const E*>(P.p_stage ? P.p_stage : P.p) + (static_cast<int64_t>(b) * (kk + 1) + L) * P.ld_p;
    const E* gq = use_q ? static_cast<const E*>(P.q_stage ? P.q_stage : P.q) + (static_cast<int64_t>(b) * kk + L) * P.ld_q
                        : nullptr;
    __threadfence();
    // level 1: chunks, one lane each, warp scans over blocks of 32 chunks (carry between blocks)
    auto chunk_mass = [&](int cc) -> double2 {
        if (cc >= nch) return make_double2(0.0, 0.0);
        const PartB t = load_cg(P.partB + static_cast<size_t>(b) * nch + cc);
        return make_double2(t.R, t.P);
    };
    double2 carry = make_double2(0.0, 0.0);
    for (int base = 0; base < nch; base += 32) {
        const double2 icb = warp_scan2(chunk_mass(base + lane), lane);
        carry.x = __dadd_rn(carry.x, __shfl_sync(0xFFFFFFFFu, icb.x, 31));
        carry.y = __dadd_rn(carry.y, __shfl_sync(0xFFFFFFFFu, icb.y, 31));
    }
    const bool zero_res = use_q && !(carry.x > 0.0);        // C-6: fall back to p_L
    const double tot = zero_res ? carry.y : carry.x;
    *Rout = tot;
    const uint4 w = verify_words(P.seed, static_cast<uint32_t>(L), P.round,
                                 P.rid_base + static_cast<uint64_t>(b));
    const double theta = unit24(w.y) * tot;                 // C-9: first x with C(x) > theta
    int cstar = -1, clast = 0;
    double th1 = INFINITY, run = 0.0;
    for (int base = 0; base < nch && cstar < 0; base += 32) {
        const double2 pb = chunk_mass(base + lane);
        const double2 icb = warp_scan2(pb, lane);
        const double icm = __dadd_rn(run, zero_res ? icb.y : icb.x);
        const double mcm = zero_res ? pb.y : pb.x;
        const unsigned h = __ballot_sync(0xFFFFFFFFu, base + lane < nch && icm > theta);
        const unsigned pm = __ballot_sync(0xFFFFFFFFu, base + lane < nch && mcm > 0.0);
        if (pm) clast = base + 31 - __clz(pm);
        if (h) {
            const int l = __ffs(h) - 1;
            double e = __shfl_up_sync(0xFFFFFFFFu, icm, 1);
            if (lane == 0) e = run;
            cstar = base + l;
            th1 = theta - __shfl_sync(0xFFFFFFFFu, e, l);
        }
        run = __shfl_sync(0xFFFFFFFFu, icm, 31);
    }
    if (cstar < 0) cstar = clast;                           // rounding: last chunk with mass
    // level 2: segments of chunk cstar (pairs per lane, warp scan: the chunk task's association)
    const int cl = min(P.CH, P.V - cstar * P.CH);
    const int cnvv = (cl + VEC - 1) / VEC;
    const int cnsg = (cnvv + SEGV - 1) / SEGV;
    const double2* gseg = P.segtab + (static_cast<size_t>(b) * nch + cstar) * P.nseg;
    const double2 a0 = 2 * lane < cnsg ? __ldcg(gseg + 2 * lane) : make_double2(0.0, 0.0);
    const double2 a1 = 2 * lane + 1 < cnsg ? __ldcg(gseg + 2 * lane + 1) : make_double2(0.0, 0.0);
    const double m0 = zero_res ? a0.y : a0.x, m1 = zero_res ? a1.y : a1.x;
    const double2 ip = warp_scan2(make_double2(__dadd_rn(a0.x, a1.x), __dadd_rn(a0.y, a1.y)), lane);
    const double ipm = zero_res ? ip.y : ip.x;
    const unsigned hs = __ballot_sync(0xFFFFFFFFu, ipm > th1);
    const unsigned ps = __ballot_sync(0xFFFFFFFFu, __dadd_rn(m0, m1) > 0.0);
    const int lp = hs ? __ffs(hs) - 1 : (ps ? 31 - __clz(ps) : 0);
    double exs = __shfl_up_sync(0xFFFFFFFFu, ipm, 1);
    if (lane == 0) exs = 0.0;
    exs = __shfl_sync(0xFFFFFFFFu, exs, lp);
    const double lm0 = __shfl_sync(0xFFFFFFFFu, m0, lp), lm1 = __shfl_sync(0xFFFFFFFFu, m1, lp);
    int sstar;
    double th2;
    if (!hs) {                                    // rounding: last segment with mass
        sstar = lm1 > 0.0 ? 2 * lp + 1 : 2 * lp;
        th2 = INFINITY;
    } else if (__dadd_rn(exs, lm0) > th1) {
        sstar = 2 * lp;
        th2 = th1 - exs;
    } else {
        sstar = 2 * lp + 1;
        th2 = th1 - __dadd_rn(exs, lm0);
    }
    // recompute the segment exactly as the chunk task did (r and p terms both; zero_res selects p)
    const int g = sstar * SEGV + lane;
    const int valid = min(VEC, max(0, cl - g * VEC));
    uint4 up = make_uint4(0u, 0u, 0u, 0u), uq = up;
    if (g < cnvv) {
        up = __ldcg(reinterpret_cast<const uint4*>(gp + cstar * P.CH) + g);
        if (use_q) uq = __ldcg(reinterpret_cast<const uint4*>(gq + cstar * P.CH) + g);
    }
    float r[VEC], pv[VEC], sr, spv;
    resid_terms<E>(up, uq, valid, rp, c2, r, pv, sr, spv);
    const double2 inc = warp_scan2(make_double2(sr, spv), lane);
    const double icv = zero_res ? inc.y : inc.x;
    const float mine = zero_res ? spv : sr;
    const unsigned hit = __ballot_sync(0xFFFFFFFFu, icv > th2);
    const unsigned posm = __ballot_sync(0xFFFFFFFFu, mine > 0.0f);
    const int ls = hit ? __ffs(hit) - 1 : (posm ? 31 - __clz(posm) : 0);
    double ex = __shfl_up_sync(0xFFFFFFFFu, icv, 1);
    if (lane == 0) ex = 0.0;
    int fe = -1;
    if (lane == ls) {
        const double th3 = hit ? th2 - ex : INFINITY;
        int lastpos = -1;
        float cum = 0.0f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            const float te = zero_res ? pv[e] : r[e];
            if (te > 0.0f) lastpos = e;
            cum = e == 0 ? te : __fadd_rn(cum, te);
            if (fe < 0 && static_cast<double>(cum) > th3) fe = e;
        }
        if (fe < 0) fe = lastpos >= 0 ? lastpos : 0;   // rounding: clamp (C-9)
    }
    fe = __shfl_sync(0xFFFFFFFFu, fe, ls);
    if (zero_res) status |= kZeroResidual;
    return cstar * P.CH + (sstar * SEGV + ls) * VEC + fe;
}

// One sampling chunk task (whole CTA); the CTA that completes the request's last task searches
// and writes the request's outputs.  Hard-faulted requests have nothing to sample (the tail kernel
// writes their outputs).
template <typename E>
__device__ __forceinline__ void sample_task(const Params& P, unsigned char* smem, uint64_t* bar,
                                            uint32_t& ph0, uint32_t& ph1, double2* s_seg,
                                            int* s_last, int b, int L, int c) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RowStat rs = load_cg(P.rowstat + static_cast<size_t>(b) * (P.k + 1) + L);
    if (rs.status & kHard) return;
    const bool last = sample_chunk<E>(P, smem, bar, ph0, ph1, s_seg, s_last, b, L, c, rs);
    if (!last || warp != 0) return;
    int32_t status = rs.status;
    double R;
    const int32_t tok = sample_search<E>(P, b, L, rs, status, lane, &R);
    if (lane == 0) {
        write_outputs(P, b, L, tok, status, false);
        P.rres[b] = R;
        SD_TRF(P, 8);
    }
}

// The slice partial of one chunk (whole CTA; valid in warp 0, zx fields in lane 0): wait for the
// bulk copies (mbarrier parities ph0 / ph1), unpack NV vectors per thread into registers, the lean
// statistics (or argmax) per thread, warp and block reductions.
template <typename E, bool GREEDY>
__device__ __forceinline__ PartA slice_partial(const Params& P, const E* sp, const E* sq, int c0,
                                               int len, bool load_q, int x, uint64_t* bar,
                                               uint32_t ph0, uint32_t ph1, float (*s_d)[kWarps],
                                               double (*s_s)[kWarps], int* s_gi, int* s_f) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int NV = rs_chunk_bytes(GREEDY, sizeof(E)) / kVecBytes / kThreads;   // vectors per thread
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ---- registers: NV vectors of p (and q) per thread; -inf past the slice end ------------
    const int nfull = len / VEC;                 // complete vectors
    const int nvv = (len + VEC - 1) / VEC;       // vectors incl. a ragged last one
    float vp[NV][VEC];
    mbar_wait(&bar[0], ph0);   // (the copy is in flight: it completes)
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int g = tid + i * kThreads;
        if (g < nfull) {
            EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), vp[i]);
        } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) vp[i][e] = -INFINITY;
            if (g < nvv) {   // ragged last vector (row end only)
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if (g * VEC + e < len) vp[i][e] = EL::one(sp, g * VEC + e);
            }
        }
    }
    int nf = 0;
    float dP = -INFINITY, dQ = -INFINITY, sP = 0.0f, sQ = 0.0f;
    float gbest = -INFINITY;
    int gidx = INT_MAX;
    if (GREEDY) {
        float nanacc = -INFINITY;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            float vm = -INFINITY;
#pragma unroll
            for (int e = 0; e < VEC; e += 2) {
                nanacc = max3nan(nanacc, vp[i][e], vp[i][e + 1]);
                vm = max3(vm, vp[i][e], vp[i][e + 1]);
            }
            if (vm > gbest) {   // ascending index within the thread: strict > keeps the first
                int fe = 0;
#pragma unroll
                for (int e = VEC - 1; e >= 0; --e)
                    if (vp[i][e] == vm) fe = e;
                gbest = vm;
                gidx = c0 + (tid + i * kThreads) * VEC + fe;
            }
        }
        if (!(nanacc < INFINITY)) nf |= kPartNonfiniteP;
    } else {
        thread_stats<NV, VEC>(vp, P.c2, kPartNonfiniteP, dP, sP, nf);
        if (load_q) {
            float vq[NV][VEC];
            mbar_wait(&bar[1], ph1);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int g = tid + i * kThreads;
                if (g < nfull) {
                    EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), vq[i]);
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) vq[i][e] = -INFINITY;
                    if (g < nvv) {
#pragma unroll
                        for (int e = 0; e < VEC; ++e)
                            if (g * VEC + e < len) vq[i][e] = EL::one(sq, g * VEC + e);
                    }
                }
            }
            thread_stats<NV, VEC>(vq, P.c2, kPartNonfiniteQ, dQ, sQ, nf);
        }
    }

    // ---- block reduction: warps, then warp 0 ---------------------------------------------
    nf = __reduce_or_sync(0xFFFFFFFFu, nf);
    if (GREEDY) {
        float v = gbest;
        int i = gidx;
        warp_argmax(v, i);
        if (lane == 0) {
            s_d[0][warp] = v;
            s_gi[warp] = i;
            s_f[warp] = nf;
        }
    } else {
        const float Dw = warp_max(dP), Ew = warp_max(dQ);
        const double Sw = warp_sum(sP > 0.0f ? static_cast<double>(sP * ex2_approx(dP - Dw)) : 0.0);
        const double Tw = warp_sum(sQ > 0.0f ? static_cast<double>(sQ * ex2_approx(dQ - Ew)) : 0.0);
        if (lane == 0) {
            s_d[0][warp] = Dw;
            s_d[1][warp] = Ew;
            s_s[0][warp] = Sw;
            s_s[1][warp] = Tw;
            s_f[warp] = nf;
        }
    }
    __syncthreads();
    PartA pa{};
    if (warp == 0) {
        const bool on = lane < kWarps;
        const int f = __reduce_or_sync(0xFFFFFFFFu, on ? s_f[lane] : 0);
        if (GREEDY) {
            float v = on ? s_d[0][lane] : -INFINITY;
            int i = on ? s_gi[lane] : INT_MAX;
            warp_argmax(v, i);
            pa.M_p = v;
            pa.M_q = -INFINITY;
            pa.S_p = pa.S_q = 0.0;
            pa.argmax = i;
        } else {
            const float wd = on ? s_d[0][lane] : -INFINITY, we = on ? s_d[1][lane] : -INFINITY;
            const double ws = on ? s_s[0][lane] : 0.0, wt = on ? s_s[1][lane] : 0.0;
            const float Dc = warp_max(wd), Ec = warp_max(we);
            pa.S_p = warp_sum(ws > 0.0 ? ws * static_cast<double>(ex2_approx(wd - Dc)) : 0.0);
            pa.S_q = warp_sum(wt > 0.0 ? wt * static_cast<double>(ex2_approx(we - Ec)) : 0.0);
            pa.M_p = Dc;   // scaled maxima D (see resid_terms)
            pa.M_q = Ec;
            pa.argmax = INT_MAX;
        }
        if (lane == 0) {
            pa.zx_p = 0.0f;
            pa.zx_q = 0.0f;
            pa.flags = f;
            if (x >= c0 && x < c0 + len) {
                pa.zx_p = EL::one(sp, x - c0);
                pa.zx_q = load_q ? EL::one(sq, x - c0) : 0.0f;
                pa.flags |= kPartHasX;
            }
        }
    }
    return pa;
}

// ------------------------------------------------------------------------------------------
// Kernel A: per-slice statistics + per-row acceptance decision (+ sampling chunk tasks)
//
// CL > 1: the grid's x extent is G * CL (chunks padded with empty ones) in clusters of CL along
// x.  A non-leader CTA sends its partial into the leader's (rank 0) shared memory with st.async
// stores that complete bytes on the leader's mbarrier, then exits: no fence, no global atomic on
// its path.  The leader combines the CL partials; with G == 1 it decides at once, else it publishes
// the cluster partial and takes the row ticket (the last of the G leaders decides).  Every CTA of
// a cluster arrives exactly once, also when it skips, so the leader outlives every remote write
// into it.
// TAG (rows of 2..64 chunks, no cluster): every CTA that loads takes a start ticket on the row
// right after issuing its copies; the one holding ticket nch-1 started last, so every other chunk
// of the row has started (and never waits on anything): it polls their tagged partials and
// decides.  Skipping CTAs take no ticket -- a needed row (j <= L) never sees a stop below j, so
// all its chunks take tickets; an unneeded row may end without a decider.
// resident CTAs per SM: registers (40 / 32 per thread) with 16 KB slices; shared memory with the
// 32 KB slices of greedy fp32 rows
constexpr int rs_min_blocks(bool greedy, int esz) {
    return rs_chunk_bytes(greedy, esz) > kMaxChunkBytes ? 6 : (greedy ? 8 : 6);
}
template <typename E, bool GREEDY, int CL, bool TAG>
__global__ void __launch_bounds__(kThreads, rs_min_blocks(GREEDY, sizeof(E))) k_row_stats(const Params P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int NV = rs_chunk_bytes(GREEDY, sizeof(E)) / kVecBytes / kThreads;   // vectors per thread
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(8) uint64_t s_pbar;                    // CL > 1, leader: peer partials
    __shared__ __align__(16) PartA s_parts[CL];
    __shared__ __align__(16) PartA s_all[TAG ? kMaxTagNch : 1]; // TAG: the row's partials
    __shared__ uint32_t s_tag;
    __shared__ int s_flag;
    __shared__ float s_d[2][kWarps];
    __shared__ double s_s[2][kWarps];
    __shared__ int s_gi[kWarps], s_f[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = P.nch, kk = P.k;
    // grid (chunk, request in group, group x position): blocks are scheduled x-fastest, so within
    // a group of gridDim.y requests all position-0 rows come first (position-major), then
    // position 1, ...; one group (gridDim.y = B) is the plain position-major order
    const int c = blockIdx.x;
    int b = blockIdx.y, j = blockIdx.z;
    if (gridDim.z != static_cast<unsigned>(kk + 1)) {   // (more than one group: STARSD_RGROUP / B > 32768)
        const int grp = j / (kk + 1);
        j -= grp * (kk + 1);
        b += grp * gridDim.y;
        if (b >= P.B) return;
    }
    const size_t pos = static_cast<size_t>(b) * (kk + 1) + j;

    const int rank = CL > 1 ? c % CL : 0;
    // launched as a programmatic dependent of the previous kernel on the stream (P.chain): its
    // results (the previous call's workspace reset, the caller's logits) are visible after this
    if (P.chain) asm volatile("griddepcontrol.wait;" ::: "memory");
    // P.early: the sampler may launch once every CTA of the last position has started (all of
    // this grid is then resident, so the sampler's settle waits cannot starve it)
    if (P.early && j == kk) asm volatile("griddepcontrol.launch_dependents;");
    // (the earliest CTAs are the first row's: only they fold their start in)
    if (P.prof_ts && tid == 0 && blockIdx.y == 0 && blockIdx.z == 0) prof_min(P.prof_ts);
    if (tid == 0) {
        SD_TR(P, 0);
        const unsigned long long s = j ? ld_relaxed_u64(P.state + b) : 0ull;
        const uint32_t m = static_cast<uint32_t>(s >> 32);
        s_flag = (m & ((1u << j) - 1u)) != 0u;
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        if (CL > 1 && rank == 0) mbar_init(&s_pbar, 1);
        fence_mbar_init();
        if (CL > 1 && rank == 0) mbar_arrive_expect_tx(&s_pbar, (CL - 1) * sizeof(PartA));
    }
    __syncthreads();
    // the leader's barrier is initialised before any peer writes into it: every thread arrives on
    // the cluster barrier now and waits on it before the first remote write (a skipping CTA at
    // once, a working one after issuing its copies, so the wait overlaps the load).  Every thread
    // takes part in both halves: a thread parked on a CTA barrier while its peers wait on the
    // cluster barrier was measured to hang it.
    if (CL > 1) cl_arrive_relaxed();
    // The request already stopped before j: this row is never needed (laziness).
    if (s_flag) {
        if (CL > 1) cl_wait_acquire();
        if (tid == 0) {
            SD_TR(P, 1);
            SD_TRF(P, 1);
            if (CL > 1) {
                if (rank != 0) {
                    PartA a{};
                    a.flags = kPartSkipped;
                    cl_send_part(cl_map(&s_parts[rank], 0), a, cl_map(&s_pbar, 0));
                } else {
                    spin_until([&] { return mbar_try_wait_cluster(&s_pbar, 0); }, 2);
                }
            }
        }
        return;
    }
    if (tid == 0) SD_TR(P, 1);

    const int c0 = c * P.CH;
    const int len = max(0, min(P.CH, P.V - c0));   // CL > 1: empty padding chunks past V
    const bool load_q = !GREEDY && j < kk && P.qmeta == nullptr;   // (lazy q: metadata instead)
    const E* gp = static_cast<const E*>(P.p) + static_cast<int64_t>(pos) * P.ld_p + c0;
    const E* gq = load_q ? static_cast<const E*>(P.q) +
                               (static_cast<int64_t>(b) * kk + j) * P.ld_q + c0
                         : nullptr;
    E* sp = reinterpret_cast<E*>(smem);
    E* sq = sp + P.CH;
    const uint32_t bytes = static_cast<uint32_t>(len) * sizeof(E);
    const uint32_t bulk = bytes & ~15u;
    // p and q slices are copied by threads of different warps: bulk copies issued by one thread
    // complete one after another (tools/tma_probe)
    uint32_t tk = 0;
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar[0], bulk);
        if (bulk) bulk_g2s(sp, gp, bulk, &bar[0]);
        // start ticket and call tag (tagged rows): both are consumed at publish time (s_tag after
        // the block reduction's barrier), so their round trips overlap the load and the statistics
        if (TAG) {
            tk = ticket_relaxed(P.ticketA + pos);
            s_tag = (ld_relaxed_u32(P.epoch) + 1u) | 0x80000000u;
        }
    } else if (tid == 32 && load_q) {
        mbar_arrive_expect_tx(&bar[1], bulk);
        if (bulk) bulk_g2s(sq, gq, bulk, &bar[1]);
    }
    for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += kThreads) {
        sp[i] = gp[i];
        if (load_q) sq[i] = gq[i];
    }
    const int x = (j < kk) ? P.ids[static_cast<size_t>(b) * kk + j] : -1;
    if (CL > 1) cl_wait_acquire();   // (copies in flight) the leader's s_pbar is initialised
    __syncthreads();

    const PartA pa0 = slice_partial<E, GREEDY>(P, sp, sq, c0, len, load_q, x, bar, 0u, 0u, s_d, s_s,
                                                s_gi, s_f);
    if (tid == 0) SD_TR(P, 4);
    if constexpr (!GREEDY) {
        if (P.p_stage) {   // sd_verify_staged: this slice also goes to the device stage
            E* dp = static_cast<E*>(P.p_stage) + static_cast<int64_t>(pos) * P.ld_p + c0;
            E* dq = load_q ? static_cast<E*>(P.q_stage) + (static_cast<int64_t>(b) * kk + j) * P.ld_q + c0
                           : nullptr;
            if (bulk && (tid == 0 || (tid == 32 && load_q))) {
                bulk_s2g(tid == 0 ? dp : dq, tid == 0 ? sp : sq, bulk);
                bulk_wait_read();   // (the slice's shared memory may be released after this)
            }
            for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += kThreads) {
                dp[i] = sp[i];
                if (load_q) dq[i] = sq[i];
            }
        }
    }
    if ((CL > 1 || TAG) && warp != 0) return;
    if (warp == 0) {
        PartA pa = pa0;
        if (CL > 1) {
            cluster_publish<GREEDY, CL>(P, pa, s_parts, &s_pbar, rank, c / CL, b, j, x, lane);
            return;
        }
        if (TAG) {
            const uint32_t tag = s_tag;
            tk = __shfl_sync(0xFFFFFFFFu, tk, 0);
            if (tk != static_cast<uint32_t>(nch - 1)) {   // plain tagged stores, then exit
                if (lane == 0) {
                    write_tagged(P, pos, c, pa, tag);
                    SD_TR(P, 5);
                    SD_TR(P, 6);
                }
                return;
            }
            // the row's decider: every other chunk of the row took its ticket before this one,
            // so it has started; its tagged partial arrives
            if (lane == 0) s_all[c] = pa;
            bool ok = true;
            for (int cc = lane; cc < nch; cc += 32) {
                if (cc == c) continue;
                PartA a;
                ok = spin_until([&] { return read_tagged(P, pos, cc, tag, a); }, 9) && ok;
                s_all[cc] = a;
            }
            ok = __all_sync(0xFFFFFFFFu, ok);
            __syncwarp();
            Comb C = combine_parts<GREEDY, true>(s_all, nch, lane);
            if (!ok) C.flags |= kPartProtocol;
            if (lane == 0) SD_TR(P, 5);
            if (!(C.flags & kPartSkipped) && lane == 0) decide<GREEDY>(P, b, j, x, C);
            if (lane == 0) { SD_TR(P, 6); SD_TRF(P, 2); }
            return;
        }
        if (lane == 0) {
            P.partA[pos * nch + c] = pa;
            uint32_t t;   // release: the partial is visible before the ticket
            asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(P.ticketA + pos) : "memory");
            s_flag = t == static_cast<uint32_t>(nch - 1);   // last arriver of the row
            SD_TR(P, 5);
        }
    }
    __syncthreads();
    if (!s_flag || warp != 0) {
        if (tid == 0) SD_TR(P, 6);
        return;
    }

    row_decide<GREEDY>(P, b, j, x, lane);
    if (tid == 0) { SD_TR(P, 6); SD_TRF(P, 2); }
}


// ------------------------------------------------------------------------------------------
// Kernel B (one CTA per request): residual (or bonus) inverse-CDF sample at the stop position L.
//
// The CTA streams row L of its request -- units of kSUnit logits of p_L and q_L -- through a ring
// of kSRing shared-memory slots (lane 0 copies p, lane 1 copies q: two issuing threads keep two
// bulk copies in flight), computes r = max(0, p - q) (or p) per 16-byte vector and one fp64 mass
// per 32-vector segment (a warp tree reduction), keeps every segment mass of the row in shared
// memory, and searches blocks of 32 segments -> segment -> lane -> token on chip; only the found
// segment is re-read (32 vectors).  No ticket, no global segment table.
constexpr int kSThreadsB = 512;
constexpr int kSRing = 3;                         // ring slots (p unit | q unit each); 6 slots of
                                                  // 16 KB units measured 1-3 % slower (c2, c3)
constexpr int kSUnitBytes = 32 * 1024;            // bytes of p (and of q) per unit: one bulk copy
                                                  // per issuing thread (tools/tma_probe)
constexpr int kSMaxSeg = 2048;                    // segments per row kept in shared memory
                                                  // (V <= 262144 fp32 / 524288 bf16)

template <typename E>
__global__ void __launch_bounds__(kSThreadsB + 32, 1) k_sample_req(const Params P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int NT = kSThreadsB, NW = NT / 32;   // consumer warps; warp NW is the producer
    constexpr int SEGV = 32;                                  // vectors per segment
    constexpr int UV = kSUnitBytes / 16;                      // vectors per unit
    constexpr int USEG = UV / SEGV;                           // segments per unit
    extern __shared__ __align__(128) unsigned char smem[];    // ring, then segment masses
    double* segm = reinterpret_cast<double*>(smem + static_cast<size_t>(kSRing) * 2 * kSUnitBytes);
    __shared__ __align__(8) uint64_t full[kSRing][2], empty[kSRing];
    __shared__ double s_blk[kSMaxSeg / 32];                   // block (32-segment) masses
    __shared__ double s_th;
    __shared__ int s_sel[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kk = P.k;
    const int b = blockIdx.x;
    if (tid == 0) {
        for (int i = 0; i < kSRing; ++i) {
            mbar_init(&full[i][0], 1);
            mbar_init(&full[i][1], 1);
            mbar_init(&empty[i], NW);
        }
        fence_mbar_init();
    }
    // the end of k_row_stats: its writes are visible, the next call may tag anew, the next
    // call's k_row_stats may be scheduled (it waits for this grid to complete)
    // (P.early: CTA B, one past the requests, is the completion probe: it only waits for
    // k_row_stats, so the call counter and the span timestamp move when that grid is complete)
    const bool lead = P.early ? blockIdx.x == static_cast<unsigned>(P.B) : blockIdx.x == 0;
    auto primary_done = [&] {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (P.prof_ts && tid == 0 && (P.early ? lead : blockIdx.x < 8)) prof_min(P.prof_ts + 1);
        if (P.tagpub && tid == 0 && lead) {
            P.epoch[0] += 1u;   // k_row_stats is complete: the next call tags with a new value
        }
        if (P.chain) asm volatile("griddepcontrol.launch_dependents;");
    };
    if (P.early && lead) {
        primary_done();
        return;
    }
    __shared__ unsigned long long s_state;
    if (P.early) {
        // launched while k_row_stats' last position wave runs (its CTAs trigger at their start,
        // so every CTA of that grid is already resident): wait for this request to settle
        if (tid == 0) {
            unsigned long long st = 0ull;
            const bool ok = spin_until([&] {
                st = ld_relaxed_u64(P.state + b);
                return settled_L(st, kk) >= 0;
            }, 12);
            __threadfence();   // acquire: the rowstat released with the settling bits
            s_state = ok ? st : ~0ull;
        }
        __syncthreads();
    } else {
        primary_done();
        if (tid == 0) s_state = __ldcg(P.state + b);
        __syncthreads();
    }
    const bool lost = s_state == ~0ull;                  // (a wait timed out: protocol fault)
    const uint32_t mask = static_cast<uint32_t>(s_state >> 32);
    const int L = lost ? 0 : (mask ? __ffs(mask) - 1 : kk);
    RowStat rs = load_cg(P.rowstat + static_cast<size_t>(b) * (kk + 1) + L);
    if (lost) rs.status = kProtocol;
    const bool hard = (rs.status & kHard) != 0;
    const bool use_q = L < kk;
    const float c2 = P.c2;
    const E* gp = static_cast<const E*>(P.p_stage ? P.p_stage : P.p) + (static_cast<int64_t>(b) * (kk + 1) + L) * P.ld_p;
    const E* gq = use_q ? static_cast<const E*>(P.q_stage ? P.q_stage : P.q) + (static_cast<int64_t>(b) * kk + L) * P.ld_q
                        : nullptr;
    const int V = P.V;
    const int nvv = (V + VEC - 1) / VEC;                      // vectors of the row
    const int nunits = (nvv + UV - 1) / UV;
    const int nseg = (nvv + SEGV - 1) / SEGV;
    const uint32_t rowbytes = static_cast<uint32_t>(nvv) * 16u;   // staged bytes (16 B rounded)
    __syncthreads();
    int32_t status = rs.status;
    int32_t tok = -1;
    if (!hard) {
        ResidParams rp;
        rp.nDp = -rs.M_p;
        rp.nDq = use_q ? -rs.M_q : 0.0f;
        rp.ip = static_cast<float>(1.0 / rs.S_p);
        rp.iq = use_q ? static_cast<float>(1.0 / rs.S_q) : 0.0f;
        rp.use_q = use_q ? 1 : 0;
        float rho = use_q ? static_cast<float>(rs.S_p / rs.S_q) : -1.0f;   // < 0: p only
        bool zero_res = false;
        for (int attempt = 0; attempt < 2; ++attempt) {
            // ---- stream the row: unit u at ring position n (slot n % kSRing) ----------------
            auto issue = [&](int n, int u) {
                const int sl = n % kSRing;
                const uint32_t off = static_cast<uint32_t>(u) * kSUnitBytes;
                const uint32_t nb = min(static_cast<uint32_t>(kSUnitBytes), rowbytes - off);
                unsigned char* dst = smem + static_cast<size_t>(sl) * 2 * kSUnitBytes;
                // a different lane pair per slot: a thread's bulk copies complete one after
                // another, so rotating issuers keeps every slot's copies in flight together
                if (lane == 2 * sl) {
                    mbar_arrive_expect_tx(&full[sl][0], nb);
                    bulk_g2s(dst, reinterpret_cast<const char*>(gp) + off, nb, &full[sl][0]);
                } else if (lane == 2 * sl + 1 && rp.use_q) {
                    mbar_arrive_expect_tx(&full[sl][1], nb);
                    bulk_g2s(dst + kSUnitBytes, reinterpret_cast<const char*>(gq) + off, nb, &full[sl][1]);
                }
            };
            const int base_u = attempt * nunits;               // ring position of unit 0
            if (warp == NW) {
                // producer warp: lane 0 streams p, lane 1 streams q, each as far ahead as the ring allows
                for (int u = 0; u < nunits; ++u) {
                    const int n = base_u + u;
                    if (n >= kSRing) {
                        mbar_wait(&empty[n % kSRing], ((n / kSRing) & 1) ^ 1);
                        // the consumers' generic-proxy reads of the slot precede this
                        // async-proxy overwrite (WAR across proxies)
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    issue(n, u);   // (the retry pass re-reads units 0.. at later ring positions)
                }
            } else {
                for (int u = 0; u < nunits; ++u) {
                    const int n = base_u + u, sl = n % kSRing;
                    const uint32_t ph = (n / kSRing) & 1;
                    mbar_wait(&full[sl][0], ph);
                    if (rp.use_q) mbar_wait(&full[sl][1], ph);
                    const uint4* sp4 = reinterpret_cast<const uint4*>(smem + static_cast<size_t>(sl) * 2 * kSUnitBytes);
                    const uint4* sq4 = sp4 + UV;
                    // warp w: segments SPW*w .. SPW*w+SPW-1 of the unit (one vector per lane
                    // each), then one transpose-reduce of the SPW fp64 masses
                    constexpr int SPW = USEG / NW;
                    static_assert(SPW == 2 || SPW == 4, "two or four segments per consumer warp");
                    double d[SPW];
#pragma unroll
                    for (int k4 = 0; k4 < SPW; ++k4) {
                        const int sg = SPW * warp + k4;
                        const int g = u * UV + sg * SEGV + lane;    // row vector index
                        uint4 up = make_uint4(0u, 0u, 0u, 0u), uq = up;
                        if (g < nvv) {
                            up = sp4[sg * SEGV + lane];
                            if (rp.use_q) uq = sq4[sg * SEGV + lane];
                        }
                        const int valid = g < nvv - 1 ? VEC : min(VEC, max(0, V - g * VEC));
                        float r[VEC];
                        d[k4] = static_cast<double>(resid_scaled<E>(up, uq, valid, c2, rp.nDp, rp.nDq, rho, r));
                    }
                    const bool b4 = (lane >> 4) & 1;
                    double m;
                    int gs;
                    if constexpr (SPW == 4) {
                        const bool b3 = (lane >> 3) & 1;
                        double a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
                        a0 = __dadd_rn(a0, __shfl_xor_sync(0xFFFFFFFFu, b4 ? d[0] : d[2], 16));
                        a1 = __dadd_rn(a1, __shfl_xor_sync(0xFFFFFFFFu, b4 ? d[1] : d[3], 16));
                        m = b3 ? a1 : a0;
                        m = __dadd_rn(m, __shfl_xor_sync(0xFFFFFFFFu, b3 ? a0 : a1, 8));
#pragma unroll
                        for (int o = 4; o > 0; o >>= 1) m = __dadd_rn(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
                        gs = u * USEG + 4 * warp + 2 * b4 + b3;   // this lane group's segment
                    } else {
                        m = b4 ? d[1] : d[0];
                        m = __dadd_rn(m, __shfl_xor_sync(0xFFFFFFFFu, b4 ? d[0] : d[1], 16));
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) m = __dadd_rn(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
                        gs = u * USEG + 2 * warp + b4;
                    }
                    if ((lane & (32 / SPW - 1)) == 0 && gs < nseg) segm[gs] = m;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[sl]);
                }
            }
            __syncthreads();
            // ---- block masses (32 segments each; warp tree sums) and the total --------------
            const int nblk = (nseg + 31) / 32;
            for (int bk = warp; bk < nblk; bk += NW) {
                const int sgi = bk * 32 + lane;
                const double t = warp_sum(sgi < nseg ? segm[sgi] : 0.0);
                if (lane == 0) s_blk[bk] = t;
            }
            __syncthreads();
            if (warp == 0) {
                const uint4 w = verify_words(P.seed, static_cast<uint32_t>(L), P.round,
                                             P.rid_base + static_cast<uint64_t>(b));
                int sgsel = 0;
                double th2 = INFINITY;
                const double tot = cdf_search_blocks([&](int i) { return s_blk[i]; },
                                                     [&](int i) { return segm[i]; }, nblk, nseg,
                                                     w.y, lane, &sgsel, &th2);
                if (lane == 0) {
                    s_sel[1] = tot > 0.0;
                    P.rres[b] = tot / rs.S_p;   // (trace) mass of the distribution sampled
                    s_sel[0] = sgsel;
                    s_th = th2;
                }
            }
            __syncthreads();
            if (s_sel[1] || !rp.use_q) {
                zero_res = attempt == 1;
                break;
            }
            // C-6: the residual has no mass (rounding only): sample from p_L instead
            rp.use_q = 0;
            rho = -1.0f;
            __syncthreads();
        }
        // ---- level 3: re-read the found segment, scan it, find the lane and the token -------
        if (warp == 0) {
            tok = cdf_search_segment<E>(gp, gq, s_sel[0], s_th, V, nvv, c2, rp.nDp, rp.nDq, rho, lane);
            if (zero_res) status |= kZeroResidual;
        }
    }
    if (tid == 0) {
        const int Lout = hard ? 0 : L;
        P.out_L[b] = Lout;
        int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
        for (int i = 0; i <= kk; ++i) {
            int32_t v = -1;
            if (!hard) v = i < L ? P.ids[static_cast<size_t>(b) * kk + i] : (i == L ? tok : -1);
            ot[i] = v;
        }
        if (P.out_status) P.out_status[b] = status;
    }
    if (P.early) primary_done();   // (no k_row_stats CTA touches the request's words any more)
    if (tid == 0) reset_request(P, b);   // leave the workspace zeroed for the next call
}

// ------------------------------------------------------------------------------------------
// Kernel B, chunked form (rows longer than k_sample_req's on-chip segment table, V > 262144 fp32
// / 524288 bf16): grid (chunk c, request b).  CTA (c, b) runs sampling chunk task c of request b
// at its stop position L; the CTA completing the request's last task searches and writes the
// outputs.  The request's last CTA to finish writes the outputs of a hard-faulted request and
// resets the request's workspace words.
template <typename E>
__global__ void __launch_bounds__(kThreads) k_sample_chunked(const Params P) {
    constexpr int MAXSEG = kMaxChunkBytes / 16 / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(16) double2 s_seg[MAXSEG];
    __shared__ int s_last;

    const int tid = threadIdx.x;
    const int kk = P.k, nch = P.nch;
    const int c = blockIdx.x, b = blockIdx.y + blockIdx.z * kGridY;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    // programmatic dependent launch: this grid may start while k_row_stats drains; wait until
    // the primary grid is complete and its writes are visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (P.prof_ts && tid == 0 && blockIdx.x < 8 && blockIdx.y == 0 && blockIdx.z == 0)
        prof_min(P.prof_ts + 1);
    if (P.tagpub && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
        P.epoch[0] += 1u;   // k_row_stats is complete: the next call tags with a new value
    }
    // the next call's k_row_stats may be scheduled now (it waits for this grid to complete)
    if (P.chain) asm volatile("griddepcontrol.launch_dependents;");
    if (b >= P.B) return;
    const unsigned long long s = __ldcg(P.state + b);
    int L = settled_L(s, kk);
    RowStat rs;
    if (L >= 0) {
        rs = load_cg(P.rowstat + static_cast<size_t>(b) * (kk + 1) + L);
    } else {   // a broken protocol (never in a correct run): void the request
        L = 0;
        rs = RowStat{};
        rs.status = kProtocol;
    }
    const bool hard = (rs.status & kHard) != 0;
    __syncthreads();
    if (!hard) {
        uint32_t ph0 = 0, ph1 = 0;
        sample_task<E>(P, smem, bar, ph0, ph1, s_seg, &s_last, b, L, c);
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(P.tailT + b, 1u);
        if (t == static_cast<uint32_t>(nch - 1)) {   // every sampling step of b is complete
            if (hard) write_outputs(P, b, L, -1, rs.status, true);
            P.state[b] = 0ull;   // leave the workspace zeroed for the next call
            P.ticketB[b] = 0u;
            P.tailT[b] = 0u;
            for (int i = 0; i <= kk; ++i) P.ticketA[static_cast<size_t>(b) * (kk + 1) + i] = 0u;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Greedy finalize: one thread per request
__global__ void k_finalize_greedy(const Params P) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (P.prof_ts && threadIdx.x == 0 && blockIdx.x < 8) prof_min(P.prof_ts + 1);
    if (P.tagpub && threadIdx.x == 0 && blockIdx.x == 0) {
        P.epoch[0] += 1u;   // k_row_stats is complete: the next call tags with a new value
    }
    if (P.chain) asm volatile("griddepcontrol.launch_dependents;");
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P.B) return;
    const int kk = P.k;
    const uint32_t mask = static_cast<uint32_t>(P.state[b] >> 32);
    const int L = mask ? __ffs(mask) - 1 : kk;
    const RowStat rs = P.rowstat[static_cast<size_t>(b) * (kk + 1) + L];
    const bool hard = (rs.status & kHard) != 0;
    P.out_L[b] = hard ? 0 : L;
    int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
    for (int i = 0; i <= kk; ++i) {
        int32_t v = -1;
        if (!hard) v = i < L ? P.ids[static_cast<size_t>(b) * kk + i] : (i == L ? rs.argmax : -1);
        ot[i] = v;
    }
    if (P.out_status) P.out_status[b] = rs.status;
    P.state[b] = 0ull;
    for (int i = 0; i <= kk; ++i) P.ticketA[static_cast<size_t>(b) * (kk + 1) + i] = 0u;
}

// ------------------------------------------------------------------------------------------
// sd_verify_trace: the statistics the last call on a workspace computed, per (b, j) thread.
//   lam = ln 2 (D + log2 S)   (natural-log log-normaliser of softmax(z / T); D, S as in RowStat)
__global__ void k_trace(const RowStat* rowstat, const double* rres, const int32_t* accept_len,
                        int B, int k, double* lam_p, double* lam_q, double* a_out, double* R_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * (k + 1)) return;
    const int b = i / (k + 1), j = i % (k + 1);
    const int L = accept_len[b];
    const RowStat rs = rowstat[i];
    const double ln2 = 0.69314718055994530942;
    const bool reached = j <= L;
    lam_p[i] = reached ? ln2 * (static_cast<double>(rs.M_p) + log2(rs.S_p)) : NAN;
    if (j < k) {
        lam_q[b * k + j] = reached ? ln2 * (static_cast<double>(rs.M_q) + log2(rs.S_q)) : NAN;
        a_out[b * k + j] = reached ? rs.a : NAN;
    }
    if (j == 0) {
        const RowStat rl = rowstat[static_cast<size_t>(b) * (k + 1) + L];
        R_out[b] = (rl.status & kHard) ? NAN : rres[b];
    }
}

// ------------------------------------------------------------------------------------------
// Row statistics only (sd_draft_qmeta): the second kernel just resets the workspace words.
__global__ void k_reset(const Params P) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (P.tagpub && threadIdx.x == 0 && blockIdx.x == 0) {
        P.epoch[0] += 1u;   // k_row_stats is complete: the next call tags with a new value
    }
    if (P.chain) asm volatile("griddepcontrol.launch_dependents;");
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P.B) return;
    if (P.out_status) P.out_status[b] = P.rowstat[static_cast<size_t>(b) * (P.k + 1)].status;
    P.state[b] = 0ull;
    for (int i = 0; i <= P.k; ++i) P.ticketA[static_cast<size_t>(b) * (P.k + 1) + i] = 0u;
}

// Draft-row metadata (NEXT-1/2): row r's statistics (k = 0 calls: one row per "request") and the
// logit of its token ids[r].
template <typename E>
__global__ void k_qmeta(const Params P, const int32_t* ids, QMeta* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.B) return;
    const RowStat rs = P.rowstat[r];
    const int x = ids[r];
    QMeta m;
    m.S = rs.S_p;
    m.D = rs.M_p;
    m.zx = (x >= 0 && x < P.V) ? Elt<E>::one(static_cast<const E*>(P.p) + static_cast<int64_t>(r) * P.ld_p, x)
                               : NAN;
    m.status = rs.status & (kNonfinite | kEmptyRow);
    m.reserved = 0;
    out[r] = m;
}

// ------------------------------------------------------------------------------------------
__global__ void k_philox(uint64_t seed, uint64_t round, const uint32_t* pos, const uint64_t* rid,
                         int n, uint32_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 w = verify_words(seed, pos[i], round, rid[i]);
    reinterpret_cast<uint4*>(out)[i] = w;
}

// ------------------------------------------------------------------------------------------
// launchers (called from abi.cu)

// Second kernel of a call: programmatic dependent launch, so its launch and prologue overlap the
// tail of k_row_stats (the kernel waits with griddepcontrol.wait before reading decisions).
template <typename K>
static cudaError_t launch_dependent(K kernel, dim3 grid, unsigned block, size_t smem,
                                    cudaStream_t st, const Params& P) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, P);
}

// Profiling event: a real timestamp record even while the stream is being captured into a
// CUDA graph (external event node), a plain record otherwise.
void record_event(cudaEvent_t ev, cudaStream_t st) {
    if (!ev) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
    else
        cudaEventRecord(ev, st);
}
// k_sample_req's dynamic shared memory (ring + segment masses) needs the opt-in attribute, which
// is per device: set it once per device (thread-safe).
template <typename K>
static cudaError_t ensure_smem_optin(K kernel, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// (dynamic shared memory: 2 x kMaxChunkBytes at most; above the 48 KB default it needs the
// per-device opt-in)
template <typename E, bool G, int CL, bool TAG = false>
static void launch_stats_cl(const Params& P, cudaStream_t st) {
    if ((G ? 1 : 2) * rs_chunk_bytes(G, sizeof(E)) > 48 * 1024) {
        static std::atomic<uint64_t> optin{0};
        ensure_smem_optin(k_row_stats<E, G, CL, TAG>, (G ? 1 : 2) * rs_chunk_bytes(G, sizeof(E)), optin);
    }
    int gr = P.B < kGridY ? P.B : kGridY;            // requests per group (grid.y)
    if (P.rgroup > 0 && P.rgroup < gr) gr = P.rgroup;
    const int ng = (P.B + gr - 1) / gr;
    const dim3 gridA(CL > 1 ? P.G * CL : P.nch, gr, (P.k + 1) * ng);
    const size_t sm = (G ? 1 : 2) * static_cast<size_t>(P.CH) * sizeof(E);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = gridA;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (P.chain) {   // overlap this launch with the tail of the previous kernel on the stream
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (CL > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CL;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, k_row_stats<E, G, CL, TAG>, P);
}
template <typename E, bool G>
static void launch_stats(const Params& P, cudaStream_t st) {
    if (P.tagpub) {   // (tagged partials: rows of 2..64 chunks without clusters)
        launch_stats_cl<E, G, 1, true>(P, st);
        return;
    }
    switch (P.CL) {
        case 8: launch_stats_cl<E, G, 8>(P, st); break;
        case 4: launch_stats_cl<E, G, 4>(P, st); break;
        case 2: launch_stats_cl<E, G, 2>(P, st); break;
        default: launch_stats_cl<E, G, 1>(P, st); break;
    }
}

template <typename E>
static cudaError_t launch_sampled(const Params& P, cudaStream_t st, cudaEvent_t ev0,
                                  cudaEvent_t ev1) {
    const size_t smem = 2 * static_cast<size_t>(P.CH) * sizeof(E);
    const int nb = (P.B + kGridY - 1) / kGridY;
    const int nseg_row = (P.V + 32 * Elt<E>::VEC - 1) / (32 * Elt<E>::VEC);
    static std::atomic<uint64_t> optin{0};
    const size_t smB = static_cast<size_t>(kSRing) * 2 * kSUnitBytes + sizeof(double) * kSMaxSeg;
    if (nseg_row <= kSMaxSeg) {
        cudaError_t e = ensure_smem_optin(k_sample_req<E>, static_cast<int>(smB), optin);
        if (e != cudaSuccess) return e;
    } else if (smem > 48 * 1024) {
        static std::atomic<uint64_t> optin2{0};
        cudaError_t e = ensure_smem_optin(k_sample_chunked<E>, static_cast<int>(smem), optin2);
        if (e != cudaSuccess) return e;
    }
    record_event(ev0, st);
    launch_stats<E, false>(P, st);
    record_event(ev1, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (nseg_row <= kSMaxSeg)   // (P.early: one more CTA, the completion probe)
        return launch_dependent(k_sample_req<E>, dim3(P.B + (P.early ? 1 : 0)), kSThreadsB + 32, smB,
                                st, P);
    return launch_dependent(k_sample_chunked<E>, dim3(P.nch, P.B < kGridY ? P.B : kGridY, nb),
                            kThreads, smem, st, P);
}

template <typename E>
static cudaError_t launch_greedy(const Params& P, cudaStream_t st, cudaEvent_t ev0,
                                 cudaEvent_t ev1) {
    record_event(ev0, st);
    launch_stats<E, true>(P, st);
    record_event(ev1, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dependent(k_finalize_greedy, dim3((P.B + 127) / 128), 128, 0, st, P);
}

cudaError_t qmeta_gather(const Params& P, bool bf16, const int32_t* ids, QMeta* out,
                         cudaStream_t st);
cudaError_t launch_verify(const Params& P, bool greedy, bool bf16, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1) {
    if (greedy)
        return bf16 ? launch_greedy<__nv_bfloat16>(P, st, ev0, ev1)
                    : launch_greedy<float>(P, st, ev0, ev1);
    return bf16 ? launch_sampled<__nv_bfloat16>(P, st, ev0, ev1)
                : launch_sampled<float>(P, st, ev0, ev1);
}

// Row statistics of B rows (P.k == 0) without sampling, then the metadata gather.
cudaError_t launch_qmeta(const Params& P, bool bf16, const int32_t* ids, QMeta* out,
                         cudaStream_t st) {
    if (bf16) launch_stats<__nv_bfloat16, false>(P, st);
    else launch_stats<float, false>(P, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = launch_dependent(k_reset, dim3((P.B + 127) / 128), 128, 0, st, P);
    if (e != cudaSuccess) return e;
    return qmeta_gather(P, bf16, ids, out, st);
}
cudaError_t qmeta_gather(const Params& P, bool bf16, const int32_t* ids, QMeta* out,
                         cudaStream_t st) {
    if (P.B == 0) return cudaSuccess;
    if (bf16) k_qmeta<__nv_bfloat16><<<(P.B + 127) / 128, 128, 0, st>>>(P, ids, out);
    else k_qmeta<float><<<(P.B + 127) / 128, 128, 0, st>>>(P, ids, out);
    return cudaGetLastError();
}

cudaError_t launch_trace(const Params& P, const int32_t* accept_len, double* lam_p, double* lam_q,
                         double* a, double* R, cudaStream_t st) {
    const int n = P.B * (P.k + 1);
    if (n > 0)
        k_trace<<<(n + 255) / 256, 256, 0, st>>>(P.rowstat, P.rres, accept_len, P.B, P.k, lam_p,
                                                 lam_q, a, R);
    return cudaGetLastError();
}

// Device-side stand-in for a model forward of a given duration (star benchmarks): one thread
// spins on %globaltimer.
__global__ void k_spin_ns(uint64_t ns) {
    const uint64_t t0 = gtimer();
    uint64_t t;
    do {
        __nanosleep(1000);
        t = gtimer();
    } while (t - t0 < ns);
}
cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t st) {
    k_spin_ns<<<1, 32, 0, st>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_philox(uint64_t seed, uint64_t round, const uint32_t* pos, const uint64_t* rid,
                          int n, uint32_t* out, cudaStream_t st) {
    if (n > 0) k_philox<<<(n + 255) / 256, 256, 0, st>>>(seed, round, pos, rid, n, out);
    return cudaGetLastError();
}

}  // namespace sd
