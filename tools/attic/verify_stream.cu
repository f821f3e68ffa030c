// verify_stream.cu -- v4 (default): persistent, warp-specialized thread-block-cluster kernel.
//
// The method (Alg. 2; readings C-1..C-12 of DESIGN.md), per request b:
//   accept x_j iff u_acc(j) < min(1, p_j(x_j) / q_j(x_j)),  L = first rejection (else k),
//   emit x_0..x_{L-1} and t ~ norm(max(0, p_L - q_L)) (L < k) or t ~ p_k (L == k).
//
// Work: the (k+1)*B row pairs (p_j, q_j) of a call in POSITION-MAJOR order (row = j*B + b).
// G persistent clusters of C CTAs (one CTA per SM); cluster g owns rows g, g+G, g+2G, ...;
// CTA `rank` owns the vocabulary slice [rank*W, rank*W + W) of every row.  Inside a CTA:
//
//   producer warp  one thread streams 16 KB pieces of its slices into a ring of shared-memory
//                  slots with TMA 1-D bulk copies (cp.async.bulk, mbarrier completion), running
//                  ahead across rows.  Just before a row's first piece it reads rej_mask[b]: if
//                  an earlier position of request b already stopped the chain the row is never
//                  needed (laziness) and only a zero-byte "skip" marker is queued.
//                  Residual re-reads requested by the row warps are queued first (priority).
//   stats warps    consume the ring in order: per-thread online max + sum of 2^(z*c2 - d)
//                  (FMNMX3.NAN, FFMA2, MUFU.EX2, FADD2), per-warp partials at the end of a row;
//                  on residual pieces, r = max(0, p - q) and p per 128-token segment (fp64
//                  segment masses).  They never wait for a decision.
//   row warps      (rows round-robin) combine the warp partials, exchange the CTA partials with
//                  the cluster through distributed shared memory (st.shared::cluster + remote
//                  mbarrier arrive, acknowledged slot reuse), take the row decision (identical
//                  in every CTA), publish a stop in rej_mask[b] at once, and for a stopping row
//                  (or the bonus row k) request the residual pass, exchange slice masses and let
//                  the CTA holding theta = u_smp * R find the token.  The last of the k+1 rows of
//                  a request writes out_accept_len / out_tokens / out_status.
//
// Every logit of a reached row is read from HBM once; the residual pass re-reads the one
// stopping row per request shortly after its stats pass (L2-resident).  No tensor cores: the
// step is a streaming reduction, not a contraction.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "philox.cuh"
#include "ptx.cuh"
#include "verify.cuh"

namespace sd {
namespace strm {

// Development instrumentation (event log, clock64 accounting, bisection knobs) is compiled in only
// with -DSD_STREAM_DEBUG (STARSD_BUILD_DEBUG=1 python -m paper_2601_21622_b200.build): the
// production kernel carries no extra branches in its hot loops.
#ifdef SD_STREAM_DEBUG
constexpr bool kDbg = true;
#else
constexpr bool kDbg = false;
#endif

constexpr int NS = kSStatsWarps;          // stats warps
constexpr int NR = kSRowWarps;            // row warps
constexpr int NT = kSThreads;             // 32 * (1 + NS + NR + 1 + producers - 1)
constexpr int NST = NS * 32;              // stats threads
constexpr uint32_t kPiece = kSPieceBytes; // 16 KB ring slots
constexpr int PV = kSPieceBytes / 16;     // 16-byte vectors per piece
constexpr int SEGV = 32;                  // vectors per residual segment (one per lane)
constexpr int NPB = 8 * NR;               // partial slots (multiple of NR)
constexpr int NX = 2 * NR;                // exchange slots (multiple of NR)
constexpr int MAXC = 16;

constexpr int32_t kBadId = 1, kNonfinite = 2, kEmptyRow = 4, kZeroQ = 8, kZeroResidual = 16;
constexpr int32_t kHard = kBadId | kNonfinite | kEmptyRow;
constexpr int kFlagNfP = 1, kFlagNfQ = 2, kFlagSkip = 8;

enum : int { kEnd = 0, kSkip = 1, kStatP = 2, kStatQ = 3, kResid = 4 };

// ---- element types -----------------------------------------------------------------------
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
};

// ---- arithmetic ----------------------------------------------------------------------------
__device__ __forceinline__ float max3nan(float a, float b, float c) {   // FMNMX3.NAN
    float d;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {      // FMNMX3
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float& lo, float& hi) {
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
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long ex2x2(unsigned long long a) {
    float lo, hi;
    upk(a, lo, hi);
    return pk(ex2_approx(lo), ex2_approx(hi));
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
__device__ __forceinline__ double warp_scan1(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, a);
    }
    return v;
}

// ---- mbarriers, DSMEM ------------------------------------------------------------------
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cl(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {   // non-blocking
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}
// Waiting.  This CTA signals mbarriers constantly, and a try_wait with a suspend hint
// (NANOSLEEP.SYNCS) wakes on any of those events, so hinted waits degenerate into spinning that
// steals issue slots from the stats warps (tools/mbar_probe, ncu instruction histogram).  Waits
// therefore poll with test_wait and back off with a plain __nanosleep, whose length depends on
// how latency-critical the waiter is.  Bounded: a protocol bug traps instead of hanging the GPU.
constexpr uint32_t kSpinLimit = 1u << 24;
__device__ __forceinline__ bool mbar_test_wait_cl(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __noinline__ void wait_fail(const char* what, const void* bar, uint32_t parity) {
    printf("verify_stream: wait on %s (smem 0x%x parity %u) exceeded its bound: block %d warp %d\n", what,
           smem_addr(bar), parity, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x >> 5));
    __trap();
}
__device__ __forceinline__ void wait_poll(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t n = 0;
    while (!mbar_test_wait(bar, parity)) {
        __nanosleep(ns);
        if (++n > kSpinLimit) wait_fail("local mbarrier", bar, parity);
    }
}
__device__ __forceinline__ void wait_local(uint64_t* bar, uint32_t parity) { wait_poll(bar, parity, 200); }
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t n = 0;
    while (!mbar_test_wait_cl(bar, parity)) {
        __nanosleep(200);
        if (++n > kSpinLimit) wait_fail("cluster mbarrier", bar, parity);
    }
}
// wait_local + cycles spent waiting, added to *acc (trace mode accounting)
__device__ __forceinline__ void wait_local_t(uint64_t* bar, uint32_t parity, unsigned long long& acc) {
    if (mbar_test_wait(bar, parity)) return;
    const unsigned long long t0 = clock64();
    wait_local(bar, parity);
    acc += clock64() - t0;
}
__device__ __forceinline__ void wait_cluster_t(uint64_t* bar, uint32_t parity, unsigned long long& acc) {
    if (mbar_test_wait_cl(bar, parity)) return;
    const unsigned long long t0 = clock64();
    wait_cluster(bar, parity);
    acc += clock64() - t0;
}
__device__ __forceinline__ void st_cl_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cl_f64(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ int ld_acq_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_s32(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {   // every thread of every CTA
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
}

// ---- development event log (sd_debug_trace) ----------------------------------------------
enum : int { kEvStart = 1, kEvIssue = 2, kEvIssueR = 3, kEvSkip = 4, kEvConsume = 5, kEvResPiece = 6,
             kEvPdone = 7, kEvXch = 8, kEvDecide = 9, kEvResDone = 10, kEvRowEnd = 11, kEvEnd = 12,
             kEvPlan = 13 };
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_ev(unsigned long long* tr, int* cnt, int type, int arg) {
    if (!tr || !(cnt[1] & 64)) return;   // event log only with debug bit 6 (globaltimer reads are slow)
    const int i = atomicAdd(cnt, 1) + 1;
    if (i < kSTraceN - 16)
        tr[static_cast<size_t>(blockIdx.x) * kSTraceN + i] =
            (static_cast<unsigned long long>(type) << 56) |
            (static_cast<unsigned long long>(arg & 0xFFFF) << 40) | (gtimer() & 0xFFFFFFFFFFull);
}

// ---- shared structures ---------------------------------------------------------------------
struct PInfo {          // what a ring slot holds (written by the producer before the arrive)
    int kind;           // kEnd / kSkip / kStatP / kStatQ / kResid
    int t;              // local row index of this cluster
    int idx;            // piece index within the slice
    int aux;            // bit0: last piece of its row / residual pass; bit1: residual has q;
                        // bits 8..: row warp that requested the residual
};
struct WPart {          // one stats warp's partial of a row
    float dP, dQ;       // warp max of fl(m*c2)      | greedy: best value (dP)
    double sP, sQ;      // sum of 2^(z*c2 - d) rel. to dP / dQ
    int flags;          // kFlagNfP | kFlagNfQ | kFlagSkip
    int gidx;           // greedy: lowest index of the best value
};
struct Xch {            // one CTA's row partial, pushed into every peer
    double sP, sQ;
    float dP, dQ;       // greedy: dP = best value
    float zxp, zxq;
    int flags;          // + kFlagHasX
    int gidx;
};
constexpr int kFlagHasX = 4;
struct RParams {        // residual pass parameters of a row warp's current row
    float nDp, nDq, ip, iq;
    int use_q;
};

__device__ __forceinline__ int x_for(const SParams& P, int b, int j) {
    return j < P.k ? __ldg(P.ids + static_cast<size_t>(b) * P.k + j) : -1;
}

// The row's result is published; the last of the k+1 rows of request b emits its output.
__device__ void arrive_row(const SParams& P, int b, int j, bool write, int token, int status) {
    const int kk = P.k;
    if (write) P.rowres[static_cast<size_t>(b) * (kk + 1) + j] = make_int2(token, status);
    __threadfence();
    const uint32_t t = atomicAdd(P.ticket + b, 1u);
    if (t != static_cast<uint32_t>(kk)) return;
    __threadfence();
    const uint32_t m = __ldcg(P.rej_mask + b);
    const int L = m ? __ffs(static_cast<int>(m)) - 1 : kk;
    const int2 rr = __ldcg(P.rowres + static_cast<size_t>(b) * (kk + 1) + L);
    const bool hard = (rr.y & kHard) != 0;
    P.out_L[b] = hard ? 0 : L;
    int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
    for (int i = 0; i <= kk; ++i) {
        int32_t v = -1;
        if (!hard) v = i < L ? __ldg(P.ids + static_cast<size_t>(b) * kk + i) : (i == L ? rr.x : -1);
        ot[i] = v;
    }
    if (P.out_status) P.out_status[b] = rr.y;
    P.rej_mask[b] = 0u;   // leave the workspace zeroed for the next call
    P.ticket[b] = 0u;
}

// Residual terms of one 16-byte vector (raw bits of p and q), ascending token order:
//   p(x) = 2^(z_p*c2 - D_p) / S_p,  r(x) = max(0, p(x) - q(x)); r = p if !use_q.
// Elements at or past `valid` are 0.  Outputs the sequential fp32 sums of r and p.
template <typename E>
__device__ __forceinline__ void vec_terms(uint4 up, uint4 uq, int valid, const RParams& rp,
                                          float c2, float (&r)[Elt<E>::VEC],
                                          float (&pv)[Elt<E>::VEC], float& sr, float& spv) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    float v[VEC];
    EL::unpack(up, v);
    const unsigned long long cc = pk(c2, c2), np = pk(rp.nDp, rp.nDp), ipp = pk(rp.ip, rp.ip);
#pragma unroll
    for (int u = 0; u < VEC; u += 2) {
        const unsigned long long e = ex2x2(ffma2(pk(v[u], v[u + 1]), cc, np));
        upk(fmul2(e, ipp), pv[u], pv[u + 1]);                       // p(x)
    }
    if (rp.use_q) {
        float w[VEC];
        EL::unpack(uq, w);
        const unsigned long long nq = pk(rp.nDq, rp.nDq), iqq = pk(rp.iq, rp.iq);
#pragma unroll
        for (int u = 0; u < VEC; u += 2) {
            const unsigned long long q = fmul2(ex2x2(ffma2(pk(w[u], w[u + 1]), cc, nq)), iqq);
            float q0, q1;
            upk(q, q0, q1);
            r[u] = fmaxf(__fsub_rn(pv[u], q0), 0.0f);
            r[u + 1] = fmaxf(__fsub_rn(pv[u + 1], q1), 0.0f);
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

// Online (max, sum) of one piece's values held by a thread: m = running max, d = fl(m*c2),
// s = sum of 2^(z*c2 - d); a NaN or +inf sets the fault flag and stops the accumulation.
template <int VEC, int KV>
__device__ __forceinline__ void online_acc(const float (&v)[KV][VEC], float c2, bool isq, float& m,
                                           float& d, float& s, int& nf) {
    static_assert(KV == 8, "max tree below assumes 8 vectors per thread and piece");
    // NaN-propagating max: independent per-vector chains, then a 2-level FMNMX3 tree
    float mv[KV];
#pragma unroll
    for (int i = 0; i < KV; ++i) {
        float t = max3nan(v[i][0], v[i][1], v[i][2]);
#pragma unroll
        for (int e = 3; e < VEC; e += 2) t = max3nan(t, v[i][e], v[i][e + 1 < VEC ? e + 1 : e]);
        mv[i] = t;
    }
    const float pm = max3nan(max3nan(mv[0], mv[1], mv[2]), max3nan(mv[3], mv[4], mv[5]),
                             max3nan(mv[6], mv[7], mv[7]));
    const int flag = isq ? kFlagNfQ : kFlagNfP;
    if (!(pm < INFINITY)) {
        nf |= flag;                                   // NaN or +inf in a reached row
        return;
    }
    if ((nf & flag) || !(pm > -INFINITY)) return;
    if (pm > m) {                                     // rescale to the new running max
        const float dn = pm * c2;
        if (s > 0.0f) s *= ex2_approx(d - dn);
        m = pm;
        d = dn;
    }
    // sum of 2^(z*c2 - d): FFMA2 + 2 MUFU.EX2 + FADD2 per pair, four independent accumulators
    const unsigned long long cc = pk(c2, c2), nd = pk(-d, -d);
    unsigned long long a[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int i = 0; i < KV; ++i)
#pragma unroll
        for (int e = 0; e < VEC; e += 2) {
            const int k = (i * (VEC / 2) + e / 2) & 3;
            a[k] = fadd2(a[k], ex2x2(ffma2(pk(v[i][e], v[i][e + 1]), cc, nd)));
        }
    const unsigned long long t = fadd2(fadd2(a[0], a[1]), fadd2(a[2], a[3]));
    float x0, x1;
    upk(t, x0, x1);
    s += x0 + x1;
}

template <typename E, bool GREEDY>
__global__ void __launch_bounds__(NT, 1) k_verify_stream(const SParams P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    extern __shared__ __align__(1024) unsigned char smem[];
    // ring slots first, then the residual segment tables [NR][P.segmax] (double2)
    unsigned char* rring = smem + static_cast<size_t>(P.nslot) * kPiece;   // residual ring
    double2* segbuf = reinterpret_cast<double2*>(rring + static_cast<size_t>(kSResSlots) * kPiece);

    __shared__ __align__(8) uint64_t full[kSMaxSlots], empty[kSMaxSlots];
    __shared__ __align__(8) uint64_t pdone[NPB], pfree[NPB];
    __shared__ __align__(8) uint64_t xbar[NX], xfree[NX];
    __shared__ __align__(8) uint64_t xrbar[NR], xrfree[NR], resdone[NR];
    __shared__ __align__(8) uint64_t full_r[kSResSlots], empty_r[kSResSlots];
    __shared__ PInfo pinfo[kSMaxSlots];
    __shared__ PInfo pinfo_r[kSResSlots];
    __shared__ WPart part[NPB][NS];
    __shared__ Xch xch[NX][MAXC];
    __shared__ double2 xres[NR][MAXC];
    __shared__ RParams rparams[NR];
    __shared__ int resreq[NR];
    __shared__ int rows_done;
    __shared__ int tr_state[2];        // event count, debug flags (trace_ev reads cnt[1])
    int& tr_cnt = tr_state[0];
    __shared__ unsigned long long ctr[16];   // clock64 accounting (trace mode)
    unsigned long long* const tr = kDbg ? P.trace : nullptr;
    const int dbg = kDbg ? P.debug : 0;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = P.C, G = P.G;
    const int rank = static_cast<int>(blockIdx.x) % C;
    const int g = static_cast<int>(blockIdx.x) / C;
    const int kk = P.k;
    const int nrows = (kk + 1) * P.B;
    const int T = g < nrows ? (nrows - g + G - 1) / G : 0;   // rows of this cluster
    const int s0 = rank * P.W;
    const int len = max(0, min(P.W, P.V - s0));               // logits in my slice
    const int nvec = (len + VEC - 1) / VEC;                   // 16-byte vectors (last may be ragged)
    const int nfull = len / VEC;
    const uint32_t sbytes = static_cast<uint32_t>(nvec) * 16u; // bytes staged per slice
    const int npc = static_cast<int>((sbytes + kPiece - 1) / kPiece);
    const int nseg = (nvec + SEGV - 1) / SEGV;
    const float c2 = P.c2;
    const int nslot = P.nslot;

    if (tid == 0) {
        for (int i = 0; i < nslot; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NS);
        }
        for (int i = 0; i < kSResSlots; ++i) {
            mbar_init(&full_r[i], 1);
            mbar_init(&empty_r[i], NS);
        }
        for (int i = 0; i < NPB; ++i) {
            mbar_init(&pdone[i], NS);
            mbar_init(&pfree[i], 1);
        }
        for (int i = 0; i < NX; ++i) {
            mbar_init(&xbar[i], C);
            mbar_init(&xfree[i], C);
        }
        for (int i = 0; i < NR; ++i) {
            mbar_init(&xrbar[i], C);
            mbar_init(&xrfree[i], C);
            mbar_init(&resdone[i], NS);
            resreq[i] = 0;
        }
        rows_done = 0;
        tr_cnt = 0;
        tr_state[1] = dbg;
        for (int i = 0; i < 16; ++i) ctr[i] = 0ull;
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();   // every CTA's barriers are initialised before any remote arrive
    if (tid == 0) trace_ev(tr, &tr_cnt, kEvStart, 0);

    auto row_of = [&](int t) { return g + t * G; };
    auto p_row = [&](int row) -> const E* {
        const int j = row / P.B, b = row % P.B;
        return static_cast<const E*>(P.p) + (static_cast<int64_t>(b) * (kk + 1) + j) * P.ld_p + s0;
    };
    auto q_row = [&](int row) -> const E* {
        const int j = row / P.B, b = row % P.B;
        return static_cast<const E*>(P.q) + (static_cast<int64_t>(b) * kk + j) * P.ld_q + s0;
    };

    // warp roles: 0 main-ring producer | 1..NS stats | NS+1..NS+NR row warps |
    // NS+NR+1 residual-ring producer

    if (warp == 0 || warp > NS + NR) {
        // =============================== producers ==========================================
        // Two rings: the main ring (stats pieces, skip markers, the end marker) and a small
        // priority ring for residual re-reads, so a residual pass never queues behind the
        // stats pieces already in flight.
        if (warp == NS + NR + 1) {
          if (lane == 0 && T > 0) {
            // ---- residual ring (its own warp: TMA copies from one thread serialise) -----------
            uint32_t m = 0;
            int rjob = 0, rt = 0, rr = 0, rpiece = 0, rhasq = 0;
            const E* rp_ = nullptr;
            const E* rq_ = nullptr;
            uint32_t pend = 0;       // row warps with a pending residual request
            int pend_t[NR];
            for (int r = 0; r < NR; ++r) pend_t[r] = 0;
            for (;;) {
                bool progress = false;
                for (int r = 0; r < NR; ++r) {
                    const int v = ld_acq_s32(&resreq[r]);
                    if (v) {
                        pend |= 1u << r;
                        pend_t[r] = v - 1;
                        resreq[r] = 0;
                    }
                }
                if (!rjob && pend) {
                    rr = __ffs(pend) - 1;
                    pend &= pend - 1;
                    rt = pend_t[rr];
                    const int row = row_of(rt);
                    rhasq = (!GREEDY && row / P.B < kk) ? 1 : 0;
                    rp_ = p_row(row);
                    rq_ = rhasq ? q_row(row) : nullptr;
                    rpiece = 0;
                    rjob = 1;
                }
                if (rjob) {
                    const int s = m % kSResSlots, s2 = (m + 1) % kSResSlots;
                    if (mbar_test_wait(&empty_r[s], ((m / kSResSlots) & 1) ^ 1) &&
                        (!rhasq || mbar_test_wait(&empty_r[s2], (((m + 1) / kSResSlots) & 1) ^ 1))) {
                        const uint32_t off = static_cast<uint32_t>(rpiece) * kPiece;
                        const uint32_t nb = min(kPiece, sbytes - off);
                        const bool last = rpiece == npc - 1;
                        pinfo_r[s] = PInfo{kResid, rt, rpiece, (last ? 1 : 0) | (rhasq << 1) | (rr << 8)};
                        mbar_arrive_expect_tx(&full_r[s], nb);
                        bulk_g2s(rring + static_cast<size_t>(s) * kPiece,
                                 reinterpret_cast<const char*>(rp_) + off, nb, &full_r[s]);
                        if (rhasq) {
                            mbar_arrive_expect_tx(&full_r[s2], nb);
                            bulk_g2s(rring + static_cast<size_t>(s2) * kPiece,
                                     reinterpret_cast<const char*>(rq_) + off, nb, &full_r[s2]);
                        }
                        m += 1 + rhasq;
                        trace_ev(tr, &tr_cnt, kEvIssueR, rt);
                        if (++rpiece == npc) rjob = 0;
                        progress = true;
                    }
                }
                if (!rjob && !pend && ld_acq_s32(&rows_done) >= T) break;
                if (!progress) __nanosleep(256);
            }
          }
        } else if (lane < kSProducers && T > 0) {
            // ---- main ring: stats pieces, skip markers, the end marker --------------------------
            // Lanes 0..kSProducers-1 run the same planning code (lane 0 reads the stop mask and
            // broadcasts it, so they agree on every skip); lane n % kSProducers
            // issues entry n.  Bulk copies issued by one thread complete one after another
            // (tools/tma_probe), so alternating issuing lanes keeps several copies in flight.
            const unsigned pm = (1u << kSProducers) - 1u;
            uint32_t n = 0;
            int s = 0, ph = 0;                  // ring slot / phase of entry n
            int t_next = 0, tp = 0, tph = 0;    // next row, its partial slot and phase
            int job = 0, jt = 0, jpiece = 0, jq = 0, jhasq = 0;
            uint32_t jleft = 0;                 // bytes of the current row slice still to stage
            const char* jsrc = nullptr;
            const char* jqsrc = nullptr;
            int row = g, jrow = row / P.B, brow = row - jrow * P.B;   // row = g + t*G = jrow*B + brow
            unsigned long long cw_e = 0, cw_p = 0;
            const unsigned long long c_t0 = clock64();
            for (;;) {
                const bool fin = !(t_next < T || job);
                if (fin) {
                    while (ld_acq_s32(&rows_done) < T) __nanosleep(256);   // end marker last
                }
                PInfo info;
                const char* src = nullptr;
                uint32_t nb = 0;
                if (fin) {
                    info = PInfo{kEnd, 0, 0, 0};
                } else {
                    if (!job) {
                        // the row's partial slot must be free before any of its entries is queued
                        wait_local_t(&pfree[tp], tph ^ 1, cw_p);
                        uint32_t msk = 0u;
                        if (lane == 0 && !(dbg & 2)) msk = ld_relaxed_u32(P.rej_mask + brow);
                        msk = __shfl_sync(pm, msk, 0);   // one read: every lane takes the same decision
                        const bool skip = (msk & ((1u << jrow) - 1u)) != 0u;
                        if (skip) {
                            info = PInfo{kSkip, t_next, 0, 1};
                        } else {
                            jt = t_next;
                            jhasq = (!GREEDY && jrow < kk) ? 1 : 0;
                            jsrc = reinterpret_cast<const char*>(
                                static_cast<const E*>(P.p) + (static_cast<int64_t>(brow) * (kk + 1) + jrow) * P.ld_p + s0);
                            jqsrc = jhasq ? reinterpret_cast<const char*>(
                                               static_cast<const E*>(P.q) + (static_cast<int64_t>(brow) * kk + jrow) * P.ld_q + s0)
                                          : nullptr;
                            jpiece = 0;
                            jq = 0;
                            jleft = sbytes;
                            job = 1;
                        }
                        // advance to the next row of this cluster (incremental: no division)
                        ++t_next;
                        if (++tp == NPB) {
                            tp = 0;
                            tph ^= 1;
                        }
                        row += G;
                        brow += G;
                        while (brow >= P.B) {
                            brow -= P.B;
                            ++jrow;
                        }
                    }
                    if (job) {
                        nb = jleft < kPiece ? jleft : kPiece;
                        src = (jq ? jqsrc : jsrc) + static_cast<size_t>(jpiece) * kPiece;
                        const bool last = nb == jleft && (jq || !jhasq);
                        info = PInfo{jq ? kStatQ : kStatP, jt, jpiece, last ? 1 : 0};
                        jleft -= nb;
                        ++jpiece;
                        if (jleft == 0) {
                            if (jhasq && !jq) {
                                jq = 1;
                                jpiece = 0;
                                jleft = sbytes;
                            } else {
                                job = 0;
                            }
                        }
                    }
                }
                if (lane == static_cast<int>(n % kSProducers)) {
                    if (!mbar_test_wait(&empty[s], ph ^ 1)) {   // critical path: short backoff
                        const unsigned long long c0 = clock64();
                        wait_poll(&empty[s], ph ^ 1, 32);
                        cw_e += clock64() - c0;
                    }
                    pinfo[s] = info;
                    if (info.kind == kStatP || info.kind == kStatQ) {
                        if (dbg & 128) {
                            mbar_arrive(&full[s]);   // bisection: no data movement
                        } else {
                            mbar_arrive_expect_tx(&full[s], nb);
                            bulk_g2s(smem + static_cast<size_t>(s) * kPiece, src, nb, &full[s]);
                        }
                    } else {
                        mbar_arrive(&full[s]);
                    }
                }
                __syncwarp(pm);
                ++n;
                if (++s == nslot) {
                    s = 0;
                    ph ^= 1;
                }
                if (fin) break;
            }
            if (tr && lane == 0) {
                atomicAdd(&ctr[4], cw_e);
                atomicAdd(&ctr[5], cw_p);
                atomicAdd(&ctr[6], clock64() - c_t0);
            }
        } else if (lane == 0 && warp == 0) {   // no rows: still terminate the stats warps
            pinfo[0] = PInfo{kEnd, 0, 0, 0};
            mbar_arrive(&full[0]);
        }
    } else if (warp <= NS) {
        // =============================== stats warps ========================================
        const int sw = warp - 1;            // stats warp index
        const int u = tid - 32;             // stats thread index
        uint32_t m = 0;                     // residual ring position
        int s = 0, ph = 0;                  // main ring slot and phase parity
        float mP = -INFINITY, mQ = -INFINITY, dP = -INFINITY, dQ = -INFINITY;
        float sP = 0.0f, sQ = 0.0f;
        int nf = 0;
        float gbest = -INFINITY;
        int gidx = INT_MAX;
        uint32_t spins = 0;
        unsigned long long cw_f = 0, c_np = 0, c_nr = 0, c_cmp = 0, c_res = 0;
        const unsigned long long c_t0 = clock64();
        unsigned long long c_w0 = 0;
        bool waiting = false;
        for (;;) {
            // ---- residual ring first (p in slot sr, q in the next slot) ---------------------
            const int sr = m % kSResSlots;
            if (mbar_test_wait(&full_r[sr], (m / kSResSlots) & 1)) {
                const unsigned long long c_r0 = tr ? clock64() : 0ull;
                const PInfo pi = pinfo_r[sr];
                const int hasq = (pi.aux >> 1) & 1;
                const int rw = pi.aux >> 8;
                const int sr2 = (m + 1) % kSResSlots;
                if (hasq) wait_poll(&full_r[sr2], ((m + 1) / kSResSlots) & 1, 32);
                const uint4* slot = reinterpret_cast<const uint4*>(rring + static_cast<size_t>(sr) * kPiece);
                const uint4* slot2 = reinterpret_cast<const uint4*>(rring + static_cast<size_t>(sr2) * kPiece);
                const RParams rp = rparams[rw];
                const int base = pi.idx * PV;
                const int pv_hi = min(nvec - base, PV);              // vectors staged in this piece
                const int nsp = (pv_hi + SEGV - 1) / SEGV;            // segments in this piece
                double2* seg = segbuf + static_cast<size_t>(rw) * P.segmax;
                for (int sg = sw; sg < nsp; sg += NS) {
                    const int vv = sg * SEGV + lane;
                    const int gv = base + vv;                         // slice vector index
                    const int valid = min(VEC, max(0, len - gv * VEC));
                    uint4 up = make_uint4(0, 0, 0, 0), uq = up;
                    if (vv < pv_hi) {
                        up = slot[vv];
                        if (hasq) uq = slot2[vv];
                    }
                    float r[VEC], pv[VEC], srr, spv;
                    vec_terms<E>(up, uq, valid, rp, c2, r, pv, srr, spv);
                    const double2 inc = warp_scan2(make_double2(srr, spv), lane);
                    if (lane == 31) seg[base / SEGV + sg] = inc;
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty_r[sr]);
                    if (hasq) mbar_arrive(&empty_r[sr2]);
                    if (pi.aux & 1) mbar_arrive(&resdone[rw]);
                    if (sw == 0) trace_ev(tr, &tr_cnt, kEvResPiece, pi.t);
                }
                m += 1 + hasq;
                ++c_nr;
                (void)c_r0;
                continue;
            }
            // ---- main ring ------------------------------------------------------------------
            if (!mbar_test_wait(&full[s], ph)) {
                __nanosleep(32);
                if (++spins > kSpinLimit) wait_fail("stats full", &full[s], ph);
                ++c_res;
                if (!waiting) {
                    waiting = true;
                    c_w0 = clock64();
                }
                continue;
            }
            if (waiting) {
                cw_f += clock64() - c_w0;
                waiting = false;
            }
            ++c_np;
            spins = 0;
            const PInfo pi = pinfo[s];
            if (pi.kind == kEnd) {
                if (tr && lane == 0) {
                    atomicAdd(&ctr[0], cw_f);
                    atomicAdd(&ctr[1], clock64() - c_t0);
                    atomicAdd(&ctr[2], c_np);
                    atomicAdd(&ctr[3], c_nr);
                    atomicAdd(&ctr[12], c_cmp);
                    atomicAdd(&ctr[13], c_res);
                }
                break;
            }
            const uint4* slot = reinterpret_cast<const uint4*>(smem + static_cast<size_t>(s) * kPiece);
            if (pi.kind == kSkip) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == nslot) {
                    s = 0;
                    ph ^= 1;
                }
                if (lane == 0) part[pi.t % NPB][sw] = WPart{0.f, 0.f, 0.0, 0.0, kFlagSkip, INT_MAX};
                __syncwarp();
                if (lane == 0) mbar_arrive(&pdone[pi.t % NPB]);
                continue;
            }
            const bool isq = pi.kind == kStatQ;
            if (!isq && pi.idx == 0) {   // first piece of a new row
                mP = mQ = dP = dQ = -INFINITY;
                sP = sQ = 0.0f;
                nf = 0;
                gbest = -INFINITY;
                gidx = INT_MAX;
            }
            const int base = pi.idx * PV;                // slice vector index of the piece
            const int hi = min(nfull - base, PV);        // complete vectors in the piece
            constexpr int KV = PV / NST;                 // vectors per thread per piece
            float v[KV][VEC];
            int nv = 0;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int vv = u + i * NST;
                if (vv < hi) {
                    EL::unpack(slot[vv], v[i]);
                    nv = i + 1;
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) v[i][e] = -INFINITY;
                }
            }
            // ragged last vector of the slice: its past-the-end lanes are -inf
            if (base + hi < nvec && hi < PV && u == hi % NST) {
                const int ir = hi / NST;
                float w[VEC];
                EL::unpack(slot[hi], w);
                const int valid = len - (base + hi) * VEC;
#pragma unroll
                for (int i = 0; i < KV; ++i)
                    if (i == ir) {
#pragma unroll
                        for (int e = 0; e < VEC; ++e) v[i][e] = e < valid ? w[e] : -INFINITY;
                    }
                nv = ir + 1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);   // values are in registers
            if (lane == 0 && sw == 0) trace_ev(tr, &tr_cnt, kEvConsume, pi.t);
            const unsigned long long c_cmp0 = tr ? clock64() : 0ull;
            if (++s == nslot) {
                s = 0;
                ph ^= 1;
            }
            if (dbg & 1) {
                // bandwidth probe: consume the values without the arithmetic
                float a = 0.0f;
#pragma unroll
                for (int i = 0; i < KV; ++i) a += v[i][0];
                if (a == 1234.5f) nf |= 16;
            } else if (GREEDY) {
                float nanacc = -INFINITY;
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    float vm = -INFINITY;
#pragma unroll
                    for (int e = 0; e < VEC; e += 2) {
                        nanacc = max3nan(nanacc, v[i][e], v[i][e + 1]);
                        vm = max3(vm, v[i][e], v[i][e + 1]);
                    }
                    if (vm > gbest) {
                        int fe = 0;
#pragma unroll
                        for (int e = VEC - 1; e >= 0; --e)
                            if (v[i][e] == vm) fe = e;
                        gbest = vm;
                        gidx = s0 + (base + u + i * NST) * VEC + fe;
                    }
                }
                if (!(nanacc < INFINITY)) nf |= kFlagNfP;
            } else if (nv > 0) {
                if (isq) online_acc<VEC, KV>(v, c2, isq, mQ, dQ, sQ, nf);
                else online_acc<VEC, KV>(v, c2, isq, mP, dP, sP, nf);
            }
            if (tr) c_cmp += clock64() - c_cmp0;
            if (pi.aux & 1) {   // last piece of the row: warp partial
                const int tp = pi.t % NPB;
                WPart wp;
                wp.flags = __reduce_or_sync(0xFFFFFFFFu, nf);
                if (GREEDY) {
                    float bv = gbest;
                    int bi = gidx;
                    warp_argmax(bv, bi);
                    wp.dP = bv;
                    wp.gidx = bi;
                    wp.dQ = -INFINITY;
                    wp.sP = wp.sQ = 0.0;
                } else {
                    const float Dw = warp_max(dP), Ew = warp_max(dQ);
                    wp.sP = warp_sum(sP > 0.0f ? static_cast<double>(sP * ex2_approx(dP - Dw)) : 0.0);
                    wp.sQ = warp_sum(sQ > 0.0f ? static_cast<double>(sQ * ex2_approx(dQ - Ew)) : 0.0);
                    wp.dP = Dw;
                    wp.dQ = Ew;
                    wp.gidx = INT_MAX;
                }
                if (lane == 0) part[tp][sw] = wp;
                __syncwarp();
                if (lane == 0) mbar_arrive(&pdone[tp]);
            }
        }
    } else {
        // =============================== row warps (warps NS+1 .. NS+NR) ====================
        const int rw = warp - 1 - NS;
        uint32_t nres = 0;                  // residual passes of this row warp
        unsigned long long cw_pd = 0, cw_x = 0, cw_rd = 0, cw_xr = 0;
        const unsigned long long c_t0 = clock64();
        for (int t = rw; t < T; t += NR) {
            const int row = row_of(t);
            const int j = row / P.B, b = row % P.B;
            const bool has_q = !GREEDY && j < kk;
            const int x = x_for(P, b, j);
            // Philox words of (j, round, rid) -- C-8
            uint4 w = make_uint4(0, 0, 0, 0);
            if (lane == 0)
                w = verify_words(P.seed, static_cast<uint32_t>(j), P.round, P.rid_base + static_cast<uint64_t>(b));
            // ---- 1. combine the stats warps' partials --------------------------------------
            const int tp = t % NPB;
            wait_local_t(&pdone[tp], (t / NPB) & 1, cw_pd);
            const bool on = lane < NS;
            WPart wp = on ? part[tp][lane] : WPart{-INFINITY, -INFINITY, 0.0, 0.0, 0, INT_MAX};
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfree[tp]);
                trace_ev(tr, &tr_cnt, kEvPdone, t);
            }
            if (dbg & 4) {   // bisection: no exchange / decision (results are wrong)
                if (lane == 0) {
                    if (rank == 0) arrive_row(P, b, j, true, -1, 0);
                    atomicAdd(&rows_done, 1);
                }
                continue;
            }
            Xch mine;
            mine.flags = __reduce_or_sync(0xFFFFFFFFu, wp.flags);
            if (GREEDY) {
                float bv = wp.dP;
                int bi = wp.gidx;
                warp_argmax(bv, bi);
                mine.dP = bv;
                mine.gidx = bi;
                mine.dQ = -INFINITY;
                mine.sP = mine.sQ = 0.0;
            } else {
                const float Dc = warp_max(wp.dP), Ec = warp_max(wp.dQ);
                mine.sP = warp_sum(wp.sP > 0.0 ? wp.sP * static_cast<double>(ex2_approx(wp.dP - Dc)) : 0.0);
                mine.sQ = warp_sum(wp.sQ > 0.0 ? wp.sQ * static_cast<double>(ex2_approx(wp.dQ - Ec)) : 0.0);
                mine.dP = Dc;
                mine.dQ = Ec;
                mine.gidx = INT_MAX;
            }
            mine.zxp = 0.0f;
            mine.zxq = 0.0f;
            if (x >= s0 && x < s0 + len && !(mine.flags & kFlagSkip)) {
                mine.flags |= kFlagHasX;
                if (lane == 0) {
                    const E* pr = p_row(row);
                    if (sizeof(E) == 4) {
                        mine.zxp = __ldg(reinterpret_cast<const float*>(pr) + (x - s0));
                        if (has_q) mine.zxq = __ldg(reinterpret_cast<const float*>(q_row(row)) + (x - s0));
                    } else {
                        mine.zxp = __uint_as_float(static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(pr) + (x - s0))) << 16);
                        if (has_q)
                            mine.zxq = __uint_as_float(static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(q_row(row)) + (x - s0))) << 16);
                    }
                }
                mine.zxp = __shfl_sync(0xFFFFFFFFu, mine.zxp, 0);
                mine.zxq = __shfl_sync(0xFFFFFFFFu, mine.zxq, 0);
            }
            // ---- 2. exchange with the cluster ----------------------------------------------
            const int sx = t % NX;
            wait_cluster_t(&xfree[sx], ((t / NX) & 1) ^ 1, cw_x);   // every peer has read the slot's last use
            if (lane < C) {
                Xch* dst = &xch[sx][rank];
                const uint32_t a = mapa(dst, lane);
                st_cl_f64(a + offsetof(Xch, sP), mine.sP);
                st_cl_f64(a + offsetof(Xch, sQ), mine.sQ);
                st_cl_u32(a + offsetof(Xch, dP), __float_as_uint(mine.dP));
                st_cl_u32(a + offsetof(Xch, dQ), __float_as_uint(mine.dQ));
                st_cl_u32(a + offsetof(Xch, zxp), __float_as_uint(mine.zxp));
                st_cl_u32(a + offsetof(Xch, zxq), __float_as_uint(mine.zxq));
                st_cl_u32(a + offsetof(Xch, flags), static_cast<uint32_t>(mine.flags));
                st_cl_u32(a + offsetof(Xch, gidx), static_cast<uint32_t>(mine.gidx));
                mbar_arrive_remote(mapa(&xbar[sx], lane));
            }
            wait_cluster_t(&xbar[sx], (t / NX) & 1, cw_x);
            const bool onc = lane < C;
            Xch pc;
            if (onc) pc = xch[sx][lane];
            __syncwarp();
            if (onc) mbar_arrive_remote(mapa(&xfree[sx], lane));   // ack: slot read
            if (lane == 0) trace_ev(tr, &tr_cnt, kEvXch, t);
            const int f = __reduce_or_sync(0xFFFFFFFFu, onc ? pc.flags : 0);
            const unsigned hx = __ballot_sync(0xFFFFFFFFu, onc && (pc.flags & kFlagHasX));
            float zxp = 0.0f, zxq = 0.0f;
            if (hx) {
                const int src = __ffs(hx) - 1;
                zxp = __shfl_sync(0xFFFFFFFFu, onc ? pc.zxp : 0.0f, src);
                zxq = __shfl_sync(0xFFFFFFFFu, onc ? pc.zxq : 0.0f, src);
            }
            float Dp, Dq = -INFINITY;
            double Sp = 0.0, Sq = 0.0;
            int Gi = INT_MAX;
            if (GREEDY) {
                Dp = onc ? pc.dP : -INFINITY;
                Gi = onc ? pc.gidx : INT_MAX;
                warp_argmax(Dp, Gi);
            } else {
                const float d = onc ? pc.dP : -INFINITY, e = onc ? pc.dQ : -INFINITY;
                const double sp = onc ? pc.sP : 0.0, sq = onc ? pc.sQ : 0.0;
                Dp = warp_max(d);
                Dq = warp_max(e);
                Sp = warp_sum(sp > 0.0 ? sp * static_cast<double>(ex2_approx(d - Dp)) : 0.0);
                Sq = warp_sum(sq > 0.0 ? sq * static_cast<double>(ex2_approx(e - Dq)) : 0.0);
            }
            // ---- 3. decision (identical in every CTA of the cluster) --------------------------
            int st = 0, stop = 0;
            if (lane == 0 && !(f & kFlagSkip)) {
                if (j < kk && (x < 0 || x >= P.V)) st = kBadId;
                if (!st) {
                    if (f & kFlagNfP) st = kNonfinite;
                    else if (Dp == -INFINITY) st = kEmptyRow;
                }
                if (!st && has_q) {
                    if (f & kFlagNfQ) st = kNonfinite;
                    else if (Dq == -INFINITY) st = kEmptyRow;
                }
                if (st) {
                    stop = 1;
                } else if (j < kk) {
                    if (GREEDY) {
                        stop = x != Gi;                                   // argmax matching (C-5)
                    } else if (zxq == -INFINITY) {
                        st = kZeroQ;                                      // q_j(x_j) = 0 (C-7)
                        stop = 1;
                    } else {
                        // a = p(x)/q(x) = 2^((z_p(x) c2 - D_p) - (z_q(x) c2 - D_q)) * S_q / S_p
                        const double c2d = static_cast<double>(c2);
                        const double l = (static_cast<double>(zxp) * c2d - static_cast<double>(Dp)) -
                                         (static_cast<double>(zxq) * c2d - static_cast<double>(Dq));
                        const double a = exp2(l) * (Sq / Sp);
                        if (!(a >= 1.0)) stop = unit24(w.x) >= a;        // reject iff u >= a (C-2)
                    }
                }
                if (rank == 0 && stop && j < kk) {   // publish the stop at once (laziness)
                    atomicOr(P.rej_mask + b, 1u << j);
                    __threadfence();
                }
            }
            st = __shfl_sync(0xFFFFFFFFu, st, 0);
            stop = __shfl_sync(0xFFFFFFFFu, stop, 0);
            const bool skipped = (f & kFlagSkip) != 0;
            const bool hard = (st & kHard) != 0;
            const bool resid = !GREEDY && !skipped && !hard && (stop || j == kk);
            if (lane == 0) trace_ev(tr, &tr_cnt, kEvDecide, t | (resid ? 0x8000 : 0) | (skipped ? 0x4000 : 0));
            if (!resid) {
                if (rank == 0 && lane == 0) {
                    if (skipped) arrive_row(P, b, j, false, -1, 0);
                    else arrive_row(P, b, j, stop || j == kk, (GREEDY && !hard) ? Gi : -1, st);
                }
            } else {
                // ---- 4. residual pass over my slice (stats warps, L2-resident re-read) -------
                RParams rp;
                rp.nDp = -Dp;
                rp.nDq = has_q ? -Dq : 0.0f;
                rp.ip = static_cast<float>(1.0 / Sp);
                rp.iq = has_q ? static_cast<float>(1.0 / Sq) : 0.0f;
                rp.use_q = has_q ? 1 : 0;
                if (lane == 0) {
                    rparams[rw] = rp;
                    st_rel_s32(&resreq[rw], t + 1);
                }
                wait_local_t(&resdone[rw], nres & 1, cw_rd);
                if (lane == 0) trace_ev(tr, &tr_cnt, kEvResDone, t);
                // slice masses: chunked prefix over the segment table (fixed association)
                const double2* seg = segbuf + static_cast<size_t>(rw) * P.segmax;
                double2 carry = make_double2(0.0, 0.0);
                for (int c0 = 0; c0 < nseg; c0 += 32) {
                    const double2 v = c0 + lane < nseg ? seg[c0 + lane] : make_double2(0.0, 0.0);
                    double2 inc = warp_scan2(v, lane);
                    inc.x = __dadd_rn(inc.x, carry.x);
                    inc.y = __dadd_rn(inc.y, carry.y);
                    carry.x = __shfl_sync(0xFFFFFFFFu, inc.x, 31);
                    carry.y = __shfl_sync(0xFFFFFFFFu, inc.y, 31);
                }
                // exchange (R_c, P_c)
                wait_cluster_t(&xrfree[rw], (nres & 1) ^ 1, cw_xr);
                if (lane < C) {
                    const uint32_t a = mapa(&xres[rw][rank], lane);
                    st_cl_f64(a, carry.x);
                    st_cl_f64(a + 8, carry.y);
                    mbar_arrive_remote(mapa(&xrbar[rw], lane));
                }
                wait_cluster_t(&xrbar[rw], nres & 1, cw_xr);
                const double2 rc = onc ? xres[rw][lane] : make_double2(0.0, 0.0);
                __syncwarp();
                if (onc) mbar_arrive_remote(mapa(&xrfree[rw], lane));
                ++nres;
                const double2 ic = warp_scan2(rc, lane);
                const double Rt = __shfl_sync(0xFFFFFFFFu, ic.x, 31);
                const bool zres = !(Rt > 0.0);          // C-6: no residual mass -> sample from p_L
                const double tot = zres ? __shfl_sync(0xFFFFFFFFu, ic.y, 31) : Rt;
                const double mc = zres ? rc.y : rc.x, icm = zres ? ic.y : ic.x;
                const double theta = unit24(__shfl_sync(0xFFFFFFFFu, w.y, 0)) * tot;   // C-9
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, onc && icm > theta);
                const unsigned posm = __ballot_sync(0xFFFFFFFFu, onc && mc > 0.0);
                const int cs = hit ? __ffs(hit) - 1 : (posm ? 31 - __clz(posm) : 0);
                double exc = __shfl_up_sync(0xFFFFFFFFu, icm, 1);
                if (lane == 0) exc = 0.0;
                exc = __shfl_sync(0xFFFFFFFFu, exc, cs);
                const int status = st | (zres ? kZeroResidual : 0);
                if (!(tot > 0.0)) {
                    // cannot happen for a finite row (its max has p >= 1/V); never hang the request
                    if (rank == 0 && lane == 0) arrive_row(P, b, j, true, -1, status);
                } else if (rank == cs) {
                    // ---- 5. token search in this slice: segment -> lane -> element ----------
                    const double th1 = hit ? theta - exc : INFINITY;
                    int sgf = -1, sglast = -1;
                    double sexc = 0.0;
                    carry = make_double2(0.0, 0.0);
                    for (int c0 = 0; c0 < nseg && sgf < 0; c0 += 32) {
                        const double2 v = c0 + lane < nseg ? seg[c0 + lane] : make_double2(0.0, 0.0);
                        double2 inc = warp_scan2(v, lane);
                        inc.x = __dadd_rn(inc.x, carry.x);
                        inc.y = __dadd_rn(inc.y, carry.y);
                        const double icv = zres ? inc.y : inc.x, mv = zres ? v.y : v.x;
                        const unsigned h = __ballot_sync(0xFFFFFFFFu, c0 + lane < nseg && icv > th1);
                        const unsigned pm = __ballot_sync(0xFFFFFFFFu, c0 + lane < nseg && mv > 0.0);
                        if (pm) sglast = c0 + 31 - __clz(pm);
                        if (h) {
                            const int l = __ffs(h) - 1;
                            sgf = c0 + l;
                            double e2 = __shfl_up_sync(0xFFFFFFFFu, icv, 1);
                            const double cz = zres ? carry.y : carry.x;
                            if (lane == 0) e2 = cz;
                            sexc = __shfl_sync(0xFFFFFFFFu, e2, l);
                        }
                        carry.x = __shfl_sync(0xFFFFFFFFu, inc.x, 31);
                        carry.y = __shfl_sync(0xFFFFFFFFu, inc.y, 31);
                    }
                    const bool sclamp = sgf < 0;
                    if (sclamp) sgf = sglast >= 0 ? sglast : 0;
                    const double th2 = sclamp ? INFINITY : th1 - sexc;
                    // recompute the segment exactly as the stats warps did (bit-identical terms)
                    const int gv = sgf * SEGV + lane;
                    const int valid = min(VEC, max(0, len - gv * VEC));
                    uint4 up = make_uint4(0, 0, 0, 0), uq = up;
                    if (valid > 0) {
                        up = __ldg(reinterpret_cast<const uint4*>(p_row(row)) + gv);
                        if (has_q) uq = __ldg(reinterpret_cast<const uint4*>(q_row(row)) + gv);
                    }
                    float r[VEC], pv[VEC], sr, spv;
                    vec_terms<E>(up, uq, valid, rp, c2, r, pv, sr, spv);
                    const double2 inc = warp_scan2(make_double2(sr, spv), lane);
                    const double icv = zres ? inc.y : inc.x;
                    const float mine_s = zres ? spv : sr;
                    const unsigned h = __ballot_sync(0xFFFFFFFFu, icv > th2);
                    const unsigned pm = __ballot_sync(0xFFFFFFFFu, mine_s > 0.0f);
                    const int ls = h ? __ffs(h) - 1 : (pm ? 31 - __clz(pm) : 0);
                    double ex = __shfl_up_sync(0xFFFFFFFFu, icv, 1);
                    if (lane == 0) ex = 0.0;
                    if (lane == ls) {
                        const double th3 = h ? th2 - ex : INFINITY;
                        int fe = -1, lastpos = -1;
                        float cum = 0.0f;
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            const float te = zres ? pv[e] : r[e];
                            if (te > 0.0f) lastpos = e;
                            cum = e == 0 ? te : __fadd_rn(cum, te);
                            if (fe < 0 && static_cast<double>(cum) > th3) fe = e;
                        }
                        if (fe < 0) fe = lastpos >= 0 ? lastpos : 0;   // rounding: clamp (C-9)
                        arrive_row(P, b, j, true, s0 + gv * VEC + fe, status);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                atomicAdd(&rows_done, 1);
                trace_ev(tr, &tr_cnt, kEvRowEnd, t);
            }
        }
        if (tr && lane == 0) {
            atomicAdd(&ctr[7], cw_pd);
            atomicAdd(&ctr[8], cw_x);
            atomicAdd(&ctr[9], cw_rd);
            atomicAdd(&ctr[10], cw_xr);
            atomicAdd(&ctr[11], clock64() - c_t0);
        }
    }
    __syncwarp();
    __syncthreads();
    if (tid < 16 && tr) tr[static_cast<size_t>(blockIdx.x) * kSTraceN + kSTraceN - 16 + tid] = ctr[tid];
    if (tid == 0 && tr) {
        trace_ev(tr, &tr_cnt, kEvEnd, 0);
        tr[static_cast<size_t>(blockIdx.x) * kSTraceN] = static_cast<unsigned long long>(min(tr_cnt, kSTraceN - 17));
    }
    cluster_sync_all();   // no CTA leaves while a peer may still signal it
}

}  // namespace strm

// ------------------------------------------------------------------------------------------
// host side

void record_event(cudaEvent_t ev, cudaStream_t st);

namespace {
template <typename E, bool G>
struct SInfo {
    static bool init;
    static int max_dyn;
};
template <typename E, bool G>
bool SInfo<E, G>::init = false;
template <typename E, bool G>
int SInfo<E, G>::max_dyn = 0;

template <typename E, bool G>
int prepare_stream() {
    if (!SInfo<E, G>::init) {
        auto k = strm::k_verify_stream<E, G>;
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        SInfo<E, G>::max_dyn = optin - static_cast<int>(fa.sharedSizeBytes);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SInfo<E, G>::max_dyn);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        SInfo<E, G>::init = true;
    }
    return SInfo<E, G>::max_dyn;
}

template <typename E, bool G>
int stream_occupancy(int C, size_t smem) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C * 64);
    cfg.blockDim = dim3(strm::NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, strm::k_verify_stream<E, G>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int dispatch_prepare(int esz, bool greedy) {
    if (esz == 4) return greedy ? prepare_stream<float, true>() : prepare_stream<float, false>();
    return greedy ? prepare_stream<__nv_bfloat16, true>() : prepare_stream<__nv_bfloat16, false>();
}
int dispatch_occ(int esz, bool greedy, int C, size_t sm) {
    if (esz == 4) return greedy ? stream_occupancy<float, true>(C, sm) : stream_occupancy<float, false>(C, sm);
    return greedy ? stream_occupancy<__nv_bfloat16, true>(C, sm)
                  : stream_occupancy<__nv_bfloat16, false>(C, sm);
}
}  // namespace

// Target logits bytes per CTA slice of one row pair (p and q).  Smaller slices = more CTAs per
// row (lower per-row latency, better laziness), larger = fewer exchanges per byte.
static int stream_slice_target() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("STARSD_SLICE_KB");
        v = (e ? atoi(e) : 128) * 1024;
        if (v < 2048) v = 2048;
    }
    return v;
}

bool stream_config(int32_t V, int esz, bool greedy, StreamPlan* out) {
    const int vec = 16 / esz;
    const int64_t pair = static_cast<int64_t>(V) * esz * (greedy ? 1 : 2);
    int c = 1;
    while (c < 16 && pair > static_cast<int64_t>(stream_slice_target()) * c) c *= 2;
    {
        const char* e = getenv("STARSD_CLUSTER");
        if (e && atoi(e) >= 1 && atoi(e) <= 16) c = atoi(e);
    }
    int64_t w = (V + c - 1) / c;
    w = (w + vec - 1) / vec * vec;
    const int64_t nvec = w / vec;
    const int64_t segmax = (nvec + strm::SEGV - 1) / strm::SEGV;
    const int max_dyn = dispatch_prepare(esz, greedy);
    const size_t segbytes = static_cast<size_t>(strm::NR) * segmax * 16;
    const int64_t nslot = (static_cast<int64_t>(max_dyn) - static_cast<int64_t>(segbytes)) / strm::kPiece -
                          kSResSlots;
    if (nslot < 4) return false;
    const int ns = static_cast<int>(nslot > kSMaxSlots ? kSMaxSlots : nslot);
    const size_t sm = static_cast<size_t>(ns + kSResSlots) * strm::kPiece + segbytes;
    struct Entry { int c; size_t sm; int esz, greedy, n; };
    static Entry cache[32];
    static int ncache = 0;
    int n = -1;
    for (int i = 0; i < ncache; ++i)
        if (cache[i].c == c && cache[i].sm == sm && cache[i].esz == esz && cache[i].greedy == (int)greedy)
            n = cache[i].n;
    if (n < 0) {
        n = dispatch_occ(esz, greedy, c, sm);
        if (ncache < 32) cache[ncache++] = Entry{c, sm, esz, (int)greedy, n};
    }
    if (n <= 0) return false;
    out->C = c;
    out->G = n;
    out->W = static_cast<int32_t>(w);
    out->segmax = static_cast<int32_t>(segmax);
    out->nslot = ns;
    out->smem = sm;
    return true;
}

cudaError_t launch_stream(const SParams& P, bool greedy, bool bf16, size_t smem, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(P.G) * P.C);
    cfg.blockDim = dim3(strm::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    record_event(ev0, st);
    cudaError_t e;
    if (greedy)
        e = bf16 ? cudaLaunchKernelEx(&cfg, strm::k_verify_stream<__nv_bfloat16, true>, P)
                 : cudaLaunchKernelEx(&cfg, strm::k_verify_stream<float, true>, P);
    else
        e = bf16 ? cudaLaunchKernelEx(&cfg, strm::k_verify_stream<__nv_bfloat16, false>, P)
                 : cudaLaunchKernelEx(&cfg, strm::k_verify_stream<float, false>, P);
    record_event(ev1, st);
    return e;
}

}  // namespace sd
