// verify_cluster.cu -- v3 (default): one thread-block CLUSTER per (request, position) row pair.
//
// The method (Alg. 2; readings C-1..C-12 of DESIGN.md), per request b:
//   accept x_j iff u_acc(j) < min(1, p_j(x_j) / q_j(x_j)),  L = first rejection (else k),
//   emit x_0..x_{L-1} and t ~ norm(max(0, p_L - q_L)) (L < k) or t ~ p_k (L == k).
//
// One launch, grid = (k+1) * B clusters of C CTAs, in POSITION-MAJOR order (all requests'
// position 0 first).  Cluster (j, b) owns the row pair (p_j, q_j) of request b; CTA `rank` of
// the cluster owns the vocabulary slice [rank*W, rank*W + W) and keeps it in shared memory for
// the whole life of the row:
//
//   A  rank 0 reads rej_mask[b]; if an earlier position already stopped the chain the row is
//      never needed (laziness) and the cluster only takes its ticket.
//   1  TMA 1-D bulk copies (16 KB pieces, one mbarrier each) stage the slice of p_j and q_j.
//      Sweep 1: NaN-propagating max per thread (FMNMX3.NAN).  Sweep 2: sum of
//      2^(z*c2 - d_t), d_t = fl(max_t * c2), with FFMA2 + MUFU.EX2 + FADD2 (c2 = log2(e)/T).
//   B  per-CTA (D, S) partials are exchanged through distributed shared memory; every CTA of
//      the cluster combines the C partials in the same order and takes the same decision
//      (ratio rule with the shared Philox uniform, C-1/C-2/C-8); rank 0 publishes a stop in
//      rej_mask[b] at once so later positions of b can skip their loads.
//   C  if this row stops (or is the bonus row k) the residual max(0, p - q) (or p) is computed
//      from the slice STILL IN SHARED MEMORY: per-thread contiguous ranges, fp64 prefix across
//      threads / warps / CTAs (DSMEM), and the CTA holding theta = u_smp * R finds the token.
//      No logit is read from HBM twice.
//   D  the row's publisher writes (token, status), takes the request's ticket; the last of the
//      k+1 rows of a request writes out_accept_len / out_tokens / out_status.
//
// Greedy (T = 0): p rows only; per-slice (max, lowest argmax) replaces the sums; no residual.
// No tensor cores: the step is a streaming reduction, not a contraction.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "philox.cuh"
#include "ptx.cuh"
#include "verify.cuh"

namespace sd {
namespace clu {

namespace cgx = cooperative_groups;

constexpr int NT = kCThreads;
constexpr int NW = NT / 32;
constexpr uint32_t kPieceBytes = 16384;   // one bulk copy (>= 16 KB copies stream at ~7.3 TB/s)
constexpr int kMaxPieces = kCMaxPieces;

constexpr int32_t kBadId = 1, kNonfinite = 2, kEmptyRow = 4, kZeroQ = 8, kZeroResidual = 16;
constexpr int32_t kHard = kBadId | kNonfinite | kEmptyRow;
constexpr int kFlagNfP = 1, kFlagNfQ = 2, kFlagHasX = 4;

// ---- element types: one 16-byte vector = 4 fp32 or 8 bf16 logits -------------------------
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

// ---- arithmetic helpers ------------------------------------------------------------------
__device__ __forceinline__ float max3nan(float a, float b, float c) {   // FMNMX3.NAN
    float d;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {      // FMNMX3 (NaN-ignoring)
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
                                                    unsigned long long c) {   // FFMA2
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
// 2^x of both halves (MUFU.EX2 x2)
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
// inclusive Kogge-Stone scan over the 32 lanes (fixed association: deterministic)
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v = __dadd_rn(v, n);
    }
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

// ---- cluster barrier (all threads of all CTAs; release/acquire at cluster scope) ----------
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// What one CTA publishes to its cluster peers (read through distributed shared memory).
struct Xch {
    double S_p, S_q;     // slice sum of 2^(z*c2 - D) (sampled)
    double R[2];         // slice residual mass (attempt 0: max(0,p-q); attempt 1: p, C-6)
    float D_p, D_q;      // slice max of fl(z_max*c2) (sampled) | raw max of p (greedy)
    float zx_p, zx_q;    // logits at the draft token if it lies in this slice
    int flags;           // kFlagNfP | kFlagNfQ | kFlagHasX
    int argmax;          // greedy: lowest index of the slice max (global token id)
    int skip;            // rank 0's view of the laziness test (the cluster's decision)
};

// Row decision, broadcast to the CTA through shared memory.
struct Dec {
    double S_p, S_q, u_smp;
    float D_p, D_q;
    int stop, status, token;
};

// The row's result is published; the last of the k+1 rows of request b emits its output.
__device__ void arrive_row(const CParams& P, int b, int j, bool write, int token, int status) {
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

// Residual terms of one 16-byte vector g of the slice, in ascending token order:
//   r(x) = max(0, p(x) - q(x)),  p(x) = 2^(z_p*c2 - D_p) / S_p  (q likewise)
//   or r = p (bonus row / zero-residual fallback, use_q = false).
// Returns the sequential fp32 sum r0 + r1 + ... (the same order the token search re-uses).
template <typename E>
__device__ __forceinline__ float vec_resid(const E* sp, const E* sq, int g, int len, bool use_q,
                                           float c2, float nDp, float nDq, float ip, float iq,
                                           float (&r)[Elt<E>::VEC]) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    float v[VEC];
    EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
    const unsigned long long cc = pk(c2, c2), np = pk(nDp, nDp), ipp = pk(ip, ip);
    float e[VEC];
#pragma unroll
    for (int u = 0; u < VEC; u += 2) {
        const unsigned long long x = ex2x2(ffma2(pk(v[u], v[u + 1]), cc, np));
        upk(x, e[u], e[u + 1]);
    }
    if (use_q) {
        float w[VEC];
        EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), w);
        const unsigned long long nq = pk(nDq, nDq), iqq = pk(iq, iq);
#pragma unroll
        for (int u = 0; u < VEC; u += 2) {
            const unsigned long long eq = ex2x2(ffma2(pk(w[u], w[u + 1]), cc, nq));
            const unsigned long long t = fmul2(eq, iqq);                 // q(x)
            float t0, t1;
            upk(t, t0, t1);
            // p(x) - q(x) with p's product exact inside the FMA
            r[u] = fmaxf(__fmaf_rn(e[u], ip, -t0), 0.0f);
            r[u + 1] = fmaxf(__fmaf_rn(e[u + 1], ip, -t1), 0.0f);
        }
    } else {
#pragma unroll
        for (int u = 0; u < VEC; u += 2) {
            const unsigned long long pp = fmul2(pk(e[u], e[u + 1]), ipp);
            upk(pp, r[u], r[u + 1]);
        }
    }
    if (g * VEC + VEC > len) {   // ragged last vector of the slice: past-the-end lanes are 0
#pragma unroll
        for (int u = 0; u < VEC; ++u)
            if (g * VEC + u >= len) r[u] = 0.0f;
    }
    float s = r[0];
#pragma unroll
    for (int u = 1; u < VEC; ++u) s = __fadd_rn(s, r[u]);
    return s;
}

template <typename E, bool GREEDY>
__global__ void __launch_bounds__(NT, 1) k_verify_cluster(const CParams P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int PV = kPieceBytes / 16;   // 16-byte vectors per piece
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2 * kMaxPieces];
    __shared__ Xch xs;
    __shared__ Dec s_dec;
    __shared__ float s_wD[2][NW];
    __shared__ double s_wS[2][NW];
    __shared__ int s_wI[NW], s_wF[NW];
    __shared__ double s_we[NW + 1];
    __shared__ double s_th;
    __shared__ int s_c[2];
    __shared__ int s_skip;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = P.C;
    const int rank = static_cast<int>(blockIdx.x) % C;
    const int row = static_cast<int>(blockIdx.x) / C;   // = j * B + b (position-major)
    const int kk = P.k;
    const int j = row / P.B, b = row % P.B;
    const bool has_q = !GREEDY && j < kk;
    const int s0 = rank * P.W;
    const int len = max(0, min(P.W, P.V - s0));
    const E* gp = static_cast<const E*>(P.p) +
                  (static_cast<int64_t>(b) * (kk + 1) + j) * P.ld_p + s0;
    const E* gq = has_q ? static_cast<const E*>(P.q) + (static_cast<int64_t>(b) * kk + j) * P.ld_q + s0
                        : nullptr;
    E* sp = reinterpret_cast<E*>(smem);
    E* sq = sp + P.W;
    const uint32_t bulk = (static_cast<uint32_t>(len) * sizeof(E)) & ~15u;
    const int npc = static_cast<int>((bulk + kPieceBytes - 1) / kPieceBytes);
    const int x = j < kk ? __ldg(P.ids + static_cast<size_t>(b) * kk + j) : -1;
    const float c2 = P.c2;

    // ---- A: laziness test + staging -------------------------------------------------------
    if (tid == 0) {
        for (int i = 0; i < npc; ++i) {
            mbar_init(&bars[i], 1);
            if (has_q) mbar_init(&bars[kMaxPieces + i], 1);
        }
        fence_mbar_init();
        const uint32_t m = ld_relaxed_u32(P.rej_mask + b);
        s_skip = (m & ((1u << j) - 1u)) != 0u;
        xs.skip = s_skip;
    }
    __syncthreads();
    const bool my_skip = s_skip != 0;
    auto issue = [&]() {
        for (int i = 0; i < npc; ++i) {
            const uint32_t off = static_cast<uint32_t>(i) * kPieceBytes;
            const uint32_t nb = min(kPieceBytes, bulk - off);
            mbar_arrive_expect_tx(&bars[i], nb);
            bulk_g2s(reinterpret_cast<char*>(sp) + off, reinterpret_cast<const char*>(gp) + off, nb,
                     &bars[i]);
            if (has_q) {
                mbar_arrive_expect_tx(&bars[kMaxPieces + i], nb);
                bulk_g2s(reinterpret_cast<char*>(sq) + off, reinterpret_cast<const char*>(gq) + off,
                         nb, &bars[kMaxPieces + i]);
            }
        }
    };
    if (tid == 0 && !my_skip) issue();
    cluster_arrive();
    cluster_wait();   // every CTA of the cluster is running: DSMEM is addressable
    cgx::cluster_group cluster = cgx::this_cluster();
    const int skip = rank == 0 ? static_cast<int>(my_skip) : cluster.map_shared_rank(&xs, 0)->skip;
    if (skip) {
        if (tid == 0 && !my_skip) {   // drain our own bulk copies before the CTA exits
            for (int i = 0; i < npc; ++i) {
                mbar_wait(&bars[i], 0);
                if (has_q) mbar_wait(&bars[kMaxPieces + i], 0);
            }
        }
        cluster_arrive();
        cluster_wait();   // rank 0's flag has been read by everyone
        if (rank == 0 && tid == 0) arrive_row(P, b, j, false, -1, 0);
        return;
    }
    if (tid == 0 && my_skip) issue();   // our view was stale: rank 0 decided to run the row
    for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += NT) {   // ragged tail
        sp[i] = gp[i];
        if (has_q) sq[i] = gq[i];
    }
    __syncthreads();

    const int nfull = len / VEC;              // complete 16-byte vectors
    const int rem = len - nfull * VEC;        // logits in the ragged last vector
    // ---- 1: per-thread statistics of the slice --------------------------------------------
    float dP = -INFINITY, dQ = -INFINITY;     // fl(max * c2) of this thread's logits
    float sP = 0.0f, sQ = 0.0f;               // sum of 2^(z*c2 - d)
    int nf = 0;                               // kFlagNfP / kFlagNfQ seen by this thread
    float gbest = -INFINITY;                  // greedy: best value, its index
    int gidx = INT_MAX;
    if (GREEDY) {
        float nanacc = -INFINITY;
        int bestg = -1;
        for (int i = 0; i < npc; ++i) {
            mbar_wait(&bars[i], 0);
            const int hi = min(nfull, (i + 1) * PV);
            for (int g = i * PV + tid; g < hi; g += NT) {
                float v[VEC];
                EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
                float vm = -INFINITY;
#pragma unroll
                for (int u = 0; u < VEC; u += 2) {
                    nanacc = max3nan(nanacc, v[u], v[u + 1]);
                    vm = max3(vm, v[u], v[u + 1]);
                }
                if (vm > gbest) {
                    gbest = vm;
                    bestg = g;
                }
            }
        }
        if (bestg >= 0) {   // first (lowest) index of the best value inside its vector
            float v[VEC];
            EL::unpack(*reinterpret_cast<const uint4*>(sp + bestg * VEC), v);
            int u = 0;
#pragma unroll
            for (int w = VEC - 1; w >= 0; --w)
                if (v[w] == gbest) u = w;
            gidx = s0 + bestg * VEC + u;
        }
        if (rem && tid == 0) {
            for (int u = 0; u < rem; ++u) {
                const float z = EL::one(sp, nfull * VEC + u);
                nanacc = max3nan(nanacc, z, z);
                if (z > gbest) {   // later index: only a strictly larger value wins
                    gbest = z;
                    gidx = s0 + nfull * VEC + u;
                }
            }
        }
        if (!(nanacc < INFINITY)) nf = kFlagNfP;   // NaN or +inf
    } else {
        // sweep 1: NaN-propagating max (a NaN makes it NaN, +inf makes it +inf: no per-element
        // fault test is needed)
        float mp = -INFINITY, mq = -INFINITY;
        for (int i = 0; i < npc; ++i) {
            mbar_wait(&bars[i], 0);
            const int hi = min(nfull, (i + 1) * PV);
            for (int g = i * PV + tid; g < hi; g += NT) {
                float v[VEC];
                EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
#pragma unroll
                for (int u = 0; u < VEC; u += 2) mp = max3nan(mp, v[u], v[u + 1]);
            }
        }
        if (has_q) {
            for (int i = 0; i < npc; ++i) {
                mbar_wait(&bars[kMaxPieces + i], 0);
                const int hi = min(nfull, (i + 1) * PV);
                for (int g = i * PV + tid; g < hi; g += NT) {
                    float v[VEC];
                    EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), v);
#pragma unroll
                    for (int u = 0; u < VEC; u += 2) mq = max3nan(mq, v[u], v[u + 1]);
                }
            }
        }
        if (rem && tid == 0) {
            for (int u = 0; u < rem; ++u) {
                const float z = EL::one(sp, nfull * VEC + u);
                mp = max3nan(mp, z, z);
                if (has_q) {
                    const float w = EL::one(sq, nfull * VEC + u);
                    mq = max3nan(mq, w, w);
                }
            }
        }
        if (!(mp < INFINITY)) nf |= kFlagNfP;
        if (has_q && !(mq < INFINITY)) nf |= kFlagNfQ;
        // sweep 2: sum of 2^(z*c2 - d), d = fl(m*c2); FFMA2 + MUFU.EX2 + FADD2
        const unsigned long long cc = pk(c2, c2);
        if (mp > -INFINITY && mp < INFINITY) {
            dP = mp * c2;
            const unsigned long long nd = pk(-dP, -dP);
            unsigned long long a0 = 0ull, a1 = 0ull;
            for (int g = tid; g < nfull; g += NT) {
                float v[VEC];
                EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
#pragma unroll
                for (int u = 0; u < VEC; u += 4) {
                    a0 = fadd2(a0, ex2x2(ffma2(pk(v[u], v[u + 1]), cc, nd)));
                    a1 = fadd2(a1, ex2x2(ffma2(pk(v[u + 2], v[u + 3]), cc, nd)));
                }
            }
            float x0, x1, x2, x3;
            upk(a0, x0, x1);
            upk(a1, x2, x3);
            sP = (x0 + x1) + (x2 + x3);
            if (rem && tid == 0)
                for (int u = 0; u < rem; ++u)
                    sP += ex2_approx(__fmaf_rn(EL::one(sp, nfull * VEC + u), c2, -dP));
        }
        if (has_q && mq > -INFINITY && mq < INFINITY) {
            dQ = mq * c2;
            const unsigned long long nd = pk(-dQ, -dQ);
            unsigned long long a0 = 0ull, a1 = 0ull;
            for (int g = tid; g < nfull; g += NT) {
                float v[VEC];
                EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), v);
#pragma unroll
                for (int u = 0; u < VEC; u += 4) {
                    a0 = fadd2(a0, ex2x2(ffma2(pk(v[u], v[u + 1]), cc, nd)));
                    a1 = fadd2(a1, ex2x2(ffma2(pk(v[u + 2], v[u + 3]), cc, nd)));
                }
            }
            float x0, x1, x2, x3;
            upk(a0, x0, x1);
            upk(a1, x2, x3);
            sQ = (x0 + x1) + (x2 + x3);
            if (rem && tid == 0)
                for (int u = 0; u < rem; ++u)
                    sQ += ex2_approx(__fmaf_rn(EL::one(sq, nfull * VEC + u), c2, -dQ));
        }
    }

    // ---- per-CTA reduction: warps, then warp 0 over the warp partials ------------------------
    nf = __reduce_or_sync(0xFFFFFFFFu, nf);
    if (GREEDY) {
        float v = gbest;
        int i = gidx;
        warp_argmax(v, i);
        if (lane == 0) {
            s_wD[0][warp] = v;
            s_wI[warp] = i;
            s_wF[warp] = nf;
        }
    } else {
        const float Dw = warp_max(dP), Ew = warp_max(dQ);
        const double Sw = warp_sum(sP > 0.0f ? static_cast<double>(sP * ex2_approx(dP - Dw)) : 0.0);
        const double Tw = warp_sum(sQ > 0.0f ? static_cast<double>(sQ * ex2_approx(dQ - Ew)) : 0.0);
        if (lane == 0) {
            s_wD[0][warp] = Dw;
            s_wD[1][warp] = Ew;
            s_wS[0][warp] = Sw;
            s_wS[1][warp] = Tw;
            s_wF[warp] = nf;
        }
    }
    __syncthreads();
    if (warp == 0) {
        const bool on = lane < NW;
        const int f = __reduce_or_sync(0xFFFFFFFFu, on ? s_wF[lane] : 0);
        if (GREEDY) {
            float v = on ? s_wD[0][lane] : -INFINITY;
            int i = on ? s_wI[lane] : INT_MAX;
            warp_argmax(v, i);
            if (lane == 0) {
                xs.D_p = v;
                xs.argmax = i;
            }
        } else {
            const float wd = on ? s_wD[0][lane] : -INFINITY, we = on ? s_wD[1][lane] : -INFINITY;
            const double ws = on ? s_wS[0][lane] : 0.0, wt = on ? s_wS[1][lane] : 0.0;
            const float Dc = warp_max(wd), Ec = warp_max(we);
            const double Sc = warp_sum(ws > 0.0 ? ws * static_cast<double>(ex2_approx(wd - Dc)) : 0.0);
            const double Tc = warp_sum(wt > 0.0 ? wt * static_cast<double>(ex2_approx(we - Ec)) : 0.0);
            if (lane == 0) {
                xs.D_p = Dc;
                xs.D_q = Ec;
                xs.S_p = Sc;
                xs.S_q = Tc;
            }
        }
        if (lane == 0) {
            int fl = f;
            xs.zx_p = 0.0f;
            xs.zx_q = 0.0f;
            if (x >= s0 && x < s0 + len) {
                xs.zx_p = EL::one(sp, x - s0);
                if (has_q) xs.zx_q = EL::one(sq, x - s0);
                fl |= kFlagHasX;
            }
            xs.flags = fl;
        }
    }
    cluster_arrive();
    cluster_wait();   // B: every CTA's partial is published

    // ---- B: cluster combine + decision (identical in every CTA) -----------------------------
    if (warp == 0) {
        const bool on = lane < C;
        const Xch* px = cluster.map_shared_rank(&xs, on ? lane : 0);
        const int fl = on ? px->flags : 0;
        const int f = __reduce_or_sync(0xFFFFFFFFu, fl);
        const unsigned hx = __ballot_sync(0xFFFFFFFFu, (fl & kFlagHasX) != 0);
        float zxp = 0.0f, zxq = 0.0f;
        if (hx) {
            const int src = __ffs(hx) - 1;
            const float a = on ? px->zx_p : 0.0f, c = on ? px->zx_q : 0.0f;
            zxp = __shfl_sync(0xFFFFFFFFu, a, src);
            zxq = __shfl_sync(0xFFFFFFFFu, c, src);
        }
        float Dp = -INFINITY, Dq = -INFINITY;
        double Sp = 0.0, Sq = 0.0;
        int G = INT_MAX;
        if (GREEDY) {
            Dp = on ? px->D_p : -INFINITY;
            G = on ? px->argmax : INT_MAX;
            warp_argmax(Dp, G);
        } else {
            const float d = on ? px->D_p : -INFINITY, e = on ? px->D_q : -INFINITY;
            const double s = on ? px->S_p : 0.0, t = on ? px->S_q : 0.0;
            Dp = warp_max(d);
            Dq = warp_max(e);
            Sp = warp_sum(s > 0.0 ? s * static_cast<double>(ex2_approx(d - Dp)) : 0.0);
            Sq = warp_sum(t > 0.0 ? t * static_cast<double>(ex2_approx(e - Dq)) : 0.0);
        }
        if (lane == 0) {
            int st = 0;
            bool stop = false;
            double u_smp = 0.0;
            if (j < kk && (x < 0 || x >= P.V)) st = kBadId;
            if (!st) {
                if (f & kFlagNfP) st = kNonfinite;
                else if (Dp == -INFINITY) st = kEmptyRow;
            }
            if (!st && has_q) {
                if (f & kFlagNfQ) st = kNonfinite;
                else if (Dq == -INFINITY) st = kEmptyRow;
            }
            const uint4 w = verify_words(P.seed, static_cast<uint32_t>(j), P.round,
                                         P.rid_base + static_cast<uint64_t>(b));
            if (st) {
                stop = true;
            } else if (j < kk) {
                if (GREEDY) {
                    stop = x != G;                                        // argmax matching (C-5)
                } else if (zxq == -INFINITY) {
                    st = kZeroQ;                                          // q_j(x_j) = 0 (C-7)
                    stop = true;
                } else {
                    // a = p(x)/q(x) = 2^((z_p(x) c2 - D_p) - (z_q(x) c2 - D_q)) * S_q / S_p
                    const double c2d = static_cast<double>(c2);
                    const double l = (static_cast<double>(zxp) * c2d - static_cast<double>(Dp)) -
                                     (static_cast<double>(zxq) * c2d - static_cast<double>(Dq));
                    const double a = exp2(l) * (Sq / Sp);
                    if (!(a >= 1.0)) stop = unit24(w.x) >= a;            // reject iff u >= a (C-2)
                }
            }
            if (rank == 0 && stop && j < kk) {   // publish the stop at once (laziness)
                atomicOr(P.rej_mask + b, 1u << j);
                __threadfence();
            }
            u_smp = unit24(w.y);
            s_dec.S_p = Sp;
            s_dec.S_q = Sq;
            s_dec.u_smp = u_smp;
            s_dec.D_p = Dp;
            s_dec.D_q = Dq;
            s_dec.stop = stop;
            s_dec.status = st;
            s_dec.token = G;
        }
    }
    __syncthreads();
    const int st = s_dec.status;
    const bool stop = s_dec.stop != 0;
    const bool hard = (st & kHard) != 0;
    const bool resid = !GREEDY && !hard && (stop || j == kk);
    if (!resid) {
        cluster_arrive();   // no more DSMEM reads by this CTA
        if (rank == 0 && tid == 0) {
            const bool write = stop || j == kk;
            arrive_row(P, b, j, write, (GREEDY && !hard) ? s_dec.token : -1, st);
        }
        cluster_wait();     // peers may still read our partial until they arrive
        return;
    }

    // ---- C: residual (or bonus) inverse-CDF sample from the slice held in shared memory -----
    const float Dp = s_dec.D_p, Dq = s_dec.D_q;
    const float ip = static_cast<float>(1.0 / s_dec.S_p);
    const float iq = has_q ? static_cast<float>(1.0 / s_dec.S_q) : 0.0f;
    const int nall = nfull + (rem ? 1 : 0);
    const int g0 = tid * P.nvr, g1 = min(nall, g0 + P.nvr);
    bool use_q = has_q;
    int status = st;
    double tsum = 0.0, incl = 0.0;
    double R = 0.0;
    int cstar = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        tsum = 0.0;
        for (int g = g0; g < g1; ++g) {
            float r[VEC];
            tsum += static_cast<double>(vec_resid<E>(sp, sq, g, len, use_q, c2, -Dp, -Dq, ip, iq, r));
        }
        incl = warp_incl_scan(tsum, lane);
        if (lane == 31) s_wS[0][warp] = incl;
        __syncthreads();
        if (tid == 0) {
            double a = 0.0;
            s_we[0] = 0.0;
            for (int w = 0; w < NW; ++w) {
                a = __dadd_rn(a, s_wS[0][w]);
                s_we[w + 1] = a;
            }
            xs.R[attempt] = a;
        }
        cluster_arrive();
        cluster_wait();   // C: every CTA's slice mass is published
        if (warp == 0) {
            const double Rr = lane < C ? cluster.map_shared_rank(&xs, lane)->R[attempt] : 0.0;
            const double ic = warp_incl_scan(Rr, lane);
            const double tot = __shfl_sync(0xFFFFFFFFu, ic, 31);
            if (lane == 0) s_th = tot;
            if (tot > 0.0) {
                const double theta = s_dec.u_smp * tot;           // C-9: first x with C(x) > theta
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, lane < C && ic > theta);
                const unsigned pos = __ballot_sync(0xFFFFFFFFu, lane < C && Rr > 0.0);
                const int cs = hit ? __ffs(hit) - 1 : 31 - __clz(pos);   // clamp: last slice with mass
                const double ex = __shfl_up_sync(0xFFFFFFFFu, ic, 1);
                const double exs = __shfl_sync(0xFFFFFFFFu, lane == 0 ? 0.0 : ex, cs);
                if (lane == 0) {
                    s_c[0] = cs;
                    s_c[1] = hit ? 0 : 1;
                    s_th = theta - exs;
                }
            }
            if (lane == 0 && !(tot > 0.0)) s_c[0] = -1;
        }
        __syncthreads();
        R = s_th;
        cstar = s_c[0];
        if (cstar >= 0 || !use_q) break;
        // C-6: the residual has no mass (rounding only) -> sample from p_L instead
        use_q = false;
        status |= kZeroResidual;
        __syncthreads();
    }
    cluster_arrive();   // no more DSMEM reads by this CTA
    if (cstar < 0 && rank == 0 && tid == 0)   // no mass even in p_L: cannot happen for a finite
        arrive_row(P, b, j, true, -1, status);  // row (its max has p >= 1/V); never hang the request
    if (rank == cstar) {
        const double th1 = R;   // theta relative to this slice
        const bool clamp = s_c[1] != 0;
        // warp holding theta (all threads compute the same)
        int ws = -1, wlast = 0;
        for (int w = 0; w < NW; ++w) {
            if (s_we[w + 1] > s_we[w]) wlast = w;
            if (ws < 0 && !clamp && s_we[w + 1] > th1) ws = w;
        }
        const bool wclamp = ws < 0;
        if (wclamp) ws = wlast;
        if (warp == ws) {
            const double th2 = th1 - s_we[ws];
            const unsigned hit = wclamp ? 0u : __ballot_sync(0xFFFFFFFFu, incl > th2);
            const unsigned pos = __ballot_sync(0xFFFFFFFFu, tsum > 0.0);
            const int ls = hit ? __ffs(hit) - 1 : (pos ? 31 - __clz(pos) : 0);
            double ex = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
            if (lane == 0) ex = 0.0;
            if (lane == ls) {
                const double th3 = hit ? th2 - ex : INFINITY;
                double acc = 0.0;
                int found = -1, lastpos = -1;
                for (int g = g0; g < g1 && found < 0; ++g) {
                    float r[VEC];
                    const float vs = vec_resid<E>(sp, sq, g, len, use_q, c2, -Dp, -Dq, ip, iq, r);
#pragma unroll
                    for (int u = 0; u < VEC; ++u)
                        if (r[u] > 0.0f) lastpos = g * VEC + u;
                    if (acc + static_cast<double>(vs) > th3) {
                        float cum = r[0];
                        if (acc + static_cast<double>(cum) > th3) {
                            found = g * VEC;
                        } else {
#pragma unroll
                            for (int u = 1; u < VEC; ++u) {
                                cum = __fadd_rn(cum, r[u]);
                                if (found < 0 && acc + static_cast<double>(cum) > th3) found = g * VEC + u;
                            }
                        }
                        if (found < 0) found = lastpos;   // rounding inside the vector
                    } else {
                        acc += static_cast<double>(vs);
                    }
                }
                if (found < 0) found = lastpos >= 0 ? lastpos : g0 * VEC;   // rounding: clamp (C-9)
                arrive_row(P, b, j, true, s0 + found, status);
            }
        }
    }
    cluster_wait();
}

}  // namespace clu

// ------------------------------------------------------------------------------------------
// host side: configuration + launch

void record_event(cudaEvent_t ev, cudaStream_t st);

namespace {
template <typename E, bool G>
struct KInfo {
    static bool init;
    static int max_dyn;
};
template <typename E, bool G>
bool KInfo<E, G>::init = false;
template <typename E, bool G>
int KInfo<E, G>::max_dyn = 0;

template <typename E, bool G>
int prepare_kernel() {
    if (!KInfo<E, G>::init) {
        auto k = clu::k_verify_cluster<E, G>;
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        KInfo<E, G>::max_dyn = optin - static_cast<int>(fa.sharedSizeBytes);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, KInfo<E, G>::max_dyn);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        KInfo<E, G>::init = true;
    }
    return KInfo<E, G>::max_dyn;
}

template <typename E, bool G>
cudaError_t launch_t(const CParams& P, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(P.k + 1) * P.B * P.C);
    cfg.blockDim = dim3(clu::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, clu::k_verify_cluster<E, G>, P);
}

template <typename E, bool G>
int occupancy_clusters(int C, size_t smem) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C * 64);
    cfg.blockDim = dim3(clu::NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, clu::k_verify_cluster<E, G>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
}  // namespace

// Target bytes of logits held per CTA (p and q slices together).  64 KB lets three CTAs share
// an SM (3 x 64 KB of the 228 KB), so one CTA's loads overlap another's reductions.
static int cta_target_bytes() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("STARSD_CTA_KB");
        v = (e ? atoi(e) : 64) * 1024;
        if (v < 4096) v = 4096;
    }
    return v;
}

// Choose the cluster shape for (V, dtype, greedy).  Returns false if the cluster kernel cannot
// serve the shape on this device (the caller then uses the two-launch path).
bool cluster_config(int32_t V, int esz, bool greedy, int32_t* C, int32_t* W, int32_t* nvr,
                    size_t* smem) {
    const int vec = 16 / esz;
    const int64_t row = static_cast<int64_t>(V) * esz * (greedy ? 1 : 2);
    int c = 1;
    while (c < 16 && row > static_cast<int64_t>(cta_target_bytes()) * c) c *= 2;
    int64_t w = (V + c - 1) / c;
    w = (w + vec - 1) / vec * vec;
    const size_t sm = static_cast<size_t>(w) * esz * (greedy ? 1 : 2);
    int max_dyn;
    if (esz == 4)
        max_dyn = greedy ? prepare_kernel<float, true>() : prepare_kernel<float, false>();
    else
        max_dyn = greedy ? prepare_kernel<__nv_bfloat16, true>() : prepare_kernel<__nv_bfloat16, false>();
    if (sm > static_cast<size_t>(max_dyn)) return false;
    if (static_cast<int64_t>(w) * esz > static_cast<int64_t>(clu::kMaxPieces) * clu::kPieceBytes) return false;
    // occupancy (cached per shape class)
    struct Entry { int esz, greedy, c; size_t sm; int n; };
    static Entry cache[32];
    static int ncache = 0;
    int n = -1;
    for (int i = 0; i < ncache; ++i)
        if (cache[i].esz == esz && cache[i].greedy == (int)greedy && cache[i].c == c && cache[i].sm == sm)
            n = cache[i].n;
    if (n < 0) {
        if (esz == 4)
            n = greedy ? occupancy_clusters<float, true>(c, sm) : occupancy_clusters<float, false>(c, sm);
        else
            n = greedy ? occupancy_clusters<__nv_bfloat16, true>(c, sm)
                       : occupancy_clusters<__nv_bfloat16, false>(c, sm);
        if (ncache < 32) cache[ncache++] = Entry{esz, (int)greedy, c, sm, n};
    }
    if (n <= 0) return false;
    const int nvec = static_cast<int>(w / vec);
    int r = (nvec + clu::NT - 1) / clu::NT;
    if (r % 2 == 0) r += 1;   // odd 16-byte stride per thread: conflict-free LDS.128
    *C = c;
    *W = static_cast<int32_t>(w);
    *nvr = r;
    *smem = sm;
    return true;
}

int cluster_max_active(int32_t V, int esz, bool greedy) {
    int32_t C, W, nvr;
    size_t sm;
    if (!cluster_config(V, esz, greedy, &C, &W, &nvr, &sm)) return 0;
    if (esz == 4)
        return greedy ? occupancy_clusters<float, true>(C, sm) : occupancy_clusters<float, false>(C, sm);
    return greedy ? occupancy_clusters<__nv_bfloat16, true>(C, sm)
                  : occupancy_clusters<__nv_bfloat16, false>(C, sm);
}

cudaError_t launch_cluster(const CParams& P, bool greedy, bool bf16, size_t smem, cudaStream_t st,
                           cudaEvent_t ev0, cudaEvent_t ev1) {
    record_event(ev0, st);
    cudaError_t e;
    if (greedy)
        e = bf16 ? launch_t<__nv_bfloat16, true>(P, smem, st) : launch_t<float, true>(P, smem, st);
    else
        e = bf16 ? launch_t<__nv_bfloat16, false>(P, smem, st) : launch_t<float, false>(P, smem, st);
    record_event(ev1, st);
    return e;
}

}  // namespace sd
