// verify_kernels.cu -- sm_100a kernels of the batched speculative-sampling verify step.
//
// The method (Alg. 2; readings C-1..C-12 of DESIGN.md), per request b:
//   accept x_j iff u_acc(j) < min(1, p_j(x_j) / q_j(x_j)),  L = first rejection (else k),
//   emit x_0..x_{L-1} and t ~ norm(max(0, p_L - q_L)) (L < k) or t ~ p_k (L == k).
//
// Data flow (two launches, stream ordered):
//   k_row_stats  grid = (k+1) * B * nch CTAs in POSITION-MAJOR order (all requests' position 0
//                first).  CTA (j, b, c) TMA-bulk-loads its 32 KB vocab slice of p_j (and q_j)
//                into shared memory, computes the slice max and sum of 2^((z - M) log2e / T)
//                (one MUFU.EX2 per element, fp64 accumulation), and gathers z(x_j).  The last
//                CTA of a row pair combines the slices (fp64), draws u_acc from Philox and
//                decides the acceptance test; a rejection sets bit j of rej_mask[b].
//                A CTA whose request already has a rejection at an earlier position skips its
//                loads: the method never needs rows after L (laziness).
//   k_sample     grid = B * nch.  CTA (b, c) re-reads slice c of row L (usually from L2),
//                computes r = max(0, p - q) in fp64 and per-warp-segment masses; the last CTA
//                of the request does the inverse-CDF search chunk -> segment -> token.
//   greedy (T = 0) replaces the sum by an (max, lowest index) reduction and k_sample by a tiny
//                finalize kernel.
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

// status bits (values of include/starsd.h SD_FAULT_*)
constexpr int32_t kBadId = 1, kNonfinite = 2, kEmptyRow = 4, kZeroQ = 8, kZeroResidual = 16;
constexpr int32_t kHard = kBadId | kNonfinite | kEmptyRow;
constexpr uint32_t kSkipArrive = 1u | (1u << 16);

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

// Probability terms of the sampling pass.  Written with explicit-rounding intrinsics so the
// main pass and the final re-read compute bit-identical values.
//   p(x) = 2^((z_p - M_p) c2) / S_p ,  r(x) = max(0, p(x) - q(x))   (fp64 after the exp)
__device__ __forceinline__ double prob_term(float z, float M, float c2, double invS) {
    return __dmul_rn(static_cast<double>(ex2_approx(__fmul_rn(__fsub_rn(z, M), c2))), invS);
}

// ------------------------------------------------------------------------------------------
// Kernel A: per-slice statistics + per-row acceptance decision
template <typename E, bool GREEDY>
__global__ void __launch_bounds__(kThreads) k_row_stats(const Params P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int TILE = kThreads * VEC;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_flag;
    __shared__ float s_mp[kWarps], s_mq[kWarps];
    __shared__ int s_gi[kWarps];
    __shared__ double s_sp[kWarps], s_sq[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = P.nch, kk = P.k;
    const int c = blockIdx.x % nch;
    const int rowid = blockIdx.x / nch;          // = j * B + b  (position-major)
    const int b = rowid % P.B, j = rowid / P.B;
    const size_t pos = static_cast<size_t>(b) * (kk + 1) + j;

    if (tid == 0) {
        const uint32_t m = ld_relaxed_u32(P.rej_mask + b);
        s_flag = (m & ((1u << j) - 1u)) != 0u;
    }
    __syncthreads();
    if (s_flag) {   // the request already stopped before j: this row is never needed
        if (tid == 0) {
            const uint32_t t = atomicAdd(P.ticketA + pos, kSkipArrive);
            if ((t & 0xFFFFu) == static_cast<uint32_t>(nch - 1)) P.ticketA[pos] = 0u;
        }
        return;
    }

    const int c0 = c * P.CH;
    const int len = min(P.CH, P.V - c0);
    const bool load_q = !GREEDY && j < kk;
    const E* gp = static_cast<const E*>(P.p) + static_cast<int64_t>(pos) * P.ld_p + c0;
    const E* gq = load_q ? static_cast<const E*>(P.q) +
                               (static_cast<int64_t>(b) * kk + j) * P.ld_q + c0
                         : nullptr;
    E* sp = reinterpret_cast<E*>(smem);
    E* sq = sp + P.CH;
    const uint32_t bytes = static_cast<uint32_t>(len) * sizeof(E);
    const uint32_t bulk = bytes & ~15u;

    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar, load_q ? 2u * bulk : bulk);
        if (bulk) {
            bulk_g2s(sp, gp, bulk, &bar);
            if (load_q) bulk_g2s(sq, gq, bulk, &bar);
        }
    }
    for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += kThreads) {
        sp[i] = gp[i];
        if (load_q) sq[i] = gq[i];
    }
    const int x = (j < kk) ? P.ids[static_cast<size_t>(b) * kk + j] : -1;
    __syncthreads();
    mbar_wait(&bar, 0);

    // ---- sweep 1: slice max (NaN-propagating: a NaN makes the max NaN, +inf makes it +inf,
    // so faults need no per-element test); greedy: lowest argmax + NaN-propagating max ------
    const int nvec = len / VEC;                  // fully valid vectors
    const bool tail = nvec * VEC < len;          // a ragged last vector (row end only)
    const int tail_tid = nvec % kThreads;
    float mp = -INFINITY, mq = -INFINITY, np = -INFINITY;
    int gi = INT_MAX;
#pragma unroll 4
    for (int g = tid; g < nvec; g += kThreads) {
        float v[VEC];
        EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
        if (GREEDY) {
#pragma unroll
            for (int u = 0; u < VEC; ++u) {
                np = fmax_nan(np, v[u]);
                if (v[u] > mp) {
                    mp = v[u];
                    gi = c0 + g * VEC + u;
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < VEC; u += 2) mp = fmax_nan(mp, fmax_nan(v[u], v[u + 1]));
            if (load_q) {
                EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), v);
#pragma unroll
                for (int u = 0; u < VEC; u += 2) mq = fmax_nan(mq, fmax_nan(v[u], v[u + 1]));
            }
        }
    }
    if (tail && tid == tail_tid) {
        float v[VEC];
        EL::unpack(*reinterpret_cast<const uint4*>(sp + nvec * VEC), v);
        for (int u = 0; u < VEC; ++u) {
            if (nvec * VEC + u < len) {
                if (GREEDY) {
                    np = fmax_nan(np, v[u]);
                    if (v[u] > mp) {
                        mp = v[u];
                        gi = c0 + nvec * VEC + u;
                    }
                } else {
                    mp = fmax_nan(mp, v[u]);
                }
            }
        }
        if (load_q) {
            EL::unpack(*reinterpret_cast<const uint4*>(sq + nvec * VEC), v);
            for (int u = 0; u < VEC; ++u)
                if (nvec * VEC + u < len) mq = fmax_nan(mq, v[u]);
        }
    }
    if (GREEDY) {
        warp_argmax(mp, gi);
        np = warp_max_nan(np);
    } else {
        mp = warp_max_nan(mp);
        mq = warp_max_nan(mq);
    }
    if (lane == 0) {
        s_mp[warp] = mp;
        s_mq[warp] = GREEDY ? np : mq;
        s_gi[warp] = gi;
    }
    __syncthreads();
    float Mp = s_mp[0], Mq = s_mq[0];
    int G = s_gi[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
        if (GREEDY) {
            if (s_mp[w] > Mp || (s_mp[w] == Mp && s_gi[w] < G)) {
                Mp = s_mp[w];
                G = s_gi[w];
            }
            Mq = fmax_nan(Mq, s_mq[w]);       // greedy: NaN-propagating max of p
        } else {
            Mp = fmax_nan(Mp, s_mp[w]);
            Mq = fmax_nan(Mq, s_mq[w]);
        }
    }
    int bad = 0;
    if (GREEDY) {
        bad = (Mq != Mq || Mq == INFINITY) ? kPartNonfiniteP : 0;
        Mq = -INFINITY;
    } else {
        bad = ((Mp != Mp || Mp == INFINITY) ? kPartNonfiniteP : 0) |
              ((Mq != Mq || Mq == INFINITY) ? kPartNonfiniteQ : 0);
    }

    // ---- sweep 2: sum of 2^((z - M) c2) against the CTA max (one MUFU.EX2 per element;
    // fp32 within a vector, fp64 across vectors) ----------------------------------------------
    double Sp = 0.0, Sq = 0.0;
    if (!GREEDY) {
        const float c2 = P.c2;
        const bool okp = Mp > -INFINITY && Mp < INFINITY;
        const bool okq = load_q && Mq > -INFINITY && Mq < INFINITY;
        const float ep = okp ? Mp : 0.0f, eq = okq ? Mq : 0.0f;
        if (okp || okq) {
#pragma unroll 4
            for (int g = tid; g < nvec; g += kThreads) {
                float v[VEC];
                if (okp) {
                    EL::unpack(*reinterpret_cast<const uint4*>(sp + g * VEC), v);
                    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                    for (int u = 0; u < VEC; u += 2) {
                        a0 += ex2_approx(__fmul_rn(__fsub_rn(v[u], ep), c2));
                        a1 += ex2_approx(__fmul_rn(__fsub_rn(v[u + 1], ep), c2));
                    }
                    Sp += static_cast<double>(a0 + a1);
                }
                if (okq) {
                    EL::unpack(*reinterpret_cast<const uint4*>(sq + g * VEC), v);
                    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                    for (int u = 0; u < VEC; u += 2) {
                        a0 += ex2_approx(__fmul_rn(__fsub_rn(v[u], eq), c2));
                        a1 += ex2_approx(__fmul_rn(__fsub_rn(v[u + 1], eq), c2));
                    }
                    Sq += static_cast<double>(a0 + a1);
                }
            }
            if (tail && tid == tail_tid) {
                float v[VEC];
                if (okp) {
                    EL::unpack(*reinterpret_cast<const uint4*>(sp + nvec * VEC), v);
                    float t = 0.0f;
                    for (int u = 0; u < VEC; ++u)
                        if (nvec * VEC + u < len) t += ex2_approx(__fmul_rn(__fsub_rn(v[u], ep), c2));
                    Sp += static_cast<double>(t);
                }
                if (okq) {
                    EL::unpack(*reinterpret_cast<const uint4*>(sq + nvec * VEC), v);
                    float t = 0.0f;
                    for (int u = 0; u < VEC; ++u)
                        if (nvec * VEC + u < len) t += ex2_approx(__fmul_rn(__fsub_rn(v[u], eq), c2));
                    Sq += static_cast<double>(t);
                }
            }
        }
        Sp = warp_sum(Sp);
        Sq = warp_sum(Sq);
        if (lane == 0) {
            s_sp[warp] = Sp;
            s_sq[warp] = Sq;
        }
        __syncthreads();
        if (tid == 0) {
            Sp = 0.0;
            Sq = 0.0;
            for (int w = 0; w < kWarps; ++w) {
                Sp += s_sp[w];
                Sq += s_sq[w];
            }
        }
    }

    // ---- publish the slice, take a ticket ------------------------------------------------
    if (tid == 0) {
        PartA pa;
        pa.S_p = Sp;
        pa.S_q = Sq;
        pa.M_p = Mp;
        pa.M_q = Mq;
        pa.zx_p = 0.0f;
        pa.zx_q = 0.0f;
        pa.flags = bad;
        pa.argmax = G;
        if (x >= c0 && x < c0 + len) {
            pa.zx_p = EL::one(sp, x - c0);
            pa.zx_q = load_q ? EL::one(sq, x - c0) : 0.0f;
            pa.flags |= kPartHasX;
        }
        P.partA[pos * nch + c] = pa;
        __threadfence();
        const uint32_t t = atomicAdd(P.ticketA + pos, 1u);
        const bool last = (t & 0xFFFFu) == static_cast<uint32_t>(nch - 1);
        if (last) P.ticketA[pos] = 0u;
        s_flag = last && (t >> 16) == 0u;   // last arriver and no slice of this row skipped
    }
    __syncthreads();
    if (!s_flag || warp != 0) return;

    // ---- last CTA of the row pair: combine the slices (fp64) and decide --------------------
    __threadfence();
    const PartA* parts = P.partA + pos * nch;
    float RMp = -INFINITY, RMq = -INFINITY, zxp = 0.0f, zxq = 0.0f;
    int flags = 0, RG = INT_MAX, hasx_lane = 0;
    for (int cc = lane; cc < nch; cc += 32) {
        const PartA a = load_cg(parts + cc);
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
            RMp = fmax_nan(RMp, a.M_p);
            RMq = fmax_nan(RMq, a.M_q);
        }
    }
    if (GREEDY) {
        warp_argmax(RMp, RG);
    } else {
        RMp = warp_max_nan(RMp);
        RMq = warp_max_nan(RMq);
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
        // rescale each slice sum from its own max to the row max: S_c * 2^((M_c - M) c2)
        for (int cc = lane; cc < nch; cc += 32) {
            const PartA a = load_cg(parts + cc);
            if (a.S_p > 0.0 && RMp < INFINITY)
                RSp += a.S_p * exp2((static_cast<double>(a.M_p) - RMp) * P.c2d);
            if (a.S_q > 0.0 && RMq < INFINITY)
                RSq += a.S_q * exp2((static_cast<double>(a.M_q) - RMq) * P.c2d);
        }
        RSp = warp_sum(RSp);
        RSq = warp_sum(RSq);
    }
    if (lane != 0) return;

    int32_t st = 0;
    bool stop = false;
    if (j < kk && (x < 0 || x >= P.V)) st = kBadId;
    if (!st) {
        if ((flags & kPartNonfiniteP) || !(RMp < INFINITY)) st = kNonfinite;
        else if (RMp == -INFINITY) st = kEmptyRow;
    }
    if (!st && load_q) {
        if ((flags & kPartNonfiniteQ) || !(RMq < INFINITY)) st = kNonfinite;
        else if (RMq == -INFINITY) st = kEmptyRow;
    }
    if (st) {
        stop = true;
    } else if (j < kk) {
        if (GREEDY) {
            stop = (x != RG);                                       // argmax matching (C-5)
        } else if (zxq == -INFINITY) {
            st = kZeroQ;                                            // q_j(x_j) = 0 (C-7)
            stop = true;
        } else {
            // log2 p_j(x_j) - log2 q_j(x_j), in fp64 on the kernel's own softmax scale
            const double ell = (static_cast<double>(zxp) - RMp) * P.c2d - log2(RSp) -
                               ((static_cast<double>(zxq) - RMq) * P.c2d - log2(RSq));
            if (ell < 0.0) {                                        // a = min(1, p/q) < 1
                const double a = exp2(ell);
                const uint4 w = verify_words(P.seed, static_cast<uint32_t>(j), P.round,
                                             P.rid_base + static_cast<uint64_t>(b));
                stop = unit24(w.x) >= a;                            // reject iff u >= a (C-2)
            }
        }
    }
    RowStat rs;
    rs.S_p = RSp;
    rs.S_q = RSq;
    rs.M_p = RMp;
    rs.M_q = RMq;
    rs.status = st;
    rs.argmax = RG;
    P.rowstat[pos] = rs;
    if (stop) atomicOr(P.rej_mask + b, 1u << j);
}

// ------------------------------------------------------------------------------------------
// Kernel B: residual (or bonus) inverse-CDF sample at the stop position L
template <typename E>
__global__ void __launch_bounds__(kThreads) k_sample(const Params P) {
    using EL = Elt<E>;
    constexpr int VEC = EL::VEC;
    constexpr int TILE = kThreads * VEC;
    constexpr int SEG = 32 * VEC;                 // tokens per warp segment
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ double2 s_seg[kMaxChunkBytes / kTileBytes * kWarps];
    __shared__ double2 s_pb[256];
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = P.nch, kk = P.k;
    const int c = blockIdx.x % nch, b = blockIdx.x / nch;
    // programmatic dependent launch: this grid may start while k_row_stats drains; wait until
    // every row decision of the primary grid is complete and visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t mask = P.rej_mask[b];
    const int L = mask ? __ffs(mask) - 1 : kk;
    const RowStat rs = P.rowstat[static_cast<size_t>(b) * (kk + 1) + L];
    const bool hard = (rs.status & kHard) != 0;
    const bool use_q = L < kk;
    const float c2 = P.c2;
    const double invSp = 1.0 / rs.S_p;
    const double invSq = use_q ? 1.0 / rs.S_q : 0.0;
    const int nseg = P.nseg;
    const E* gp = static_cast<const E*>(P.p) +
                  (static_cast<int64_t>(b) * (kk + 1) + L) * P.ld_p;
    const E* gq = use_q ? static_cast<const E*>(P.q) + (static_cast<int64_t>(b) * kk + L) * P.ld_q
                        : nullptr;

    if (!hard) {
        const int c0 = c * P.CH;
        const int len = min(P.CH, P.V - c0);
        E* sp = reinterpret_cast<E*>(smem);
        E* sq = sp + P.CH;
        const uint32_t bytes = static_cast<uint32_t>(len) * sizeof(E);
        const uint32_t bulk = bytes & ~15u;
        if (tid == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid == 0) {
            mbar_arrive_expect_tx(&bar, use_q ? 2u * bulk : bulk);
            if (bulk) {
                bulk_g2s(sp, gp + c0, bulk, &bar);
                if (use_q) bulk_g2s(sq, gq + c0, bulk, &bar);
            }
        }
        for (int i = static_cast<int>(bulk / sizeof(E)) + tid; i < len; i += kThreads) {
            sp[i] = gp[c0 + i];
            if (use_q) sq[i] = gq[c0 + i];
        }
        __syncthreads();
        mbar_wait(&bar, 0);

        // warp w computes segments w*PER .. w*PER+PER-1 of the chunk (SEG contiguous tokens
        // each); PER <= 4 independent Kogge-Stone scans run interleaved.  Segment totals are
        // the scans' last lanes -- the same routine the final search re-runs on one segment.
        const int PER = nseg / kWarps;
        double vr[4], vpm[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            vr[i] = 0.0;
            vpm[i] = 0.0;
            const int e0 = (warp * PER + i) * SEG + lane * VEC;
            if (i < PER && e0 < len) {
                float vp[VEC], vq[VEC];
                EL::unpack(*reinterpret_cast<const uint4*>(sp + e0), vp);
                if (use_q) EL::unpack(*reinterpret_cast<const uint4*>(sq + e0), vq);
                double r4 = 0.0, p4 = 0.0;
#pragma unroll
                for (int u = 0; u < VEC; ++u) {
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
                vr[i] = r4;
                vpm[i] = p4;
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
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
            for (int i = 0; i < 4; ++i)
                if (i < PER) s_seg[warp * PER + i] = make_double2(vr[i], vpm[i]);
        }
        __syncthreads();
        double2* gseg = P.segtab + (static_cast<size_t>(b) * nch + c) * nseg;
        for (int s = tid; s < nseg; s += kThreads) gseg[s] = s_seg[s];
        if (tid == 0) {
            double R = 0.0, Pm = 0.0;
            for (int s = 0; s < nseg; ++s) {
                R = __dadd_rn(R, s_seg[s].x);
                Pm = __dadd_rn(Pm, s_seg[s].y);
            }
            P.partB[static_cast<size_t>(b) * nch + c] = PartB{R, Pm};
        }
        __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t t = atomicAdd(P.ticketB + b, 1u);
        s_last = t == static_cast<uint32_t>(nch - 1);
    }
    __syncthreads();
    if (!s_last || warp != 0) return;

    // ---- last CTA of request b: inverse CDF, chunk -> segment -> token ------------------
    __threadfence();
    int32_t status = rs.status;
    int32_t tok = -1;
    if (!hard) {
        for (int cc = lane; cc < nch; cc += 32) {
            const PartB pb = load_cg(P.partB + static_cast<size_t>(b) * nch + cc);
            s_pb[cc] = make_double2(pb.R, pb.P);
        }
        __syncwarp();
        int cstar = 0, sstar = 0;
        double th1 = 0.0;
        bool zero_res = false;
        if (lane == 0) {
            double R = 0.0, Pm = 0.0;
            for (int cc = 0; cc < nch; ++cc) {
                R = __dadd_rn(R, s_pb[cc].x);
                Pm = __dadd_rn(Pm, s_pb[cc].y);
            }
            zero_res = use_q && !(R > 0.0);                 // C-6: fall back to p_L
            const double tot = zero_res ? Pm : R;
            const uint4 w = verify_words(P.seed, static_cast<uint32_t>(L), P.round,
                                         P.rid_base + static_cast<uint64_t>(b));
            const double theta = unit24(w.y) * tot;
            double run = 0.0;
            cstar = -1;
            int lastpos = 0;
            for (int cc = 0; cc < nch; ++cc) {
                const double m = zero_res ? s_pb[cc].y : s_pb[cc].x;
                if (m > 0.0) lastpos = cc;
                const double nr = __dadd_rn(run, m);
                if (nr > theta) {
                    cstar = cc;
                    break;
                }
                run = nr;
            }
            if (cstar < 0) {          // rounding: clamp to the last chunk with mass (C-9)
                cstar = lastpos;
                th1 = INFINITY;
            } else {
                th1 = theta - run;
            }
        }
        cstar = __shfl_sync(0xFFFFFFFFu, cstar, 0);
        th1 = __shfl_sync(0xFFFFFFFFu, th1, 0);
        zero_res = __shfl_sync(0xFFFFFFFFu, static_cast<int>(zero_res), 0) != 0;
        const double2* gseg = P.segtab + (static_cast<size_t>(b) * nch + cstar) * nseg;
        for (int s = lane; s < nseg; s += 32) s_seg[s] = __ldcg(gseg + s);
        __syncwarp();
        double th2 = 0.0;
        if (lane == 0) {
            double run = 0.0;
            sstar = -1;
            int lastpos = 0;
            for (int s = 0; s < nseg; ++s) {
                const double m = zero_res ? s_seg[s].y : s_seg[s].x;
                if (m > 0.0) lastpos = s;
                const double nr = __dadd_rn(run, m);
                if (nr > th1) {
                    sstar = s;
                    break;
                }
                run = nr;
            }
            if (sstar < 0) {
                sstar = lastpos;
                th2 = INFINITY;
            } else {
                th2 = th1 - run;
            }
        }
        sstar = __shfl_sync(0xFFFFFFFFu, sstar, 0);
        th2 = __shfl_sync(0xFFFFFFFFu, th2, 0);
        // re-read the segment's 32*VEC tokens and scan them exactly as the main pass did
        const int base = cstar * P.CH + (sstar / kWarps) * TILE + (sstar % kWarps) * SEG;
        const int my0 = base + lane * VEC;
        double rv[VEC];
        double r4 = 0.0;
#pragma unroll
        for (int u = 0; u < VEC; ++u) {
            rv[u] = 0.0;
            const int xx = my0 + u;
            if (xx < P.V && xx < (cstar + 1) * P.CH) {
                const double pd = prob_term(EL::one(gp, xx), rs.M_p, c2, invSp);
                double rd = pd;
                if (use_q && !zero_res) {
                    const double qd = prob_term(EL::one(gq, xx), rs.M_q, c2, invSq);
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
                double run = excl;
                int lastpos = -1;
#pragma unroll
                for (int u = 0; u < VEC; ++u) {
                    if (rv[u] > 0.0) lastpos = u;
                    run = __dadd_rn(run, rv[u]);
                    if (fu < 0 && run > th2) fu = u;
                }
                if (fu < 0) fu = lastpos;
            }
        } else {
            // rounding: the last token of the segment with positive mass
            int lastpos = -1;
#pragma unroll
            for (int u = 0; u < VEC; ++u)
                if (rv[u] > 0.0) lastpos = u;
            const unsigned pos = __ballot_sync(0xFFFFFFFFu, lastpos >= 0);
            fl = pos ? 31 - __clz(pos) : 0;
            if (lane == fl) fu = lastpos >= 0 ? lastpos : 0;
        }
        fu = __shfl_sync(0xFFFFFFFFu, fu, fl);
        tok = base + fl * VEC + fu;
        if (zero_res) status |= kZeroResidual;
    }
    if (lane == 0) {
        const int Lout = hard ? 0 : L;
        P.out_L[b] = Lout;
        int32_t* ot = P.out_tok + static_cast<size_t>(b) * (kk + 1);
        for (int i = 0; i <= kk; ++i) {
            int32_t v = -1;
            if (!hard) v = i < L ? P.ids[static_cast<size_t>(b) * kk + i] : (i == L ? tok : -1);
            ot[i] = v;
        }
        if (P.out_status) P.out_status[b] = status;
        P.rej_mask[b] = 0u;      // leave the workspace zeroed for the next call
        P.ticketB[b] = 0u;
    }
}

// ------------------------------------------------------------------------------------------
// Greedy finalize: one thread per request
__global__ void k_finalize_greedy(const Params P) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P.B) return;
    const int kk = P.k;
    const uint32_t mask = P.rej_mask[b];
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
    P.rej_mask[b] = 0u;
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
static cudaError_t launch_dependent(K kernel, unsigned grid, unsigned block, size_t smem,
                                    cudaStream_t st, const Params& P) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
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
template <typename E>
static cudaError_t launch_sampled(const Params& P, cudaStream_t st, cudaEvent_t ev0,
                                  cudaEvent_t ev1) {
    const size_t smem = 2 * static_cast<size_t>(P.CH) * sizeof(E);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_row_stats<E, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxChunkBytes * 2);
        cudaFuncSetAttribute(k_sample<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxChunkBytes * 2);

        attr = true;
    }
    const unsigned gridA = static_cast<unsigned>(P.k + 1) * P.B * P.nch;
    record_event(ev0, st);
    k_row_stats<E, false><<<gridA, kThreads, smem, st>>>(P);
    record_event(ev1, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dependent(k_sample<E>, static_cast<unsigned>(P.B) * P.nch, kThreads, smem, st, P);
}

template <typename E>
static cudaError_t launch_greedy(const Params& P, cudaStream_t st, cudaEvent_t ev0,
                                 cudaEvent_t ev1) {
    const size_t smem = static_cast<size_t>(P.CH) * sizeof(E);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_row_stats<E, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxChunkBytes * 2);
        attr = true;
    }
    const unsigned gridA = static_cast<unsigned>(P.k + 1) * P.B * P.nch;
    record_event(ev0, st);
    k_row_stats<E, true><<<gridA, kThreads, smem, st>>>(P);
    record_event(ev1, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dependent(k_finalize_greedy, (P.B + 127) / 128, 128, 0, st, P);
}

cudaError_t launch_verify(const Params& P, bool greedy, bool bf16, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1) {
    if (greedy)
        return bf16 ? launch_greedy<__nv_bfloat16>(P, st, ev0, ev1)
                    : launch_greedy<float>(P, st, ev0, ev1);
    return bf16 ? launch_sampled<__nv_bfloat16>(P, st, ev0, ev1)
                : launch_sampled<float>(P, st, ev0, ev1);
}

cudaError_t launch_philox(uint64_t seed, uint64_t round, const uint32_t* pos, const uint64_t* rid,
                          int n, uint32_t* out, cudaStream_t st) {
    if (n > 0) k_philox<<<(n + 255) / 256, 256, 0, st>>>(seed, round, pos, rid, n, out);
    return cudaGetLastError();
}

}  // namespace sd
