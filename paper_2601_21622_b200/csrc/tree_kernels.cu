// tree_kernels.cu -- lossless tree verification on sm_100a (sd_tree_verify).
//
// The paper drafts a depth-d tree with branching k (Alg. 2) and keeps the best
// of its independently verified paths, which is not lossless.  Reading
// D-2 of DESIGN.md replaces it with recursive rejection sampling over the children of each node
// (SpecInfer's multi-candidate rule, the paper's ref. [miao2024specinfer]): the m children
// c_1..c_m of a node are i.i.d. draws from the node's draft distribution q; with d_0 = p,
//   accept c_i iff u_i < min(1, d_{i-1}(x_i) / q(x_i)), else d_i = norm(max(0, d_{i-1} - q));
//   all m rejected: t ~ d_m;  a leaf reached: the bonus t ~ p_leaf.
// m = 1 is the chain of sd_verify (same Philox counters).  Full m-ary trees in level order: node 0
// is the root, the children of n are m n + 1 .. m n + m.
//
// One CTA per request walks its tree: per visited node a statistics pass over p (and q), one
// residual-mass pass per rejected candidate, and an inverse-CDF pass for the emitted token, all
// over the node's rows with 16-byte read-only loads (fp32 terms, fp64 sums -- reading C-11).  The
// walk is inherently sequential per request (each decision picks the next node), so requests are
// the parallel dimension; rows of the nodes not visited are never read.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <atomic>
#include <cstdlib>

#include "philox.cuh"
#include "ptx.cuh"
#include "verify.cuh"

namespace sd {

constexpr int kTT = 512;                 // threads per request CTA
constexpr int kTW = kTT / 32;
constexpr int kTreeMaxM = 8;

struct TreeParams {
    const void* p;                       // [B][N][ld_p]
    const void* q;                       // [B][Nint][ld_q]
    const int32_t* tok;                  // [B][N]
    int32_t B, m, d, V, N, Nint;
    int64_t ld_p, ld_q;
    float c2;                            // fl32(log2(e) / T); 0 = greedy
    uint64_t seed, round, rid_base;
    int32_t* out_L;
    int32_t* out_tok;                    // [B][d+1]
    int32_t* out_status;
    int32_t* out_node;
};

template <typename E>
struct TElt;
template <>
struct TElt<float> {
    static constexpr int VEC = 4;
    __device__ static void vec(const void* row, int g, float (&v)[4]) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(row) + g);
        v[0] = __uint_as_float(u.x);
        v[1] = __uint_as_float(u.y);
        v[2] = __uint_as_float(u.z);
        v[3] = __uint_as_float(u.w);
    }
    __device__ static float one(const void* row, int i) { return __ldg(static_cast<const float*>(row) + i); }
};
template <>
struct TElt<__nv_bfloat16> {
    static constexpr int VEC = 8;
    __device__ static void vec(const void* row, int g, float (&v)[8]) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(row) + g);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ static float one(const void* row, int i) {
        return __uint_as_float(static_cast<uint32_t>(__ldg(static_cast<const unsigned short*>(row) + i)) << 16);
    }
};

struct TreeSmem {
    float redf[kTW];
    double redd[kTW];
    int redi[kTW];
    double scan[kTT];
    float bc_f[4];
    double bc_d[4];
    int bc_i[4];
};

__device__ __forceinline__ float t_max_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// block reductions (every thread gets the result)
__device__ float tblock_max(float v, TreeSmem& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = t_max_nan(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    __syncthreads();
    if (lane == 0) s.redf[w] = v;
    __syncthreads();
    float r = s.redf[0];
    for (int i = 1; i < kTW; ++i) r = t_max_nan(r, s.redf[i]);
    return r;
}
__device__ double tblock_sum(double v, TreeSmem& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) s.redd[w] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < kTW; ++i) r += s.redd[i];   // fixed order: deterministic
    return r;
}
// (value, lowest index) max
__device__ void tblock_argmax(float& v, int& i, TreeSmem& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, i, o);
        if (ov > v || (ov == v && oi < i)) v = ov, i = oi;
    }
    __syncthreads();
    if (lane == 0) s.redf[w] = v, s.redi[w] = i;
    __syncthreads();
    v = s.redf[0];
    i = s.redi[0];
    for (int k = 1; k < kTW; ++k)
        if (s.redf[k] > v || (s.redf[k] == v && s.redi[k] < i)) v = s.redf[k], i = s.redi[k];
}

// Row statistics: D = fl32(max z * c2), S = sum 2^(z c2 - D); fault bits for NaN / +inf / empty.
template <typename E>
__device__ void trow_stats(const void* row, int V, float c2, float& D, double& S, int& fault,
                           TreeSmem& s) {
    constexpr int VEC = TElt<E>::VEC;
    const int nvv = (V + VEC - 1) / VEC;
    float m = -INFINITY;
    for (int g = threadIdx.x; g < nvv; g += kTT) {
        float v[VEC];
        TElt<E>::vec(row, g, v);
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (g * VEC + e < V) m = t_max_nan(m, v[e]);
    }
    m = tblock_max(m, s);
    fault = !(m < INFINITY) ? kNonfinite : (!(m > -INFINITY) ? kEmptyRow : 0);
    D = m * c2;
    double acc = 0.0;
    if (!fault) {
        for (int g = threadIdx.x; g < nvv; g += kTT) {
            float v[VEC];
            TElt<E>::vec(row, g, v);
            float t = 0.0f;
#pragma unroll
            for (int e = 0; e < VEC; ++e)
                if (g * VEC + e < V) t += ex2_approx(__fmaf_rn(v[e], c2, -D));
            acc += t;
        }
    }
    S = tblock_sum(acc, s);
}

// The walk state of one node: d_0 = p (D_p, S_p), q (D_q, S_q) and the residual masses R_1..R_i.
struct NodeDist {
    float Dp, Dq, ip, iq;            // fp32 terms: p(y) = 2^(z c2 - Dp) ip, q(y) likewise
    double Sp, Sq;
    float iR[kTreeMaxM + 1];         // 1 / R_l (fp32), or < 0: R_l == 0 (C-6: d_l = d_{l-1})
    double R[kTreeMaxM + 1];
};

// d_lv(y) in fp32 (lv = 0: p itself).  `raw`: the last level unnormalised, max(0, d_{lv-1} - q).
__device__ __forceinline__ float dlevel(float zp, float zq, float c2, const NodeDist& nd, int lv,
                                        bool raw) {
    float dcur = ex2_approx(__fmaf_rn(zp, c2, -nd.Dp)) * nd.ip;
    if (lv == 0) return dcur;
    const float qy = ex2_approx(__fmaf_rn(zq, c2, -nd.Dq)) * nd.iq;
    for (int l = 1; l <= lv; ++l) {
        const float r = fmaxf(dcur - qy, 0.0f);
        if (l == lv && raw) return nd.iR[l] < 0.0f ? dcur : r;
        if (nd.iR[l] >= 0.0f) dcur = r * nd.iR[l];
    }
    return dcur;
}

// Mass of max(0, d_{lv-1} - q) over the row (fp64 across vectors and threads).
template <typename E>
__device__ double residual_mass(const void* prow, const void* qrow, int V, float c2,
                                const NodeDist& nd, int lv, TreeSmem& s) {
    constexpr int VEC = TElt<E>::VEC;
    const int nvv = (V + VEC - 1) / VEC;
    double acc = 0.0;
    for (int g = threadIdx.x; g < nvv; g += kTT) {
        float vp[VEC], vq[VEC];
        TElt<E>::vec(prow, g, vp);
        TElt<E>::vec(qrow, g, vq);
        float t = 0.0f;
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (g * VEC + e < V) {
                const float prev = dlevel(vp[e], vq[e], c2, nd, lv - 1, false);
                const float qy = ex2_approx(__fmaf_rn(vq[e], c2, -nd.Dq)) * nd.iq;
                t += fmaxf(prev - qy, 0.0f);
            }
        acc += t;
    }
    return tblock_sum(acc, s);
}

// Inverse CDF (C-9) over the terms t(y) = d_lv(y) (raw last level) in ascending token id:
// thread t owns a contiguous range of vectors; its fp64 range mass, an exclusive block scan, and
// the owning thread's sequential walk find the first y with C(y) > theta = u * total.
template <typename E>
__device__ int tree_sample(const void* prow, const void* qrow, int V, float c2, const NodeDist& nd,
                           int lv, double u, TreeSmem& s) {
    constexpr int VEC = TElt<E>::VEC;
    const int nvv = (V + VEC - 1) / VEC;
    const int W = (nvv + kTT - 1) / kTT;
    const int g0 = threadIdx.x * W, g1 = min(nvv, g0 + W);
    auto term = [&](float zp, float zq) { return dlevel(zp, zq, c2, nd, lv, true); };
    double mine = 0.0;
    int lastpos = -1;
    for (int g = g0; g < g1; ++g) {
        float vp[VEC], vq[VEC];
        TElt<E>::vec(prow, g, vp);
        if (qrow) TElt<E>::vec(qrow, g, vq);
        float t = 0.0f;
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (g * VEC + e < V) {
                const float x = term(vp[e], qrow ? vq[e] : 0.0f);
                t += x;
                if (x > 0.0f) lastpos = g * VEC + e;
            }
        mine += t;
    }
    s.scan[threadIdx.x] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {            // sequential exclusive scan, fixed order
        double run = 0.0;
        for (int i = 0; i < kTT; ++i) {
            const double v = s.scan[i];
            s.scan[i] = run;
            run += v;
        }
        s.bc_d[0] = run;               // total
    }
    __syncthreads();
    const double total = s.bc_d[0];
    const double theta = u * total;
    const double lo = s.scan[threadIdx.x];
    if (threadIdx.x == 0) s.bc_i[0] = -1;
    __syncthreads();
    // the owner: lo <= theta < lo + mine (strict C(y) > theta); the last thread with mass also
    // records itself for the rounding clamp
    if (mine > 0.0 && theta >= lo && theta < lo + mine) {
        double run = lo;
        int found = -1;
        for (int g = g0; g < g1 && found < 0; ++g) {
            float vp[VEC], vq[VEC];
            TElt<E>::vec(prow, g, vp);
            if (qrow) TElt<E>::vec(qrow, g, vq);
            float t = 0.0f;
            for (int e = 0; e < VEC && found < 0; ++e)
                if (g * VEC + e < V) {
                    const float x = term(vp[e], qrow ? vq[e] : 0.0f);
                    // (the same fp32 vector sum the range mass used, walked element by element)
                    if (x > 0.0f && run + static_cast<double>(t + x) > theta) found = g * VEC + e;
                    t += x;
                }
            run += t;
        }
        if (found < 0) found = lastpos;   // rounding: the range's last positive-mass token
        atomicMax(&s.bc_i[0], found);     // (one owner in exact arithmetic)
    }
    __syncthreads();
    int tok = s.bc_i[0];
    if (tok < 0) {                        // theta past every range (rounding): the last positive
        if (lastpos >= 0) atomicMax(&s.bc_i[1], lastpos);
        __syncthreads();
        tok = s.bc_i[1];
    }
    __syncthreads();
    return tok;
}

template <typename E>
__global__ void __launch_bounds__(kTT) k_tree_verify(const TreeParams P) {
    __shared__ TreeSmem s;
    const int b = blockIdx.x;
    const int m = P.m, d = P.d, V = P.V;
    const size_t esz = sizeof(E);
    const uint64_t rid = P.rid_base + static_cast<uint64_t>(b);
    const bool greedy = P.c2 == 0.0f;
    const int32_t* tok = P.tok + static_cast<size_t>(b) * P.N;
    int node = 0, depth = 0, status = 0;
    int32_t path[32];                    // d <= 31
    int emitted = -1;
    if (threadIdx.x == 0) s.bc_i[1] = -1;
    while (true) {
        const void* prow = static_cast<const char*>(P.p) + (static_cast<size_t>(b) * P.N + node) * P.ld_p * esz;
        if (greedy) {
            float v = -INFINITY, nanacc = -INFINITY;
            int gi = INT_MAX;
            constexpr int VEC = TElt<E>::VEC;
            const int nvv = (V + VEC - 1) / VEC;
            for (int g = threadIdx.x; g < nvv; g += kTT) {
                float x[VEC];
                TElt<E>::vec(prow, g, x);
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if (g * VEC + e < V) {
                        nanacc = t_max_nan(nanacc, x[e]);
                        if (x[e] > v) v = x[e], gi = g * VEC + e;
                    }
            }
            nanacc = tblock_max(nanacc, s);
            tblock_argmax(v, gi, s);
            if (!(nanacc < INFINITY)) { status = kNonfinite; break; }
            if (!(v > -INFINITY)) { status = kEmptyRow; break; }
            if (depth == d) { emitted = gi; break; }
            int next = -1;
            for (int i = 0; i < m; ++i) {
                const int x = tok[m * node + 1 + i];
                if (x < 0 || x >= V) { status = kBadId; break; }
                if (x == gi) { next = m * node + 1 + i; break; }
            }
            if (status) break;
            if (next < 0) { emitted = gi; break; }
            path[depth++] = gi;
            node = next;
            continue;
        }
        NodeDist nd;
        int fp;
        trow_stats<E>(prow, V, P.c2, nd.Dp, nd.Sp, fp, s);
        if (fp) { status = fp; break; }
        nd.ip = static_cast<float>(1.0 / nd.Sp);
        if (depth == d) {                                      // leaf: bonus t ~ p_leaf (C-3)
            const double u = unit24(verify_words(P.seed, static_cast<uint32_t>(depth), P.round, rid).y);
            emitted = tree_sample<E>(prow, nullptr, V, P.c2, nd, 0, u, s);
            break;
        }
        const void* qrow = static_cast<const char*>(P.q) + (static_cast<size_t>(b) * P.Nint + node) * P.ld_q * esz;
        int fq;
        trow_stats<E>(qrow, V, P.c2, nd.Dq, nd.Sq, fq, s);
        if (fq) { status = fq; break; }
        nd.iq = static_cast<float>(1.0 / nd.Sq);
        int next = -1;
        for (int i = 0; i < m && next < 0; ++i) {
            const int x = tok[m * node + 1 + i];
            if (x < 0 || x >= V) { status = kBadId; break; }
            if (i > 0) {                                       // d_i = norm(max(0, d_{i-1} - q))
                const double R = residual_mass<E>(prow, qrow, V, P.c2, nd, i, s);
                nd.R[i] = R;
                nd.iR[i] = R > 0.0 ? static_cast<float>(1.0 / R) : -1.0f;
                if (!(R > 0.0)) status |= kZeroResidual;
            }
            // d_{i}(x) and q(x) at the candidate, fp64 from the same fp32 terms
            const float zp = TElt<E>::one(prow, x), zq = TElt<E>::one(qrow, x);
            const double dx = static_cast<double>(dlevel(zp, zq, P.c2, nd, i, false));
            const double qx = static_cast<double>(ex2_approx(__fmaf_rn(zq, P.c2, -nd.Dq)) * nd.iq);
            const double a = qx > 0.0 ? dx / qx : 0.0;       // (C-7: q(x) = 0 rejects)
            if (zq == -INFINITY) status |= kZeroQ;
            if (!(a >= 1.0)) {
                const double u = unit24(verify_words(P.seed, static_cast<uint32_t>(depth + 32 * i), P.round, rid).x);
                if (u >= a) continue;                          // reject: the next candidate
            }
            next = m * node + 1 + i;
            path[depth] = x;
        }
        if (status & kHard) break;
        if (next >= 0) {
            ++depth;
            node = next;
            continue;
        }
        // every candidate rejected: t ~ d_m
        const double R = residual_mass<E>(prow, qrow, V, P.c2, nd, m, s);
        nd.R[m] = R;
        nd.iR[m] = R > 0.0 ? static_cast<float>(1.0 / R) : -1.0f;
        if (!(R > 0.0)) status |= kZeroResidual;
        const double u = unit24(verify_words(P.seed, static_cast<uint32_t>(depth), P.round, rid).y);
        emitted = tree_sample<E>(prow, qrow, V, P.c2, nd, m, u, s);
        break;
    }
    if (threadIdx.x == 0) {
        const bool hard = (status & kHard) != 0;
        const int L = hard ? 0 : depth;
        P.out_L[b] = L;
        int32_t* ot = P.out_tok + static_cast<size_t>(b) * (d + 1);
        for (int i = 0; i <= d; ++i) ot[i] = hard ? -1 : (i < L ? path[i] : (i == L ? emitted : -1));
        if (P.out_status) P.out_status[b] = status;
        if (P.out_node) P.out_node[b] = node;
    }
}


// ------------------------------------------------------------------------------------------
// k_tree_cluster: the same walk with one 8-CTA cluster per request.  CTA rank r keeps its slice
// of the current node's p and q rows (vectors [r SV, (r+1) SV)) in shared memory -- one TMA load
// per row per node, the algorithmic minimum -- and every pass of the node (statistics, the
// residual masses of the rejected candidates, the inverse CDF) runs on chip; the cluster combines
// the slices' partials through distributed shared memory (each CTA posts its partial, a cluster
// barrier, every CTA reads all eight in rank order, so every CTA takes the same decisions).
// Same readings and counters as k_tree_verify (D-2, C-8, C-9); sums fp64 above one vector.
constexpr int kTCMax = 16;               // CTAs per cluster (one request): 8 or 16
constexpr int kTCT = 256;                // threads per CTA
constexpr int kTCW = kTCT / 32;
constexpr int kTCMaxBytes = 200 * 1024;  // shared memory for the two slices

struct TCSmem {
    float redf[kTCW];
    double redd[kTCW];
    int redi[kTCW];
    double scan[kTCT];
    double post[2][4];                   // this CTA's partials, double-buffered by phase
    int bc;
};

__device__ __forceinline__ float tc_max(float v, TCSmem& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = t_max_nan(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    __syncthreads();
    if (lane == 0) s.redf[w] = v;
    __syncthreads();
    float r = s.redf[0];
    for (int i = 1; i < kTCW; ++i) r = t_max_nan(r, s.redf[i]);
    return r;
}
__device__ __forceinline__ double tc_sum(double v, TCSmem& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) s.redd[w] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < kTCW; ++i) r += s.redd[i];
    return r;
}
// every CTA posts K values; after the cluster barrier every thread holds all ranks' posts
template <int kTC, int K>
__device__ __forceinline__ void tc_exchange(TCSmem& s, int& ph, const double (&mine)[K],
                                            double (&all)[kTC][K]) {
    double* slot = s.post[ph & 1];
    if (threadIdx.x == 0)
        #pragma unroll
        for (int i = 0; i < K; ++i) slot[i] = mine[i];
    cl_sync();
    #pragma unroll
    for (int r = 0; r < kTC; ++r)
        #pragma unroll
        for (int i = 0; i < K; ++i) all[r][i] = cl_ld_f64(cl_map(slot + i, r));
    ++ph;
}

template <typename E, int kTC>
__global__ void __launch_bounds__(kTCT, kTC == 16 ? 2 : 1) k_tree_cluster(const TreeParams P) {
    using TE = TElt<E>;
    constexpr int VEC = TE::VEC;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ TCSmem s;
    __shared__ __align__(8) uint64_t bar[2];
    const int b = blockIdx.x / kTC;
    const int rank = static_cast<int>(cl_rank());
    const int m = P.m, d = P.d, V = P.V;
    const bool greedy = P.c2 == 0.0f;
    const uint64_t rid = P.rid_base + static_cast<uint64_t>(b);
    const int32_t* tok = P.tok + static_cast<size_t>(b) * P.N;
    const int nvv = (V + VEC - 1) / VEC;
    const int SV = (nvv + kTC - 1) / kTC;                  // vectors per slice
    const int v0 = rank * SV, nv = max(0, min(SV, nvv - v0));
    const uint4* sp = reinterpret_cast<const uint4*>(smem);
    const uint4* sq = sp + SV;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    int ph = 0;                                            // cluster exchange phase
    uint32_t lp = 0;                                       // node loads (mbarrier parity)
    int node = 0, depth = 0, status = 0, emitted = -1, writer = 0;
    int32_t path[32];
    auto elem = [&](const uint4* base, int g, float (&v)[VEC]) {
        const uint4 u = base[g];
        if constexpr (VEC == 4) {
            v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
            v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
        } else {
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                v[2 * i] = __uint_as_float(w[i] << 16);
                v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
            }
        }
    };
    while (true) {
        const bool internal = depth < d;
        const char* prow = static_cast<const char*>(P.p) + (static_cast<size_t>(b) * P.N + node) * P.ld_p * sizeof(E);
        const char* qrow = internal && !greedy
                               ? static_cast<const char*>(P.q) + (static_cast<size_t>(b) * P.Nint + node) * P.ld_q * sizeof(E)
                               : nullptr;
        // ---- this node's slices into shared memory (the previous node's reads are done) ------
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(&bar[0], nv * 16u);
            if (nv) bulk_g2s(smem, prow + static_cast<size_t>(v0) * 16, nv * 16u, &bar[0]);
        } else if (threadIdx.x == 32) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t nb = qrow ? nv * 16u : 0u;
            mbar_arrive_expect_tx(&bar[1], nb);
            if (nb) bulk_g2s(smem + static_cast<size_t>(SV) * 16, qrow + static_cast<size_t>(v0) * 16, nb, &bar[1]);
        }
        mbar_wait(&bar[0], lp & 1u);
        mbar_wait(&bar[1], lp & 1u);
        ++lp;
        if (greedy) {
            // (max, lowest index) over the row; NaN / +inf faults
            float v = -INFINITY, nanacc = -INFINITY;
            int gi = INT_MAX;
            for (int g = threadIdx.x; g < nv; g += kTCT) {
                float x[VEC];
                elem(sp, g, x);
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if ((v0 + g) * VEC + e < V) {
                        nanacc = t_max_nan(nanacc, x[e]);
                        if (x[e] > v) v = x[e], gi = (v0 + g) * VEC + e;
                    }
            }
            nanacc = tc_max(nanacc, s);
            // block argmax (value, lowest index)
            {
                const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xFFFFFFFFu, v, o);
                    const int oi = __shfl_xor_sync(0xFFFFFFFFu, gi, o);
                    if (ov > v || (ov == v && oi < gi)) v = ov, gi = oi;
                }
                __syncthreads();
                if (lane == 0) s.redf[w] = v, s.redi[w] = gi;
                __syncthreads();
                v = s.redf[0];
                gi = s.redi[0];
                for (int i = 1; i < kTCW; ++i)
                    if (s.redf[i] > v || (s.redf[i] == v && s.redi[i] < gi)) v = s.redf[i], gi = s.redi[i];
            }
            double all[kTC][3];
            const double mine[3] = {static_cast<double>(v), static_cast<double>(gi), static_cast<double>(nanacc)};
            tc_exchange<kTC, 3>(s, ph, mine, all);
            float V_ = -INFINITY, nan_ = -INFINITY;
            int G_ = INT_MAX;
            #pragma unroll
            for (int r = 0; r < kTC; ++r) {
                const float rv = static_cast<float>(all[r][0]);
                const int ri = static_cast<int>(all[r][1]);
                nan_ = t_max_nan(nan_, static_cast<float>(all[r][2]));
                if (rv > V_ || (rv == V_ && ri < G_)) V_ = rv, G_ = ri;
            }
            if (!(nan_ < INFINITY)) { status = kNonfinite; break; }
            if (!(V_ > -INFINITY)) { status = kEmptyRow; break; }
            if (depth == d) { emitted = G_; break; }
            int next = -1;
            for (int i = 0; i < m; ++i) {
                const int x = tok[m * node + 1 + i];
                if (x < 0 || x >= V) { status = kBadId; break; }
                if (x == G_) { next = m * node + 1 + i; break; }
            }
            if (status) break;
            if (next < 0) { emitted = G_; break; }
            path[depth++] = G_;
            node = next;
            continue;
        }
        // ---- statistics of p (and q): slice (max, sum), combined over the cluster -------------
        float Dl[2] = {-INFINITY, -INFINITY};
        double Sl[2] = {0.0, 0.0};
        for (int w = 0; w < (qrow ? 2 : 1); ++w) {
            const uint4* base = w ? sq : sp;
            float mx = -INFINITY;
            for (int g = threadIdx.x; g < nv; g += kTCT) {
                float x[VEC];
                elem(base, g, x);
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if ((v0 + g) * VEC + e < V) mx = t_max_nan(mx, x[e]);
            }
            mx = tc_max(mx, s);
            const float D = mx * P.c2;
            double acc = 0.0;
            if (mx < INFINITY && mx > -INFINITY) {
                for (int g = threadIdx.x; g < nv; g += kTCT) {
                    float x[VEC];
                    elem(base, g, x);
                    float t = 0.0f;
#pragma unroll
                    for (int e = 0; e < VEC; ++e)
                        if ((v0 + g) * VEC + e < V) t += ex2_approx(__fmaf_rn(x[e], P.c2, -D));
                    acc += t;
                }
            }
            Dl[w] = !(mx < INFINITY) ? NAN : D;
            Sl[w] = tc_sum(acc, s);
        }
        double all[kTC][4];
        {
            const double mine[4] = {static_cast<double>(Dl[0]), Sl[0], static_cast<double>(Dl[1]), Sl[1]};
            tc_exchange<kTC, 4>(s, ph, mine, all);
        }
        NodeDist nd;
        int fp = 0, fq = 0;
        {
            float Dp = -INFINITY, Dq = -INFINITY;
            #pragma unroll
            for (int r = 0; r < kTC; ++r) {
                Dp = t_max_nan(Dp, static_cast<float>(all[r][0]));
                Dq = t_max_nan(Dq, static_cast<float>(all[r][2]));
            }
            double Sp = 0.0, Sq = 0.0;
            #pragma unroll
            for (int r = 0; r < kTC; ++r) {
                if (all[r][1] > 0.0) Sp += all[r][1] * exp2(all[r][0] - static_cast<double>(Dp));
                if (all[r][3] > 0.0) Sq += all[r][3] * exp2(all[r][2] - static_cast<double>(Dq));
            }
            fp = !(Dp < INFINITY) ? kNonfinite : (!(Dp > -INFINITY) ? kEmptyRow : 0);
            if (qrow) fq = !(Dq < INFINITY) ? kNonfinite : (!(Dq > -INFINITY) ? kEmptyRow : 0);
            nd.Dp = Dp; nd.Sp = Sp; nd.ip = static_cast<float>(1.0 / Sp);
            nd.Dq = Dq; nd.Sq = Sq; nd.iq = qrow ? static_cast<float>(1.0 / Sq) : 0.0f;
        }
        if (fp) { status = fp; break; }
        // the slice's terms of level lv (raw last level), and the inverse CDF over the cluster
        auto slice_mass = [&](int lv, bool use_q) -> double {
            double acc = 0.0;
            for (int g = threadIdx.x; g < nv; g += kTCT) {
                float vp[VEC], vq[VEC];
                elem(sp, g, vp);
                if (use_q) elem(sq, g, vq);
                float t = 0.0f;
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if ((v0 + g) * VEC + e < V) t += dlevel(vp[e], use_q ? vq[e] : 0.0f, P.c2, nd, lv, true);
                acc += t;
            }
            return tc_sum(acc, s);
        };
        // Inverse CDF over the cluster: per-thread contiguous ranges of the slice, the slice
        // total posted with the slice's last positive-mass token (one exchange), the owner rank
        // found in rank order, and the owner CTA's owner thread walks its range.  Returns the
        // total mass (every CTA); *owner_out = the writing rank, *tok_out = the token (valid in
        // the writing CTA).
        auto sample = [&](int lv, bool use_q, int* owner_out, int* tok_out) -> double {
            const int W = (nv + kTCT - 1) / kTCT;
            const int g0 = threadIdx.x * W, g1 = min(nv, g0 + W);
            double mine = 0.0;
            int lastpos = -1;
            for (int g = g0; g < g1; ++g) {
                float vp[VEC], vq[VEC];
                elem(sp, g, vp);
                if (use_q) elem(sq, g, vq);
                float t = 0.0f;
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                    if ((v0 + g) * VEC + e < V) {
                        const float x = dlevel(vp[e], use_q ? vq[e] : 0.0f, P.c2, nd, lv, true);
                        t += x;
                        if (x > 0.0f) lastpos = (v0 + g) * VEC + e;
                    }
                mine += t;
            }
            s.scan[threadIdx.x] = mine;
            __syncthreads();
            if (threadIdx.x == 0) {                        // sequential exclusive scan, fixed order
                double run = 0.0;
                for (int i = 0; i < kTCT; ++i) {
                    const double v = s.scan[i];
                    s.scan[i] = run;
                    run += v;
                }
                s.redd[0] = run;
                s.bc = -1;
            }
            __syncthreads();
            const double tot_r = s.redd[0];
            int lp2 = lastpos;                             // the slice's last positive-mass token
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lp2 = max(lp2, __shfl_xor_sync(0xFFFFFFFFu, lp2, o));
            if ((threadIdx.x & 31) == 0) atomicMax(&s.bc, lp2);
            __syncthreads();
            const int last_r = s.bc;
            double allm[kTC][2];
            const double post[2] = {tot_r, static_cast<double>(last_r)};
            tc_exchange<kTC, 2>(s, ph, post, allm);
            double total = 0.0;
#pragma unroll
            for (int r = 0; r < kTC; ++r) total += allm[r][0];
            const double u = unit24(verify_words(P.seed, static_cast<uint32_t>(depth), P.round, rid).y);
            const double theta = u * total;
            int owner = -1, lastr = -1;
            double before = 0.0, acc = 0.0;
#pragma unroll
            for (int r = 0; r < kTC; ++r) {
                if (allm[r][0] > 0.0) lastr = r;
                if (owner < 0 && allm[r][0] > 0.0 && theta >= acc && theta < acc + allm[r][0]) {
                    owner = r;
                    before = acc;
                }
                acc += allm[r][0];
            }
            if (owner < 0) {                               // rounding: the last token with mass
                *owner_out = 0;
                *tok_out = lastr >= 0 ? static_cast<int>(allm[lastr][1]) : 0;
                return total;
            }
            *owner_out = owner;
            *tok_out = -1;
            if (owner == rank) {
                __syncthreads();
                if (threadIdx.x == 0) s.bc = -1;
                __syncthreads();
                const double lo = before + s.scan[threadIdx.x];
                if (mine > 0.0 && theta >= lo && theta < lo + mine) {
                    double run = lo;
                    int found = -1;
                    for (int g = g0; g < g1 && found < 0; ++g) {
                        float vp[VEC], vq[VEC];
                        elem(sp, g, vp);
                        if (use_q) elem(sq, g, vq);
                        float t = 0.0f;
                        for (int e = 0; e < VEC && found < 0; ++e)
                            if ((v0 + g) * VEC + e < V) {
                                const float x = dlevel(vp[e], use_q ? vq[e] : 0.0f, P.c2, nd, lv, true);
                                if (x > 0.0f && run + static_cast<double>(t + x) > theta) found = (v0 + g) * VEC + e;
                                t += x;
                            }
                        run += t;
                    }
                    if (found < 0) found = lastpos;
                    atomicMax(&s.bc, found);
                }
                __syncthreads();
                *tok_out = s.bc >= 0 ? s.bc : last_r;
            }
            return total;
        };
        if (depth == d) {                                  // leaf: bonus t ~ p_leaf (C-3)
            sample(0, false, &writer, &emitted);
            break;
        }
        if (fq) { status = fq; break; }
        int next = -1;
        for (int i = 0; i < m && next < 0; ++i) {
            const int x = tok[m * node + 1 + i];
            if (x < 0 || x >= V) { status = kBadId; break; }
            if (i > 0) {                                   // d_i = norm(max(0, d_{i-1} - q))
                nd.iR[i] = 0.0f;                           // (raw level i: max(0, d_{i-1} - q))
                const double loc = slice_mass(i, true);
                double allr[kTC][1];
                const double mine1[1] = {loc};
                tc_exchange<kTC, 1>(s, ph, mine1, allr);
                double R = 0.0;
                #pragma unroll
                for (int r = 0; r < kTC; ++r) R += allr[r][0];
                nd.R[i] = R;
                nd.iR[i] = R > 0.0 ? static_cast<float>(1.0 / R) : -1.0f;
                if (!(R > 0.0)) status |= kZeroResidual;
            }
            const float zp = TE::one(prow, x), zq = TE::one(qrow, x);
            const double dx = static_cast<double>(dlevel(zp, zq, P.c2, nd, i, false));
            const double qx = static_cast<double>(ex2_approx(__fmaf_rn(zq, P.c2, -nd.Dq)) * nd.iq);
            const double a = qx > 0.0 ? dx / qx : 0.0;
            if (zq == -INFINITY) status |= kZeroQ;
            if (!(a >= 1.0)) {
                const double u = unit24(verify_words(P.seed, static_cast<uint32_t>(depth + 32 * i), P.round, rid).x);
                if (u >= a) continue;
            }
            next = m * node + 1 + i;
            path[depth] = x;
        }
        if (status & kHard) break;
        if (next >= 0) {
            ++depth;
            node = next;
            continue;
        }
        {                                                  // every candidate rejected: t ~ d_m
            // the sampling exchange also yields R_m = max(0, d_{m-1} - q)'s total mass
            nd.iR[m] = 0.0f;                               // (raw level m: max(0, d_{m-1} - q))
            const double R = sample(m, true, &writer, &emitted);
            nd.R[m] = R;
            if (!(R > 0.0)) {                              // C-6: d_m = d_{m-1}
                status |= kZeroResidual;
                nd.iR[m] = -1.0f;
                sample(m, true, &writer, &emitted);
            }
        }
        break;
    }
    if (rank == writer && threadIdx.x == 0) {   // (the rank that holds the emitted token)
        const bool hard = (status & kHard) != 0;
        const int L = hard ? 0 : depth;
        P.out_L[b] = L;
        int32_t* ot = P.out_tok + static_cast<size_t>(b) * (d + 1);
        for (int i = 0; i <= d; ++i) ot[i] = hard ? -1 : (i < L ? path[i] : (i == L ? emitted : -1));
        if (P.out_status) P.out_status[b] = status;
        if (P.out_node) P.out_node[b] = node;
    }
    cl_sync();   // (no CTA leaves while a peer may still read its posts)
}

template <typename E, int CT>
static cudaError_t launch_tree_cluster(const TreeParams& P, size_t smem, cudaStream_t st) {
    static std::atomic<uint64_t> optin{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(optin.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(k_tree_cluster<E, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kTCMaxBytes));
        if (e != cudaSuccess) return e;
        if (CT > 8) {
            e = cudaFuncSetAttribute(k_tree_cluster<E, CT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        optin.fetch_or(bit, std::memory_order_acq_rel);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(P.B) * CT);
    cfg.blockDim = dim3(kTCT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CT;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_tree_cluster<E, CT>, P);
}

cudaError_t launch_tree(const TreeParams& P, bool bf16, cudaStream_t st) {
    if (P.B == 0) return cudaSuccess;
    // one 8-CTA cluster per request when the node's two row slices fit in shared memory
    // (V <= ~200K fp32 / ~400K bf16); else one CTA per request streaming the rows
    // (STARSD_TREE_CLUSTER = 0: off; 8 (default) or 16 CTAs per cluster -- 16 measured slower)
    static const int cl = getenv("STARSD_TREE_CLUSTER") ? atoi(getenv("STARSD_TREE_CLUSTER")) : 8;
    const int VEC = bf16 ? 8 : 4;
    const int CT = cl == 8 ? 8 : 16;
    const size_t SV = ((P.V + VEC - 1) / VEC + CT - 1) / CT;
    const size_t smem = 2 * SV * 16;
    if (cl && smem <= static_cast<size_t>(kTCMaxBytes) && P.d <= 31) {
        if (CT == 8)
            return bf16 ? launch_tree_cluster<__nv_bfloat16, 8>(P, smem, st)
                        : launch_tree_cluster<float, 8>(P, smem, st);
        return bf16 ? launch_tree_cluster<__nv_bfloat16, 16>(P, smem, st)
                    : launch_tree_cluster<float, 16>(P, smem, st);
    }
    if (bf16) k_tree_verify<__nv_bfloat16><<<P.B, kTT, 0, st>>>(P);
    else k_tree_verify<float><<<P.B, kTT, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace sd
