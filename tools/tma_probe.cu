// tma_probe.cu -- per-SM throughput of TMA 1-D bulk copies (cp.async.bulk) in a persistent
// one-CTA-per-SM ring, the structure of verify_stream.cu: copy size, number of issuing threads,
// and source pattern (sequential chunks vs 64 KB row slices 512 KB apart).  Design evidence.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!try_wait(b, par)) {} }

// pattern 0: chunk i of this CTA = global chunk blockIdx + i*grid (sequential stripes)
// pattern 1: rows of 512 KB; CTA reads a 64 KB slice [rank*64K, +64K) of rows g, g+G, ...
__device__ __forceinline__ size_t chunk_off(int pattern, size_t i, int cb, size_t total) {
    if (pattern == 0) return ((size_t)blockIdx.x + i * gridDim.x) * cb % total;
    const size_t per_slice = 65536 / cb;               // chunks per 64 KB slice
    const size_t row = (blockIdx.x / 8) + (i / per_slice) * (gridDim.x / 8);
    const size_t rank = blockIdx.x % 8;
    return (row * 524288 + rank * 65536 + (i % per_slice) * cb) % total;
}

__device__ __forceinline__ float ex2a(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float max3nan(float a, float b, float c) { float d; asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

__global__ void __launch_bounds__(512, 1)
k_probe(const char* __restrict__ src, size_t total, size_t per_cta, int cb, int stages, int nprod,
        int pattern, float* out, unsigned long long* issue_cyc, int compute) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)stages * cb);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sa(empty + s)));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + stages)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t mine = per_cta;
    if (warp > 8) {   // extra warps: wait on a barrier nobody completes until the end (like row warps)
        if (lane == 0) {
            uint64_t* never = empty + stages;   // spare slot past the ring barriers
            uint32_t n = 0;
            while (!try_wait(never, 0) && n < 2000000) { ++n; if (n % 64 == 0) __nanosleep(500); }
        }
        return;
    }
    if (warp == 8) {
        if (lane < nprod) {
            unsigned long long cyc = 0, nis = 0;
            for (size_t i = lane; i < mine; i += nprod) {
                const int s = i % stages;
                wait(empty + s, ((i / stages) & 1) ^ 1);
                const char* g = src + chunk_off(pattern, i, cb, total);
                const unsigned long long t0 = clock64();
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(cb) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + (size_t)s * cb)), "l"(g), "r"(cb), "r"(sa(full + s)) : "memory");
                cyc += clock64() - t0;
                ++nis;
            }
            if (blockIdx.x == 0 && lane == 0) { issue_cyc[0] = cyc; issue_cyc[1] = nis; }
        }
        return;
    }
    float acc = 0.f;
    for (size_t i = 0; i < mine; ++i) {
        const int s = i % stages;
        wait(full + s, (i / stages) & 1);
        const float4* v = (const float4*)(sm + (size_t)s * cb);
        if (!compute) {
            for (int k = warp * 32 + lane; k < cb / 16; k += 256) { float4 x = v[k]; acc += x.x + x.y + x.z + x.w; }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
        } else {
            // 32 KB chunk: 8 vectors per thread into registers, release, then max + sum of ex2
            float4 x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = i < cb / 4096 ? v[warp * 32 + lane + i * 256] : make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = max3nan(m, max3nan(x[i].x, x[i].y, x[i].z), x[i].w);
            const float c2 = 1.4427f, nd = -m * c2;
            float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a0 += ex2a(fmaf(x[i].x, c2, nd)); a1 += ex2a(fmaf(x[i].y, c2, nd));
                a2 += ex2a(fmaf(x[i].z, c2, nd)); a3 += ex2a(fmaf(x[i].w, c2, nd));
            }
            acc += (a0 + a1) + (a2 + a3);
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// plain 128-bit loads into registers, 1 CTA/SM of 256 threads, U loads in flight per thread,
// same patterns (pattern 1: each warp reads consecutive 512 B of the CTA's current slice)
template <int U>
__global__ void __launch_bounds__(256, 1) k_ldg(const float4* __restrict__ src, size_t total, size_t per_cta_bytes,
                                               int pattern, float* out) {
    float acc = 0.f;
    const size_t chunks = per_cta_bytes / (U * 4096);
    for (size_t i = 0; i < chunks; ++i) {
        const size_t off = chunk_off(pattern, i, U * 4096, total) / 16;
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs(src + off + threadIdx.x + u * 256);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += x[u].x + x[u].y + x[u].z + x[u].w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const size_t total = 4ull << 30;
    char* src; float* out; unsigned long long* ic;
    cudaMalloc(&src, total); cudaMalloc(&out, 16); cudaMalloc(&ic, 16);
    cudaMemset(src, 0, total);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms / 8 * 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t per_cta = 24ull << 20;   // 24 MB per CTA (~3.4 GB total)
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("SMs=%d grid=%d\n", sms, grid);
    // sweep: copy size x ring depth x issuing threads (192 KB ring, 1 CTA per SM, stats consumers)
    for (int pattern : {0, 1})
    for (int cb : {16384, 32768})
    for (int nprod : {1, 2, 4, 12}) {
        const int stages = 196608 / cb, threads = 288, compute = 1;
        if (nprod > stages) continue;
        const size_t smem = (size_t)stages * cb + 2 * (stages + 1) * 8;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.numAttrs = 0;
        const int g = cfg.gridDim.x;
        auto launch = [&] { cudaLaunchKernelEx(&cfg, k_probe, (const char*)src, total, per_cta / cb, cb, stages, nprod, pattern, out, ic, compute); };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("pattern=%d copy=%d KB stages=%d issuers=%d: %7.1f GB/s (%6.1f GB/s per SM) %s\n", pattern, cb / 1024, stages, nprod,
               (double)g * per_cta * 3 / (ms * 1e-3) / 1e9, (double)per_cta * 3 / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
    }
    for (int pattern : {0, 1}) {
        auto l8 = [&] { k_ldg<8><<<grid, 256>>>((const float4*)src, total / 16, per_cta, pattern, out); };
        auto l4 = [&] { k_ldg<4><<<grid, 256>>>((const float4*)src, total / 16, per_cta, pattern, out); };
        for (int which = 0; which < 2; ++which) {
            auto f = [&] { if (which) l8(); else l4(); };
            f(); cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) f();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("ldg pattern=%d U=%d (1 CTA/SM, 256 thr): %7.1f GB/s\n", pattern, which ? 8 : 4,
                   (double)grid * per_cta * 3 / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
