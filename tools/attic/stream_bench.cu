// stream_bench.cu -- HBM read-streaming microbenchmark on B200 (design evidence for the verify
// kernel): TMA 1-D bulk copies through an mbarrier ring vs plain 128-bit loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!try_wait(b, par)) {} }

// consumers: warps 0..NC-1 each take items n % NC; producer = warp NC lane 0
template <int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1)
k_tma_ring(const float* __restrict__ src, size_t n_chunks, int chunk_bytes, int stages, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)stages * chunk_bytes);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + s)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t mine = (n_chunks > blockIdx.x) ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == NC) {
        if (lane == 0) {
            for (size_t i = 0; i < mine; ++i) {
                const int s = i % stages;
                if (i >= (size_t)stages) wait(empty + s, ((i / stages) - 1) & 1);
                const char* g = (const char*)src + (blockIdx.x + i * gridDim.x) * (size_t)chunk_bytes;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(chunk_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + (size_t)s * chunk_bytes)), "l"(g), "r"(chunk_bytes), "r"(sa(full + s)) : "memory");
            }
        }
        return;
    }
    float acc = 0.f;
    for (size_t i = warp; i < mine; i += NC) {
        const int s = i % stages;
        wait(full + s, (i / stages) & 1);
        const float4* v = (const float4*)(sm + (size_t)s * chunk_bytes);
        for (int k = lane; k < chunk_bytes / 16; k += 32) { float4 x = v[k]; acc += x.x + x.y + x.z + x.w; }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
    }
    if (acc == 1234.5f) out[0] = acc;
}

// kernel-shaped ring: stage = two 16 KB copies from two distant rows; every consumer warp reads
// its 1/NC share of every stage; a shared-memory counter elects the last warp, which releases
template <int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1)
k_coop_ring(const float* __restrict__ src, size_t n_items, int stages, size_t half, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    constexpr int CB = 16384;
    uint64_t* full = (uint64_t*)(sm + (size_t)stages * 2 * CB);
    uint64_t* empty = full + stages;
    uint32_t* cnt = (uint32_t*)(empty + stages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + s)));
            cnt[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t mine = (n_items > blockIdx.x) ? (n_items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == NC) {
        if (lane == 0) {
            for (size_t i = 0; i < mine; ++i) {
                const int s = i % stages;
                if (i >= (size_t)stages) wait(empty + s, ((i / stages) - 1) & 1);
                const char* g = (const char*)src + (blockIdx.x + i * gridDim.x) * (size_t)CB;
                unsigned char* d = sm + (size_t)s * 2 * CB;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(2 * CB) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(d)), "l"(g), "r"(CB), "r"(sa(full + s)) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(d + CB)), "l"(g + half), "r"(CB), "r"(sa(full + s)) : "memory");
            }
        }
        return;
    }
    float acc = 0.f;
    for (size_t i = 0; i < mine; ++i) {
        const int s = i % stages;
        wait(full + s, (i / stages) & 1);
        const float4* v = (const float4*)(sm + (size_t)s * 2 * CB);
        for (int k = warp * 32 + lane; k < 2 * CB / 16; k += 32 * NC) { float4 x = v[k]; acc += x.x + x.y + x.z + x.w; }
        __syncwarp();
        __threadfence_block();
        uint32_t old = 0;
        if (lane == 0) old = atomicAdd(cnt + s, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == NC - 1) {
            if (lane == 0) { cnt[s] = 0; asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory"); }
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// plain loads: each thread U independent 16B loads in flight per iteration
template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float4* __restrict__ src, size_t n4, float* out) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += x[u].x + x[u].y + x[u].z + x[u].w;
    }
    for (; i < n4; i += stride) { float4 x = __ldcs(src + i); acc += x.x + x.y + x.z + x.w; }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const size_t bytes = 2ull << 30;   // 2 GiB >> L2
    float* src; float* out;
    cudaMalloc(&src, bytes); cudaMalloc(&out, 16);
    cudaMemset(src, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        return bytes * 5.0 / (ms * 1e-3) / 1e9;
    };
    printf("SMs=%d\n", sms);
    for (int U : {4, 8, 16}) {
        for (int bpsm : {2, 4, 8}) {
            double gbs = timeit([&] {
                const int grid = sms * bpsm;
                if (U == 4) k_ldg<4><<<grid, 256>>>((const float4*)src, bytes / 16, out);
                if (U == 8) k_ldg<8><<<grid, 256>>>((const float4*)src, bytes / 16, out);
                if (U == 16) k_ldg<16><<<grid, 256>>>((const float4*)src, bytes / 16, out);
            });
            printf("ldg U=%2d blocks/SM=%d : %7.1f GB/s\n", U, bpsm, gbs);
        }
    }
    // stages must be a multiple of the consumer-warp count (slot s always belongs to warp s % NC,
    // otherwise a warp can wait on a slot two mbarrier phases ahead and the parity aliases)
    auto ring = [&](auto kern, int nc, int cb, int st) {
        const size_t smem = (size_t)st * cb + 2 * st * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        double gbs = timeit([&] { kern<<<sms, 32 * (nc + 1), smem>>>(src, bytes / cb, cb, st, out); });
        cudaError_t e = cudaGetLastError();
        printf("tma consumers=%d chunk=%5d stages=%2d (ring %3zu KB): %7.1f GB/s %s\n", nc, cb, st,
               smem / 1024, gbs, e ? cudaGetErrorString(e) : "");
    };
    for (int st : {4, 6, 8}) {
        const size_t smem = (size_t)st * 32768 + 2 * st * 8 + st * 4 + 64;
        cudaFuncSetAttribute(k_coop_ring<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        double gbs = timeit([&] { k_coop_ring<8><<<sms, 288, smem>>>(src, bytes / 2 / 16384, st, bytes / 2, out); });
        cudaError_t e = cudaGetLastError();
        printf("coop 8 warps, stage = 2 x 16 KB rows, stages=%d: %7.1f GB/s %s\n", st, gbs, e ? cudaGetErrorString(e) : "");
    }
    ring(k_tma_ring<4>, 4, 16384, 8);
    ring(k_tma_ring<4>, 4, 16384, 12);
    ring(k_tma_ring<6>, 6, 16384, 12);
    ring(k_tma_ring<6>, 6, 8192, 12);
    ring(k_tma_ring<6>, 6, 8192, 24);
    ring(k_tma_ring<8>, 8, 8192, 16);
    ring(k_tma_ring<8>, 8, 12288, 16);
    ring(k_tma_ring<8>, 8, 16384, 8);
    ring(k_tma_ring<8>, 8, 24576, 8);
    ring(k_tma_ring<4>, 4, 32768, 4);
    return 0;
}
