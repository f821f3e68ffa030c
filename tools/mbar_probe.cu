// mbar_probe.cu -- wake-up latency of an mbarrier waiter after the arrive that completes the
// phase (same CTA, clock64), for the wait styles used in verify_stream.cu.  Design evidence.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ bool try_wait_hint(uint64_t* b, uint32_t par, uint32_t ns) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(par), "r"(ns) : "memory"); return ok; }
__device__ __forceinline__ bool test_wait(uint64_t* b, uint32_t par) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory"); return ok; }

__global__ void k(int mode, int reps, long long* out, int extra_spin) {
    __shared__ uint64_t bar;
    __shared__ long long t_arr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar))); }
    __syncthreads();
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
        const uint32_t par = r & 1;
        if (warp == 0) {
            if (lane == 0) {
                const long long t0 = clock64();
                while (clock64() - t0 < 2000 + (r * 37) % 1000) {}
                t_arr = clock64();
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
            }
        } else if (warp == 1) {
            if (mode == 0) { while (!try_wait(&bar, par)) {} }
            else if (mode == 1) { while (!try_wait_hint(&bar, par, 256)) {} }
            else if (mode == 2) { while (!try_wait_hint(&bar, par, 4000)) {} }
            else { while (!test_wait(&bar, par)) {} }
            const long long t1 = clock64();
            if (lane == 0) acc += t1 - *(volatile long long*)&t_arr;
        } else if (extra_spin) {   // other warps spinning on the same barrier style (contention)
            if (mode == 0) { while (!try_wait(&bar, par)) {} }
            else if (mode == 1) { while (!try_wait_hint(&bar, par, 256)) {} }
            else if (mode == 2) { while (!try_wait_hint(&bar, par, 4000)) {} }
            else { while (!test_wait(&bar, par)) {} }
        }
        __syncthreads();
    }
    if (threadIdx.x == 32) out[0] = acc / reps;
}
int main() {
    long long* out; cudaMalloc(&out, 8);
    const char* names[4] = {"try_wait", "try_wait hint 256ns", "try_wait hint 4000ns", "test_wait spin"};
    for (int extra : {0, 1})
        for (int mode = 0; mode < 4; ++mode) {
            k<<<1, extra ? 512 : 64>>>(mode, 2000, out, extra);
            long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("%-22s %s: wake-up latency %lld cycles %s\n", names[mode], extra ? "(+14 waiting warps)" : "", h, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
