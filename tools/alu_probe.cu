// alu_probe.cu -- per-SM throughput of the stats-pass instructions on this GPU (design evidence):
// MUFU.EX2 (ex2.approx.ftz.f32), FFMA2 (fma.rn.f32x2), FMNMX3 (max.NaN.f32 3-input), FADD.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_probe tools/alu_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
constexpr int ITER = 4096, ILP = 8;
__global__ void k_ex2(float* out, float s) {
    float x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = s * (threadIdx.x + i) * 1e-6f;
    for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    float a = 0; for (int i = 0; i < ILP; ++i) a += x[i];
    if (a == 1234.5f) out[0] = a;
}
__global__ void k_ffma2(float* out, float s) {
    unsigned long long x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = (unsigned long long)(threadIdx.x + i);
    const unsigned long long c = 0x3f8000003f800000ull;
    for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x[i]) : "l"(c));
    unsigned long long a = 0; for (int i = 0; i < ILP; ++i) a ^= x[i];
    if (a == 12345) out[0] = (float)a;
}
__global__ void k_max3(float* out, float s) {
    float x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = s * (threadIdx.x + i);
    const float y = s * 3.f, z = s * 5.f;
    for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("max.NaN.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(y), "f"(z));
    float a = 0; for (int i = 0; i < ILP; ++i) a += x[i];
    if (a == 1234.5f) out[0] = a;
}
__global__ void k_fadd(float* out, float s) {
    float x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = s * (threadIdx.x + i);
    for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(s));
    float a = 0; for (int i = 0; i < ILP; ++i) a += x[i];
    if (a == 1234.5f) out[0] = a;
}
int main() {
    float* out; cudaMalloc(&out, 16);
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, void (*k)(float*, float), int per) {
        for (int tpb : {256, 512, 1024}) {
            const int grid = sms * (2048 / tpb);
            k<<<grid, tpb>>>(out, 1.0f); cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) k<<<grid, tpb>>>(out, 1.0f);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double ops = 5.0 * grid * tpb * (double)ITER * ILP * per;
            const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
            printf("%-8s tpb=%4d: %8.1f Gop/s  %6.2f lane-ops/clk/SM (at %d MHz nominal)\n", name, tpb,
                   ops / (ms * 1e-3) / 1e9, per_clk_sm, clk / 1000);
        }
    };
    run("ex2", k_ex2, 1);
    run("ffma2", k_ffma2, 2);
    run("max3", k_max3, 1);
    run("fadd", k_fadd, 1);
    return 0;
}
