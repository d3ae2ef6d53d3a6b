// microbench.cu — FP32 pipe peaks on this B200 (the roofline denominators of DESIGN.md §6).
// FFMA (scalar), FFMA2 (packed f32x2, sm_100a) and MUFU.RCP throughput, all SMs, many
// independent chains per thread, timed with CUDA events.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
    unsigned long long x[kChains];
    const unsigned long long A = pk(a, a * 0.5f), B = pk(b, b * 0.25f);
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = pk(threadIdx.x * 1e-3f + c, c * 0.5f);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[c]));
        s += lo + hi;
    }
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void rcp_kernel(float* out, float a) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = 1.0f + threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
            x[c] += 0.5f;   // keeps ptxas from folding rcp(rcp(x))
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1234.5f) out[threadIdx.x] = s * a;
}

template <typename F>
float time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char** argv) {
    const int dev = argc > 1 ? atoi(argv[1]) : 0;
    cudaSetDevice(dev);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, dev);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    float* out;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    const double thr = (double)blocks * threads;
    float t1 = time_ms([&] { ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    float t2 = time_ms([&] { ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    float t3 = time_ms([&] { rcp_kernel<<<blocks, threads>>>(out, 1.0f); });
    const double ffma_tflops = thr * kIters * kChains * 2.0 / (t1 * 1e-3) / 1e12;
    const double ffma2_tflops = thr * kIters * kChains * 4.0 / (t2 * 1e-3) / 1e12;
    const double rcp_gops = thr * kIters * kChains / (t3 * 1e-3) / 1e9;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
           "\"mufu_rcp_gops\": %.1f, \"ffma_per_sm_per_clk_at_attr\": %.1f, \"ffma2_fma_per_sm_per_clk_at_attr\": %.1f, "
           "\"rcp_per_sm_per_clk_at_attr\": %.2f}\n",
           p.multiProcessorCount, clk_khz / 1e3, ffma_tflops, ffma2_tflops, rcp_gops,
           ffma_tflops * 1e12 / 2 / p.multiProcessorCount / (clk_khz * 1e3),
           ffma2_tflops * 1e12 / 2 / p.multiProcessorCount / (clk_khz * 1e3),
           rcp_gops * 1e9 / p.multiProcessorCount / (clk_khz * 1e3));
    return 0;
}
