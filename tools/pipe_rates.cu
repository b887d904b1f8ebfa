// pipe_rates.cu -- B200 issue/pipe microbenchmarks behind the roofline
// denominator (MEASURED_PEAKS.json has HBM and bf16 only).  Each kernel runs
// 8 independent dependency chains per thread, 148*8 blocks x 256 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_rates tools/pipe_rates.cu
#include <cuda_runtime.h>

#include <cstdio>

#define CHAINS 8
#define UNROLL 16

__global__ void k_ffma_rcc(float* out, int iters, float a, float b) {
    float x[CHAINS];
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
    float r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5f) out[0] = r;
}

// three register sources: y, z differ per thread and per chain
__global__ void k_ffma_rrr(float* out, const float* in, int iters) {
    float x[CHAINS], y[CHAINS], z[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
        z[c] = in[(threadIdx.x * 7 + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], y[c], z[c]);
    float r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5f) out[0] = r;
}

__global__ void k_fmul_rr(float* out, const float* in, int iters) {
    float x[CHAINS], y[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = x[c] * y[c];
    float r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5f) out[0] = r;
}

// FMNMX with |.| modifiers, register sources
__global__ void k_fmnmx(float* out, const float* in, int iters) {
    float x[CHAINS], y[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = -fmaxf(fabsf(x[c]), fabsf(y[c]));
    float r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5f) out[0] = r;
}

// mix close to the fused search inner loop: per step 3 FFMA (rrr) + 1 FMNMX
__global__ void k_mix(float* out, const float* in, int iters) {
    float x[CHAINS], y[CHAINS], z[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
        z[c] = in[(threadIdx.x * 3 + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL / 4; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                float t = fmaf(x[c], y[c], z[c]);
                t = fmaf(t, y[c], z[c]);
                t = fmaf(t, y[c], z[c]);
                x[c] = fmaxf(fabsf(t), y[c]);
            }
    float r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5f) out[0] = r;
}

// FP64: dependent chains of DFMA (reg,reg,reg) and DMUL/DADD pairs
__global__ void k_dfma(float* out, const float* in, int iters) {
    double x[CHAINS], y[CHAINS], z[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
        z[c] = in[(threadIdx.x * 5 + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], y[c], z[c]);
    double r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5) out[0] = (float)r;
}

__global__ void k_dmul_dadd(float* out, const float* in, int iters) {
    double x[CHAINS], y[CHAINS], z[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = threadIdx.x + c;
        y[c] = in[(threadIdx.x + c) & 255];
        z[c] = in[(threadIdx.x * 5 + c) & 255];
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < UNROLL / 2; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = __dadd_rn(__dmul_rn(x[c], y[c]), z[c]);
    double r = 0;
    for (int c = 0; c < CHAINS; ++c) r += x[c];
    if (r == 1234.5) out[0] = (float)r;
}

template <typename F>
double time_kernel(F launch, double ops) {
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
    return ops / (best * 1e-3);
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    float *out, *in;
    cudaMalloc(&out, 4);
    cudaMalloc(&in, 256 * 4);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.999f + i * 1e-6f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    const double lanes = double(blocks) * threads * iters;
    const double per_clk_sm = 1.0 / (sms * clk_khz * 1e3);
    struct R { const char* name; double v; } res[7];
    res[0] = {"ffma_reg_const_const", time_kernel([&] { k_ffma_rcc<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f); }, lanes * UNROLL * CHAINS)};
    res[1] = {"ffma_reg_reg_reg", time_kernel([&] { k_ffma_rrr<<<blocks, threads>>>(out, in, iters); }, lanes * UNROLL * CHAINS)};
    res[2] = {"fmul_reg_reg", time_kernel([&] { k_fmul_rr<<<blocks, threads>>>(out, in, iters); }, lanes * UNROLL * CHAINS)};
    res[3] = {"fmnmx_abs", time_kernel([&] { k_fmnmx<<<blocks, threads>>>(out, in, iters); }, lanes * UNROLL * CHAINS)};
    res[4] = {"mix_3ffma_1fmnmx", time_kernel([&] { k_mix<<<blocks, threads>>>(out, in, iters); }, lanes * UNROLL * CHAINS)};
    res[5] = {"dfma_reg", time_kernel([&] { k_dfma<<<blocks, threads>>>(out, in, iters / 8); }, lanes / 8 * UNROLL * CHAINS)};
    res[6] = {"dmul_dadd_ops", time_kernel([&] { k_dmul_dadd<<<blocks, threads>>>(out, in, iters / 8); }, lanes / 8 * UNROLL * CHAINS)};
    printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f", sms, clk_khz / 1e3);
    for (auto& r : res) printf(", \"%s_Tops\": %.3f, \"%s_per_sm_clk_at_attr\": %.1f", r.name, r.v / 1e12, r.name, r.v * per_clk_sm);
    printf("}\n");
    return cudaGetLastError() != cudaSuccess;
}
