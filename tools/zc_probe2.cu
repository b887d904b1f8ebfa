// Can a few SMs stream HBM -> mapped host memory at PCIe rate, and does that
// slow a compute kernel running on the other SMs?  (streamed-search design probe)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/zc_probe2.cu -o zc_probe2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stream_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

__global__ void busy(float* out, int iters, unsigned* tickets, unsigned n_items) {
    // claims items from a ticket like phase 1 (atomics + FFMA work)
    __shared__ unsigned item;
    float x = threadIdx.x;
    while (true) {
        if (threadIdx.x == 0) item = atomicAdd(tickets, 1u);
        __syncthreads();
        if (item >= n_items) break;
        for (int i = 0; i < iters; ++i) x = fmaf(x, 0.999f, 0.001f);
        __syncthreads();
    }
    if (x == 1234.5f) out[0] = x;
}

int main() {
    const size_t bytes = 38ull << 20;
    void *h = nullptr, *d = nullptr;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    void* hd = nullptr;
    cudaHostGetDevicePointer(&hd, h, 0);
    float* out;
    cudaMalloc(&out, 4);
    unsigned* tk;
    cudaMalloc(&tk, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a0, a1, b0, b1;
    cudaEventCreate(&a0); cudaEventCreate(&a1); cudaEventCreate(&b0); cudaEventCreate(&b1);
    const int big_smem = 200 * 1024;
    cudaFuncSetAttribute(stream_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    const unsigned items = 40000;
    auto run_busy = [&](cudaStream_t s) {
        cudaMemsetAsync(tk, 0, 4, s);
        busy<<<4 * sms, 256, 0, s>>>(out, 2000, tk, items);
    };
    // busy alone
    for (int r = 0; r < 2; ++r) { cudaEventRecord(a0, s1); run_busy(s1); cudaEventRecord(a1, s1); cudaDeviceSynchronize(); }
    float ms_busy;
    cudaEventElapsedTime(&ms_busy, a0, a1);
    printf("busy alone: %.3f ms\n", ms_busy);
    for (int R : {2, 4, 8, 16, 32, 148}) {
        for (int threads : {512, 1024}) {
            // copy alone
            cudaEventRecord(b0, s2);
            stream_copy<<<R, threads, big_smem, s2>>>(static_cast<uint4*>(d), static_cast<uint4*>(hd), bytes / 16);
            cudaEventRecord(b1, s2);
            cudaDeviceSynchronize();
            float ms_c;
            cudaEventElapsedTime(&ms_c, b0, b1);
            // concurrent: copy first (occupies R SMs), then busy
            cudaEventRecord(b0, s2);
            stream_copy<<<R, threads, big_smem, s2>>>(static_cast<uint4*>(d), static_cast<uint4*>(hd), bytes / 16);
            cudaEventRecord(b1, s2);
            cudaEventRecord(a0, s1);
            run_busy(s1);
            cudaEventRecord(a1, s1);
            cudaDeviceSynchronize();
            float ms_cc, ms_bc;
            cudaEventElapsedTime(&ms_cc, b0, b1);
            cudaEventElapsedTime(&ms_bc, a0, a1);
            printf("R=%3d thr=%4d copy alone %.3f ms (%.1f GB/s) | concurrent: copy %.3f ms (%.1f GB/s) busy %.3f ms\n", R,
                   threads, ms_c, bytes / ms_c / 1e6, ms_cc, bytes / ms_cc / 1e6, ms_bc);
        }
    }
    // DMA copy concurrent with busy
    cudaEventRecord(b0, s2);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b1, s2);
    cudaEventRecord(a0, s1);
    run_busy(s1);
    cudaEventRecord(a1, s1);
    cudaDeviceSynchronize();
    float ms_cc, ms_bc;
    cudaEventElapsedTime(&ms_cc, b0, b1);
    cudaEventElapsedTime(&ms_bc, a0, a1);
    printf("DMA concurrent: copy %.3f ms (%.1f GB/s) busy %.3f ms\n", ms_cc, bytes / ms_cc / 1e6, ms_bc);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
