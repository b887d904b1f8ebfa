// Zero-copy write probe: SM stores into mapped pinned host memory vs a
// cudaMemcpy D2H of the same bytes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/zc_probe.cu -o zc_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename T>
__global__ void write_kernel(T* __restrict__ dst, size_t n, T v) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) dst[i] = v;
}

// per warp: 32 x 6 bytes staged as 96 u16 (3 contiguous 64-byte stores), like a packed code record
__global__ void write_codes6(uint16_t* __restrict__ dst, size_t n_rec) {
    const unsigned lane = threadIdx.x & 31;
    const size_t warps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    for (size_t w = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5; w * 32 < n_rec; w += warps) {
        uint16_t* p = dst + w * 96;
        p[lane] = static_cast<uint16_t>(lane);
        p[32 + lane] = static_cast<uint16_t>(lane);
        p[64 + lane] = static_cast<uint16_t>(lane);
    }
}

int main() {
    const size_t bytes = 38ull << 20;
    void* h = nullptr;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    void* hd = nullptr;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto time_it = [&](const char* what, auto fn) {
        fn();
        cudaDeviceSynchronize();
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-44s %8.3f ms  %6.1f GB/s\n", what, best, bytes / (best * 1e-3) / 1e9);
    };
    time_it("cudaMemcpyAsync D2H", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); });
    for (int blocks_per_sm : {1, 4}) {
        for (int threads : {128, 256}) {
            char name[96];
            snprintf(name, sizeof(name), "zero-copy u32  grid %dx%d thr %d", blocks_per_sm, sms, threads);
            time_it(name, [&] {
                write_kernel<uint32_t><<<blocks_per_sm * sms, threads>>>(static_cast<uint32_t*>(hd), bytes / 4, 7u);
            });
            snprintf(name, sizeof(name), "zero-copy uint4 grid %dx%d thr %d", blocks_per_sm, sms, threads);
            time_it(name, [&] {
                write_kernel<uint4><<<blocks_per_sm * sms, threads>>>(static_cast<uint4*>(hd), bytes / 16,
                                                                       make_uint4(1, 2, 3, 4));
            });
            snprintf(name, sizeof(name), "zero-copy u16  grid %dx%d thr %d", blocks_per_sm, sms, threads);
            time_it(name, [&] {
                write_kernel<uint16_t><<<blocks_per_sm * sms, threads>>>(static_cast<uint16_t*>(hd), bytes / 2, 7);
            });
            snprintf(name, sizeof(name), "zero-copy codes6 grid %dx%d thr %d", blocks_per_sm, sms, threads);
            time_it(name, [&] {
                write_codes6<<<blocks_per_sm * sms, threads>>>(static_cast<uint16_t*>(hd), bytes / 6);
            });
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
