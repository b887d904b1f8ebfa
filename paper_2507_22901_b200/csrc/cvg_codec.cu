// cvg_codec.cu -- the codec's image passes on the device (sm_100a).
//
// Reference: src/codec.cpp.  embed_blocks (:65-99) paints each block's
// selected pair over the base image; decode_blocks (:108-165) reduces each
// block to per-channel means.  Both are byte passes over RGB8 rasters, so
// they are bound by HBM bandwidth, not arithmetic: the kernels move 4-byte
// words with every warp access coalesced, keep per-byte work to a few
// integer instructions, and size their grids in multiples of the SM count.
//
// Layout lookup.  The host turns the block list into a per-row span table
// (CSR over rows: for row y, the x0 of every block crossing it, sorted, and
// the block index).  Blocks have one size and do not overlap, so the spans
// of a row are disjoint and sorted by both ends: a pixel's block is found by
// a binary search over its row, and rows without blocks (most of an image)
// cost one comparison per 4 pixels.
#include <cuda_runtime.h>

#include <cstdint>

#include "cvg_internal.h"

namespace cvg {
namespace {

struct SpanTable {
    const int32_t* row_ptr;  // [H + 1]
    const int32_t* x0;       // [n_spans] sorted per row
    const int32_t* blk;      // [n_spans]
    int32_t bw;
};

// First span of [s, e) whose right end lies past x (spans sorted by x0 and
// disjoint, so their right ends are sorted too).
__device__ __forceinline__ int first_span_after(const SpanTable& t, int s, int e, int x) {
    while (s < e) {
        const int mid = (s + e) >> 1;
        if (__ldg(&t.x0[mid]) + t.bw <= x) {
            s = mid + 1;
        } else {
            e = mid;
        }
    }
    return s;
}

__device__ __forceinline__ uint32_t put_byte(uint32_t w, int byte, uint32_t v) {
    const int sh = 8 * byte;
    return (w & ~(0xffu << sh)) | (v << sh);
}

// 4 pixels (12 bytes = 3 words) per thread; needs width % 4 == 0 so every
// group starts on a word boundary inside one row.
__global__ void __launch_bounds__(256) paint4_kernel(const uint32_t* __restrict__ base, uint32_t* __restrict__ fa,
                                                     uint32_t* __restrict__ fb, int width, int height, SpanTable t,
                                                     const uint8_t* __restrict__ plus,
                                                     const uint8_t* __restrict__ minus) {
    const int gpr = width >> 2;
    const long long total = static_cast<long long>(gpr) * height;
    for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
         g += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint32_t w0 = __ldcs(base + 3 * g), w1 = __ldcs(base + 3 * g + 1), w2 = __ldcs(base + 3 * g + 2);
        const int y = static_cast<int>(g / gpr);
        const int x = static_cast<int>(g - static_cast<long long>(y) * gpr) << 2;
        const int s = __ldg(&t.row_ptr[y]), e = __ldg(&t.row_ptr[y + 1]);
        uint32_t a[3] = {w0, w1, w2}, b[3] = {w0, w1, w2};
        if (s != e) {
            int j = first_span_after(t, s, e, x);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                while (j < e && __ldg(&t.x0[j]) + t.bw <= x + p) ++j;
                if (j < e && __ldg(&t.x0[j]) <= x + p) {
                    const int k = __ldg(&t.blk[j]);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int byte = 3 * p + c;  // compile-time after unrolling
                        a[byte >> 2] = put_byte(a[byte >> 2], byte & 3, __ldg(&plus[3 * k + c]));
                        b[byte >> 2] = put_byte(b[byte >> 2], byte & 3, __ldg(&minus[3 * k + c]));
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            __stcs(fa + 3 * g + q, a[q]);
            __stcs(fb + 3 * g + q, b[q]);
        }
    }
}

// Any width: one pixel per thread.
__global__ void __launch_bounds__(256) paint1_kernel(const uint8_t* __restrict__ base, uint8_t* __restrict__ fa,
                                                     uint8_t* __restrict__ fb, int width, int height, SpanTable t,
                                                     const uint8_t* __restrict__ plus,
                                                     const uint8_t* __restrict__ minus) {
    const long long total = static_cast<long long>(width) * height;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(i / width);
        const int x = static_cast<int>(i - static_cast<long long>(y) * width);
        const int s = __ldg(&t.row_ptr[y]), e = __ldg(&t.row_ptr[y + 1]);
        int k = -1;
        if (s != e) {
            const int j = first_span_after(t, s, e, x);
            if (j < e && __ldg(&t.x0[j]) <= x) k = __ldg(&t.blk[j]);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint8_t v = base[3 * i + c];
            fa[3 * i + c] = k < 0 ? v : plus[3 * k + c];
            fb[3 * i + c] = k < 0 ? v : minus[3 * k + c];
        }
    }
}

// Block sums.  One CTA of 192 threads (a multiple of 3) per (block, row
// slice).  A row segment of a block is split into an unaligned head and
// tail (<= 3 bytes each, done bytewise) and a word-aligned middle.  Byte 0
// of word w belongs to channel (4w) % 3 = w % 3, and a thread strides by
// 192 words, so each thread sees one fixed byte->channel phase: it adds the
// words' even and odd bytes into two packed 16-bit-lane accumulators (two
// instructions per word and frame) and unpacks them into channels per row.
constexpr int kSumThreads = 192;

__device__ __forceinline__ void unpack_add(uint32_t even, uint32_t odd, int phase, unsigned long long* ch) {
    // bytes 0..3 of the words -> channels (phase + k) % 3
    const uint32_t s[4] = {even & 0xffffu, odd & 0xffffu, even >> 16, odd >> 16};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int c = (phase + k) % 3;
        ch[0] += c == 0 ? s[k] : 0u;
        ch[1] += c == 1 ? s[k] : 0u;
        ch[2] += c == 2 ? s[k] : 0u;
    }
}

__global__ void __launch_bounds__(kSumThreads) block_sums_kernel(const uint8_t* __restrict__ fa,
                                                                 const uint8_t* __restrict__ fb, int width,
                                                                 int block_w, int block_h,
                                                                 const int32_t* __restrict__ xy,
                                                                 unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long red[6];
    if (threadIdx.x < 6) red[threadIdx.x] = 0;
    __syncthreads();
    const int blk = blockIdx.x;
    const int bx = __ldg(&xy[2 * blk]), by = __ldg(&xy[2 * blk + 1]);
    unsigned long long ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    const uint32_t* wa = reinterpret_cast<const uint32_t*>(fa);
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(fb);
    for (int r = blockIdx.y; r < block_h; r += gridDim.y) {
        const long long s = 3 * (static_cast<long long>(by + r) * width + bx);  // segment [s, e)
        const long long e = s + 3ll * block_w;
        const long long ws = (s + 3) >> 2, we = e >> 2;  // whole words inside the segment
        if (ws < we) {
            const int phase = static_cast<int>((ws + threadIdx.x) % 3);
            uint32_t ea = 0, oa = 0, eb = 0, ob = 0;
            int n = 0;
            for (long long w = ws + threadIdx.x; w < we; w += kSumThreads) {
                const uint32_t va = __ldcs(wa + w), vb = __ldcs(wb + w);
                ea += va & 0x00ff00ffu;
                oa += (va >> 8) & 0x00ff00ffu;
                eb += vb & 0x00ff00ffu;
                ob += (vb >> 8) & 0x00ff00ffu;
                if (++n == 256) {  // 16-bit lanes hold 257 bytes of 255
                    unpack_add(ea, oa, phase, ca);
                    unpack_add(eb, ob, phase, cb);
                    ea = oa = eb = ob = 0;
                    n = 0;
                }
            }
            unpack_add(ea, oa, phase, ca);
            unpack_add(eb, ob, phase, cb);
        }
        // head bytes [s, 4*ws) and tail bytes [4*we, e) (all bytes when the
        // segment holds no whole word)
        const long long h_end = ws < we ? 4 * ws : e;
        const long long t_beg = ws < we ? 4 * we : e;
        const int n_head = static_cast<int>(h_end - s), n_tail = static_cast<int>(e - t_beg);
        const int tid = threadIdx.x;
        if (tid < n_head + n_tail) {
            const long long i = tid < n_head ? s + tid : t_beg + (tid - n_head);
            const int c = static_cast<int>(i % 3);
            const unsigned long long va = fa[i], vb = fb[i];
            ca[0] += c == 0 ? va : 0ull;
            ca[1] += c == 1 ? va : 0ull;
            ca[2] += c == 2 ? va : 0ull;
            cb[0] += c == 0 ? vb : 0ull;
            cb[1] += c == 1 ? vb : 0ull;
            cb[2] += c == 2 ? vb : 0ull;
        }
    }
    // CTA reduction: warp shuffles, then one shared atomic per warp and channel
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        for (int o = 16; o; o >>= 1) {
            ca[c] += __shfl_xor_sync(0xffffffffu, ca[c], o);
            cb[c] += __shfl_xor_sync(0xffffffffu, cb[c], o);
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            atomicAdd(&red[c], ca[c]);
            atomicAdd(&red[3 + c], cb[c]);
        }
    }
    __syncthreads();
    if (threadIdx.x < 6 && red[threadIdx.x]) atomicAdd(&sums[6 * blk + threadIdx.x], red[threadIdx.x]);
}

int grid_for(long long items, int threads, int sms) {
    const long long want = (items + threads - 1) / threads;
    const long long cap = static_cast<long long>(sms) * 16;  // 16 x 256 threads per SM: full occupancy
    return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_paint(const uint8_t* base, uint8_t* fa, uint8_t* fb, int width, int height,
                         const int32_t* row_ptr, const int32_t* x0, const int32_t* blk, int block_w,
                         const uint8_t* plus, const uint8_t* minus, int sms, cudaStream_t st) {
    const SpanTable t{row_ptr, x0, blk, block_w};
    const bool words = width % 4 == 0 && (reinterpret_cast<uintptr_t>(base) & 3) == 0 &&
                       (reinterpret_cast<uintptr_t>(fa) & 3) == 0 && (reinterpret_cast<uintptr_t>(fb) & 3) == 0;
    if (words) {
        const long long groups = static_cast<long long>(width / 4) * height;
        paint4_kernel<<<grid_for(groups, 256, sms), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(base),
                                                                 reinterpret_cast<uint32_t*>(fa),
                                                                 reinterpret_cast<uint32_t*>(fb), width, height, t,
                                                                 plus, minus);
    } else {
        const long long px = static_cast<long long>(width) * height;
        paint1_kernel<<<grid_for(px, 256, sms), 256, 0, st>>>(base, fa, fb, width, height, t, plus, minus);
    }
    return cudaGetLastError();
}

cudaError_t launch_block_sums(const uint8_t* fa, const uint8_t* fb, int width, int block_w, int block_h,
                              int n_blocks, const int32_t* xy, unsigned long long* sums, int sms, cudaStream_t st) {
    if (n_blocks <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * 6 * static_cast<size_t>(n_blocks), st);
    if (e != cudaSuccess) return e;
    // enough CTAs for ~8 per SM in total, row slices of each block
    const long long want = (static_cast<long long>(sms) * 8 + n_blocks - 1) / n_blocks;
    int slices = static_cast<int>(want < block_h ? (want > 0 ? want : 1) : block_h);
    if (slices > 65535) slices = 65535;
    if ((reinterpret_cast<uintptr_t>(fa) & 3) || (reinterpret_cast<uintptr_t>(fb) & 3)) return cudaErrorMisalignedAddress;
    block_sums_kernel<<<dim3(n_blocks, slices), kSumThreads, 0, st>>>(fa, fb, width, block_w, block_h, xy, sums);
    return cudaGetLastError();
}

}  // namespace cvg
