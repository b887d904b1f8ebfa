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

// Painting.  One CTA per image row (grid-stride over rows), so rows without
// blocks -- most of a carrier -- are a plain 16-byte copy per thread with
// fully coalesced loads and stores, no per-pixel work.  In a row with
// blocks, each 16-byte chunk covers pixels px0..px0+5 (3 bytes each); its
// byte k belongs to pixel (phase + k) / 3 and channel (phase + k) % 3 with
// phase = chunk % 3 (16 = 1 mod 3), so the merge is unrolled per phase with
// compile-time byte positions.  Block colors come packed as r | g << 8 |
// b << 16 words.  Needs 3 * width % 16 == 0 (rows start on 16 bytes).
__device__ __forceinline__ uint32_t put_byte(uint32_t w, int byte, uint32_t v) {
    const int sh = 8 * byte;
    return (w & ~(0xffu << sh)) | ((v & 0xffu) << sh);
}

template <int kPhase>
__device__ __forceinline__ void merge_chunk(uint32_t (&a)[4], uint32_t (&b)[4], const int (&blk)[6],
                                            const uint32_t (&pc)[6], const uint32_t (&mc)[6]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int q = (kPhase + k) / 3, ch = (kPhase + k) % 3;
        if (blk[q] >= 0) {
            a[k >> 2] = put_byte(a[k >> 2], k & 3, pc[q] >> (8 * ch));
            b[k >> 2] = put_byte(b[k >> 2], k & 3, mc[q] >> (8 * ch));
        }
    }
}

__global__ void __launch_bounds__(256) paint16_kernel(const uint4* __restrict__ base, uint4* __restrict__ fa,
                                                      uint4* __restrict__ fb, int width, int height, SpanTable t,
                                                      const uint32_t* __restrict__ plus,
                                                      const uint32_t* __restrict__ minus) {
    const int cpr = (3 * width) >> 4;  // 16-byte chunks per row
    for (int y = blockIdx.x; y < height; y += gridDim.x) {
        const int s = __ldg(&t.row_ptr[y]), e = __ldg(&t.row_ptr[y + 1]);
        const size_t row0 = static_cast<size_t>(y) * cpr;
        if (s == e) {
            for (int c = threadIdx.x; c < cpr; c += blockDim.x) {
                const uint4 v = __ldcs(base + row0 + c);
                __stcs(fa + row0 + c, v);
                __stcs(fb + row0 + c, v);
            }
            continue;
        }
        int j = -1;  // span cursor: this thread's chunks come in increasing x
        for (int c = threadIdx.x; c < cpr; c += blockDim.x) {
            const uint4 v = __ldcs(base + row0 + c);
            const int px0 = (c << 4) / 3, px1 = ((c << 4) + 15) / 3;
            if (j < 0) {
                j = first_span_after(t, s, e, px0);
            } else {
                while (j < e && __ldg(&t.x0[j]) + t.bw <= px0) ++j;
            }
            if (j >= e || __ldg(&t.x0[j]) > px1) {  // no block touches this chunk
                __stcs(fa + row0 + c, v);
                __stcs(fb + row0 + c, v);
                continue;
            }
            int blk[6];
            uint32_t pc[6], mc[6];
            int jj = j;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const int px = px0 + q;
                while (jj < e && __ldg(&t.x0[jj]) + t.bw <= px) ++jj;
                const bool in = px <= px1 && jj < e && __ldg(&t.x0[jj]) <= px;
                blk[q] = in ? __ldg(&t.blk[jj]) : -1;
                pc[q] = in ? __ldg(&plus[blk[q]]) : 0u;
                mc[q] = in ? __ldg(&minus[blk[q]]) : 0u;
            }
            uint32_t a[4] = {v.x, v.y, v.z, v.w}, b[4] = {v.x, v.y, v.z, v.w};
            const int phase = c % 3;
            if (phase == 0) {
                merge_chunk<0>(a, b, blk, pc, mc);
            } else if (phase == 1) {
                merge_chunk<1>(a, b, blk, pc, mc);
            } else {
                merge_chunk<2>(a, b, blk, pc, mc);
            }
            __stcs(fa + row0 + c, make_uint4(a[0], a[1], a[2], a[3]));
            __stcs(fb + row0 + c, make_uint4(b[0], b[1], b[2], b[3]));
        }
    }
}

// Any width: one CTA per row, one pixel per thread.
__global__ void __launch_bounds__(256) paint1_kernel(const uint8_t* __restrict__ base, uint8_t* __restrict__ fa,
                                                     uint8_t* __restrict__ fb, int width, int height, SpanTable t,
                                                     const uint32_t* __restrict__ plus,
                                                     const uint32_t* __restrict__ minus) {
    for (int y = blockIdx.x; y < height; y += gridDim.x) {
        const int s = __ldg(&t.row_ptr[y]), e = __ldg(&t.row_ptr[y + 1]);
        const size_t row0 = 3 * static_cast<size_t>(y) * width;
        int j = -1;
        for (int x = threadIdx.x; x < width; x += blockDim.x) {
            int k = -1;
            if (s != e) {
                if (j < 0) {
                    j = first_span_after(t, s, e, x);
                } else {
                    while (j < e && __ldg(&t.x0[j]) + t.bw <= x) ++j;
                }
                if (j < e && __ldg(&t.x0[j]) <= x) k = __ldg(&t.blk[j]);
            }
            const size_t i = row0 + 3 * static_cast<size_t>(x);
            const uint32_t pw = k < 0 ? 0u : __ldg(&plus[k]), mw = k < 0 ? 0u : __ldg(&minus[k]);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint8_t v = base[i + c];
                fa[i + c] = k < 0 ? v : static_cast<uint8_t>(pw >> (8 * c));
                fb[i + c] = k < 0 ? v : static_cast<uint8_t>(mw >> (8 * c));
            }
        }
    }
}

// Block sums.  CTAs of 8 warps per (block, row slice); a warp sums one row
// segment of the block at a time, lanes over its 4-byte words (byte 0 of
// word w is channel w % 3, since 4 = 1 mod 3) plus the unaligned head and
// tail bytes, in exact integers; then warp shuffles, one shared atomic per
// warp and channel, and one global atomic per CTA and channel.
constexpr int kSumThreads = 256;

__device__ __forceinline__ void add_word(uint32_t v, int phase, unsigned long long (&ch)[3]) {
    const uint32_t x0 = (v & 0xffu) + (v >> 24), x1 = (v >> 8) & 0xffu, x2 = (v >> 16) & 0xffu;
    ch[0] += phase == 0 ? x0 : (phase == 1 ? x2 : x1);
    ch[1] += phase == 0 ? x1 : (phase == 1 ? x0 : x2);
    ch[2] += phase == 0 ? x2 : (phase == 1 ? x1 : x0);
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
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    const uint32_t* wa = reinterpret_cast<const uint32_t*>(fa);
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(fb);
    for (int r = blockIdx.y * (kSumThreads / 32) + warp; r < block_h; r += gridDim.y * (kSumThreads / 32)) {
        const long long s = 3 * (static_cast<long long>(by + r) * width + bx);  // segment [s, e)
        const long long e = s + 3ll * block_w;
        long long ws = (s + 3) >> 2, we = e >> 2;  // whole words inside the segment
        if (ws > we) ws = we;
        for (long long w = ws + lane; w < we; w += 32) {
            const int phase = static_cast<int>(w % 3);
            add_word(__ldcs(wa + w), phase, ca);
            add_word(__ldcs(wb + w), phase, cb);
        }
        // head [s, 4 ws) and tail [4 we, e) bytes (the whole segment when it
        // holds no whole word)
        const long long h_end = ws < we ? 4 * ws : e;
        const long long t_beg = ws < we ? 4 * we : e;
        const int n_head = static_cast<int>(h_end - s), n_tail = static_cast<int>(e - t_beg);
        for (int k = lane; k < n_head + n_tail; k += 32) {
            const long long i = k < n_head ? s + k : t_beg + (k - n_head);
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
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        for (int o = 16; o; o >>= 1) {
            ca[c] += __shfl_xor_sync(0xffffffffu, ca[c], o);
            cb[c] += __shfl_xor_sync(0xffffffffu, cb[c], o);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (ca[c]) atomicAdd(&red[c], ca[c]);
            if (cb[c]) atomicAdd(&red[3 + c], cb[c]);
        }
    }
    __syncthreads();
    if (threadIdx.x < 6 && red[threadIdx.x]) atomicAdd(&sums[6 * blk + threadIdx.x], red[threadIdx.x]);
}

}  // namespace

cudaError_t launch_paint(const uint8_t* base, uint8_t* fa, uint8_t* fb, int width, int height,
                         const int32_t* row_ptr, const int32_t* x0, const int32_t* blk, int block_w,
                         const uint32_t* plus, const uint32_t* minus, int sms, cudaStream_t st) {
    const SpanTable t{row_ptr, x0, blk, block_w};
    const int grid = height < sms * 8 ? height : sms * 8;  // 8 x 256 threads per SM, rows grid-strided
    const bool vec = (3 * width) % 16 == 0 && ((reinterpret_cast<uintptr_t>(base) | reinterpret_cast<uintptr_t>(fa) |
                                                reinterpret_cast<uintptr_t>(fb)) & 15) == 0;
    if (vec) {
        paint16_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(base), reinterpret_cast<uint4*>(fa),
                                             reinterpret_cast<uint4*>(fb), width, height, t, plus, minus);
    } else {
        paint1_kernel<<<grid, 256, 0, st>>>(base, fa, fb, width, height, t, plus, minus);
    }
    return cudaGetLastError();
}

cudaError_t launch_block_sums(const uint8_t* fa, const uint8_t* fb, int width, int block_w, int block_h,
                              int n_blocks, const int32_t* xy, unsigned long long* sums, int sms, cudaStream_t st) {
    if (n_blocks <= 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(fa) | reinterpret_cast<uintptr_t>(fb)) & 3) return cudaErrorMisalignedAddress;
    cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * 6 * static_cast<size_t>(n_blocks), st);
    if (e != cudaSuccess) return e;
    // row slices of 8 rows per CTA, at most what fills ~8 CTAs per SM in total
    const long long rows8 = (block_h + 7) / 8;
    const long long want = (static_cast<long long>(sms) * 8 + n_blocks - 1) / n_blocks;
    long long slices = want < rows8 ? want : rows8;
    if (slices < 1) slices = 1;
    if (slices > 65535) slices = 65535;
    block_sums_kernel<<<dim3(n_blocks, static_cast<unsigned>(slices)), kSumThreads, 0, st>>>(fa, fb, width, block_w,
                                                                                             block_h, xy, sums);
    return cudaGetLastError();
}

}  // namespace cvg
