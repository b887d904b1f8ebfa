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

// Warp tasks: a task is 128 consecutive 16-byte chunks (2 KB) of one row;
// lane l takes chunks l, l+32, l+64, l+96, all four loads issued before any
// store (4 x 16 B in flight per lane).  Row spans are warp-uniform; a lane's
// span cursor only moves forward across its chunks.
constexpr int kTaskChunks = 128;

template <int kPhase>
__device__ __forceinline__ uint4 merge_pixels(uint4 v, int px0, int px1, int& j, int e, const SpanTable& t,
                                              const uint32_t* __restrict__ colors, uint4& other,
                                              const uint32_t* __restrict__ colors2) {
    int blk[6];
    uint32_t pc[6], mc[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int px = px0 + q;
        while (j < e && __ldg(&t.x0[j]) + t.bw <= px) ++j;
        const bool in = px <= px1 && j < e && __ldg(&t.x0[j]) <= px;
        blk[q] = in ? __ldg(&t.blk[j]) : -1;
        pc[q] = in ? __ldg(&colors[blk[q]]) : 0u;
        mc[q] = in ? __ldg(&colors2[blk[q]]) : 0u;
    }
    uint32_t a[4] = {v.x, v.y, v.z, v.w}, b[4] = {v.x, v.y, v.z, v.w};
    merge_chunk<kPhase>(a, b, blk, pc, mc);
    other = make_uint4(b[0], b[1], b[2], b[3]);
    return make_uint4(a[0], a[1], a[2], a[3]);
}

__global__ void __launch_bounds__(256) paint16_kernel(const uint4* __restrict__ base, uint4* __restrict__ fa,
                                                      uint4* __restrict__ fb, int width, int height, SpanTable t,
                                                      const uint32_t* __restrict__ plus,
                                                      const uint32_t* __restrict__ minus) {
    const int cpr = (3 * width) >> 4;  // 16-byte chunks per row
    const int tpr = (cpr + kTaskChunks - 1) / kTaskChunks;
    const long long tasks = static_cast<long long>(tpr) * height;
    const int lane = threadIdx.x & 31;
    const long long nwarps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long task = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; task < tasks;
         task += nwarps) {
        const int y = static_cast<int>(task / tpr);
        const int c0 = static_cast<int>(task - static_cast<long long>(y) * tpr) * kTaskChunks + lane;
        const size_t row0 = static_cast<size_t>(y) * cpr;
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u;
            if (c < cpr) v[u] = __ldcs(base + row0 + c);
        }
        const int s = __ldg(&t.row_ptr[y]), e = __ldg(&t.row_ptr[y + 1]);
        if (s == e) {  // no block crosses this row: a copy
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + 32 * u;
                if (c < cpr) {
                    __stcs(fa + row0 + c, v[u]);
                    __stcs(fb + row0 + c, v[u]);
                }
            }
            continue;
        }
        int j = c0 < cpr ? first_span_after(t, s, e, (c0 << 4) / 3) : e;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u;
            if (c >= cpr) break;
            const int px0 = (c << 4) / 3, px1 = ((c << 4) + 15) / 3;
            while (j < e && __ldg(&t.x0[j]) + t.bw <= px0) ++j;
            uint4 ra = v[u], rb = v[u];
            if (j < e && __ldg(&t.x0[j]) <= px1) {  // a block touches this chunk
                int jj = j;
                const int phase = c % 3;
                if (phase == 0) {
                    ra = merge_pixels<0>(v[u], px0, px1, jj, e, t, plus, rb, minus);
                } else if (phase == 1) {
                    ra = merge_pixels<1>(v[u], px0, px1, jj, e, t, plus, rb, minus);
                } else {
                    ra = merge_pixels<2>(v[u], px0, px1, jj, e, t, plus, rb, minus);
                }
            }
            __stcs(fa + row0 + c, ra);
            __stcs(fb + row0 + c, rb);
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

// Block sums.  A CTA takes one block (or a slice of its rows) and flattens
// it into (row, 16-byte chunk) items, so every thread issues independent
// 16-byte loads however narrow the block is.  Byte i of the chunk starting
// at byte offset 16c belongs to channel (c + i) % 3 (16 = 1 mod 3): bytes are
// summed into three chunk-relative accumulators with compile-time indices and
// rotated into r, g, b once per chunk.  Chunks that straddle the block's row
// segment [s, e) mask their bytes; a chunk running past the end of the image
// is read bytewise.  Sums are exact integers.
constexpr int kSumThreads = 256;

__device__ __forceinline__ void rotate_add(const uint32_t (&rel)[3], int phase, unsigned long long (&ch)[3]) {
    ch[0] += phase == 0 ? rel[0] : (phase == 1 ? rel[2] : rel[1]);
    ch[1] += phase == 0 ? rel[1] : (phase == 1 ? rel[0] : rel[2]);
    ch[2] += phase == 0 ? rel[2] : (phase == 1 ? rel[1] : rel[0]);
}

__device__ __forceinline__ void sum_chunk(uint4 v, long long o, long long s, long long e, bool full,
                                          uint32_t (&rel)[3]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    rel[0] = rel[1] = rel[2] = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        uint32_t byte = (w[i >> 2] >> (8 * (i & 3))) & 0xffu;
        if (!full) byte = (o + i >= s && o + i < e) ? byte : 0u;
        rel[i % 3] += byte;
    }
}

__global__ void __launch_bounds__(kSumThreads) block_sums_kernel(const uint8_t* __restrict__ fa,
                                                                 const uint8_t* __restrict__ fb, int width,
                                                                 int block_w, int block_h, long long total_bytes,
                                                                 const int32_t* __restrict__ xy,
                                                                 unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long red[6];
    if (threadIdx.x < 6) red[threadIdx.x] = 0;
    __syncthreads();
    const int blk = blockIdx.x;
    const int bx = __ldg(&xy[2 * blk]), by = __ldg(&xy[2 * blk + 1]);
    const int cpr = (3 * block_w + 15) / 16 + 1;  // chunks a row segment can touch
    const int r0 = static_cast<int>((static_cast<long long>(block_h) * blockIdx.y) / gridDim.y);
    const int r1 = static_cast<int>((static_cast<long long>(block_h) * (blockIdx.y + 1)) / gridDim.y);
    const long long items = static_cast<long long>(r1 - r0) * cpr;
    unsigned long long ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    const uint4* va4 = reinterpret_cast<const uint4*>(fa);
    const uint4* vb4 = reinterpret_cast<const uint4*>(fb);
    for (long long it = threadIdx.x; it < items; it += kSumThreads) {
        const int r = r0 + static_cast<int>(it / cpr);
        const int k = static_cast<int>(it - static_cast<long long>(r - r0) * cpr);
        const long long s = 3 * (static_cast<long long>(by + r) * width + bx);
        const long long e = s + 3ll * block_w;
        const long long c = (s >> 4) + k;
        const long long o = c << 4;
        if (o >= e) continue;
        const int phase = static_cast<int>(c % 3);
        uint32_t rel[3];
        if (o + 16 <= total_bytes) {
            const bool full = o >= s && o + 16 <= e;
            sum_chunk(__ldcs(va4 + c), o, s, e, full, rel);
            rotate_add(rel, phase, ca);
            sum_chunk(__ldcs(vb4 + c), o, s, e, full, rel);
            rotate_add(rel, phase, cb);
        } else {  // the image's last partial chunk
            for (long long i = (o > s ? o : s); i < e; ++i) {
                const int ch = static_cast<int>(i % 3);
                const unsigned long long x = fa[i], y = fb[i];
                ca[0] += ch == 0 ? x : 0ull;
                ca[1] += ch == 1 ? x : 0ull;
                ca[2] += ch == 2 ? x : 0ull;
                cb[0] += ch == 0 ? y : 0ull;
                cb[1] += ch == 1 ? y : 0ull;
                cb[2] += ch == 2 ? y : 0ull;
            }
        }
    }
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
    const int grid = height < sms * 8 ? height : sms * 8;  // 8 x 256 threads per SM
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

cudaError_t launch_block_sums(const uint8_t* fa, const uint8_t* fb, int width, int height, int block_w, int block_h,
                              int n_blocks, const int32_t* xy, unsigned long long* sums, int sms, cudaStream_t st) {
    const long long total_bytes = 3ll * width * height;
    if (n_blocks <= 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(fa) | reinterpret_cast<uintptr_t>(fb)) & 15) return cudaErrorMisalignedAddress;
    cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * 6 * static_cast<size_t>(n_blocks), st);
    if (e != cudaSuccess) return e;
    // row slices so that ~8 CTAs per SM are in flight in total
    const long long want = (static_cast<long long>(sms) * 8 + n_blocks - 1) / n_blocks;
    long long slices = want < block_h ? want : block_h;
    if (slices < 1) slices = 1;
    if (slices > 65535) slices = 65535;
    block_sums_kernel<<<dim3(n_blocks, static_cast<unsigned>(slices)), kSumThreads, 0, st>>>(
        fa, fb, width, block_w, block_h, total_bytes, xy, sums);
    return cudaGetLastError();
}

}  // namespace cvg
