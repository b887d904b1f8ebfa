// cvg_codec.cu -- the codec's image passes on the device (sm_100a).
//
// Reference: src/codec.cpp.  embed_blocks (:65-99) paints each block's
// selected pair over the base image; decode_blocks (:108-165) reduces each
// block to per-channel means.  Both are byte passes over RGB8 rasters, so
// they are bound by HBM bandwidth, not arithmetic: the kernels move 16-byte
// chunks with every warp access coalesced, keep per-byte work to a few
// integer instructions, and size their grids in multiples of the SM count.
//
// The host validates the layout (bounds, no overlaps: cvg_codec_host.cpp
// layout_spans) and uploads the block positions and packed colors
// (r | g << 8 | b << 16); the kernels address pixels by byte offset: the
// pixel (x, y) occupies bytes 3 (y W + x) .. +2, so byte offset o is channel
// o % 3 wherever it lies.
#include <cuda_runtime.h>

#include <cstdint>

#include "cvg_internal.h"

namespace cvg {
namespace {

constexpr int kBlockThreads = 256;  // 8 warps; the fill and the block sums run one task per warp

// Programmatic dependent launch: the fill is launched while the copy drains;
// its blocks set up their geometry and wait (griddepcontrol.wait: the copy
// grid complete and its writes visible) before their first store.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Painting, in two passes over device memory:
//  1. copy2_kernel: frame_a = frame_b = base, a flat 16-byte copy (read once,
//     write twice: the 9 B/pixel minimum) with four loads in flight per thread;
//  2. fill_kernel: every block's row segments as coalesced 32-bit stores of
//     the color pattern plus <= 6 unaligned edge bytes per row (below).
// The fused alternative (one pass, a span lookup per chunk) measured slower:
// its per-chunk lookups are dependent loads that stall the copy's stream of
// independent loads.
__global__ void __launch_bounds__(256) copy2_kernel(const uint4* __restrict__ base, uint4* __restrict__ fa,
                                                    uint4* __restrict__ fb, long long n16,
                                                    const uint8_t* __restrict__ base_b, uint8_t* __restrict__ fa_b,
                                                    uint8_t* __restrict__ fb_b, long long n_bytes) {
    pdl_trigger();  // the fill may launch now (it waits for this grid before storing)
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(base + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            fa[i + u * stride] = v[u];  // default policy: the fill pass merges into these lines in L2
            fb[i + u * stride] = v[u];
        }
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldcs(base + i);
        fa[i] = v;
        fb[i] = v;
    }
    // the last n_bytes % 16 bytes
    const long long t = 16 * n16 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n_bytes) {
        fa_b[t] = base_b[t];
        fb_b[t] = base_b[t];
    }
}

__global__ void __launch_bounds__(256) copy2_bytes_kernel(const uint8_t* __restrict__ base, uint8_t* __restrict__ fa,
                                                          uint8_t* __restrict__ fb, long long n_bytes) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_bytes;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        fa[i] = base[i];
        fb[i] = base[i];
    }
}

// The 4-byte word of a color's repeating r,g,b pattern whose first byte is
// channel `phase` (word w of the raster starts at channel (4w) % 3 = w % 3).
__device__ __forceinline__ uint32_t color_word(uint32_t rgb, int phase) {
    const uint32_t r = rgb & 0xffu, g = (rgb >> 8) & 0xffu, b = (rgb >> 16) & 0xffu;
    const uint32_t w0 = r | g << 8 | b << 16 | r << 24;  // channels 0,1,2,0
    const uint32_t w1 = g | b << 8 | r << 16 | g << 24;  // 1,2,0,1
    const uint32_t w2 = b | r << 8 | g << 16 | b << 24;  // 2,0,1,2
    return phase == 0 ? w0 : (phase == 1 ? w1 : w2);
}

// A warp takes one block (or a slice of its rows); its lanes form
// groups of G (a power of two, about the words of one row segment), one
// group per row, so narrow blocks still fill whole warps.  A group stores
// the row segment's whole 4-byte words (coalesced 32-bit stores of the
// pattern word of the word's phase) and its <= 3 + 3 unaligned head and tail
// bytes (a segment holding no whole word has <= 6 bytes, all written as head).  Every byte written belongs to this block: neighbouring blocks
// never race.
// kUniform (width % 4 == 0): a row is 3W = 0 mod 12 bytes, so every row of a
// block has the same word alignment and phases; the geometry is set up once
// and a row costs its stores and one address add.
template <bool kUniform>
__global__ void __launch_bounds__(256) fill_kernel(uint8_t* __restrict__ fa, uint8_t* __restrict__ fb, int width,
                                                   int block_w, int block_h, int slices, int rows_per_slice,
                                                   int log2_group, int n_tasks, const int32_t* __restrict__ xy,
                                                   const uint32_t* __restrict__ plus,
                                                   const uint32_t* __restrict__ minus) {
    const int task = static_cast<int>(blockIdx.x) * (kBlockThreads / 32) + static_cast<int>(threadIdx.x >> 5);
    if (task >= n_tasks) {
        pdl_wait();
        return;
    }
    const int blk = task / slices, slice = task - blk * slices;
    const int bx = __ldg(&xy[2 * blk]), by = __ldg(&xy[2 * blk + 1]);
    const uint32_t pc = __ldg(&plus[blk]), mc = __ldg(&minus[blk]);
    const uint32_t pw[3] = {color_word(pc, 0), color_word(pc, 1), color_word(pc, 2)};
    const uint32_t mw[3] = {color_word(mc, 0), color_word(mc, 1), color_word(mc, 2)};
    const int r0 = slice * rows_per_slice;
    const int r1 = min(r0 + rows_per_slice, block_h);
    const int group = 1 << log2_group, lane = threadIdx.x & 31;
    const int g = lane >> log2_group, li = lane & (group - 1), groups = 32 >> log2_group;
    const int gmod3 = group % 3;
    uint32_t* wa = reinterpret_cast<uint32_t*>(fa);
    uint32_t* wb = reinterpret_cast<uint32_t*>(fb);
    // geometry of a row segment (for kUniform: of every row, relative to its start)
    auto geometry = [&](long long s, long long& ws, int& nw, int& ph0, int& nh, long long& t_beg, int& nt) {
        const long long e = s + 3ll * block_w;
        ws = (s + 3) >> 2;
        const long long we = e >> 2;
        if (ws > we) ws = we;  // no whole word (segments of <= 6 bytes): every byte is a head byte
        nw = static_cast<int>(we - ws);
        ph0 = static_cast<int>(ws % 3);
        nh = static_cast<int>((nw > 0 ? 4 * ws : e) - s);
        t_beg = nw > 0 ? 4 * we : e;
        nt = static_cast<int>(e - t_beg);
    };
    long long ws = 0, t_beg = 0;
    int nw = 0, ph0 = 0, nh = 0, nt = 0, tch = 0;
    const long long row_bytes = 3ll * width;
    if (kUniform) {
        const long long s0 = 3 * (static_cast<long long>(by) * width + bx);
        geometry(s0, ws, nw, ph0, nh, t_beg, nt);
        tch = static_cast<int>(t_beg - s0) % 3;
    }
    pdl_wait();  // the copy pass complete: these bytes are ours now
    for (int r = r0 + g; r < r1; r += groups) {
        const long long s = 3 * (static_cast<long long>(by + r) * width + bx);
        long long wrow;
        long long tb;
        if (kUniform) {
            wrow = ws + static_cast<long long>(r) * (row_bytes >> 2);
            tb = t_beg + static_cast<long long>(r) * row_bytes;
        } else {
            geometry(s, wrow, nw, ph0, nh, tb, nt);
            tch = static_cast<int>(tb - s) % 3;
        }
        int ph = (ph0 + li) % 3;
        for (int k = li; k < nw; k += group) {
            wa[wrow + k] = ph == 0 ? pw[0] : (ph == 1 ? pw[1] : pw[2]);
            wb[wrow + k] = ph == 0 ? mw[0] : (ph == 1 ? mw[1] : mw[2]);
            ph += gmod3;
            ph = ph >= 3 ? ph - 3 : ph;
        }
        if (li < 6) {
            long long i = -1;
            int ch = 0;
            if (nw == 0) {  // no whole word: <= 6 bytes (3 + 3 around a word boundary), all "head"
                if (li < nh) {
                    i = s + li;
                    ch = li % 3;
                }
            } else if (li < 3 && li < nh) {
                i = s + li;
                ch = li;  // s starts a pixel
            } else if (li >= 3 && li - 3 < nt) {
                i = tb + (li - 3);
                ch = (tch + li - 3) % 3;
            }
            if (i >= 0) {
                fa[i] = static_cast<uint8_t>(pc >> (8 * ch));
                fb[i] = static_cast<uint8_t>(mc >> (8 * ch));
            }
        }
    }
}

// Block sums.  A warp takes one block (or a slice of its rows); lane groups of
// G (a power of two, about the 16-byte chunks of a row segment) take one row
// each, so every thread issues independent 16-byte loads however narrow the
// block is.  A chunk's bytes are summed per channel with byte dot products
// (dp4a against 0/1 selector words): byte i of the chunk at offset o is
// channel o + i mod 3, and the selectors also drop bytes outside the row
// segment.  kUniform (width % 16 == 0): every row of a block has the same
// chunk alignment and phases, so a lane's selectors are built once.  Sums
// are exact integers (32-bit lane partials flushed to 64 bits).
constexpr int kSumThreads = kBlockThreads;

// selector words of one chunk: sel[q][c] has 0x01 in the bytes of word q that
// belong to channel c and lie in [s, e)
__device__ __forceinline__ void chunk_selectors(long long o, long long s, long long e, uint32_t (&sel)[4][3]) {
    const int ph = static_cast<int>(((o % 3) + 3) % 3);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t m[3] = {0, 0, 0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const long long x = o + 4 * q + b;
            const int ch = (ph + 4 * q + b) % 3;
            const uint32_t bit = (x >= s && x < e) ? (1u << (8 * b)) : 0u;
            m[0] |= ch == 0 ? bit : 0u;
            m[1] |= ch == 1 ? bit : 0u;
            m[2] |= ch == 2 ? bit : 0u;
        }
        sel[q][0] = m[0];
        sel[q][1] = m[1];
        sel[q][2] = m[2];
    }
}

__device__ __forceinline__ void dot_chunk(uint4 v, const uint32_t (&sel)[4][3], uint32_t (&acc)[3]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = __dp4a(w[q], sel[q][c], acc[c]);
    }
}

template <bool kUniform>
__global__ void __launch_bounds__(kSumThreads) block_sums_kernel(const uint8_t* __restrict__ fa,
                                                                 const uint8_t* __restrict__ fb, int width,
                                                                 int block_w, int block_h, int slices,
                                                                 int rows_per_slice, int log2_group, int n_tasks,
                                                                 long long total_bytes,
                                                                 const int32_t* __restrict__ xy,
                                                                 unsigned long long* __restrict__ sums) {
    const int task = static_cast<int>(blockIdx.x) * (kSumThreads / 32) + static_cast<int>(threadIdx.x >> 5);
    if (task >= n_tasks) return;
    const int blk = task / slices, slice = task - blk * slices;
    const int bx = __ldg(&xy[2 * blk]), by = __ldg(&xy[2 * blk + 1]);
    const int r0 = slice * rows_per_slice;
    const int r1 = min(r0 + rows_per_slice, block_h);
    const int group = 1 << log2_group, lane = threadIdx.x & 31;
    const int g = lane >> log2_group, li = lane & (group - 1), groups = 32 >> log2_group;
    unsigned long long ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    uint32_t pa[3] = {0, 0, 0}, pb[3] = {0, 0, 0};
    int pending = 0;
    const uint4* va4 = reinterpret_cast<const uint4*>(fa);
    const uint4* vb4 = reinterpret_cast<const uint4*>(fb);
    const long long row_bytes = 3ll * width;
    const long long s0 = 3 * (static_cast<long long>(by) * width + bx);
    const int nc0 = static_cast<int>(((s0 + 3ll * block_w + 15) >> 4) - (s0 >> 4));
    uint32_t sel0[4][3];
    if (kUniform && li < nc0) chunk_selectors(((s0 >> 4) + li) << 4, s0, s0 + 3ll * block_w, sel0);
    for (int r = r0 + g; r < r1; r += groups) {
        const long long s = s0 + static_cast<long long>(r) * row_bytes;
        const long long e = s + 3ll * block_w;
        const long long c0 = s >> 4;
        const int nc = static_cast<int>(((e + 15) >> 4) - c0);
        for (int k = li; k < nc; k += group) {
            const long long c = c0 + k, o = c << 4;
            if (o + 16 <= total_bytes) {
                uint32_t sel[4][3];
                if (kUniform && k == li) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
#pragma unroll
                        for (int x = 0; x < 3; ++x) sel[q][x] = sel0[q][x];
                    }
                } else {
                    chunk_selectors(o, s, e, sel);
                }
                dot_chunk(__ldcs(va4 + c), sel, pa);
                dot_chunk(__ldcs(vb4 + c), sel, pb);
                if (++pending == 65536) {  // 65536 chunks x 16 x 255 < 2^32
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        ca[x] += pa[x];
                        cb[x] += pb[x];
                        pa[x] = pb[x] = 0;
                    }
                    pending = 0;
                }
            } else {  // the image's last partial chunk
                const long long lo = o > s ? o : s;
                int ch = static_cast<int>(lo - s) % 3;
                for (long long i = lo; i < e; ++i) {
                    const unsigned long long x = fa[i], y = fb[i];
                    ca[0] += ch == 0 ? x : 0ull;
                    ca[1] += ch == 1 ? x : 0ull;
                    ca[2] += ch == 2 ? x : 0ull;
                    cb[0] += ch == 0 ? y : 0ull;
                    cb[1] += ch == 1 ? y : 0ull;
                    cb[2] += ch == 2 ? y : 0ull;
                    ch = ch == 2 ? 0 : ch + 1;
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < 3; ++x) {
        ca[x] += pa[x];
        cb[x] += pb[x];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        for (int o = 16; o; o >>= 1) {
            ca[c] += __shfl_xor_sync(0xffffffffu, ca[c], o);
            cb[c] += __shfl_xor_sync(0xffffffffu, cb[c], o);
        }
    }
    if (lane == 0) {  // one atomic per warp task and channel
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (ca[c]) atomicAdd(&sums[6 * blk + c], ca[c]);
            if (cb[c]) atomicAdd(&sums[6 * blk + 3 + c], cb[c]);
        }
    }
}

// log2 of the lanes per row: the power of two >= the items of a row
// segment, in [8, 32] (>= 6 lanes for the fill's edge bytes).
int lane_group_log2(int items) {
    int l = 3;
    while ((1 << l) < items && l < 5) ++l;
    return l;
}

// Row slices of a block (one warp task each) so that >= 16 warps per SM are
// in flight in total.
int rows_per_slice(int n_blocks, int block_h, int sms, unsigned* slices_out, int warps_per_sm = 16) {
    const long long want = (static_cast<long long>(sms) * warps_per_sm + n_blocks - 1) / n_blocks;
    long long slices = want < block_h ? want : block_h;
    if (slices < 1) slices = 1;
    const int rps = static_cast<int>((block_h + slices - 1) / slices);
    *slices_out = static_cast<unsigned>((block_h + rps - 1) / rps);
    return rps;
}

}  // namespace

cudaError_t launch_paint(const uint8_t* base, uint8_t* fa, uint8_t* fb, int width, int height, int block_w,
                         int block_h, int n_blocks, const int32_t* xy, const uint32_t* plus, const uint32_t* minus,
                         int sms, cudaStream_t st) {
    const long long n_bytes = 3ll * width * height;
    const bool vec = ((reinterpret_cast<uintptr_t>(base) | reinterpret_cast<uintptr_t>(fa) |
                       reinterpret_cast<uintptr_t>(fb)) & 15) == 0;
    const int grid = sms * 8;  // 8 x 256 threads per SM
    if (vec) {
        copy2_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(base), reinterpret_cast<uint4*>(fa),
                                           reinterpret_cast<uint4*>(fb), n_bytes / 16, base, fa, fb, n_bytes);
    } else {
        copy2_bytes_kernel<<<grid, 256, 0, st>>>(base, fa, fb, n_bytes);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || n_blocks <= 0) return e;
    unsigned slices = 1;
    // the fill is store-latency bound: ~48 warps per SM in flight (16 measured slower)
    const int rps = rows_per_slice(n_blocks, block_h, sms, &slices, 48);
    if ((reinterpret_cast<uintptr_t>(fa) | reinterpret_cast<uintptr_t>(fb)) & 3) return cudaErrorMisalignedAddress;
    const int lg = lane_group_log2((3 * block_w) / 4 + 1);
    const long long tasks = static_cast<long long>(n_blocks) * slices;
    if (tasks > (1ll << 31) - 1) return cudaErrorInvalidConfiguration;
    const int nt = static_cast<int>(tasks);
    const unsigned grid2 = static_cast<unsigned>((tasks + 7) / 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid2);
    cfg.blockDim = dim3(kBlockThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int sl = static_cast<int>(slices);
    return width % 4 == 0 ? cudaLaunchKernelEx(&cfg, fill_kernel<true>, fa, fb, width, block_w, block_h, sl, rps, lg,
                                               nt, xy, plus, minus)
                          : cudaLaunchKernelEx(&cfg, fill_kernel<false>, fa, fb, width, block_w, block_h, sl, rps,
                                               lg, nt, xy, plus, minus);
}

cudaError_t launch_block_sums(const uint8_t* fa, const uint8_t* fb, int width, int height, int block_w, int block_h,
                              int n_blocks, const int32_t* xy, unsigned long long* sums, int sms, cudaStream_t st) {
    const long long total_bytes = 3ll * width * height;
    if (n_blocks <= 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(fa) | reinterpret_cast<uintptr_t>(fb)) & 15) return cudaErrorMisalignedAddress;
    cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * 6 * static_cast<size_t>(n_blocks), st);
    if (e != cudaSuccess) return e;
    unsigned slices = 1;
    const int rps = rows_per_slice(n_blocks, block_h, sms, &slices);
    const int lg = lane_group_log2((3 * block_w + 15) / 16 + 1);
    const long long tasks = static_cast<long long>(n_blocks) * slices;
    if (tasks > (1ll << 31) - 1) return cudaErrorInvalidConfiguration;
    const int nt = static_cast<int>(tasks);
    const unsigned grid = static_cast<unsigned>((tasks + 7) / 8);
    if (width % 16 == 0) {
        block_sums_kernel<true><<<grid, kSumThreads, 0, st>>>(fa, fb, width, block_w, block_h, static_cast<int>(slices),
                                                               rps, lg, nt, total_bytes, xy, sums);
    } else {
        block_sums_kernel<false><<<grid, kSumThreads, 0, st>>>(fa, fb, width, block_w, block_h,
                                                                static_cast<int>(slices), rps, lg, nt, total_bytes, xy,
                                                                sums);
    }
    return cudaGetLastError();
}

}  // namespace cvg
