// cvg_codec_host.cpp -- the codec passes' C-ABI (include/cvg.h): layout
// validation and span tables, prepared layouts, and the launches of the
// paint and block-sum kernels (cvg_codec.cu).
#include "cvg_host.h"

using namespace cvg::host;

// ============================================================================
// Codec passes (include/cvg.h; kernels in cvg_codec.cu).
namespace {

// Per-row span table of a block layout (CSR over rows, x0 sorted), with the
// reference's BlockLayout::validate checks (codec.cpp:25-54).  Equal-size
// blocks overlap iff two of them share a row with overlapping x ranges, and
// then two neighbours in that row's sorted list overlap: one pass over the
// sorted rows replaces the reference's all-pairs test.
struct SpanCsr {
    std::vector<int32_t> row_ptr, x0, blk;
};

int layout_spans(int32_t width, int32_t height, int32_t bw, int32_t bh, int32_t n, const int32_t* xy, SpanCsr& t) {
    if (width <= 0 || height <= 0) return fail(CVG_EINVAL, "image dimensions must be positive");
    if (bw <= 0 || bh <= 0) return fail(CVG_EINVAL, "layout: block size must be positive");
    if (n < 0 || (n > 0 && !xy)) return fail(CVG_EINVAL, "layout: block positions missing");
    for (int32_t i = 0; i < n; ++i) {
        const int64_t x = xy[2 * i], y = xy[2 * i + 1];
        if (x < 0 || y < 0 || x + bw > width || y + bh > height) {
            return fail(CVG_EINVAL, "layout: block " + std::to_string(i) + " exceeds image bounds");
        }
    }
    t.row_ptr.assign(static_cast<size_t>(height) + 1, 0);
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t r = 0; r < bh; ++r) ++t.row_ptr[xy[2 * i + 1] + r + 1];
    }
    for (int32_t y = 0; y < height; ++y) t.row_ptr[y + 1] += t.row_ptr[y];
    const size_t spans = static_cast<size_t>(t.row_ptr[height]);
    t.x0.resize(spans);
    t.blk.resize(spans);
    std::vector<int32_t> fill(t.row_ptr.begin(), t.row_ptr.end() - 1);
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t r = 0; r < bh; ++r) {
            const int32_t k = fill[xy[2 * i + 1] + r]++;
            t.x0[k] = xy[2 * i];
            t.blk[k] = i;
        }
    }
    std::vector<std::pair<int32_t, int32_t>> row;
    for (int32_t y = 0; y < height; ++y) {
        const int32_t s = t.row_ptr[y], e = t.row_ptr[y + 1];
        if (e - s < 2) continue;
        bool sorted = true;
        for (int32_t k = s + 1; k < e; ++k) sorted = sorted && t.x0[k - 1] <= t.x0[k];
        if (!sorted) {
            row.clear();
            for (int32_t k = s; k < e; ++k) row.emplace_back(t.x0[k], t.blk[k]);
            std::sort(row.begin(), row.end());
            for (int32_t k = s; k < e; ++k) std::tie(t.x0[k], t.blk[k]) = row[k - s];
        }
        for (int32_t k = s + 1; k < e; ++k) {
            if (t.x0[k - 1] + bw > t.x0[k]) {
                const int32_t a = std::min(t.blk[k - 1], t.blk[k]), b = std::max(t.blk[k - 1], t.blk[k]);
                return fail(CVG_EINVAL, "layout: blocks " + std::to_string(a) + " and " + std::to_string(b) +
                                            " overlap");
            }
        }
    }
    return CVG_OK;
}

template <typename T>
size_t blob_put(std::vector<unsigned char>& blob, const T* p, size_t n) {
    const size_t off = (blob.size() + 255) & ~size_t(255);
    blob.resize(off + sizeof(T) * n);
    if (n) std::memcpy(blob.data() + off, p, sizeof(T) * n);
    return off;
}

// Device scratch for host-memory rasters (from the context's pool).
struct DevScratch {
    cvg_ctx* ctx;
    std::vector<void*> blocks;
    ~DevScratch() {
        for (void* b : blocks) ctx->dev.release(b);
    }
    void* get(size_t bytes) {
        void* p = ctx->dev.alloc(bytes);
        if (p) blocks.push_back(p);
        return p;
    }
};

}  // namespace

// A validated block layout on the device: positions and the packed block
// colors of the last paint, in one allocation.  `done` follows the last pass
// that read it; anything that rewrites the tables first makes its stream wait
// on it (or waits on the host when the allocation must grow).
struct cvg_layout {
    cvg_ctx* ctx = nullptr;
    int32_t width = 0, height = 0, bw = 0, bh = 0, n = 0;
    unsigned char* d = nullptr;
    size_t cap = 0;
    size_t o_xy = 0, o_pl = 0, o_mi = 0;
    cudaEvent_t done = nullptr;
    bool pending = false;
    std::vector<uint32_t> colors;  // packed colors the device holds (plus then minus)
    bool colors_valid = false;
};

namespace {

int layout_reserve(cvg_layout* L, size_t bytes, cudaStream_t st) {
    if (!L->done) CVG_CUDA(cudaEventCreateWithFlags(&L->done, cudaEventDisableTiming));
    if (bytes > L->cap) {
        if (L->pending) CVG_CUDA(cudaEventSynchronize(L->done));
        if (L->d) CVG_CUDA(cudaFree(L->d));
        L->d = nullptr;
        L->cap = 0;
        const size_t cap = std::max<size_t>(bytes, 1u << 16);
        CVG_CUDA(cudaMalloc(reinterpret_cast<void**>(&L->d), cap));
        L->cap = cap;
    } else if (L->pending) {
        CVG_CUDA(cudaStreamWaitEvent(st, L->done, 0));
    }
    return CVG_OK;
}

// Validates the geometry, builds the span table and uploads it on `st`
// (pageable source: the driver stages the bytes before the call returns).
int layout_prepare(cvg_layout* L, int32_t width, int32_t height, int32_t bw, int32_t bh, int32_t n,
                   const int32_t* xy, cudaStream_t st) {
    SpanCsr t;
    if (int e = layout_spans(width, height, bw, bh, n, xy, t)) return e;
    std::vector<unsigned char> blob;  // the span table only validates; the kernels take positions
    L->o_xy = blob_put(blob, xy, 2 * static_cast<size_t>(n));
    L->o_pl = (blob.size() + 255) & ~size_t(255);  // colors: plus then minus, written by the paints
    L->o_mi = L->o_pl + 4 * static_cast<size_t>(n);
    L->colors_valid = false;
    const size_t total = L->o_mi + 4 * static_cast<size_t>(n);
    if (int e = layout_reserve(L, total, st)) return e;
    CVG_CUDA(cudaMemcpyAsync(L->d, blob.data(), blob.size(), cudaMemcpyHostToDevice, st));
    L->width = width;
    L->height = height;
    L->bw = bw;
    L->bh = bh;
    L->n = n;
    return CVG_OK;
}

// Packs the block colors and uploads them (one copy; plus then minus are
// adjacent) unless they equal what the device already holds -- a codec
// stream paints the same message frame after frame.
int layout_colors(cvg_layout* L, const uint8_t* plus, const uint8_t* minus, cudaStream_t st) {
    if (L->n == 0) return CVG_OK;
    if (!plus || !minus) return fail(CVG_EINVAL, "block colors missing");
    const size_t n = static_cast<size_t>(L->n);
    std::vector<uint32_t> w(2 * n);
    for (size_t i = 0; i < n; ++i) {
        w[i] = plus[3 * i] | (uint32_t(plus[3 * i + 1]) << 8) | (uint32_t(plus[3 * i + 2]) << 16);
        w[n + i] = minus[3 * i] | (uint32_t(minus[3 * i + 1]) << 8) | (uint32_t(minus[3 * i + 2]) << 16);
    }
    if (L->colors_valid && L->colors == w) return CVG_OK;
    if (L->pending) CVG_CUDA(cudaStreamWaitEvent(st, L->done, 0));
    CVG_CUDA(cudaMemcpyAsync(L->d + L->o_pl, w.data(), 8 * n, cudaMemcpyHostToDevice, st));
    L->colors.swap(w);
    L->colors_valid = true;
    return CVG_OK;
}

int layout_finish(cvg_layout* L, cudaStream_t st) {
    CVG_CUDA(cudaEventRecord(L->done, st));
    L->pending = true;
    return CVG_OK;
}

int paint_pass(cvg_layout* L, const uint8_t* base, uint8_t* fa, uint8_t* fb, const uint8_t* plus,
               const uint8_t* minus, int32_t mem, cudaStream_t st) {
    cvg_ctx* ctx = L->ctx;
    if (int e = layout_colors(L, plus, minus, st)) return e;
    const size_t bytes = 3 * static_cast<size_t>(L->width) * static_cast<size_t>(L->height);
    DevScratch scratch{ctx};
    const uint8_t* d_base = base;
    uint8_t *d_a = fa, *d_b = fb;
    if (mem == CVG_MEM_HOST) {
        auto* db = static_cast<uint8_t*>(scratch.get(bytes));
        d_a = static_cast<uint8_t*>(scratch.get(bytes));
        d_b = static_cast<uint8_t*>(scratch.get(bytes));
        if (!db || !d_a || !d_b) return fail(CVG_ENOMEM, "device allocation of the frames failed");
        CVG_CUDA(cudaMemcpyAsync(db, base, bytes, cudaMemcpyHostToDevice, st));
        d_base = db;
    }
    CVG_CUDA(cvg::launch_paint(d_base, d_a, d_b, L->width, L->height, L->bw, L->bh, L->n,
                               reinterpret_cast<const int32_t*>(L->d + L->o_xy),
                               reinterpret_cast<const uint32_t*>(L->d + L->o_pl),
                               reinterpret_cast<const uint32_t*>(L->d + L->o_mi), ctx->sms, st));
    if (int e = layout_finish(L, st)) return e;
    if (mem == CVG_MEM_HOST) {
        CVG_CUDA(cudaMemcpyAsync(fa, d_a, bytes, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaMemcpyAsync(fb, d_b, bytes, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaStreamSynchronize(st));
    }
    return CVG_OK;
}

int sums_pass(cvg_layout* L, const uint8_t* fa, const uint8_t* fb, uint64_t* sums, int32_t mem, cudaStream_t st) {
    if (L->n == 0) return CVG_OK;
    cvg_ctx* ctx = L->ctx;
    const size_t bytes = 3 * static_cast<size_t>(L->width) * static_cast<size_t>(L->height);
    DevScratch scratch{ctx};
    const uint8_t *d_a = fa, *d_b = fb;
    auto* d_sums = reinterpret_cast<unsigned long long*>(sums);
    if (mem == CVG_MEM_HOST) {
        auto* da = static_cast<uint8_t*>(scratch.get(bytes));
        auto* db = static_cast<uint8_t*>(scratch.get(bytes));
        d_sums = static_cast<unsigned long long*>(scratch.get(sizeof(uint64_t) * 6 * L->n));
        if (!da || !db || !d_sums) return fail(CVG_ENOMEM, "device allocation of the frames failed");
        CVG_CUDA(cudaMemcpyAsync(da, fa, bytes, cudaMemcpyHostToDevice, st));
        CVG_CUDA(cudaMemcpyAsync(db, fb, bytes, cudaMemcpyHostToDevice, st));
        d_a = da;
        d_b = db;
    }
    CVG_CUDA(cvg::launch_block_sums(d_a, d_b, L->width, L->height, L->bw, L->bh, L->n,
                                    reinterpret_cast<const int32_t*>(L->d + L->o_xy), d_sums, ctx->sms, st));
    if (int e = layout_finish(L, st)) return e;
    if (mem == CVG_MEM_HOST) {
        CVG_CUDA(cudaMemcpyAsync(sums, d_sums, sizeof(uint64_t) * 6 * L->n, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaStreamSynchronize(st));
    }
    return CVG_OK;
}

int codec_common(cvg_ctx* ctx, int32_t mem, const void* a, const void* b, const void* c) {
    if (!ctx) return fail(CVG_EINVAL, "null context");
    if (mem != CVG_MEM_HOST && mem != CVG_MEM_DEVICE) return fail(CVG_EINVAL, "mem must be CVG_MEM_HOST or CVG_MEM_DEVICE");
    if (!a || !b || !c) return fail(CVG_EINVAL, "null raster pointer");
    return ensure_device(ctx);
}

cvg_layout* scratch_layout(cvg_ctx* ctx) {
    if (!ctx->codec_layout) {
        ctx->codec_layout = new cvg_layout();
        ctx->codec_layout->ctx = ctx;
    }
    return ctx->codec_layout;
}

}  // namespace

void layout_free(cvg_layout* L) {
    if (!L) return;
    cudaSetDevice(L->ctx->device);
    if (L->pending) cudaEventSynchronize(L->done);
    if (L->done) cudaEventDestroy(L->done);
    if (L->d) cudaFree(L->d);
    delete L;
}

extern "C" {

int cvg_paint_blocks(cvg_ctx* ctx, const uint8_t* base, uint8_t* frame_a, uint8_t* frame_b, int32_t width,
                     int32_t height, int32_t block_w, int32_t block_h, int32_t n_blocks, const int32_t* xy,
                     const uint8_t* plus_rgb, const uint8_t* minus_rgb, int32_t mem, void* stream) {
    if (int e = codec_common(ctx, mem, base, frame_a, frame_b)) return e;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    try {
        cudaStream_t st = mem == CVG_MEM_DEVICE ? static_cast<cudaStream_t>(stream) : ctx->stream;
        cvg_layout* L = scratch_layout(ctx);
        if (int e = layout_prepare(L, width, height, block_w, block_h, n_blocks, xy, st)) return e;
        return paint_pass(L, base, frame_a, frame_b, plus_rgb, minus_rgb, mem, st);
    } catch (const std::bad_alloc&) {
        return fail(CVG_ENOMEM, "host allocation failed");
    }
}

int cvg_block_sums(cvg_ctx* ctx, const uint8_t* frame_a, const uint8_t* frame_b, int32_t width, int32_t height,
                   int32_t block_w, int32_t block_h, int32_t n_blocks, const int32_t* xy, uint64_t* sums,
                   int32_t mem, void* stream) {
    if (int e = codec_common(ctx, mem, frame_a, frame_b, n_blocks > 0 ? static_cast<const void*>(sums) : frame_a)) {
        return e;
    }
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    try {
        cudaStream_t st = mem == CVG_MEM_DEVICE ? static_cast<cudaStream_t>(stream) : ctx->stream;
        cvg_layout* L = scratch_layout(ctx);
        if (int e = layout_prepare(L, width, height, block_w, block_h, n_blocks, xy, st)) return e;
        return sums_pass(L, frame_a, frame_b, sums, mem, st);
    } catch (const std::bad_alloc&) {
        return fail(CVG_ENOMEM, "host allocation failed");
    }
}

int cvg_layout_create(cvg_ctx* ctx, int32_t width, int32_t height, int32_t block_w, int32_t block_h, int32_t n_blocks,
                      const int32_t* xy, cvg_layout** out) {
    if (!ctx || !out) return fail(CVG_EINVAL, "null context or output pointer");
    *out = nullptr;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    if (int e = ensure_device(ctx)) return e;
    auto* L = new (std::nothrow) cvg_layout();
    if (!L) return fail(CVG_ENOMEM, "host allocation failed");
    L->ctx = ctx;
    int e;
    try {
        e = layout_prepare(L, width, height, block_w, block_h, n_blocks, xy, ctx->stream);
    } catch (const std::bad_alloc&) {
        e = fail(CVG_ENOMEM, "host allocation failed");
    }
    if (!e) {
        const cudaError_t ce = cudaStreamSynchronize(ctx->stream);
        if (ce != cudaSuccess) e = cuda_fail(ce, "layout upload");
    }
    if (e) {
        layout_free(L);
        return e;
    }
    *out = L;
    return CVG_OK;
}

void cvg_layout_destroy(cvg_layout* L) {
    if (!L) return;
    std::lock_guard<std::recursive_mutex> lk(L->ctx->mu);
    layout_free(L);
}

int cvg_layout_paint(cvg_layout* L, const uint8_t* base, uint8_t* frame_a, uint8_t* frame_b, const uint8_t* plus_rgb,
                     const uint8_t* minus_rgb, int32_t mem, void* stream) {
    if (!L) return fail(CVG_EINVAL, "null layout");
    if (int e = codec_common(L->ctx, mem, base, frame_a, frame_b)) return e;
    std::lock_guard<std::recursive_mutex> lk(L->ctx->mu);
    try {
        cudaStream_t st = mem == CVG_MEM_DEVICE ? static_cast<cudaStream_t>(stream) : L->ctx->stream;
        return paint_pass(L, base, frame_a, frame_b, plus_rgb, minus_rgb, mem, st);
    } catch (const std::bad_alloc&) {
        return fail(CVG_ENOMEM, "host allocation failed");
    }
}

int cvg_layout_block_sums(cvg_layout* L, const uint8_t* frame_a, const uint8_t* frame_b, uint64_t* sums, int32_t mem,
                          void* stream) {
    if (!L) return fail(CVG_EINVAL, "null layout");
    if (int e = codec_common(L->ctx, mem, frame_a, frame_b, L->n > 0 ? static_cast<const void*>(sums) : frame_a)) {
        return e;
    }
    std::lock_guard<std::recursive_mutex> lk(L->ctx->mu);
    try {
        cudaStream_t st = mem == CVG_MEM_DEVICE ? static_cast<cudaStream_t>(stream) : L->ctx->stream;
        return sums_pass(L, frame_a, frame_b, sums, mem, st);
    } catch (const std::bad_alloc&) {
        return fail(CVG_ENOMEM, "host allocation failed");
    }
}

int cvg_layout_launches(const cvg_layout* L, int32_t pass) {
    if (!L) return 0;
    return pass == 0 ? (L->n > 0 ? 2 : 1) : (L->n > 0 ? 1 : 0);  // paint: copy + fill; sums: 1 (+ a memset)
}

}  // extern "C"

