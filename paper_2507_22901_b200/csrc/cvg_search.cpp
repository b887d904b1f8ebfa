// cvg_search.cpp -- cvg_search: one host call over a batch of searches, and
// its pipelined paths (search ranges whose host prep and read-back overlap
// the kernels of other ranges).
#include "cvg_host.h"

namespace cvg::host {

// ---- pipelined PAIRS search ------------------------------------------------
// The end-to-end cost of a large PAIRS search is the PCIe read-back of 10
// bytes per pair (cfg1: 38 MB, 0.69 ms at ~55 GB/s) after the device work.
// Splitting the batch into K search ranges lets chunk c's read-back (copy
// stream) overlap chunk c+1's build and kernels (compute stream); the
// host learns chunk c's pair total from a 8-byte tail copy behind its
// kernels and appends its pairs to one contiguous pinned result.
int pipeline_chunks(const cvg_search_desc* d) {
    if (d->output != CVG_OUT_PAIRS || d->n_searches < 2) return 1;
    const uint64_t cands = static_cast<uint64_t>(d->n_searches) * static_cast<uint64_t>(d->n_radii) *
                           static_cast<uint64_t>(d->n_angles);
    static const int forced = [] {
        const char* e = std::getenv("CVG_PIPELINE_K");  // tuning override; 1 disables pipelining
        return e ? std::atoi(e) : 0;
    }();
    uint64_t k;
    if (forced > 0) {
        k = static_cast<uint64_t>(forced);
    } else {
        // each range pays ~80 us of kernel tail and the last range's read-back
        // overlaps nothing; measured optimum (tools/sweep_pipeline.sh):
        // cfg1 (198M candidates) K=2, cfg3 (1.07G) K=4..6
        if (cands < (1ull << 26)) return 1;
        k = cands < (1ull << 29) ? 2 : (cands < (1ull << 31) ? 4 : 6);
    }
    return static_cast<int>(std::min<uint64_t>(k, static_cast<uint64_t>(d->n_searches)));
}

// Range boundaries growing linearly (sizes 1:2:...:K): the first range is
// small so the read-back starts early; the later ranges carry the bulk.
std::vector<size_t> ramp_bounds(size_t n, int K) {
    std::vector<size_t> lo(K + 1);
    static const bool even = std::getenv("CVG_PIPELINE_EVEN") != nullptr;  // tuning override
    if (even) {
        for (int c = 0; c <= K; ++c) lo[c] = n * c / K;
        return lo;
    }
    const size_t den = static_cast<size_t>(K) * (K + 1) / 2;
    for (int c = 0; c <= K; ++c) {
        const size_t num = static_cast<size_t>(c) * (c + 1) / 2;
        lo[c] = std::max(static_cast<size_t>(c), std::min(n - (K - c), n * num / den));
    }
    return lo;
}

// Range boundaries for the COUNTS / FIRST ranges: a small first range (its
// prep is the only one the device waits for), sizes doubling up to a plateau
// (the host prepares ~2.5x faster than the device computes, so range c + 1
// is ready before range c ends), and a taper so that the last range's
// read-back, the only one not overlapped, is small.  Weights per range; the
// batch is cut in proportion.  CVG_RANGE_SHAPE=0: the linear ramp above.
std::vector<size_t> shaped_bounds(size_t n, int K) {
    static const int shape = [] {
        const char* e = std::getenv("CVG_RANGE_SHAPE");
        return e ? std::atoi(e) : 1;
    }();
    if (shape == 0 || K < 6) return ramp_bounds(n, K);
    std::vector<double> w(K);
    static const std::vector<double> forced = [] {  // tuning override: CVG_RANGE_WEIGHTS="1,2,4,4,2,1"
        std::vector<double> v;
        if (const char* e = std::getenv("CVG_RANGE_WEIGHTS")) {
            for (const char* q = e; *q;) {
                char* end = nullptr;
                const double x = std::strtod(q, &end);
                if (end == q) break;
                if (x > 0) v.push_back(x);
                q = *end == ',' ? end + 1 : end;
            }
        }
        return v;
    }();
    if (static_cast<int>(forced.size()) == K) {
        w = forced;
    } else {
        const int up = std::min(5, K / 3), down = std::min(4, K / 3);
        double top = 1.0;
        for (int c = 0; c < up; ++c, top *= 2.0) w[c] = top;
        for (int c = up; c < K - down; ++c) w[c] = top;
        double t = top;
        for (int c = K - down; c < K; ++c) w[c] = (t *= 0.5);
    }
    double sum = 0.0;
    for (double x : w) sum += x;
    std::vector<size_t> lo(K + 1);
    double acc = 0.0;
    for (int c = 0; c <= K; ++c) {
        const size_t b = c == K ? n : static_cast<size_t>(static_cast<double>(n) * (acc / sum));
        lo[c] = std::max(static_cast<size_t>(c), std::min(n - (K - c), b));  // every range holds a search
        if (c < K) acc += w[c];
    }
    return lo;
}

struct ChunkTail {
    union {
        cvg::Stats st;
        unsigned char pad[256];
    };
    unsigned long long total;
};
static_assert(sizeof(cvg::Stats) <= 256 && offsetof(ChunkTail, total) == 256, "ChunkTail mirrors the workspace");

struct PinnedPairs {
    cvg_ctx* ctx;
    uint32_t* idx = nullptr;
    uint8_t* codes = nullptr;
    uint64_t cap = 0;

    // grows to `need` pairs keeping the first `used` (waits for in-flight copies)
    bool ensure(uint64_t need, uint64_t want, uint64_t used) {
        if (need <= cap) return true;
        const uint64_t ncap = std::max(need, want);
        auto* ni = static_cast<uint32_t*>(ctx->host.alloc(ncap * 4));
        auto* nc = static_cast<uint8_t*>(ctx->host.alloc(ncap * 6));
        if (!ni || !nc) {
            ctx->host.release(ni);
            ctx->host.release(nc);
            return false;
        }
        if (used) {
            cudaStreamSynchronize(ctx->copy_stream);
            const size_t parts = used >= (1u << 20) ? 16 : 1;
            parallel_for(
                parts,
                [&](size_t c) {
                    const size_t lo = used * c / parts, hi = used * (c + 1) / parts;
                    std::memcpy(ni + lo, idx + lo, 4 * (hi - lo));
                    std::memcpy(nc + 6 * lo, codes + 6 * lo, 6 * (hi - lo));
                },
                1);
        }
        ctx->host.release(idx);
        ctx->host.release(codes);
        idx = ni;
        codes = nc;
        cap = ncap;
        return true;
    }
};

// ---- pipelined COUNTS / FIRST search -----------------------------------------
// Per-pixel batches (cfg4: 8.3M searches) spend ~13 ms of host prep and
// ~3 ms of read-back around ~230 ms of kernels.  Split into K search ranges:
// range c+1 is built on the host while range c computes, and range c's
// counts (+ first pairs) are read back on the copy stream while later
// ranges compute.  Only range 0's prep and the last range's read-back stay
// exposed.  Every result array is sized up front (n searches).
int fixed_chunks(const cvg_search_desc* d) {
    if (d->output == CVG_OUT_PAIRS || d->n_searches < (1 << 20)) return 1;
    static const int forced = [] {
        const char* e = std::getenv("CVG_PIPELINE_K");
        return e ? std::atoi(e) : 0;
    }();
    return forced > 0 ? std::min(forced, d->n_searches) : 8;
}

int search_ranges_fixed(cvg_ctx* ctx, const cvg_search_desc* d, cvg_result* r, int K) {
    const double t0 = now_ms();
    const size_t n = static_cast<size_t>(d->n_searches);
    const uint64_t cps = static_cast<uint64_t>(d->n_radii) * static_cast<uint64_t>(d->n_angles);
    const bool first = d->output == CVG_OUT_FIRST;
    r->n_searches = d->n_searches;
    r->counts = static_cast<uint64_t*>(ctx->host.alloc(sizeof(uint64_t) * n));
    if (first) {
        r->first_idx = static_cast<uint32_t*>(ctx->host.alloc(4 * n));
        r->first_codes = static_cast<uint8_t*>(ctx->host.alloc(6 * n));
    }
    auto* tails = static_cast<ChunkTail*>(ctx->host.alloc(sizeof(ChunkTail) * K));
    if (!r->counts || !tails || (first && (!r->first_idx || !r->first_codes))) {
        ctx->host.release(tails);
        return fail(CVG_ENOMEM, "pinned host allocation failed");
    }
    std::vector<cvg_plan> plans(K);
    std::vector<cudaEvent_t> kdone(K, nullptr);
    GridTables grid;  // built once range 0 has validated the grid
    double prep = 0, h2d = 0, t_first_enqueued = 0;
    int err = CVG_OK;
    // growing ranges: the first range's prep (the only one not overlapped)
    // is short.  Measured cfg4 e2e (C-side ms): K=4 even 224-225,
    // K=4 ramp 227.7, K=8 even 231.0, K=8 ramp 220.2, K=16 ramp 221.2
    // shaped ranges, K = 8 (weights 1,2,4,4,4,4,2,1): cfg4 call 86.4 -> 84.2 ms against the
    // linear ramp (tools/sweep_ranges_cfg4.sh, tools/sweep_range_weights_cfg4.sh)
    const std::vector<size_t> bounds = shaped_bounds(n, K);
    for (int c = 0; c < K && !err; ++c) {
        const size_t lo = bounds[c], hi = bounds[c + 1];
        cvg_search_desc sub = *d;
        sub.n_searches = static_cast<int32_t>(hi - lo);
        sub.target_rgb = d->target_rgb + 3 * lo;
        sub.pattern_bits = d->pattern_bits + lo;
        sub.v_th = d->v_th + lo;
        sub.r_novib = d->r_novib + lo;
        const double tb = now_ms();
        err = validate_desc(&sub);  // cvg_search left the per-search scan to the ranges
        if (err) break;
        const double tv = now_ms();
        if (c == 0) grid = make_grid_tables(d);
        const double tg = now_ms();
        err = plan_build_safe(ctx, &sub, &plans[c], &grid);
        if (err) break;
        static const bool trace = std::getenv("CVG_TRACE") != nullptr;
        if (trace) {
            std::fprintf(stderr, "[cvg range %d] start@%.3f validate %.3f grid %.3f build %.3f (n = %zu)\n", c, tb - t0,
                         tv - tb, tg - tv, now_ms() - tg, hi - lo);
        }
        prep += (plans[c].t_prep_end ? plans[c].t_prep_end : now_ms()) - tb;
        h2d += plans[c].t_upload_end ? plans[c].t_upload_end - plans[c].t_prep_end : 0.0;
        if (!ctx->events.empty()) {
            kdone[c] = ctx->events.back();
            ctx->events.pop_back();
        } else if (cudaEventCreate(&kdone[c]) != cudaSuccess) {
            err = fail(CVG_ECUDA, "event creation failed");
            break;
        }
        // ranges alternate between two streams: range c + 1's phase-1 blocks
        // take the SMs that range c's tail leaves idle (CVG_RANGE_STREAMS=1: one)
        static const bool two = [] {
            const char* e = std::getenv("CVG_RANGE_STREAMS");
            return !e || std::atoi(e) != 1;
        }();
        cudaStream_t ps = two && (c & 1) ? ctx->tail_stream : ctx->stream;
        if (ps != ctx->stream) {  // the plan's constants were uploaded on ctx->stream
            if (cudaEventRecord(kdone[c], ctx->stream) != cudaSuccess ||
                cudaStreamWaitEvent(ps, kdone[c], 0) != cudaSuccess) {
                err = fail(CVG_ECUDA, "range stream ordering failed");
                break;
            }
        }
        err = plan_enqueue(&plans[c], ps);
        if (err) break;
        if (c == 0) t_first_enqueued = now_ms();
        const cvg_plan& p = plans[c];
        auto copy = [&]() -> int {
            cudaStream_t cs = ctx->copy_stream;
            CVG_CUDA(cudaEventRecord(kdone[c], ps));
            CVG_CUDA(cudaStreamWaitEvent(cs, kdone[c], 0));
            CVG_CUDA(cudaMemcpyAsync(r->counts + lo, p.args.counts, sizeof(uint64_t) * (hi - lo),
                                     cudaMemcpyDeviceToHost, cs));
            CVG_CUDA(cudaMemcpyAsync(&tails[c], p.args.stats, sizeof(ChunkTail), cudaMemcpyDeviceToHost, cs));
            if (first) {
                CVG_CUDA(cudaMemcpyAsync(r->first_idx + lo, p.args.first_idx, 4 * (hi - lo), cudaMemcpyDeviceToHost,
                                         cs));
                CVG_CUDA(cudaMemcpyAsync(r->first_codes + 6 * lo, p.args.first_codes, 6 * (hi - lo),
                                         cudaMemcpyDeviceToHost, cs));
            }
            return CVG_OK;
        };
        err = copy();
    }
    const double t_enqueued = now_ms();
    if (!err) {
        const cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
        if (ce != cudaSuccess) err = cuda_fail(ce, "result read-back");
    }
    const double t1 = now_ms();
    if (!err) {
        cvg::Stats agg{};
        float ratio_max = 0.f, kernel_ms = 0.f;
        uint64_t in_bytes = 0;
        for (int c = 0; c < K; ++c) {
            const cvg::Stats& st = tails[c].st;
            if (st.undecided && !err) err = undecided_fail(st.undecided);
            agg.band_repairs += st.band_repairs;
            agg.code_repairs += st.code_repairs;
            agg.audit_violations += st.audit_violations;
            agg.class_mismatch += st.class_mismatch;
            float ratio;
            std::memcpy(&ratio, &st.audit_max_ratio_bits, sizeof(float));
            ratio_max = std::max(ratio_max, ratio);
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, plans[c].ev0, plans[c].ev1) == cudaSuccess) kernel_ms += ms;
            in_bytes += plans[c].input_bytes;
        }
        r->n_pairs = sum_counts(r->counts, n);
        r->n_candidates = cps * n;
        r->n_band_repairs = agg.band_repairs;
        r->n_code_repairs = agg.code_repairs;
        r->n_audit_violations = agg.audit_violations;
        r->n_class_mismatch = agg.class_mismatch;
        r->audit_max_ratio = ratio_max;
        r->kernel_ms = kernel_ms;
        r->h2d_bytes = in_bytes;
        r->d2h_bytes = (sizeof(uint64_t) + (first ? 10 : 0)) * n + sizeof(ChunkTail) * K;
        r->prep_ms = static_cast<float>(prep);
        r->h2d_ms = static_cast<float>(h2d);
        r->device_ms = static_cast<float>(t1 - t_first_enqueued);  // ranges after the first overlap their prep
        r->d2h_ms = 0.f;                                               // overlapped except the last range's
        r->total_ms = static_cast<float>(t1 - t0);
        (void)t_enqueued;
    }
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->tail_stream);
    for (int c = 0; c < K; ++c) {
        if (kdone[c]) ctx->events.push_back(kdone[c]);
        if (plans[c].ctx) plan_release(&plans[c]);
    }
    ctx->host.release(tails);
    return err;
}

// One plan for the whole batch (constants and grid tables uploaded once),
// run as K search-range views back to back on the compute stream: phase 1,
// scan and emit of view c, then view c+1 with no host work in between.  The
// tail stream reads each view's counts and [stats | total] behind its emit;
// the host then queues the copy of the view's pairs (one contiguous slice of
// the canonical result, at the running total) on the copy stream, so the
// D2H engine drains view c while views c+1.. compute.  Only the first
// view's kernels and the last view's copy are exposed.
int search_pipelined(cvg_ctx* ctx, const cvg_search_desc* d, cvg_result* r, int K) {
    const double t0 = now_ms();
    const size_t n = static_cast<size_t>(d->n_searches);
    const uint64_t cps = static_cast<uint64_t>(d->n_radii) * static_cast<uint64_t>(d->n_angles);
    const uint32_t tps = static_cast<uint32_t>((cps + cvg::kTile - 1) / cvg::kTile);
    const uint64_t sig[4] = {n, cps, static_cast<uint64_t>(d->delta_basis), static_cast<uint64_t>(d->path)};
    const bool hinted = std::equal(sig, sig + 4, ctx->hint_sig);
    cvg_plan p;
    p.external_out = true;
    if (int e = plan_build_safe(ctx, d, &p)) {
        plan_release(&p);
        return e;
    }
    const double t_built = now_ms();
    struct Cleanup {
        cvg_ctx* ctx;
        cvg_plan* p;
        std::vector<void*> host;
        std::vector<cudaEvent_t> events;
        void* dev = nullptr;
        ~Cleanup() {
            cudaStreamSynchronize(ctx->copy_stream);
            cudaStreamSynchronize(ctx->tail_stream);
            cudaStreamSynchronize(ctx->stream);
            for (void* h : host) ctx->host.release(h);
            for (cudaEvent_t e : events) ctx->events.push_back(e);
            ctx->dev.release(dev);
            plan_release(p);
        }
    } cl{ctx, &p, {}, {}, nullptr};
    auto event = [&]() -> cudaEvent_t {
        cudaEvent_t e = nullptr;
        if (!ctx->events.empty()) {
            e = ctx->events.back();
            ctx->events.pop_back();
        } else if (cudaEventCreate(&e) != cudaSuccess) {
            return nullptr;
        }
        cl.events.push_back(e);
        return e;
    };
    // device pair buffer: the previous total of this shape (+25%), else
    // plan_reserve's default; a view that overflows reruns the batch at the
    // exact size
    {
        const uint64_t fit = static_cast<uint64_t>(ctx->total_mem / 4 / 10);
        const uint64_t cap = hinted ? ctx->hint_pairs + ctx->hint_pairs / 4 + (1u << 16)
                                    : std::min<uint64_t>(p.candidates, std::max<uint64_t>(fit, 1u << 20));
        if (hinted) plan_set_density(&p, ctx->hint_pairs);
        if (int e = plan_reserve(&p, cap)) return e;
    }

    // ---- per-view workspace: [Stats | total | tickets] x K | cum[K+1] | status | claim ----
    const std::vector<size_t> lo = ramp_bounds(n, K);
    constexpr size_t kHdr = 512;
    size_t status_words = 0;
    for (int c = 0; c < K; ++c) {
        status_words += ((lo[c + 1] - lo[c]) * tps + cvg::kScanTile - 1) / cvg::kScanTile;
    }
    const size_t o_cum = kHdr * K, o_st = o_cum + 8 * (K + 1), o_claim = o_st + 8 * status_words;
    const size_t vbytes = o_claim + 4 * n;
    auto* stage = static_cast<unsigned char*>(ctx->host.alloc(vbytes));
    auto* tails = static_cast<unsigned char*>(ctx->host.alloc(kHdr * K));
    cl.host = {stage, tails};
    cl.dev = ctx->dev.alloc(vbytes);
    r->n_searches = d->n_searches;
    r->counts = static_cast<uint64_t*>(ctx->host.alloc(sizeof(uint64_t) * n));
    r->offsets = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (n + 1)));
    if (!stage || !tails || !cl.dev || !r->counts || !r->offsets) return fail(CVG_ENOMEM, "allocation failed");
    auto* dv = static_cast<unsigned char*>(cl.dev);
    std::memset(stage, 0, o_claim);
    auto* claim = reinterpret_cast<uint32_t*>(stage + o_claim);
    std::vector<LaunchArgs> views(K, p.args);
    size_t st_off = 0;
    for (int c = 0; c < K; ++c) {
        LaunchArgs& V = views[c];
        const size_t b = lo[c], e = lo[c + 1];
        V.search_begin = static_cast<uint32_t>(b);
        V.range_searches = static_cast<uint32_t>(e - b);
        V.tile_begin = static_cast<uint64_t>(b) * tps;
        V.n_tiles = static_cast<uint64_t>(e - b) * tps;
        V.n_claims = static_cast<uint32_t>((e - b) * p.args.claim_per_search);
        V.stats = reinterpret_cast<cvg::Stats*>(dv + kHdr * c);
        V.total = reinterpret_cast<unsigned long long*>(dv + kHdr * c + 256);
        V.ticket = reinterpret_cast<unsigned int*>(dv + kHdr * c + 264);
        V.base_offset = reinterpret_cast<const unsigned long long*>(dv + o_cum + 8 * c);
        V.grand_total = reinterpret_cast<unsigned long long*>(dv + o_cum + 8 * (c + 1));
        V.status = reinterpret_cast<unsigned long long*>(dv + o_st + 8 * st_off);
        st_off += (V.n_tiles + cvg::kScanTile - 1) / cvg::kScanTile;
        V.worklist = p.args.worklist + V.tile_begin * (cvg::kTile / cvg::kEmitSpan);
        // claim order inside the view: searches grouped by loud count (one
        // hot-loop specialization per group), as plan_build does for a batch
        V.claim_order = nullptr;
        if (p.mode == cvg::kModeBand && e - b > 1) {
            std::array<uint32_t, 4> bucket{};
            for (size_t i = b; i < e; ++i) ++bucket[__builtin_popcount(d->pattern_bits[i] & 7)];
            if ((bucket[1] > 0) + (bucket[2] > 0) + (bucket[3] > 0) > 1) {
                V.group_end[0] = bucket[1];
                V.group_end[1] = bucket[1] + bucket[2];
                V.group_end[2] = bucket[1] + bucket[2] + bucket[3];
                std::array<uint32_t, 4> next{0, 0, V.group_end[0], V.group_end[1]};
                for (size_t i = b; i < e; ++i) {
                    claim[b + next[__builtin_popcount(d->pattern_bits[i] & 7)]++] = static_cast<uint32_t>(i);
                }
                V.claim_order = reinterpret_cast<const uint32_t*>(dv + o_claim) + b;
            }
        }
    }
    std::vector<cudaEvent_t> kdone(K), done(K), copied(K);
    for (int c = 0; c < K; ++c) {
        kdone[c] = event();
        done[c] = event();
        copied[c] = event();
        if (!kdone[c] || !done[c] || !copied[c]) return fail(CVG_ECUDA, "event creation failed");
    }
    cudaStream_t st = ctx->stream, ts = ctx->tail_stream, cs = ctx->copy_stream;
    CVG_CUDA(cudaMemcpyAsync(dv, stage, vbytes, cudaMemcpyHostToDevice, st));
    auto enqueue = [&]() -> int {
        CVG_CUDA(cudaMemsetAsync(p.d_work, 0, p.work_bytes, st));
        CVG_CUDA(cudaMemsetAsync(dv, 0, o_claim, st));  // headers, cum, status (a rerun starts clean)
        CVG_CUDA(cudaEventRecord(p.ev0, st));
        for (int c = 0; c < K; ++c) {
            LaunchArgs& V = views[c];
            V.out_idx = p.args.out_idx;  // plan_reserve may have replaced the buffers
            V.out_codes = p.args.out_codes;
            V.capacity = p.args.capacity;
            CVG_CUDA(cvg::launch_phase1(V, p.mode, p.out, p.path, p.grid, st));
            CVG_CUDA(cvg::launch_scan(V, st));
            CVG_CUDA(cvg::launch_emit(V, p.mode, p.path, p.grid, st));
            CVG_CUDA(cudaEventRecord(kdone[c], st));
            CVG_CUDA(cudaStreamWaitEvent(ts, kdone[c], 0));
            CVG_CUDA(cudaMemcpyAsync(r->counts + lo[c], p.args.counts + lo[c], sizeof(uint64_t) * (lo[c + 1] - lo[c]),
                                     cudaMemcpyDeviceToHost, ts));
            CVG_CUDA(cudaMemcpyAsync(tails + kHdr * c, dv + kHdr * c, 264, cudaMemcpyDeviceToHost, ts));
            CVG_CUDA(cudaEventRecord(done[c], ts));
        }
        CVG_CUDA(cudaEventRecord(p.ev1, st));
        return CVG_OK;
    };
    if (int e = enqueue()) return e;
    const double t_enq = now_ms();

    // ---- drain: copy each view's pairs as soon as its tail lands ----
    PinnedPairs out{ctx};
    uint64_t used = 0;
    bool overflow = false;
    cvg::Stats agg{};
    float ratio_max = 0.f;
    double t_last_done = t_enq;
    for (int c = 0; c < K; ++c) {
        CVG_CUDA(cudaEventSynchronize(done[c]));
        t_last_done = now_ms();
        const auto& s = *reinterpret_cast<const cvg::Stats*>(tails + kHdr * c);
        const uint64_t tc = *reinterpret_cast<const unsigned long long*>(tails + kHdr * c + 256);
        if (s.undecided) return undecided_fail(s.undecided);
        agg.band_repairs += s.band_repairs;
        agg.code_repairs += s.code_repairs;
        agg.audit_violations += s.audit_violations;
        agg.class_mismatch += s.class_mismatch;
        float ratio;
        std::memcpy(&ratio, &s.audit_max_ratio_bits, sizeof(float));
        ratio_max = std::max(ratio_max, ratio);
        overflow |= s.overflow != 0;
        if (!overflow && tc) {
            // pinned result sized for the whole batch up front when hinted
            const uint64_t seen = cps * lo[c + 1];
            const uint64_t extrap = (used + tc) * ((cps * n + seen - 1) / seen) + (used + tc) / 4 + (1u << 16);
            const uint64_t want = hinted ? std::max(ctx->hint_pairs, used + tc) : extrap;
            if (!out.ensure(used + tc, std::min<uint64_t>(want, cps * n), used)) {
                return fail(CVG_ENOMEM, "pinned host allocation failed");
            }
            CVG_CUDA(cudaStreamWaitEvent(cs, done[c], 0));
            CVG_CUDA(cudaMemcpyAsync(out.idx + used, p.args.out_idx + used, tc * 4, cudaMemcpyDeviceToHost, cs));
            CVG_CUDA(cudaMemcpyAsync(out.codes + 6 * used, p.args.out_codes + 6 * used, tc * 6, cudaMemcpyDeviceToHost,
                                     cs));
        }
        CVG_CUDA(cudaEventRecord(copied[c], cs));
        used += tc;
    }
    if (overflow) {
        // a view's pairs did not fit the device buffer: rerun at the exact size
        CVG_CUDA(cudaStreamSynchronize(cs));
        if (int e = plan_reserve(&p, used)) return e;
        if (int e = enqueue()) return e;
        CVG_CUDA(cudaStreamSynchronize(ts));
        for (int c = 0; c < K; ++c) {
            if (reinterpret_cast<const cvg::Stats*>(tails + kHdr * c)->overflow) {
                return fail(CVG_ECUDA, "pair buffer overflow after resizing");
            }
        }
        if (!out.ensure(used, used, 0)) return fail(CVG_ENOMEM, "pinned host allocation failed");
        if (used) {
            CVG_CUDA(cudaStreamWaitEvent(cs, done[K - 1], 0));
            CVG_CUDA(cudaMemcpyAsync(out.idx, p.args.out_idx, used * 4, cudaMemcpyDeviceToHost, cs));
            CVG_CUDA(cudaMemcpyAsync(out.codes, p.args.out_codes, used * 6, cudaMemcpyDeviceToHost, cs));
        }
    }
    CVG_CUDA(cudaStreamSynchronize(cs));
    const double t1 = now_ms();
    static const bool trace = std::getenv("CVG_TRACE") != nullptr;
    if (trace) {
        std::string line = "[cvg pipeline] K=" + std::to_string(K) + " built@" + std::to_string(t_built - t0).substr(0, 6) +
                           " enq@" + std::to_string(t_enq - t0).substr(0, 6) + " end@" + std::to_string(t1 - t0).substr(0, 6);
        for (int c = 0; c < K; ++c) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, p.ev0, kdone[c]);
            cudaEventElapsedTime(&b, p.ev0, copied[c]);
            line += " | v" + std::to_string(c) + " n=" + std::to_string(lo[c + 1] - lo[c]) + " kernels@" +
                    std::to_string(a).substr(0, 5) + " copied@" + std::to_string(b).substr(0, 5);
        }
        std::fprintf(stderr, "%s\n", line.c_str());
    }

    // ---- result ----
    r->offsets[0] = 0;
    for (size_t s = 0; s < n; ++s) r->offsets[s + 1] = r->offsets[s] + r->counts[s];
    if (r->offsets[n] != used) return fail(CVG_ECUDA, "pipelined search: counts and pair totals disagree");
    r->n_pairs = used;
    r->idx = used ? out.idx : nullptr;
    r->codes = used ? out.codes : nullptr;
    if (!used) {
        ctx->host.release(out.idx);
        ctx->host.release(out.codes);
    }
    r->n_candidates = cps * n;
    r->n_band_repairs = agg.band_repairs;
    r->n_code_repairs = agg.code_repairs;
    r->n_audit_violations = agg.audit_violations;
    r->n_class_mismatch = agg.class_mismatch;
    r->audit_max_ratio = ratio_max;
    CVG_CUDA(cudaEventElapsedTime(&r->kernel_ms, p.ev0, p.ev1));
    r->h2d_bytes = p.input_bytes + vbytes;
    r->d2h_bytes = sizeof(uint64_t) * n + 264 * K + used * 10;
    r->prep_ms = static_cast<float>((p.t_prep_end ? p.t_prep_end : t_built) - t0);
    r->h2d_ms = static_cast<float>(p.t_upload_end ? p.t_upload_end - p.t_prep_end : 0.0);
    r->device_ms = static_cast<float>(t_last_done - t_enq);
    r->d2h_ms = static_cast<float>(t1 - t_last_done);
    r->total_ms = static_cast<float>(t1 - t0);
    std::copy(sig, sig + 4, ctx->hint_sig);
    ctx->hint_pairs = used;
    return CVG_OK;
}

}  // namespace cvg::host

using namespace cvg::host;

extern "C" {

int cvg_search(cvg_ctx* ctx, const cvg_search_desc* desc, cvg_result* out) {
    if (!ctx || !out) return fail(CVG_EINVAL, "null context or result");
    result_zero(out);
    if (int e = validate_header(desc)) return e;
    // Search ranges (COUNTS / FIRST) validate range by range, each just
    // before its plan is built, so that the scan of range c + 1 overlaps
    // range c's kernels (cfg4: ~4 ms of an 88 ms call).  The ranges run in
    // order, so the first failure reported is the batch's first, with the
    // reference's message; the other paths validate the whole batch here.
    const bool ranged_fixed = desc->output != CVG_OUT_PAIRS && desc->path != CVG_PATH_MEMO &&
                              desc->output != CVG_OUT_BEST && fixed_chunks(desc) > 1;
    if (!ranged_fixed) {
        if (int e = validate_desc(desc)) return e;
    }
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    if (int e = ensure_device(ctx)) return e;
    // A plan holds < 2^28 tiles (32-bit tile ids with 16 emit items each):
    // larger batches always run as search ranges, each well under the limit.
    int K_min = 1;
    {
        const uint64_t cps = static_cast<uint64_t>(desc->n_radii) * static_cast<uint64_t>(desc->n_angles);
        const uint64_t tiles = (cps + cvg::kTile - 1) / cvg::kTile * static_cast<uint64_t>(desc->n_searches);
        const uint64_t per_range = 1ull << 26;  // ramp ranges reach 2/(K+1) of the batch
        if (tiles >= per_range) K_min = static_cast<int>(std::min<uint64_t>((tiles + per_range - 1) / per_range,
                                                                             static_cast<uint64_t>(desc->n_searches)));
    }
    // memoized batches run as one plan: the color dedup must see the whole batch
    // and BEST runs one plan (select_best reads each search's whole list on the device)
    const bool single = desc->path == CVG_PATH_MEMO || desc->output == CVG_OUT_BEST;
    if (const int K = single ? 1 : std::max({pipeline_chunks(desc), fixed_chunks(desc), K_min});
        K > 1) {
        int e;
        try {
            e = desc->output == CVG_OUT_PAIRS ? search_pipelined(ctx, desc, out, K)
                                              : search_ranges_fixed(ctx, desc, out, K);
        } catch (const std::bad_alloc&) {
            e = fail(CVG_ENOMEM, "host allocation failed");
        } catch (const std::exception& ex) {
            e = fail(CVG_EUNSUPPORTED, ex.what());
        }
        remember_owner(out, ctx);
        if (e) cvg_result_free(out);
        return e;
    }
    const double t0 = now_ms();
    cvg_plan plan;
    int e = plan_build_safe(ctx, desc, &plan);
    const double t_built = now_ms();
    if (!e) e = plan_enqueue(&plan, ctx->stream);
    if (!e) e = plan_fetch_impl(&plan, out, true);
    if (!e) {
        const double t1 = now_ms();
        out->prep_ms = static_cast<float>((plan.t_prep_end ? plan.t_prep_end : t_built) - t0);
        out->h2d_ms = static_cast<float>(plan.t_upload_end ? plan.t_upload_end - plan.t_prep_end : 0.0);
        out->total_ms = static_cast<float>(t1 - t0);
        out->device_ms = static_cast<float>(t1 - t_built - out->d2h_ms);
    }
    if (plan.ran) cudaStreamSynchronize(ctx->stream);
    plan_release(&plan);
    plan.ctx = nullptr;
    remember_owner(out, ctx);
    if (e) cvg_result_free(out);
    return e;
}

}  // extern "C"
