// cvg_plan.cpp -- plans (build once, run many) and the context, plan and
// scalar parts of the C-ABI (include/cvg.h).
#include "cvg_host.h"

namespace cvg::host {

thread_local std::string g_error;

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(CVG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int ensure_device(cvg_ctx* ctx) {
    CVG_CUDA(cudaSetDevice(ctx->device));
    return CVG_OK;
}

void plan_free_outputs(cvg_plan* p) {
    p->ctx->dev.release(p->d_out_idx);
    p->ctx->dev.release(p->d_out_codes);
    p->d_out_idx = p->d_out_codes = nullptr;
    p->capacity = 0;
}

// Emit item size from the expected pair count: batches averaging >= 256
// pairs per tile (cfg2: ~750) take 512-pair items, half the item set-ups
// (cfg2 emit 3.32 -> 3.04 ms); sparse batches keep 256 so that the last
// items stay short (cfg1: 512 everywhere measured 0.051 -> 0.054 ms).
void plan_set_density(cvg_plan* p, uint64_t expected_pairs) {
    const uint64_t tiles = p->args.n_tiles ? p->args.n_tiles : 1;
    p->args.emit_shift = expected_pairs >= 256 * tiles ? 9u : 8u;
    if (const char* e = std::getenv("CVG_EMIT_SHIFT")) {  // A/B override (8..12)
        const int v = std::atoi(e);
        if (v >= 8 && v <= 12) p->args.emit_shift = static_cast<uint32_t>(v);
    }
}

int plan_reserve(cvg_plan* p, uint64_t cap) {
    if (p->out != cvg::kOutPairs || p->empty) return CVG_OK;
    if (cap == 0) cap = 1;
    if (cap == p->capacity && p->d_out_idx) return CVG_OK;
    plan_free_outputs(p);
    p->d_out_idx = p->ctx->dev.alloc(cap * sizeof(uint32_t));
    p->d_out_codes = p->ctx->dev.alloc(cap * 6);
    if (!p->d_out_idx || !p->d_out_codes) {
        plan_free_outputs(p);
        return fail(CVG_ENOMEM, "device allocation of the pair buffer failed");
    }
    p->capacity = cap;
    p->args.out_idx = static_cast<uint32_t*>(p->d_out_idx);
    p->args.out_codes = static_cast<uint8_t*>(p->d_out_codes);
    p->args.capacity = cap;
    return CVG_OK;
}

// Bump layout of several arrays inside one allocation (256-byte aligned).
struct Layout {
    size_t off = 0;
    size_t take(size_t bytes) {
        off = (off + 255) & ~size_t(255);
        const size_t o = off;
        off += bytes;
        return o;
    }
};

template <typename T>
T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(static_cast<unsigned char*>(base) + off);
}

// sc_index[s] -> record of search s; uniq[u] -> first search with record u.
// sc_index stays empty when every search is distinct (identity mapping).
// Returns true if every search has the same (pattern, v_th, r_novib).
bool dedup_searches(const cvg_search_desc* d, std::vector<uint32_t>& sc_index, std::vector<int32_t>& uniq) {
    const int n = d->n_searches;
    sc_index.clear();
    uniq.clear();
    if (n <= 0) return true;
    // uniform classifier? (chunked so a per-pixel screen runs on all cores;
    // 16K searches per chunk at least)
    const size_t parts = std::min<size_t>(64, std::max<size_t>(1, static_cast<size_t>(n) >> 14));
    std::vector<char> same(parts, 1);
    parallel_for(
        parts,
        [&](size_t c) {
            const size_t lo = std::max<size_t>(1, n * c / parts), hi = n * (c + 1) / parts;
            const int32_t b0 = d->pattern_bits[0];
            const double v0 = d->v_th[0], r0 = d->r_novib[0];
            bool ok = true;
            for (size_t s = lo; s < hi; ++s) {
                ok &= (d->pattern_bits[s] == b0) & (d->v_th[s] == v0) & (d->r_novib[s] == r0);
            }
            same[c] = ok;
        },
        1);
    bool uniform = true;
    for (char c : same) uniform = uniform && c;
    auto key24 = [&](size_t s) {
        const int32_t* t = d->target_rgb + 3 * s;
        return static_cast<uint32_t>(t[0]) << 16 | static_cast<uint32_t>(t[1]) << 8 | static_cast<uint32_t>(t[2]);
    };
    sc_index.resize(n);
    if (uniform && n > 4096) {
        // Same classifier everywhere: records keyed by the 24-bit color.
        // Presence bitmap over the 2^24 colors (2 MB) + per-word rank, so the
        // record id of a color is rank(color): no table to clear, cache-resident.
        // Both passes run chunked over all cores; the representative of a
        // record is its first search (atomic min), so the result is
        // independent of the thread count.
        std::vector<uint64_t> bits(1u << 18, 0);
        const size_t chunks = parts;
        parallel_for(
            chunks,
            [&](size_t c) {
                for (size_t s = n * c / chunks; s < n * (c + 1) / chunks; ++s) {
                    const uint32_t k = key24(s);
                    const uint64_t m = 1ull << (k & 63);
                    if (!(__atomic_load_n(&bits[k >> 6], __ATOMIC_RELAXED) & m)) {
                        __atomic_fetch_or(&bits[k >> 6], m, __ATOMIC_RELAXED);
                    }
                }
            },
            1);
        std::vector<uint32_t> rank(1u << 18);
        uint32_t acc = 0;
        for (size_t w = 0; w < bits.size(); ++w) {
            rank[w] = acc;
            acc += static_cast<uint32_t>(__builtin_popcountll(bits[w]));
        }
        uniq.assign(acc, INT32_MAX);
        parallel_for(
            chunks,
            [&](size_t c) {
                for (size_t s = n * c / chunks; s < n * (c + 1) / chunks; ++s) {
                    const uint32_t k = key24(s);
                    const uint32_t id = rank[k >> 6] +
                                        static_cast<uint32_t>(__builtin_popcountll(bits[k >> 6] & ((1ull << (k & 63)) - 1)));
                    sc_index[s] = id;
                    int32_t cur = __atomic_load_n(&uniq[id], __ATOMIC_RELAXED);
                    const int32_t me = static_cast<int32_t>(s);
                    while (me < cur &&
                           !__atomic_compare_exchange_n(&uniq[id], &cur, me, true, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
                    }
                }
            },
            1);
    } else {
        // Open-addressing table of search ids keyed by (color, pattern, v_th,
        // r_novib) bits: no per-entry allocation (4096 searches: ~40 us
        // instead of ~450 us with std::unordered_map).
        auto same = [&](size_t a, size_t b) {
            return key24(a) == key24(b) && d->pattern_bits[a] == d->pattern_bits[b] &&
                   std::memcmp(&d->v_th[a], &d->v_th[b], 8) == 0 && std::memcmp(&d->r_novib[a], &d->r_novib[b], 8) == 0;
        };
        auto hash = [&](size_t s) {
            uint64_t a, b;
            std::memcpy(&a, &d->v_th[s], 8);
            std::memcpy(&b, &d->r_novib[s], 8);
            uint64_t h = (static_cast<uint64_t>(key24(s)) << 3 | static_cast<uint64_t>(d->pattern_bits[s] & 7)) *
                         0x9E3779B97F4A7C15ull;
            h ^= (a + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2)) * 0xBF58476D1CE4E5B9ull;
            h ^= (b + 0x85157AF5ull + (h << 6) + (h >> 2)) * 0x94D049BB133111EBull;
            return h ^ (h >> 31);
        };
        size_t cap = 16;
        while (cap < 2 * static_cast<size_t>(n)) cap <<= 1;
        std::vector<int32_t> slot(cap, -1);  // search id of the record's representative
        for (int s = 0; s < n; ++s) {
            size_t i = hash(static_cast<size_t>(s)) & (cap - 1);
            while (slot[i] >= 0 && !same(static_cast<size_t>(slot[i]), static_cast<size_t>(s))) i = (i + 1) & (cap - 1);
            if (slot[i] < 0) {
                slot[i] = s;
                sc_index[s] = static_cast<uint32_t>(uniq.size());
                uniq.push_back(s);
            } else {
                sc_index[s] = sc_index[slot[i]];
            }
        }
    }
    if (static_cast<int>(uniq.size()) == n) {
        sc_index.clear();  // all distinct: records are in search order
    }
    return uniform;
}

GridTables make_grid_tables(const cvg_search_desc* d) {
    GridTables g;
    g.radii_f.resize(d->n_radii);
    for (int k = 0; k < d->n_radii; ++k) g.radii_f[k] = static_cast<float>(d->radii[k]);
    // float trig table padded by 128 entries (loads of a partial last chunk stay in bounds)
    g.trig_f.assign(2 * (static_cast<size_t>(d->n_angles) + 128), 0.0f);
    g.trig_d.resize(2 * static_cast<size_t>(d->n_angles));
    for (int j = 0; j < d->n_angles; ++j) {  // search.cpp:414-419
        const double sn = std::sin(d->angles[j]);
        const double cs = std::cos(d->angles[j]);
        g.trig_d[2 * j] = sn;
        g.trig_d[2 * j + 1] = cs;
        g.trig_f[2 * j] = static_cast<float>(sn * kInv500);
        g.trig_f[2 * j + 1] = static_cast<float>(cs * kInv200);
    }
    return g;
}

// Twin tiles: the grid maps onto itself under theta -> theta + pi,
// so candidate (k, m + na/2) is candidate (k, m) with its endpoints swapped.
// The reference's sin/cos of the twin angles are not exactly the negated ones;
// this bounds what that changes in the FP64 linear values (search.cpp:243-262)
// of every search of the plan: the derivative of a linear value in sin (cos) is
// M_c0 wx f^-1'(fx) r / 500 (M_c2 wz f^-1'(fz) r / 200), f^-1' <= max(3 u^2,
// 116 / kappa) for |u| <= the largest |fx| (|fz|), plus the FP64 rounding of
// both evaluations (< 2^-46 of the terms' magnitude).  Twins are used only
// when that is <= 2^-33; the emit widens its code bound by 2^-32 (kTwinSlack).
bool twin_grid(const std::vector<double>& trig_d, int na, const double* radii, int nr, const SearchConst* recs,
               size_t n_sc) {
    if (na < 2 || na % 2 != 0 || nr < 1) return false;
    const int h = na / 2;
    double ds = 0.0, dc = 0.0;
    for (int m = 0; m < h; ++m) {
        ds = std::max(ds, std::fabs(trig_d[2 * m] + trig_d[2 * (m + h)]));
        dc = std::max(dc, std::fabs(trig_d[2 * m + 1] + trig_d[2 * (m + h) + 1]));
    }
    if (!(ds <= 1e-12 && dc <= 1e-12)) return false;  // also NaN
    double rmax = 0.0;
    for (int k = 0; k < nr; ++k) rmax = std::max(rmax, std::fabs(radii[k]));
    double fy = 0.0, ta = 0.0, tb = 0.0, wx = 0.0, wz = 0.0, cy = 0.0;
    for (size_t u = 0; u < n_sc; ++u) {
        const SearchConst& r = recs[u];
        fy = std::max(fy, std::fabs(r.fy));
        ta = std::max(ta, std::fabs(r.ta));
        tb = std::max(tb, std::fabs(r.tb));
        wx = std::max(wx, std::fabs(r.wx));
        wz = std::max(wz, std::fabs(r.wz));
        for (int q = 0; q < 3; ++q) cy = std::max(cy, std::fabs(r.cy64[q]));
    }
    constexpr double kM = 3.25;  // >= every |kXyzToRgb| entry (convert_kernel.hpp:47)
    const double fxm = fy + (ta + rmax) / 500.0, fzm = fy + (tb + rmax) / 200.0;
    const double ls = kM * wx * std::max(3.0 * fxm * fxm, 0.13) * rmax / 500.0;
    const double lc = kM * wz * std::max(3.0 * fzm * fzm, 0.13) * rmax / 200.0;
    const double mag = kM * (wx * fxm * fxm * fxm + wz * fzm * fzm * fzm) + cy + 1.0;
    const double delta = 2.0 * (ls * ds + lc * dc) + std::ldexp(mag, -46);
    return std::isfinite(delta) && delta <= std::ldexp(1.0, -33);
}

int plan_build(cvg_ctx* ctx, const cvg_search_desc* d, cvg_plan* p, const GridTables* grid = nullptr,
               const SearchConst* pre = nullptr) {
    const double tb0 = now_ms();
    static const bool trace = std::getenv("CVG_TRACE") != nullptr;
    std::vector<std::pair<const char*, double>> tl;
    auto mark = [&](const char* w) {
        if (trace) tl.emplace_back(w, now_ms() - tb0);
    };
    struct TraceOut {
        std::vector<std::pair<const char*, double>>& tl;
        ~TraceOut() {
            if (tl.empty()) return;
            std::string line = "[cvg build]";
            for (auto& [w, t] : tl) line += std::string(" ") + w + "@" + std::to_string(t).substr(0, 6);
            std::fprintf(stderr, "%s\n", line.c_str());
        }
    } trace_out{tl};
    const Tables& T = tables();
    mark("tables");
    p->ctx = ctx;
    p->mode = search_mode(d);
    p->best = d->output == CVG_OUT_BEST;
    p->out = p->best ? CVG_OUT_PAIRS : d->output;  // BEST runs the PAIRS kernels, then best_kernel
    // pruning is a flag of the FAST path; so is memoization (distinct searches only)
    p->path = (d->path == CVG_PATH_PRUNED || d->path == CVG_PATH_MEMO) ? CVG_PATH_FAST : d->path;
    p->memo = d->path == CVG_PATH_MEMO && !pre;
    p->n = d->n_searches;
    p->nr = d->n_radii;
    p->na = d->n_angles;
    const uint64_t cps = static_cast<uint64_t>(p->nr) * static_cast<uint64_t>(p->na);
    p->candidates = cps * static_cast<uint64_t>(p->n);
    p->empty = p->candidates == 0;
    if (p->empty) return CVG_OK;  // search.cpp:409-411

    // Strip tiles (32 angles x up to 512 rows, lane per angle, uniform
    // radii) for COUNTS / FIRST on the band FAST path; a tile holds ~16K
    // candidates (cfg4: one whole 64 x 256 search).  Else row-major tiles of
    // kTile canonical candidates.  CVG_STRIPS=0 turns them off (A/B).
    static const int strips_env = [] {
        const char* e = std::getenv("CVG_STRIPS");
        return e ? std::atoi(e) : 1;
    }();
    // PAIRS (and BEST, on the PAIRS kernels) on strip tiles need canonical
    // tiles of whole strips within a 32-row block: n_angles % 32 == 0 and
    // either tiles of <= 32 whole rows (n_strips | 128, n_strips >= 4) or
    // rows of whole tiles (128 | n_strips)
    const bool pairs_out = d->output == CVG_OUT_PAIRS || d->output == CVG_OUT_BEST;
    const uint32_t n_strips = static_cast<uint32_t>((p->na + 31) / 32);
    const bool lists_ok = p->na % 32 == 0 && ((n_strips >= 4 && 128 % n_strips == 0) || n_strips % 128 == 0);
    const bool strips = strips_env != 0 && search_mode(d) == cvg::kModeBand &&
                        (d->path == CVG_PATH_FAST || d->path == CVG_PATH_MEMO) && (!pairs_out || lists_ok);
    // ~16K candidates per strip tile (a strip's set-up amortized over up to
    // 512 rows), made finer for small batches until there are claims for
    // every resident warp twice over (cfg0: one search of 256 x 1024)
    uint32_t strip_rows = static_cast<uint32_t>(std::min(p->nr, 512));  // 512: a multiple of 32
    uint32_t strips_per_tile = std::max<uint32_t>(1, 16384u / (32u * strip_rows));
    {
        const uint64_t want = 2ull * static_cast<uint64_t>(ctx->sms) * 32;
        auto claims = [&] {
            return static_cast<uint64_t>(p->n) * ((p->nr + strip_rows - 1) / strip_rows) *
                   ((n_strips + strips_per_tile - 1) / strips_per_tile);
        };
        while (claims() < want && (strips_per_tile > 1 || strip_rows > 32)) {
            if (strips_per_tile > 1) {
                strips_per_tile /= 2;
            } else {
                strip_rows = std::max<uint32_t>(32, (strip_rows / 2 + 31) / 32 * 32);
            }
        }
    }
    const uint32_t strip_tiles = (n_strips + strips_per_tile - 1) / strips_per_tile;
    const uint32_t tps = strips && !pairs_out
                             ? static_cast<uint32_t>((p->nr + strip_rows - 1) / strip_rows) * strip_tiles
                             : static_cast<uint32_t>((cps + cvg::kTile - 1) / cvg::kTile);
    const uint32_t claim_per_search =
        strips ? static_cast<uint32_t>((p->nr + strip_rows - 1) / strip_rows) * strip_tiles : tps;
    const uint32_t mask_rows = static_cast<uint32_t>((p->nr + 31) / 32 * 32);

    // ---- host tables ----
    // Per-search constants, deduplicated: searches with the same (target,
    // pattern, v_th, r_novib) share one record (per-pixel batches repeat
    // colors); every candidate of every search is still evaluated.
    // The records are built straight into the pinned staging block below.
    std::vector<uint32_t> sc_index;
    std::vector<int32_t> uniq;  // representative search of each record
    size_t n_sc = static_cast<size_t>(p->n);
    bool uniform = false;  // one classifier for the whole batch (one loud count: no claim groups)
    if (!pre) {
        uniform = dedup_searches(d, sc_index, uniq);
        n_sc = uniq.size();
    }
    mark("dedup");
    p->n_unique = static_cast<int32_t>(n_sc);
    if (p->memo && sc_index.empty()) p->memo = false;  // all distinct: nothing to memoize
    // the searches the kernels run: all of them, or (memo) one per record
    p->n_exec = p->memo ? static_cast<int32_t>(n_sc) : p->n;
    const uint64_t n_tiles = static_cast<uint64_t>(tps) * static_cast<uint64_t>(p->n_exec);
    const uint64_t n_claims = static_cast<uint64_t>(claim_per_search) * static_cast<uint64_t>(p->n_exec);
    if (n_tiles >= (1ull << 28)) return fail(CVG_EINVAL, "batch too large for one plan (split the searches)");
    auto exec_bits = [&](int32_t i) { return d->pattern_bits[p->memo ? uniq[i] : i] & 7; };
    GridTables own;
    if (!grid) {
        own = make_grid_tables(d);
        grid = &own;
    }
    const std::vector<float>& radii_f = grid->radii_f;
    const std::vector<float>& trig_f = grid->trig_f;
    const std::vector<double>& trig_d = grid->trig_d;
    mark("grid");

    // Claim order (band mode, more than one loud count in the batch): all
    // tiles of the searches with one loud count, then the next, so the warps
    // resident together run one band_row specialization (instruction cache).
    std::vector<uint32_t> claim;
    std::array<uint32_t, 3> group_end{};
    static const bool group_claims = [] {
        const char* e = std::getenv("CVG_CLAIM_GROUP");  // A/B switch; default on
        return !e || std::atoi(e) != 0;
    }();
    if (group_claims && p->mode == cvg::kModeBand && p->n_exec > 1 && !uniform) {
        std::array<uint32_t, 4> bucket{};
        for (int32_t i = 0; i < p->n_exec; ++i) ++bucket[__builtin_popcount(exec_bits(i))];
        int kinds = 0;
        for (uint32_t b : bucket) kinds += b > 0;
        if (kinds > 1) {
            // positions: loud count 1 first ([0, group_end[0])), then 2, then 3
            group_end[0] = bucket[1];
            group_end[1] = bucket[1] + bucket[2];
            group_end[2] = bucket[1] + bucket[2] + bucket[3];
            std::array<uint32_t, 4> next{0, 0, group_end[0], group_end[1]};
            claim.resize(p->n_exec);
            for (int32_t i = 0; i < p->n_exec; ++i) claim[next[__builtin_popcount(exec_bits(i))]++] = i;
        }
    }

    // ---- one constant blob: [sc | sc_index | claim | radii | trig | thresholds | code table] ----
    Layout L;
    const size_t o_sc = L.take(sizeof(SearchConst) * n_sc);
    const size_t o_si = L.take(sizeof(uint32_t) * sc_index.size());
    const size_t o_co = L.take(sizeof(uint32_t) * claim.size());
    const size_t o_rd = L.take(sizeof(double) * p->nr);
    const size_t o_rf = L.take(sizeof(float) * p->nr);
    const size_t o_td = L.take(sizeof(double) * trig_d.size());
    const size_t o_tf = L.take(sizeof(float) * trig_f.size());
    const size_t o_thd = L.take(sizeof(double) * 256);
    const size_t o_ctab = L.take(sizeof(T.ctab));
    const bool signal = p->mode == cvg::kModeSignal;
    const size_t o_stab = signal ? L.take(sizeof(T.stab)) : 0;
    const size_t o_bands = p->best ? L.take(sizeof(double) * 2 * p->n) : 0;
    const size_t o_sinv = strips ? L.take(sizeof(float) * 2 * n_strips) : 0;
    // COUNTS / FIRST strips walk the angles in order of decreasing |cos|
    // (lane slot j -> angle perm[j]): a strip's angles then reach the linear
    // branch of f^-1 at nearly the same radius, so fewer rows need the
    // general form (cfg4: 13% of the candidates instead of 19.5%).  PAIRS
    // strips keep the canonical order (their pass words are canonical).
    const bool permute = strips && !pairs_out;
    const size_t o_perm = permute ? L.take(sizeof(uint32_t) * 32 * n_strips) : 0;
    const size_t o_ptrig = permute ? L.take(sizeof(float) * 2 * 32 * n_strips) : 0;
    const size_t n_rgroups = static_cast<size_t>((p->nr + 3) / 4);
    const size_t o_rg = strips ? L.take(sizeof(float) * 12 * n_rgroups) : 0;
    const size_t bytes = L.off;
    p->input_bytes = bytes;
    p->t_prep_end = now_ms();
    unsigned char* stage = static_cast<unsigned char*>(ctx->host.alloc(bytes));
    p->d_const = ctx->dev.alloc(bytes);
    if (!stage || !p->d_const) {
        ctx->host.release(stage);
        return fail(CVG_ENOMEM, "allocation of the search tables failed");
    }
    p->stage = stage;  // released with the plan (also if a record throws below)
    mark("alloc");
    if (pre) {
        std::memcpy(stage + o_sc, pre, sizeof(SearchConst) * n_sc);
    } else {
        auto* recs = reinterpret_cast<SearchConst*>(stage + o_sc);
        const double rmax = d->radii[p->nr - 1];
        parallel_for(n_sc, [&](size_t u) { make_search_const(d, uniq[u], rmax, p->mode, T, recs[u]); }, 8);
    }
    mark("records");
    if (!sc_index.empty()) {
        const size_t m = sc_index.size(), parts = m >= (1u << 20) ? 16 : 1;
        parallel_for(
            parts,
            [&](size_t c) {
                const size_t lo = m * c / parts, hi = m * (c + 1) / parts;
                std::memcpy(stage + o_si + 4 * lo, sc_index.data() + lo, 4 * (hi - lo));
            },
            1);
    }
    if (!claim.empty()) std::memcpy(stage + o_co, claim.data(), sizeof(uint32_t) * claim.size());
    std::memcpy(stage + o_rd, d->radii, sizeof(double) * p->nr);
    std::memcpy(stage + o_rf, radii_f.data(), sizeof(float) * p->nr);
    std::memcpy(stage + o_td, trig_d.data(), sizeof(double) * trig_d.size());
    std::memcpy(stage + o_tf, trig_f.data(), sizeof(float) * trig_f.size());
    std::memcpy(stage + o_thd, T.thr, sizeof(double) * 256);
    std::memcpy(stage + o_ctab, T.ctab, sizeof(T.ctab));
    if (signal) std::memcpy(stage + o_stab, T.stab, sizeof(T.stab));
    if (strips) {
        // radius groups of 4 rows: r, r^2, r^3 of the double radii, each
        // rounded once to float (strip form); padded with the last radius
        auto* rg = reinterpret_cast<float*>(stage + o_rg);
        for (size_t j = 0; j < n_rgroups; ++j) {
            for (int i = 0; i < 4; ++i) {
                const double r = d->radii[std::min<size_t>(4 * j + i, static_cast<size_t>(p->nr - 1))];
                rg[12 * j + i] = static_cast<float>(r);
                rg[12 * j + 4 + i] = static_cast<float>(r * r);
                rg[12 * j + 8 + i] = static_cast<float>(r * r * r);
            }
        }
        // per strip of 32 angles: 1 / max |s'|, 1 / max |c'| over the float
        // trig values the kernel uses, rounded down (FLT_MAX for an all-zero
        // column: 0 * FLT_MAX stays 0 in the kernel's bound)
        std::vector<uint32_t> order(static_cast<size_t>(p->na));
        for (int m = 0; m < p->na; ++m) order[m] = static_cast<uint32_t>(m);
        if (permute) {
            std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
                return std::fabs(trig_f[2 * a + 1]) > std::fabs(trig_f[2 * b + 1]);
            });
            auto* perm = reinterpret_cast<uint32_t*>(stage + o_perm);
            auto* ptrig = reinterpret_cast<float*>(stage + o_ptrig);
            for (size_t j = 0; j < 32 * static_cast<size_t>(n_strips); ++j) {
                const uint32_t m = order[std::min<size_t>(j, order.size() - 1)];  // idle slots: a valid angle
                perm[j] = j < order.size() ? m : 0xffffffffu;
                ptrig[2 * j] = trig_f[2 * m];
                ptrig[2 * j + 1] = trig_f[2 * m + 1];
            }
        }
        auto* inv = reinterpret_cast<float*>(stage + o_sinv);
        for (uint32_t q = 0; q < n_strips; ++q) {
            float gs = 0.f, gc = 0.f;
            for (int j = 32 * static_cast<int>(q); j < std::min(p->na, 32 * static_cast<int>(q) + 32); ++j) {
                const uint32_t m = order[static_cast<size_t>(j)];
                gs = std::max(gs, std::fabs(trig_f[2 * m]));
                gc = std::max(gc, std::fabs(trig_f[2 * m + 1]));
            }
            for (int c = 0; c < 2; ++c) {
                const double g = c ? gc : gs;
                float v = g > 0 ? static_cast<float>(1.0 / g) : FLT_MAX;
                if (g > 0 && static_cast<double>(v) > 1.0 / g) v = std::nextafter(v, 0.0f);
                inv[2 * q + c] = std::min(v, FLT_MAX);
            }
        }
    }
    if (p->best) {
        // (v_th, low_band) per search for classification_margin (search.hpp:29-35: low = v_th * r_novib)
        auto* bands = reinterpret_cast<double*>(stage + o_bands);
        for (int32_t s = 0; s < p->n; ++s) {
            bands[2 * s] = d->v_th[s];
            bands[2 * s + 1] = d->v_th[s] * d->r_novib[s];
        }
        p->d_bands = at<const double>(p->d_const, o_bands);
    }
    LaunchArgs& A = p->args;
    std::memset(&A, 0, sizeof(A));
    A.sc = at<const SearchConst>(p->d_const, o_sc);
    A.sc_index = sc_index.empty() || p->memo ? nullptr : at<const uint32_t>(p->d_const, o_si);
    p->d_map = p->memo ? at<const uint32_t>(p->d_const, o_si) : nullptr;
    A.claim_order = claim.empty() ? nullptr : at<const uint32_t>(p->d_const, o_co);
    for (int g = 0; g < 3; ++g) A.group_end[g] = group_end[g];
    A.radii_d = at<const double>(p->d_const, o_rd);
    A.radii_f = at<const float>(p->d_const, o_rf);
    A.trig_d = at<const double>(p->d_const, o_td);
    A.trig_f = at<const float>(p->d_const, o_tf);
    A.thr_d = at<const double>(p->d_const, o_thd);
    A.ctab = at<const float>(p->d_const, o_ctab);
    A.stab = signal ? at<const float>(p->d_const, o_stab) : nullptr;
    // No sync: the staging block stays with the plan until it is released,
    // which happens after the stream has passed this copy.
    cudaError_t e = cudaMemcpyAsync(p->d_const, stage, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "upload of the search tables");
    p->t_upload_end = now_ms();
    mark("upload");

    for (int i = 0; i < 9; ++i) A.minv[i] = kXyzToRgb.m[i / 3][i % 3];
    A.n_searches = p->n_exec;
    A.nr = p->nr;
    A.na = p->na;
    A.aligned = (p->na % 32) == 0;
    A.tiles_per_search = tps;
    A.cand_per_search = static_cast<uint32_t>(cps);
    A.na_magic = p->na > 1 ? (UINT64_MAX / static_cast<uint64_t>(p->na)) + 1 : 0;
    A.emit_shift = 8;  // kEmitSpan until an expected pair count says otherwise (plan_set_density)
    A.prune = d->path == CVG_PATH_PRUNED ? 1u : 0u;
    A.strips = strips ? 1u : 0u;
    A.n_claims = static_cast<uint32_t>(n_claims);
    A.claim_per_search = claim_per_search;
    A.mask_rows = mask_rows;
    A.lst_rpt = strips && pairs_out && n_strips <= 128 ? 128u / n_strips : 0u;
    A.lst_tpr = strips && pairs_out && n_strips > 128 ? n_strips / 128u : 0u;
    A.lst_unit_rows = std::max<uint32_t>(8u, A.lst_rpt);
    A.strip_rows = strip_rows;
    A.strips_per_tile = strips_per_tile;
    A.strip_tiles = strip_tiles;
    A.strip_inv = strips ? at<const float>(p->d_const, o_sinv) : nullptr;
    A.strip_perm = permute ? at<const uint32_t>(p->d_const, o_perm) : nullptr;
    A.strip_trig = permute ? at<const float>(p->d_const, o_ptrig) : nullptr;
    A.radius_groups = strips ? at<const float>(p->d_const, o_rg) : nullptr;
    // Bulk skip of the inner rows of strip tiles (strip_run): COUNTS / FIRST
    // always; PAIRS on strips of 512 rows (cfg2: phase 1 + lists 1.86 ->
    // 1.49 ms), not on short strips (cfg1 / cfg3: its instantiation is 10-17%
    // slower there).  CVG_BULK_SKIP=0/1 forces it off / on (A/B).
    A.bulk_skip = [&] {
        if (const char* e = std::getenv("CVG_BULK_SKIP")) return static_cast<uint32_t>(std::atoi(e) != 0);
        return static_cast<uint32_t>(!pairs_out || strip_rows >= 512);
    }();
    A.n_tiles = n_tiles;

    // ---- per-run workspace --------------------------------------------------
    // zeroed each run:  status[n_scan_blocks] | tickets[8] | counts[n] | stats | total
    // written each run: tile_count[n_tiles] | tile_base[n_tiles] | worklist   (PAIRS)
    const bool pairs = p->out == cvg::kOutPairs;
    const int per_sm = cvg::search_blocks_per_sm(p->mode, p->out, p->path);
    if (per_sm <= 0) {
        cudaError_t le = cudaGetLastError();
        return fail(CVG_ECUDA, std::string("search kernel cannot be resident on this device (") +
                                   cudaGetErrorString(le) + "); sm_100a image required");
    }
    const uint64_t scan_blocks = pairs ? (n_tiles + cvg::kScanTile - 1) / cvg::kScanTile : 0;
    Layout W;
    const size_t o_st = W.take(sizeof(unsigned long long) * scan_blocks);
    const size_t o_tk = W.take(sizeof(unsigned int) * 8);
    const size_t o_ct = W.take(sizeof(unsigned long long) * p->n_exec);
    const size_t o_ss = W.take(sizeof(cvg::Stats));
    const size_t o_to = W.take(sizeof(unsigned long long));  // stats+total read back as one ChunkTail
    p->work_bytes = W.off;  // memset span
    const size_t o_tc = W.take(sizeof(uint32_t) * (pairs ? n_tiles : 0));
    const size_t o_tb = W.take(sizeof(unsigned long long) * (pairs ? n_tiles : 0));
    const size_t o_wl = W.take(sizeof(uint32_t) * (pairs ? n_tiles * (cvg::kTile / cvg::kEmitSpan) : 0));
    const size_t o_bk = W.take(p->best ? sizeof(unsigned long long) * 2 * n_tiles : 0);  // written each run
    // Twin tiles: PAIRS strip plans whose rows hold an even number of whole
    // tiles, on a grid twin_grid proves symmetric.  CVG_TWIN=0 turns them off
    // (A/B); CVG_TWIN_SPLIT_TEST=1 builds both lists of every odd row (tests).
    const int twin_env = [] {
        const char* e = std::getenv("CVG_TWIN");
        return e ? std::atoi(e) : 1;
    }();
    const bool twin = pairs && strips && twin_env != 0 && A.lst_tpr >= 2 && A.lst_tpr % 2 == 0 &&
                      A.lst_unit_rows == 8 &&
                      twin_grid(trig_d, p->na, d->radii, p->nr, at<const SearchConst>(stage, o_sc), n_sc);
    const size_t o_tw = W.take(twin ? n_tiles : 0);
    p->d_work = ctx->dev.alloc(W.off);
    if (!p->d_work) return fail(CVG_ENOMEM, "device allocation of the workspace failed");
    A.status = at<unsigned long long>(p->d_work, o_st);
    A.ticket = at<unsigned int>(p->d_work, o_tk);
    A.counts = at<unsigned long long>(p->d_work, o_ct);
    A.stats = at<cvg::Stats>(p->d_work, o_ss);
    A.tile_count = at<uint32_t>(p->d_work, o_tc);
    A.tile_base = at<unsigned long long>(p->d_work, o_tb);
    A.total = at<unsigned long long>(p->d_work, o_to);
    A.best_key = p->best ? at<unsigned long long>(p->d_work, o_bk) : nullptr;
    A.worklist = at<uint32_t>(p->d_work, o_wl);
    A.twin = twin ? at<uint8_t>(p->d_work, o_tw) : nullptr;
    A.twin_tiles = twin ? A.lst_tpr / 2 : 0u;
    A.twin_m = twin ? static_cast<uint32_t>(p->na / 2) : 0u;
    A.twin_split_test = [] {
        const char* e = std::getenv("CVG_TWIN_SPLIT_TEST");
        return e && std::atoi(e) != 0 ? 1u : 0u;
    }();
    p->twin = twin;
    A.search_begin = 0;
    A.range_searches = static_cast<uint32_t>(p->n_exec);
    A.tile_begin = 0;
    A.base_offset = nullptr;
    A.grand_total = nullptr;
    if (pairs) {
        p->d_scratch = ctx->dev.alloc(static_cast<size_t>(n_tiles) * cvg::kTile * sizeof(uint16_t));
        if (!p->d_scratch) return fail(CVG_ENOMEM, "device allocation of the tile lists failed");
        A.scratch = static_cast<uint16_t*>(p->d_scratch);
        if (strips) {  // pass words of the strip tiles (every word is written each run)
            p->d_masks = ctx->dev.alloc(static_cast<size_t>(p->n_exec) * n_strips * mask_rows * sizeof(uint32_t));
            if (!p->d_masks) return fail(CVG_ENOMEM, "device allocation of the pass masks failed");
            A.masks = static_cast<uint32_t*>(p->d_masks);
        }
    }
    if (p->out == cvg::kOutFirst || p->best) {
        Layout F;
        const size_t o_fi = F.take(sizeof(uint32_t) * p->n_exec);
        const size_t o_fc = F.take(static_cast<size_t>(p->n_exec) * 6);
        p->first_bytes = F.off;
        p->d_first = ctx->dev.alloc(p->first_bytes);
        if (!p->d_first) return fail(CVG_ENOMEM, "device allocation of the first-pair buffer failed");
        A.first_idx = at<uint32_t>(p->d_first, o_fi);
        A.first_codes = at<uint8_t>(p->d_first, o_fc);
    }
    p->res_counts = A.counts;
    p->res_first_idx = A.first_idx;
    p->res_first_codes = A.first_codes;
    if (p->memo) {
        // every search's result, scattered from its record's
        Layout M;
        const size_t o_mc = M.take(sizeof(unsigned long long) * p->n);
        const bool first = p->out == cvg::kOutFirst;
        const size_t o_mi = M.take(first ? sizeof(uint32_t) * p->n : 0);
        const size_t o_mf = M.take(first ? static_cast<size_t>(p->n) * 6 : 0);
        p->d_memo = ctx->dev.alloc(M.off);
        if (!p->d_memo) return fail(CVG_ENOMEM, "device allocation of the memoized results failed");
        p->res_counts = at<unsigned long long>(p->d_memo, o_mc);
        p->res_first_idx = first ? at<uint32_t>(p->d_memo, o_mi) : nullptr;
        p->res_first_codes = first ? at<uint8_t>(p->d_memo, o_mf) : nullptr;
    }

    const uint64_t want = (n_claims + cvg::kWarpsPerBlock - 1) / cvg::kWarpsPerBlock;
    static const int cap_per_sm = [] {
        const char* e = std::getenv("CVG_BLOCKS_PER_SM");  // tuning override (occupancy experiments)
        return e ? std::atoi(e) : 0;
    }();
    const int use_per_sm = cap_per_sm > 0 ? std::min(cap_per_sm, per_sm) : per_sm;
    p->grid = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(use_per_sm) * ctx->sms, want));
    if (p->grid < 1) p->grid = 1;
    for (cudaEvent_t* ev : {&p->ev0, &p->ev1, &p->marks[0], &p->marks[1], &p->marks[2], &p->marks[3]}) {
        if (!ctx->events.empty()) {
            *ev = ctx->events.back();
            ctx->events.pop_back();
        } else {
            CVG_CUDA(cudaEventCreate(ev));
        }
    }

    mark("workspace");
    if (p->out == cvg::kOutPairs && !p->external_out) {
        // Initial capacity: every candidate when it fits in half the free memory.
        const uint64_t fit = static_cast<uint64_t>(ctx->total_mem / 4 / 10);  // a quarter of HBM at most
        uint64_t cap = std::min<uint64_t>(p->candidates, std::max<uint64_t>(fit, 1u << 20));
        if (int e2 = plan_reserve(p, cap)) return e2;
    }
    return CVG_OK;
}

int plan_build_safe(cvg_ctx* ctx, const cvg_search_desc* d, cvg_plan* p, const GridTables* grid,
                    const SearchConst* pre) {
    try {
        return plan_build(ctx, d, p, grid, pre);
    } catch (const std::bad_alloc&) {
        return fail(CVG_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(CVG_EUNSUPPORTED, e.what());
    }
}

void plan_release(cvg_plan* p) {
    if (!p->ctx) return;
    if (p->ran && !p->empty && p->ev1) cudaEventSynchronize(p->ev1);  // buffers go back to the pool
    plan_free_outputs(p);
    p->ctx->dev.release(p->d_const);
    p->ctx->dev.release(p->d_work);
    p->ctx->dev.release(p->d_first);
    p->ctx->dev.release(p->d_scratch);
    p->ctx->dev.release(p->d_memo);
    p->d_memo = nullptr;
    p->ctx->dev.release(p->d_masks);
    p->d_masks = nullptr;
    if (p->stage) cudaStreamSynchronize(p->ctx->stream);  // the constant upload may still be in flight
    for (cudaEvent_t* ev : {&p->ev0, &p->ev1, &p->marks[0], &p->marks[1], &p->marks[2], &p->marks[3]}) {
        if (*ev) p->ctx->events.push_back(*ev);
        *ev = nullptr;
    }
    p->ctx->host.release(p->stage);
    p->stage = nullptr;
    p->ctx->host.release(p->h_counts);
    p->h_counts = nullptr;
}

int plan_enqueue(cvg_plan* p, cudaStream_t st) {
    p->last_stream = st;
    p->ran = true;
    if (p->empty) return CVG_OK;
    CVG_CUDA(cudaMemsetAsync(p->d_work, 0, p->work_bytes, st));
    if (p->out == cvg::kOutFirst) CVG_CUDA(cudaMemsetAsync(p->d_first, 0xff, static_cast<size_t>(p->n_exec) * 4, st));
    CVG_CUDA(cudaEventRecord(p->ev0, st));
    p->marked = p->phase_marks;
    CVG_CUDA(cvg::launch_search(p->args, p->mode, p->out, p->path, p->grid, st, p->marked ? p->marks : nullptr));
    if (p->out == cvg::kOutFirst) CVG_CUDA(cvg::launch_first_codes(p->args, st));
    if (p->best) CVG_CUDA(cvg::launch_best(p->args, p->d_bands, st));
    if (p->memo) {
        const bool first = p->out == cvg::kOutFirst;
        CVG_CUDA(cvg::launch_scatter(p->d_map, p->n, p->args.counts, first ? p->args.first_idx : nullptr,
                                     first ? p->args.first_codes : nullptr, p->res_counts, p->res_first_idx,
                                     p->res_first_codes, st));
    }
    CVG_CUDA(cudaEventRecord(p->ev1, st));
    return CVG_OK;
}

int plan_collect(cvg_plan* p, uint64_t* counts, HostStats& hs) {
    if (p->empty) {
        if (p->n) std::memset(counts, 0, sizeof(uint64_t) * p->n);
        return CVG_OK;
    }
    cudaStream_t st = p->last_stream;
    CVG_CUDA(cudaMemcpyAsync(counts, p->res_counts, sizeof(uint64_t) * p->n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaMemcpyAsync(&hs.st, p->args.stats, sizeof(cvg::Stats), cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    CVG_CUDA(cudaEventElapsedTime(&hs.ms, p->ev0, p->ev1));
    return CVG_OK;
}

uint64_t sum_counts(const uint64_t* c, size_t n) {
    const size_t parts = n >= (1u << 20) ? 16 : 1;
    std::vector<uint64_t> part(parts, 0);
    parallel_for(
        parts,
        [&](size_t k) {
            uint64_t acc = 0;
            for (size_t i = n * k / parts; i < n * (k + 1) / parts; ++i) acc += c[i];
            part[k] = acc;
        },
        1);
    uint64_t t = 0;
    for (uint64_t v : part) t += v;
    return t;
}

void result_zero(cvg_result* r) { std::memset(r, 0, sizeof(*r)); }

int undecided_fail(unsigned long long n) {
    return fail(CVG_EUNDECIDED, std::to_string(n) +
                                    " continuous FrameDiff decision(s) lie within the device/glibc pow error "
                                    "margin of a threshold; the device cannot prove the reference's result");
}

int plan_fetch_impl(cvg_plan* p, cvg_result* r, bool allow_rerun) {
    result_zero(r);
    r->n_searches = p->n;
    cvg_ctx* ctx = p->ctx;
    const size_t n = static_cast<size_t>(p->n);
    // counts land straight in the pinned block that becomes r->counts
    r->counts = static_cast<uint64_t*>(ctx->host.alloc(sizeof(uint64_t) * (n ? n : 1)));
    if (!r->counts) return fail(CVG_ENOMEM, "pinned host allocation failed");
    HostStats hs;
    if (int e = plan_collect(p, r->counts, hs)) return e;
    const double t_counts = now_ms();
    const uint64_t total = sum_counts(r->counts, n);
    if (hs.st.undecided) return undecided_fail(hs.st.undecided);
    if (p->out == cvg::kOutPairs && hs.st.overflow) {
        if (!allow_rerun) {
            r->n_pairs = total;
            return fail(CVG_EOVERFLOW, "pair buffer too small; call cvg_plan_reserve and rerun");
        }
        if (int e = plan_reserve(p, total)) return e;
        if (int e = plan_enqueue(p, p->last_stream)) return e;
        ctx->host.release(r->counts);
        return plan_fetch_impl(p, r, false);
    }
    r->n_pairs = total;
    r->n_candidates = p->candidates;
    r->n_band_repairs = hs.st.band_repairs;
    r->n_code_repairs = hs.st.code_repairs;
    r->n_audit_violations = hs.st.audit_violations;
    r->n_class_mismatch = hs.st.class_mismatch;
    std::memcpy(&r->audit_max_ratio, &hs.st.audit_max_ratio_bits, sizeof(float));
    r->kernel_ms = hs.ms;
    r->h2d_bytes = p->input_bytes;
    r->d2h_bytes = sizeof(uint64_t) * n + sizeof(cvg::Stats);
    if (p->out == cvg::kOutPairs && !p->best) {
        r->d2h_bytes += total * 10;
        r->offsets = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (n + 1)));
        if (!r->offsets) return fail(CVG_ENOMEM, "host allocation failed");
        r->offsets[0] = 0;
        for (size_t s = 0; s < n; ++s) r->offsets[s + 1] = r->offsets[s] + r->counts[s];
        if (total) {
            r->idx = static_cast<uint32_t*>(ctx->host.alloc(total * 4));
            r->codes = static_cast<uint8_t*>(ctx->host.alloc(total * 6));
            if (!r->idx || !r->codes) return fail(CVG_ENOMEM, "pinned host allocation failed");
            cudaStream_t st = p->last_stream;
            CVG_CUDA(cudaMemcpyAsync(r->idx, p->d_out_idx, total * 4, cudaMemcpyDeviceToHost, st));
            CVG_CUDA(cudaMemcpyAsync(r->codes, p->d_out_codes, total * 6, cudaMemcpyDeviceToHost, st));
            CVG_CUDA(cudaStreamSynchronize(st));
        }
        r->d2h_ms = static_cast<float>(now_ms() - t_counts);
    } else if ((p->out == cvg::kOutFirst || p->best) && n) {
        r->d2h_bytes += n * 10;
        r->first_idx = static_cast<uint32_t*>(ctx->host.alloc(n * 4));
        r->first_codes = static_cast<uint8_t*>(ctx->host.alloc(n * 6));
        if (!r->first_idx || !r->first_codes) return fail(CVG_ENOMEM, "pinned host allocation failed");
        cudaStream_t st = p->last_stream;
        CVG_CUDA(cudaMemcpyAsync(r->first_idx, p->res_first_idx, n * 4, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaMemcpyAsync(r->first_codes, p->res_first_codes, n * 6, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaStreamSynchronize(st));
    }
    return CVG_OK;
}

// cvg_result keeps a pointer to its context in a side table so that
// cvg_result_free can return pinned blocks to the right pool.  A result may
// outlive its context: cvg_destroy detaches the blocks still held by results
// (owner nullptr) and cvg_result_free then releases them with cudaFreeHost.
std::mutex g_owner_mu;
std::map<const void*, cvg_ctx*> g_owner;

void remember_owner(cvg_result* r, cvg_ctx* ctx) {
    std::lock_guard<std::mutex> lk(g_owner_mu);
    for (const void* ptr : {static_cast<const void*>(r->counts), static_cast<const void*>(r->idx),
                            static_cast<const void*>(r->codes),
                            static_cast<const void*>(r->first_idx), static_cast<const void*>(r->first_codes)}) {
        if (ptr) g_owner[ptr] = ctx;
    }
}

}  // namespace cvg::host

// ============================================================================
// C-ABI
// ============================================================================

using namespace cvg::host;

extern "C" {

const char* cvg_last_error(void) { return g_error.c_str(); }
const char* cvg_version(void) { return "colorvibe-b200 0.1.0 (sm_100a)"; }

int cvg_create(int device, cvg_ctx** out) {
    if (!out) return fail(CVG_EINVAL, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(CVG_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    }
    if (device < 0 || device >= count) return fail(CVG_EINVAL, "device index out of range");
    auto* ctx = new cvg_ctx();
    ctx->device = device;
    ctx->dev.device = true;
    ctx->host.device = false;
    e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->tail_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        size_t free_b = 0;
        e = cudaMemGetInfo(&free_b, &ctx->total_mem);
    }
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "context creation");
    }
    (void)tables();
    *out = ctx;
    return CVG_OK;
}

void cvg_destroy(cvg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    {
        // results still alive keep their pinned blocks (they outlive the pool)
        std::lock_guard<std::mutex> lk(g_owner_mu);
        for (auto& kv : g_owner) {
            if (kv.second == ctx && ctx->host.detach(const_cast<void*>(kv.first))) kv.second = nullptr;
        }
    }
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamSynchronize(ctx->tail_stream);
    cudaStreamSynchronize(ctx->aux_stream);
    layout_free(ctx->codec_layout);
    for (cudaEvent_t ev : ctx->events) cudaEventDestroy(ev);
    cudaStreamDestroy(ctx->stream);
    cudaStreamDestroy(ctx->copy_stream);
    cudaStreamDestroy(ctx->tail_stream);
    cudaStreamDestroy(ctx->aux_stream);
    delete ctx;
}

int cvg_plan_create(cvg_ctx* ctx, const cvg_search_desc* desc, cvg_plan** out) {
    if (!ctx || !out) return fail(CVG_EINVAL, "null context or output pointer");
    *out = nullptr;
    if (int e = validate_desc(desc)) return e;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    if (int e = ensure_device(ctx)) return e;
    auto* p = new cvg_plan();
    if (int e = plan_build_safe(ctx, desc, p)) {
        plan_release(p);
        delete p;
        return e;
    }
    *out = p;
    return CVG_OK;
}

void cvg_plan_destroy(cvg_plan* p) {
    if (!p) return;
    if (p->ctx) {
        std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
        cudaSetDevice(p->ctx->device);
        if (p->ran) cudaStreamSynchronize(p->last_stream);
        plan_release(p);
    }
    delete p;
}

int cvg_plan_reserve(cvg_plan* p, uint64_t cap) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    plan_set_density(p, cap);  // the caller's expected pair count
    return plan_reserve(p, cap);
}

int cvg_plan_run(cvg_plan* p, void* stream) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    return plan_enqueue(p, static_cast<cudaStream_t>(stream));
}

int cvg_plan_sync(cvg_plan* p, uint64_t* n_pairs) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    if (!p->h_counts) {
        p->h_counts = static_cast<uint64_t*>(p->ctx->host.alloc(sizeof(uint64_t) * (p->n ? p->n : 1)));
        if (!p->h_counts) return fail(CVG_ENOMEM, "pinned host allocation failed");
    }
    HostStats hs;
    if (int e = plan_collect(p, p->h_counts, hs)) return e;
    const uint64_t total = sum_counts(p->h_counts, static_cast<size_t>(p->n));
    if (n_pairs) *n_pairs = total;
    if (hs.st.undecided) return undecided_fail(hs.st.undecided);
    if (p->out == cvg::kOutPairs && hs.st.overflow) return fail(CVG_EOVERFLOW, "pair buffer too small");
    return CVG_OK;
}

int cvg_plan_fetch(cvg_plan* p, cvg_result* out) {
    if (!p || !out) return fail(CVG_EINVAL, "null plan or result");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    const int e = plan_fetch_impl(p, out, false);
    remember_owner(out, p->ctx);
    if (e) cvg_result_free(out);
    return e;
}

int cvg_plan_copy_outputs(cvg_plan* p, uint64_t* counts, uint32_t* idx, uint8_t* codes, uint64_t n_pairs,
                          void* stream) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    if (p->empty) return CVG_OK;
    if ((idx || codes) && (p->out != cvg::kOutPairs || n_pairs > p->capacity)) {
        return fail(CVG_EINVAL, "n_pairs exceeds the plan's pair buffer (or not a PAIRS plan)");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (counts) {
        CVG_CUDA(cudaMemcpyAsync(counts, p->res_counts, sizeof(uint64_t) * p->n, cudaMemcpyDeviceToDevice, st));
    }
    if (idx && n_pairs) CVG_CUDA(cudaMemcpyAsync(idx, p->d_out_idx, 4 * n_pairs, cudaMemcpyDeviceToDevice, st));
    if (codes && n_pairs) CVG_CUDA(cudaMemcpyAsync(codes, p->d_out_codes, 6 * n_pairs, cudaMemcpyDeviceToDevice, st));
    return CVG_OK;
}

int cvg_plan_device_outputs(cvg_plan* p, uint64_t** counts, uint32_t** idx, uint8_t** codes, uint64_t* capacity) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    if (counts) *counts = reinterpret_cast<uint64_t*>(p->res_counts);
    if (idx) *idx = static_cast<uint32_t*>(p->d_out_idx);
    if (codes) *codes = static_cast<uint8_t*>(p->d_out_codes);
    if (capacity) *capacity = p->capacity;
    return CVG_OK;
}

int cvg_plan_last_kernel_ms(cvg_plan* p, float* ms) {
    if (!p || !ms) return fail(CVG_EINVAL, "null plan or output");
    *ms = 0.f;
    if (p->empty || !p->ran) return CVG_OK;
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    CVG_CUDA(cudaEventSynchronize(p->ev1));
    CVG_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
    return CVG_OK;
}

uint64_t cvg_plan_input_bytes(const cvg_plan* p) { return p ? p->input_bytes : 0; }

int32_t cvg_plan_evaluated_searches(const cvg_plan* p) { return p ? (p->empty ? 0 : p->n_exec) : 0; }

int cvg_plan_twin_tiles(const cvg_plan* p) { return p && p->twin ? 1 : 0; }

int cvg_plan_copy_first(cvg_plan* p, uint32_t* first_idx, uint8_t* first_codes, void* stream) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    if (p->out != cvg::kOutFirst && !p->best) return fail(CVG_EINVAL, "not a FIRST / BEST plan");
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (int e = ensure_device(p->ctx)) return e;
    if (p->empty || !p->n) return CVG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = static_cast<size_t>(p->n);
    if (first_idx) CVG_CUDA(cudaMemcpyAsync(first_idx, p->res_first_idx, 4 * n, cudaMemcpyDeviceToDevice, st));
    if (first_codes) CVG_CUDA(cudaMemcpyAsync(first_codes, p->res_first_codes, 6 * n, cudaMemcpyDeviceToDevice, st));
    return CVG_OK;
}

int cvg_plan_last_phase_ms(cvg_plan* p, float* phase1_ms, float* scan_ms, float* emit_ms) {
    if (!p || !phase1_ms || !scan_ms || !emit_ms) return fail(CVG_EINVAL, "null plan or output");
    *phase1_ms = *scan_ms = *emit_ms = 0.f;
    if (p->empty || !p->ran) return CVG_OK;
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    CVG_CUDA(cudaEventSynchronize(p->ev1));
    if (p->out != cvg::kOutPairs) return cudaEventElapsedTime(phase1_ms, p->ev0, p->ev1) == cudaSuccess
                                             ? CVG_OK : fail(CVG_ECUDA, "event timing failed");
    if (!p->marked) return fail(CVG_EINVAL, "the last run recorded no phase marks (cvg_plan_set_phase_marks)");
    CVG_CUDA(cudaEventElapsedTime(phase1_ms, p->ev0, p->marks[0]));
    CVG_CUDA(cudaEventElapsedTime(scan_ms, p->marks[0], p->marks[1]));
    CVG_CUDA(cudaEventElapsedTime(emit_ms, p->marks[1], p->ev1));
    return CVG_OK;
}

int cvg_plan_set_phase_marks(cvg_plan* p, int on) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    p->phase_marks = on != 0;
    return CVG_OK;
}

int cvg_plan_launches(const cvg_plan* p) {
    if (!p || p->empty) return 0;
    // phase 1 [+ tile lists (strip plans) + scan + emit] [+ first codes] [+ best: tile pass + search pass] [+ memo scatter]
    const int pairs = p->out == cvg::kOutPairs ? (p->args.masks ? 4 : 3) : 0;
    return (pairs ? pairs : p->out == cvg::kOutFirst ? 2 : 1) + (p->best ? 2 : 0) + (p->memo ? 1 : 0);
}

uint64_t cvg_plan_candidates(const cvg_plan* p) { return p ? p->candidates : 0; }

int cvg_validate(const cvg_search_desc* desc) { return validate_desc(desc); }

void cvg_result_free(cvg_result* r) {
    if (!r) return;
    std::free(r->offsets);
    for (void* ptr : {static_cast<void*>(r->counts), static_cast<void*>(r->idx), static_cast<void*>(r->codes), static_cast<void*>(r->first_idx),
                      static_cast<void*>(r->first_codes)}) {
        if (!ptr) continue;
        cvg_ctx* owner = nullptr;
        bool orphan = false;
        {
            std::lock_guard<std::mutex> lk(g_owner_mu);
            auto it = g_owner.find(ptr);
            if (it != g_owner.end()) {
                owner = it->second;
                orphan = owner == nullptr;
                g_owner.erase(it);
            }
        }
        if (orphan) {
            cudaFreeHost(ptr);  // its context was destroyed first
        } else if (owner) {
            std::lock_guard<std::recursive_mutex> lk(owner->mu);
            owner->host.release(ptr);
        }
    }
    std::memset(r, 0, sizeof(*r));
}

int cvg_srgb_to_lab(const int32_t rgb[3], const double* wp, double lab[3]) {
    if (!rgb || !lab) return fail(CVG_EINVAL, "null argument");
    if (int e = validate_color(rgb)) return e;
    to_lab(rgb, white_or_d65(wp), lab);
    return CVG_OK;
}

static int validate_lab(const double lab[3]) {
    if (!(std::isfinite(lab[0]) && std::isfinite(lab[1]) && std::isfinite(lab[2])) || lab[0] < 0.0 || lab[0] > 100.0) {
        return fail(CVG_EINVAL, "Lab color with L* outside [0, 100]");
    }
    return CVG_OK;
}

int cvg_lab_to_srgb_clipped(const double lab[3], const double* wp, int32_t rgb[3]) {
    if (!rgb || !lab) return fail(CVG_EINVAL, "null argument");
    if (int e = validate_lab(lab)) return e;
    double lin[3];
    to_linear(lab, white_or_d65(wp), lin);
    for (int c = 0; c < 3; ++c) rgb[c] = quantize(lin[c]);
    return CVG_OK;
}

int cvg_lab_to_srgb(const double lab[3], const double* wp, int32_t rgb[3]) {
    if (!rgb || !lab) return -fail(CVG_EINVAL, "null argument");
    if (validate_lab(lab)) return -CVG_EINVAL;
    double lin[3];
    to_linear(lab, white_or_d65(wp), lin);
    for (int c = 0; c < 3; ++c) {
        if (!(lin[c] >= -kGamutEps && lin[c] <= 1.0 + kGamutEps)) return 0;
    }
    for (int c = 0; c < 3; ++c) rgb[c] = quantize(lin[c]);
    return 1;
}

int cvg_pair_eval(const double lab[3], double radius, double angle, const double* wp, int32_t sp[3], int32_t sm[3],
                  double gp[3], double gm[3]) {
    if (!lab || !sp || !sm || !gp || !gm) return fail(CVG_EINVAL, "null argument");
    // displaced_pair (search.cpp:113-123) -> lab_to_linear (convert_kernel.hpp:
    // 94-105) -> quantize_signal / signal_value (:109-117), per candidate
    const double da = radius * std::sin(angle);
    const double db = radius * std::cos(angle);
    const double plus[3] = {lab[0], lab[1] + da, lab[2] + db};
    const double minus[3] = {lab[0], lab[1] - da, lab[2] - db};
    double lp[3], lm[3];
    to_linear(plus, white_or_d65(wp), lp);
    to_linear(minus, white_or_d65(wp), lm);
    for (int c = 0; c < 3; ++c) {
        sp[c] = quantize(lp[c]);
        sm[c] = quantize(lm[c]);
        gp[c] = signal_value(lp[c]);
        gm[c] = signal_value(lm[c]);
    }
    return CVG_OK;
}

int cvg_pair_signal(const double lab[3], double radius, double angle, const double* wp, double sp[3],
                    double sm[3]) {
    if (!lab || !sp || !sm) return fail(CVG_EINVAL, "null argument");
    if (int e = validate_lab(lab)) return e;
    // displaced_pair (search.cpp:113-123) -> lab_to_linear -> signal_value
    const double da = radius * std::sin(angle);
    const double db = radius * std::cos(angle);
    const double plus[3] = {lab[0], lab[1] + da, lab[2] + db};
    const double minus[3] = {lab[0], lab[1] - da, lab[2] - db};
    double lp[3], lm[3];
    to_linear(plus, white_or_d65(wp), lp);
    to_linear(minus, white_or_d65(wp), lm);
    for (int c = 0; c < 3; ++c) {
        sp[c] = signal_value(lp[c]);
        sm[c] = signal_value(lm[c]);
    }
    return CVG_OK;
}

void cvg_d65_white(double out[3]) {
    const double* w = white_or_d65(nullptr);
    out[0] = w[0];
    out[1] = w[1];
    out[2] = w[2];
}

void cvg_quant_thresholds(double out[256]) { std::memcpy(out, tables().thr, sizeof(double) * 256); }
void cvg_code_table(float out[8194]) { std::memcpy(out, tables().ctab, sizeof(tables().ctab)); }
void cvg_signal_table(float out[8194]) { std::memcpy(out, tables().stab, sizeof(tables().stab)); }
float cvg_code_slack(void) { return cvg::kCodeSlack; }

double cvg_measure_ffma_peak(int device, float* ms_out) { return cvg::measure_ffma_peak(device, ms_out); }

}  // extern "C"
