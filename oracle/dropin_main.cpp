// dropin_main.cpp -- TEST INFRASTRUCTURE ONLY (C++ drop-in check).
//
// One driver, built twice by oracle/Makefile from the reference's own,
// unmodified callers of the hot path -- src/feasibility.cpp (sweep,
// feasibility.cpp:261-292), src/bench.cpp (run_benchmark / sweep,
// bench.cpp:18-34, 84-85, 104), src/codec.cpp (embed_blocks,
// codec.cpp:80-81) and src/util.cpp -- compiled where they lie:
//
//   _ref/dropin_gpu  against include/colorvibe/*.hpp, the search and color
//                    API resolved from libcolorvibe_gpu.so (the swap
//                    INTEGRATION.md section 1 describes);
//   _ref/dropin_ref  against the reference headers with the reference's own
//                    src/color.cpp + src/search.cpp (CPU).
//
// Both print the same report (tests/test_dropin.py compares them line by
// line): the reference test_search.cpp:177-255 cases, the feasibility
// matrix exports, run_benchmark's pair total and parity flag, and the codec
// frames/decode of a test card and a multi-block layout.  image.cpp needs
// libpng and is not compiled; the one Image member the codec calls,
// Image::solid, comes from libcolorvibe_gpu.so (GPU build) or is restated
// from its declaration below (CPU build).

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "colorvibe/bench.hpp"
#include "colorvibe/codec.hpp"
#include "colorvibe/feasibility.hpp"
#include "colorvibe/search.hpp"

using namespace colorvibe;

#ifdef DROPIN_REF
namespace colorvibe {
Image Image::solid(int width, int height, const SrgbColor& fill) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("image dimensions must be positive");
    validate(fill);
    Image img;
    img.width = width;
    img.height = height;
    img.pixels.resize(3 * static_cast<std::size_t>(width) * height);
    for (std::size_t i = 0; i < img.pixels.size(); i += 3) {
        img.pixels[i] = static_cast<std::uint8_t>(fill.r);
        img.pixels[i + 1] = static_cast<std::uint8_t>(fill.g);
        img.pixels[i + 2] = static_cast<std::uint8_t>(fill.b);
    }
    return img;
}
}  // namespace colorvibe
#endif

namespace {

uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}

uint64_t hash_pairs(const std::vector<ColorPair>& v) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const auto& p : v) {
        const int c[9] = {p.target.r, p.target.g, p.target.b, p.plus.r, p.plus.g, p.plus.b,
                          p.minus.r, p.minus.g, p.minus.b};
        const double d[5] = {p.radius, p.angle, p.deltas.dr, p.deltas.dg, p.deltas.db};
        h = fnv(h, c, sizeof(c));
        h = fnv(h, d, sizeof(d));
    }
    return h;
}

uint64_t hash_image(const Image& img) { return fnv(0xcbf29ce484222325ull, img.pixels.data(), img.pixels.size()); }

VibrationGrid small_grid() { return VibrationGrid::uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0); }

}  // namespace

int main() {
    // ---- test_search.cpp:177-201: serial == batch, every mode and basis ----
    const VibrationGrid grid = small_grid();
    const SrgbColor targets[] = {{170, 170, 170}, {240, 240, 240}, {100, 100, 240}, {240, 100, 240}};
    const char* patterns[] = {"100", "001", "101", "110", "111"};
    const Thresholds ths[] = {{50.0, 0.5}, {100.0, 0.25}, {150.0, 0.125}};
    int agree = 0, cases = 0;
    for (const auto& t : targets) {
        for (const char* ps : patterns) {
            const BitPattern pat = BitPattern::parse(ps);
            for (const auto& th : ths) {
                for (DeltaMode mode : {DeltaMode::Quantized, DeltaMode::Continuous}) {
                    for (DeltaBasis basis : {DeltaBasis::TargetSwing, DeltaBasis::FrameDiff}) {
                        SearchOptions opts;
                        opts.delta_mode = mode;
                        opts.delta_basis = basis;
                        const auto s = serial_search(t, grid, pat, th, opts);
                        const auto b = batch_search(t, grid, pat, th, opts);
                        agree += s == b;
                        ++cases;
                        std::printf("search %d,%d,%d %s %g,%g mode=%d basis=%d n=%zu h=%016llx\n", t.r, t.g, t.b, ps,
                                    th.v_th, th.r_novib, static_cast<int>(mode), static_cast<int>(basis), b.size(),
                                    static_cast<unsigned long long>(hash_pairs(b)));
                    }
                }
            }
        }
    }
    std::printf("serial_equals_batch %d/%d\n", agree, cases);

    // ---- test_search.cpp:203-219: independent of the worker count ----------
    {
        SearchOptions one;
        one.workers = 1;
        const auto base = batch_search(SrgbColor{170, 170, 170}, grid, BitPattern::parse("101"), Thresholds{50.0, 0.5}, one);
        bool same = !base.empty();
        for (int w : {2, 3, 5, 16, 64}) {
            SearchOptions o;
            o.workers = w;
            same = same && batch_search(SrgbColor{170, 170, 170}, grid, BitPattern::parse("101"), Thresholds{50.0, 0.5}, o) == base;
        }
        std::printf("workers_independent %d\n", same ? 1 : 0);
    }

    // ---- test_search.cpp:221-255: canonical order, re-verification ---------
    {
        const auto pairs = batch_search(SrgbColor{170, 170, 170}, grid, BitPattern::parse("101"), Thresholds{50.0, 0.5});
        bool ordered = pairs.size() > 1;
        for (size_t i = 1; i < pairs.size(); ++i) {
            ordered = ordered && (pairs[i - 1].radius < pairs[i].radius ||
                                  (pairs[i - 1].radius == pairs[i].radius && pairs[i - 1].angle < pairs[i].angle));
        }
        std::printf("canonical_order %d\n", ordered ? 1 : 0);
        const Thresholds th{50.0, 0.5};
        const auto wp = batch_search(SrgbColor{240, 240, 240}, grid, BitPattern::parse("110"), th);
        const LabColor lab = srgb_to_lab(SrgbColor{240, 240, 240});
        bool ok = !wp.empty();
        for (const auto& p : wp) {
            const auto [lp, lm] = displaced_pair(lab, p.radius, p.angle);
            ok = ok && lab_to_srgb_clipped(lp) == p.plus && lab_to_srgb_clipped(lm) == p.minus &&
                 channel_deltas(p.target, p.plus, p.minus) == p.deltas &&
                 classify_pair(p.deltas, BitPattern::parse("110"), th) && lp.l == lab.l && lm.l == lab.l;
        }
        std::printf("reverified %d n=%zu\n", ok ? 1 : 0, wp.size());
        VibrationGrid zero;
        zero.radii = {0.0};
        zero.angles = grid.angles;
        bool none = true;
        for (const char* ps : {"100", "010", "001", "110", "101", "011", "111"}) {
            none = none && batch_search(SrgbColor{170, 170, 170}, zero, BitPattern::parse(ps), Thresholds{50.0, 0.5}).empty() &&
                   serial_search(SrgbColor{170, 170, 170}, zero, BitPattern::parse(ps), Thresholds{50.0, 0.5}).empty();
        }
        std::printf("zero_radius_empty %d\n", none ? 1 : 0);
    }

    // ---- the reference's feasibility sweep (feasibility.cpp:261-292) -------
    {
        const SearchConfig cfg = SearchConfig::defaults();
        const FeasibilityMatrix m = feasibility_matrix(cfg);
        std::printf("config_hash %s\n", config_hash(cfg).c_str());
        std::printf("matrix_csv_aggregated\n%s", export_matrix(m, ExportFormat::Csv, true).c_str());
        const std::string full = export_matrix(m, ExportFormat::Csv, false);
        std::printf("matrix_csv_full bytes=%zu h=%016llx\n", full.size(),
                    static_cast<unsigned long long>(fnv(0xcbf29ce484222325ull, full.data(), full.size())));
        const std::string js = export_matrix(m, ExportFormat::Json, false);
        std::printf("matrix_json_full bytes=%zu h=%016llx\n", js.size(),
                    static_cast<unsigned long long>(fnv(0xcbf29ce484222325ull, js.data(), js.size())));
    }

    // ---- the reference's benchmark harness (bench.cpp) ---------------------
    {
        const BenchReport r = run_benchmark(SearchConfig::benchmark_defaults(), 1);
        std::printf("bench combos=%zu candidates=%zu pairs=%zu parity=%d\n", static_cast<size_t>(r.combos),
                    static_cast<size_t>(r.candidates), static_cast<size_t>(r.pairs_found), r.result_parity ? 1 : 0);
    }

    // ---- the reference's codec (codec.cpp:65-165) --------------------------
    {
        const DisplayParams disp;
        const VibrationGrid g = VibrationGrid::uniform(1.0, 76.0, 15.0, 9.0, 359.0, 12.0);
        const Thresholds th{50.0, 0.5};
        const FramePair tc = make_testcard(SrgbColor{170, 170, 170}, BitPattern::parse("101"), th, g, disp, 48, 32);
        std::printf("testcard a=%016llx b=%016llx\n", static_cast<unsigned long long>(hash_image(tc.frame_a)),
                    static_cast<unsigned long long>(hash_image(tc.frame_b)));
        BlockLayout layout;
        layout.block_width = 16;
        layout.block_height = 12;
        const SrgbColor cols[] = {{170, 170, 170}, {240, 100, 100}, {170, 170, 170}, {100, 100, 240}};
        const char* pats[] = {"101", "101", "001", "110"};
        for (int i = 0; i < 4; ++i) {
            BlockSpec b;
            b.x = 20 * i;
            b.y = 5 + 3 * i;
            b.color_name = "block" + std::to_string(i);
            b.color = cols[i];
            b.pattern = BitPattern::parse(pats[i]);
            layout.blocks.push_back(b);
        }
        const Image base = Image::solid(96, 40, SrgbColor{128, 128, 128});
        try {
            const FramePair fp = embed_blocks(base, layout, th, g, disp);
            std::printf("embed a=%016llx b=%016llx\n", static_cast<unsigned long long>(hash_image(fp.frame_a)),
                        static_cast<unsigned long long>(hash_image(fp.frame_b)));
            for (const auto& r : decode_blocks(fp, th)) {
                std::printf("decode status=%d pattern=%s deltas=%.17g,%.17g,%.17g\n", static_cast<int>(r.status),
                            r.pattern.str().c_str(), r.mean_deltas[0], r.mean_deltas[1], r.mean_deltas[2]);
            }
        } catch (const std::exception& e) {
            std::printf("embed error: %s\n", e.what());
        }
        // error behaviour: the reference's exception types and messages
        layout.blocks[2].pattern = BitPattern::parse("010");
        layout.blocks[2].color = SrgbColor{100, 240, 100};
        try {
            embed_blocks(base, layout, th, g, disp);
            std::printf("embed_unsatisfiable no error\n");
        } catch (const std::runtime_error& e) {
            std::printf("embed_unsatisfiable runtime_error: %s\n", e.what());
        }
        try {
            batch_search(SrgbColor{256, 0, 0}, grid, BitPattern::parse("111"), Thresholds{50.0, 0.5});
        } catch (const std::invalid_argument& e) {
            std::printf("bad_color invalid_argument: %s\n", e.what());
        }
        try {
            batch_search(SrgbColor{1, 2, 3}, grid, BitPattern{}, Thresholds{50.0, 0.5});
        } catch (const std::invalid_argument& e) {
            std::printf("empty_pattern invalid_argument: %s\n", e.what());
        }
        try {
            batch_search(SrgbColor{1, 2, 3}, grid, BitPattern::parse("111"), Thresholds{50.0, 1.5});
        } catch (const std::invalid_argument& e) {
            std::printf("bad_thresholds invalid_argument: %s\n", e.what());
        }
    }
    return 0;
}
