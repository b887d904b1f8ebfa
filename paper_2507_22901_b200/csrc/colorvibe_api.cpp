// colorvibe_api.cpp -- the reference C++ API (include/colorvibe/*.hpp) over
// the C-ABI of libcolorvibe_gpu.so.  Searches run on the GPU; this file only
// validates, marshals and materializes std::vector<ColorPair>
// (reference: src/search.cpp, src/color.cpp).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <string>

#include "../../include/cvg.h"
#include "colorvibe/search.hpp"
#include "colorvibe_detail.h"

namespace colorvibe {

namespace detail {

[[noreturn]] void throw_status(int status) {
    const std::string msg = cvg_last_error();
    if (status == CVG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void check(int status) {
    if (status != CVG_OK) throw_status(status);
}

// Process-wide context on the device named by CVG_DEVICE (default: 0).
cvg_ctx* default_ctx() {
    static std::once_flag once;
    static cvg_ctx* ctx = nullptr;
    static int status = CVG_OK;
    static std::string error;
    std::call_once(once, [] {
        const char* env = std::getenv("CVG_DEVICE");
        status = cvg_create(env ? std::atoi(env) : 0, &ctx);
        if (status != CVG_OK) error = cvg_last_error();
    });
    if (status != CVG_OK) throw std::runtime_error("colorvibe: no usable CUDA device: " + error);
    return ctx;
}

int pattern_bits(const BitPattern& p) { return (p.r ? 4 : 0) | (p.g ? 2 : 0) | (p.b ? 1 : 0); }

// One device call for a batch of searches sharing the grid and options.
void run(const std::vector<SearchSpec>& specs, const VibrationGrid& grid, const SearchOptions& opts,
         int output, int path, ResultGuard& g) {
    std::vector<int32_t> rgb(3 * specs.size());
    std::vector<int32_t> bits(specs.size());
    std::vector<double> vth(specs.size()), rn(specs.size());
    for (size_t s = 0; s < specs.size(); ++s) {
        rgb[3 * s] = specs[s].target.r;
        rgb[3 * s + 1] = specs[s].target.g;
        rgb[3 * s + 2] = specs[s].target.b;
        bits[s] = pattern_bits(specs[s].pattern);
        vth[s] = specs[s].thresholds.v_th;
        rn[s] = specs[s].thresholds.r_novib;
    }
    const double wp[3] = {opts.white_point.x, opts.white_point.y, opts.white_point.z};
    cvg_search_desc d{};
    d.n_searches = static_cast<int32_t>(specs.size());
    d.target_rgb = rgb.data();
    d.pattern_bits = bits.data();
    d.v_th = vth.data();
    d.r_novib = rn.data();
    d.n_radii = static_cast<int32_t>(grid.radii.size());
    d.radii = grid.radii.data();
    d.n_angles = static_cast<int32_t>(grid.angles.size());
    d.angles = grid.angles.data();
    d.delta_mode = opts.delta_mode == DeltaMode::Quantized ? CVG_DELTA_QUANTIZED : CVG_DELTA_CONTINUOUS;
    d.delta_basis = opts.delta_basis == DeltaBasis::TargetSwing ? CVG_BASIS_TARGET_SWING : CVG_BASIS_FRAME_DIFF;
    d.white_point = wp;
    d.output = output;
    d.path = path;
    d.workers = opts.workers;
    check(cvg_search(default_ctx(), &d, &g.r));
}

// ColorPair of record (i, c) of a search around `target` (Continuous: `lab`
// is the target's Lab, deltas from the host's glibc signal values).
ColorPair make_pair(uint32_t i, const uint8_t* c, const SrgbColor& target, const double* radii, const double* angles,
                    uint32_t na, const SearchOptions& opts, const double* lab) {
    const bool swing = opts.delta_basis == DeltaBasis::TargetSwing;
    const bool continuous = opts.delta_mode == DeltaMode::Continuous;
    const double wp[3] = {opts.white_point.x, opts.white_point.y, opts.white_point.z};
    ColorPair cp;
    cp.target = target;
    cp.plus = SrgbColor{c[0], c[1], c[2]};
    cp.minus = SrgbColor{c[3], c[4], c[5]};
    cp.radius = radii[i / na];
    cp.angle = angles[i % na];
    if (continuous) {
        // continuous_deltas (search.cpp:161-180) on the host's glibc signal values
        double sp[3], sm[3];
        check(cvg_pair_signal(lab, cp.radius, cp.angle, wp, sp, sm));
        const double t[3] = {static_cast<double>(target.r), static_cast<double>(target.g),
                             static_cast<double>(target.b)};
        double d[3];
        for (int q = 0; q < 3; ++q) {
            d[q] = swing ? std::max(std::abs(sp[q] - t[q]), std::abs(sm[q] - t[q])) : std::abs(sp[q] - sm[q]);
        }
        cp.deltas = ChannelDeltas{d[0], d[1], d[2]};
    } else {
        cp.deltas = swing ? channel_deltas(target, cp.plus, cp.minus) : frame_deltas(cp.plus, cp.minus);
    }
    return cp;
}

std::vector<ColorPair> materialize(const cvg_result& r, size_t s, const SrgbColor& target, const VibrationGrid& grid,
                                   const SearchOptions& opts) {
    std::vector<ColorPair> out;
    const uint64_t b = r.offsets[s], e = r.offsets[s + 1];
    out.reserve(e - b);
    const uint32_t na = static_cast<uint32_t>(grid.angles.size());
    double lab[3] = {0, 0, 0};
    if (opts.delta_mode == DeltaMode::Continuous) {
        const int32_t rgb[3] = {target.r, target.g, target.b};
        const double wp[3] = {opts.white_point.x, opts.white_point.y, opts.white_point.z};
        check(cvg_srgb_to_lab(rgb, wp, lab));
    }
    for (uint64_t p = b; p < e; ++p) {
        out.push_back(make_pair(r.idx[p], r.codes + 6 * p, target, grid.radii.data(), grid.angles.data(), na, opts, lab));
    }
    return out;
}

}  // namespace detail

using namespace detail;

namespace {

void validate_one(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                  const Thresholds& th) {
    // search.cpp:22-30 order: color, grid, thresholds, pattern.
    validate(target);
    grid.validate();
    th.validate();
    if (!pattern.any()) throw std::invalid_argument("bit pattern has no set bits");
}

std::vector<ColorPair> search_one(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                                  const Thresholds& th, const SearchOptions& opts, int path) {
    validate_one(target, grid, pattern, th);
    if (grid.radii.empty() || grid.angles.empty()) return {};
    ResultGuard g;
    run({SearchSpec{target, pattern, th}}, grid, opts, CVG_OUT_PAIRS, path, g);
    return materialize(g.r, 0, target, grid, opts);
}

}  // namespace

// ---- color.hpp -------------------------------------------------------------

const WhitePoint& d65_white() {
    static const WhitePoint wp = [] {
        double w[3];
        cvg_d65_white(w);
        return WhitePoint{w[0], w[1], w[2]};
    }();
    return wp;
}

bool is_valid(const SrgbColor& c) {
    return c.r >= 0 && c.r <= 255 && c.g >= 0 && c.g <= 255 && c.b >= 0 && c.b <= 255;
}

void validate(const SrgbColor& c) {
    if (!is_valid(c)) {
        throw std::invalid_argument("sRGB channel code outside [0, 255]: (" + std::to_string(c.r) + ", " +
                                    std::to_string(c.g) + ", " + std::to_string(c.b) + ")");
    }
}

void validate(const LabColor& lab) {
    if (!(std::isfinite(lab.l) && std::isfinite(lab.a) && std::isfinite(lab.b)) || lab.l < 0.0 || lab.l > 100.0) {
        throw std::invalid_argument("Lab color with L* outside [0, 100]");
    }
}

double srgb_to_linear(int code) {
    if (code < 0 || code > 255) {
        throw std::invalid_argument("channel code outside [0, 255]: " + std::to_string(code));
    }
    const double u = code / 255.0;
    return u <= 0.04045 ? u / 12.92 : std::pow((u + 0.055) / 1.055, 2.4);
}

LabColor srgb_to_lab(const SrgbColor& c, const WhitePoint& wp) {
    validate(c);
    const int32_t rgb[3] = {c.r, c.g, c.b};
    const double w[3] = {wp.x, wp.y, wp.z};
    double lab[3];
    check(cvg_srgb_to_lab(rgb, w, lab));
    return LabColor{lab[0], lab[1], lab[2]};
}

std::optional<SrgbColor> lab_to_srgb(const LabColor& lab, const WhitePoint& wp) {
    validate(lab);
    const double l[3] = {lab.l, lab.a, lab.b};
    const double w[3] = {wp.x, wp.y, wp.z};
    int32_t rgb[3];
    const int st = cvg_lab_to_srgb(l, w, rgb);
    if (st < 0) throw_status(-st);
    if (st == 0) return std::nullopt;
    return SrgbColor{rgb[0], rgb[1], rgb[2]};
}

SrgbColor lab_to_srgb_clipped(const LabColor& lab, const WhitePoint& wp) {
    validate(lab);
    const double l[3] = {lab.l, lab.a, lab.b};
    const double w[3] = {wp.x, wp.y, wp.z};
    int32_t rgb[3];
    check(cvg_lab_to_srgb_clipped(l, w, rgb));
    return SrgbColor{rgb[0], rgb[1], rgb[2]};
}

bool in_gamut(const LabColor& lab, const WhitePoint& wp) { return lab_to_srgb(lab, wp).has_value(); }

// ---- search.hpp ------------------------------------------------------------

BitPattern BitPattern::parse(std::string_view s) {
    if (s.size() != 3 || s.find_first_not_of("01") != std::string_view::npos) {
        throw std::invalid_argument("bit pattern must be three binary digits");
    }
    BitPattern p{s[0] == '1', s[1] == '1', s[2] == '1'};
    if (!p.any()) throw std::invalid_argument("bit pattern \"000\" carries no signal");
    return p;
}

std::string BitPattern::str() const { return {r ? '1' : '0', g ? '1' : '0', b ? '1' : '0'}; }

void Thresholds::validate() const {
    if (!(std::isfinite(v_th) && v_th > 0.0)) throw std::invalid_argument("v_th must be positive");
    if (!(std::isfinite(r_novib) && r_novib > 0.0 && r_novib <= 1.0)) {
        throw std::invalid_argument("r_novib must be in (0, 1]");
    }
}

VibrationGrid VibrationGrid::uniform(double radius_min, double radius_max, double radius_step, double angle_min_deg,
                                     double angle_max_deg, double angle_step_deg) {
    if (!(radius_step > 0.0) || !(angle_step_deg > 0.0)) throw std::invalid_argument("grid steps must be positive");
    if (radius_min < 0.0 || radius_max < radius_min) throw std::invalid_argument("invalid radius range");
    if (angle_min_deg < 0.0 || angle_max_deg < angle_min_deg || angle_max_deg >= 360.0) {
        throw std::invalid_argument("angle range must lie within [0, 360)");
    }
    VibrationGrid g;
    for (int k = 0;; ++k) {
        const double v = radius_min + k * radius_step;
        if (v > radius_max + 1e-9) break;
        g.radii.push_back(v);
    }
    constexpr double kDegToRad = std::numbers::pi / 180.0;
    for (int k = 0;; ++k) {
        const double deg = angle_min_deg + k * angle_step_deg;
        if (deg > angle_max_deg + 1e-9) break;
        g.angles.push_back(deg * kDegToRad);
    }
    g.validate();
    return g;
}

VibrationGrid VibrationGrid::standard() { return uniform(1.0, 100.0, 1.0, 0.0, 359.0, 1.0); }

void VibrationGrid::validate() const {
    constexpr double kTwoPi = 2.0 * std::numbers::pi;
    for (size_t i = 0; i < radii.size(); ++i) {
        if (!(std::isfinite(radii[i]) && radii[i] >= 0.0)) throw std::invalid_argument("grid radii must be non-negative");
        if (i > 0 && !(radii[i] > radii[i - 1])) throw std::invalid_argument("grid radii must be strictly increasing");
    }
    for (size_t i = 0; i < angles.size(); ++i) {
        if (!(std::isfinite(angles[i]) && angles[i] >= 0.0 && angles[i] < kTwoPi)) {
            throw std::invalid_argument("grid angles must lie in [0, 2pi)");
        }
        if (i > 0 && !(angles[i] > angles[i - 1])) throw std::invalid_argument("grid angles must be strictly increasing");
    }
}

std::pair<LabColor, LabColor> displaced_pair(const LabColor& target, double radius, double angle) {
    validate(target);
    if (!(std::isfinite(radius) && radius >= 0.0) || !std::isfinite(angle)) {
        throw std::invalid_argument("displacement radius must be >= 0");
    }
    const double da = radius * std::sin(angle);
    const double db = radius * std::cos(angle);
    return {LabColor{target.l, target.a + da, target.b + db}, LabColor{target.l, target.a - da, target.b - db}};
}

ChannelDeltas channel_deltas(const SrgbColor& target, const SrgbColor& plus, const SrgbColor& minus) {
    validate(target);
    validate(plus);
    validate(minus);
    auto dev = [](int t, int p, int m) { return static_cast<double>(std::max(std::abs(p - t), std::abs(m - t))); };
    return ChannelDeltas{dev(target.r, plus.r, minus.r), dev(target.g, plus.g, minus.g), dev(target.b, plus.b, minus.b)};
}

ChannelDeltas frame_deltas(const SrgbColor& plus, const SrgbColor& minus) {
    validate(plus);
    validate(minus);
    return ChannelDeltas{static_cast<double>(std::abs(plus.r - minus.r)), static_cast<double>(std::abs(plus.g - minus.g)),
                         static_cast<double>(std::abs(plus.b - minus.b))};
}

bool classify_pair(const ChannelDeltas& d, const BitPattern& pattern, const Thresholds& th) {
    th.validate();
    if (!pattern.any()) throw std::invalid_argument("bit pattern has no set bits");
    const double low = th.low_band();
    const bool r_ok = pattern.r ? d.dr > th.v_th : d.dr <= low;
    const bool g_ok = pattern.g ? d.dg > th.v_th : d.dg <= low;
    const bool b_ok = pattern.b ? d.db > th.v_th : d.db <= low;
    return r_ok && g_ok && b_ok;
}

// The reference's scalar "previous method" (search.cpp:184-218), kept as
// what it is in the reference: one candidate after another on the host, the
// baseline the batched search is measured against (run_benchmark's serial
// column).  It is not a fallback: batch_search and every other
// search entry point run on the device only.
std::vector<ColorPair> serial_search(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                                     const Thresholds& th, const SearchOptions& opts) {
    validate_one(target, grid, pattern, th);
    const double wp[3] = {opts.white_point.x, opts.white_point.y, opts.white_point.z};
    const int32_t rgb[3] = {target.r, target.g, target.b};
    double lab[3];
    check(cvg_srgb_to_lab(rgb, wp, lab));
    const bool quantized = opts.delta_mode == DeltaMode::Quantized;
    const bool swing = opts.delta_basis == DeltaBasis::TargetSwing;
    const double t[3] = {static_cast<double>(target.r), static_cast<double>(target.g), static_cast<double>(target.b)};
    std::vector<ColorPair> hits;
    for (double radius : grid.radii) {
        for (double angle : grid.angles) {
            int32_t p[3], m[3];
            double gp[3], gm[3];
            check(cvg_pair_eval(lab, radius, angle, wp, p, m, gp, gm));
            const SrgbColor sp{p[0], p[1], p[2]}, sm{m[0], m[1], m[2]};
            ChannelDeltas d;
            if (quantized) {
                d = swing ? channel_deltas(target, sp, sm) : frame_deltas(sp, sm);
            } else {
                // continuous_deltas (search.cpp:161-180)
                double e[3];
                for (int q = 0; q < 3; ++q) {
                    e[q] = swing ? std::max(std::abs(gp[q] - t[q]), std::abs(gm[q] - t[q])) : std::abs(gp[q] - gm[q]);
                }
                d = ChannelDeltas{e[0], e[1], e[2]};
            }
            if (classify_pair(d, pattern, th)) hits.push_back(ColorPair{target, sp, sm, radius, angle, d});
        }
    }
    return hits;
}

std::vector<ColorPair> batch_search(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                                    const Thresholds& th, const SearchOptions& opts) {
    return search_one(target, grid, pattern, th, opts, CVG_PATH_PRUNED);  // FAST + certified row pruning: same pairs
}

// ---- PairView ----------------------------------------------------------------

struct PairView::Impl {
    cvg_result r{};
    SrgbColor target{};
    std::vector<double> radii, angles;
    SearchOptions opts{};
    double lab[3] = {0, 0, 0};
    ~Impl() { cvg_result_free(&r); }
};

std::size_t PairView::size() const { return impl_ ? static_cast<std::size_t>(impl_->r.n_pairs) : 0; }

const std::uint32_t* PairView::idx() const { return impl_ ? impl_->r.idx : nullptr; }

const std::uint8_t* PairView::codes() const { return impl_ ? impl_->r.codes : nullptr; }

ColorPair PairView::at(std::size_t i) const {
    if (i >= size()) throw std::out_of_range("PairView index out of range");
    const Impl& m = *impl_;
    return make_pair(m.r.idx[i], m.r.codes + 6 * i, m.target, m.radii.data(), m.angles.data(),
                     static_cast<uint32_t>(m.angles.size()), m.opts, m.lab);
}

std::vector<ColorPair> PairView::to_vector() const {
    std::vector<ColorPair> out;
    out.reserve(size());
    for (std::size_t i = 0; i < size(); ++i) out.push_back(at(i));
    return out;
}

PairView batch_search_view(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                           const Thresholds& th, const SearchOptions& opts) {
    validate_one(target, grid, pattern, th);
    PairView v;
    auto impl = std::make_shared<PairView::Impl>();
    impl->target = target;
    impl->opts = opts;
    if (!grid.radii.empty() && !grid.angles.empty()) {
        ResultGuard g;
        run({SearchSpec{target, pattern, th}}, grid, opts, CVG_OUT_PAIRS, CVG_PATH_PRUNED, g);
        impl->r = g.r;  // the view owns the result from here
        g.r = cvg_result{};
        impl->radii = grid.radii;
        impl->angles = grid.angles;
        if (opts.delta_mode == DeltaMode::Continuous) {
            const int32_t rgb[3] = {target.r, target.g, target.b};
            const double wp[3] = {opts.white_point.x, opts.white_point.y, opts.white_point.z};
            check(cvg_srgb_to_lab(rgb, wp, impl->lab));
        }
    }
    v.impl_ = std::move(impl);
    return v;
}

double classification_margin(const ColorPair& pair, const Thresholds& th) {
    th.validate();
    const double low = th.low_band();
    auto chan = [&](double d) { return d > th.v_th ? d - th.v_th : low - d; };
    return std::min({chan(pair.deltas.dr), chan(pair.deltas.dg), chan(pair.deltas.db)});
}

const ColorPair& select_best(const std::vector<ColorPair>& pairs, const Thresholds& th) {
    if (pairs.empty()) throw std::invalid_argument("select_best: empty pair list");
    const ColorPair* best = &pairs.front();
    double best_margin = classification_margin(*best, th);
    for (size_t i = 1; i < pairs.size(); ++i) {
        const double m = classification_margin(pairs[i], th);
        const bool better = m > best_margin ||
                            (m == best_margin && (pairs[i].radius < best->radius ||
                                                  (pairs[i].radius == best->radius && pairs[i].angle < best->angle)));
        if (better) {
            best = &pairs[i];
            best_margin = m;
        }
    }
    return *best;
}

std::vector<std::vector<ColorPair>> batch_search_many(const std::vector<SearchSpec>& specs, const VibrationGrid& grid,
                                                      const SearchOptions& opts) {
    for (const auto& s : specs) validate_one(s.target, grid, s.pattern, s.thresholds);
    std::vector<std::vector<ColorPair>> out(specs.size());
    if (specs.empty() || grid.radii.empty() || grid.angles.empty()) return out;
    ResultGuard g;
    run(specs, grid, opts, CVG_OUT_PAIRS, CVG_PATH_PRUNED, g);
    for (size_t s = 0; s < specs.size(); ++s) out[s] = materialize(g.r, s, specs[s].target, grid, opts);
    return out;
}

std::vector<std::uint64_t> batch_count_many(const std::vector<SearchSpec>& specs, const VibrationGrid& grid,
                                            const SearchOptions& opts) {
    for (const auto& s : specs) validate_one(s.target, grid, s.pattern, s.thresholds);
    std::vector<std::uint64_t> out(specs.size(), 0);
    if (specs.empty() || grid.radii.empty() || grid.angles.empty()) return out;
    ResultGuard g;
    run(specs, grid, opts, CVG_OUT_COUNTS, CVG_PATH_FAST, g);  // counts: the strip tiles outrun row pruning
    for (size_t s = 0; s < specs.size(); ++s) out[s] = g.r.counts[s];
    return out;
}

}  // namespace colorvibe
