// colorvibe/search.hpp -- the color-pair search API of the B200 build.
//
// Declaration-compatible with the reference header
// proj/include/colorvibe/search.hpp:13-140: same types, same functions, same
// defaults, same exceptions.  batch_search and serial_search run on the GPU
// through the C-ABI in include/cvg.h (batch: FP32 fast path with FP64 repair;
// serial: FP64 op-for-op for every candidate); both return lists identical to
// the reference's.  There is no CPU fallback: without a usable sm_100a device
// the searches throw std::runtime_error.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "colorvibe/color.hpp"

namespace colorvibe {

/// Information bits carried by the R, G and B channels ("000" is rejected).
struct BitPattern {
    bool r = false;
    bool g = false;
    bool b = false;

    static BitPattern parse(std::string_view s);
    std::string str() const;
    bool any() const { return r || g || b; }

    bool operator==(const BitPattern&) const = default;
};

/// A 1-bit channel needs delta > v_th; a 0-bit channel needs
/// delta <= v_th * r_novib (low_band); between the two is a dead zone.
struct Thresholds {
    double v_th = 0.0;
    double r_novib = 0.0;

    double low_band() const { return v_th * r_novib; }
    void validate() const;
};

/// Explicit displacement grid: radii >= 0 ascending, angles in radians,
/// ascending within [0, 2pi).
struct VibrationGrid {
    std::vector<double> radii;
    std::vector<double> angles;

    /// Inclusive uniform ranges, angles in degrees.
    static VibrationGrid uniform(double radius_min, double radius_max, double radius_step,
                                 double angle_min_deg, double angle_max_deg, double angle_step_deg);
    /// 1..100 by 1 radius x 0..359 by 1 degree.
    static VibrationGrid standard();

    void validate() const;
    std::size_t candidate_count() const { return radii.size() * angles.size(); }
};

/// Per-channel deviation of a pair.
struct ChannelDeltas {
    double dr = 0.0;
    double dg = 0.0;
    double db = 0.0;

    bool operator==(const ChannelDeltas&) const = default;
};

/// One passing pair: quantized endpoints, its grid point and deltas.
struct ColorPair {
    SrgbColor target{};
    SrgbColor plus{};
    SrgbColor minus{};
    double radius = 0.0;
    double angle = 0.0;
    ChannelDeltas deltas{};

    bool operator==(const ColorPair&) const = default;
};

enum class DeltaMode {
    Quantized,   // deltas between 8-bit codes (default)
    Continuous,  // pre-quantization deltas (device path for both bases)
};

enum class DeltaBasis {
    TargetSwing,  // max(|plus - target|, |minus - target|) (default)
    FrameDiff,    // |plus - minus|
};

struct SearchOptions {
    DeltaMode delta_mode = DeltaMode::Quantized;
    DeltaBasis delta_basis = DeltaBasis::TargetSwing;
    int workers = 0;  // accepted for compatibility; results never depend on it
    WhitePoint white_point = d65_white();
};

/// (L, a + r sin(angle), b + r cos(angle)) and its mirror.
std::pair<LabColor, LabColor> displaced_pair(const LabColor& target, double radius, double angle);

ChannelDeltas channel_deltas(const SrgbColor& target, const SrgbColor& plus, const SrgbColor& minus);
ChannelDeltas frame_deltas(const SrgbColor& plus, const SrgbColor& minus);
bool classify_pair(const ChannelDeltas& deltas, const BitPattern& pattern, const Thresholds& th);

/// Reference "previous method": every candidate through the FP64 scalar
/// conversion (on the device).  Canonical (radius, angle) order.
std::vector<ColorPair> serial_search(const SrgbColor& target, const VibrationGrid& grid,
                                     const BitPattern& pattern, const Thresholds& th,
                                     const SearchOptions& opts = {});

/// The hot path: fused B200 kernel, list-identical to serial_search.
std::vector<ColorPair> batch_search(const SrgbColor& target, const VibrationGrid& grid,
                                    const BitPattern& pattern, const Thresholds& th,
                                    const SearchOptions& opts = {});

double classification_margin(const ColorPair& pair, const Thresholds& th);

/// Maximum margin; ties to smaller radius, then smaller angle.
const ColorPair& select_best(const std::vector<ColorPair>& pairs, const Thresholds& th);

// ---- B200 extension: many searches in one launch ------------------------
// One entry of a batch; all entries share the grid and options.
struct SearchSpec {
    SrgbColor target{};
    BitPattern pattern{};
    Thresholds thresholds{};
};

/// Runs every spec in one device launch; result[s] equals
/// batch_search(specs[s].target, grid, specs[s].pattern, specs[s].thresholds, opts).
std::vector<std::vector<ColorPair>> batch_search_many(const std::vector<SearchSpec>& specs,
                                                      const VibrationGrid& grid,
                                                      const SearchOptions& opts = {});

/// Pair counts only (no list materialization).
std::vector<std::uint64_t> batch_count_many(const std::vector<SearchSpec>& specs, const VibrationGrid& grid,
                                            const SearchOptions& opts = {});

// ---- B200 extension: lazy result -------------------------------------------
/// The pairs of one search, kept as the packed records the device returned
/// (u32 idx = k * n_angles + m, then plus r,g,b and minus r,g,b) in pinned
/// host memory; ColorPair (80 B, search.hpp:58-79) is built on access, so a
/// search with hundreds of millions of pairs costs 10 B per pair until
/// elements are read.  at(i) / to_vector() equal batch_search(...)[i] / (...).
class PairView {
public:
    PairView() = default;
    std::size_t size() const;
    bool empty() const { return size() == 0; }
    ColorPair at(std::size_t i) const;  // std::out_of_range past the end
    ColorPair operator[](std::size_t i) const { return at(i); }
    std::vector<ColorPair> to_vector() const;
    const std::uint32_t* idx() const;    // [size()] packed records
    const std::uint8_t* codes() const;   // [6 * size()]
    struct Impl;

private:
    std::shared_ptr<const Impl> impl_;
    friend PairView batch_search_view(const SrgbColor&, const VibrationGrid&, const BitPattern&, const Thresholds&,
                                      const SearchOptions&);
};

/// batch_search returning a PairView instead of materializing the list.
PairView batch_search_view(const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern,
                           const Thresholds& th, const SearchOptions& opts = {});

}  // namespace colorvibe
