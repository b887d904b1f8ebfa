// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper over the UNMODIFIED reference hot path, compiled
// together with the reference's own sources where they lie
// (<ref>/proj/src/color.cpp, <ref>/proj/src/search.cpp) by oracle/Makefile
// into oracle/_ref/.  Nothing from the reference is copied into this repo.
// Used (a) to pin oracle/cv_oracle.c bit-for-bit against the reference and
// (b) as bench.py's CPU baseline / `--impl reference` arm, which times the
// reference's own colorvibe::batch_search (search.cpp:403-456).

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "colorvibe/search.hpp"
#include "convert_kernel.hpp"

using namespace colorvibe;

namespace {

thread_local std::string g_err;

BitPattern pattern_of(int bits) {
    BitPattern p;
    p.r = (bits >> 2) & 1;
    p.g = (bits >> 1) & 1;
    p.b = bits & 1;
    return p;
}

VibrationGrid grid_of(const double* radii, int nr, const double* angles, int na) {
    VibrationGrid g;
    g.radii.assign(radii, radii + nr);
    g.angles.assign(angles, angles + na);
    return g;
}

SearchOptions options_of(int mode, int basis, int workers, const double* wp) {
    SearchOptions o;
    o.delta_mode = mode == 0 ? DeltaMode::Quantized : DeltaMode::Continuous;
    o.delta_basis = basis == 0 ? DeltaBasis::TargetSwing : DeltaBasis::FrameDiff;
    o.workers = workers;
    if (wp) o.white_point = WhitePoint{wp[0], wp[1], wp[2]};
    return o;
}

}  // namespace

extern "C" {

const char* cvr_last_error() { return g_err.c_str(); }

void cvr_thresholds(double out[256]) {
    const auto& qt = detail::quant_table();
    std::memcpy(out, qt.thresholds.data(), 256 * sizeof(double));
}

int cvr_table_code(double x) { return detail::quant_table().code(x); }
int cvr_quantize(double x) { return detail::quantize_signal(x); }

void cvr_xyz_to_rgb(double out[9]) {
    std::memcpy(out, detail::kXyzToRgb.m, 9 * sizeof(double));
}

void cvr_white(double out[3]) {
    const WhitePoint& w = d65_white();
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
}

void cvr_srgb_to_lab(const int32_t rgb[3], double lab[3]) {
    const LabColor l = srgb_to_lab(SrgbColor{rgb[0], rgb[1], rgb[2]});
    lab[0] = l.l;
    lab[1] = l.a;
    lab[2] = l.b;
}

// Returns the pair count (records beyond cap are dropped), -1 on
// std::invalid_argument, -2 on any other exception.
int64_t cvr_search(const int32_t rgb[3], int pattern_bits, double v_th,
                   double r_novib, const double* radii, int nr,
                   const double* angles, int na, int delta_mode,
                   int delta_basis, const double* wp, int method, int workers,
                   uint32_t* idx, uint8_t* codes, double* deltas, int64_t cap) {
    try {
        const VibrationGrid grid = grid_of(radii, nr, angles, na);
        const SrgbColor t{rgb[0], rgb[1], rgb[2]};
        const Thresholds th{v_th, r_novib};
        const SearchOptions o = options_of(delta_mode, delta_basis, workers, wp);
        const std::vector<ColorPair> pairs =
            method == 0 ? serial_search(t, grid, pattern_of(pattern_bits), th, o)
                        : batch_search(t, grid, pattern_of(pattern_bits), th, o);
        const int64_t n = static_cast<int64_t>(pairs.size());
        const int64_t w = std::min(n, cap);
        for (int64_t q = 0; q < w; ++q) {
            const ColorPair& p = pairs[q];
            if (idx) {
                const auto k = std::lower_bound(grid.radii.begin(), grid.radii.end(), p.radius) -
                               grid.radii.begin();
                const auto m = std::lower_bound(grid.angles.begin(), grid.angles.end(), p.angle) -
                               grid.angles.begin();
                idx[q] = static_cast<uint32_t>(static_cast<uint64_t>(k) * na + m);
            }
            if (codes) {
                uint8_t* c = codes + 6 * q;
                c[0] = p.plus.r; c[1] = p.plus.g; c[2] = p.plus.b;
                c[3] = p.minus.r; c[4] = p.minus.g; c[5] = p.minus.b;
            }
            if (deltas) {
                deltas[3 * q] = p.deltas.dr;
                deltas[3 * q + 1] = p.deltas.dg;
                deltas[3 * q + 2] = p.deltas.db;
            }
        }
        return n;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}

// Many searches on one grid through the reference batch_search, one call
// per search exactly as the reference's sweep does (feasibility.cpp:273-275).
// Writes per-search pair counts; returns the total or a negative error.
int64_t cvr_search_many(int n, const int32_t* rgb, const int32_t* pattern_bits,
                        const double* v_th, const double* r_novib,
                        const double* radii, int nr, const double* angles,
                        int na, int workers, uint64_t* counts) {
    try {
        const VibrationGrid grid = grid_of(radii, nr, angles, na);
        SearchOptions o;
        o.workers = workers;
        int64_t total = 0;
        for (int s = 0; s < n; ++s) {
            const auto pairs = batch_search(
                SrgbColor{rgb[3 * s], rgb[3 * s + 1], rgb[3 * s + 2]}, grid,
                pattern_of(pattern_bits[s]), Thresholds{v_th[s], r_novib[s]}, o);
            counts[s] = pairs.size();
            total += static_cast<int64_t>(pairs.size());
        }
        return total;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}

}  // extern "C"
