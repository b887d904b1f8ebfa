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
#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
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

// Address of colorvibe::batch_search as THIS library binds it.  The library
// is linked with -Bsymbolic (oracle/Makefile), so the reference's own
// definition is used even when libcolorvibe_gpu.so (which exports the same
// mangled symbol) is loaded into the same process first with RTLD_GLOBAL;
// tests/test_oracle.py checks this with dladdr.
void* cvr_batch_search_addr() {
    using Fn = std::vector<ColorPair> (*)(const SrgbColor&, const VibrationGrid&, const BitPattern&,
                                          const Thresholds&, const SearchOptions&);
    return reinterpret_cast<void*>(static_cast<Fn>(&batch_search));
}

// cfg4's CPU baseline as BASELINE.md section 3 plans it: dedupe the pixels
// by color -- with one pattern and one threshold pair for the batch, results
// depend only on it -- evaluate each unique color with the reference
// batch_search (workers = 1 per call) on an outer pool of `threads`
// std::threads, then scatter count + first canonical pair to every pixel.
// Writes counts[n], first_idx[n] (0xFFFFFFFF if none), first_codes[6n];
// returns the number of unique colors, or a negative error.  memo = 0: no
// dedup, every pixel is searched (the same outer pool; the per-candidate
// CPU rate of the per-pixel batch).
int64_t cvr_search_memo(int64_t n, const int32_t* rgb, int pattern_bits, double v_th,
                        double r_novib, const double* radii, int nr, const double* angles, int na,
                        int threads, int memo, uint64_t* counts, uint32_t* first_idx, uint8_t* first_codes) {
    try {
        const VibrationGrid grid = grid_of(radii, nr, angles, na);
        std::vector<int32_t> slot(memo ? size_t(1) << 24 : 0, -1);  // key = rgb
        std::vector<uint32_t> keys;
        std::vector<int32_t> of(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const int32_t* c = rgb + 3 * i;
            if ((c[0] | c[1] | c[2]) & ~0xff) throw std::invalid_argument("color channel out of range");
            const uint32_t key = (static_cast<uint32_t>(c[0]) << 16) | (static_cast<uint32_t>(c[1]) << 8) |
                                 static_cast<uint32_t>(c[2]);
            if (!memo) {
                of[static_cast<size_t>(i)] = static_cast<int32_t>(keys.size());
                keys.push_back(key);
                continue;
            }
            int32_t& u = slot[key];
            if (u < 0) {
                u = static_cast<int32_t>(keys.size());
                keys.push_back(key);
            }
            of[static_cast<size_t>(i)] = u;
        }
        const size_t nu = keys.size();
        std::vector<uint64_t> ucount(nu);
        std::vector<uint32_t> ufirst(nu, 0xffffffffu);
        std::vector<uint8_t> ucodes(6 * nu, 0);
        std::atomic<size_t> next{0};
        std::string err;
        std::atomic<bool> failed{false};
        auto work = [&] {
            SearchOptions o;
            o.workers = 1;
            try {
                for (size_t u; (u = next.fetch_add(1)) < nu && !failed.load();) {
                    const uint32_t key = keys[u];
                    const auto pairs = batch_search(
                        SrgbColor{int((key >> 16) & 0xff), int((key >> 8) & 0xff), int(key & 0xff)}, grid,
                        pattern_of(pattern_bits), Thresholds{v_th, r_novib}, o);
                    ucount[u] = pairs.size();
                    if (!pairs.empty()) {
                        const ColorPair& p = pairs.front();
                        const auto k = std::lower_bound(grid.radii.begin(), grid.radii.end(), p.radius) -
                                       grid.radii.begin();
                        const auto m = std::lower_bound(grid.angles.begin(), grid.angles.end(), p.angle) -
                                       grid.angles.begin();
                        ufirst[u] = static_cast<uint32_t>(static_cast<uint64_t>(k) * na + m);
                        uint8_t* c = &ucodes[6 * u];
                        c[0] = p.plus.r; c[1] = p.plus.g; c[2] = p.plus.b;
                        c[3] = p.minus.r; c[4] = p.minus.g; c[5] = p.minus.b;
                    }
                }
            } catch (const std::exception& e) {
                if (!failed.exchange(true)) err = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < std::max(1, threads); ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
        if (failed) throw std::invalid_argument(err);
        for (int64_t i = 0; i < n; ++i) {
            const size_t u = static_cast<size_t>(of[static_cast<size_t>(i)]);
            counts[i] = ucount[u];
            first_idx[i] = ufirst[u];
            std::memcpy(first_codes + 6 * i, &ucodes[6 * u], 6);
        }
        return static_cast<int64_t>(nu);
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}

}  // extern "C"
