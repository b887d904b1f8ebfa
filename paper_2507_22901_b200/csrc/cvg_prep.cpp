// cvg_prep.cpp -- reference-exact host preparation: scalar conversions
// (convert_kernel.hpp restated), the quantization threshold table,
// validation with the reference's messages, the continuous-mode signal
// bands, and the per-search record with its proven FP32 error bounds.
#include "cvg_host.h"

namespace cvg::host {

double f_lab(double t) { return t > kEps ? std::cbrt(t) : (kKappa * t + 16.0) / 116.0; }

double f_lab_inv(double u) {
    const double u3 = (u * u) * u;
    return u3 > kEps ? u3 : (116.0 * u - 16.0) * kInvKappa;
}

double eotf(double u) { return u <= 0.04045 ? u / 12.92 : std::pow((u + 0.055) / 1.055, 2.4); }
double oetf(double x) { return x <= 0.0031308 ? 12.92 * x : 1.055 * std::pow(x, 1.0 / 2.4) - 0.055; }

int quantize(double linear) {
    const double x = linear < 0.0 ? 0.0 : (linear > 1.0 ? 1.0 : linear);
    return static_cast<int>(std::floor(255.0 * oetf(x) + 0.5));
}

const double* white_or_d65(const double* wp) {
    static const double d65[3] = {(kRgbToXyz.m[0][0] + kRgbToXyz.m[0][1]) + kRgbToXyz.m[0][2],
                                  (kRgbToXyz.m[1][0] + kRgbToXyz.m[1][1]) + kRgbToXyz.m[1][2],
                                  (kRgbToXyz.m[2][0] + kRgbToXyz.m[2][1]) + kRgbToXyz.m[2][2]};
    return wp ? wp : d65;
}

void to_lab(const int32_t c[3], const double* wp, double lab[3]) {
    const double rl = eotf(c[0] / 255.0), gl = eotf(c[1] / 255.0), bl = eotf(c[2] / 255.0);
    const auto& m = kRgbToXyz.m;
    const double x = (m[0][0] * rl + m[0][1] * gl) + m[0][2] * bl;
    const double y = (m[1][0] * rl + m[1][1] * gl) + m[1][2] * bl;
    const double z = (m[2][0] * rl + m[2][1] * gl) + m[2][2] * bl;
    const double fx = f_lab(x / wp[0]), fy = f_lab(y / wp[1]), fz = f_lab(z / wp[2]);
    lab[0] = 116.0 * fy - 16.0;
    lab[1] = 500.0 * (fx - fy);
    lab[2] = 200.0 * (fy - fz);
}

void to_linear(const double lab[3], const double* wp, double lin[3]) {
    const double fy = (lab[0] + 16.0) / 116.0;
    const double fx = fy + lab[1] * kInv500;
    const double fz = fy - lab[2] * kInv200;
    const double x = wp[0] * f_lab_inv(fx), y = wp[1] * f_lab_inv(fy), z = wp[2] * f_lab_inv(fz);
    const auto& m = kXyzToRgb.m;
    for (int c = 0; c < 3; ++c) lin[c] = (m[c][0] * x + m[c][1] * y) + m[c][2] * z;
}

const Tables& tables() {
    static const Tables t;
    return t;
}

// ---------------------------------------------------------------------------
// Validation, mirroring the reference's checks and messages
// (color.cpp:27-39, search.cpp:22-30, 49-56, 92-111).

int validate_color(const int32_t* c) {
    if (c[0] < 0 || c[0] > 255 || c[1] < 0 || c[1] > 255 || c[2] < 0 || c[2] > 255) {
        return fail(CVG_EINVAL, "sRGB channel code outside [0, 255]: (" + std::to_string(c[0]) + ", " +
                                    std::to_string(c[1]) + ", " + std::to_string(c[2]) + ")");
    }
    return CVG_OK;
}

int validate_grid(const double* radii, int nr, const double* angles, int na) {
    if (nr < 0 || na < 0 || (nr > 0 && !radii) || (na > 0 && !angles)) {
        return fail(CVG_EINVAL, "grid arrays missing");
    }
    for (int i = 0; i < nr; ++i) {
        if (!(std::isfinite(radii[i]) && radii[i] >= 0.0)) return fail(CVG_EINVAL, "grid radii must be non-negative");
        if (i > 0 && !(radii[i] > radii[i - 1])) return fail(CVG_EINVAL, "grid radii must be strictly increasing");
    }
    for (int i = 0; i < na; ++i) {
        if (!(std::isfinite(angles[i]) && angles[i] >= 0.0 && angles[i] < kTwoPi)) {
            return fail(CVG_EINVAL, "grid angles must lie in [0, 2pi)");
        }
        if (i > 0 && !(angles[i] > angles[i - 1])) return fail(CVG_EINVAL, "grid angles must be strictly increasing");
    }
    return CVG_OK;
}

int validate_thresholds(double v_th, double r_novib) {
    if (!(std::isfinite(v_th) && v_th > 0.0)) return fail(CVG_EINVAL, "v_th must be positive");
    if (!(std::isfinite(r_novib) && r_novib > 0.0 && r_novib <= 1.0)) return fail(CVG_EINVAL, "r_novib must be in (0, 1]");
    return CVG_OK;
}

// True when every search of the batch is valid (colors in [0, 255],
// 0 < v_th < inf, 0 < r_novib <= 1, pattern in 1..7).  Accumulates with
// bitwise ORs so the compiler vectorizes it: ~1 ns per search.
bool batch_clean_range(const cvg_search_desc* d, size_t lo, size_t hi) {
    uint32_t bad = 0;
    const int32_t* c = d->target_rgb;
    for (size_t i = 3 * lo; i < 3 * hi; ++i) bad |= static_cast<uint32_t>(c[i]) > 255u;
    const int32_t* pb = d->pattern_bits;
    for (size_t i = lo; i < hi; ++i) bad |= static_cast<uint32_t>(pb[i] - 1) > 6u;
    const double* v = d->v_th;
    const double* r = d->r_novib;
    for (size_t i = lo; i < hi; ++i) {
        bad |= static_cast<uint32_t>(!(v[i] > 0.0)) | static_cast<uint32_t>(!(v[i] < HUGE_VAL)) |
               static_cast<uint32_t>(!(r[i] > 0.0)) | static_cast<uint32_t>(!(r[i] <= 1.0));
    }
    return bad == 0;
}

bool batch_clean(const cvg_search_desc* d) {
    const size_t n = static_cast<size_t>(d->n_searches);
    const size_t chunk = 1u << 14;  // a 377K-search range of cfg4 spreads over every core (1.26 -> ~0.15 ms)
    const size_t parts = (n + chunk - 1) / chunk;
    std::vector<char> ok(parts, 1);
    parallel_for(
        parts, [&](size_t c) { ok[c] = batch_clean_range(d, c * chunk, std::min(n, (c + 1) * chunk)); }, 1);
    for (char o : ok) {
        if (!o) return false;
    }
    return true;
}

// The descriptor's scalar fields (no per-search arrays scanned).
int validate_header(const cvg_search_desc* d) {
    if (!d) return fail(CVG_EINVAL, "null search descriptor");
    if (d->n_searches < 0) return fail(CVG_EINVAL, "n_searches must be >= 0");
    if (d->n_searches > 0 && (!d->target_rgb || !d->pattern_bits || !d->v_th || !d->r_novib)) {
        return fail(CVG_EINVAL, "search arrays missing");
    }
    if (d->delta_mode != CVG_DELTA_QUANTIZED && d->delta_mode != CVG_DELTA_CONTINUOUS) {
        return fail(CVG_EINVAL, "unknown delta_mode");
    }
    if (d->delta_basis != CVG_BASIS_TARGET_SWING && d->delta_basis != CVG_BASIS_FRAME_DIFF) {
        return fail(CVG_EINVAL, "unknown delta_basis");
    }
    if (d->output < CVG_OUT_PAIRS || d->output > CVG_OUT_BEST) return fail(CVG_EINVAL, "unknown output mode");
    if (d->path < CVG_PATH_FAST || d->path > CVG_PATH_MEMO) return fail(CVG_EINVAL, "unknown path");
    if (d->output == CVG_OUT_BEST && d->delta_mode != CVG_DELTA_QUANTIZED) {
        return fail(CVG_EUNSUPPORTED, "CVG_OUT_BEST ranks integer (Quantized) deltas; continuous deltas need the "
                                      "host's glibc pow (select_best over CVG_OUT_PAIRS)");
    }
    if (d->path == CVG_PATH_MEMO && (d->output == CVG_OUT_PAIRS || d->output == CVG_OUT_BEST)) {
        return fail(CVG_EINVAL, "CVG_PATH_MEMO returns per-search counts / first pairs (CVG_OUT_COUNTS or CVG_OUT_FIRST)");
    }
    return CVG_OK;
}

int validate_desc(const cvg_search_desc* d) {
    if (int e = validate_header(d)) return e;
    // Fast screen: branch-free, vectorizable pass over the whole batch.  Only
    // if it finds a problem does the ordered per-search loop below run, to
    // report the first failure with the reference's message and order.
    if (batch_clean(d) && validate_grid(d->radii, d->n_radii, d->angles, d->n_angles) == CVG_OK) {
        goto checked;
    }
    {
    // Per search in the reference order: target, grid, thresholds, pattern.
    int grid_checked = 0;
    for (int s = 0; s < d->n_searches; ++s) {
        if (int e = validate_color(d->target_rgb + 3 * s)) return e;
        if (!grid_checked) {
            if (int e = validate_grid(d->radii, d->n_radii, d->angles, d->n_angles)) return e;
            grid_checked = 1;
        }
        if (int e = validate_thresholds(d->v_th[s], d->r_novib[s])) return e;
        const int p = d->pattern_bits[s];
        if (p < 0 || p > 7) return fail(CVG_EINVAL, "bit pattern must be three binary digits");
        if (p == 0) return fail(CVG_EINVAL, "bit pattern has no set bits");
    }
    if (!grid_checked) {
        if (int e = validate_grid(d->radii, d->n_radii, d->angles, d->n_angles)) return e;
    }
    }
checked:
    if (static_cast<uint64_t>(d->n_radii) * static_cast<uint64_t>(d->n_angles) >= (1ull << 32)) {
        return fail(CVG_EINVAL, "grid too large: n_radii * n_angles must be < 2^32");
    }
    return CVG_OK;
}

// ---------------------------------------------------------------------------
// Per-search constants and the FP32 error bound.

float round_up_f(double x) {
    if (std::isinf(x)) return static_cast<float>(x);
    float f = static_cast<float>(x);
    if (static_cast<double>(f) < x) f = std::nextafter(f, INFINITY);
    return f;
}

float round_down_f(double x) {
    if (std::isinf(x)) return static_cast<float>(x);
    float f = static_cast<float>(x);
    if (static_cast<double>(f) > x) f = std::nextafter(f, -INFINITY);
    return f;
}

// Continuous-mode bands.  With s(x) = signal_value(x) = 255 * oetf(clamp(x))
// (convert_kernel.hpp:109-112, glibc pow), the reference's per-endpoint
// condition fabs(s(x) - t) <= T (search.cpp:171-179, 146-157) holds exactly
// on an interval [a, b] of doubles because s is monotone non-decreasing.
// a and b are found by bisection over the reference's own double
// computation; the band handed to the kernel is [a, nextafter(b, +inf)).
// Monotonicity is checked on 64 doubles either side of each bound.
double signal_value(double linear) {
    const double x = linear < 0.0 ? 0.0 : (linear > 1.0 ? 1.0 : linear);
    return 255.0 * oetf(x);
}

struct SignalBand {
    double lo, hi;
};

SignalBand signal_band(int target, double T) {
    const double t = static_cast<double>(target);
    auto low_ok = [&](double x) { return signal_value(x) - t >= -T; };   // true for x >= a
    auto high_ok = [&](double x) { return signal_value(x) - t <= T; };   // true for x <= b
    // smallest x in (0, 1] with low_ok, by bisection over doubles
    auto first_true = [](auto pred) {
        double lo = 0.0, hi = 1.0;  // pred(hi) assumed true, pred(lo) false
        while (std::nextafter(lo, 1.0) < hi) {
            const double mid = 0.5 * (lo + hi);
            (pred(mid) ? hi : lo) = mid;
        }
        return hi;
    };
    SignalBand b;
    if (low_ok(0.0)) {
        b.lo = -HUGE_VAL;  // s(x) = 0 for x <= 0 already satisfies it
    } else if (!low_ok(1.0)) {
        return SignalBand{HUGE_VAL, HUGE_VAL};  // never inside (empty band)
    } else {
        b.lo = first_true(low_ok);
    }
    if (high_ok(1.0)) {
        b.hi = HUGE_VAL;
    } else if (!high_ok(0.0)) {
        return SignalBand{HUGE_VAL, HUGE_VAL};
    } else {
        b.hi = first_true([&](double x) { return !high_ok(x); });  // first x above b
    }
    // monotonicity around each bound (pow is accurate to < 1 ulp; a violation
    // here would mean the interval model does not hold)
    for (double edge : {b.lo, b.hi}) {
        if (std::isinf(edge)) continue;
        double x = edge;
        for (int i = 0; i < 64; ++i) x = std::nextafter(x, -1.0);
        double prev = signal_value(x);
        for (int i = 0; i < 128; ++i) {
            x = std::nextafter(x, 2.0);
            const double v = signal_value(x);
            if (v < prev) throw std::runtime_error("signal_value not monotone near a band edge");
            prev = v;
        }
    }
    return b;
}

// signal_band depends only on (target code, threshold): a batch repeats few
// pairs (cfg1: 9 targets x 16 thresholds over 756 searches), and each band
// costs ~380 glibc pow calls, so bands are memoized process-wide.
SignalBand signal_band_cached(int target, double T) {
    static std::mutex mu;
    static std::map<std::pair<int, uint64_t>, SignalBand> cache;
    uint64_t bits;
    std::memcpy(&bits, &T, sizeof(bits));
    const std::pair<int, uint64_t> key(target, bits);
    {
        std::lock_guard<std::mutex> lk(mu);
        const auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const SignalBand b = signal_band(target, T);
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= (1u << 16)) cache.clear();
    cache.emplace(key, b);
    return b;
}

// Continuous x FrameDiff linear-space bounds for a channel threshold T on
// d = |s(x_p) - s(x_m)| (search.cpp:161-173).  s = signal_value is increasing
// and concave on [0, 1] with s(0) = 0 and s(1) = 255, so for dx = |x_p - x_m|
//   d <= s(dx)               (subadditivity): dx <= a, s(a) <= T - 1e-6,
//                            gives d < T, and a loud channel fails;
//   d >= 255 - s(1 - dx)     (the flattest end): dx >= 1 - b with
//                            s(b) <= 255 - T - 1e-6 gives d > T, and a quiet
//                            channel fails.
// Returns {a, 1 - b} (largest such a, b by bisection over the reference's own
// signal_value, glibc pow); a = -1: no loud region, a = 2: a loud channel
// never passes; 1 - b = 2: a quiet channel never fails.  Memoized per T.
std::pair<double, double> frame_signal_bounds(double T) {
    static std::mutex mu;
    static std::map<double, std::pair<double, double>> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        const auto it = cache.find(T);
        if (it != cache.end()) return it->second;
    }
    auto largest_below = [](double v) {  // largest x in [0, 1] with s(x) <= v (v in [0, 255))
        double lo = 0.0, hi = 1.0;
        for (int i = 0; i < 80; ++i) {
            const double mid = 0.5 * (lo + hi);
            (signal_value(mid) <= v ? lo : hi) = mid;
        }
        return lo;
    };
    const double la = T - 1e-6, lq = 255.0 - T - 1e-6;
    const double a = la <= 0.0 ? -1.0 : (la >= 255.0 ? 2.0 : largest_below(la));
    const double q = lq < 0.0 ? 2.0 : 1.0 - largest_below(lq);
    const std::pair<double, double> r{a, q};
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 4096) cache.clear();
    cache.emplace(T, r);
    return r;
}

struct BoundTerms {
    double err;  // |g32 - f^-1(f)| bound
    double gmax; // max |f^-1(f)|
};

// Forward error of g = f^-1(f) computed in FP32 as in fast_linear():
// f = fma(+-r, s', f0) with r, s', f0 rounded to float, then either
// (f*f)*f or fma(f, K1, -K2).  u = 2^-24 (round to nearest).
BoundTerms finv_bound(double f0, double rmax_scaled) {
    const double u = std::ldexp(1.0, -24);
    const double F0 = std::fabs(f0);
    const double ef = 3.01 * u * rmax_scaled + 2.01 * u * F0;  // |f32 - f|
    const double fm = F0 + rmax_scaled;                        // max |f|
    const double cube_err = 3.0 * fm * fm * ef + 3.0 * fm * ef * ef + ef * ef * ef +
                            2.01 * u * (fm + ef) * (fm + ef) * (fm + ef);
    const double k1 = 3132.0 / 24389.0, k2 = 432.0 / 24389.0;
    const double lin_err = k1 * ef + 2.01 * u * (k1 * fm + k2) + 2.0 * u * k1 * ef;
    BoundTerms b;
    b.err = std::max(cube_err, lin_err);
    b.gmax = std::max(fm * fm * fm, k1 * fm + k2);
    return b;
}

// Cube-only rows (every endpoint in the cube branch), sum/difference form as
// in the kernel's band_cube(): with f+- = f0 +- U (U = r*s') the half-sum and
// half-difference of the cubes are
//   A = (f+^3 + f-^3)/2 = f0^3 + 3 f0 U^2   = fma(u*u, C3, C1)
//   B = (f+^3 - f-^3)/2 = U (3 f0^2 + U^2)  = u * fma(u, u, C2),   u = r*s'
// with C1 = fl(f0^3), C2 = fl(3 f0^2), C3 = fl(3 f0) rounded once from double
// (1.01u each).  Forward errors (u = 2^-24):
//   u:         3.01u |U|   (r, s' rounded to float, product)
//   u*u:       7.04u U^2;   times C3: 8.06u relative to 3 F0 U^2
//   A:         8.06u 3F0U^2 + 1.01u F0^3 + u |A|
//   fma(u,u,C2): 6.03u U^2 + 3.03u F0^2 + u |T|,  T = U^2 + 3 F0^2
//   B:         |u| etx + 3.01u |U| T + u |U| T
struct CubeTerms {
    BoundTerms a, b;
};

CubeTerms cube_bound(double f0, double umax) {
    const double u = std::ldexp(1.0, -24);
    const double F = std::fabs(f0), U = umax;
    CubeTerms t;
    t.a.gmax = F * F * F + 3.0 * F * U * U;
    t.a.err = u * (9.07 * 3.0 * F * U * U + 2.02 * F * F * F);
    const double T = U * U + 3.0 * F * F;
    const double etx = u * (7.04 * U * U + 6.04 * F * F);
    t.b.gmax = U * T;
    t.b.err = U * (1.0 + 3.02 * u) * etx + 4.03 * u * U * T;
    return t;
}

void make_search_const(const cvg_search_desc* d, int s, double rmax, int mode, const Tables& T,
                       SearchConst& S) {
    std::memset(&S, 0, sizeof(S));
    const double* wp = white_or_d65(d->white_point);
    const int32_t* t = d->target_rgb + 3 * s;
    // srgb_to_lab of the target (color.cpp:57-70: 3 glibc pow + 3 cbrt, most
    // of a record's cost); batches repeat a target over consecutive searches,
    // so each thread remembers its last one
    thread_local int32_t last_t[3] = {-1, -1, -1};
    thread_local double last_wp[3] = {0, 0, 0}, last_lab[3];
    double lab[3];
    if (t[0] == last_t[0] && t[1] == last_t[1] && t[2] == last_t[2] && wp[0] == last_wp[0] && wp[1] == last_wp[1] &&
        wp[2] == last_wp[2]) {
        std::memcpy(lab, last_lab, sizeof(lab));
    } else {
        to_lab(t, wp, lab);
        std::memcpy(last_t, t, sizeof(last_t));
        std::memcpy(last_wp, wp, sizeof(last_wp));
        std::memcpy(last_lab, lab, sizeof(lab));
    }
    // search.cpp:345-355
    const auto& m = kXyzToRgb.m;
    const double fy = (lab[0] + 16.0) / 116.0;
    const double yv = wp[1] * f_lab_inv(fy);
    S.fy = fy;
    S.ta = lab[1];
    S.tb = lab[2];
    S.wx = wp[0];
    S.wz = wp[2];
    for (int c = 0; c < 3; ++c) S.cy64[c] = m[c][1] * yv;

    const int bits[3] = {(d->pattern_bits[s] >> 2) & 1, (d->pattern_bits[s] >> 1) & 1, d->pattern_bits[s] & 1};
    const double v_th = d->v_th[s];
    const double low = v_th * d->r_novib[s];
    const int k1 = v_th >= 255.0 ? 256 : static_cast<int>(v_th) + 1;
    const int q0 = low >= 255.0 ? 255 : static_cast<int>(low);
    S.k1 = k1;
    S.q0 = q0;
    S.flags = static_cast<uint32_t>(bits[0] | (bits[1] << 1) | (bits[2] << 2));
    if (d->delta_basis == CVG_BASIS_FRAME_DIFF) S.flags |= 1u << 8;
    const bool continuous = d->delta_mode == CVG_DELTA_CONTINUOUS;
    if (continuous) S.flags |= 1u << 9;  // bands on signal values: no integer-code self-check
    for (int c = 0; c < 3; ++c) S.t[c] = t[c];
    // make_bands (search.cpp:291-329): exact only for Quantized x TargetSwing.
    for (int c = 0; c < 3; ++c) {
        if (mode == cvg::kModeSignal) {
            // continuous FrameDiff (search.cpp:146-173): the channel's threshold on |s(p) - s(m)|
            S.lo[c] = bits[c] ? v_th : low;
            S.hi[c] = HUGE_VAL;
        } else if (mode == cvg::kModeBand && continuous) {
            // continuous_deltas (search.cpp:161-180): pass iff |s(x) - t| <= T
            // for both endpoints (quiet, T = low) / not for both (loud, T = v_th)
            const SignalBand b = signal_band_cached(t[c], bits[c] ? v_th : low);
            S.lo[c] = b.lo;
            S.hi[c] = b.hi;
        } else if (mode != cvg::kModeBand) {
            S.lo[c] = -HUGE_VAL;
            S.hi[c] = HUGE_VAL;
        } else if (bits[c]) {
            S.lo[c] = t[c] - k1 + 1 >= 1 ? T.thr[t[c] - k1 + 1] : -HUGE_VAL;
            S.hi[c] = t[c] + k1 <= 255 ? T.thr[t[c] + k1] : HUGE_VAL;
        } else {
            S.lo[c] = t[c] - q0 >= 1 ? T.thr[t[c] - q0] : -HUGE_VAL;
            S.hi[c] = t[c] + q0 + 1 <= 255 ? T.thr[t[c] + q0 + 1] : HUGE_VAL;
        }
    }

    // FP32 constants.
    const double fx0 = fy + lab[1] * kInv500;
    const double fz0 = fy - lab[2] * kInv200;
    S.fx0 = static_cast<float>(fx0);
    S.fz0 = static_cast<float>(fz0);
    const double u0 = 6.0 / 29.0;
    const double rc = std::min((fx0 - u0) * 500.0, (fz0 - u0) * 200.0) * (1.0 - 1e-6) - 1e-6;
    S.rcube = rc > 0.0 ? round_down_f(rc) : -1.0f;
    const double u = std::ldexp(1.0, -24);
    const BoundTerms bx = finv_bound(fx0, rmax * kInv500);
    const BoundTerms bz = finv_bound(fz0, rmax * kInv200);
    const CubeTerms cx = cube_bound(fx0, rmax * kInv500);
    const CubeTerms cz = cube_bound(fz0, rmax * kInv200);
    const double cube_c[6] = {fx0 * fx0 * fx0, 3.0 * fx0 * fx0, 3.0 * fx0, fz0 * fz0 * fz0, 3.0 * fz0 * fz0, 3.0 * fz0};
    for (int i = 0; i < 6; ++i) S.cube[i] = static_cast<float>(cube_c[i]);
    double eps_q = 0.0, eps_l = 0.0;
    // band form channel slots: loud channels first (the kernel specializes on
    // the loud count L and reads slots [0, L) as loud, [L, 3) as quiet)
    int slot_of[3], n_loud = 0;
    for (int c = 0; c < 3; ++c) n_loud += bits[c];
    {
        // Loud channels ordered most selective first: the strip loop tests
        // slot 0 alone first and skips the other channels when no candidate
        // of a group can leave slot 0's band.  Selectivity estimate: the
        // band statistic of the target itself plus its first-order growth
        // over half the radius range, in band units (small = rarely > 1).
        double sigma[3];
        for (int c = 0; c < 3; ++c) {
            const double mx = m[c][0] * wp[0], mz = m[c][2] * wp[2];
            const double lo = std::isinf(S.lo[c]) ? -10.0 : S.lo[c], hi = std::isinf(S.hi[c]) ? 10.0 : S.hi[c];
            const double hh = std::max(0.5 * (hi - lo), 1e-30), cc = 0.5 * (lo + hi);
            const double centre = (mx * fx0 * fx0 * fx0 + mz * fz0 * fz0 * fz0 + S.cy64[c] - cc) / hh;
            const double growth = (std::fabs(mx) * 3.0 * fx0 * fx0 * kInv500 + std::fabs(mz) * 3.0 * fz0 * fz0 * kInv200) *
                                  0.5 * rmax / hh;
            sigma[c] = std::fabs(centre) + growth;
        }
        int order[3] = {0, 1, 2};
        std::stable_sort(order, order + 3, [&](int a, int b) {
            if (bits[a] != bits[b]) return bits[a] > bits[b];  // loud first
            return bits[a] ? sigma[a] < sigma[b] : false;
        });
        for (int j = 0; j < 3; ++j) slot_of[order[j]] = j;
    }
    S.flags |= static_cast<uint32_t>(n_loud) << 10;
    for (int c = 0; c < 3; ++c) {
        const double mx = m[c][0] * wp[0], mz = m[c][2] * wp[2], cy = S.cy64[c];
        // Forward error of fma(cx, gx, fma(cz, gz, add)) with float-rounded
        // constants (|cx|, |cz| magnitudes, `add` exact value).  Returns
        // (bound, max |result|).
        auto lin_err_of = [&](const BoundTerms& gx, const BoundTerms& gz, double acx, double acz, double add) {
            const double aadd = std::fabs(add);
            const double inner_max = acz * gz.gmax + aadd;
            const double e_inner = acz * gz.err * (1 + u) + u * acz * gz.gmax + u * aadd + u * (inner_max + acz * gz.err);
            const double lin_max = acx * gx.gmax + inner_max;
            return std::pair<double, double>(acx * gx.err * (1 + u) + u * acx * gx.gmax + e_inner +
                                                 u * (lin_max + acx * gx.err),
                                             lin_max);
        };
        auto lin_err = [&](double acx, double acz, double add) { return lin_err_of(bx, bz, acx, acz, add); };
        S.mx[c] = static_cast<float>(mx);
        S.mz[c] = static_cast<float>(mz);
        S.cy[c] = static_cast<float>(cy);
        const auto [e_lin, lin_max] = lin_err(std::fabs(mx), std::fabs(mz), cy);
        const double eps = 1.05 * e_lin + 1e-12;
        S.eps[c] = round_up_f(eps);
        S.eps_code[c] = round_up_f(eps + std::ldexp(1.0, -23));
        // Band form.  With centre cc and half-width hh of [lo, hi] (an
        // infinite edge replaced by -+L, L above every |lin| on the grid,
        // which leaves the test unchanged), channel c is inside iff
        // M' = max(|vp - cc|, |vm - cc|) / hh <= 1: the matrix constants are
        // pre-divided by hh so the kernel gets (v - cc) / hh directly.
        const double L = lin_max + e_lin + 1.0;
        double lo = std::isinf(S.lo[c]) ? -L : S.lo[c];
        double hi = std::isinf(S.hi[c]) ? L : S.hi[c];
        if (S.lo[c] == HUGE_VAL || !(S.lo[c] < S.hi[c])) {  // empty band: never inside
            lo = L + 1.0;
            hi = L + 2.0;
        }
        const double cc = 0.5 * (lo + hi), hh = 0.5 * (hi - lo);
        const int j = slot_of[c];
        S.mxs[j] = static_cast<float>(mx / hh);
        S.mzs[j] = static_cast<float>(mz / hh);
        S.cys[j] = static_cast<float>((cy - cc) / hh);
        const auto [e_d, d_max] = lin_err(std::fabs(mx / hh), std::fabs(mz / hh), (cy - cc) / hh);
        // cube-only rows: M' = |A_c| + |B_c| with A_c = fma(mxs, Ax, fma(mzs, Az, cys)) and
        // B_c = fma(mxs, Bx, -(mzs * Bz)) (the kernel's band_cube); the thresholds cover both forms
        const auto [e_a, a_max] = lin_err_of(cx.a, cz.a, std::fabs(mx / hh), std::fabs(mz / hh), (cy - cc) / hh);
        const auto [e_b, b_max] = lin_err_of(cx.b, cz.b, std::fabs(mx / hh), std::fabs(mz / hh), 0.0);
        const double e_ab = e_a + e_b + u * (a_max + b_max + e_a + e_b);
        // strip form (the kernel's strip_stat, cube-only rows of a strip):
        // A_c = fma(K2_c, r^2, K0_c), B_c = fma(L3_c, r^3, fl(L1_c * r)) with
        // K0_c = mxs fx0^3 + mzs fz0^3 + cys, K2_c = mxs 3fx0 s'^2 + mzs 3fz0 c'^2,
        // L1_c = mxs 3fx0^2 s' - mzs 3fz0^2 c', L3_c = mxs s'^3 - mzs c'^3, all
        // in FP32 from the float constants and the float trig / r, r^2, r^3
        // tables.  Term by term (u = 2^-24; strip_setup's operation order):
        // |err K0| <= 4u TA0, |err K2 r^2| <= 10u TA2, final rounding u |A|
        // (TA = TA0 + TA2 the magnitudes of the cube and U^2 parts), and
        // |err fl(L1 r)| <= 8u TB1, |err L3 r^3| <= 9u TB3, rounding u |B|;
        // bounded here by 20u TA and 20u TB.
        const double fxa = std::fabs(fx0), fza = std::fabs(fz0);
        const double uxm = rmax * kInv500, uzm = rmax * kInv200;
        const double amx = std::fabs(mx / hh), amz = std::fabs(mz / hh);
        const double ta_s = amx * (fxa * fxa * fxa + 3.0 * fxa * uxm * uxm) +
                            amz * (fza * fza * fza + 3.0 * fza * uzm * uzm) + std::fabs((cy - cc) / hh);
        const double tb_s = amx * uxm * (3.0 * fxa * fxa + uxm * uxm) + amz * uzm * (3.0 * fza * fza + uzm * uzm);
        const double e_as = 20.0 * u * ta_s, e_bs = 20.0 * u * tb_s;
        const double e_abs = e_as + e_bs + u * (ta_s + tb_s + e_as + e_bs);
        const double m_max = std::max({d_max, a_max + b_max, ta_s + tb_s});
        const double e_m = 1.05 * (std::max({e_d, e_ab, e_abs}) + 4 * std::ldexp(1.0, -53) * (m_max + 2.0)) + 1e-12 / hh;
        (bits[c] ? eps_l : eps_q) = std::max(bits[c] ? eps_l : eps_q, e_m);
    }
    S.la = round_down_f(1.0 - eps_l);
    S.lp = round_up_f(1.0 + eps_l);
    S.qa = round_up_f(1.0 + eps_q);
    S.qp = round_down_f(1.0 - eps_q);
    if (mode == cvg::kModeSignal) {
        // Continuous x FrameDiff: the same prefilter on the signal's
        // linear-space bounds (frame_signal_bounds), before the signal table
        for (int c = 0; c < 3; ++c) {
            const double m = 2.0 * S.eps[c] + std::ldexp(1.0, -22) + 1e-9;
            const auto [a, q] = frame_signal_bounds(S.lo[c]);
            if (bits[c]) {
                S.fd_bounds[2 * c] = a > 1.5 ? INFINITY : (a < 0.0 ? -1.0f : round_down_f(a - m));
                S.fd_bounds[2 * c + 1] = INFINITY;
            } else {
                S.fd_bounds[2 * c] = -1.0f;
                S.fd_bounds[2 * c + 1] = q > 1.5 ? INFINITY : round_up_f(q + m);
            }
        }
    }
    if (mode == cvg::kModeCodes) {
        // FrameDiff prefilter bounds (frame_row): |sat(v32) - sat(v64)| <= eps
        // per endpoint and the FP32 difference rounds by <= 2^-24, so a
        // channel whose |d32| is at most fd_loud - 2 eps - 2^-22 (loud) or at
        // least fd_quiet + 2 eps + 2^-22 (quiet) surely fails.
        for (int c = 0; c < 3; ++c) {
            const double m = 2.0 * S.eps[c] + std::ldexp(1.0, -22);
            if (bits[c]) {
                const double lo = T.fd_loud[k1];
                S.fd_bounds[2 * c] = std::isinf(lo) ? INFINITY : round_down_f(lo - m);
                S.fd_bounds[2 * c + 1] = INFINITY;
            } else {
                const double hi = T.fd_quiet[q0];
                S.fd_bounds[2 * c] = -1.0f;
                S.fd_bounds[2 * c + 1] = std::isinf(hi) ? INFINITY : round_up_f(hi + m);
            }
        }
    }
}

}  // namespace cvg::host
