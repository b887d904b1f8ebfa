// cvg_host.cpp -- host side of libcolorvibe_gpu.so: the C-ABI in include/cvg.h.
//
// Compiled with the reference's FP flags (-ffp-contract=off, no errno/traps)
// so every double computed here -- target Lab (glibc pow/cbrt), per-angle
// sin/cos (glibc), the quantization threshold table (bisection over glibc
// pow), the per-target hoisted constants -- carries the same bits as the
// reference (src/color.cpp:57-70, src/search.cpp:341-370, 414-419,
// src/convert_kernel.hpp:123-146).  Those are one-off per-call tables; every
// candidate is evaluated on the GPU (cvg_kernels.cu).
#include <cuda_runtime.h>

#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/cvg.h"
#include "cvg_internal.h"
#include "cvg_layout.h"

using cvg::LaunchArgs;
using cvg::SearchConst;

namespace {

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

#define CVG_CUDA(call)                                  \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// ---------------------------------------------------------------------------
// Pinned constants and scalar conversions (restating convert_kernel.hpp).

struct Mat3 {
    double m[3][3];
};

constexpr Mat3 kRgbToXyz{{{0.4124, 0.3576, 0.1805}, {0.2126, 0.7152, 0.0722}, {0.0193, 0.1192, 0.9505}}};

// Adjugate over determinant with the reference's association
// (convert_kernel.hpp:27-43), evaluated at compile time.
constexpr Mat3 adjugate_inverse(const Mat3& a) {
    const auto& m = a.m;
    const double c00 = m[1][1] * m[2][2] - m[1][2] * m[2][1];
    const double c01 = m[1][0] * m[2][2] - m[1][2] * m[2][0];
    const double c02 = m[1][0] * m[2][1] - m[1][1] * m[2][0];
    const double det = m[0][0] * c00 - m[0][1] * c01 + m[0][2] * c02;
    Mat3 r{};
    r.m[0][0] = c00 / det;
    r.m[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
    r.m[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
    r.m[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
    r.m[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
    r.m[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
    r.m[2][0] = c02 / det;
    r.m[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
    r.m[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
    return r;
}

constexpr Mat3 kXyzToRgb = adjugate_inverse(kRgbToXyz);
constexpr double kEps = 216.0 / 24389.0;
constexpr double kKappa = 24389.0 / 27.0;
constexpr double kInvKappa = 27.0 / 24389.0;
constexpr double kInv500 = 1.0 / 500.0;
constexpr double kInv200 = 1.0 / 200.0;
constexpr double kGamutEps = 1e-12;
constexpr double kTwoPi = 2.0 * std::numbers::pi;

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

// Quantization thresholds: thr[c] = smallest double x with quantize(x) >= c,
// found by bisection over the glibc-pow quantizer (convert_kernel.hpp:127-141).
struct Tables {
    double thr[256];
    float thr3[256][4];  // {tf[g], tf[g+1], tf[g+2], 0}: tf[0] = -inf, tf[c] = float(thr[c]), tf[256..] = +inf
    uint8_t guess[cvg::kGuessBuckets + 1];
    Tables() {
        thr[0] = 0.0;
        for (int code = 1; code <= 255; ++code) {
            double lo = thr[code - 1], hi = 1.0;
            while (std::nextafter(lo, 1.0) < hi) {
                const double mid = 0.5 * (lo + hi);
                (quantize(mid) >= code ? hi : lo) = mid;
            }
            thr[code] = hi;
        }
        float tf[258];
        tf[0] = -INFINITY;
        for (int c = 1; c < 256; ++c) tf[c] = static_cast<float>(thr[c]);
        tf[256] = tf[257] = INFINITY;
        for (int g = 0; g < 256; ++g) {
            thr3[g][0] = tf[g];
            thr3[g][1] = tf[g + 1];
            thr3[g][2] = tf[g + 2];
            thr3[g][3] = 0.0f;
        }
        // Round-to-nearest buckets: bucket i holds x * 4096 in [i - 1/2, i + 1/2);
        // guess = code at the bucket's lower edge (<= 1 threshold per bucket).
        for (int i = 0; i <= cvg::kGuessBuckets; ++i) guess[i] = static_cast<uint8_t>(code((i - 0.5) / 4096.0));
    }
    int code(double x) const {
        if (x <= 0.0) return 0;
        if (x >= 1.0) return 255;
        return static_cast<int>(std::upper_bound(thr + 1, thr + 256, x) - thr) - 1;
    }
};

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

// Process-wide worker threads for parallel_for: spawning threads per call
// costs ~10 us each, more than the host work of a sweep-sized batch.  The
// caller takes part; nested calls and calls from a forked child run inline.
class WorkerPool {
public:
    static WorkerPool& get() {
        static WorkerPool pool;
        return pool;
    }
    size_t width() const { return workers_.size() + 1; }

    // job(w) for w in [0, n_jobs) on the pool and the calling thread
    void run(size_t n_jobs, const std::function<void(size_t)>& job) {
        if (n_jobs <= 1 || workers_.empty() || in_job_ || getpid() != pid_) {
            for (size_t w = 0; w < n_jobs; ++w) job(w);
            return;
        }
        std::lock_guard<std::mutex> one(run_mu_);  // one batch at a time
        Batch b;
        {
            std::lock_guard<std::mutex> lk(mu_);
            b = Batch{++generation_, static_cast<uint32_t>(n_jobs), &job};
            batch_ = b;
            pending_ = n_jobs;
            state_.store(b.gen << 32);
        }
        cv_.notify_all();
        work(b);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

private:
    struct Batch {
        uint64_t gen = 0;
        uint32_t n = 0;
        const std::function<void(size_t)>* job = nullptr;
    };
    WorkerPool() : pid_(getpid()) {
        const size_t hw = std::max(1u, std::thread::hardware_concurrency());
        for (size_t i = 0; i + 1 < std::min<size_t>(hw, 64); ++i) {
            workers_.emplace_back([this] { loop(); });
        }
    }
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // Claims jobs of batch b only: state_ = generation << 32 | next job, so a
    // worker holding an older batch can never take a job of a newer one.
    void work(const Batch& b) {
        in_job_ = true;
        size_t done = 0;
        uint64_t st = state_.load();
        for (;;) {
            if ((st >> 32) != (b.gen & 0xffffffffu) || (st & 0xffffffffu) >= b.n) break;
            if (!state_.compare_exchange_weak(st, st + 1)) continue;
            (*b.job)(static_cast<size_t>(st & 0xffffffffu));
            ++done;
            st = state_.load();
        }
        in_job_ = false;
        if (done) {
            std::lock_guard<std::mutex> lk(mu_);
            pending_ -= done;
            if (pending_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            Batch b;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || generation_ != seen; });
                if (stop_) return;
                seen = generation_;
                b = batch_;
            }
            work(b);
        }
    }

    pid_t pid_;
    std::vector<std::thread> workers_;
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    Batch batch_;
    size_t pending_ = 0;
    std::atomic<uint64_t> state_{0};
    uint64_t generation_ = 0;
    bool stop_ = false;
    static thread_local bool in_job_;
};
thread_local bool WorkerPool::in_job_ = false;

// Runs f(0..n-1) on the worker pool, at least `grain` items per job
// (contiguous ranges); inline for small n.  Exceptions are rethrown on the
// caller's thread.
template <typename F>
void parallel_for(size_t n, F&& f, size_t grain = 512) {
    WorkerPool& pool = WorkerPool::get();
    const size_t jobs = std::min<size_t>(pool.width(), n / std::max<size_t>(grain, 1));
    if (jobs <= 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::exception_ptr err;
    std::mutex err_mu;
    pool.run(jobs, [&](size_t w) {
        try {
            for (size_t i = n * w / jobs; i < n * (w + 1) / jobs; ++i) f(i);
        } catch (...) {
            std::lock_guard<std::mutex> lk(err_mu);
            if (!err) err = std::current_exception();
        }
    });
    if (err) std::rethrow_exception(err);
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
    const size_t chunk = 1u << 18;
    const size_t parts = (n + chunk - 1) / chunk;
    std::vector<char> ok(parts, 1);
    parallel_for(
        parts, [&](size_t c) { ok[c] = batch_clean_range(d, c * chunk, std::min(n, (c + 1) * chunk)); }, 1);
    for (char o : ok) {
        if (!o) return false;
    }
    return true;
}

int validate_desc(const cvg_search_desc* d) {
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
    if (d->output < CVG_OUT_PAIRS || d->output > CVG_OUT_FIRST) return fail(CVG_EINVAL, "unknown output mode");
    if (d->path < CVG_PATH_FAST || d->path > CVG_PATH_AUDIT) return fail(CVG_EINVAL, "unknown path");
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
    if (d->delta_mode == CVG_DELTA_CONTINUOUS && d->delta_basis == CVG_BASIS_FRAME_DIFF) {
        return fail(CVG_EUNSUPPORTED,
                    "DeltaMode::Continuous with DeltaBasis::FrameDiff is not implemented on the device path "
                    "(no CPU fallback)");
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

void make_search_const(const cvg_search_desc* d, int s, double rmax, int mode, const Tables& T,
                       SearchConst& S) {
    std::memset(&S, 0, sizeof(S));
    const double* wp = white_or_d65(d->white_point);
    const int32_t* t = d->target_rgb + 3 * s;
    double lab[3];
    to_lab(t, wp, lab);
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
        if (mode == cvg::kModeBand && continuous) {
            // continuous_deltas (search.cpp:161-180): pass iff |s(x) - t| <= T
            // for both endpoints (quiet, T = low) / not for both (loud, T = v_th)
            const SignalBand b = signal_band(t[c], bits[c] ? v_th : low);
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
    double eps_q = 0.0, eps_l = 0.0;
    // band form channel slots: loud channels first (the kernel specializes on
    // the loud count L and reads slots [0, L) as loud, [L, 3) as quiet)
    int slot_of[3], n_loud = 0;
    for (int c = 0; c < 3; ++c) n_loud += bits[c];
    {
        int nl = 0, nq = n_loud;
        for (int c = 0; c < 3; ++c) slot_of[c] = bits[c] ? nl++ : nq++;
    }
    S.flags |= static_cast<uint32_t>(n_loud) << 10;
    for (int c = 0; c < 3; ++c) {
        const double mx = m[c][0] * wp[0], mz = m[c][2] * wp[2], cy = S.cy64[c];
        // Forward error of fma(cx, gx, fma(cz, gz, add)) with float-rounded
        // constants (|cx|, |cz| magnitudes, `add` exact value).  Returns
        // (bound, max |result|).
        auto lin_err = [&](double acx, double acz, double add) {
            const double aadd = std::fabs(add);
            const double inner_max = acz * bz.gmax + aadd;
            const double e_inner = acz * bz.err * (1 + u) + u * acz * bz.gmax + u * aadd + u * (inner_max + acz * bz.err);
            const double lin_max = acx * bx.gmax + inner_max;
            return std::pair<double, double>(acx * bx.err * (1 + u) + u * acx * bx.gmax + e_inner +
                                                 u * (lin_max + acx * bx.err),
                                             lin_max);
        };
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
        const double e_m = 1.05 * (e_d + 4 * std::ldexp(1.0, -53) * (d_max + 2.0)) + 1e-12 / hh;
        (bits[c] ? eps_l : eps_q) = std::max(bits[c] ? eps_l : eps_q, e_m);
    }
    S.la = round_down_f(1.0 - eps_l);
    S.lp = round_up_f(1.0 + eps_l);
    S.qa = round_up_f(1.0 + eps_q);
    S.qp = round_down_f(1.0 - eps_q);
}

// ---------------------------------------------------------------------------
// Caching allocators (device and pinned host), per context.

struct Pool {
    bool device = true;
    std::multimap<size_t, void*> free_blocks;
    std::map<void*, size_t> sizes;
    size_t cached = 0;

    static size_t round(size_t n) {
        const size_t g = 2u << 20;
        return ((n ? n : 1) + g - 1) / g * g;
    }

    void* alloc(size_t n) {
        n = round(n);
        auto it = free_blocks.lower_bound(n);
        if (it != free_blocks.end() && it->first <= 2 * n) {
            void* p = it->second;
            cached -= it->first;
            free_blocks.erase(it);
            return p;
        }
        void* p = nullptr;
        cudaError_t e = device ? cudaMalloc(&p, n) : cudaMallocHost(&p, n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            trim();
            e = device ? cudaMalloc(&p, n) : cudaMallocHost(&p, n);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
        }
        sizes[p] = n;
        return p;
    }

    void release(void* p) {
        if (!p) return;
        auto it = sizes.find(p);
        if (it == sizes.end()) return;
        free_blocks.emplace(it->second, p);
        cached += it->second;
    }

    void trim() {
        for (auto& kv : free_blocks) {
            if (device) cudaFree(kv.second); else cudaFreeHost(kv.second);
            sizes.erase(kv.second);
        }
        free_blocks.clear();
        cached = 0;
    }

    ~Pool() {
        for (auto& kv : sizes) {
            if (device) cudaFree(kv.first); else cudaFreeHost(kv.first);
        }
    }
};

}  // namespace

struct cvg_ctx {
    int device = 0;
    int sms = 0;
    size_t total_mem = 0;
    std::vector<cudaEvent_t> events;  // recycled timing events
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // D2H of finished chunks while later chunks compute
    cudaStream_t tail_stream = nullptr;  // per-range counts/totals of a pipelined search
    cudaStream_t aux_stream = nullptr;   // second range view of split plans
    std::recursive_mutex mu;
    // pair total of the last pipelined search of the same shape: sizes the
    // pinned result so repeated searches never grow it
    uint64_t hint_sig[4] = {0, 0, 0, 0};
    uint64_t hint_pairs = 0;
    // scratch layout of the one-shot codec calls (cvg_paint_blocks / cvg_block_sums)
    cvg_layout* codec_layout = nullptr;
    Pool dev;
    Pool host;
};

void layout_free(cvg_layout* L);  // codec section below

struct cvg_plan {
    cvg_ctx* ctx = nullptr;
    int mode = 0, out = 0, path = 0;
    int32_t n = 0, nr = 0, na = 0;
    uint64_t candidates = 0;
    int grid = 0;
    bool empty = false;
    LaunchArgs args{};
    // device allocations (from ctx->dev)
    void* d_const = nullptr;  // search consts + grid tables + thresholds
    void* d_work = nullptr;   // status + ticket + counts + stats (memset per run)
    size_t work_bytes = 0;
    void* d_first = nullptr;
    size_t first_bytes = 0;
    void* d_scratch = nullptr;
    void* d_out_idx = nullptr;
    void* d_out_codes = nullptr;
    uint64_t capacity = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // PAIRS: after phase 1, after the scan; split: [0] phase 1 of view a, [1]
    // phase 1 of view b, [2] scan of view a (fork/join), [3] join of view b
    cudaEvent_t marks[4] = {nullptr, nullptr, nullptr, nullptr};
    bool split = false;
    LaunchArgs va{}, vb{};  // the two range views of a split plan
    bool ran = false;
    cudaStream_t last_stream = nullptr;
    uint64_t input_bytes = 0;
    void* stage = nullptr;  // pinned staging of the constant blob (held until the plan is released)
    uint64_t* h_counts = nullptr;  // pinned per-search counts for cvg_plan_sync
    int32_t n_unique = 0;
    double t_prep_end = 0, t_upload_end = 0;
};

namespace {

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
void dedup_searches(const cvg_search_desc* d, std::vector<uint32_t>& sc_index, std::vector<int32_t>& uniq) {
    const int n = d->n_searches;
    sc_index.clear();
    uniq.clear();
    if (n <= 0) return;
    // uniform classifier? (chunked so the 8M-search screen runs on all cores)
    const size_t parts = n >= (1 << 20) ? 64 : 1;
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
        const size_t chunks = n >= (1 << 20) ? 64 : 1;
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
        struct Key {
            uint32_t rgb;
            int32_t bits;
            double v, r;
            bool operator==(const Key& o) const {
                return rgb == o.rgb && bits == o.bits && std::memcmp(&v, &o.v, 8) == 0 &&
                       std::memcmp(&r, &o.r, 8) == 0;
            }
        };
        struct Hash {
            size_t operator()(const Key& k) const {
                uint64_t a, b;
                std::memcpy(&a, &k.v, 8);
                std::memcpy(&b, &k.r, 8);
                uint64_t h = (static_cast<uint64_t>(k.rgb) << 3 | static_cast<uint64_t>(k.bits)) * 0x9E3779B97F4A7C15ull;
                h ^= a + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
                h ^= b + 0x85157AF5ull + (h << 6) + (h >> 2);
                return static_cast<size_t>(h);
            }
        };
        std::unordered_map<Key, int32_t, Hash> seen;
        seen.reserve(static_cast<size_t>(n) * 2);
        for (int s = 0; s < n; ++s) {
            const Key k{key24(static_cast<size_t>(s)), d->pattern_bits[s], d->v_th[s], d->r_novib[s]};
            auto [it, fresh] = seen.emplace(k, static_cast<int32_t>(uniq.size()));
            if (fresh) uniq.push_back(s);
            sc_index[s] = static_cast<uint32_t>(it->second);
        }
    }
    if (static_cast<int>(uniq.size()) == n) {
        sc_index.clear();  // all distinct: records are in search order
    }
}

// Grid tables shared by every search (and every range of a pipelined search).
struct GridTables {
    std::vector<float> radii_f;
    std::vector<float> trig_f;   // (sin/500, cos/200) per angle, padded by 128 entries
    std::vector<double> trig_d;  // (sin, cos) per angle
};

GridTables make_grid_tables(const cvg_search_desc* d) {
    GridTables g;
    g.radii_f.resize(d->n_radii);
    for (int k = 0; k < d->n_radii; ++k) g.radii_f[k] = static_cast<float>(d->radii[k]);
    // float trig table padded by 128 entries: the hot loop prefetches two chunks ahead
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

int plan_build(cvg_ctx* ctx, const cvg_search_desc* d, cvg_plan* p, const GridTables* grid = nullptr,
               const SearchConst* pre = nullptr) {
    const Tables& T = tables();
    p->ctx = ctx;
    // TargetSwing (quantized or continuous) is a per-endpoint interval test:
    // band mode.  Quantized FrameDiff classifies on the codes of both endpoints.
    p->mode = d->delta_basis == CVG_BASIS_TARGET_SWING ? cvg::kModeBand : cvg::kModeCodes;
    p->out = d->output;
    p->path = d->path;
    p->n = d->n_searches;
    p->nr = d->n_radii;
    p->na = d->n_angles;
    const uint64_t cps = static_cast<uint64_t>(p->nr) * static_cast<uint64_t>(p->na);
    p->candidates = cps * static_cast<uint64_t>(p->n);
    p->empty = p->candidates == 0;
    if (p->empty) return CVG_OK;  // search.cpp:409-411

    const uint32_t tps = static_cast<uint32_t>((cps + cvg::kTile - 1) / cvg::kTile);
    const uint64_t n_tiles = static_cast<uint64_t>(tps) * static_cast<uint64_t>(p->n);
    if (n_tiles >= (1ull << 28)) return fail(CVG_EINVAL, "batch too large for one plan (split the searches)");

    // ---- host tables ----
    // Per-search constants, deduplicated: searches with the same (target,
    // pattern, v_th, r_novib) share one record (per-pixel batches repeat
    // colors); every candidate of every search is still evaluated.
    std::vector<uint32_t> sc_index;
    std::vector<SearchConst> sc_own;
    const SearchConst* sc_ptr = pre;  // one record per search, built by the caller
    size_t n_sc = static_cast<size_t>(p->n);
    if (!pre) {
        std::vector<int32_t> uniq;  // representative search of each record
        dedup_searches(d, sc_index, uniq);
        sc_own.resize(uniq.size());
        const double rmax = d->radii[p->nr - 1];
        parallel_for(uniq.size(), [&](size_t u) { make_search_const(d, uniq[u], rmax, p->mode, T, sc_own[u]); });
        sc_ptr = sc_own.data();
        n_sc = sc_own.size();
    }
    p->n_unique = static_cast<int32_t>(n_sc);
    GridTables own;
    if (!grid) {
        own = make_grid_tables(d);
        grid = &own;
    }
    const std::vector<float>& radii_f = grid->radii_f;
    const std::vector<float>& trig_f = grid->trig_f;
    const std::vector<double>& trig_d = grid->trig_d;

    // Claim order (band mode, more than one loud count in the batch): all
    // tiles of the searches with one loud count, then the next, so the warps
    // resident together run one band_row specialization (instruction cache).
    std::vector<uint32_t> claim;
    std::array<uint32_t, 3> group_end{};
    static const bool group_claims = [] {
        const char* e = std::getenv("CVG_CLAIM_GROUP");  // A/B switch; default on
        return !e || std::atoi(e) != 0;
    }();
    if (group_claims && p->mode == cvg::kModeBand && p->n > 1) {
        std::array<uint32_t, 4> bucket{};
        for (int32_t i = 0; i < p->n; ++i) ++bucket[__builtin_popcount(d->pattern_bits[i] & 7)];
        int kinds = 0;
        for (uint32_t b : bucket) kinds += b > 0;
        if (kinds > 1) {
            // positions: loud count 1 first ([0, group_end[0])), then 2, then 3
            group_end[0] = bucket[1];
            group_end[1] = bucket[1] + bucket[2];
            group_end[2] = bucket[1] + bucket[2] + bucket[3];
            std::array<uint32_t, 4> next{0, 0, group_end[0], group_end[1]};
            claim.resize(p->n);
            for (int32_t i = 0; i < p->n; ++i) claim[next[__builtin_popcount(d->pattern_bits[i] & 7)]++] = i;
        }
    }

    // ---- one constant blob: [sc | sc_index | claim | radii | trig | thresholds | guess] ----
    Layout L;
    const size_t o_sc = L.take(sizeof(SearchConst) * n_sc);
    const size_t o_si = L.take(sizeof(uint32_t) * sc_index.size());
    const size_t o_co = L.take(sizeof(uint32_t) * claim.size());
    const size_t o_rd = L.take(sizeof(double) * p->nr);
    const size_t o_rf = L.take(sizeof(float) * p->nr);
    const size_t o_td = L.take(sizeof(double) * trig_d.size());
    const size_t o_tf = L.take(sizeof(float) * trig_f.size());
    const size_t o_thd = L.take(sizeof(double) * 256);
    const size_t o_thf = L.take(sizeof(float) * 256 * 4);
    const size_t o_gs = L.take(cvg::kGuessBuckets + 1);
    const size_t bytes = L.off;
    p->input_bytes = bytes;
    p->t_prep_end = now_ms();
    unsigned char* stage = static_cast<unsigned char*>(ctx->host.alloc(bytes));
    p->d_const = ctx->dev.alloc(bytes);
    if (!stage || !p->d_const) {
        ctx->host.release(stage);
        return fail(CVG_ENOMEM, "allocation of the search tables failed");
    }
    std::memcpy(stage + o_sc, sc_ptr, sizeof(SearchConst) * n_sc);
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
    std::memcpy(stage + o_thf, T.thr3, sizeof(float) * 256 * 4);
    std::memcpy(stage + o_gs, T.guess, cvg::kGuessBuckets + 1);
    LaunchArgs& A = p->args;
    std::memset(&A, 0, sizeof(A));
    A.sc = at<const SearchConst>(p->d_const, o_sc);
    A.sc_index = sc_index.empty() ? nullptr : at<const uint32_t>(p->d_const, o_si);
    A.claim_order = claim.empty() ? nullptr : at<const uint32_t>(p->d_const, o_co);
    for (int g = 0; g < 3; ++g) A.group_end[g] = group_end[g];
    A.radii_d = at<const double>(p->d_const, o_rd);
    A.radii_f = at<const float>(p->d_const, o_rf);
    A.trig_d = at<const double>(p->d_const, o_td);
    A.trig_f = at<const float>(p->d_const, o_tf);
    A.thr_d = at<const double>(p->d_const, o_thd);
    A.thr3 = at<const float>(p->d_const, o_thf);
    A.guess = at<const uint8_t>(p->d_const, o_gs);
    // No sync: the staging block stays with the plan until it is released,
    // which happens after the stream has passed this copy.
    p->stage = stage;
    cudaError_t e = cudaMemcpyAsync(p->d_const, stage, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "upload of the search tables");
    p->t_upload_end = now_ms();

    for (int i = 0; i < 9; ++i) A.minv[i] = kXyzToRgb.m[i / 3][i % 3];
    A.n_searches = p->n;
    A.nr = p->nr;
    A.na = p->na;
    A.aligned = (p->na % 32) == 0;
    A.tiles_per_search = tps;
    A.cand_per_search = static_cast<uint32_t>(cps);
    A.na_magic = p->na > 1 ? (UINT64_MAX / static_cast<uint64_t>(p->na)) + 1 : 0;
    A.n_tiles = n_tiles;

    // ---- per-run workspace --------------------------------------------------
    // zeroed each run:  status[n_scan_blocks] | tickets[8] | counts[n] | stats | total | total_a | total_b
    // written each run: tile_count[n_tiles] | tile_base[n_tiles] | worklist   (PAIRS)
    const bool pairs = p->out == cvg::kOutPairs;
    const int per_sm = cvg::search_blocks_per_sm(p->mode, p->out, p->path);
    if (per_sm <= 0) {
        cudaError_t le = cudaGetLastError();
        return fail(CVG_ECUDA, std::string("search kernel cannot be resident on this device (") +
                                   cudaGetErrorString(le) + "); sm_100a image required");
    }
    // Two range views on two streams (PAIRS): the second range's phase 1
    // fills the first's tail, and the first's scan + emit fill the second's.
    // Measured neutral on cfg1/cfg2/cfg3 (the second range's persistent
    // blocks hold every slot until its own tail, so the first range's emit
    // only starts there), hence off unless CVG_SPLIT=1.
    static const bool allow_split = [] {
        const char* e = std::getenv("CVG_SPLIT");
        return e && std::atoi(e) != 0;
    }();
    const uint64_t resident_warps = static_cast<uint64_t>(per_sm) * ctx->sms * cvg::kWarpsPerBlock;
    p->split = allow_split && pairs && p->n >= 2 && n_tiles >= 8 * resident_warps;
    const uint32_t n_a = p->split ? static_cast<uint32_t>(p->n / 2) : static_cast<uint32_t>(p->n);
    const uint64_t tiles_a = static_cast<uint64_t>(n_a) * tps, tiles_b = n_tiles - tiles_a;
    const uint64_t scan_a = pairs ? (tiles_a + cvg::kScanTile - 1) / cvg::kScanTile : 0;
    const uint64_t scan_b = p->split ? (tiles_b + cvg::kScanTile - 1) / cvg::kScanTile : 0;
    Layout W;
    const size_t o_st = W.take(sizeof(unsigned long long) * (scan_a + scan_b));
    const size_t o_tk = W.take(sizeof(unsigned int) * 8);
    const size_t o_ct = W.take(sizeof(unsigned long long) * p->n);
    const size_t o_ss = W.take(sizeof(cvg::Stats));
    const size_t o_to = W.take(sizeof(unsigned long long));  // stats+total read back as one ChunkTail
    const size_t o_ta = W.take(sizeof(unsigned long long) * 2);  // per-view totals (split)
    p->work_bytes = W.off;  // memset span
    const size_t o_tc = W.take(sizeof(uint32_t) * (pairs ? n_tiles : 0));
    const size_t o_tb = W.take(sizeof(unsigned long long) * (pairs ? n_tiles : 0));
    const size_t o_wl = W.take(sizeof(uint32_t) * (pairs ? n_tiles * (cvg::kTile / cvg::kEmitSpan) : 0));
    p->d_work = ctx->dev.alloc(W.off);
    if (!p->d_work) return fail(CVG_ENOMEM, "device allocation of the workspace failed");
    A.status = at<unsigned long long>(p->d_work, o_st);
    A.ticket = at<unsigned int>(p->d_work, o_tk);
    A.counts = at<unsigned long long>(p->d_work, o_ct);
    A.stats = at<cvg::Stats>(p->d_work, o_ss);
    A.tile_count = at<uint32_t>(p->d_work, o_tc);
    A.tile_base = at<unsigned long long>(p->d_work, o_tb);
    A.total = at<unsigned long long>(p->d_work, o_to);
    A.worklist = at<uint32_t>(p->d_work, o_wl);
    A.search_begin = 0;
    A.range_searches = static_cast<uint32_t>(p->n);
    A.tile_begin = 0;
    A.base_offset = nullptr;
    A.grand_total = nullptr;
    if (pairs) {
        p->d_scratch = ctx->dev.alloc(static_cast<size_t>(n_tiles) * cvg::kTile * sizeof(uint16_t));
        if (!p->d_scratch) return fail(CVG_ENOMEM, "device allocation of the tile lists failed");
        A.scratch = static_cast<uint16_t*>(p->d_scratch);
    }
    if (p->out == cvg::kOutFirst) {
        Layout F;
        const size_t o_fi = F.take(sizeof(uint32_t) * p->n);
        const size_t o_fc = F.take(static_cast<size_t>(p->n) * 6);
        p->first_bytes = F.off;
        p->d_first = ctx->dev.alloc(p->first_bytes);
        if (!p->d_first) return fail(CVG_ENOMEM, "device allocation of the first-pair buffer failed");
        A.first_idx = at<uint32_t>(p->d_first, o_fi);
        A.first_codes = at<uint8_t>(p->d_first, o_fc);
    }

    if (p->split) {
        unsigned long long* totals = at<unsigned long long>(p->d_work, o_ta);
        A.claim_order = nullptr;  // range views claim in search order
        p->va = A;
        p->va.range_searches = n_a;
        p->va.n_tiles = tiles_a;
        p->va.total = totals;
        p->vb = A;
        p->vb.search_begin = n_a;
        p->vb.range_searches = static_cast<uint32_t>(p->n) - n_a;
        p->vb.tile_begin = tiles_a;
        p->vb.n_tiles = tiles_b;
        p->vb.status = A.status + scan_a;
        p->vb.ticket = A.ticket + 4;
        p->vb.total = totals + 1;
        p->vb.worklist = A.worklist + tiles_a * (cvg::kTile / cvg::kEmitSpan);
        p->vb.base_offset = totals;
        p->vb.grand_total = A.total;
    }
    const uint64_t want = (n_tiles + cvg::kWarpsPerBlock - 1) / cvg::kWarpsPerBlock;
    p->grid = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(per_sm) * ctx->sms, want));
    if (p->grid < 1) p->grid = 1;
    for (cudaEvent_t* ev : {&p->ev0, &p->ev1, &p->marks[0], &p->marks[1], &p->marks[2], &p->marks[3]}) {
        if (!ctx->events.empty()) {
            *ev = ctx->events.back();
            ctx->events.pop_back();
        } else {
            CVG_CUDA(cudaEventCreate(ev));
        }
    }

    if (p->out == cvg::kOutPairs) {
        // Initial capacity: every candidate when it fits in half the free memory.
        const uint64_t fit = static_cast<uint64_t>(ctx->total_mem / 4 / 10);  // a quarter of HBM at most
        uint64_t cap = std::min<uint64_t>(p->candidates, std::max<uint64_t>(fit, 1u << 20));
        if (int e2 = plan_reserve(p, cap)) return e2;
    }
    return CVG_OK;
}

int plan_build_safe(cvg_ctx* ctx, const cvg_search_desc* d, cvg_plan* p, const GridTables* grid = nullptr,
                    const SearchConst* pre = nullptr) {
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
    if (p->out == cvg::kOutFirst) CVG_CUDA(cudaMemsetAsync(p->d_first, 0xff, static_cast<size_t>(p->n) * 4, st));
    CVG_CUDA(cudaEventRecord(p->ev0, st));
    if (p->split) {
        // the views copy the output buffers, which cvg_plan_reserve may have replaced
        for (LaunchArgs* v : {&p->va, &p->vb}) {
            v->out_idx = p->args.out_idx;
            v->out_codes = p->args.out_codes;
            v->capacity = p->args.capacity;
        }
        cudaStream_t aux = p->ctx->aux_stream;
        CVG_CUDA(cudaStreamWaitEvent(aux, p->ev0, 0));
        CVG_CUDA(cvg::launch_phase1(p->va, p->mode, p->out, p->path, p->grid, st));
        CVG_CUDA(cudaEventRecord(p->marks[0], st));
        CVG_CUDA(cvg::launch_phase1(p->vb, p->mode, p->out, p->path, p->grid, aux));
        CVG_CUDA(cudaEventRecord(p->marks[1], aux));
        CVG_CUDA(cvg::launch_scan(p->va, st));
        CVG_CUDA(cudaEventRecord(p->marks[2], st));
        CVG_CUDA(cvg::launch_emit(p->va, p->mode, p->path, p->grid, st));
        CVG_CUDA(cvg::launch_scan(p->vb, aux));
        CVG_CUDA(cudaStreamWaitEvent(aux, p->marks[2], 0));  // view b's pairs start after view a's total
        CVG_CUDA(cvg::launch_emit(p->vb, p->mode, p->path, p->grid, aux));
        CVG_CUDA(cudaEventRecord(p->marks[3], aux));
        CVG_CUDA(cudaStreamWaitEvent(st, p->marks[3], 0));
    } else {
        CVG_CUDA(cvg::launch_search(p->args, p->mode, p->out, p->path, p->grid, st, p->marks));
        if (p->out == cvg::kOutFirst) CVG_CUDA(cvg::launch_first_codes(p->args, st));
    }
    CVG_CUDA(cudaEventRecord(p->ev1, st));
    return CVG_OK;
}

struct HostStats {
    cvg::Stats st{};
    float ms = 0.f;
};

// Waits for the last run; copies counts (into pinned `counts`) and stats to host.
int plan_collect(cvg_plan* p, uint64_t* counts, HostStats& hs) {
    if (p->empty) {
        if (p->n) std::memset(counts, 0, sizeof(uint64_t) * p->n);
        return CVG_OK;
    }
    cudaStream_t st = p->last_stream;
    CVG_CUDA(cudaMemcpyAsync(counts, p->args.counts, sizeof(uint64_t) * p->n, cudaMemcpyDeviceToHost, st));
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
    if (p->out == cvg::kOutPairs) {
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
    } else if (p->out == cvg::kOutFirst && n) {
        r->d2h_bytes += n * 10;
        r->first_idx = static_cast<uint32_t*>(ctx->host.alloc(n * 4));
        r->first_codes = static_cast<uint8_t*>(ctx->host.alloc(n * 6));
        if (!r->first_idx || !r->first_codes) return fail(CVG_ENOMEM, "pinned host allocation failed");
        cudaStream_t st = p->last_stream;
        CVG_CUDA(cudaMemcpyAsync(r->first_idx, p->args.first_idx, n * 4, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaMemcpyAsync(r->first_codes, p->args.first_codes, n * 6, cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaStreamSynchronize(st));
    }
    return CVG_OK;
}

// cvg_result keeps a pointer to its context in a side table so that
// cvg_result_free can return pinned blocks to the right pool.
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
    return forced > 0 ? std::min(forced, d->n_searches) : 4;
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
    const GridTables grid = make_grid_tables(d);
    double prep = 0, h2d = 0, t_first_enqueued = 0;
    int err = CVG_OK;
    for (int c = 0; c < K && !err; ++c) {
        const size_t lo = n * c / K, hi = n * (c + 1) / K;
        cvg_search_desc sub = *d;
        sub.n_searches = static_cast<int32_t>(hi - lo);
        sub.target_rgb = d->target_rgb + 3 * lo;
        sub.pattern_bits = d->pattern_bits + lo;
        sub.v_th = d->v_th + lo;
        sub.r_novib = d->r_novib + lo;
        const double tb = now_ms();
        err = plan_build_safe(ctx, &sub, &plans[c], &grid);
        if (err) break;
        prep += (plans[c].t_prep_end ? plans[c].t_prep_end : now_ms()) - tb;
        h2d += plans[c].t_upload_end ? plans[c].t_upload_end - plans[c].t_prep_end : 0.0;
        if (!ctx->events.empty()) {
            kdone[c] = ctx->events.back();
            ctx->events.pop_back();
        } else if (cudaEventCreate(&kdone[c]) != cudaSuccess) {
            err = fail(CVG_ECUDA, "event creation failed");
            break;
        }
        err = plan_enqueue(&plans[c], ctx->stream);
        if (err) break;
        if (c == 0) t_first_enqueued = now_ms();
        const cvg_plan& p = plans[c];
        auto copy = [&]() -> int {
            cudaStream_t cs = ctx->copy_stream;
            CVG_CUDA(cudaEventRecord(kdone[c], ctx->stream));
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
    for (int c = 0; c < K; ++c) {
        if (kdone[c]) ctx->events.push_back(kdone[c]);
        if (plans[c].ctx) plan_release(&plans[c]);
    }
    ctx->host.release(tails);
    return err;
}

int search_pipelined(cvg_ctx* ctx, const cvg_search_desc* d, cvg_result* r, int K) {
    const double t0 = now_ms();
    const size_t n = static_cast<size_t>(d->n_searches);
    const uint64_t cps = static_cast<uint64_t>(d->n_radii) * static_cast<uint64_t>(d->n_angles);
    const GridTables grid = make_grid_tables(d);
    // every record up front, on all cores (ranges are too small to thread well)
    std::vector<SearchConst> recs(n);
    {
        const Tables& T = tables();
        const int mode = d->delta_basis == CVG_BASIS_TARGET_SWING ? cvg::kModeBand : cvg::kModeCodes;
        const double rmax = d->radii[d->n_radii - 1];
        parallel_for(n, [&](size_t s) { make_search_const(d, static_cast<int>(s), rmax, mode, T, recs[s]); }, 64);
    }
    const double t_recs = now_ms();
    r->n_searches = d->n_searches;
    r->counts = static_cast<uint64_t*>(ctx->host.alloc(sizeof(uint64_t) * n));
    r->offsets = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (n + 1)));
    auto* tails = static_cast<ChunkTail*>(ctx->host.alloc(sizeof(ChunkTail) * K));
    if (!r->counts || !r->offsets || !tails) {
        ctx->host.release(tails);
        return fail(CVG_ENOMEM, "host allocation failed");
    }
    std::vector<cvg_plan> plans(K);
    const std::vector<size_t> lo = ramp_bounds(n, K);
    std::vector<cudaEvent_t> done(K, nullptr), kdone(K, nullptr);  // tails landed / kernels finished
    PinnedPairs out{ctx};
    const uint64_t sig[4] = {n, cps, static_cast<uint64_t>(d->delta_basis), static_cast<uint64_t>(d->path)};
    const bool hinted = std::equal(sig, sig + 4, ctx->hint_sig);
    uint64_t used = 0;
    double prep = t_recs - t0, h2d = 0, t_last_done = 0;
    cvg::Stats agg{};
    float agg_ratio = 0.f, kernel_ms = 0.f;
    int err = CVG_OK;
    static const bool trace = std::getenv("CVG_TRACE") != nullptr;
    std::vector<cudaEvent_t> copied(trace ? K : 0, nullptr);
    for (auto& e : copied) cudaEventCreate(&e);
    std::vector<std::pair<const char*, double>> tl;
    auto mark = [&](const char* what) {
        if (trace) tl.emplace_back(what, now_ms() - t0);
    };

    auto enqueue_tail = [&](int c) -> int {
        // counts and [stats | total] of the range on the tail stream: the
        // compute stream goes on with the next range, never queued behind
        // a pair copy on the D2H engine
        cvg_plan& p = plans[c];
        cudaStream_t st = ctx->tail_stream;
        CVG_CUDA(cudaEventRecord(kdone[c], ctx->stream));
        CVG_CUDA(cudaStreamWaitEvent(st, kdone[c], 0));
        CVG_CUDA(cudaMemcpyAsync(r->counts + lo[c], p.args.counts, sizeof(uint64_t) * (lo[c + 1] - lo[c]),
                                 cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaMemcpyAsync(&tails[c], p.args.stats, sizeof(ChunkTail), cudaMemcpyDeviceToHost, st));
        CVG_CUDA(cudaEventRecord(done[c], st));
        return CVG_OK;
    };
    auto drain = [&](int c) -> int {
        cvg_plan& p = plans[c];
        mark("drain");
        CVG_CUDA(cudaEventSynchronize(done[c]));
        mark("done");
        if (tails[c].st.overflow) {  // device pair buffer too small: rerun this range at its exact size
            if (int e = plan_reserve(&p, tails[c].total)) return e;
            if (int e = plan_enqueue(&p, ctx->stream)) return e;
            if (int e = enqueue_tail(c)) return e;
            CVG_CUDA(cudaEventSynchronize(done[c]));
            if (tails[c].st.overflow) return fail(CVG_ECUDA, "pair buffer overflow after resizing");
        }
        t_last_done = now_ms();
        const uint64_t tc = tails[c].total;
        const uint64_t seen = cps * lo[c + 1];  // candidates through this chunk
        const uint64_t extrap = (used + tc) * ((cps * n + seen - 1) / seen) + (used + tc) / 4 + (1u << 16);
        const uint64_t want = hinted ? std::max(ctx->hint_pairs, used + tc) : extrap;
        if (!out.ensure(used + tc, std::min<uint64_t>(want, cps * n), used)) {
            return fail(CVG_ENOMEM, "pinned host allocation failed");
        }
        if (tc) {
            CVG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, done[c], 0));
            CVG_CUDA(cudaMemcpyAsync(out.idx + used, p.d_out_idx, tc * 4, cudaMemcpyDeviceToHost, ctx->copy_stream));
            CVG_CUDA(cudaMemcpyAsync(out.codes + 6 * used, p.d_out_codes, tc * 6, cudaMemcpyDeviceToHost,
                                     ctx->copy_stream));
        }
        if (trace) cudaEventRecord(copied[c], ctx->copy_stream);
        mark("issued");
        used += tc;
        const cvg::Stats& s = tails[c].st;
        agg.band_repairs += s.band_repairs;
        agg.code_repairs += s.code_repairs;
        agg.audit_violations += s.audit_violations;
        agg.class_mismatch += s.class_mismatch;
        float ratio;
        std::memcpy(&ratio, &s.audit_max_ratio_bits, sizeof(float));
        agg_ratio = std::max(agg_ratio, ratio);
        float ms = 0.f;
        CVG_CUDA(cudaEventElapsedTime(&ms, p.ev0, p.ev1));
        kernel_ms += ms;
        return CVG_OK;
    };

    mark("grid");
    int next = 0;  // first range not yet drained
    for (int c = 0; c < K && !err; ++c) {
        cvg_search_desc sub = *d;
        sub.n_searches = static_cast<int32_t>(lo[c + 1] - lo[c]);
        sub.target_rgb = d->target_rgb + 3 * lo[c];
        sub.pattern_bits = d->pattern_bits + lo[c];
        sub.v_th = d->v_th + lo[c];
        sub.r_novib = d->r_novib + lo[c];
        const double tb = now_ms();
        err = plan_build_safe(ctx, &sub, &plans[c], &grid, recs.data() + lo[c]);
        if (err) break;
        prep += (plans[c].t_prep_end ? plans[c].t_prep_end : now_ms()) - tb;
        h2d += plans[c].t_upload_end ? plans[c].t_upload_end - plans[c].t_prep_end : 0.0;
        for (cudaEvent_t* ev : {&done[c], &kdone[c]}) {
            if (!ctx->events.empty()) {
                *ev = ctx->events.back();
                ctx->events.pop_back();
            } else if (cudaEventCreate(ev) != cudaSuccess) {
                err = fail(CVG_ECUDA, "event creation failed");
            }
        }
        if (err) break;
        mark("built");
        err = plan_enqueue(&plans[c], ctx->stream);
        if (!err) err = enqueue_tail(c);
        mark("enqueued");
        // start the read-back of every finished range without blocking the builds
        while (!err && next < c) {
            const cudaError_t q = cudaEventQuery(done[next]);
            if (q == cudaErrorNotReady) {
                cudaGetLastError();  // not an error: the range is still running
                break;
            }
            err = q == cudaSuccess ? drain(next++) : cuda_fail(q, "range completion");
        }
    }
    while (!err && next < K) err = drain(next++);
    if (!err) {
        cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
        if (ce != cudaSuccess) err = cuda_fail(ce, "pair read-back");
    }
    const double t1 = now_ms();
    if (!err) {
        r->idx = used ? out.idx : nullptr;
        r->codes = used ? out.codes : nullptr;
        if (!used) {
            ctx->host.release(out.idx);
            ctx->host.release(out.codes);
        }
        r->offsets[0] = 0;
        for (size_t s = 0; s < n; ++s) r->offsets[s + 1] = r->offsets[s] + r->counts[s];
        r->n_pairs = used;
        r->n_candidates = cps * n;
        r->n_band_repairs = agg.band_repairs;
        r->n_code_repairs = agg.code_repairs;
        r->n_audit_violations = agg.audit_violations;
        r->n_class_mismatch = agg.class_mismatch;
        r->audit_max_ratio = agg_ratio;
        r->kernel_ms = kernel_ms;
        uint64_t in_bytes = 0;
        for (const cvg_plan& p : plans) in_bytes += p.input_bytes;
        r->h2d_bytes = in_bytes;
        r->d2h_bytes = sizeof(uint64_t) * n + (sizeof(ChunkTail)) * K + used * 10;
        r->prep_ms = static_cast<float>(prep);
        r->h2d_ms = static_cast<float>(h2d);
        r->device_ms = static_cast<float>(t_last_done - t0 - prep - h2d);
        r->d2h_ms = static_cast<float>(t1 - t_last_done);
        r->total_ms = static_cast<float>(t1 - t0);
        std::copy(sig, sig + 4, ctx->hint_sig);
        ctx->hint_pairs = used;
    } else {
        cudaStreamSynchronize(ctx->copy_stream);
        ctx->host.release(out.idx);
        ctx->host.release(out.codes);
    }
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->tail_stream);
    if (trace) {
        mark("end");
        std::string line = "[cvg trace] K=" + std::to_string(K);
        for (auto& [w, t] : tl) line += std::string(" ") + w + "@" + std::to_string(t).substr(0, 6);
        for (int c = 0; c < K && !err; ++c) {
            float a = 0, b = 0, x = 0, m0 = 0, m1 = 0;
            cudaEventElapsedTime(&a, plans[0].ev0, plans[c].ev0);
            cudaEventElapsedTime(&b, plans[0].ev0, plans[c].ev1);
            cudaEventElapsedTime(&x, plans[0].ev0, copied[c]);
            cudaEventElapsedTime(&m0, plans[c].ev0, plans[c].marks[0]);
            cudaEventElapsedTime(&m1, plans[c].ev0, plans[c].marks[1]);
            line += " | r" + std::to_string(c) + " n=" + std::to_string(lo[c + 1] - lo[c]) + " pairs=" +
                    std::to_string(tails[c].total) + " gpu " + std::to_string(a).substr(0, 5) + "-" +
                    std::to_string(b).substr(0, 5) + " (p1 " + std::to_string(m0).substr(0, 5) + " scan@" +
                    std::to_string(m1).substr(0, 5) + ") copied@" + std::to_string(x).substr(0, 5);
        }
        std::fprintf(stderr, "%s\n", line.c_str());
        for (auto& e : copied) cudaEventDestroy(e);
    }
    for (int c = 0; c < K; ++c) {
        if (done[c]) ctx->events.push_back(done[c]);
        if (kdone[c]) ctx->events.push_back(kdone[c]);
        if (plans[c].ctx) plan_release(&plans[c]);
    }
    ctx->host.release(tails);
    return err;
}

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================

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
        std::lock_guard<std::mutex> lk(g_owner_mu);
        for (auto it = g_owner.begin(); it != g_owner.end();) {
            it = it->second == ctx ? g_owner.erase(it) : std::next(it);
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
        CVG_CUDA(cudaMemcpyAsync(counts, p->args.counts, sizeof(uint64_t) * p->n, cudaMemcpyDeviceToDevice, st));
    }
    if (idx && n_pairs) CVG_CUDA(cudaMemcpyAsync(idx, p->d_out_idx, 4 * n_pairs, cudaMemcpyDeviceToDevice, st));
    if (codes && n_pairs) CVG_CUDA(cudaMemcpyAsync(codes, p->d_out_codes, 6 * n_pairs, cudaMemcpyDeviceToDevice, st));
    return CVG_OK;
}

int cvg_plan_device_outputs(cvg_plan* p, uint64_t** counts, uint32_t** idx, uint8_t** codes, uint64_t* capacity) {
    if (!p) return fail(CVG_EINVAL, "null plan");
    if (counts) *counts = reinterpret_cast<uint64_t*>(p->args.counts);
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

int cvg_plan_last_phase_ms(cvg_plan* p, float* phase1_ms, float* scan_ms, float* emit_ms) {
    if (!p || !phase1_ms || !scan_ms || !emit_ms) return fail(CVG_EINVAL, "null plan or output");
    *phase1_ms = *scan_ms = *emit_ms = 0.f;
    if (p->empty || !p->ran) return CVG_OK;
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    CVG_CUDA(cudaEventSynchronize(p->ev1));
    if (p->out != cvg::kOutPairs) return cudaEventElapsedTime(phase1_ms, p->ev0, p->ev1) == cudaSuccess
                                             ? CVG_OK : fail(CVG_ECUDA, "event timing failed");
    if (p->split) {
        // phase 1 = until both views' phase 1 ended; scan + emit = the rest
        // (view a's scan and emit overlap view b's phase 1 and are not split out)
        float a = 0.f, b = 0.f, all = 0.f;
        CVG_CUDA(cudaEventElapsedTime(&a, p->ev0, p->marks[0]));
        CVG_CUDA(cudaEventElapsedTime(&b, p->ev0, p->marks[1]));
        CVG_CUDA(cudaEventElapsedTime(&all, p->ev0, p->ev1));
        *phase1_ms = std::max(a, b);
        *emit_ms = all - *phase1_ms;
        return CVG_OK;
    }
    CVG_CUDA(cudaEventElapsedTime(phase1_ms, p->ev0, p->marks[0]));
    CVG_CUDA(cudaEventElapsedTime(scan_ms, p->marks[0], p->marks[1]));
    CVG_CUDA(cudaEventElapsedTime(emit_ms, p->marks[1], p->ev1));
    return CVG_OK;
}

int cvg_plan_launches(const cvg_plan* p) {
    if (!p || p->empty) return 0;
    if (p->split) return 6;
    return p->out == cvg::kOutPairs ? 3 : p->out == cvg::kOutFirst ? 2 : 1;
}

uint64_t cvg_plan_candidates(const cvg_plan* p) { return p ? p->candidates : 0; }

int cvg_search(cvg_ctx* ctx, const cvg_search_desc* desc, cvg_result* out) {
    if (!ctx || !out) return fail(CVG_EINVAL, "null context or result");
    result_zero(out);
    if (int e = validate_desc(desc)) return e;
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
    if (const int K = std::max({pipeline_chunks(desc), fixed_chunks(desc), K_min}); K > 1) {
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

int cvg_validate(const cvg_search_desc* desc) { return validate_desc(desc); }

void cvg_result_free(cvg_result* r) {
    if (!r) return;
    std::free(r->offsets);
    for (void* ptr : {static_cast<void*>(r->counts), static_cast<void*>(r->idx), static_cast<void*>(r->codes), static_cast<void*>(r->first_idx),
                      static_cast<void*>(r->first_codes)}) {
        if (!ptr) continue;
        cvg_ctx* owner = nullptr;
        {
            std::lock_guard<std::mutex> lk(g_owner_mu);
            auto it = g_owner.find(ptr);
            if (it != g_owner.end()) {
                owner = it->second;
                g_owner.erase(it);
            }
        }
        if (owner) {
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

double cvg_measure_ffma_peak(int device, float* ms_out) { return cvg::measure_ffma_peak(device, ms_out); }

}  // extern "C"

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
