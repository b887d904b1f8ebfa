// cvg_host.h -- internal header of the host library (libcolorvibe_gpu.so):
// the context, plan and pools shared by the host translation units
//   cvg_prep.cpp        reference-exact host tables, validation, per-search constants
//   cvg_plan.cpp        plans (build / run / fetch) and the plan, context and scalar C-ABI
//   cvg_search.cpp      cvg_search and its pipelined read-back paths
//   cvg_codec_host.cpp  the codec passes' C-ABI
// Compiled with the reference's FP flags (-ffp-contract=off, no errno/traps)
// so every double computed on the host -- target Lab (glibc pow/cbrt),
// per-angle sin/cos (glibc), the quantization threshold table (bisection over
// glibc pow), the per-target hoisted constants -- carries the same bits as the
// reference (src/color.cpp:57-70, src/search.cpp:341-370, 414-419,
// src/convert_kernel.hpp:123-146).  Every candidate is evaluated on the GPU
// (cvg_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <unistd.h>

#include <algorithm>
#include <array>
#include <bit>
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

namespace cvg::host {

extern thread_local std::string g_error;  // cvg_last_error()
double now_ms();
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace cvg::host

#define CVG_CUDA(call)                                                  \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) return ::cvg::host::cuda_fail(_e, #call); \
    } while (0)

namespace cvg::host {

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

double f_lab(double t);
double f_lab_inv(double u);
double eotf(double u);
double oetf(double x);
int quantize(double linear);
double signal_value(double linear);  // 255 * oetf(clamp(x, 0, 1)) (convert_kernel.hpp:109-112)
const double* white_or_d65(const double* wp);
void to_lab(const int32_t c[3], const double* wp, double lab[3]);
void to_linear(const double lab[3], const double* wp, double lin[3]);

// Quantization thresholds: thr[c] = smallest double x with quantize(x) >= c,
// found by bisection over the glibc-pow quantizer (convert_kernel.hpp:127-141).
struct Tables {
    double thr[256];
    // Code table over kGuessBuckets + 1 round-to-nearest buckets of linear
    // [0, 1] (bucket i: x * 4096 in [i - 1/2, i + 1/2]), each widened by
    // cvg::kCodeSlack on both sides.  Entry {t, c}: c = number of float
    // thresholds tf = float(thr[1..255]) below the widened bucket, t = the one
    // tf inside it (+inf if none, NaN if two or more).  For x in the bucket and
    // E = eps_code <= kCodeSlack, |x - t| > E proves code(x64) = c + (x >= t).
    float ctab[cvg::kGuessBuckets + 1][2];
    // Signal table (Continuous x FrameDiff prefilter) over the same buckets:
    // {L, U} with L <= signal_value(x) <= U for every double x in
    // [(i - 1/2) / 4096, (i + 1/2) / 4096] (signal_value is monotone; the
    // bounds are rounded outward to float with a 1e-9 allowance for glibc pow).
    float stab[cvg::kGuessBuckets + 1][2];
    // FrameDiff linear-space bounds (QuantTable thresholds, clamped values):
    // |code(p) - code(m)| >= k1 needs |x_p - x_m| > fd_loud[k1] =
    // min_c (thr[c + k1 - 1] - thr[c]); |code(p) - code(m)| <= q0 needs
    // |x_p - x_m| < fd_quiet[q0] = max_c (thr[min(c + q0 + 1, 256)] - thr[c]),
    // thr[256] = 1 (x clamped to [0, 1]).  k1 = 256 / q0 = 255: +inf.
    double fd_loud[257];
    double fd_quiet[256];
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
        for (int i = 0; i <= cvg::kGuessBuckets; ++i) {
            const double lo = (i - 0.5) / cvg::kGuessBuckets - cvg::kCodeSlack;
            const double hi = (i + 0.5) / cvg::kGuessBuckets + cvg::kCodeSlack;
            int below = 0, inside = 0;
            float t = INFINITY;
            for (int c = 1; c < 256; ++c) {
                const double tf = static_cast<float>(thr[c]);
                if (tf < lo) {
                    ++below;
                } else if (tf <= hi) {
                    ++inside;
                    t = static_cast<float>(tf);
                }
            }
            ctab[i][0] = inside > 1 ? NAN : t;
            ctab[i][1] = std::bit_cast<float>(below);
            const double sl = signal_value((i - 0.5) / cvg::kGuessBuckets) - 1e-9;
            const double su = signal_value((i + 0.5) / cvg::kGuessBuckets) + 1e-9;
            float fl = static_cast<float>(sl), fu = static_cast<float>(su);
            if (fl > sl) fl = std::nextafter(fl, -INFINITY);
            if (fu < su) fu = std::nextafter(fu, INFINITY);
            stab[i][0] = fl;
            stab[i][1] = fu;
        }
        for (int k1 = 1; k1 <= 256; ++k1) {
            double d = INFINITY;
            for (int c = 1; k1 <= 255 && c + k1 - 1 <= 255; ++c) d = std::min(d, thr[c + k1 - 1] - thr[c]);
            fd_loud[k1] = d;
        }
        fd_loud[0] = -INFINITY;  // unused (k1 >= 1)
        for (int q0 = 0; q0 <= 255; ++q0) {
            double d = 0.0;
            for (int c = 0; q0 < 255 && c <= 255; ++c) d = std::max(d, (c + q0 + 1 >= 256 ? 1.0 : thr[c + q0 + 1]) - thr[c]);
            fd_quiet[q0] = q0 >= 255 ? INFINITY : d;
        }
    }
    int code(double x) const {
        if (x <= 0.0) return 0;
        if (x >= 1.0) return 255;
        return static_cast<int>(std::upper_bound(thr + 1, thr + 256, x) - thr) - 1;
    }
};

const Tables& tables();

// Validation, mirroring the reference's checks and messages
// (color.cpp:27-39, search.cpp:22-30, 49-56, 92-111).
int validate_color(const int32_t* c);
int validate_grid(const double* radii, int nr, const double* angles, int na);
int validate_thresholds(double v_th, double r_novib);
int validate_desc(const cvg_search_desc* d);
int validate_header(const cvg_search_desc* d);  // validate_desc without the per-search scan

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
            published_.store(b.gen, std::memory_order_release);
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
            // A search runs several short parallel sections back to back:
            // poll for the next batch for a while before sleeping on the
            // condition variable (a futex wake-up costs tens of microseconds).
            static const int spin_us = [] {
                const char* e = std::getenv("CVG_POOL_SPIN_US");
                return e ? std::atoi(e) : 200;
            }();
            const auto t0 = std::chrono::steady_clock::now();
            while (published_.load(std::memory_order_acquire) == seen &&
                   std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(spin_us)) {
                __builtin_ia32_pause();
            }
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
    std::atomic<uint64_t> published_{0};  // generation_, readable without the lock
    uint64_t generation_ = 0;
    bool stop_ = false;
    static thread_local bool in_job_;
};
inline thread_local bool WorkerPool::in_job_ = false;

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

float round_up_f(double x);
float round_down_f(double x);
double signal_value(double linear);
// The per-search record: FP32 constants with their proven error bounds and
// the FP64 hoisted values of the reference (cvg_prep.cpp).
void make_search_const(const cvg_search_desc* d, int s, double rmax, int mode, const Tables& T, SearchConst& S);

// Kernel family of a search (cvg_layout.h Mode): TargetSwing (quantized or
// continuous) is a per-endpoint interval test (band); Quantized FrameDiff
// classifies on the codes of both endpoints; Continuous FrameDiff on the
// difference of the two signal values.
inline int search_mode(const cvg_search_desc* d) {
    if (d->delta_basis == CVG_BASIS_TARGET_SWING) return cvg::kModeBand;
    return d->delta_mode == CVG_DELTA_QUANTIZED ? cvg::kModeCodes : cvg::kModeSignal;
}

// CVG_EUNDECIDED with the count of continuous-FrameDiff decisions that fell
// inside the device/glibc pow margin.
int undecided_fail(unsigned long long n);

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

    // Hands an outstanding block to its holder: the pool forgets it (its
    // destructor will not free it); the holder frees it with the raw API.
    bool detach(void* p) {
        auto it = sizes.find(p);
        if (it == sizes.end()) return false;
        sizes.erase(it);
        return true;
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

}  // namespace cvg::host

struct cvg_ctx {
    int device = 0;
    int sms = 0;
    size_t total_mem = 0;
    std::vector<cudaEvent_t> events;  // recycled timing events
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // D2H of finished chunks while later chunks compute
    cudaStream_t tail_stream = nullptr;  // per-range counts/totals of a pipelined search
    cudaStream_t aux_stream = nullptr;   // emits of a streamed search (concurrent with phase 1)
    std::recursive_mutex mu;
    // pair total of the last pipelined search of the same shape: sizes the
    // pinned result so repeated searches never grow it
    uint64_t hint_sig[4] = {0, 0, 0, 0};
    uint64_t hint_pairs = 0;
    // scratch layout of the one-shot codec calls (cvg_paint_blocks / cvg_block_sums)
    cvg_layout* codec_layout = nullptr;
    cvg::host::Pool dev;
    cvg::host::Pool host;
};

void layout_free(cvg_layout* L);  // cvg_codec_host.cpp

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
    // PAIRS: [0] after phase 1, [1] after the scan (pipelined searches use [2], [3] per view)
    cudaEvent_t marks[4] = {nullptr, nullptr, nullptr, nullptr};
    bool phase_marks = false;  // record marks between the kernels (breaks their PDL overlap)
    bool marked = false;       // the last run recorded them
    bool external_out = false;  // the caller supplies the pair buffers (streamed search): no reserve
    bool ran = false;
    cudaStream_t last_stream = nullptr;
    uint64_t input_bytes = 0;
    void* stage = nullptr;  // pinned staging of the constant blob (held until the plan is released)
    uint64_t* h_counts = nullptr;  // pinned per-search counts for cvg_plan_sync
    int32_t n_unique = 0;
    double t_prep_end = 0, t_upload_end = 0;
    // CVG_PATH_MEMO: the kernels run the n_exec distinct searches (records in
    // representative order); scatter_kernel expands their counts / first
    // pairs to all n searches through map (= sc_index, device)
    bool memo = false;
    // CVG_OUT_BEST: the PAIRS kernels, then best_kernel (select_best per
    // search on the device pair buffer) into the first_* arrays
    bool best = false;
    bool twin = false;  // PAIRS: twin tiles (LaunchArgs::twin)
    const double* d_bands = nullptr;  // BEST: (v_th, low_band) per search
    int32_t n_exec = 0;
    const uint32_t* d_map = nullptr;
    void* d_memo = nullptr;
    void* d_masks = nullptr;  // PAIRS on strip tiles: pass words (LaunchArgs::masks)
    // where the per-search results of a run land (args.* unless memo)
    unsigned long long* res_counts = nullptr;
    uint32_t* res_first_idx = nullptr;
    uint8_t* res_first_codes = nullptr;
};

namespace cvg::host {

// Grid tables shared by every search (and every range of a pipelined search).
struct GridTables {
    std::vector<float> radii_f;
    std::vector<float> trig_f;   // (sin/500, cos/200) per angle, padded by 128 entries
    std::vector<double> trig_d;  // (sin, cos) per angle
};
GridTables make_grid_tables(const cvg_search_desc* d);

int ensure_device(cvg_ctx* ctx);
void plan_free_outputs(cvg_plan* p);
int plan_reserve(cvg_plan* p, uint64_t cap);
void plan_set_density(cvg_plan* p, uint64_t expected_pairs);
int plan_build_safe(cvg_ctx* ctx, const cvg_search_desc* d, cvg_plan* p, const GridTables* grid = nullptr,
                    const SearchConst* pre = nullptr);
void plan_release(cvg_plan* p);
int plan_enqueue(cvg_plan* p, cudaStream_t st);
struct HostStats {
    cvg::Stats st{};
    float ms = 0.f;
};

// Waits for the last run; copies counts (into pinned `counts`) and stats to host.
int plan_collect(cvg_plan* p, uint64_t* counts, HostStats& hs);
uint64_t sum_counts(const uint64_t* c, size_t n);
void result_zero(cvg_result* r);
int plan_fetch_impl(cvg_plan* p, cvg_result* r, bool allow_rerun);
// cvg_result_free returns pinned blocks to the pool of the context recorded here.
void remember_owner(cvg_result* r, cvg_ctx* ctx);

}  // namespace cvg::host
