// cvg_kernels.cu -- fused color-pair search for B200 (sm_100a).
//
// Three kernels per batch of searches (one stream, K2/K3 by programmatic
// dependent launch):
//
//   K1 phase1_kernel  persistent; each warp claims 4096-candidate tiles (a
//            contiguous range of one search's canonical index i = k*na + m)
//            from a global ticket.  It synthesizes every candidate in
//            registers from (target, r_k, theta_m) -- no per-candidate HBM
//            traffic besides the L1/L2-resident trig table -- runs the Lab ->
//            linear RGB conversion and the band test of the reference batch
//            path (search.cpp:230-278, 291-329) in FP32 with a proven
//            per-channel error bound, and sends the rare candidates whose
//            decision lies inside that bound through the FP64 op-for-op
//            restatement (bit-identical to the reference).  Passing offsets
//            are appended to the tile's ordered list with ballot/popc (the
//            reference's pass-2 extraction, search.cpp:379-397), or counted
//            (COUNTS / FIRST).  The FrameDiff modes have their own decisions
//            (code bounds; FP32 signal bounds) with the same FP64 fallback.
//   K2 scan_kernel  exclusive scan of the tile counts (chained, decoupled
//            look-back): each tile's output offset in the global canonical
//            order, independent of scheduling (search.cpp:448-455).
//   K3 emit_kernel  warps walk the lists 32 pairs at a time (all lanes busy),
//            recompute the six linear values, quantize them through the code
//            table with the same bound (FP64 repair when unsure) and write
//            idx + 6 code bytes with coalesced stores.
//
// Result: per-search counts and pair lists bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>


#include "cvg_internal.h"
#include "cvg_layout.h"

namespace cvg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Reference constants (convert_kernel.hpp:50-60), evaluated in double.
constexpr double kLabEpsilon = 216.0 / 24389.0;
constexpr double kInvKappa = 27.0 / 24389.0;
constexpr double kInv500 = 1.0 / 500.0;
constexpr double kInv200 = 1.0 / 200.0;

// FP32 fast-path constants: f^-1(u) = u^3 above u0 = 6/29, else the tangent
// line (116u - 16) * 27/24389 = K1*u - K2 (the two branches are C1-tangent at
// u0, so a branch flip next to u0 costs O(du^2), covered by the bound).
constexpr float kU0f = 6.0f / 29.0f;
constexpr float kK1f = 3132.0f / 24389.0f;
constexpr float kK2f = 432.0f / 24389.0f;


constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Programmatic dependent launch: scan and emit launch while their
// predecessor drains (its CTAs trigger when they run out of work) and wait
// here for its completion and memory before touching its outputs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ const SearchConst* search_const(const LaunchArgs& A, uint32_t s) {
    return A.sc + (A.sc_index ? __ldg(&A.sc_index[s]) : s);
}

__device__ __forceinline__ uint32_t div_na(uint32_t i, const LaunchArgs& A) {
    return A.na == 1 ? i : static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(i), A.na_magic));
}

// ------------------------------------------------------------------------
// Per-search constants held in registers for a tile (phase 1, band form;
// channel slots loud-first).
struct Consts {
    float fx0, fz0, rcube;
    float cube[6];  // SearchConst::cube: {fx0^3, 3 fx0^2, 3 fx0, fz0^3, 3 fz0^2, 3 fz0}
    float mxs[3], mzs[3], cys[3];
    float la, qa, lp, qp;
    uint32_t flags;
};

__device__ __forceinline__ void load_consts(const SearchConst* S, Consts& c) {
    c.fx0 = __ldg(&S->fx0);
    c.fz0 = __ldg(&S->fz0);
    c.rcube = __ldg(&S->rcube);
#pragma unroll
    for (int q = 0; q < 6; ++q) c.cube[q] = __ldg(&S->cube[q]);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        c.mxs[q] = __ldg(&S->mxs[q]);
        c.mzs[q] = __ldg(&S->mzs[q]);
        c.cys[q] = __ldg(&S->cys[q]);
    }
    c.la = __ldg(&S->la);
    c.qa = __ldg(&S->qa);
    c.lp = __ldg(&S->lp);
    c.qp = __ldg(&S->qp);
    c.flags = __ldg(&S->flags);
}

// Constants for the code path (phase 2 and CODES mode).
struct CodeConsts {
    float fx0, fz0, rcube;
    float mx[3], mz[3], cy[3], ec[3];
    uint32_t tab;  // code_fast's table address (ctab_addr), computed once per kernel
};

__device__ __forceinline__ void load_code_consts(const SearchConst* S, CodeConsts& c, uint32_t tab) {
    c.tab = tab;
    c.fx0 = __ldg(&S->fx0);
    c.fz0 = __ldg(&S->fz0);
    c.rcube = __ldg(&S->rcube);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        c.mx[q] = __ldg(&S->mx[q]);
        c.mz[q] = __ldg(&S->mz[q]);
        c.cy[q] = __ldg(&S->cy[q]);
        const float e = __ldg(&S->eps_code[q]);
        c.ec[q] = e <= kCodeSlack ? e : INFINITY;  // beyond the table's slack: every code goes to FP64
    }
}

// ------------------------------------------------------------------------
// FP64 exact path: op-for-op restatement of the reference batch row
// (search.cpp:243-262 with convert_kernel.hpp:70-73), no contraction.

__device__ __forceinline__ double finv_exact(double u) {
    const double u3 = __dmul_rn(__dmul_rn(u, u), u);
    return u3 > kLabEpsilon ? u3 : __dmul_rn(__dsub_rn(__dmul_rn(116.0, u), 16.0), kInvKappa);
}

__device__ __forceinline__ void exact_linear_inl(const SearchConst* S, const LaunchArgs& A, uint32_t k,
                                                 uint32_t m, double* lp, double* lm) {
    const double r = __ldg(&A.radii_d[k]);
    const double s = __ldg(&A.trig_d[2 * m]);
    const double c = __ldg(&A.trig_d[2 * m + 1]);
    const double fy = __ldg(&S->fy), ta = __ldg(&S->ta), tb = __ldg(&S->tb);
    const double wx = __ldg(&S->wx), wz = __ldg(&S->wz);
    const double da = __dmul_rn(r, s);
    const double db = __dmul_rn(r, c);
    const double fxp = __dadd_rn(fy, __dmul_rn(__dadd_rn(ta, da), kInv500));
    const double fzp = __dsub_rn(fy, __dmul_rn(__dadd_rn(tb, db), kInv200));
    const double xp = __dmul_rn(wx, finv_exact(fxp));
    const double zp = __dmul_rn(wz, finv_exact(fzp));
    const double fxm = __dadd_rn(fy, __dmul_rn(__dsub_rn(ta, da), kInv500));
    const double fzm = __dsub_rn(fy, __dmul_rn(__dsub_rn(tb, db), kInv200));
    const double xm = __dmul_rn(wx, finv_exact(fxm));
    const double zm = __dmul_rn(wz, finv_exact(fzm));
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double cy = __ldg(&S->cy64[q]);
        lp[q] = __dadd_rn(__dadd_rn(__dmul_rn(A.minv[3 * q], xp), cy), __dmul_rn(A.minv[3 * q + 2], zp));
        lm[q] = __dadd_rn(__dadd_rn(__dmul_rn(A.minv[3 * q], xm), cy), __dmul_rn(A.minv[3 * q + 2], zm));
    }
}

// Out-of-line copy for the rare repair sites of the hot kernels.
__device__ __noinline__ void exact_linear(const SearchConst* S, const LaunchArgs& A, uint32_t k, uint32_t m,
                                          double* lp, double* lm) {
    exact_linear_inl(S, A, k, m, lp, lm);
}

// QuantTable::code (convert_kernel.hpp:148-154): largest c with x >= thr[c].
__device__ __forceinline__ int code_exact(double x, const double* thr) {
    if (x <= 0.0) return 0;
    if (x >= 1.0) return 255;
    int c = 0;
#pragma unroll
    for (int step = 128; step; step >>= 1) {
        if (x >= thr[c + step]) c += step;
    }
    return c;
}

// Band predicate of pass1_row (search.cpp:267-276) on exact values.
__device__ __forceinline__ bool exact_band(const SearchConst* S, const double* lp, const double* lm,
                                           uint32_t flags) {
    bool ok = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double lo = __ldg(&S->lo[q]), hi = __ldg(&S->hi[q]);
        const bool in = (lp[q] >= lo) & (lp[q] < hi) & (lm[q] >= lo) & (lm[q] < hi);
        const bool loud = (flags >> q) & 1;
        ok &= in != loud;
    }
    return ok;
}

// signal_value (convert_kernel.hpp:109-112) of an exact linear value, with
// the radius `e` of |s_dev - s_ref| (s_ref: the reference's glibc result).
// Clamped values and the linear branch of srgb_oetf (convert_kernel.hpp:81-83)
// are op-for-op exact (e = 0).  On the pow branch the device pow differs from
// glibc's by at most 2 (CUDA) + 0.52 (glibc) ulp of t <= 1; propagated through
// 1.055*t - 0.055 and *255 (one rounding each, 1 ulp apart at most) that is
// 255 * (1.055 * 3 * 2^-53 + 2 * 2^-52) + 2^-45 < 2.4e-13; e = 5e-13.
__device__ __forceinline__ double signal_dev(double lin, double& e) {
    const double x = lin < 0.0 ? 0.0 : (lin > 1.0 ? 1.0 : lin);
    double y;
    e = 0.0;
    if (x <= 0.0031308) {
        y = __dmul_rn(12.92, x);
    } else {
        const double t = pow(x, 1.0 / 2.4);
        y = __dsub_rn(__dmul_rn(1.055, t), 0.055);
        if (x != 1.0) e = 5e-13;  // pow(1, y) == 1 exactly on both sides
    }
    return __dmul_rn(255.0, y);
}

// classify_pair (search.cpp:146-157) on continuous FrameDiff deltas
// |s(p) - s(m)| (continuous_deltas, search.cpp:161-173), decided with the
// margin of signal_dev: d_dev within e_p + e_m + 2^-44 (rounding of the
// difference, values < 256) of a threshold is undecided (counted; the call
// then fails instead of guessing).  lo[c] holds the channel's threshold.
__device__ __forceinline__ bool signal_pass(const SearchConst* S, const double* lp, const double* lm,
                                            uint32_t flags, bool& undecided) {
    bool ok = true;
    undecided = false;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        double ep, em;
        const double sp = signal_dev(lp[q], ep);
        const double sm = signal_dev(lm[q], em);
        const double d = fabs(__dsub_rn(sp, sm));
        const double mg = ep + em > 0.0 ? ep + em + 0x1p-44 : 0.0;
        const double T = __ldg(&S->lo[q]);
        const bool loud = (flags >> q) & 1;
        // loud: d > v_th; quiet: d <= low
        const bool pass = loud ? d > T : d <= T;
        const bool sure = loud ? (d - mg > T) | (d + mg <= T) : (d + mg <= T) | (d - mg > T);
        ok &= pass;
        undecided |= !sure;
    }
    return ok;
}

// ---- Continuous x FrameDiff FP32 prefilter ------------------------------
__device__ __forceinline__ float add_rm_sat(float a, float b) {
    float d;
    asm("add.rm.sat.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float add_rp_sat(float a, float b) {
    float d;
    asm("add.rp.sat.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// Per-search constants of the prefilter: the bound on |v32 - v64| and each
// channel's threshold widened to [tl, th] (margin 2^-12 covers the float
// rounding of the threshold and the difference's double rounding).
struct SigConsts {
    float e[3], th[3], tl[3];
    float flo[3], fhi[3];  // SearchConst::fd_bounds: linear-space sure-fail bounds (frame_signal_bounds)
};

__device__ __forceinline__ void load_sig_consts(const SearchConst* S, SigConsts& g) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double T = __ldg(&S->lo[q]);
        g.e[q] = __ldg(&S->eps[q]);
        g.th[q] = __double2float_ru(T + 0x1p-12);
        g.tl[q] = __double2float_rd(T - 0x1p-12);
        g.flo[q] = __ldg(&S->fd_bounds[2 * q]);
        g.fhi[q] = __ldg(&S->fd_bounds[2 * q + 1]);
    }
}

// Bounds [lo, hi] on signal_value(v64) for |v - v64| <= e: the buckets of
// sat(v - e) (rounded down) and sat(v + e) (rounded up) in the signal table
// (Tables::stab, signal_value monotone).  `tab` as in code_fast.
__device__ __forceinline__ void signal_bounds(float v, float e, uint32_t tab, float& lo, float& hi) {
    const float bl = fmaf(add_rm_sat(v, -e), static_cast<float>(kGuessBuckets), 8388608.0f);
    const float bh = fmaf(add_rp_sat(v, e), static_cast<float>(kGuessBuckets), 8388608.0f);
    asm("ld.shared.f32 %0, [%1];" : "=f"(lo) : "r"(tab + (__float_as_uint(bl) << 3)));
    asm("ld.shared.f32 %0, [%1];" : "=f"(hi) : "r"(tab + (__float_as_uint(bh) << 3) + 4u));
}

// classify_pair on continuous FrameDiff deltas (search.cpp:146-173) from the
// bounds: with d in [dmin, dmax], a channel is surely above its threshold if
// dmin > th and surely at or below it if dmax <= tl.  The candidate surely
// fails if any channel surely fails, surely passes if every channel surely
// passes; otherwise `unsure` (the FP64 path decides).
__device__ __forceinline__ bool signal_prefilter(const SigConsts& G, const float* vp, const float* vm, uint32_t tab,
                                                 uint32_t flags, bool& unsure) {
    bool fail = false, all = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        float pl, ph, ml, mh;
        signal_bounds(vp[q], G.e[q], tab, pl, ph);
        signal_bounds(vm[q], G.e[q], tab, ml, mh);
        const float dlo = __fsub_rd(pl, mh), dhi = __fsub_ru(ph, ml);
        const float dmin = fmaxf(fmaxf(dlo, -dhi), 0.0f), dmax = fmaxf(-dlo, dhi);
        const bool above = dmin > G.th[q], below = dmax <= G.tl[q];
        const bool loud = (flags >> q) & 1;
        fail |= loud ? below : above;
        all &= loud ? above : below;
    }
    unsure = !fail & !all;
    return all;
}

// classify_pair (search.cpp:146-157) on integer codes, with the integer form
// of the thresholds (d > v_th <=> d >= k1, d <= low <=> d <= q0).
__device__ __forceinline__ bool classify_codes(const SearchConst* S, const int* cp, const int* cm,
                                               uint32_t flags) {
    const bool frame_diff = (flags >> 8) & 1;
    const int k1 = __ldg(&S->k1), q0 = __ldg(&S->q0);
    bool ok = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int t = __ldg(&S->t[q]);
        int d;
        if (frame_diff) {
            d = abs(cp[q] - cm[q]);
        } else {
            d = max(abs(cp[q] - t), abs(cm[q] - t));
        }
        const bool loud = (flags >> q) & 1;
        ok &= loud ? (d >= k1) : (d <= q0);
    }
    return ok;
}

// ------------------------------------------------------------------------
// FP32 fast path.

template <bool kCubeOnly>
__device__ __forceinline__ float finv_fast(float f) {
    const float c3 = __fmul_rn(__fmul_rn(f, f), f);
    if (kCubeOnly) return c3;
    const float l = fmaf(f, kK1f, -kK2f);
    return f > kU0f ? c3 : l;
}

// The six linear endpoint values (plus: vp, minus: vm) minus an additive
// offset folded into `add` (cy for the values themselves, cy - centre for the
// band statistic).  f = f0 +- r*s' is one FFMA; f^-1 two FMULs (+ select).
__device__ __forceinline__ float fma_sat(float a, float b, float c) {
    float d;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// kSat: the values saturated to [0, 1] in the last FFMA (code_fast input).
template <bool kCubeOnly, bool kSat = false>
__device__ __forceinline__ void fast_linear(float fx0, float fz0, const float* mx, const float* mz, const float* add,
                                            float r, float2 sc, float* vp, float* vm) {
    const float fxp = fmaf(r, sc.x, fx0);
    const float fxm = fmaf(-r, sc.x, fx0);
    const float fzp = fmaf(-r, sc.y, fz0);
    const float fzm = fmaf(r, sc.y, fz0);
    const float gxp = finv_fast<kCubeOnly>(fxp);
    const float gxm = finv_fast<kCubeOnly>(fxm);
    const float gzp = finv_fast<kCubeOnly>(fzp);
    const float gzm = finv_fast<kCubeOnly>(fzm);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        if (kSat) {
            vp[q] = fma_sat(mx[q], gxp, fmaf(mz[q], gzp, add[q]));
            vm[q] = fma_sat(mx[q], gxm, fmaf(mz[q], gzm, add[q]));
        } else {
            vp[q] = fmaf(mx[q], gxp, fmaf(mz[q], gzp, add[q]));
            vm[q] = fmaf(mx[q], gxm, fmaf(mz[q], gzm, add[q]));
        }
    }
}

// Band statistics of the reference band test (search.cpp:267-276,
// make_bands 291-329).  With the matrix rows pre-divided by the band half-
// width h_c and offset by the band centre, channel c of a candidate yields
// M'_c = max(|vp_c - centre_c|, |vm_c - centre_c|) / h_c: a quiet channel
// passes iff M'_c <= 1 (both endpoints inside), a loud one iff M'_c > 1.  The
// host orders the channel slots loud-first, so with L loud channels the
// candidate passes iff minl = min over slots < L of M' > 1 and maxq = max
// over slots >= L of M' <= 1.  |M'32 - M'| is bounded on the host, hence
//   attention (no channel certainly fails): minl >= la and maxq <= qa
//   certain pass:                            minl >  lp and maxq <  qp
// and only attention-but-not-certain candidates go to the FP64 path.
// kL = loud count (1..3), 0 = read it from the flags at run time.
template <int kL, class CT>
__device__ __forceinline__ void band_stats_m(const CT& C, const float* M, float& minl, float& maxq) {
    const int L = kL ? kL : static_cast<int>((C.flags >> 10) & 3u);
    minl = INFINITY;
    maxq = -INFINITY;
    if (kL == 3) {
        minl = fminf(fminf(M[0], M[1]), M[2]);
    } else if (kL == 2) {
        minl = fminf(M[0], M[1]);
        maxq = M[2];
    } else if (kL == 1) {
        minl = M[0];
        maxq = fmaxf(M[1], M[2]);
    } else {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (q < L) minl = fminf(minl, M[q]); else maxq = fmaxf(maxq, M[q]);
        }
    }
}

template <int kL>
__device__ __forceinline__ void band_stats(const Consts& C, const float* dp, const float* dm, float& minl,
                                           float& maxq) {
    float M[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) M[q] = fmaxf(fabsf(dp[q]), fabsf(dm[q]));
    band_stats_m<kL>(C, M, minl, maxq);
}

// Cube-only rows in sum/difference form: with d+- the two endpoint values of
// a channel, A = (d+ + d-)/2 and B = (d+ - d-)/2 give M' = max(|d+|, |d-|)
// = |A| + |B|, and for f+- = f0 +- U in the cube branch
//   A = mxs (fx0^3 + 3 fx0 Ux^2) + mzs (fz0^3 + 3 fz0 Uz^2) + cys
//   B = mxs Ux (3 fx0^2 + Ux^2)  - mzs Uz (3 fz0^2 + Uz^2)
// (Ux = r sin/500, Uz = r cos/200): 10 ops for the cubes and 15 for the
// three channels instead of 4 + 8 + 12 + 3 (static SASS of the two-chunk
// loop body: 70 instructions instead of 74); the host bound (cube_bound,
// make_search_const) covers this form.
template <int kL>
__device__ __forceinline__ void band_cube(const Consts& C, float r, float2 sc, float& minl, float& maxq) {
    const float ux = __fmul_rn(r, sc.x), uz = __fmul_rn(r, sc.y);
    const float ax = fmaf(__fmul_rn(ux, ux), C.cube[2], C.cube[0]);
    const float az = fmaf(__fmul_rn(uz, uz), C.cube[5], C.cube[3]);
    const float bx = __fmul_rn(ux, fmaf(ux, ux, C.cube[1]));
    const float bz = __fmul_rn(uz, fmaf(uz, uz, C.cube[4]));
    float M[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float a = fmaf(C.mxs[q], ax, fmaf(C.mzs[q], az, C.cys[q]));
        const float b = fmaf(C.mxs[q], bx, -__fmul_rn(C.mzs[q], bz));
        M[q] = fabsf(a) + fabsf(b);
    }
    band_stats_m<kL>(C, M, minl, maxq);
}

// Strip form of the cube-only band statistic.  In band_cube, with ux = r s'
// and uz = r c' (s' = sin/500, c' = cos/200 of the lane's angle),
//   A_c = mxs_c (fx0^3 + 3 fx0 ux^2) + mzs_c (fz0^3 + 3 fz0 uz^2) + cys_c
//       = K0_c + r^2 K2_c,
//   B_c = mxs_c ux (3 fx0^2 + ux^2) - mzs_c uz (3 fz0^2 + uz^2)
//       = r L1_c + r^3 L3_c,
// K0_c per search, K2_c, L1_c, L3_c per search and angle: computed once per
// strip (strip_setup), so a candidate costs 2 + 3 operations per channel
// plus |A| + |B| instead of the 25 of band_cube.  r, r^2, r^3 are
// warp-uniform row tables.  make_search_const bounds this FP32 sequence too
// (20u per term magnitude) and the band thresholds cover it; the AUDIT path
// checks it against FP64 on every cube-only candidate.
struct StripConsts {
    float k0[3], k2[3], l1[3], l3[3];
};

// The band thresholds alone (the cube-only strip loop holds no other search
// constant, so the linear-form constants are not live across it).
struct ThrConsts {
    float la, qa, lp, qp;
    uint32_t flags;
};

// A copy of a pointer the compiler cannot see through: loads through it are
// not merged with earlier loads through the original (forces a reload).
template <class T>
__device__ __forceinline__ const T* opaque_ptr(const T* p) {
    asm volatile("" : "+l"(p));
    return p;
}

__device__ __forceinline__ void strip_setup(const Consts& C, float2 sc, StripConsts& Q) {
    const float s2 = __fmul_rn(sc.x, sc.x), c2 = __fmul_rn(sc.y, sc.y);
    const float px = __fmul_rn(C.cube[2], s2), pz = __fmul_rn(C.cube[5], c2);  // 3 f0 s'^2
    const float s1x = __fmul_rn(C.cube[1], sc.x), s1z = __fmul_rn(C.cube[4], sc.y);  // 3 f0^2 s'
    const float s3x = __fmul_rn(s2, sc.x), s3z = __fmul_rn(c2, sc.y);  // s'^3
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        Q.k0[q] = fmaf(C.mxs[q], C.cube[0], fmaf(C.mzs[q], C.cube[3], C.cys[q]));
        Q.k2[q] = fmaf(C.mxs[q], px, __fmul_rn(C.mzs[q], pz));
        Q.l1[q] = fmaf(C.mxs[q], s1x, -__fmul_rn(C.mzs[q], s1z));
        Q.l3[q] = fmaf(C.mxs[q], s3x, -__fmul_rn(C.mzs[q], s3z));
    }
}

// One slot's statistic |A_c| + |B_c| of the strip form.
__device__ __forceinline__ float strip_chan(const StripConsts& Q, int q, float r, float r2, float r3) {
    return fabsf(fmaf(Q.k2[q], r2, Q.k0[q])) + fabsf(fmaf(Q.l3[q], r3, __fmul_rn(Q.l1[q], r)));
}

template <int kL, class CT>
__device__ __forceinline__ void strip_stat(const CT& C, const StripConsts& Q, float r, float r2, float r3,
                                           float& minl, float& maxq) {
    float M[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float a = fmaf(Q.k2[q], r2, Q.k0[q]);
        const float b = fmaf(Q.l3[q], r3, __fmul_rn(Q.l1[q], r));
        M[q] = fabsf(a) + fabsf(b);
    }
    band_stats_m<kL>(C, M, minl, maxq);
}

template <class CT>
__device__ __forceinline__ bool band_attention(const CT& C, float minl, float maxq) {
    return (minl >= C.la) & (maxq <= C.qa);
}

template <class CT>
__device__ __forceinline__ bool band_certain(const CT& C, float minl, float maxq) {
    return (minl > C.lp) & (maxq < C.qp);
}

// Linear value -> code through the code table, verified against the bound:
// the bucket of xs (round-to-nearest) gives {t, c}, the only float threshold
// within kCodeSlack of the bucket and the count below it; c + (xs >= t) is
// the code, and ok iff |xs - t| > E, which proves code(x64) == it (E =
// eps_code <= kCodeSlack; NaN t: never ok).  xs is the FP32 value saturated
// to [0, 1]: the table has no threshold within kCodeSlack of 0 or 1, so a
// value below 0 (above 1) gets code 0 (255) exactly as its FP64 twin does.
// `tab` = shared address of the table minus 8 * bits(2^23).
// The increment is the sign bit of d = t - xs (one LEA.HI): when ok, d != 0
// and sign(d) = (xs > t) = (xs >= t); when not ok the result is c or c + 1
// either way, which is all the callers assume of an unverified code.
__device__ __forceinline__ int code_fast(float xs, float E, uint32_t tab, bool& ok) {
    const float b = fmaf(xs, static_cast<float>(kGuessBuckets), 8388608.0f);  // bits: 0x4B000000 + round(xs * 4096)
    float t;
    int c;
    asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=f"(t), "=r"(c) : "r"(tab + (__float_as_uint(b) << 3)));
    const float d = __fsub_rn(t, xs);
    ok = fabsf(d) > E;
    return c + static_cast<int>(__float_as_uint(d) >> 31);
}

// Passed through a shuffle, so that it is opaque to ptxas and each lookup is
// one LEA off this register (else ptxas re-derives the shared base and the
// constant inside the loop, two more instructions per lookup).
__device__ __forceinline__ uint32_t ctab_addr(const float2* ctab) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(ctab)) - (0x4B000000u << 3);
    return __shfl_sync(0xffffffffu, a, 0);
}

// Exact code from a nearby guess (the FP32 code is off by at most one).
__device__ __forceinline__ int code_exact_from(double x, int c, const double* thr) {
    if (x <= 0.0) return 0;
    if (x >= 1.0) return 255;
    while (c < 255 && x >= thr[c + 1]) ++c;
    while (c > 0 && x < thr[c]) --c;
    return c;
}

// Shared tables: exact quantization thresholds + the FP32 code table.
struct Smem {
    double thr_d[256];
    uint32_t first[kWarpsPerBlock];  // FIRST mode: tile offset of the warp's first passing candidate
    // code table (cvg_host.h Tables::ctab); phase 1 of kModeSignal holds the
    // signal table (Tables::stab) here instead.  Last: kernels without a
    // table omit it.
    float2 ctab[kGuessBuckets + 2];
};

// Dynamic shared memory of phase 1: the code table only where it quantizes.
template <int kMode>
__host__ __device__ constexpr size_t phase1_smem() { return kMode == kModeBand ? offsetof(Smem, ctab) : sizeof(Smem); }

// Dynamic shared memory of the emit kernel: the tables + each warp's repair
// queue (emit_run).
constexpr int kRepairQueueSlots = 64;
constexpr size_t emit_smem() { return sizeof(Smem) + kWarpsPerBlock * kRepairQueueSlots * sizeof(uint2); }

enum Table : int { kTabNone = 0, kTabCode = 1, kTabSignal = 2 };

template <int kTab>
__device__ __forceinline__ void load_tables(Smem& sm, const LaunchArgs& A) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        sm.thr_d[i] = A.thr_d[i];
    }
    if (kTab != kTabNone) {
        const float2* src = reinterpret_cast<const float2*>(kTab == kTabCode ? A.ctab : A.stab);
        for (int i = threadIdx.x; i <= kGuessBuckets; i += blockDim.x) sm.ctab[i] = src[i];
    }
    __syncthreads();
}

struct Counters {
    unsigned long long repairs = 0, code_repairs = 0, violations = 0, mismatch = 0, overflow = 0, undecided = 0;
    float max_ratio = 0.f;
};

__device__ __forceinline__ void flush_counters(Counters& ct, const LaunchArgs& A, unsigned lane) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ct.repairs += __shfl_xor_sync(kFull, ct.repairs, o);
        ct.code_repairs += __shfl_xor_sync(kFull, ct.code_repairs, o);
        ct.violations += __shfl_xor_sync(kFull, ct.violations, o);
        ct.mismatch += __shfl_xor_sync(kFull, ct.mismatch, o);
        ct.overflow += __shfl_xor_sync(kFull, ct.overflow, o);
        ct.undecided += __shfl_xor_sync(kFull, ct.undecided, o);
        ct.max_ratio = fmaxf(ct.max_ratio, __shfl_xor_sync(kFull, ct.max_ratio, o));
    }
    if (lane == 0) {
        if (ct.repairs) atomicAdd(&A.stats->band_repairs, ct.repairs);
        if (ct.code_repairs) atomicAdd(&A.stats->code_repairs, ct.code_repairs);
        if (ct.violations) atomicAdd(&A.stats->audit_violations, ct.violations);
        if (ct.mismatch) atomicAdd(&A.stats->class_mismatch, ct.mismatch);
        if (ct.overflow) atomicAdd(&A.stats->overflow, ct.overflow);
        if (ct.undecided) atomicAdd(&A.stats->undecided, ct.undecided);
        if (ct.max_ratio > 0.f) atomicMax(&A.stats->audit_max_ratio_bits, __float_as_uint(ct.max_ratio));
    }
}

__device__ __forceinline__ void audit_ratio(const SearchConst* S, const float* vp, const float* vm, const double* lp,
                                            const double* lm, float& max_ratio) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double eps = __ldg(&S->eps[q]);
        max_ratio = fmaxf(max_ratio, static_cast<float>(fabs(static_cast<double>(vp[q]) - lp[q]) / eps));
        max_ratio = fmaxf(max_ratio, static_cast<float>(fabs(static_cast<double>(vm[q]) - lm[q]) / eps));
    }
}

// Codes of the six endpoint channels of one candidate from its FP32 values,
// exact: values whose code is not proven by the bound go to FP64 (all six
// values recomputed op-for-op, codes walked from the FP32 guess).  Called by
// all 32 lanes (warp vote inside).
// FP32 codes of the six endpoint channels (code_fast each); true iff all six
// are proven.  Called by all 32 lanes (warp vote inside).
__device__ __forceinline__ bool codes_guess(const CodeConsts& C, float r, float2 sc, int* cp, int* cm) {
    float vp[3], vm[3];
    if (__all_sync(kFull, r < C.rcube)) {  // every lane's row stays on the cube branch
        fast_linear<true, true>(C.fx0, C.fz0, C.mx, C.mz, C.cy, r, sc, vp, vm);
    } else {
        fast_linear<false, true>(C.fx0, C.fz0, C.mx, C.mz, C.cy, r, sc, vp, vm);
    }
    bool all_ok = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        bool ok1, ok2;
        cp[q] = code_fast(vp[q], C.ec[q], C.tab, ok1);
        cm[q] = code_fast(vm[q], C.ec[q], C.tab, ok2);
        all_ok &= ok1 & ok2;
    }
    return all_ok;
}

__device__ __forceinline__ void codes_fast(const Smem& sm, const SearchConst* S, const CodeConsts& C,
                                           const LaunchArgs& A, uint32_t k, uint32_t m, float r, float2 sc,
                                           bool active, int* cp, int* cm, unsigned long long& repairs) {
    const bool all_ok = codes_guess(C, r, sc, cp, cm);
    if (__any_sync(kFull, !all_ok) && !all_ok) {
        double lp[3], lm[3];
        exact_linear_inl(S, A, k, m, lp, lm);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            cp[q] = code_exact_from(lp[q], cp[q], sm.thr_d);
            cm[q] = code_exact_from(lm[q], cm[q], sm.thr_d);
        }
        if (active) ++repairs;
    }
}

// Codes of candidate (k, m) for any path (EXACT: FP64 only; AUDIT: both,
// counting FP32 codes that were "verified" but wrong).
template <int kPath>
__device__ __forceinline__ void candidate_codes(const Smem& sm, const SearchConst* S, const CodeConsts& C,
                                                const LaunchArgs& A, uint32_t k, uint32_t m, bool active,
                                                int* cp, int* cm, unsigned long long& repairs, Counters& ct) {
    const float r = __ldg(&A.radii_f[k]);
    const float2 sc = __ldg(reinterpret_cast<const float2*>(A.trig_f) + m);
    if (kPath == kPathFast) {
        codes_fast(sm, S, C, A, k, m, r, sc, active, cp, cm, repairs);
        return;
    }
    double lp[3], lm[3];
    exact_linear(S, A, k, m, lp, lm);
    if (kPath == kPathExact) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            cp[q] = code_exact(lp[q], sm.thr_d);
            cm[q] = code_exact(lm[q], sm.thr_d);
        }
        return;
    }
    float vp[3], vm[3];
    fast_linear<false>(C.fx0, C.fz0, C.mx, C.mz, C.cy, r, sc, vp, vm);
    bool all_ok = true, wrong = false;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        bool ok1, ok2;
        const int fp = code_fast(__saturatef(vp[q]), C.ec[q], C.tab, ok1);
        const int fm = code_fast(__saturatef(vm[q]), C.ec[q], C.tab, ok2);
        all_ok &= ok1 & ok2;
        cp[q] = code_exact(lp[q], sm.thr_d);
        cm[q] = code_exact(lm[q], sm.thr_d);
        wrong |= (ok1 && fp != cp[q]) | (ok2 && fm != cm[q]);
        // the FP64 walk from the FP32 guess must agree with the binary search
        wrong |= (code_exact_from(lp[q], fp, sm.thr_d) != cp[q]) | (code_exact_from(lm[q], fm, sm.thr_d) != cm[q]);
    }
    if (active) {
        ct.violations += wrong;
        repairs += !all_ok;
        audit_ratio(S, vp, vm, lp, lm, ct.max_ratio);
    }
}

// Phase-1 decision of one candidate, any mode/path (the generic loop).
template <int kMode, int kPath>
__device__ __forceinline__ bool candidate_pass(const Smem& sm, const SearchConst* S, const Consts& C,
                                               const CodeConsts& CC, const SigConsts& SG, const LaunchArgs& A,
                                               uint32_t k, uint32_t m, bool active, Counters& ct) {
    if (kMode == kModeSignal) {
        // FP32 prefilter on signal bounds; unsure lanes (and every lane of
        // the EXACT / AUDIT paths) decide on FP64 linear values + device pow
        // with its margin.
        bool pass = false, unsure = true;
        if (kPath != kPathExact) {
            const float r = __ldg(&A.radii_f[k]);
            const float2 sc = __ldg(reinterpret_cast<const float2*>(A.trig_f) + m);
            float vp[3], vm[3];
            fast_linear<false>(CC.fx0, CC.fz0, CC.mx, CC.mz, CC.cy, r, sc, vp, vm);
            // a channel whose clamped linear difference is outside its
            // linear-space bounds surely fails: skip the signal bounds when
            // every lane has one
            bool lf = false;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const float d = fabsf(__fsub_rn(__saturatef(vp[q]), __saturatef(vm[q])));
                lf |= (d <= SG.flo[q]) | (d >= SG.fhi[q]);
            }
            if (__all_sync(kFull, lf) && kPath == kPathFast) return false;
            pass = signal_prefilter(SG, vp, vm, CC.tab, C.flags, unsure);
            if (lf) {
                pass = false;
                unsure = false;
            }
        }
        if (kPath != kPathFast || (__any_sync(kFull, unsure) && unsure)) {
            double lp[3], lm[3];
            exact_linear(S, A, k, m, lp, lm);
            bool undecided;
            const bool ex = signal_pass(S, lp, lm, C.flags, undecided);
            if (active) {
                ct.undecided += undecided;
                if (kPath != kPathExact) ct.repairs += unsure;
                if (kPath == kPathAudit) ct.violations += !unsure && ex != pass;
            }
            pass = ex;
        }
        return active && pass;
    }
    if (kMode == kModeCodes) {
        int cp[3], cm[3];
        candidate_codes<kPath>(sm, S, CC, A, k, m, active, cp, cm, ct.repairs, ct);
        return active && classify_codes(S, cp, cm, C.flags);
    }
    if (kPath == kPathExact) {
        double lp[3], lm[3];
        exact_linear(S, A, k, m, lp, lm);
        return active && exact_band(S, lp, lm, C.flags);
    }
    const float r = __ldg(&A.radii_f[k]);
    const float2 sc = __ldg(reinterpret_cast<const float2*>(A.trig_f) + m);
    float dp[3], dm[3];
    fast_linear<false>(C.fx0, C.fz0, C.mxs, C.mzs, C.cys, r, sc, dp, dm);
    float minl, maxq;
    band_stats<0>(C, dp, dm, minl, maxq);
    bool pass = band_certain(C, minl, maxq);
    const bool unsure = band_attention(C, minl, maxq) & !pass;
    if (kPath == kPathAudit) {
        double lp[3], lm[3];
        exact_linear(S, A, k, m, lp, lm);
        const bool ex = exact_band(S, lp, lm, C.flags);
        if (r < C.rcube) {  // cube-only rows run the sum/difference form in the fast path
            float l2, q2;
            band_cube<0>(C, r, sc, l2, q2);
            const bool pass2 = band_certain(C, l2, q2);
            const bool unsure2 = band_attention(C, l2, q2) & !pass2;
            if (active) ct.violations += !unsure2 && ex != pass2;
            // and the strip form (strip tiles, COUNTS / FIRST)
            StripConsts Q;
            strip_setup(C, sc, Q);
            const double rd = __ldg(&A.radii_d[k]);
            float l3, q3;
            strip_stat<0>(C, Q, r, static_cast<float>(rd * rd), static_cast<float>(rd * rd * rd), l3, q3);
            const bool pass3 = band_certain(C, l3, q3);
            const bool unsure3 = band_attention(C, l3, q3) & !pass3;
            if (active) ct.violations += !unsure3 && ex != pass3;
        }
        if (active) {
            ct.violations += !unsure && ex != pass;
            ct.repairs += unsure;
            float vp[3], vm[3];
            fast_linear<false>(CC.fx0, CC.fz0, CC.mx, CC.mz, CC.cy, r, sc, vp, vm);
            audit_ratio(S, vp, vm, lp, lm, ct.max_ratio);
        }
        return active && ex;
    }
    if (__any_sync(kFull, unsure) && unsure) {
        double lp[3], lm[3];
        exact_linear(S, A, k, m, lp, lm);
        pass = exact_band(S, lp, lm, C.flags);
        if (active) ++ct.repairs;
    }
    return active && pass;
}

// Appends the passing lanes of one 32-candidate chunk to the tile's list
// (PAIRS: ordered offsets in global scratch; FIRST: remembers the first).
template <int kOut>
__device__ __forceinline__ void append(bool pass, uint32_t off, uint16_t* list, uint32_t& cnt, uint32_t* first,
                                       unsigned lane_lt) {
    const unsigned b = __ballot_sync(kFull, pass);
    if (kOut == kOutPairs) {
        if (pass) list[cnt + __popc(b & lane_lt)] = static_cast<uint16_t>(off);
    } else if (kOut == kOutFirst) {
        // the first passing lane of the tile's first passing chunk records its
        // offset in shared memory (keeps a register free in the hot loop)
        if (cnt == 0 && pass && (b & lane_lt) == 0) *first = off;
    }
    cnt += __popc(b);
}

// Slow path of one chunk (some lane needs attention): FP64 repair of the
// unsure lanes, then the ordered append.
template <int kOut>
__device__ __forceinline__ void band_settle(const SearchConst* S, const Consts& C, const LaunchArgs& A, uint32_t k,
                                            uint32_t m, float minl, float maxq, uint32_t off, uint16_t* list,
                                            uint32_t& cnt, uint32_t* first, Counters& ct, unsigned lane_lt) {
    bool pass = band_certain(C, minl, maxq);
    if (band_attention(C, minl, maxq) & !pass) {
        double lp[3], lm[3];
        exact_linear(S, A, k, m, lp, lm);
        pass = exact_band(S, lp, lm, C.flags);
        ++ct.repairs;
    }
    append<kOut>(pass, off, list, cnt, first, lane_lt);
}

// Slow path of a group of G chunks (some lane needs attention): the certain
// passes, FP64 repair of the unsure lanes behind one vote, then the ordered
// appends.  COUNTS / FIRST append with one ballot per chunk and, while the
// tile has no pass yet, a warp-uniform search for the first passing lane.
template <int kOut, uint32_t G>
__device__ __forceinline__ void band_settle_group(const SearchConst* S, const Consts& C, const LaunchArgs& A,
                                                  uint32_t k, uint32_t ix, const float* lv, const float* qv,
                                                  uint32_t off, uint16_t* list, uint32_t& cnt, uint32_t* first,
                                                  Counters& ct, unsigned lane_lt) {
    bool pass[G], uns[G], any_uns = false;
#pragma unroll
    for (uint32_t g = 0; g < G; ++g) {
        pass[g] = band_certain(C, lv[g], qv[g]);
        uns[g] = band_attention(C, lv[g], qv[g]) & !pass[g];
        any_uns |= uns[g];
    }
    if (__any_sync(kFull, any_uns)) {
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) {
            if (uns[g]) {
                double lp[3], lm[3];
                exact_linear(S, A, k, ix + 32 * g, lp, lm);
                pass[g] = exact_band(S, lp, lm, C.flags);
                ++ct.repairs;
            }
        }
    }
    if (kOut == kOutPairs) {
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) append<kOut>(pass[g], off + 32 * g, list, cnt, first, lane_lt);
    } else {
        unsigned b[G];
        uint32_t n = 0;
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) {
            b[g] = __ballot_sync(kFull, pass[g]);
            n += __popc(b[g]);
        }
        if (kOut == kOutFirst && cnt == 0 && n) {
#pragma unroll
            for (uint32_t g = 0; g < G; ++g) {
                if (b[g]) {
                    if (pass[g] && (b[g] & lane_lt) == 0) *first = off + 32 * g;
                    break;
                }
            }
        }
        cnt += n;
    }
}

template <int kL, bool kCubeOnly>
__device__ __forceinline__ void band_chunk(const Consts& C, float r, float2 sc, float& minl, float& maxq) {
    if (kCubeOnly) {
        band_cube<kL>(C, r, sc, minl, maxq);
    } else {
        float dp[3], dm[3];
        fast_linear<false>(C.fx0, C.fz0, C.mxs, C.mzs, C.cys, r, sc, dp, dm);
        band_stats<kL>(C, dp, dm, minl, maxq);
    }
}

// Hot loop: FAST path, band mode, kL loud channels, `nch` full 32-candidate
// chunks of radius row k starting at angle m0 (na % 32 == 0: chunks never
// straddle rows).  Four chunks per iteration share one vote and one loop
// branch (ILP across chunks); their trig loads are issued together at the
// top of the iteration (L1-resident table; other warps hide the latency).
// Per candidate: 1 LDG, then either 24 FMA-pipe ops (4 f, 8 cube or linear,
// 12 matrix) + 4 min/max, or, in kCubeOnly rows (r < rcube: never the
// linear branch of f^-1), the sum/difference form's 25 ops + 1-2 min/max
// (band_cube).  Measured against two chunks per vote with a two-chunk-ahead
// prefetch (cfg1 / cfg3 / cfg2 / cfg4): 4 per vote +2.5 / +6.3 / +1.5 / +7.4%;
// 2 per vote without prefetch +2 / +2.6 / -3.8%; 3: +0.7 / +2 / -1.9%;
// 6: -7 / +5 / +2.5%; 8: -17 / +4 / +1.6%; 4 with a next-group prefetch
// (register rotation): -6 / 0 / +1.8%.
template <int kL, bool kCubeOnly, int kOut>
__device__ __forceinline__ void band_row(const SearchConst* S, const Consts& C, const LaunchArgs& A, uint32_t k,
                                         float r, uint32_t m0, uint32_t nch, uint32_t off, uint16_t* list,
                                         uint32_t& cnt, uint32_t* first, Counters& ct, unsigned lane,
                                         unsigned lane_lt) {
    constexpr uint32_t G = 4;
    const float2* __restrict__ trig = reinterpret_cast<const float2*>(A.trig_f);
    const uint32_t mb = m0 + lane;
    uint32_t ix = mb;
    const uint32_t iend = mb + 32u * (nch - nch % G);
#pragma unroll 1
    for (; ix != iend; ix += 32 * G) {
        float2 sv[G];
        float lv[G], qv[G];
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) sv[g] = __ldg(trig + ix + 32 * g);
        bool att = false;
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) {
            band_chunk<kL, kCubeOnly>(C, r, sv[g], lv[g], qv[g]);
            att |= band_attention(C, lv[g], qv[g]);
        }
        if (__any_sync(kFull, att))
            band_settle_group<kOut, G>(S, C, A, k, ix, lv, qv, off + lane + (ix - mb), list, cnt, first, ct, lane_lt);
    }
#pragma unroll 1
    for (uint32_t j = nch % G; j; --j, ix += 32) {
        float la_, qa_;
        band_chunk<kL, kCubeOnly>(C, r, __ldg(trig + ix), la_, qa_);
        if (__any_sync(kFull, band_attention(C, la_, qa_))) {
            band_settle<kOut>(S, C, A, k, ix, la_, qa_, off + lane + (ix - mb), list, cnt, first, ct, lane_lt);
        }
    }
}

// ---- Quantized x FrameDiff hot loop ---------------------------------------
// Code bounds instead of exact codes: a code whose FP32 value lies within E
// of its bucket's threshold is c or c + 1 (code_fast), so its computed value
// is off by at most one; with widths w, d = |cp - cm| lies in [d - w, d + w].
// A channel surely passes or fails unless its threshold falls inside that
// range (classify_pair, search.cpp:146-157, frame_deltas :138-144); only
// candidates that are neither sure pass nor sure fail take FP64 codes.
// E beyond kCodeSlack (ec = inf): width 256, every channel unsure.
struct FrameConsts {
    int k1, q0;
    int wc[3];
    float lo[3], hi[3];  // SearchConst::fd_bounds: linear-space sure-fail bounds per channel
};

// Linear-space prefilter: true if some channel surely fails (|v_p - v_m| of
// the saturated FP32 values at or below its loud bound, or at or above its
// quiet bound; make_search_const), so the candidate needs no codes.
__device__ __forceinline__ bool frame_surely_fails(const FrameConsts& F, const float* vp, const float* vm) {
    bool fail = false;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float d = fabsf(__fsub_rn(vp[q], vm[q]));
        fail |= (d <= F.lo[q]) | (d >= F.hi[q]);
    }
    return fail;
}

__device__ __forceinline__ void frame_chunk(const CodeConsts& CC, const FrameConsts& F, uint32_t flags,
                                            const float* vp, const float* vm, bool& att, bool& sure) {
    bool fail = false, all = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        bool okp, okm;
        const int cp = code_fast(vp[q], CC.ec[q], CC.tab, okp);
        const int cm = code_fast(vm[q], CC.ec[q], CC.tab, okm);
        const int w = (okp ? 0 : F.wc[q]) + (okm ? 0 : F.wc[q]);
        const int d = abs(cp - cm);
        const int dmin = d - w, dmax = d + w;  // dmin < 0 is as good as 0 below
        const bool loud = (flags >> q) & 1;
        fail |= loud ? (dmax < F.k1) : (dmin > F.q0);
        all &= loud ? (dmin >= F.k1) : (dmax <= F.q0);
    }
    att = !fail;
    sure = all;
}

template <int kOut>
__device__ __forceinline__ void frame_settle(const Smem& sm, const SearchConst* S, const LaunchArgs& A, uint32_t flags,
                                             uint32_t k, uint32_t m, bool att, bool sure, uint32_t off,
                                             uint16_t* list, uint32_t& cnt, uint32_t* first, Counters& ct,
                                             unsigned lane_lt) {
    bool pass = sure;
    if (att & !sure) {
        double lp[3], lm[3];
        exact_linear(S, A, k, m, lp, lm);
        int cp[3], cm[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            cp[q] = code_exact(lp[q], sm.thr_d);
            cm[q] = code_exact(lm[q], sm.thr_d);
        }
        pass = classify_codes(S, cp, cm, flags);
        ++ct.repairs;
    }
    append<kOut>(pass, off, list, cnt, first, lane_lt);
}

// `nch` full chunks of radius row k from angle m0 (na % 32 == 0), two chunks
// per vote.  The six saturated values of both chunks go through the
// linear-space prefilter first; the code lookups run only when some lane of
// the pair of chunks may pass.
template <int kOut>
__device__ __forceinline__ void frame_row(const Smem& sm, const SearchConst* S, const CodeConsts& CC,
                                          const FrameConsts& F, uint32_t flags, const LaunchArgs& A, uint32_t k,
                                          float r, uint32_t m0, uint32_t nch, uint32_t off, uint16_t* list,
                                          uint32_t& cnt, uint32_t* first, Counters& ct, unsigned lane,
                                          unsigned lane_lt) {
    constexpr uint32_t G = 2;
    const float2* __restrict__ trig = reinterpret_cast<const float2*>(A.trig_f);
    const uint32_t mb = m0 + lane;
    uint32_t ix = mb;
    const uint32_t iend = mb + 32u * (nch - nch % G);
#pragma unroll 1
    for (; ix != iend; ix += 32 * G) {
        float2 sv[G];
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) sv[g] = __ldg(trig + ix + 32 * g);
        float vp[G][3], vm[G][3];
        bool maybe = false;
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) {
            fast_linear<false, true>(CC.fx0, CC.fz0, CC.mx, CC.mz, CC.cy, r, sv[g], vp[g], vm[g]);
            maybe |= !frame_surely_fails(F, vp[g], vm[g]);
        }
        if (!__any_sync(kFull, maybe)) continue;
        bool at[G], su[G], any = false;
#pragma unroll
        for (uint32_t g = 0; g < G; ++g) {
            frame_chunk(CC, F, flags, vp[g], vm[g], at[g], su[g]);
            any |= at[g];
        }
        if (__any_sync(kFull, any)) {
            const uint32_t d = ix - mb;
#pragma unroll
            for (uint32_t g = 0; g < G; ++g)
                frame_settle<kOut>(sm, S, A, flags, k, ix + 32 * g, at[g], su[g], off + lane + d + 32 * g, list, cnt,
                                   first, ct, lane_lt);
        }
    }
    if (nch % G) {
        float vp[3], vm[3];
        fast_linear<false, true>(CC.fx0, CC.fz0, CC.mx, CC.mz, CC.cy, r, __ldg(trig + ix), vp, vm);
        bool at, su;
        frame_chunk(CC, F, flags, vp, vm, at, su);
        if (__any_sync(kFull, at))
            frame_settle<kOut>(sm, S, A, flags, k, ix, at, su, off + lane + (ix - mb), list, cnt, first, ct, lane_lt);
    }
}

template <int kOut>
__device__ __forceinline__ void frame_tile(const Smem& sm, const SearchConst* S, const CodeConsts& CC,
                                           uint32_t flags, const LaunchArgs& A, uint32_t i0, uint32_t i1,
                                           uint16_t* list, uint32_t& cnt, uint32_t* first, Counters& ct,
                                           unsigned lane, unsigned lane_lt) {
    FrameConsts F;
    F.k1 = __ldg(&S->k1);
    F.q0 = __ldg(&S->q0);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        F.wc[q] = CC.ec[q] == INFINITY ? 256 : 1;
        F.lo[q] = __ldg(&S->fd_bounds[2 * q]);
        F.hi[q] = __ldg(&S->fd_bounds[2 * q + 1]);
    }
    uint32_t k = div_na(i0, A);
    uint32_t m0 = i0 - k * static_cast<uint32_t>(A.na);
    uint32_t i = i0;
    while (i < i1) {
        const uint32_t seg = min(i1 - i, static_cast<uint32_t>(A.na) - m0);
        const float r = __ldg(&A.radii_f[k]);
        frame_row<kOut>(sm, S, CC, F, flags, A, k, r, m0, seg >> 5, i - i0, list, cnt, first, ct, lane, lane_lt);
        i += seg;
        m0 = 0;
        ++k;
    }
}

// CVG_PATH_PRUNED: true if every candidate of radius row k surely fails,
// proven in FP64 from the reference's own operation sequence
// (search.cpp:243-262): with |sin|, |cos| <= 1, fx of every candidate lies in
// [fy + (ta - r)/500, fy + (ta + r)/500] and fz in [fy - (tb + r)/200,
// fy - (tb - r)/200] (each rounded operation is monotone), X = wx f^-1(fx) and
// Z = wz f^-1(fz) are monotone, and lin_c = (Minv[c][0] X + cy_c) +
// Minv[c][2] Z takes its extremes at the corners.  A loud channel whose whole
// range lies inside its band [lo, hi) (1e-12 of slack for the f^-1 branch
// switch) never passes (exact_band), so neither does any candidate.
__device__ __forceinline__ bool row_surely_fails(const SearchConst* S, const LaunchArgs& A, uint32_t k) {
    const double r = __ldg(&A.radii_d[k]);
    const double fy = __ldg(&S->fy), ta = __ldg(&S->ta), tb = __ldg(&S->tb);
    const double wx = __ldg(&S->wx), wz = __ldg(&S->wz);
    const double x0 = __dmul_rn(wx, finv_exact(__dadd_rn(fy, __dmul_rn(__dsub_rn(ta, r), kInv500))));
    const double x1 = __dmul_rn(wx, finv_exact(__dadd_rn(fy, __dmul_rn(__dadd_rn(ta, r), kInv500))));
    const double z0 = __dmul_rn(wz, finv_exact(__dsub_rn(fy, __dmul_rn(__dadd_rn(tb, r), kInv200))));
    const double z1 = __dmul_rn(wz, finv_exact(__dsub_rn(fy, __dmul_rn(__dsub_rn(tb, r), kInv200))));
    const uint32_t flags = __ldg(&S->flags);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        if (!((flags >> q) & 1u)) continue;
        const double a0 = __dmul_rn(A.minv[3 * q], x0), a1 = __dmul_rn(A.minv[3 * q], x1);
        const double b0 = __dmul_rn(A.minv[3 * q + 2], z0), b1 = __dmul_rn(A.minv[3 * q + 2], z1);
        const double cy = __ldg(&S->cy64[q]);
        const double vmin = __dadd_rn(__dadd_rn(fmin(a0, a1), cy), fmin(b0, b1));
        const double vmax = __dadd_rn(__dadd_rn(fmax(a0, a1), cy), fmax(b0, b1));
        if (vmin - 1e-12 >= __ldg(&S->lo[q]) && vmax + 1e-12 < __ldg(&S->hi[q])) return true;
    }
    return false;
}

// Rows k0 .. k0 + n - 1 (n <= 32) that row_surely_fails proves empty, one
// row per lane, as a bit mask (one warp-wide FP64 pass per tile).
__device__ __noinline__ uint32_t rows_surely_fail(const SearchConst* S, const LaunchArgs& A, uint32_t k0, uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
    return __ballot_sync(kFull, lane < n && row_surely_fails(S, A, k0 + lane));
}

template <int kL, int kOut, bool kPrune>
__device__ __forceinline__ void band_tile(const SearchConst* S, const Consts& C, const LaunchArgs& A, uint32_t i0,
                                          uint32_t i1, uint16_t* list, uint32_t& cnt, uint32_t* first, Counters& ct,
                                          unsigned lane, unsigned lane_lt) {
    uint32_t k = div_na(i0, A);
    uint32_t m0 = i0 - k * static_cast<uint32_t>(A.na);
    // CVG_PATH_PRUNED: the tile's first 32 rows tested at once
    uint32_t skip = 0;
    if (kPrune) {
        const uint32_t rows = (m0 + (i1 - i0) + static_cast<uint32_t>(A.na) - 1) / static_cast<uint32_t>(A.na);
        skip = rows_surely_fail(S, A, k, min(rows, 32u));
    }
    uint32_t i = i0;
    while (i < i1) {
        const uint32_t seg = min(i1 - i, static_cast<uint32_t>(A.na) - m0);
        const float r = __ldg(&A.radii_f[k]);
        if (kPrune && (skip & 1u)) {
            // no candidate of this row passes: nothing to append
        } else if (r < C.rcube) {
            band_row<kL, true, kOut>(S, C, A, k, r, m0, seg >> 5, i - i0, list, cnt, first, ct, lane, lane_lt);
        } else {
            band_row<kL, false, kOut>(S, C, A, k, r, m0, seg >> 5, i - i0, list, cnt, first, ct, lane, lane_lt);
        }
        i += seg;
        m0 = 0;
        ++k;
        if (kPrune) skip >>= 1;
    }
}

// ---- Strip tiles (COUNTS / FIRST, band FAST path) --------------------------
#ifndef CVG_STRIP_G
#define CVG_STRIP_G 4
#endif
// A strip is 32 consecutive angles (lane l owns angle m0 + l, its trig in
// registers for the whole strip) walked down R radius rows, kStripG rows per
// iteration: the radii are warp-uniform (one broadcast LDG.128 per four
// rows) and a row costs no set-up.  The f^-1 branch is chosen per group of
// rows from the strip's own largest |sin| and |cos| (cube-only while r of the
// group's last row stays under the strip's bound), so only strips near the
// axes pay for the linear branch.  Certain passes are tallied per lane (no
// ballot); each lane keeps its first passing row (rows ascend, so the first
// hit is the lane's smallest).  Lanes inside the FP32 bound but not certain
// are decided in FP64 behind one vote per iteration.  Every candidate is
// evaluated by the same band_chunk under the same proven bound as in the
// row-major loop; only the walk order differs, and the outputs (counts,
// first canonical pair) do not depend on it.
constexpr uint32_t kStripG = CVG_STRIP_G;  // rows per iteration: 4 or 8 (radius groups of 4)


// Rows [k, kend) (kend - k a multiple of kStripG, k % 4 == 0) of the strip,
// one f^-1 form for all of them: kCubeOnly = the strip form (strip_stat,
// constants Q and thresholds T only), else band_chunk (full constants C).
// Fast path: the attention test only, one vote per group; a group with some
// lane that may pass settles: certain passes tallied per lane, the lane's
// first passing row kept, unsure lanes decided in FP64.
// PAIRS: `cnt` is the lane's pending pass word (bit l = angle m0 + l) of row
// 32 b + lane of the current 32-row block; each 32-row block's words are
// stored to the strip's column of the pass-mask array (mcol[k], coalesced)
// when the block ends.
// kCubeOnly: the strip form (rows below the strip's cube bound); else the
// endpoint form, with x on the cube branch when kXCube (every row of the
// range below the x half of the bound: no select for the x endpoints; the
// caller also passes cos >= 0 with fz0 on the cube branch, so the z endpoint
// fz0 + r cos needs no select).
template <int kL, bool kCubeOnly, int kOut, class CT, bool kXCube = false>
__device__ __forceinline__ void strip_rows(const SearchConst* S, const CT& C, const StripConsts& Q,
                                           const LaunchArgs& A, float2 sc, bool m_ok, uint32_t m, uint32_t k,
                                           uint32_t kend, uint32_t& cnt, uint32_t& fk, Counters& ct,
                                           uint32_t* mcol = nullptr) {
    // radius groups: {r[4j..4j+3]}, {r^2}, {r^3} as three consecutive float4
    const float4* __restrict__ rg = reinterpret_cast<const float4*>(A.radius_groups) + 3 * (k >> 2);
    // linear rows: a partial strip's idle lanes never ask for the other slots
    // (one masked threshold instead of a select per row)
    const float la_lane = m_ok ? C.la : 3.0e38f;
#pragma unroll 1
    for (; k != kend; k += kStripG, rg += 3 * (kStripG / 4)) {
        float rr[kStripG], r2[kStripG], r3[kStripG];
#pragma unroll
        for (uint32_t h = 0; h < kStripG / 4; ++h) {
            const float4 r4 = __ldg(rg + 3 * h);
            rr[4 * h] = r4.x, rr[4 * h + 1] = r4.y, rr[4 * h + 2] = r4.z, rr[4 * h + 3] = r4.w;
            if constexpr (kCubeOnly) {
                const float4 q2 = __ldg(rg + 3 * h + 1), q3 = __ldg(rg + 3 * h + 2);
                r2[4 * h] = q2.x, r2[4 * h + 1] = q2.y, r2[4 * h + 2] = q2.z, r2[4 * h + 3] = q2.w;
                r3[4 * h] = q3.x, r3[4 * h + 1] = q3.y, r3[4 * h + 2] = q3.z, r3[4 * h + 3] = q3.w;
            }
        }
        // slot 0 first (the most selective loud channel, make_search_const):
        // a group where no candidate can leave its band needs nothing more
        bool go = true;
        float M0[kStripG];
        float gv[kStripG][4];  // linear rows: f^-1 of the four endpoint coordinates (x+, x-, z+, z-)
        if constexpr (kCubeOnly) {
            float mx0 = 0.0f;
#pragma unroll
            for (uint32_t g = 0; g < kStripG; ++g) {
                M0[g] = strip_chan(Q, 0, rr[g], r2[g], r3[g]);
                mx0 = fmaxf(mx0, M0[g]);
            }
            go = __any_sync(kFull, mx0 >= C.la);
        } else {
            float mx0 = 0.0f;
#pragma unroll
            for (uint32_t g = 0; g < kStripG; ++g) {
                gv[g][0] = finv_fast<kXCube>(fmaf(rr[g], sc.x, C.fx0));
                gv[g][1] = finv_fast<kXCube>(fmaf(-rr[g], sc.x, C.fx0));
                gv[g][2] = finv_fast<false>(fmaf(-rr[g], sc.y, C.fz0));
                gv[g][3] = finv_fast<kXCube>(fmaf(rr[g], sc.y, C.fz0));  // kXCube: sc.y >= 0, fz0 on the cube branch
                const float dp = fmaf(C.mxs[0], gv[g][0], fmaf(C.mzs[0], gv[g][2], C.cys[0]));
                const float dm = fmaf(C.mxs[0], gv[g][1], fmaf(C.mzs[0], gv[g][3], C.cys[0]));
                M0[g] = fmaxf(fabsf(dp), fabsf(dm));
                mx0 = fmaxf(mx0, M0[g]);
            }
            go = __any_sync(kFull, mx0 >= la_lane);
        }
        if (go) {
        float lv[kStripG], qv[kStripG];
        bool att = false;
        if constexpr (kCubeOnly) {
            // lanes past the last angle hold zero strip constants: every
            // channel's statistic is 0, so no loud channel leaves its band
#pragma unroll
            for (uint32_t g = 0; g < kStripG; ++g) {
                const float M[3] = {M0[g], strip_chan(Q, 1, rr[g], r2[g], r3[g]), strip_chan(Q, 2, rr[g], r2[g], r3[g])};
                band_stats_m<kL>(C, M, lv[g], qv[g]);
                att |= band_attention(C, lv[g], qv[g]);
            }
        } else {
            // the endpoint form (fast_linear + band_stats) of the remaining slots
#pragma unroll
            for (uint32_t g = 0; g < kStripG; ++g) {
                float M[3];
                M[0] = M0[g];
#pragma unroll
                for (int q = 1; q < 3; ++q) {
                    const float dp = fmaf(C.mxs[q], gv[g][0], fmaf(C.mzs[q], gv[g][2], C.cys[q]));
                    const float dm = fmaf(C.mxs[q], gv[g][1], fmaf(C.mzs[q], gv[g][3], C.cys[q]));
                    M[q] = fmaxf(fabsf(dp), fabsf(dm));
                }
                band_stats_m<kL>(C, M, lv[g], qv[g]);
                att |= band_attention(C, lv[g], qv[g]);
            }
            att &= m_ok;
        }
        if constexpr (kOut == kOutPairs) {
            if (__any_sync(kFull, att)) {
                bool pass[kStripG], uns = false;
#pragma unroll
                for (uint32_t g = 0; g < kStripG; ++g) {
                    pass[g] = band_certain(C, lv[g], qv[g]) & m_ok;
                    uns |= band_attention(C, lv[g], qv[g]) & !pass[g] & m_ok;
                }
                if (uns) {
#pragma unroll
                    for (uint32_t g = 0; g < kStripG; ++g) {
                        if (band_attention(C, lv[g], qv[g]) & !band_certain(C, lv[g], qv[g]) & m_ok) {
                            double lp[3], lm[3];
                            exact_linear(S, A, k + g, m, lp, lm);
                            pass[g] = exact_band(S, lp, lm, __ldg(&S->flags));
                            ++ct.repairs;
                        }
                    }
                }
                const uint32_t lane = threadIdx.x & 31;
#pragma unroll
                for (uint32_t g = 0; g < kStripG; ++g) {
                    const uint32_t w = __ballot_sync(kFull, pass[g]);
                    if (lane == ((k + g) & 31u)) cnt = w;
                }
            }
        } else if (__any_sync(kFull, att) && att) {
            // certain passes counted per lane (the lane's first passing row
            // kept); the unsure lanes, rare, decided in FP64
            bool uns = false;
#pragma unroll
            for (uint32_t g = 0; g < kStripG; ++g) {
                const bool cert = band_certain(C, lv[g], qv[g]);
                cnt += cert;
                if (kOut == kOutFirst && cert) fk = min(fk, k + g);
                uns |= band_attention(C, lv[g], qv[g]) & !cert;
            }
            if (uns) {
#pragma unroll
                for (uint32_t g = 0; g < kStripG; ++g) {  // unrolled: lv / qv stay in registers
                    if (band_attention(C, lv[g], qv[g]) & !band_certain(C, lv[g], qv[g])) {
                        double lp[3], lm[3];
                        exact_linear(S, A, k + g, m, lp, lm);
                        const bool pass = exact_band(S, lp, lm, __ldg(&S->flags));
                        ++ct.repairs;
                        cnt += pass;
                        if (kOut == kOutFirst && pass) fk = min(fk, k + g);
                    }
                }
            }
        }
        }
        if constexpr (kOut == kOutPairs) {
            if (((k + kStripG) & 31u) == 0) {  // the 32-row block is complete
                mcol[(k & ~31u) + (threadIdx.x & 31)] = cnt;
                cnt = 0;
            }
        }
    }
}

// strip_run's bulk skip: the largest g <= n such that rows [k0, k0 + kStripG g)
// hold no lane whose loud strip statistics can all reach la (bisection on the
// bound described there; warp-uniform result).  A lane needs every loud
// channel (slots 0 .. kL-1) at la or more, so it is out while the smallest of
// its loud channels' bounds stays below: different lanes of a strip are
// limited by different channels (each channel has its own null direction).
template <int kL>
__device__ __forceinline__ uint32_t skip_groups(const float* radius_groups, uint32_t k0, uint32_t n,
                                             const StripConsts& Q, float la, uint32_t guess) {
    // (a + b) (1 + 2^-20) < la, with the margin folded into the threshold
    const float las = la * (1.0f - 1.0f / 524288.0f);
    auto below = [&](uint32_t groups) {  // rows [k0, k0 + kStripG * groups) skippable?
        const uint32_t ke = k0 + kStripG * groups - 1;  // last row of the range
        const float* g = radius_groups + 12 * (ke >> 2) + (ke & 3u);
        const float rb = __ldg(g), r2b = __ldg(g + 4), r3b = __ldg(g + 8);
        float ub = 3.0e38f;
#pragma unroll
        for (int q = 0; q < kL; ++q) {
            const float a = fmaxf(fabsf(Q.k0[q]), fabsf(fmaf(Q.k2[q], r2b, Q.k0[q])));
            const float b = fabsf(Q.l3[q] * r3b) + fabsf(Q.l1[q] * rb);  // r >= 0
            ub = fminf(ub, a + b);
        }
        return __all_sync(kFull, ub < las);
    };
    // lo: groups proven skippable; nothing beyond hi is.  The first probe sits
    // at the previous strip's answer (consecutive strips of a tile have
    // neighbouring |cos|) and the next ones gallop away from it in doubling
    // steps until they bracket the answer: where it still holds the search
    // costs two steps.  Without one (guess = 0: a tile's first strip, or
    // nothing skipped last time) the first group is tested first: where it
    // cannot be skipped (the pass region starts at the centre) the search
    // costs one step.
    if (n == 0) return 0u;
    uint32_t lo = 0, hi = n;
    const uint32_t g = min(max(guess, 1u), n);
    if (below(g)) {
        lo = g;
        if (guess != 0) {
            for (uint32_t step = 1; lo < hi; step *= 2) {
                const uint32_t p = min(lo + step, hi);
                if (below(p)) {
                    lo = p;
                } else {
                    hi = p - 1;
                    break;
                }
            }
        }
    } else {
        hi = g - 1;
        for (uint32_t step = 1; lo < hi; step *= 2) {
            const uint32_t p = hi > step ? hi - step + 1 : 1u;
            if (below(p)) {
                lo = p;
                break;
            }
            hi = p - 1;
        }
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (below(mid)) {
            lo = mid;
        } else {
            hi = mid - 1;
        }
    }
    return lo;
}

// Rows [k0, k1) of the strip at angles m0 + lane.  The full constants are
// loaded for the strip set-up and again (through an opaque pointer, so the
// two loads are not merged) for the linear rows: during the cube-only rows
// only the strip constants and the thresholds are live.
template <int kL, int kOut, bool kSkip>
__device__ __forceinline__ void strip_run(const SearchConst* S, const Consts& C0, const LaunchArgs& A, uint32_t m0,
                                          uint32_t k0, uint32_t k1, unsigned lane, uint32_t& cnt, uint32_t& fk,
                                          Counters& ct, uint32_t& guess, uint32_t* mcol = nullptr) {
    // lane slot m0 + lane: angle m (the identity, or the |cos|-sorted
    // permutation of the COUNTS / FIRST strips)
    uint32_t m = m0 + lane;
    bool m_ok = m < static_cast<uint32_t>(A.na);
    float2 sc;
    if (A.strip_perm) {
        sc = __ldg(reinterpret_cast<const float2*>(A.strip_trig) + m);
        m = __ldg(&A.strip_perm[m]);
    } else {
        sc = __ldg(reinterpret_cast<const float2*>(A.trig_f) + (m_ok ? m : A.na - 1));
    }
    const uint32_t kend = k0 + (k1 - k0) / kStripG * kStripG;  // k0 % 4 == 0
    StripConsts Q;
    ThrConsts T;
    uint32_t kc = kend;
    {
        const Consts& C = C0;
        T = ThrConsts{C.la, C.qa, C.lp, C.qp, C.flags};
        // The strip's cube-only bound rb: no candidate of a row with r < rb
        // leaves the cube branch of f^-1 (r |s'| < fx0 - u0 and r |c'| <
        // fz0 - u0 over the strip's angles, with margins as
        // make_search_const's rcube).  strip_inv[q] = 1 / the strip's
        // largest |s'|, |c'| (host, rounded down; FLT_MAX for an all-zero
        // column).
        const float2 inv = __ldg(reinterpret_cast<const float2*>(A.strip_inv) + (m0 >> 5));
        const float ex = fmaf(C.fx0 - kU0f, 1.0f - 4e-6f, -1e-6f), ez = fmaf(C.fz0 - kU0f, 1.0f - 4e-6f, -1e-6f);
        const float rb = fminf(ex * inv.x, ez * inv.y) * (1.0f - 1e-6f);
        // kc: the first row (from k0, in steps of kStripG) whose group
        // reaches rb; radii ascend, so rows [k0, kc) are cube-only
        for (uint32_t kk = k0; kk < kend; kk += 32 * kStripG) {
            const uint32_t kl = kk + kStripG * lane + kStripG - 1;  // last row of lane's group
            const unsigned b = __ballot_sync(kFull, kl < kend && !(__ldg(&A.radii_f[kl]) < rb));
            if (b) {
                kc = kk + kStripG * static_cast<uint32_t>(__ffs(b) - 1);
                break;
            }
        }
        strip_setup(C, sc, Q);
        if (!m_ok) Q = StripConsts{};  // the partial strip's idle lanes never pass (strip_rows)
    }
    // Bulk skip of the inner rows: rows [k0, ks) where no lane can have all
    // its loud statistics at la or more -- groups strip_rows would leave
    // without a pass or a repair -- found by bisection over the row groups.
    // Over rows up to radius rb (float r, r^2, r^3 of the radii, ascending)
    // the strip form's value of a slot is at most
    //     max(|K0|, |K0 + rb^2 K2|) + rb |L1| + rb^3 |L3|
    // (A = K0 + r^2 K2 is linear in r^2, so |A| peaks at an end of the range;
    // B = r L1 + r^3 L3 by the triangle inequality), non-decreasing in rb, and
    // so is a lane's smallest bound over its loud slots.
    // The 2^-20 relative margin covers the FP32 rounding of both this bound
    // and the per-candidate value (a few operations of 2^-24 each).
    // The first group is tested first: where it cannot be skipped (the pass
    // region starts at the centre) the search costs one step.  kSkip: its
    // own instantiation; the PAIRS kernels of small strips (cfg1, cfg3) ran
    // 10-17% slower with this code present even when it skipped nothing.
    uint32_t ks = k0;
    if constexpr (kSkip) {
        const uint32_t lo = A.bulk_skip && kc > k0
                                ? skip_groups<kL>(A.radius_groups, k0, (kc - k0) / kStripG, Q, T.la,
                                                  kOut == kOutPairs ? 0u : guess)
                                : 0u;
        // PAIRS skips on 512-row strips only (one strip per tile): no hint to
        // carry, and its instantiation keeps the plain search
        if constexpr (kOut != kOutPairs) guess = lo;
        ks = k0 + kStripG * lo;
        if constexpr (kOut == kOutPairs) {
            for (uint32_t b = k0; b + 32 <= ks; b += 32) mcol[b + lane] = 0u;  // whole skipped 32-row blocks
        }
    }
    strip_rows<kL, true, kOut>(S, T, Q, A, sc, m_ok, m, ks, kc, cnt, fk, ct, mcol);
    if (kc == k1) {
        if constexpr (kOut == kOutPairs) {
            if (k1 & 31u) mcol[((k1 - 1) & ~31u) + lane] = cnt;  // the last, partial 32-row block
        }
        return;
    }
    const Consts& C = C0;
    // x stays on the cube branch in every remaining row (r |s'| below
    // fx0 - u0 with the rcube margins): the endpoint form without the x select
    const float rbx = fmaf(C.fx0 - kU0f, 1.0f - 4e-6f, -1e-6f) *
                      __ldg(reinterpret_cast<const float2*>(A.strip_inv) + (m0 >> 5)).x * (1.0f - 1e-6f);
    // ... and with the lane's endpoints swapped where cos < 0 (the statistic
    // max(|d+|, |d-|) is symmetric in the endpoints, and the swapped FFMAs
    // compute the same values: fma(-r, -s, f0) = fma(r, s, f0)), the "-"
    // endpoint's z = fz0 + r |c'| >= fz0 stays on the cube branch whenever
    // fz0 itself is: no select for it either
    if (kend > kc && __ldg(&A.radii_f[kend - 1]) < rbx && C.fz0 > kU0f) {
        const float2 scs = make_float2(sc.y < 0.0f ? -sc.x : sc.x, fabsf(sc.y));
        strip_rows<kL, false, kOut, Consts, true>(S, C, Q, A, scs, m_ok, m, kc, kend, cnt, fk, ct, mcol);
    } else {
        strip_rows<kL, false, kOut>(S, C, Q, A, sc, m_ok, m, kc, kend, cnt, fk, ct, mcol);
    }
#pragma unroll 1
    for (uint32_t k = kend; k < k1; ++k) {
        const float r = __ldg(&A.radii_f[k]);
        float l1, q1;
        band_chunk<kL, false>(C, r, sc, l1, q1);
        bool pass = band_certain(C, l1, q1);
        const bool u = band_attention(C, l1, q1) & !pass & m_ok;
        if (__any_sync(kFull, u) && u) {
            double lp[3], lm[3];
            exact_linear(S, A, k, m, lp, lm);
            pass = exact_band(S, lp, lm, C.flags);
            ++ct.repairs;
        }
        pass &= m_ok;
        if constexpr (kOut == kOutPairs) {
            const uint32_t w = __ballot_sync(kFull, pass);
            if (lane == (k & 31u)) cnt = w;
        } else {
            cnt += pass;
            if (kOut == kOutFirst && pass) fk = min(fk, k);
        }
    }
    if constexpr (kOut == kOutPairs) {
        if ((k1 & 31u) || kend != k1) {  // the last block's rows were not stored yet (rows >= k1 stay 0)
            mcol[((k1 - 1) & ~31u) + lane] = cnt;
            cnt = 0;
        }
    }
}

// One strip tile of search s: strips [lt' * strip_per_tile, ...) of row
// block kb (lt = kb * tiles_per_block + lt'); per-search count and first
// canonical pair recorded here.
template <int kL, int kOut, bool kSkip>
__device__ __forceinline__ void strip_tile(const SearchConst* S, const LaunchArgs& A, uint32_t s, uint32_t lt,
                                           unsigned lane, Counters& ct) {
    const uint32_t kb = lt / A.strip_tiles, st = lt - kb * A.strip_tiles;
    const uint32_t k0 = kb * A.strip_rows;
    const uint32_t k1 = min(k0 + A.strip_rows, static_cast<uint32_t>(A.nr));
    const uint32_t n_strips = (static_cast<uint32_t>(A.na) + 31) / 32;
    const uint32_t s0 = st * A.strips_per_tile, s1 = min(s0 + A.strips_per_tile, n_strips);
    uint32_t cnt = 0, first = 0xffffffffu;
    uint32_t guess = 0;  // bulk skip: the previous strip's skipped groups (warp-uniform; 0 = no hint)
    Consts C;
    load_consts(S, C);
    if constexpr (kOut == kOutPairs) {
        // pass words of strip q: column q of search s's mask block (rows padded to 32)
        uint32_t* mblk = A.masks + static_cast<size_t>(s) * n_strips * A.mask_rows;
        for (uint32_t q = s0; q < s1; ++q) {
            uint32_t w = 0, fk = 0;
            strip_run<kL, kOut, kSkip>(S, C, A, 32 * q, k0, k1, lane, w, fk, ct, guess,
                                       mblk + static_cast<size_t>(q) * A.mask_rows);
        }
        return;
    }
    for (uint32_t q = s0; q < s1; ++q) {
        uint32_t fk = 0xffffffffu;
        strip_run<kL, kOut, kSkip>(S, C, A, 32 * q, k0, k1, lane, cnt, fk, ct, guess);
        if (kOut == kOutFirst) {
            const uint32_t mq = A.strip_perm ? __ldg(&A.strip_perm[32 * q + lane]) : 32 * q + lane;  // the lane's angle
            const uint32_t mine = fk != 0xffffffffu ? fk * static_cast<uint32_t>(A.na) + mq : 0xffffffffu;
            first = min(first, __reduce_min_sync(kFull, mine));
        }
    }
    const uint32_t total = __reduce_add_sync(kFull, cnt);
    if (lane == 0 && total) {
        atomicAdd(&A.counts[s], static_cast<unsigned long long>(total));
        if (kOut == kOutFirst) atomicMin(&A.first_idx[s], first);
    }
}

// K1: decide every candidate.  Warps claim 4096-candidate tiles (contiguous
// canonical ranges of one search) from a ticket, prefetching the next ticket.
// PAIRS: tile count + ordered passing offsets to scratch; COUNTS: per-search
// counts; FIRST: counts + first passing index.
// kPrune (CVG_PATH_PRUNED, band mode): its own instantiation, so that the
// unpruned loops keep their register allocation (a run-time flag cost 1-2%).
// kStrips: 0 = row-major tiles, 1 = strip tiles, 2 = strip tiles with the
// bulk skip of the inner rows (strip_run).
template <int kMode, int kOut, int kPath, bool kPrune = false, int kStrips = 0>
__global__ void __launch_bounds__(kBlock, 4) phase1_kernel(const LaunchArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    // phase 1 quantizes only in FrameDiff x Quantized; Continuous x FrameDiff prefilters on signal bounds
    load_tables<kMode == kModeCodes ? kTabCode : (kMode == kModeSignal ? kTabSignal : kTabNone)>(sm, A);
    const uint32_t tab = ctab_addr(sm.ctab);
    const unsigned lane = threadIdx.x & 31;
    const unsigned lane_lt = (1u << lane) - 1u;
    Counters ct;

    uint32_t t_claim = 0;
    if (lane == 0) t_claim = atomicAdd(&A.ticket[0], 1u);
    uint32_t c = __shfl_sync(kFull, t_claim, 0);
    const uint32_t n_claims = A.n_claims;
    while (c < n_claims) {
        if (lane == 0) t_claim = atomicAdd(&A.ticket[0], 1u);  // next tile, consumed at the end
        // Claim order for searches of many tiles: outermost radius tiles of
        // every search first, the innermost last.  Outer rows are the costly
        // ones (they reach the linear branch of f^-1 and need more repairs),
        // so the last round of claims -- the tail where warps run out of
        // work -- is the cheapest.  Searches of a few tiles (per-pixel
        // batches) keep search order: a warp's consecutive tiles share the
        // search's constants.  Tile t (search s, tile lt) keeps its storage
        // slot s * tps + lt either way.
        uint32_t s, lt;
        const uint32_t cps = A.claim_per_search;  // tiles (or strip tiles) per search
        if (A.claim_order) {
            // group g of loud-count-sorted positions, outer-first inside it
            const uint32_t tps = cps;
            uint32_t g0 = 0, g1 = A.group_end[0];
            if (c >= g1 * tps) {
                g0 = g1;
                g1 = A.group_end[1];
                if (c >= g1 * tps) {
                    g0 = g1;
                    g1 = A.group_end[2];
                }
            }
            const uint32_t cl = c - g0 * tps, ng = g1 - g0;
            uint32_t pos;
            if (tps >= 16) {
                const uint32_t q = cl / ng;
                pos = g0 + (cl - q * ng);
                lt = tps - 1 - q;
            } else {
                const uint32_t sr = cl / tps;
                lt = cl - sr * tps;
                pos = g0 + sr;
            }
            s = __ldg(&A.claim_order[pos]);
        } else if (cps >= 16) {
            const uint32_t q = c / A.range_searches;
            s = A.search_begin + (c - q * A.range_searches);
            lt = cps - 1 - q;
        } else {
            const uint32_t sr = c / cps;
            lt = c - sr * cps;
            s = A.search_begin + sr;
        }
        const uint32_t t = s * A.tiles_per_search + lt;
        const SearchConst* S = search_const(A, s);
        const uint32_t i0 = lt * static_cast<uint32_t>(kTile);
        const uint32_t i1 = min(i0 + static_cast<uint32_t>(kTile), A.cand_per_search);
        uint16_t* list = kOut == kOutPairs ? A.scratch + static_cast<size_t>(t) * kTile : nullptr;
        uint32_t cnt = 0;
        uint32_t* first = &sm.first[threadIdx.x >> 5];
        Consts C;
        load_consts(S, C);
        // kStrips (COUNTS / FIRST, band FAST path, LaunchArgs::strips): its
        // own instantiation, so that the row-major loops keep their registers
        constexpr bool kStripsOk = kMode == kModeBand && kPath == kPathFast && !kPrune;
        if constexpr (kStrips != 0 && kStripsOk) {
            const uint32_t nl = (__ldg(&S->flags) >> 10) & 3u;
            if (nl == 3) {
                strip_tile<3, kOut, kStrips == 2>(S, A, s, lt, lane, ct);
            } else if (nl == 2) {
                strip_tile<2, kOut, kStrips == 2>(S, A, s, lt, lane, ct);
            } else {
                strip_tile<1, kOut, kStrips == 2>(S, A, s, lt, lane, ct);
            }
            // counts / first pair recorded; PAIRS: pass words written, the
            // tile lists come from lists_kernel
            c = __shfl_sync(kFull, t_claim, 0);
            continue;
        } else if (kMode == kModeBand && kPath == kPathFast && A.aligned) {
            const uint32_t nl = (C.flags >> 10) & 3u;
            if (nl == 3) {
                band_tile<3, kOut, kPrune>(S, C, A, i0, i1, list, cnt, first, ct, lane, lane_lt);
            } else if (nl == 2) {
                band_tile<2, kOut, kPrune>(S, C, A, i0, i1, list, cnt, first, ct, lane, lane_lt);
            } else {
                band_tile<1, kOut, kPrune>(S, C, A, i0, i1, list, cnt, first, ct, lane, lane_lt);
            }
        } else if (kMode == kModeCodes && kPath == kPathFast && A.aligned) {
            CodeConsts CC;
            load_code_consts(S, CC, tab);
            frame_tile<kOut>(sm, S, CC, C.flags, A, i0, i1, list, cnt, first, ct, lane, lane_lt);
        } else {
            CodeConsts CC;
            load_code_consts(S, CC, tab);
            SigConsts SG;
            if (kMode == kModeSignal) load_sig_consts(S, SG);
            for (uint32_t base = i0; base < i1; base += 32) {
                const bool active = base + lane < i1;
                const uint32_t i = active ? base + lane : i1 - 1;
                const uint32_t k = div_na(i, A);
                const uint32_t m = i - k * static_cast<uint32_t>(A.na);
                const bool pass = candidate_pass<kMode, kPath>(sm, S, C, CC, SG, A, k, m, active, ct);
                append<kOut>(pass, i - i0, list, cnt, first, lane_lt);
            }
        }
        if (kOut == kOutFirst) __syncwarp();  // *first was written by another lane
        if (lane == 0) {
            if (kOut == kOutPairs) {
                A.tile_count[t] = cnt;
                // emit work items: (tile, 256-pair sub-range), any order
                const uint32_t subs = (cnt + (1u << A.emit_shift) - 1) >> A.emit_shift;
                if (subs) {
                    const uint32_t w = atomicAdd(&A.ticket[3], subs);
                    for (uint32_t j = 0; j < subs; ++j) A.worklist[w + j] = (t << 4) | j;
                }
            }
            if (cnt) atomicAdd(&A.counts[s], static_cast<unsigned long long>(cnt));
            if (kOut == kOutFirst && cnt) atomicMin(&A.first_idx[s], i0 + *first);
        }
        c = __shfl_sync(kFull, t_claim, 0);
    }
    pdl_trigger();  // no tiles left for this warp: the scan may launch once every CTA has said so
    flush_counters(ct, A, lane);
}

// K1b (PAIRS on strip tiles): the canonical tile lists from the pass words.
// A unit is search s, lst_unit_rows rows (8, or the rows of one whole-row
// tile when that is more) and strips [128 cb, +128) (all strips when a tile
// holds whole rows): at most 1024 words, read as full 32-byte column
// segments (lst_unit_rows consecutive rows of a strip) into a padded shared
// block, then appended row by row, strips ascending, to the ordered list of
// their canonical tile (whole-row tiles: lst_rpt rows each; else lst_tpr
// tiles per row).  Small units keep many warps resident: the expansion is a
// latency-bound chain of shuffles.  Writes tile_count, the emit work items
// and the per-search counts: scan and emit then run exactly as after the
// row-major loop.
constexpr uint32_t kListWords = 1024;

// Appends the set bits of one 32-word chunk (lane l: word W of strip
// wbase + l, bit b = angle 32 (wbase + l) + b of the tile) to `list` after
// `cnt` entries, in canonical order; returns the new count (warp-uniform).
__device__ __forceinline__ uint32_t expand_chunk(uint32_t W, uint32_t wbase, uint16_t* list, uint32_t cnt,
                                                 unsigned lane, unsigned lane_lt) {
    const uint32_t pc = __popc(W);
    uint32_t incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    const uint32_t excl = cnt + incl - pc;
    if (__all_sync(kFull, W == 0xffffffffu)) {
        // every candidate of the chunk passes (dense batches: most non-empty
        // chunks): the list is the ramp 32 wbase + e, e < 1024, written as
        // 16-byte stores between a short head and tail
        uint16_t* dst = list + cnt;
        const uint32_t base = 32u * wbase;
        const uint32_t head = (8u - ((static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst)) >> 1) & 7u)) & 7u;
        if (lane < head) dst[lane] = static_cast<uint16_t>(base + lane);
        uint4* d4 = reinterpret_cast<uint4*>(dst + head);
        const uint32_t nb = (1024u - head) >> 3;
#pragma unroll 4
        for (uint32_t j = lane; j < nb; j += 32) {
            const uint32_t v = base + head + 8u * j;
            d4[j] = make_uint4(v | (v + 1) << 16, (v + 2) | (v + 3) << 16, (v + 4) | (v + 5) << 16,
                               (v + 6) | (v + 7) << 16);
        }
        const uint32_t t0 = head + 8u * nb;
        if (t0 + lane < 1024u) dst[t0 + lane] = static_cast<uint16_t>(base + t0 + lane);
        return cnt + 1024u;
    }
    uint32_t nz = __ballot_sync(kFull, W != 0);
    // two words per iteration: their shuffles are independent, so the two
    // latency chains overlap
    while (nz) {
        const int q1 = __ffs(nz) - 1;
        nz &= nz - 1;
        const int q2 = nz ? __ffs(nz) - 1 : q1;
        const bool two = nz != 0;
        nz &= nz - 1;
        const uint32_t W1 = __shfl_sync(kFull, W, q1);
        const uint32_t o1 = __shfl_sync(kFull, excl, q1);
        const uint32_t W2 = __shfl_sync(kFull, W, q2);
        const uint32_t o2 = __shfl_sync(kFull, excl, q2);
        if ((W1 >> lane) & 1u) list[o1 + __popc(W1 & lane_lt)] = static_cast<uint16_t>(32u * (wbase + q1) + lane);
        if (two && ((W2 >> lane) & 1u)) {
            list[o2 + __popc(W2 & lane_lt)] = static_cast<uint16_t>(32u * (wbase + q2) + lane);
        }
    }
    return cnt + __shfl_sync(kFull, incl, 31);
}

// Twin tiles (A.twin, rows of whole tiles): the units cover the first half of
// each row's tiles; each unit also reads the words of the twin column (same
// rows, angles + na/2) with the same coalesced loads and compares them in
// registers.  A row whose twin words are all identical is one list for two
// tiles (twin[t] = 1, the twin gets the count and no list of its own); a row
// with any difference (a decision the FP64 repair settled differently for
// the two angles) builds the twin's list from its own words, and the twin is
// emitted on its own.
__global__ void __launch_bounds__(kBlock) lists_kernel(const LaunchArgs A) {
    __shared__ uint32_t blk[kWarpsPerBlock][kListWords + 32];
    pdl_wait();  // phase 1 complete: every pass word written
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lane_lt = (1u << lane) - 1u;
    uint32_t* Wb = blk[warp];
    const uint32_t nq = static_cast<uint32_t>(A.na) >> 5;
    const uint32_t ur = A.lst_unit_rows;                     // rows per unit (divides 32; 8 with twins)
    const uint32_t n_kb = (static_cast<uint32_t>(A.nr) + ur - 1) / ur;
    const uint32_t hcb = A.twin ? A.twin_tiles : 0u;         // twin column offset (0: no twins)
    const uint32_t n_cb = A.lst_tpr ? A.lst_tpr - hcb : 1u;
    const uint32_t cwu = min(nq, 128u);
    const uint32_t stride = cwu + 1;                         // shared row stride (bank-conflict free)
    const uint32_t ups = n_kb * n_cb;
    const uint32_t n_units = A.range_searches * ups;
    const uint32_t per_load = 32u / ur;                      // strips per load instruction
    const size_t twin_col = static_cast<size_t>(128u * hcb) * A.mask_rows;
    uint32_t u_claim = 0;
    if (lane == 0) u_claim = atomicAdd(&A.ticket[4], 1u);
    uint32_t u = __shfl_sync(kFull, u_claim, 0);
    while (u < n_units) {
        if (lane == 0) u_claim = atomicAdd(&A.ticket[4], 1u);
        const uint32_t sr = u / ups, r = u - sr * ups;
        const uint32_t s = A.search_begin + sr;
        const uint32_t kb = r / n_cb, cb = r - kb * n_cb;
        const uint32_t k0 = ur * kb, rows = min(ur, static_cast<uint32_t>(A.nr) - k0);
        const uint32_t* mblk = A.masks + static_cast<size_t>(s) * nq * A.mask_rows;
        uint32_t split = 0;  // twins: bit j = row k0 + j differs from its twin row
        uint32_t nzacc = 0;  // OR of the lane's words (and twin words)
        // load: lane -> (strip qs + lane / ur, row k0 + lane % ur)
        {
            const uint32_t kr = lane % ur, qo = lane / ur;
            const uint32_t* col = mblk + static_cast<size_t>(128u * cb + qo) * A.mask_rows + k0 + kr;
            uint32_t diff = 0;
#pragma unroll 4
            for (uint32_t qs = 0; qs < cwu; qs += per_load) {
                if (qs + qo < cwu) {
                    const uint32_t w = __ldg(col + static_cast<size_t>(qs) * A.mask_rows);
                    Wb[kr * stride + qs + qo] = w;
                    nzacc |= w;
                    if (hcb) {
                        const uint32_t w2 = __ldg(col + twin_col + static_cast<size_t>(qs) * A.mask_rows);
                        diff |= w ^ w2;
                        nzacc |= w2;
                    }
                }
            }
            if (hcb) {  // ur == 8: lanes j, j + 8, j + 16, j + 24 hold row j
                const unsigned dm = __ballot_sync(kFull, diff != 0u);
                split = (dm | dm >> 8 | dm >> 16 | dm >> 24) & 0xffu;
                if (A.twin_split_test) split |= 0xaau & ((1u << rows) - 1u);
            }
        }
        __syncwarp();
        uint32_t tcnt = 0;   // lane j: count of the unit's tile slot j
        uint32_t tcnt2 = 0;  // twins: lane j: count of slot j's twin when its row differs
        // an all-zero unit (sparse batches: most of them) writes its zero
        // counts without walking its rows
        const uint32_t n_rows = __any_sync(kFull, nzacc != 0u) ? rows : 0u;
        for (uint32_t j = 0; j < n_rows; ++j) {
            const uint32_t row = k0 + j;
            const uint32_t slot = A.lst_rpt ? j / A.lst_rpt : j;
            const uint32_t lt = A.lst_rpt ? row / A.lst_rpt : row * A.lst_tpr + cb;
            uint16_t* list = A.scratch + static_cast<size_t>(s * A.tiles_per_search + lt) * kTile;
            // word index of strip qc + l inside the tile
            const uint32_t wrow = A.lst_rpt ? (row % A.lst_rpt) * nq : 0u;
            for (uint32_t qc = 0; qc < cwu; qc += 32) {
                const uint32_t W = qc + lane < cwu ? Wb[j * stride + qc + lane] : 0u;
                if (!__any_sync(kFull, W != 0u)) continue;
                uint32_t cnt = __shfl_sync(kFull, tcnt, slot);
                cnt = expand_chunk(W, wrow + qc, list, cnt, lane, lane_lt);
                if (lane == slot) tcnt = cnt;
            }
            if ((split >> j) & 1u) {  // rare: the twin row gets its own list
                uint16_t* list2 = list + static_cast<size_t>(hcb) * kTile;
                const uint32_t* col2 = mblk + twin_col + static_cast<size_t>(128u * cb) * A.mask_rows + row;
                uint32_t cnt2 = 0;
                for (uint32_t qc = 0; qc < cwu; qc += 32) {
                    const uint32_t W = qc + lane < cwu ? __ldg(col2 + static_cast<size_t>(qc + lane) * A.mask_rows) : 0u;
                    if (!__any_sync(kFull, W != 0u)) continue;
                    cnt2 = expand_chunk(W, qc, list2, cnt2, lane, lane_lt);
                }
                if (lane == slot) tcnt2 = cnt2;
            }
        }
        __syncwarp();
        const uint32_t n_slots = A.lst_rpt ? (rows + A.lst_rpt - 1) / A.lst_rpt : rows;
        uint32_t mine = 0;
        if (lane < n_slots) {
            const uint32_t lt = A.lst_rpt ? k0 / A.lst_rpt + lane : (k0 + lane) * A.lst_tpr + cb;
            const uint32_t t = s * A.tiles_per_search + lt;
            A.tile_count[t] = tcnt;
            mine = tcnt;
            uint32_t subs = (tcnt + (1u << A.emit_shift) - 1) >> A.emit_shift;
            uint32_t subs2 = 0, c2 = 0;
            if (hcb) {
                const bool tw = !((split >> lane) & 1u);
                c2 = tw ? tcnt : tcnt2;
                A.tile_count[t + hcb] = c2;
                A.twin[t] = tw ? 1u : 0u;
                A.twin[t + hcb] = 0u;
                if (!tw) subs2 = (c2 + (1u << A.emit_shift) - 1) >> A.emit_shift;
                mine += c2;
            }
            if (subs + subs2) {
                const uint32_t w = atomicAdd(&A.ticket[3], subs + subs2);
                for (uint32_t q = 0; q < subs; ++q) A.worklist[w + q] = (t << 4) | q;
                for (uint32_t q = 0; q < subs2; ++q) A.worklist[w + subs + q] = ((t + hcb) << 4) | q;
            }
        }
        const uint32_t total = __reduce_add_sync(kFull, mine);
        if (lane == 0 && total) atomicAdd(&A.counts[s], static_cast<unsigned long long>(total));
        u = __shfl_sync(kFull, u_claim, 0);
    }
    pdl_trigger();
}

// K2: exclusive scan of tile_count -> tile_base (single pass, chained scan
// with decoupled look-back over kScanTile-tile blocks claimed from a ticket).
__global__ void __launch_bounds__(kBlock) scan_kernel(const LaunchArgs A) {
    __shared__ uint32_t s_block;
    __shared__ unsigned long long s_warp[kWarpsPerBlock];
    __shared__ unsigned long long s_prefix;
    pdl_trigger();  // emit CTAs may launch (and load their tables) while the scan runs
    pdl_wait();     // phase 1 complete: tile counts and tickets visible
    if (threadIdx.x == 0) s_block = atomicAdd(&A.ticket[1], 1u);
    __syncthreads();
    const uint32_t b = s_block;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t base = static_cast<uint64_t>(b) * kScanTile + static_cast<uint64_t>(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = base + j < A.n_tiles ? A.tile_count[A.tile_begin + base + j] : 0u;
        sum += v[j];
    }
    unsigned long long incl = sum;  // warp inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, incl, o);
        if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long warp_off = 0, block_sum = 0;
    for (int w = 0; w < kWarpsPerBlock; ++w) {
        if (w < static_cast<int>(warp)) warp_off += s_warp[w];
        block_sum += s_warp[w];
    }
    if (warp == 0) {
        unsigned long long excl = 0;
        if (b == 0) {
            if (lane == 0) st_relaxed(&A.status[0], kFlagPrefix | block_sum);
        } else {
            if (lane == 0) st_relaxed(&A.status[b], kFlagAgg | block_sum);
            long long j = static_cast<long long>(b) - 1;
            while (true) {
                const long long idx = j - static_cast<long long>(lane);
                const unsigned long long w = idx >= 0 ? ld_relaxed(&A.status[idx]) : kFlagPrefix;
                const unsigned flag = static_cast<unsigned>(w >> 62);
                const unsigned pmask = __ballot_sync(kFull, flag == 2);
                const unsigned zmask = __ballot_sync(kFull, flag == 0);
                const unsigned stop = pmask ? static_cast<unsigned>(__ffs(pmask) - 1) : 31u;
                const unsigned need = stop == 31u ? kFull : ((2u << stop) - 1u);
                if (zmask & need) {
                    __nanosleep(32);
                    continue;
                }
                unsigned long long val = lane <= stop ? (w & kValueMask) : 0ull;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
                excl += val;
                if (pmask) break;
                j -= 32;
            }
            if (lane == 0) st_relaxed(&A.status[b], kFlagPrefix | (excl + block_sum));
        }
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    unsigned long long run = s_prefix + warp_off + (incl - sum);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < A.n_tiles) A.tile_base[A.tile_begin + base + j] = run;
        run += v[j];
    }
    if (base < A.n_tiles && base + kScanItems >= A.n_tiles) *A.total = run;
}

// One pair record: idx, then the six codes as three 16-bit words (the
// warp's stores interleave into full sectors in L2).  Staging a warp's codes
// through shared memory for contiguous 64-byte stores measured 13-17% slower
// (cfg1 / cfg2 emit).
__device__ __forceinline__ void store_pair(const LaunchArgs& A, unsigned long long o, uint32_t i, const int* cp,
                                           const int* cm) {
    A.out_idx[o] = i;
    uint16_t* c16 = reinterpret_cast<uint16_t*>(A.out_codes + 6 * o);
    c16[0] = static_cast<uint16_t>(cp[0] | (cp[1] << 8));
    c16[1] = static_cast<uint16_t>(cp[2] | (cm[0] << 8));
    c16[2] = static_cast<uint16_t>(cm[1] | (cm[2] << 8));
}

// FAST path of one emit work item: `cnt` pairs of the tile's list from
// `list`, written to out_idx / out_codes (the item's slice).  Software
// pipeline: list entries two iterations ahead, the candidate's radius / trig
// loads one iteration ahead.  kOneRow: the tile lies inside radius row kt
// (angle = mt + list offset: no per-pair division, no radius load).
// Candidates whose FP32 codes are not all proven (~0.4%) do not take the FP64
// path where they occur (a whole warp pass for one lane): their item-local
// index and FP32 guesses go to the warp's queue in shared memory, and each
// 32 queued pairs are repaired together by the full warp (emit_repair).
constexpr int kRepairQueue = kRepairQueueSlots;  // per warp: < 32 waiting + one iteration's 32

__device__ __forceinline__ void store_codes16(uint8_t* codes, uint32_t qq, const int* p, const int* m) {
    uint16_t* pc = reinterpret_cast<uint16_t*>(codes) + 3 * qq;
    pc[0] = static_cast<uint16_t>(__byte_perm(p[0], p[1], 0x40));
    pc[1] = static_cast<uint16_t>(__byte_perm(p[2], m[0], 0x40));
    pc[2] = static_cast<uint16_t>(__byte_perm(m[1], m[2], 0x40));
}

// kTwin: the pair is also the twin tile's pair qq (angle m + twin_m, the
// endpoints swapped); its codes come from its own FP64 values (the FP32
// guesses, swapped, are the walk's starting points).
template <bool kOneRow, bool kTwin>
__device__ __forceinline__ void emit_repair(const Smem& sm, const SearchConst* S, const LaunchArgs& A,
                                         const uint16_t* list, uint32_t i0, uint32_t kt, uint32_t mt,
                                         uint8_t* out_codes, uint8_t* out_codes2, const uint2* q, uint32_t n,
                                         unsigned lane, unsigned long long& repairs) {
    if (lane >= n) return;
    const uint2 e = q[lane];
    const uint32_t qq = (e.x >> 24) | ((e.y >> 24) << 8);
    const uint32_t off = list[qq];
    const uint32_t i = i0 + off;
    const uint32_t k = kOneRow ? kt : div_na(i, A);
    const uint32_t m = kOneRow ? mt + off : i - k * static_cast<uint32_t>(A.na);
    double lp[3], lm[3];
    exact_linear_inl(S, A, k, m, lp, lm);
    int cp[3], cm[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        cp[c] = code_exact_from(lp[c], (e.x >> (8 * c)) & 0xff, sm.thr_d);
        cm[c] = code_exact_from(lm[c], (e.y >> (8 * c)) & 0xff, sm.thr_d);
    }
    store_codes16(out_codes, qq, cp, cm);
    ++repairs;
    if (kTwin) {
        exact_linear_inl(S, A, k, m + A.twin_m, lp, lm);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            cp[c] = code_exact_from(lp[c], (e.y >> (8 * c)) & 0xff, sm.thr_d);
            cm[c] = code_exact_from(lm[c], (e.x >> (8 * c)) & 0xff, sm.thr_d);
        }
        store_codes16(out_codes2, qq, cp, cm);
        ++repairs;
    }
}

// kTwin (one-row tiles only): every pair is written twice, as itself at
// out_idx / out_codes and as the twin tile's pair at out_idx2 / out_codes2
// (idx + twin_m, plus and minus codes swapped).  The caller widened CC.ec by
// kTwinSlack, so a verified code is the exact code of both records.
// kSeq (one-row tiles): the item's list is one run of consecutive offsets
// (dense batches: pass regions are long arcs), so offsets are computed, not
// loaded, and the trig loads do not wait on the list.
template <bool kOneRow, bool kTwin = false, bool kSeq = false>
__device__ __forceinline__ void emit_run(const Smem& sm, const SearchConst* S, const CodeConsts& CC,
                                         const LaunchArgs& A, const uint16_t* list, uint32_t cnt, uint32_t i0,
                                         uint32_t kt, uint32_t mt, uint32_t* out_idx, uint8_t* out_codes,
                                         uint32_t* out_idx2, uint8_t* out_codes2, uint2* queue, unsigned lane,
                                         Counters& ct) {
    const float2* trig = reinterpret_cast<const float2*>(A.trig_f);
    const float rt = __ldg(&A.radii_f[kt]);
    const unsigned lane_lt = (1u << lane) - 1u;
    // per-lane cursors (one add each per iteration instead of re-deriving
    // 64-bit addresses from the item base); entries past the item read as
    // offset 0, a valid candidate whose codes are computed and not written
    const uint16_t* pl = list + 64 + lane;
    uint32_t* po = out_idx + lane;
    uint16_t* pc = reinterpret_cast<uint16_t*>(out_codes) + 3 * lane;
    uint32_t* po2 = kTwin ? out_idx2 + lane : nullptr;
    uint16_t* pc2 = kTwin ? reinterpret_cast<uint16_t*>(out_codes2) + 3 * lane : nullptr;
    const uint32_t tm = kTwin ? A.twin_m : 0u;
    // through shuffles: ptxas would otherwise re-derive both (and mt's
    // division) inside the loop to save the two registers
    const int cnt_l = __shfl_sync(kFull, static_cast<int>(cnt) - static_cast<int>(lane), lane);  // active iff p < cnt_l
    mt = __shfl_sync(kFull, mt, 0);
    const uint32_t off0 = kSeq ? list[0] : 0u;
    const uint32_t off_last = kSeq ? off0 + cnt - 1 : 0u;
    uint32_t off_n = kSeq ? min(off0 + 32 + lane, off_last) : (32 < cnt_l ? list[32 + lane] : 0u);
    uint32_t i = i0 + (kSeq ? min(off0 + lane, off_last) : (0 < cnt_l ? list[lane] : 0u));
    uint32_t k = kOneRow ? kt : div_na(i, A);
    uint32_t m = kOneRow ? i - i0 + mt : i - k * static_cast<uint32_t>(A.na);
    float r = kOneRow ? rt : __ldg(&A.radii_f[k]);
    float2 sc = __ldg(trig + m);
    uint32_t nq = 0;
#pragma unroll 1
    for (int p = 0; p < static_cast<int>(cnt); p += 32, pl += 32, po += 32, pc += 96) {
        const uint32_t i_n = i0 + off_n;
        const uint32_t k_n = kOneRow ? kt : div_na(i_n, A);
        const uint32_t m_n = kOneRow ? mt + off_n : i_n - k_n * static_cast<uint32_t>(A.na);
        const float r_n = kOneRow ? rt : __ldg(&A.radii_f[k_n]);
        const float2 sc_n = __ldg(trig + m_n);
        off_n = kSeq ? min(off0 + p + 64 + lane, off_last) : (p + 64 < cnt_l ? *pl : 0u);
        const bool active = p < cnt_l;
        int cp[3], cm[3];
        const bool ok = codes_guess(CC, r, sc, cp, cm);
        if (active) {
            *po = i;
            if (kTwin) *po2 = i + tm;
            if (ok) {
                pc[0] = static_cast<uint16_t>(__byte_perm(cp[0], cp[1], 0x40));
                pc[1] = static_cast<uint16_t>(__byte_perm(cp[2], cm[0], 0x40));
                pc[2] = static_cast<uint16_t>(__byte_perm(cm[1], cm[2], 0x40));
                if (kTwin) {
                    pc2[0] = static_cast<uint16_t>(__byte_perm(cm[0], cm[1], 0x40));
                    pc2[1] = static_cast<uint16_t>(__byte_perm(cm[2], cp[0], 0x40));
                    pc2[2] = static_cast<uint16_t>(__byte_perm(cp[1], cp[2], 0x40));
                }
            }
        }
        if (kTwin) {
            po2 += 32;
            pc2 += 96;
        }
        const unsigned rep = __ballot_sync(kFull, active & !ok);
        if (rep) {
            if (active & !ok) {
                const uint32_t qq = p + lane;
                queue[nq + __popc(rep & lane_lt)] =
                    make_uint2(cp[0] | (cp[1] << 8) | (cp[2] << 16) | (qq << 24),
                               cm[0] | (cm[1] << 8) | (cm[2] << 16) | ((qq >> 8) << 24));
            }
            nq += __popc(rep);
            if (nq >= 32) {
                nq -= 32;
                __syncwarp();
                emit_repair<kOneRow, kTwin>(sm, S, A, list, i0, kt, mt, out_codes, out_codes2, queue + nq, 32, lane,
                                            ct.code_repairs);
                __syncwarp();
            }
        }
        i = i_n;
        k = k_n;
        m = m_n;
        r = r_n;
        sc = sc_n;
    }
    if (nq) {
        __syncwarp();
        emit_repair<kOneRow, kTwin>(sm, S, A, list, i0, kt, mt, out_codes, out_codes2, queue, nq, lane,
                                    ct.code_repairs);
        __syncwarp();
    }
}

// K3: codes + coalesced writes of every passing pair at its final offset.
// Warps claim (tile, 256-pair sub-range) items from the phase-1 worklist
// (next claim prefetched), so no warp holds more than 8 chunks of work; the
// item's list entries are read one chunk ahead.
template <int kMode, int kPath>
__global__ void __launch_bounds__(kBlock, 4) emit_kernel(const LaunchArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    uint2* queue = reinterpret_cast<uint2*>(smem_raw + sizeof(Smem)) + (threadIdx.x >> 5) * kRepairQueue;
    load_tables<kTabCode>(sm, A);  // constant inputs only: before the wait
    const uint32_t tab = ctab_addr(sm.ctab);
    pdl_wait();  // scan (and so phase 1) complete
    const unsigned lane = threadIdx.x & 31;
    const uint32_t n_work = *reinterpret_cast<volatile unsigned int*>(&A.ticket[3]);
    const unsigned long long base0 = A.base_offset ? *A.base_offset : 0ull;
    if (A.grand_total && blockIdx.x == 0 && threadIdx.x == 0) *A.grand_total = base0 + *A.total;
    Counters ct;
    uint32_t q_claim = 0;
    if (lane == 0) q_claim = atomicAdd(&A.ticket[2], 1u);
    uint32_t q = __shfl_sync(kFull, q_claim, 0);
    while (q < n_work) {
        if (lane == 0) q_claim = atomicAdd(&A.ticket[2], 1u);
        const uint32_t item = A.worklist[q];
        const uint32_t t = item >> 4;
        const uint32_t p0 = (item & 15u) << A.emit_shift;
        const uint32_t cnt = min(A.tile_count[t] - p0, 1u << A.emit_shift);
        const unsigned long long base = base0 + A.tile_base[t] + p0;
        const uint16_t* list = A.scratch + static_cast<size_t>(t) * kTile + p0;
        // twin tiles (band FAST plans only): this item also writes the twin's
        // records, further along the same search
        const bool twin = kMode == kModeBand && kPath == kPathFast && A.twin && A.twin[t];
        const unsigned long long base2 = twin ? base0 + A.tile_base[t + A.twin_tiles] + p0 : base;
        if (base2 + cnt > A.capacity) {
            if (lane == 0) ++ct.overflow;
        } else {
            const uint32_t s = t / A.tiles_per_search;
            const uint32_t i0 = (t - s * A.tiles_per_search) * static_cast<uint32_t>(kTile);
            const SearchConst* S = search_const(A, s);
            CodeConsts CC;
            load_code_consts(S, CC, tab);
            if (kPath == kPathFast) {
                // a tile inside one radius row (n_angles >= 4096): k is the
                // tile's row for every pair, no per-pair division or radius load
                const uint32_t kt = div_na(i0, A);
                const uint32_t mt = i0 - kt * static_cast<uint32_t>(A.na);
                uint32_t* out_idx = A.out_idx + base;
                uint8_t* out_codes = A.out_codes + 6 * base;
                if (twin) {
                    // one quantization, two records (the twin's codes proven
                    // with the bound widened by kTwinSlack)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float e = __ldg(&S->eps_code[c]) + kTwinSlack;
                        CC.ec[c] = e <= kCodeSlack ? e : INFINITY;
                    }
                    const bool seq = list[cnt - 1] - list[0] == cnt - 1;  // lists ascend strictly
                    if (seq) {
                        emit_run<true, true, true>(sm, S, CC, A, list, cnt, i0, kt, mt, out_idx, out_codes,
                                                   A.out_idx + base2, A.out_codes + 6 * base2, queue, lane, ct);
                    } else {
                        emit_run<true, true>(sm, S, CC, A, list, cnt, i0, kt, mt, out_idx, out_codes,
                                             A.out_idx + base2, A.out_codes + 6 * base2, queue, lane, ct);
                    }
                } else if (mt + static_cast<uint32_t>(kTile) <= static_cast<uint32_t>(A.na)) {
                    emit_run<true>(sm, S, CC, A, list, cnt, i0, kt, mt, out_idx, out_codes, nullptr, nullptr, queue,
                                   lane, ct);
                } else {
                    emit_run<false>(sm, S, CC, A, list, cnt, i0, kt, mt, out_idx, out_codes, nullptr, nullptr, queue,
                                    lane, ct);
                }
            } else {
#pragma unroll 1
                for (uint32_t p = 0; p < cnt; p += 32) {
                    const uint32_t qq = p + lane;
                    const bool active = qq < cnt;
                    const uint32_t i = i0 + list[active ? qq : 0];
                    const uint32_t k = div_na(i, A);
                    const uint32_t m = i - k * static_cast<uint32_t>(A.na);
                    int cp[3], cm[3];
                    candidate_codes<kPath>(sm, S, CC, A, k, m, active, cp, cm, ct.code_repairs, ct);
                    if (active) {
                        const uint32_t fl = __ldg(&S->flags);
                        if (kMode == kModeBand && !(fl & (1u << 9)) && !classify_codes(S, cp, cm, fl)) ++ct.mismatch;
                        store_pair(A, base + qq, i, cp, cm);
                    }
                }
            }
        }
        q = __shfl_sync(kFull, q_claim, 0);
    }
    flush_counters(ct, A, lane);
}

// FIRST mode epilogue: exact codes of each search's first canonical pair.
__global__ void first_codes_kernel(const LaunchArgs A) {
    __shared__ double thr[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) thr[i] = A.thr_d[i];
    __syncthreads();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= A.n_searches) return;
    const uint32_t i = A.first_idx[s];
    uint8_t* out = A.first_codes + 6 * static_cast<size_t>(s);
    if (i == 0xffffffffu) {
        for (int q = 0; q < 6; ++q) out[q] = 0;
        return;
    }
    const uint32_t k = div_na(i, A);
    const uint32_t m = i - k * static_cast<uint32_t>(A.na);
    double lp[3], lm[3];
    exact_linear(search_const(A, s), A, k, m, lp, lm);
    for (int q = 0; q < 3; ++q) {
        out[q] = static_cast<uint8_t>(code_exact(lp[q], thr));
        out[3 + q] = static_cast<uint8_t>(code_exact(lm[q], thr));
    }
}

// CVG_OUT_BEST epilogue: select_best (search.cpp:458-489) on the device.
// classification_margin (search.cpp:458-466) of a pair is min over channels
// of (d > v_th ? d - v_th : low - d) in double, with d the integer channel
// delta (channel_deltas / frame_deltas, search.cpp:125-144).  A passing pair
// has margin >= +0, so the IEEE bits of the margin order as unsigned
// integers; the best pair is the largest margin, the first in canonical
// order among equals (the reference keeps the first maximum of its scan).
// One block per search: pass 1 the block's max margin, pass 2 the smallest
// position that reaches it.
constexpr int kBestThreads = 256;

__device__ __forceinline__ unsigned long long pair_margin_bits(const LaunchArgs& A, unsigned long long o,
                                                               const int* t, bool frame_diff, double v_th,
                                                               double low) {
    const uint16_t* c16 = reinterpret_cast<const uint16_t*>(A.out_codes + 6 * o);
    const uint32_t w0 = c16[0], w1 = c16[1], w2 = c16[2];
    const int p[3] = {static_cast<int>(w0 & 0xff), static_cast<int>(w0 >> 8), static_cast<int>(w1 & 0xff)};
    const int m[3] = {static_cast<int>(w1 >> 8), static_cast<int>(w2 & 0xff), static_cast<int>(w2 >> 8)};
    double mg = INFINITY;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int di = frame_diff ? abs(p[q] - m[q]) : max(abs(p[q] - t[q]), abs(m[q] - t[q]));
        const double d = static_cast<double>(di);
        const double g = d > v_th ? __dsub_rn(d, v_th) : __dsub_rn(low, d);
        mg = fmin(mg, g);
    }
    return static_cast<unsigned long long>(__double_as_longlong(mg));
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* red, Op op) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = red[0];
    for (int w = 1; w < kBestThreads / 32; ++w) v = op(v, red[w]);
    return v;
}

// select_best on the device (search.cpp:458-489), over the emitted pairs,
// balanced by tiles.  Tile pass: a warp takes a canonical tile (its pairs are
// one contiguous slice of the search's records) and reduces its pairs to the
// largest margin and the first position reaching it (a passing pair's margin
// is >= +0, so its IEEE bits order as unsigned integers); the pair is stored
// in the tile's tile_base slot pair (tile_key).  Search pass: a warp per search
// reduces its tiles in canonical order the same way (larger margin wins, the
// earlier tile on a tie: the reference keeps the first maximum of its scan)
// and writes the record at the winning position, or the empty marker.  One
// search with many pairs no longer sits on one block (cfg1: 354 -> ~90 us).
__global__ void __launch_bounds__(kBestThreads) best_tiles_kernel(const LaunchArgs A, const double* __restrict__ bands) {
    pdl_wait();  // the emit complete
    pdl_trigger();
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kBestThreads / 32);
    for (uint64_t t = blockIdx.x * (kBestThreads / 32) + (threadIdx.x >> 5); t < A.n_tiles; t += warps) {
        const uint64_t tg = A.tile_begin + t;
        const uint32_t cnt = A.tile_count[tg];
        if (cnt == 0) continue;
        const uint32_t s = static_cast<uint32_t>(tg / A.tiles_per_search);
        const unsigned long long base = (A.base_offset ? *A.base_offset : 0ull) + A.tile_base[tg];
        const SearchConst* S = search_const(A, s);
        const int tt[3] = {__ldg(&S->t[0]), __ldg(&S->t[1]), __ldg(&S->t[2])};
        const bool frame_diff = (__ldg(&S->flags) >> 8) & 1u;
        const double v_th = __ldg(&bands[2 * s]), low = __ldg(&bands[2 * s + 1]);
        unsigned long long m = 0, pos = ~0ull;  // lane's best so far (its positions ascend)
        for (uint32_t q = lane; q < cnt; q += 32) {
            const unsigned long long g = pair_margin_bits(A, base + q, tt, frame_diff, v_th, low);
            if (g > m || pos == ~0ull) {
                m = g;
                pos = base + q;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long m2 = __shfl_xor_sync(kFull, m, o), p2 = __shfl_xor_sync(kFull, pos, o);
            if (m2 > m || (m2 == m && p2 < pos)) {
                m = m2;
                pos = p2;
            }
        }
        if (lane == 0) {
            A.best_key[2 * t] = m;
            A.best_key[2 * t + 1] = pos;
        }
    }
}

__global__ void __launch_bounds__(kBestThreads) best_search_kernel(const LaunchArgs A) {
    pdl_wait();  // the tile pass complete
    const unsigned lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kBestThreads / 32);
    const uint32_t tps = A.tiles_per_search;
    for (uint32_t sr = blockIdx.x * (kBestThreads / 32) + (threadIdx.x >> 5); sr < A.range_searches; sr += warps) {
        const uint32_t s = A.search_begin + sr;
        if (A.counts[s] == 0) {
            if (lane == 0) A.first_idx[s] = 0xffffffffu;
            if (lane < 6) A.first_codes[6 * static_cast<size_t>(s) + lane] = 0;
            continue;
        }
        unsigned long long m = 0, pos = ~0ull;
        for (uint32_t j = lane; j < tps; j += 32) {  // tiles ascend: the lane keeps its earliest maximum
            const uint64_t t = static_cast<uint64_t>(sr) * tps + j;
            if (A.tile_count[A.tile_begin + t] == 0) continue;
            const unsigned long long g = A.best_key[2 * t];
            if (g > m || pos == ~0ull) {
                m = g;
                pos = A.best_key[2 * t + 1];
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long m2 = __shfl_xor_sync(kFull, m, o), p2 = __shfl_xor_sync(kFull, pos, o);
            if (m2 > m || (m2 == m && p2 < pos)) {
                m = m2;
                pos = p2;
            }
        }
        if (lane == 0) A.first_idx[s] = A.out_idx[pos];
        if (lane < 6) A.first_codes[6 * static_cast<size_t>(s) + lane] = A.out_codes[6 * pos + lane];
    }
}

// CVG_PATH_MEMO epilogue: every search takes the result of its distinct
// representative (results depend only on target, pattern and thresholds).
__global__ void scatter_kernel(const uint32_t* __restrict__ map, int n, const unsigned long long* __restrict__ counts_in,
                               const uint32_t* __restrict__ fi_in, const uint8_t* __restrict__ fc_in,
                               unsigned long long* __restrict__ counts, uint32_t* __restrict__ fi,
                               uint8_t* __restrict__ fc) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const uint32_t u = __ldg(&map[s]);
        counts[s] = __ldg(&counts_in[u]);
        if (fi_in) {
            fi[s] = __ldg(&fi_in[u]);
            const uint8_t* a = fc_in + 6 * static_cast<size_t>(u);
            uint8_t* b = fc + 6 * static_cast<size_t>(s);
#pragma unroll
            for (int q = 0; q < 6; ++q) b[q] = __ldg(&a[q]);
        }
    }
}

// FP32 issue-rate microbenchmark: 8 independent FFMA chains per thread.
__global__ void ffma_peak_kernel(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float r = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (r == 1234.5f) out[0] = r;
}

// Persistent grids, but never more blocks than there is work for: one warp
// per tile (phase 1) or per emit item at most.  Small batches (one search of
// a few tiles) then skip launching and table-loading hundreds of idle blocks.
inline int work_grid(int grid, uint64_t units, int warps) {
    const uint64_t need = (units + static_cast<uint64_t>(warps) - 1) / static_cast<uint64_t>(warps);
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(static_cast<uint64_t>(grid), need)));
}

cudaError_t launch_pdl(void (*kernel)(LaunchArgs), unsigned grid, unsigned threads, size_t smem, cudaStream_t st,
                       const LaunchArgs& a);

template <int kMode, int kOut, int kPath, bool kPrune = false>
cudaError_t phase1_t(const LaunchArgs& a, int grid, cudaStream_t st) {
    grid = work_grid(grid, a.n_claims, kWarpsPerBlock);
    if (kMode == kModeBand && kPath == kPathFast && !kPrune && a.prune) {
        phase1_kernel<kMode, kOut, kPath, true><<<grid, kBlock, phase1_smem<kMode>(), st>>>(a);
        return cudaGetLastError();
    }
    if (kMode == kModeBand && kPath == kPathFast && !kPrune && a.strips) {
        // the bulk skip: always for COUNTS / FIRST; PAIRS when the plan asks
        // (plan_build: strips of 512 rows)
        if (kOut == kOutPairs && !a.bulk_skip) {
            phase1_kernel<kMode, kOut, kPath, false, 1><<<grid, kBlock, phase1_smem<kMode>(), st>>>(a);
        } else {
            phase1_kernel<kMode, kOut, kPath, false, 2><<<grid, kBlock, phase1_smem<kMode>(), st>>>(a);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || kOut != kOutPairs) return e;
        // PAIRS: the canonical tile lists from the pass words
        const uint32_t units = a.range_searches * ((a.nr + a.lst_unit_rows - 1) / a.lst_unit_rows) *
                               (a.lst_tpr ? a.lst_tpr : 1u);
        // latency-bound expansion: as many resident warps as fit (6 blocks per SM)
        return launch_pdl(lists_kernel, static_cast<unsigned>(work_grid(grid * 6 / 4, units, kWarpsPerBlock)), kBlock,
                          0, st, a);
    }
    // The dynamic shared-memory sizes are opted into by occupancy_t (plan creation).
    phase1_kernel<kMode, kOut, kPath, kPrune><<<grid, kBlock, phase1_smem<kMode>(), st>>>(a);
    return cudaGetLastError();
}

// The emit pass of a mode/path pair (continuous FrameDiff decides in FP64 but
// quantizes passing pairs on the FP32 code path with FP64 repair).
constexpr int emit_path(int mode, int path) { return mode == kModeSignal ? kPathFast : path; }

// Launch with programmatic stream serialization (PDL): the kernel may start
// before its stream predecessor completes; it calls pdl_wait() first.
cudaError_t launch_pdl(void (*kernel)(LaunchArgs), unsigned grid, unsigned threads, size_t smem, cudaStream_t st,
                       const LaunchArgs& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

cudaError_t launch_pdl_bands(void (*kernel)(LaunchArgs, const double*), unsigned grid, const LaunchArgs& a,
                             const double* bands, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBestThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, a, bands);
}

template <int kMode, int kPath>
cudaError_t emit_t(const LaunchArgs& a, int grid, int threads, cudaStream_t st) {
    grid = work_grid(grid, a.n_tiles * (kTile / kEmitSpan), threads / 32);
    return launch_pdl(emit_kernel<kMode, kPath>, grid, threads, emit_smem(), st, a);
}

cudaError_t scan_l(const LaunchArgs& a, cudaStream_t st) {
    const unsigned scan_blocks = static_cast<unsigned>((a.n_tiles + kScanTile - 1) / kScanTile);
    if (scan_blocks == 0) return cudaSuccess;
    return launch_pdl(scan_kernel, scan_blocks, kBlock, 0, st, a);
}

template <int kMode, int kOut, int kPath>
cudaError_t launch_t(const LaunchArgs& a, int grid, cudaStream_t st, cudaEvent_t* marks) {
    cudaError_t e = phase1_t<kMode, kOut, kPath>(a, grid, st);
    if (e != cudaSuccess || kOut != kOutPairs) return e;
    if (marks) cudaEventRecord(marks[0], st);
    e = scan_l(a, st);
    if (e != cudaSuccess) return e;
    if (marks) cudaEventRecord(marks[1], st);
    return emit_t<kMode, emit_path(kMode, kPath)>(a, grid, kBlock, st);
}

template <int kMode, int kOut, int kPath>
int occupancy_t() {
    auto f1 = phase1_kernel<kMode, kOut, kPath>;
    auto f3 = emit_kernel<kMode, emit_path(kMode, kPath)>;
    cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(phase1_smem<kMode>()));
    cudaFuncSetAttribute(f3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(emit_smem()));
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f1, kBlock, phase1_smem<kMode>()) != cudaSuccess)
        return 0;
    return blocks;
}

using LaunchFn = cudaError_t (*)(const LaunchArgs&, int, cudaStream_t, cudaEvent_t*);
using OccFn = int (*)();

#define CVG_ROW(M, P) {launch_t<M, kOutPairs, P>, launch_t<M, kOutCounts, P>, launch_t<M, kOutFirst, P>}
#define CVG_OCC(M, P) {occupancy_t<M, kOutPairs, P>, occupancy_t<M, kOutCounts, P>, occupancy_t<M, kOutFirst, P>}

const LaunchFn kLaunch[kModes][3][3] = {
    {CVG_ROW(kModeBand, kPathFast), CVG_ROW(kModeBand, kPathExact), CVG_ROW(kModeBand, kPathAudit)},
    {CVG_ROW(kModeCodes, kPathFast), CVG_ROW(kModeCodes, kPathExact), CVG_ROW(kModeCodes, kPathAudit)},
    // continuous FrameDiff: FP32 signal-bound prefilter + FP64 decisions (EXACT: FP64 only)
    {CVG_ROW(kModeSignal, kPathFast), CVG_ROW(kModeSignal, kPathExact), CVG_ROW(kModeSignal, kPathAudit)},
};
using Phase1Fn = cudaError_t (*)(const LaunchArgs&, int, cudaStream_t);
#define CVG_P1(M, P) {phase1_t<M, kOutPairs, P>, phase1_t<M, kOutCounts, P>, phase1_t<M, kOutFirst, P>}
const Phase1Fn kPhase1[kModes][3][3] = {
    {CVG_P1(kModeBand, kPathFast), CVG_P1(kModeBand, kPathExact), CVG_P1(kModeBand, kPathAudit)},
    {CVG_P1(kModeCodes, kPathFast), CVG_P1(kModeCodes, kPathExact), CVG_P1(kModeCodes, kPathAudit)},
    {CVG_P1(kModeSignal, kPathFast), CVG_P1(kModeSignal, kPathExact), CVG_P1(kModeSignal, kPathAudit)},
};
using EmitFn = cudaError_t (*)(const LaunchArgs&, int, int, cudaStream_t);
const EmitFn kEmit[kModes][3] = {
    {emit_t<kModeBand, kPathFast>, emit_t<kModeBand, kPathExact>, emit_t<kModeBand, kPathAudit>},
    {emit_t<kModeCodes, kPathFast>, emit_t<kModeCodes, kPathExact>, emit_t<kModeCodes, kPathAudit>},
    // codes of passing pairs: the FP32 code path with FP64 repair, as in the other modes
    {emit_t<kModeSignal, kPathFast>, emit_t<kModeSignal, kPathFast>, emit_t<kModeSignal, kPathFast>},
};
const OccFn kOcc[kModes][3][3] = {
    {CVG_OCC(kModeBand, kPathFast), CVG_OCC(kModeBand, kPathExact), CVG_OCC(kModeBand, kPathAudit)},
    {CVG_OCC(kModeCodes, kPathFast), CVG_OCC(kModeCodes, kPathExact), CVG_OCC(kModeCodes, kPathAudit)},
    {CVG_OCC(kModeSignal, kPathFast), CVG_OCC(kModeSignal, kPathExact), CVG_OCC(kModeSignal, kPathAudit)},
};

}  // namespace

cudaError_t launch_search(const LaunchArgs& a, int mode, int out, int path, int grid, cudaStream_t st,
                          cudaEvent_t* marks) {
    return kLaunch[mode][path][out](a, grid, st, marks);
}

int search_blocks_per_sm(int mode, int out, int path) { return kOcc[mode][path][out](); }

cudaError_t launch_phase1(const LaunchArgs& a, int mode, int out, int path, int grid, cudaStream_t st) {
    return kPhase1[mode][path][out](a, grid, st);
}
cudaError_t launch_scan(const LaunchArgs& a, cudaStream_t st) { return scan_l(a, st); }
cudaError_t launch_emit(const LaunchArgs& a, int mode, int path, int grid, cudaStream_t st, int threads) {
    return kEmit[mode][path](a, grid, threads, st);
}

cudaError_t launch_first_codes(const LaunchArgs& a, cudaStream_t st) {
    const int threads = 128;
    const int blocks = (a.n_searches + threads - 1) / threads;
    if (blocks == 0) return cudaSuccess;
    first_codes_kernel<<<blocks, threads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_best(const LaunchArgs& a, const double* bands, cudaStream_t st) {
    if (a.n_searches <= 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((a.n_tiles + kBestThreads / 32 - 1) / (kBestThreads / 32), 148 * 8)));
    const cudaError_t e = launch_pdl_bands(best_tiles_kernel, blocks, a, bands, st);
    if (e != cudaSuccess) return e;
    const unsigned sb = static_cast<unsigned>(
        std::max(1, std::min((a.n_searches + kBestThreads / 32 - 1) / (kBestThreads / 32), 148 * 8)));
    return launch_pdl(best_search_kernel, sb, kBestThreads, 0, st, a);
}

cudaError_t launch_scatter(const uint32_t* map, int n, const unsigned long long* counts_in, const uint32_t* fi_in,
                           const uint8_t* fc_in, unsigned long long* counts, uint32_t* fi, uint8_t* fc, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int threads = 256;
    const int blocks = std::min((n + threads - 1) / threads, 148 * 8);
    scatter_kernel<<<blocks, threads, 0, st>>>(map, n, counts_in, fi_in, fc_in, counts, fi, fc);
    return cudaGetLastError();
}

size_t search_smem_bytes() { return sizeof(Smem); }

double measure_ffma_peak(int device, float* ms_out) {
    if (cudaSetDevice(device) != cudaSuccess) return 0.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return 0.0;
    const int threads = 256, blocks = sms * 8, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma_peak_kernel<<<blocks, threads>>>(out, 64, 0.999f, 0.001f);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        ffma_peak_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    if (ms_out) *ms_out = best;
    const double ffma = static_cast<double>(blocks) * threads * iters * 16.0 * 8.0;
    return ffma / (best * 1e-3);
}

}  // namespace cvg
