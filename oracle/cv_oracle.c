/*
 * cv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference color-pair search (arXiv 2507.22901,
 * `colorvibe`), used as the parity checker for the B200 kernels.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library; the product path (paper_2507_22901_b200) never links it.
 *
 * Every function follows the reference file:line it cites (paths relative to
 * the reference checkout's proj/ directory).  The arithmetic is IEEE binary64
 * with round-to-nearest and NO fused multiply-add (build flag
 * -ffp-contract=off, as src/CMakeLists.txt:21-28), evaluated in the same
 * order as the reference, so that results are bit-identical to it.  libm
 * (sin, cos, pow, cbrt, floor) is the host glibc, exactly as the reference.
 *
 * Parity of this restatement is pinned by tests/test_oracle.py against
 *   - the reference sources themselves compiled into oracle/_ref (ref_shim.cpp),
 *   - tests/golden/* fixtures (known-answer constants, per-search counts and
 *     record hashes, the reference's own tests/golden/matrix_aggregated.csv).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CVO_EXPORT __attribute__((visibility("default")))

/* ---- pinned constants: src/convert_kernel.hpp:21-60 ------------------- */

static const double kRgbToXyz[3][3] = {
    {0.4124, 0.3576, 0.1805},
    {0.2126, 0.7152, 0.0722},
    {0.0193, 0.1192, 0.9505},
};
static const double kLabEpsilon = 216.0 / 24389.0; /* convert_kernel.hpp:50 */
static const double kLabKappa = 24389.0 / 27.0;    /* :51 */
static const double kInvKappa = 27.0 / 24389.0;    /* :58 */
static const double kInv500 = 1.0 / 500.0;         /* :59 */
static const double kInv200 = 1.0 / 200.0;         /* :60 */

static double kXyzToRgb[3][3]; /* adjugate / det, convert_kernel.hpp:27-47 */
static double kD65[3];         /* row sums, src/color.cpp:13-20 */
static double kThr[256];       /* QuantTable::thresholds, convert_kernel.hpp:123-141 */

/* convert_kernel.hpp:27-43 -- same expressions, same association. */
static void make_inverse(void) {
    const double(*m)[3] = kRgbToXyz;
    const double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                       m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                       m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
    double(*r)[3] = kXyzToRgb;
    r[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
    r[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
    r[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
    r[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
    r[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
    r[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
    r[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / det;
    r[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
    r[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
}

/* ---- scalar conversion kernel: convert_kernel.hpp:66-117 --------------- */

static double lab_f(double t) { /* :66-68 */
    return t > kLabEpsilon ? cbrt(t) : (kLabKappa * t + 16.0) / 116.0;
}

static double lab_f_inv(double u) { /* :70-73 */
    const double u3 = (u * u) * u;
    return u3 > kLabEpsilon ? u3 : (116.0 * u - 16.0) * kInvKappa;
}

static double srgb_eotf(double u) { /* :76-78 */
    return u <= 0.04045 ? u / 12.92 : pow((u + 0.055) / 1.055, 2.4);
}

static double srgb_oetf(double x) { /* :81-83 */
    return x <= 0.0031308 ? 12.92 * x : 1.055 * pow(x, 1.0 / 2.4) - 0.055;
}

static double signal_value(double linear) { /* :109-112 */
    const double x = linear < 0.0 ? 0.0 : (linear > 1.0 ? 1.0 : linear);
    return 255.0 * srgb_oetf(x);
}

static int quantize_signal(double linear) { /* :115-117 */
    return (int)floor(signal_value(linear) + 0.5);
}

/* QuantTable() bisection, convert_kernel.hpp:127-141. */
static void make_thresholds(void) {
    kThr[0] = 0.0;
    for (int code = 1; code <= 255; ++code) {
        double lo = kThr[code - 1];
        double hi = 1.0;
        while (nextafter(lo, 1.0) < hi) {
            const double mid = 0.5 * (lo + hi);
            if (quantize_signal(mid) >= code) {
                hi = mid;
            } else {
                lo = mid;
            }
        }
        kThr[code] = hi;
    }
}

/* QuantTable::code, convert_kernel.hpp:148-154, restated as a binary search
 * for the largest c with x >= thresholds[c] (equivalent by construction of the
 * table; pinned against the reference's guess-and-walk in the tests). */
static int table_code(double x) {
    if (x <= 0.0) return 0;
    if (x >= 1.0) return 255;
    int lo = 0, hi = 255; /* invariant: thr[lo] <= x, answer in [lo, hi] */
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (x >= kThr[mid]) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__attribute__((constructor)) static void cvo_init(void) {
    make_inverse();
    const double(*m)[3] = kRgbToXyz;
    kD65[0] = (m[0][0] + m[0][1]) + m[0][2];
    kD65[1] = (m[1][0] + m[1][1]) + m[1][2];
    kD65[2] = (m[2][0] + m[2][1]) + m[2][2];
    make_thresholds();
}

/* src/color.cpp:57-70 */
static void srgb_to_lab(const int32_t c[3], const double wp[3], double lab[3]) {
    const double rl = srgb_eotf(c[0] / 255.0);
    const double gl = srgb_eotf(c[1] / 255.0);
    const double bl = srgb_eotf(c[2] / 255.0);
    const double(*m)[3] = kRgbToXyz;
    const double x = (m[0][0] * rl + m[0][1] * gl) + m[0][2] * bl;
    const double y = (m[1][0] * rl + m[1][1] * gl) + m[1][2] * bl;
    const double z = (m[2][0] * rl + m[2][1] * gl) + m[2][2] * bl;
    const double fx = lab_f(x / wp[0]);
    const double fy = lab_f(y / wp[1]);
    const double fz = lab_f(z / wp[2]);
    lab[0] = 116.0 * fy - 16.0;
    lab[1] = 500.0 * (fx - fy);
    lab[2] = 200.0 * (fy - fz);
}

/* convert_kernel.hpp:94-105 */
static void lab_to_linear(const double lab[3], const double wp[3], double lin[3]) {
    const double fy = (lab[0] + 16.0) / 116.0;
    const double fx = fy + lab[1] * kInv500;
    const double fz = fy - lab[2] * kInv200;
    const double x = wp[0] * lab_f_inv(fx);
    const double y = wp[1] * lab_f_inv(fy);
    const double z = wp[2] * lab_f_inv(fz);
    const double(*m)[3] = kXyzToRgb;
    lin[0] = (m[0][0] * x + m[0][1] * y) + m[0][2] * z;
    lin[1] = (m[1][0] * x + m[1][1] * y) + m[1][2] * z;
    lin[2] = (m[2][0] * x + m[2][1] * y) + m[2][2] * z;
}

/* ---- search: src/search.cpp ------------------------------------------- */

enum { CVO_QUANTIZED = 0, CVO_CONTINUOUS = 1 };
enum { CVO_TARGET_SWING = 0, CVO_FRAME_DIFF = 1 };

typedef struct {
    int32_t t[3];
    int bits[3];
    double v_th, low;
    int mode, basis;
} Classifier;

static double dmax(double a, double b) { return a > b ? a : b; } /* std::max */

/* channel_deltas :125-136, frame_deltas :138-144, continuous_deltas :161-180 */
static void deltas_of(const Classifier* c, const int sp[3], const int sm[3],
                      const double lp[3], const double lm[3], double d[3]) {
    for (int k = 0; k < 3; ++k) {
        if (c->mode == CVO_QUANTIZED) {
            if (c->basis == CVO_TARGET_SWING) {
                const int a = abs(sp[k] - c->t[k]), b = abs(sm[k] - c->t[k]);
                d[k] = (double)(a > b ? a : b);
            } else {
                d[k] = (double)abs(sp[k] - sm[k]);
            }
        } else {
            const double p = signal_value(lp[k]);
            const double m = signal_value(lm[k]);
            if (c->basis == CVO_FRAME_DIFF) {
                d[k] = fabs(p - m);
            } else {
                d[k] = dmax(fabs(p - c->t[k]), fabs(m - c->t[k]));
            }
        }
    }
}

/* classify_pair :146-157 */
static int classify(const Classifier* c, const double d[3]) {
    int ok = 1;
    for (int k = 0; k < 3; ++k) {
        ok &= c->bits[k] ? (d[k] > c->v_th) : (d[k] <= c->low);
    }
    return ok;
}

typedef struct {
    uint32_t* idx;
    uint8_t* codes;
    double* deltas;
    int64_t cap;
    int64_t n;
} Sink;

static void emit(Sink* s, uint32_t idx, const int sp[3], const int sm[3], const double d[3]) {
    if (s->n < s->cap) {
        if (s->idx) s->idx[s->n] = idx;
        if (s->codes) {
            uint8_t* c = s->codes + 6 * s->n;
            c[0] = (uint8_t)sp[0]; c[1] = (uint8_t)sp[1]; c[2] = (uint8_t)sp[2];
            c[3] = (uint8_t)sm[0]; c[4] = (uint8_t)sm[1]; c[5] = (uint8_t)sm[2];
        }
        if (s->deltas) memcpy(s->deltas + 3 * s->n, d, 3 * sizeof(double));
    }
    s->n++;
}

/* serial_search :184-218 -- one candidate at a time through the scalar API
 * (displaced_pair :113-123 computes sin/cos per candidate). */
static void serial_rows(const Classifier* c, const double lab[3], const double wp[3],
                        const double* radii, int nr, const double* angles, int na,
                        Sink* out) {
    for (int k = 0; k < nr; ++k) {
        for (int j = 0; j < na; ++j) {
            const double da = radii[k] * sin(angles[j]);
            const double db = radii[k] * cos(angles[j]);
            const double plus[3] = {lab[0], lab[1] + da, lab[2] + db};
            const double minus[3] = {lab[0], lab[1] - da, lab[2] - db};
            double lp[3], lm[3];
            lab_to_linear(plus, wp, lp);
            lab_to_linear(minus, wp, lm);
            const int sp[3] = {quantize_signal(lp[0]), quantize_signal(lp[1]), quantize_signal(lp[2])};
            const int sm[3] = {quantize_signal(lm[0]), quantize_signal(lm[1]), quantize_signal(lm[2])};
            double d[3];
            deltas_of(c, sp, sm, lp, lm, d);
            if (classify(c, d)) emit(out, (uint32_t)((uint64_t)k * na + j), sp, sm, d);
        }
    }
}

/* make_bands :291-329 */
static void make_bands(const Classifier* c, double lo[3], double hi[3], int inv[3]) {
    const int exact = c->mode == CVO_QUANTIZED && c->basis == CVO_TARGET_SWING;
    const int k1 = c->v_th >= 255.0 ? 256 : (int)c->v_th + 1;
    const int q0 = c->low >= 255.0 ? 255 : (int)c->low;
    for (int k = 0; k < 3; ++k) {
        const int t = c->t[k];
        if (!exact) {
            lo[k] = -HUGE_VAL; hi[k] = HUGE_VAL; inv[k] = 0;
        } else if (c->bits[k]) {
            lo[k] = t - k1 + 1 >= 1 ? kThr[t - k1 + 1] : -HUGE_VAL;
            hi[k] = t + k1 <= 255 ? kThr[t + k1] : HUGE_VAL;
            inv[k] = 1;
        } else {
            lo[k] = t - q0 >= 1 ? kThr[t - q0] : -HUGE_VAL;
            hi[k] = t + q0 + 1 <= 255 ? kThr[t + q0 + 1] : HUGE_VAL;
            inv[k] = 0;
        }
    }
}

typedef struct {
    const Classifier* c;
    const double* lab;
    const double* wp;
    const double* radii;
    const double* angles;
    const double* sin_a;
    const double* cos_a;
    int na;
    int row_begin, row_end;
    Sink sink;
} BatchJob;

/* batch_rows :335-399 with pass1_row :230-278 inlined per candidate. */
static void* batch_rows(void* arg) {
    BatchJob* J = (BatchJob*)arg;
    const Classifier* c = J->c;
    const double(*m)[3] = kXyzToRgb;
    const double fy = (J->lab[0] + 16.0) / 116.0;
    const double yv = J->wp[1] * lab_f_inv(fy);
    const double cy[3] = {m[0][1] * yv, m[1][1] * yv, m[2][1] * yv};
    const double ta = J->lab[1], tb = J->lab[2];
    const double wx = J->wp[0], wz = J->wp[2];
    double lo[3], hi[3];
    int inv[3];
    make_bands(c, lo, hi, inv);
    for (int k = J->row_begin; k < J->row_end; ++k) {
        const double r = J->radii[k];
        for (int j = 0; j < J->na; ++j) {
            const double da = r * J->sin_a[j];
            const double db = r * J->cos_a[j];
            const double fxp = fy + (ta + da) * kInv500;
            const double fzp = fy - (tb + db) * kInv200;
            const double xp = wx * lab_f_inv(fxp);
            const double zp = wz * lab_f_inv(fzp);
            const double fxm = fy + (ta - da) * kInv500;
            const double fzm = fy - (tb - db) * kInv200;
            const double xm = wx * lab_f_inv(fxm);
            const double zm = wz * lab_f_inv(fzm);
            double lp[3], lm[3];
            for (int q = 0; q < 3; ++q) {
                lp[q] = (m[q][0] * xp + cy[q]) + m[q][2] * zp;
                lm[q] = (m[q][0] * xm + cy[q]) + m[q][2] * zm;
            }
            int ok = 1;
            for (int q = 0; q < 3; ++q) {
                const int in = (lp[q] >= lo[q]) & (lp[q] < hi[q]) & (lm[q] >= lo[q]) & (lm[q] < hi[q]);
                ok &= in ^ inv[q];
            }
            if (!ok) continue;
            const int sp[3] = {table_code(lp[0]), table_code(lp[1]), table_code(lp[2])};
            const int sm[3] = {table_code(lm[0]), table_code(lm[1]), table_code(lm[2])};
            double d[3];
            deltas_of(c, sp, sm, lp, lm, d);
            if (classify(c, d)) emit(&J->sink, (uint32_t)((uint64_t)k * J->na + j), sp, sm, d);
        }
    }
    return NULL;
}

/* ---- exported API ------------------------------------------------------ */

CVO_EXPORT void cvo_thresholds(double out[256]) { memcpy(out, kThr, sizeof(kThr)); }
CVO_EXPORT void cvo_xyz_to_rgb(double out[9]) { memcpy(out, kXyzToRgb, sizeof(kXyzToRgb)); }
CVO_EXPORT void cvo_white(double out[3]) { memcpy(out, kD65, sizeof(kD65)); }
CVO_EXPORT int cvo_quantize(double linear) { return quantize_signal(linear); }
CVO_EXPORT int cvo_table_code(double linear) { return table_code(linear); }

CVO_EXPORT void cvo_srgb_to_lab(const int32_t rgb[3], const double* wp, double lab[3]) {
    srgb_to_lab(rgb, wp ? wp : kD65, lab);
}

CVO_EXPORT void cvo_lab_to_linear(const double lab[3], const double* wp, double lin[3]) {
    lab_to_linear(lab, wp ? wp : kD65, lin);
}

/*
 * One search (target, pattern, thresholds) over an explicit grid; the grid
 * and inputs are assumed valid (validation is the product's job; the tests
 * check it against the reference separately).  method 0 = serial_search,
 * 1 = batch_search with `threads` contiguous radius slices (search.cpp:421-455).
 * Records go to idx[] (k*na+m), codes[] (plus rgb, minus rgb) and deltas[]
 * (any may be NULL) up to cap; the return value is the full pair count.
 */
CVO_EXPORT int64_t cvo_search(const int32_t rgb[3], int pattern_bits, double v_th,
                              double r_novib, const double* radii, int nr,
                              const double* angles, int na, int delta_mode,
                              int delta_basis, const double* wp, int method,
                              int threads, uint32_t* idx, uint8_t* codes,
                              double* deltas, int64_t cap) {
    if (nr <= 0 || na <= 0) return 0;
    if (!wp) wp = kD65;
    Classifier c;
    memcpy(c.t, rgb, sizeof(c.t));
    c.bits[0] = (pattern_bits >> 2) & 1;
    c.bits[1] = (pattern_bits >> 1) & 1;
    c.bits[2] = pattern_bits & 1;
    c.v_th = v_th;
    c.low = v_th * r_novib; /* Thresholds::low_band, search.hpp:33 */
    c.mode = delta_mode;
    c.basis = delta_basis;
    double lab[3];
    srgb_to_lab(rgb, wp, lab);
    Sink top = {idx, codes, deltas, cap, 0};
    if (method == 0) {
        serial_rows(&c, lab, wp, radii, nr, angles, na, &top);
        return top.n;
    }
    double* sin_a = (double*)malloc(sizeof(double) * na);
    double* cos_a = (double*)malloc(sizeof(double) * na);
    for (int j = 0; j < na; ++j) { /* search.cpp:414-419 */
        sin_a[j] = sin(angles[j]);
        cos_a[j] = cos(angles[j]);
    }
    if (threads < 1) threads = 1;
    if (threads > nr) threads = nr;
    /* counts only when the caller asked for no records */
    const int store = idx || codes || deltas;
    BatchJob* jobs = (BatchJob*)calloc(threads, sizeof(BatchJob));
    pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
    /* Per-slice scratch sinks; concatenated in slice order (search.cpp:448-455). */
    for (int w = 0; w < threads; ++w) {
        BatchJob* J = &jobs[w];
        J->c = &c; J->lab = lab; J->wp = wp; J->radii = radii; J->angles = angles;
        J->sin_a = sin_a; J->cos_a = cos_a; J->na = na;
        J->row_begin = (int)((int64_t)nr * w / threads);
        J->row_end = (int)((int64_t)nr * (w + 1) / threads);
        const int64_t slice_cap = store ? (int64_t)(J->row_end - J->row_begin) * na : 0;
        J->sink.cap = slice_cap;
        J->sink.idx = (uint32_t*)malloc(sizeof(uint32_t) * (slice_cap ? slice_cap : 1));
        J->sink.codes = (uint8_t*)malloc(6 * (slice_cap ? slice_cap : 1));
        J->sink.deltas = deltas ? (double*)malloc(sizeof(double) * 3 * (slice_cap ? slice_cap : 1)) : NULL;
        J->sink.n = 0;
        if (threads == 1) batch_rows(J); else pthread_create(&tid[w], NULL, batch_rows, J);
    }
    for (int w = 0; w < threads; ++w) {
        BatchJob* J = &jobs[w];
        if (threads > 1) pthread_join(tid[w], NULL);
        if (!store) top.n += J->sink.n;
        for (int64_t q = 0; store && q < J->sink.n; ++q) {
            const uint8_t* cc = J->sink.codes + 6 * q;
            const int sp[3] = {cc[0], cc[1], cc[2]};
            const int sm[3] = {cc[3], cc[4], cc[5]};
            double d[3] = {0, 0, 0};
            if (J->sink.deltas) memcpy(d, J->sink.deltas + 3 * q, sizeof(d));
            emit(&top, J->sink.idx[q], sp, sm, d);
        }
        free(J->sink.idx); free(J->sink.codes); free(J->sink.deltas);
    }
    free(jobs); free(tid); free(sin_a); free(cos_a);
    return top.n;
}
