/*
 * cvg.h -- C-ABI of the B200 color-pair search (libcolorvibe_gpu.so).
 *
 * Drop-in boundary for the reference hot path `colorvibe::batch_search`
 * (reference proj/include/colorvibe/search.hpp:126-130, src/search.cpp:403-456)
 * and its pybind binding `colorvibe.batch_search` (proj/bindings/module.cpp:121-131).
 * One `cvg_search` call evaluates a whole batch of searches -- the loop the
 * reference runs one call at a time in feasibility_matrix
 * (src/feasibility.cpp:261-292) and the bench sweep (src/bench.cpp:18-34).
 *
 * Plain C types only: no torch, no C++ in any signature.  All functions are
 * thread-safe; a context may be shared by threads (calls on one context are
 * serialized internally).  Errors are reported as status codes plus a
 * thread-local message (cvg_last_error); the C++ wrapper maps CVG_EINVAL to
 * std::invalid_argument and everything else to std::runtime_error, the
 * exception types the reference throws (search.cpp:22-30, 49-56, 92-111).
 *
 * There is no CPU fallback: if the CUDA kernels cannot run, calls fail with
 * CVG_ECUDA.  Options the device path does not implement fail with
 * CVG_EUNSUPPORTED instead of silently computing on the host.
 */
#ifndef CVG_H_
#define CVG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVG_API __attribute__((visibility("default")))

/* status codes */
#define CVG_OK 0
#define CVG_EINVAL 1       /* invalid color / grid / thresholds / pattern (reference: invalid_argument) */
#define CVG_ECUDA 2        /* CUDA runtime failure, no device, kernel image missing */
#define CVG_ENOMEM 3       /* host or device allocation failed */
#define CVG_EOVERFLOW 4    /* device pair buffer too small (counts are still valid) */
#define CVG_EUNSUPPORTED 5 /* option combination not implemented on the device path */
#define CVG_EUNDECIDED 6   /* Continuous x FrameDiff: a decision depends on the last bits of glibc pow
                              (|s(p) - s(m)| within ~1e-12 of a threshold); never observed, fails loudly */

/* SearchOptions::delta_mode / delta_basis (search.hpp:81-96).  All four
 * combinations run on the device.  Continuous x FrameDiff compares
 * |s(p) - s(m)| of device-pow signal values against the thresholds with the
 * device/glibc pow error margin; a decision inside it returns CVG_EUNDECIDED. */
#define CVG_DELTA_QUANTIZED 0
#define CVG_DELTA_CONTINUOUS 1
#define CVG_BASIS_TARGET_SWING 0
#define CVG_BASIS_FRAME_DIFF 1

/* what a search returns */
#define CVG_OUT_PAIRS 0  /* every passing pair, canonical (search, radius, angle) order */
#define CVG_OUT_COUNTS 1 /* per-search pair count only */
#define CVG_OUT_FIRST 2  /* per-search count + first pair in canonical order (per-pixel mode) */
#define CVG_OUT_BEST 3   /* per-search count + select_best's pair (search.cpp:458-489): the largest
                            classification_margin, ties to the first in canonical order; chosen
                            on the device (first_idx / first_codes hold it).  DeltaMode::Quantized
                            only (continuous deltas need glibc pow: CVG_EUNSUPPORTED) */

/* evaluation path (all give identical results) */
#define CVG_PATH_FAST 0  /* FP32 with a proven error bound + FP64 repair of near-boundary values */
#define CVG_PATH_EXACT 1 /* FP64 op-for-op restatement for every candidate (serial_search) */
#define CVG_PATH_AUDIT 2 /* both; counts bound violations (tests) */
#define CVG_PATH_PRUNED 3 /* FAST, plus whole radius rows decided by a certified FP64 bound
                             (TargetSwing, aligned grids): same results; candidates of a
                             pruned row are decided without being evaluated one by one */
#define CVG_PATH_MEMO 4   /* COUNTS / FIRST only: FAST over the DISTINCT searches of the batch
                             (target, pattern, v_th, r_novib), each search's count / first pair
                             then scattered from its representative on the device.  Same
                             results (they depend only on those four values); a per-pixel batch
                             of 8.3M pixels with ~22K distinct colors evaluates ~22K searches.
                             Reported apart from the per-candidate figures (memoized). */

typedef struct cvg_ctx cvg_ctx;
typedef struct cvg_plan cvg_plan;
typedef struct cvg_layout cvg_layout;

/*
 * A batch of searches over one explicit grid.  Search s is
 * (target_rgb[3s..3s+2], pattern_bits[s], v_th[s], r_novib[s]); pattern bits
 * are r<<2 | g<<1 | b ("101" == 5), BitPattern search.hpp:14-24.  The grid is
 * VibrationGrid (search.hpp:39-53): radii >= 0 strictly increasing, angles in
 * [0, 2pi) strictly increasing, radians.  n_radii * n_angles must be < 2^32.
 */
typedef struct {
    int32_t n_searches;
    const int32_t* target_rgb;   /* [n_searches * 3], codes in [0, 255] */
    const int32_t* pattern_bits; /* [n_searches], 1..7 */
    const double* v_th;          /* [n_searches], > 0 */
    const double* r_novib;       /* [n_searches], (0, 1] */
    int32_t n_radii;
    const double* radii;
    int32_t n_angles;
    const double* angles;
    int32_t delta_mode;         /* CVG_DELTA_* */
    int32_t delta_basis;        /* CVG_BASIS_* */
    const double* white_point;  /* [3] or NULL for d65_white() (color.cpp:13-20) */
    int32_t output;             /* CVG_OUT_* */
    int32_t path;               /* CVG_PATH_* */
    int32_t workers;            /* accepted for API parity, ignored: results never depend on it */
} cvg_search_desc;

/*
 * Host-side result (library-owned; release with cvg_result_free).  Its
 * buffers are pinned blocks of the context's pool; a result may outlive its
 * context (cvg_destroy hands the blocks of live results over to them).
 * Pair p: idx[p] = k * n_angles + m (radius index k, angle index m),
 * codes[6p .. 6p+5] = plus r,g,b then minus r,g,b.  Pairs of search s are
 * [offsets[s], offsets[s+1]).  FIRST and BEST modes fill first_idx/first_codes
 * instead (first_idx = 0xFFFFFFFF when a search has no pair).
 */
typedef struct {
    int32_t n_searches;
    uint64_t n_pairs;
    uint64_t* counts;      /* [n_searches] */
    uint64_t* offsets;     /* [n_searches + 1] (PAIRS) */
    uint32_t* idx;         /* [n_pairs] (PAIRS) */
    uint8_t* codes;        /* [n_pairs * 6] (PAIRS) */
    uint32_t* first_idx;   /* [n_searches] (FIRST / BEST) */
    uint8_t* first_codes;  /* [n_searches * 6] (FIRST / BEST) */
    /* diagnostics */
    uint64_t n_candidates;
    uint64_t n_band_repairs;  /* candidates whose band decision went to FP64 */
    uint64_t n_code_repairs;  /* passing candidates whose codes went to FP64 */
    uint64_t n_audit_violations; /* PATH_AUDIT: FP32 "certain" decisions that were wrong (must be 0) */
    uint64_t n_class_mismatch;   /* band decision != classify_pair on exact codes (must be 0) */
    float audit_max_ratio;       /* PATH_AUDIT: max |lin32 - lin64| / bound (must be < 1) */
    float kernel_ms;             /* device time of the search kernels of this call */
    uint64_t h2d_bytes;          /* host->device bytes this call copied (tables + constants) */
    uint64_t d2h_bytes;          /* device->host bytes this call copied (counts, stats, pairs) */
    /* wall-clock breakdown of a cvg_search call (ms): host prep (validation,
     * glibc tables, per-target constants), H2D upload, launch -> counts on
     * host, pair D2H, whole call */
    float prep_ms, h2d_ms, device_ms, d2h_ms, total_ms;
} cvg_result;

/* ---- context ----------------------------------------------------------- */
CVG_API int cvg_create(int device, cvg_ctx** out);
CVG_API void cvg_destroy(cvg_ctx* ctx);
CVG_API const char* cvg_last_error(void);
CVG_API const char* cvg_version(void);

/* ---- one-shot host API: host buffers in, host result out ------------------
 * Validates exactly like the reference (messages included), prepares the
 * per-target constants and glibc tables on the host, copies them to the
 * device, runs the fused kernel, and copies counts + pairs back. */
CVG_API int cvg_search(cvg_ctx* ctx, const cvg_search_desc* desc, cvg_result* out);
/* validation only (no device needed): CVG_OK or the status/message cvg_search would fail with */
CVG_API int cvg_validate(const cvg_search_desc* desc);
CVG_API void cvg_result_free(cvg_result* res);

/* ---- plan API: device-resident repeated runs (benchmarks, pipelines) -----
 * cvg_plan_create does validation + host prep + upload once.  cvg_plan_run
 * enqueues the search on `stream` (a cudaStream_t, 0 = legacy default) with
 * inputs already in HBM; results stay on the device.  cvg_plan_sync waits
 * and reports overflow (CVG_EOVERFLOW if pair capacity was short: counts are
 * valid, rerun after cvg_plan_reserve).  cvg_plan_fetch copies results to a
 * host cvg_result. */
CVG_API int cvg_plan_create(cvg_ctx* ctx, const cvg_search_desc* desc, cvg_plan** out);
CVG_API void cvg_plan_destroy(cvg_plan* plan);
CVG_API int cvg_plan_reserve(cvg_plan* plan, uint64_t pair_capacity);
CVG_API int cvg_plan_run(cvg_plan* plan, void* stream);
CVG_API int cvg_plan_sync(cvg_plan* plan, uint64_t* n_pairs);
CVG_API int cvg_plan_fetch(cvg_plan* plan, cvg_result* out);
/* device pointers of the plan's outputs (valid until the plan is destroyed) */
CVG_API int cvg_plan_device_outputs(cvg_plan* plan, uint64_t** counts, uint32_t** idx,
                                    uint8_t** codes, uint64_t* capacity);
/* Copies the last run's per-search counts (u64, n_searches), pair idx (u32)
 * and codes (6 B) -- n_pairs of each, as cvg_plan_sync reported -- into
 * caller device buffers, enqueued on `stream` (NULL pointers skip an array).
 * For collectives on framework tensors (e.g. NCCL all_gather of results). */
CVG_API int cvg_plan_copy_outputs(cvg_plan* plan, uint64_t* counts, uint32_t* idx, uint8_t* codes,
                                  uint64_t n_pairs, void* stream);
/* FIRST plans: copies the last run's per-search first pair (u32 idx, 6 code
 * bytes) into caller device buffers, enqueued on `stream`. */
CVG_API int cvg_plan_copy_first(cvg_plan* plan, uint32_t* first_idx, uint8_t* first_codes, void* stream);
/* searches the plan's kernels evaluate (MEMO: the distinct ones; else all) */
CVG_API int32_t cvg_plan_evaluated_searches(const cvg_plan* plan);
/* 1 if the plan's PAIRS emit uses twin tiles: on a grid symmetric under
 * theta -> theta + pi (proven on the host), each pair of tiles whose pass
 * words are identical is quantized once and written twice */
CVG_API int cvg_plan_twin_tiles(const cvg_plan* plan);
/* device time (ms) of the search kernel(s) of the plan's last completed run */
CVG_API int cvg_plan_last_kernel_ms(cvg_plan* plan, float* ms);
/* per-kernel device time (ms) of the last run: phase 1 (candidate decisions),
 * offset scan, pair emit (scan/emit are 0 outside CVG_OUT_PAIRS; the FIRST
 * epilogue is counted in phase 1) */
CVG_API int cvg_plan_last_phase_ms(cvg_plan* plan, float* phase1_ms, float* scan_ms, float* emit_ms);
/* Record events between the three kernels of the next runs, so that
 * cvg_plan_last_phase_ms can split a run (default off: the kernels then
 * launch with programmatic dependent launch and overlap their hand-off). */
CVG_API int cvg_plan_set_phase_marks(cvg_plan* plan, int on);
/* bytes of device-resident input the plan uploaded (constants + grid tables) */
CVG_API uint64_t cvg_plan_input_bytes(const cvg_plan* plan);
/* number of kernel launches one cvg_plan_run enqueues */
CVG_API int cvg_plan_launches(const cvg_plan* plan);
CVG_API uint64_t cvg_plan_candidates(const cvg_plan* plan);

/* ---- host-side scalar helpers of the reference API (color.hpp:34-66) ------
 * Exact host conversions (same glibc pow/cbrt as the reference); used by the
 * C++ / Python API surface, never by the search itself. */
CVG_API int cvg_srgb_to_lab(const int32_t rgb[3], const double* white_point, double lab[3]);
CVG_API int cvg_lab_to_srgb_clipped(const double lab[3], const double* white_point, int32_t rgb[3]);
/* returns 1 if in gamut (rgb filled), 0 if not, negative status on error */
CVG_API int cvg_lab_to_srgb(const double lab[3], const double* white_point, int32_t rgb[3]);
CVG_API void cvg_d65_white(double out[3]);
/* pre-quantization signal values 255*oetf(clamp(lin)) of both endpoints of the
 * pair (radius, angle) around `lab` (search.cpp:113-123, convert_kernel.hpp:
 * 109-112): materializes DeltaMode::Continuous deltas of emitted pairs */
CVG_API int cvg_pair_signal(const double lab[3], double radius, double angle, const double* white_point,
                            double sp[3], double sm[3]);
/* Both endpoints of the pair (radius, angle) around `lab`, evaluated on the
 * host exactly as the reference's serial_search does per candidate
 * (search.cpp:184-218: displaced_pair, lab_to_linear, quantize_signal /
 * signal_value): codes sp/sm and pre-quantization signals gp/gm.  The scalar
 * "previous method" of the API (colorvibe::serial_search), never used by the
 * device search. */
CVG_API int cvg_pair_eval(const double lab[3], double radius, double angle, const double* white_point,
                          int32_t sp[3], int32_t sm[3], double gp[3], double gm[3]);
CVG_API void cvg_quant_thresholds(double out[256]);
/* The kernels' FP32 code table: 4097 buckets of linear [0, 1] x {threshold t,
 * code below (int32 bits)}; 8194 floats.  Exposed so tests can check it on
 * the host. */
CVG_API void cvg_code_table(float out[8194]);
/* The Continuous x FrameDiff prefilter's signal bounds: 4097 buckets x
 * {L, U}, L <= signal_value(x) <= U over bucket i = [(i - 1/2), (i + 1/2)] / 4096. */
CVG_API void cvg_signal_table(float out[8194]);
CVG_API float cvg_code_slack(void);

/* FP32 FFMA issue-rate microbenchmark (roofline denominator); returns
 * lane-FFMA per second measured on `device`, 0 on failure. */
CVG_API double cvg_measure_ffma_peak(int device, float* ms_out);

/* ---- codec image passes (reference src/codec.cpp:65-165) -------------------
 * Rasters are 8-bit RGB, interleaved, row-major, width*height*3 bytes
 * (image.hpp:12-14).  A layout is n_blocks block_w x block_h rectangles with
 * top-left corners xy[2i], xy[2i+1]; they must lie inside the image and must
 * not overlap (BlockLayout::validate, codec.cpp:25-54: CVG_EINVAL with the
 * reference's message otherwise).
 *
 * `mem` says where the raster and sum pointers live:
 *   CVG_MEM_HOST    host memory; the call copies in and out and returns when done;
 *   CVG_MEM_DEVICE  device memory of the context's device; the passes are
 *                   enqueued on `stream` (a cudaStream_t, 0 = legacy default)
 *                   and the call returns without waiting.
 * xy / plus_rgb / minus_rgb are always host arrays. */
#define CVG_MEM_HOST 0
#define CVG_MEM_DEVICE 1

/* embed_blocks' painting (codec.cpp:65-99, paint :58-64): frame_a = base with
 * every block filled with plus_rgb[3i..3i+2], frame_b the same with minus_rgb.
 * Pixels outside the blocks are copied unchanged.  One pass over the image. */
CVG_API int cvg_paint_blocks(cvg_ctx* ctx, const uint8_t* base, uint8_t* frame_a, uint8_t* frame_b, int32_t width,
                             int32_t height, int32_t block_w, int32_t block_h, int32_t n_blocks, const int32_t* xy,
                             const uint8_t* plus_rgb, const uint8_t* minus_rgb, int32_t mem, void* stream);

/* decode_blocks' reduction (codec.cpp:124-137): per block, exact integer sums
 * of each channel over the block's pixels in both frames.
 * sums[6i..6i+5] = (a.r, a.g, a.b, b.r, b.g, b.b).  The reference's double
 * accumulation of 8-bit values is exact below 2^53, so these sums equal its
 * sum_a / sum_b bit for bit once converted to double. */
CVG_API int cvg_block_sums(cvg_ctx* ctx, const uint8_t* frame_a, const uint8_t* frame_b, int32_t width,
                           int32_t height, int32_t block_w, int32_t block_h, int32_t n_blocks, const int32_t* xy,
                           uint64_t* sums, int32_t mem, void* stream);

/* Prepared layouts for repeated passes over one geometry (a video stream, a
 * benchmark): validation and the per-row span table are built and uploaded
 * once; each pass is then one kernel launch (plus a copy of the 6 B/block
 * colors for painting).  Same semantics as the one-shot calls above, which
 * are a prepared layout used once. */
CVG_API int cvg_layout_create(cvg_ctx* ctx, int32_t width, int32_t height, int32_t block_w, int32_t block_h,
                              int32_t n_blocks, const int32_t* xy, cvg_layout** out);
CVG_API void cvg_layout_destroy(cvg_layout* layout);
CVG_API int cvg_layout_paint(cvg_layout* layout, const uint8_t* base, uint8_t* frame_a, uint8_t* frame_b,
                             const uint8_t* plus_rgb, const uint8_t* minus_rgb, int32_t mem, void* stream);
CVG_API int cvg_layout_block_sums(cvg_layout* layout, const uint8_t* frame_a, const uint8_t* frame_b, uint64_t* sums,
                                  int32_t mem, void* stream);
/* kernel launches one cvg_layout_paint / cvg_layout_block_sums enqueues */
CVG_API int cvg_layout_launches(const cvg_layout* layout, int32_t pass);

#ifdef __cplusplus
}
#endif

#endif /* CVG_H_ */
