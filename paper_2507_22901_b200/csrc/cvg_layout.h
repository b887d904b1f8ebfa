// cvg_layout.h -- HBM data layout shared by the host library (g++) and the
// CUDA kernels (nvcc).  Plain structs only.
#pragma once

#include <cstdint>

namespace cvg {

// Candidates per warp tile: the unit of the ordered (decoupled look-back)
// compaction.  A tile is a contiguous range of one search's canonical
// (radius-major, angle-minor) candidate index.
constexpr int kTile = 4096;
constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr int kGuessBuckets = 4096;  // code-table buckets over linear [0, 1]
constexpr float kCodeSlack = 1.0f / 65536;  // code-table bucket widening (>= every usable eps_code)
constexpr int kEmitSpan = 256;      // pairs per emit work item (tile sub-range)
constexpr int kScanItems = 8;        // tile counts per thread in the offset scan
constexpr int kScanTile = kBlock * kScanItems;
// Twin tiles: |lin64(k, m) - lin64 of the swapped twin endpoint| <= 2^-33 is
// proven on the host (plan_build); the emit widens its code-verification
// bound by this much for the twin's records.
constexpr float kTwinSlack = 1.0f / 4294967296.0f;  // 2^-32

// Per-search constants, one 288-byte record per (target, pattern, thresholds).
// The FP32 half feeds the fast path; the FP64 half is the bit-exact restatement
// of the reference hoisting (search.cpp:341-370) used by the repair path.
struct alignas(16) SearchConst {
    // --- FP32 fast path -------------------------------------------------
    float fx0;         // Fy + a/500   (fx of both endpoints = fx0 +- r*sin/500)
    float fz0;         // Fz = Fy - b/200 (fz = fz0 -+ r*cos/200)
    float rcube;       // rows with r < rcube never leave the cube branch of f^-1
    float la;          // band attention: min over loud M' >= la (= 1 - eps_l, rounded down)
    float mx[3];       // Minv[c][0] * wx
    float mz[3];       // Minv[c][2] * wz
    float cy[3];       // Minv[c][1] * wy * f^-1(Fy)
    float mxs[3];      // band form, channels permuted loud-first: mx / h_c   (h_c: band half-width)
    float mzs[3];      //            mz / h_c
    float cys[3];      //            (cy - centre_c) / h_c
    union {
        float cube[6];       // cube-only rows, sum/difference form: {fx0^3, 3 fx0^2, 3 fx0, fz0^3, 3 fz0^2, 3 fz0}
        float fd_bounds[6];  // Quantized x FrameDiff: per channel {lo, hi}; the channel surely fails if the
                             // saturated FP32 |v_p - v_m| <= lo or >= hi (make_search_const)
    };
    float qa, qp, lp;  // attention: max quiet M' <= qa; certain pass: max quiet M' < qp and min loud M' > lp
    float eps[3];      // proven bound |lin32 - lin64| per channel (linear units)
    float eps_code[3]; // eps + float rounding of the code thresholds
    uint32_t flags;    // bit c (c=0,1,2 -> r,g,b): loud channel; bit 8 FrameDiff; bit 9 continuous; bits 10-11: loud count
    int32_t t[3];      // target codes
    int32_t k1;        // d > v_th   <=> d >= k1 (integer deltas); 256 = never
    int32_t q0;        // d <= low   <=> d <= q0
    // --- FP64 exact path (bit-identical to the reference) ----------------
    double fy, ta, tb, wx, wz;
    double cy64[3];
    double lo[3], hi[3];  // band edges (kModeBand); lo[c] = the channel's threshold, v_th or low (kModeSignal)
};
static_assert(sizeof(SearchConst) == 288, "SearchConst layout");

// Device statistics block.
struct Stats {
    unsigned long long band_repairs;
    unsigned long long code_repairs;
    unsigned long long audit_violations;
    unsigned long long class_mismatch;
    unsigned long long overflow;
    unsigned long long undecided;  // kModeSignal: decisions inside the device/glibc pow margin (call fails)
    unsigned int audit_max_ratio_bits;  // float bits, atomicMax on non-negative floats
    unsigned int pad;
};

// kModeBand: TargetSwing (quantized or continuous), interval test per endpoint;
// kModeCodes: Quantized x FrameDiff, classify on the codes of both endpoints;
// kModeSignal: Continuous x FrameDiff, classify on |s(p) - s(m)| of the
// pre-rounding signal values (FP64 on the device, glibc-pow error margin).
enum Mode : int { kModeBand = 0, kModeCodes = 1, kModeSignal = 2 };
constexpr int kModes = 3;
enum Out : int { kOutPairs = 0, kOutCounts = 1, kOutFirst = 2 };
enum Path : int { kPathFast = 0, kPathExact = 1, kPathAudit = 2 };

// Everything one launch needs (passed by value as the kernel parameter).
struct LaunchArgs {
    const SearchConst* sc;     // [n_unique] per-search constant records
    const uint32_t* sc_index;  // [n_searches] record of each search, nullptr = identity
    // Claim order (band mode, mixed patterns): claim_order[p] is the search at
    // position p; positions [group_end[g-1], group_end[g]) hold the searches
    // of one loud count, claimed group after group so that concurrently
    // resident warps run one hot-loop specialization.  nullptr = identity.
    const uint32_t* claim_order;
    uint32_t group_end[3];
    const float* radii_f;      // [nr]
    const double* radii_d;     // [nr]
    const float* trig_f;       // [na][2] = (sin/500, cos/200) as float
    const double* trig_d;      // [na][2] = (sin, cos), glibc doubles (search.cpp:414-419)
    const double* thr_d;       // [256] QuantTable thresholds (convert_kernel.hpp:123-141)
    const float* ctab;         // [kGuessBuckets + 1][2] code table {t, bits(c)} (cvg_host.h Tables)
    const float* stab;         // [kGuessBuckets + 1][2] signal bounds {L, U} (kModeSignal plans only)
    double minv[9];            // kXyzToRgb (convert_kernel.hpp:47), row-major
    int32_t n_searches;
    int32_t nr;
    int32_t na;
    int32_t aligned;           // na % 32 == 0: a 32-candidate chunk never straddles rows
    uint32_t tiles_per_search;
    uint32_t cand_per_search;  // nr * na (< 2^32)
    uint64_t na_magic;         // ceil(2^64 / na): k = umul64hi(i, na_magic)
    uint64_t n_tiles;              // tiles of this range view
    // Work units the phase-1 warps claim: tiles, or strip tiles.
    uint32_t n_claims;             // units of this range view
    uint32_t claim_per_search;
    // PAIRS on strip tiles: pass words, column-major per search:
    // masks[(s * n_strips + q) * mask_rows + k] (bit l = angle 32 q + l);
    // lists_kernel builds the canonical tile lists from them
    uint32_t* masks;
    uint32_t mask_rows;            // n_radii rounded up to 32
    uint32_t lst_rpt;              // tiles of whole rows: rows per tile (0 otherwise)
    uint32_t lst_tpr;              // rows of whole tiles: tiles per row (0 otherwise)
    uint32_t lst_unit_rows;        // rows per lists_kernel unit: max(8, lst_rpt)
    // Range view: the launch covers searches [search_begin, search_begin +
    // range_searches) = tiles [tile_begin, tile_begin + n_tiles).  A plan may
    // run two views on two streams so that one range's scan and emit fill
    // the other range's phase-1 tail; tile indices stay global.
    uint32_t search_begin;
    uint32_t range_searches;
    uint64_t tile_begin;
    const unsigned long long* base_offset;  // emit: pair positions start at *base_offset (nullptr = 0)
    unsigned long long* grand_total;        // emit of the last view: *grand_total = *base_offset + *total
    unsigned long long* status;    // [n_scan_blocks] chained-scan status words (flag << 62 | value)
    unsigned int* ticket;          // [4]: phase-1 tiles, scan blocks, emit worklist, worklist size
    unsigned long long* counts;    // [n_searches]
    uint32_t* tile_count;          // [n_tiles] passing candidates per tile (PAIRS)
    unsigned long long* tile_base; // [n_tiles] exclusive prefix of tile_count (PAIRS)
    uint16_t* scratch;             // [n_tiles * kTile] per-tile passing offsets (PAIRS)
    uint32_t* worklist;            // [n_tiles * kTile / kEmitSpan] emit items tile << 4 | sub, any order
    uint32_t emit_shift;           // log2 of the pairs per emit item: 8 (kEmitSpan), 9 for dense batches
    uint32_t prune;                // CVG_PATH_PRUNED: skip radius rows that row_surely_fails proves empty
    // Strip tiles (COUNTS / FIRST, band FAST path): a strip is 32 angles x
    // strip_rows radius rows (lane l owns angle 32 q + l, the warp walks the
    // rows).  Tile lt of a search = row block kb = lt / strip_tiles, strips
    // [(lt % strip_tiles) * strips_per_tile, +strips_per_tile).  0 = row-major tiles.
    uint32_t strips;
    uint32_t strip_rows;           // rows per row block (multiple of 4, or nr)
    uint32_t strips_per_tile;
    uint32_t strip_tiles;          // tiles per row block
    const float* strip_inv;        // [n_strips][2]: 1 / the strip's largest |sin/500|, |cos/200| (rounded down)
    // COUNTS / FIRST strips: lane slot j walks angle strip_perm[j] (angles by
    // decreasing |cos|; 0xFFFFFFFF past the last), its trig in strip_trig[j]
    // (nullptr: identity, PAIRS)
    const uint32_t* strip_perm;
    const float* strip_trig;
    uint32_t bulk_skip;            // strip tiles: bisect the inner rows no lane can pass (strip_run)
    const float* radius_groups;    // [ceil(nr/4)][3][4]: per 4 rows float(r), float(r^2), float(r^3)
                                   // of the double radii (strip form; padded with the last radius)
    // Twin tiles (PAIRS on rows of whole tiles, grid symmetric under
    // theta -> theta + pi; plan_build proves it): candidate (k, m + na/2) is
    // candidate (k, m) with the endpoints swapped.  lists_kernel compares the
    // pass words of tile t (first half of a row) and its twin t + twin_tiles
    // word for word; twin[t] = 1 when they are identical, and the emit then
    // quantizes each pair of t once and writes both records (codes swapped).
    // nullptr = off.
    uint8_t* twin;                 // [n_tiles]
    uint32_t twin_tiles;           // lst_tpr / 2
    uint32_t twin_m;               // na / 2
    uint32_t twin_split_test;      // test hook: treat odd rows as differing (both lists built)
    unsigned long long* total;     // [1] sum of tile_count (PAIRS)
    uint32_t* out_idx;           // [capacity]
    uint8_t* out_codes;          // [capacity * 6]
    uint64_t capacity;
    // BEST: per tile of the view, the largest margin bits of its pairs and
    // the first position reaching it (best_tiles_kernel)
    unsigned long long* best_key;  // [2 * n_tiles]
    uint32_t* first_idx;         // [n_searches] (FIRST)
    uint8_t* first_codes;        // [n_searches * 6] (FIRST)
    Stats* stats;
};

}  // namespace cvg
