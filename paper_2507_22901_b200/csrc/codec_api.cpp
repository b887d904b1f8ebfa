// codec_api.cpp -- the reference codec API (include/colorvibe/codec.hpp,
// image.hpp) over the C-ABI.  Reference: src/codec.cpp, src/image.cpp:11-27.
//
// embed_blocks: every block's search in one device launch (the reference
// runs one batch_search per block, codec.cpp:80-81), select_best on the
// packed records, then one device pass paints both frames (cvg_paint_blocks).
// decode_blocks: one device pass of exact integer block sums
// (cvg_block_sums), then the reference's double arithmetic on the host.
// The sidecar JSON functions reproduce the reference's nlohmann
// ordered_json dump(2) text (codec.cpp:167-258).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "../../include/cvg.h"
#include "colorvibe/codec.hpp"
#include "colorvibe_detail.h"
#include "json_lite.h"

namespace colorvibe {

using namespace detail;
using namespace json;

namespace {

std::string fmt_g6(double v) {  // util.cpp:12-16
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.6g", v);
    return buf;
}

bool overlaps(const BlockSpec& b, const BlockSpec& c, int w, int h) {
    return b.x < c.x + w && c.x < b.x + w && b.y < c.y + h && c.y < b.y + h;
}

}  // namespace

// ---- image.hpp ---------------------------------------------------------------

Image Image::solid(int width, int height, const SrgbColor& fill) {  // image.cpp:11-27
    if (width <= 0 || height <= 0) throw std::invalid_argument("image dimensions must be positive");
    validate(fill);
    Image img;
    img.width = width;
    img.height = height;
    img.pixels.resize(3 * static_cast<std::size_t>(width) * height);
    for (std::size_t i = 0; i < img.pixels.size(); i += 3) {
        img.pixels[i] = static_cast<std::uint8_t>(fill.r);
        img.pixels[i + 1] = static_cast<std::uint8_t>(fill.g);
        img.pixels[i + 2] = static_cast<std::uint8_t>(fill.b);
    }
    return img;
}

// ---- codec.hpp ---------------------------------------------------------------

void DisplayParams::validate() const {  // codec.cpp:14-23
    if (!(std::isfinite(refresh_hz) && refresh_hz > 0.0)) {
        throw std::invalid_argument("display: refresh_hz must be positive");
    }
    if (!(refresh_hz / 2.0 > ccff_hz)) {
        throw std::invalid_argument("display: refresh_hz / 2 must exceed the color fusion frequency (" +
                                    fmt_g6(ccff_hz) + " Hz); got " + fmt_g6(refresh_hz) + " Hz");
    }
}

void BlockLayout::validate(int image_width, int image_height) const {  // codec.cpp:25-54
    if (block_width <= 0 || block_height <= 0) throw std::invalid_argument("layout: block size must be positive");
    // Fast screen: every color valid, every block in bounds and no two
    // overlapping (sorted sweep over rows of equal-size blocks).  Only a
    // failing layout runs the reference's ordered checks, which name the
    // first offending block or pair exactly as the reference does.
    bool ok = true;
    for (const auto& b : blocks) {
        ok = ok && is_valid(b.color) && b.x >= 0 && b.y >= 0 &&
             static_cast<long long>(b.x) + block_width <= image_width &&
             static_cast<long long>(b.y) + block_height <= image_height;
    }
    if (ok && blocks.size() > 1) {
        std::vector<int> order(blocks.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            return blocks[a].y != blocks[b].y ? blocks[a].y < blocks[b].y : blocks[a].x < blocks[b].x;
        });
        // any overlapping pair has |dy| < h; scan forward while rows can still meet
        for (size_t i = 0; i < order.size() && ok; ++i) {
            const BlockSpec& b = blocks[order[i]];
            for (size_t j = i + 1; j < order.size(); ++j) {
                const BlockSpec& c = blocks[order[j]];
                if (c.y >= b.y + block_height) break;
                if (overlaps(b, c, block_width, block_height)) {
                    ok = false;
                    break;
                }
            }
        }
    }
    if (ok) return;
    for (std::size_t i = 0; i < blocks.size(); ++i) {
        const auto& b = blocks[i];
        colorvibe::validate(b.color);
        if (b.x < 0 || b.y < 0 || b.x + block_width > image_width || b.y + block_height > image_height) {
            throw std::invalid_argument("layout: block " + std::to_string(i) + " (" + b.color_name +
                                        ") exceeds image bounds");
        }
        for (std::size_t j = i + 1; j < blocks.size(); ++j) {
            if (overlaps(b, blocks[j], block_width, block_height)) {
                throw std::invalid_argument("layout: blocks " + std::to_string(i) + " and " + std::to_string(j) +
                                            " overlap");
            }
        }
    }
}

namespace {

// classification_margin (search.cpp:458-466) of pair p of search s, deltas
// recomputed from the packed codes as materialize() does.
double margin_of(const cvg_result& r, uint64_t p, const SrgbColor& t, const Thresholds& th,
                 const SearchOptions& opts) {
    const uint8_t* c = r.codes + 6 * p;
    const int tc[3] = {t.r, t.g, t.b};
    const bool swing = opts.delta_basis == DeltaBasis::TargetSwing;
    const double low = th.low_band();
    double m = INFINITY;
    for (int q = 0; q < 3; ++q) {
        const int pv = c[q], mv = c[3 + q];
        const double d = swing ? static_cast<double>(std::max(std::abs(pv - tc[q]), std::abs(mv - tc[q])))
                               : static_cast<double>(std::abs(pv - mv));
        m = std::min(m, d > th.v_th ? d - th.v_th : low - d);
    }
    return m;
}

void copy_image(const Image& from, Image& to) {
    to.width = from.width;
    to.height = from.height;
    to.pixels = from.pixels;
}

}  // namespace

FramePair embed_blocks(const Image& base, const BlockLayout& layout, const Thresholds& th, const VibrationGrid& grid,
                       const DisplayParams& disp, const SearchOptions& opts) {
    disp.validate();  // codec.cpp:68-71
    th.validate();
    grid.validate();
    layout.validate(base.width, base.height);
    if (base.pixels.size() != 3 * static_cast<std::size_t>(base.width) * base.height) {
        throw std::invalid_argument("image pixel buffer does not match its dimensions");
    }

    FramePair fp;
    fp.layout = layout;
    const size_t n = layout.blocks.size();
    if (n == 0) {
        copy_image(base, fp.frame_a);
        copy_image(base, fp.frame_b);
        return fp;
    }
    // The reference searches block by block and throws at the first block
    // that is infeasible (runtime_error) or whose search rejects its inputs.
    // Colors, grid and thresholds are validated above, so only a "000"
    // pattern can fail a search: search the blocks before the first such
    // block in one launch, report an infeasible one first, then the pattern.
    size_t first_bad = n;
    for (size_t i = 0; i < n; ++i) {
        if (!layout.blocks[i].pattern.any()) {
            first_bad = i;
            break;
        }
    }
    std::vector<SearchSpec> specs;
    specs.reserve(first_bad);
    for (size_t i = 0; i < first_bad; ++i) specs.push_back({layout.blocks[i].color, layout.blocks[i].pattern, th});
    std::vector<uint8_t> plus(3 * n), minus(3 * n);
    std::vector<int32_t> xy(2 * n);
    const bool empty_grid = grid.radii.empty() || grid.angles.empty();
    ResultGuard g;
    if (!specs.empty() && !empty_grid) run(specs, grid, opts, CVG_OUT_PAIRS, CVG_PATH_PRUNED, g);
    for (size_t i = 0; i < first_bad; ++i) {
        const BlockSpec& b = layout.blocks[i];
        const uint64_t lo = empty_grid ? 0 : g.r.offsets[i], hi = empty_grid ? 0 : g.r.offsets[i + 1];
        if (lo == hi) {
            throw std::runtime_error("embed: block " + std::to_string(i) + " (" + b.color_name + ", pattern " +
                                     b.pattern.str() + "): no pair satisfies the thresholds on this grid");
        }
        // select_best (search.cpp:468-489): the first maximum margin in
        // canonical (radius, angle) order
        uint64_t best = lo;
        if (opts.delta_mode == DeltaMode::Continuous) {
            const std::vector<ColorPair> pairs = materialize(g.r, i, b.color, grid, opts);
            best = lo + static_cast<uint64_t>(&select_best(pairs, th) - pairs.data());
        } else {
            double best_m = margin_of(g.r, lo, b.color, th, opts);
            for (uint64_t p = lo + 1; p < hi; ++p) {
                const double m = margin_of(g.r, p, b.color, th, opts);
                if (m > best_m) {
                    best_m = m;
                    best = p;
                }
            }
        }
        std::memcpy(&plus[3 * i], g.r.codes + 6 * best, 3);
        std::memcpy(&minus[3 * i], g.r.codes + 6 * best + 3, 3);
        xy[2 * i] = b.x;
        xy[2 * i + 1] = b.y;
    }
    if (first_bad < n) throw std::invalid_argument("bit pattern has no set bits");  // search.cpp:26-28

    fp.frame_a.width = fp.frame_b.width = base.width;
    fp.frame_a.height = fp.frame_b.height = base.height;
    fp.frame_a.pixels.resize(base.pixels.size());
    fp.frame_b.pixels.resize(base.pixels.size());
    check(cvg_paint_blocks(default_ctx(), base.pixels.data(), fp.frame_a.pixels.data(), fp.frame_b.pixels.data(),
                           base.width, base.height, layout.block_width, layout.block_height,
                           static_cast<int32_t>(n), xy.data(), plus.data(), minus.data(), CVG_MEM_HOST, nullptr));
    return fp;
}

FramePair make_testcard(const SrgbColor& color, const BitPattern& pattern, const Thresholds& th,
                        const VibrationGrid& grid, const DisplayParams& disp, int width, int height,
                        const SearchOptions& opts) {  // codec.cpp:101-111
    BlockLayout layout;
    layout.block_width = width;
    layout.block_height = height;
    layout.blocks.push_back(BlockSpec{0, 0, "target", color, pattern});
    return embed_blocks(Image::solid(width, height, color), layout, th, grid, disp, opts);
}

std::vector<BlockResult> decode_blocks(const FramePair& fp, const Thresholds& th) {  // codec.cpp:113-165
    th.validate();
    if (fp.frame_a.width != fp.frame_b.width || fp.frame_a.height != fp.frame_b.height) {
        throw std::invalid_argument("decode: frame dimensions differ");
    }
    fp.layout.validate(fp.frame_a.width, fp.frame_a.height);
    const size_t expect = 3 * static_cast<std::size_t>(fp.frame_a.width) * fp.frame_a.height;
    if (fp.frame_a.pixels.size() != expect || fp.frame_b.pixels.size() != expect) {
        throw std::invalid_argument("image pixel buffer does not match its dimensions");
    }
    const size_t n_blocks = fp.layout.blocks.size();
    std::vector<BlockResult> results;
    results.reserve(n_blocks);
    if (n_blocks == 0) return results;
    std::vector<int32_t> xy(2 * n_blocks);
    for (size_t i = 0; i < n_blocks; ++i) {
        xy[2 * i] = fp.layout.blocks[i].x;
        xy[2 * i + 1] = fp.layout.blocks[i].y;
    }
    std::vector<uint64_t> sums(6 * n_blocks);
    check(cvg_block_sums(default_ctx(), fp.frame_a.pixels.data(), fp.frame_b.pixels.data(), fp.frame_a.width,
                         fp.frame_a.height, fp.layout.block_width, fp.layout.block_height,
                         static_cast<int32_t>(n_blocks), xy.data(), sums.data(), CVG_MEM_HOST, nullptr));
    const double low = th.low_band();
    const double n = static_cast<double>(fp.layout.block_width) * fp.layout.block_height;
    for (size_t i = 0; i < n_blocks; ++i) {
        const auto& block = fp.layout.blocks[i];
        const int tgt[3] = {block.color.r, block.color.g, block.color.b};
        BlockResult res;
        bool ambiguous = false, any_high = false;
        bool bits[3] = {false, false, false};
        for (int c = 0; c < 3; ++c) {
            // integer sums are exact; as doubles they equal the reference's
            // running double sums of 8-bit values (exact below 2^53)
            const double sa = static_cast<double>(sums[6 * i + c]);
            const double sb = static_cast<double>(sums[6 * i + 3 + c]);
            const double dev = std::max(std::abs(sa / n - tgt[c]), std::abs(sb / n - tgt[c]));
            res.mean_deltas[c] = dev;
            if (dev > th.v_th) {
                bits[c] = true;
                any_high = true;
            } else if (!(dev <= low)) {
                ambiguous = true;  // inside (v_th * r_novib, v_th]
            }
        }
        if (ambiguous) {
            res.status = BlockStatus::Ambiguous;
        } else if (!any_high) {
            res.status = BlockStatus::NoSignal;
        } else {
            res.status = BlockStatus::Pattern;
            res.pattern = BitPattern{bits[0], bits[1], bits[2]};
        }
        results.push_back(res);
    }
    return results;
}

// ---- sidecar JSON (codec.cpp:167-258), text of nlohmann ordered_json dump(2) ------------

std::string layout_to_json(const BlockLayout& layout, const Thresholds& th) {  // codec.cpp:167-186
    Json j = Json::object();
    j.add("version", Json::integer(1));
    j.add("block_width", Json::integer(layout.block_width));
    j.add("block_height", Json::integer(layout.block_height));
    j.add("v_th", Json::number(th.v_th));
    j.add("r_novib", Json::number(th.r_novib));
    Json blocks = Json::array();
    for (const auto& b : layout.blocks) {
        Json rgb = Json::array();
        rgb.push(Json::integer(b.color.r)).push(Json::integer(b.color.g)).push(Json::integer(b.color.b));
        Json e = Json::object();
        e.add("x", Json::integer(b.x));
        e.add("y", Json::integer(b.y));
        e.add("color_name", Json::string(b.color_name));
        e.add("rgb", rgb);
        e.add("pattern", Json::string(b.pattern.str()));
        blocks.push(e);
    }
    j.add("blocks", blocks);
    std::string out;
    dump(j, out, 0);
    return out + "\n";
}

Sidecar layout_from_json(const std::string& text) {  // codec.cpp:188-222
    Json j;
    try {
        j = Parser{text}.parse();
    } catch (const JsonError& e) {
        throw std::invalid_argument(std::string("sidecar: invalid JSON: ") + e.what());
    }
    Sidecar sc;
    try {
        // j.value("version", 0)
        int version = 0;
        if (j.kind != Json::Object) type_error(306, std::string("cannot use value() with ") + j.type_name());
        if (const Json* v = find(j, "version")) version = get_int(*v);
        if (version != 1) throw std::invalid_argument("sidecar: missing or unsupported version");
        sc.layout.block_width = get_int(at(j, "block_width"));
        sc.layout.block_height = get_int(at(j, "block_height"));
        sc.thresholds.v_th = get_double(at(j, "v_th"));
        sc.thresholds.r_novib = get_double(at(j, "r_novib"));
        // range-for over a json value: array elements, object values, one
        // element for a primitive, none for null (nlohmann iteration rules)
        const Json& blocks = at(j, "blocks");
        std::vector<const Json*> items;
        if (blocks.kind == Json::Array) {
            for (const Json& b : *blocks.arr) items.push_back(&b);
        } else if (blocks.kind == Json::Object) {
            for (const auto& kv : *blocks.obj) items.push_back(&kv.second);
        } else if (blocks.kind != Json::Null) {
            items.push_back(&blocks);
        }
        for (const Json* bp : items) {
            const Json& b = *bp;
            const Json& rgbj = at(b, "rgb");
            if (rgbj.kind != Json::Array) type_error(302, std::string("type must be array, but is ") + rgbj.type_name());
            std::vector<int> rgb;
            for (const Json& c : *rgbj.arr) rgb.push_back(get_int(c));
            if (rgb.size() != 3) throw std::invalid_argument("sidecar: rgb must have 3 entries");
            // BlockSpec{x, y, color_name, rgb, pattern}: left-to-right evaluation
            const int x = get_int(at(b, "x"));
            const int y = get_int(at(b, "y"));
            std::string name;
            if (const Json* v = find(b, "color_name")) name = get_string(*v);
            const BitPattern pat = BitPattern::parse(get_string(at(b, "pattern")));
            sc.layout.blocks.push_back(BlockSpec{x, y, name, SrgbColor{rgb[0], rgb[1], rgb[2]}, pat});
        }
    } catch (const JsonError& e) {
        throw std::invalid_argument(std::string("sidecar: ") + e.what());
    }
    sc.thresholds.validate();
    return sc;
}

std::string decode_report_json(const BlockLayout& layout, const Thresholds& th,
                               const std::vector<BlockResult>& results) {  // codec.cpp:224-258
    if (layout.blocks.size() != results.size()) throw std::invalid_argument("decode report: result count mismatch");
    Json j = Json::object();
    j.add("version", Json::integer(1));
    j.add("v_th", Json::number(th.v_th));
    j.add("r_novib", Json::number(th.r_novib));
    Json blocks = Json::array();
    for (size_t i = 0; i < results.size(); ++i) {
        const auto& b = layout.blocks[i];
        const auto& r = results[i];
        Json e = Json::object();
        e.add("index", Json::integer(static_cast<long long>(i)));
        e.add("x", Json::integer(b.x));
        e.add("y", Json::integer(b.y));
        e.add("color_name", Json::string(b.color_name));
        e.add("embedded_pattern", Json::string(b.pattern.str()));
        switch (r.status) {
            case BlockStatus::Pattern:
                e.add("result", Json::string("pattern"));
                e.add("pattern", Json::string(r.pattern.str()));
                break;
            case BlockStatus::NoSignal: e.add("result", Json::string("no_signal")); break;
            case BlockStatus::Ambiguous: e.add("result", Json::string("ambiguous")); break;
        }
        Json md = Json::array();
        md.push(Json::number(r.mean_deltas[0])).push(Json::number(r.mean_deltas[1])).push(Json::number(r.mean_deltas[2]));
        e.add("mean_deltas", md);
        blocks.push(e);
    }
    j.add("blocks", blocks);
    std::string out;
    dump(j, out, 0);
    return out + "\n";
}

}  // namespace colorvibe
