// ref_codec_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper over the UNMODIFIED reference codec and feasibility
// sweep (src/codec.cpp, src/feasibility.cpp, with src/search.cpp,
// src/color.cpp, src/util.cpp), compiled where those sources lie by
// oracle/Makefile into oracle/_ref/libcolorvibe_ref_codec.so.
// Nothing from the reference is copied into this repo.  image.cpp is not
// compiled (it needs libpng); the one Image member the codec calls,
// Image::solid, is restated below from its declaration (image.hpp).
// Used to pin the codec tests and oracle/codec_oracle.py to the reference.

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "colorvibe/codec.hpp"
#include "colorvibe/feasibility.hpp"
#include "colorvibe/image.hpp"

namespace colorvibe {

Image Image::solid(int width, int height, const SrgbColor& fill) {
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

}  // namespace colorvibe

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

BlockLayout layout_of(int bw, int bh, int n, const int32_t* xy, const int32_t* rgb, const int32_t* bits,
                      const char* const* names) {
    BlockLayout L;
    L.block_width = bw;
    L.block_height = bh;
    for (int i = 0; i < n; ++i) {
        L.blocks.push_back(BlockSpec{xy[2 * i], xy[2 * i + 1], names ? names[i] : "",
                                     SrgbColor{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]}, pattern_of(bits[i])});
    }
    return L;
}

Image image_of(const uint8_t* px, int w, int h) {
    Image img;
    img.width = w;
    img.height = h;
    img.pixels.assign(px, px + 3 * static_cast<size_t>(w) * h);
    return img;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

}  // namespace

extern "C" {

const char* cvrc_last_error() { return g_err.c_str(); }

// embed_blocks (codec.cpp:65-99); returns 0, 1 (invalid_argument), 2 (other)
int cvrc_embed(const uint8_t* base, int w, int h, int bw, int bh, int n, const int32_t* xy, const int32_t* rgb,
               const int32_t* bits, const char* const* names, double v_th, double r_novib, double refresh_hz,
               const double* radii, int nr, const double* angles, int na, int basis, uint8_t* fa, uint8_t* fb) {
    return guarded([&] {
        VibrationGrid g;
        g.radii.assign(radii, radii + nr);
        g.angles.assign(angles, angles + na);
        DisplayParams disp;
        disp.refresh_hz = refresh_hz;
        SearchOptions opts;
        opts.delta_basis = basis == 0 ? DeltaBasis::TargetSwing : DeltaBasis::FrameDiff;
        const FramePair fp = embed_blocks(image_of(base, w, h), layout_of(bw, bh, n, xy, rgb, bits, names),
                                          Thresholds{v_th, r_novib}, g, disp, opts);
        std::memcpy(fa, fp.frame_a.pixels.data(), fp.frame_a.pixels.size());
        std::memcpy(fb, fp.frame_b.pixels.data(), fp.frame_b.pixels.size());
    });
}

// decode_blocks (codec.cpp:113-165): status (0 Pattern, 1 NoSignal, 2 Ambiguous),
// pattern bits, mean deltas per block
int cvrc_decode(const uint8_t* fa, const uint8_t* fb, int w, int h, int wb, int hb, int bw, int bh, int n,
                const int32_t* xy, const int32_t* rgb, const int32_t* bits, double v_th, double r_novib,
                int32_t* status, int32_t* pattern, double* mean_deltas) {
    return guarded([&] {
        FramePair fp;
        fp.frame_a = image_of(fa, w, h);
        fp.frame_b = image_of(fb, wb, hb);
        fp.layout = layout_of(bw, bh, n, xy, rgb, bits, nullptr);
        const auto res = decode_blocks(fp, Thresholds{v_th, r_novib});
        for (size_t i = 0; i < res.size(); ++i) {
            status[i] = static_cast<int32_t>(res[i].status);
            pattern[i] = (res[i].pattern.r ? 4 : 0) | (res[i].pattern.g ? 2 : 0) | (res[i].pattern.b ? 1 : 0);
            for (int c = 0; c < 3; ++c) mean_deltas[3 * i + c] = res[i].mean_deltas[c];
        }
    });
}

// layout_to_json / decode_report_json text into out (returns needed length)
int cvrc_layout_json(int bw, int bh, int n, const int32_t* xy, const int32_t* rgb, const int32_t* bits,
                     const char* const* names, double v_th, double r_novib, char* out, int cap) {
    std::string s;
    if (guarded([&] { s = layout_to_json(layout_of(bw, bh, n, xy, rgb, bits, names), Thresholds{v_th, r_novib}); })) {
        return -1;
    }
    if (static_cast<int>(s.size()) < cap) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

int cvrc_report_json(int bw, int bh, int n, const int32_t* xy, const int32_t* rgb, const int32_t* bits,
                     const char* const* names, double v_th, double r_novib, const int32_t* status,
                     const int32_t* pattern, const double* mean_deltas, char* out, int cap) {
    std::string s;
    const int rc = guarded([&] {
        std::vector<BlockResult> res(n);
        for (int i = 0; i < n; ++i) {
            res[i].status = static_cast<BlockStatus>(status[i]);
            res[i].pattern = pattern_of(pattern[i]);
            for (int c = 0; c < 3; ++c) res[i].mean_deltas[c] = mean_deltas[3 * i + c];
        }
        s = decode_report_json(layout_of(bw, bh, n, xy, rgb, bits, names), Thresholds{v_th, r_novib}, res);
    });
    if (rc) return -1;
    if (static_cast<int>(s.size()) < cap) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

// ---- feasibility.cpp: config JSON round trip, hash, matrix exports ----
int copy_out(const std::string& s, char* out, int cap) {
    if (static_cast<int>(s.size()) < cap) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

// config_to_json(config_from_json(text)) (+ config_hash into hash[17])
int cvrf_config_roundtrip(const char* text, char* out, int cap, char* hash) {
    std::string s, h;
    const int rc = guarded([&] {
        const SearchConfig cfg = config_from_json(text);
        s = config_to_json(cfg);
        h = config_hash(cfg);
    });
    if (rc) return -rc;
    std::memcpy(hash, h.c_str(), h.size() + 1);
    return copy_out(s, out, cap);
}

// export_matrix(feasibility_matrix(config_from_json(text)), format, aggregated)
int cvrf_export(const char* text, int json_format, int aggregated, char* out, int cap) {
    std::string s;
    const int rc = guarded([&] {
        const FeasibilityMatrix m = feasibility_matrix(config_from_json(text));
        s = export_matrix(m, json_format ? ExportFormat::Json : ExportFormat::Csv, aggregated != 0);
    });
    if (rc) return -rc;
    return copy_out(s, out, cap);
}

}  // extern "C"
