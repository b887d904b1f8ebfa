// colorvibe_detail.h -- helpers shared by the C++ API translation units
// (colorvibe_api.cpp: search/color API, codec_api.cpp: codec API).
#pragma once

#include <string>
#include <vector>

#include "../../include/cvg.h"
#include "colorvibe/search.hpp"

namespace colorvibe::detail {

[[noreturn]] void throw_status(int status);
void check(int status);  // CVG_EINVAL -> std::invalid_argument, else std::runtime_error
// Process-wide context on the device named by CVG_DEVICE (default: 0).
cvg_ctx* default_ctx();
int pattern_bits(const BitPattern& p);

struct ResultGuard {
    cvg_result r{};
    ~ResultGuard() { cvg_result_free(&r); }
};

// One device call for a batch of searches sharing the grid and options.
void run(const std::vector<SearchSpec>& specs, const VibrationGrid& grid, const SearchOptions& opts, int output,
         int path, ResultGuard& g);
// The ColorPair list of search s of a PAIRS result (deltas as the options say).
std::vector<ColorPair> materialize(const cvg_result& r, size_t s, const SrgbColor& target, const VibrationGrid& grid,
                                   const SearchOptions& opts);

}  // namespace colorvibe::detail
