// cvg_internal.h -- launch entry points of cvg_kernels.cu used by the host library.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "cvg_layout.h"

namespace cvg {

// Enqueues the fused search kernel (mode: kModeBand/kModeCodes, out: kOut*,
// path: kPath*) with `grid` persistent blocks on `st`.
// `marks` (optional, 2 events) are recorded after phase 1 and after the scan.
cudaError_t launch_search(const LaunchArgs& a, int mode, int out, int path, int grid, cudaStream_t st,
                          cudaEvent_t* marks = nullptr);
// The three PAIRS-mode kernels separately (range views on two streams).
cudaError_t launch_phase1(const LaunchArgs& a, int mode, int out, int path, int grid, cudaStream_t st);
cudaError_t launch_scan(const LaunchArgs& a, cudaStream_t st);
// threads: any multiple of 32 up to kBlock (streamed searches run 128-thread emits beside phase 1)
cudaError_t launch_emit(const LaunchArgs& a, int mode, int path, int grid, cudaStream_t st, int threads = kBlock);
// Resident blocks per SM for that instantiation; also opts the kernel into its
// dynamic shared memory size on the current device (call before launching).
int search_blocks_per_sm(int mode, int out, int path);
cudaError_t launch_first_codes(const LaunchArgs& a, cudaStream_t st);
// CVG_OUT_BEST epilogue after the PAIRS kernels: per search, the pair of
// largest classification_margin (first in canonical order on ties) from the
// device pair buffer into a.first_idx / a.first_codes.  bands = (v_th, low) per search.
cudaError_t launch_best(const LaunchArgs& a, const double* bands, cudaStream_t st);
// CVG_PATH_MEMO: out[s] = in[map[s]] for counts (and first pairs when fi_in is set), s < n.
cudaError_t launch_scatter(const uint32_t* map, int n, const unsigned long long* counts_in, const uint32_t* fi_in,
                           const uint8_t* fc_in, unsigned long long* counts, uint32_t* fi, uint8_t* fc, cudaStream_t st);
size_t search_smem_bytes();

// Codec passes (cvg_codec.cu).  Block positions xy[2i], xy[2i+1]; colors
// packed r | g << 8 | b << 16.  Paint = copy pass + block fill pass.
cudaError_t launch_paint(const uint8_t* base, uint8_t* fa, uint8_t* fb, int width, int height, int block_w,
                         int block_h, int n_blocks, const int32_t* xy, const uint32_t* plus, const uint32_t* minus,
                         int sms, cudaStream_t st);
cudaError_t launch_block_sums(const uint8_t* fa, const uint8_t* fb, int width, int height, int block_w, int block_h,
                              int n_blocks, const int32_t* xy, unsigned long long* sums, int sms, cudaStream_t st);
double measure_ffma_peak(int device, float* ms_out);

}  // namespace cvg
