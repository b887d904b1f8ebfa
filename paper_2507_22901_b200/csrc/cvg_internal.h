// cvg_internal.h -- launch entry points of cvg_kernels.cu used by the host library.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "cvg_layout.h"

namespace cvg {

// Enqueues the fused search kernel (mode: kModeBand/kModeCodes, out: kOut*,
// path: kPath*) with `grid` persistent blocks on `st`.
// `marks` (optional, 2 events) are recorded after phase 1 and after the scan.
cudaError_t launch_search(const LaunchArgs& a, int mode, int out, int path, int grid, cudaStream_t st,
                          cudaEvent_t* marks = nullptr);
// Resident blocks per SM for that instantiation; also opts the kernel into its
// dynamic shared memory size on the current device (call before launching).
int search_blocks_per_sm(int mode, int out, int path);
cudaError_t launch_first_codes(const LaunchArgs& a, cudaStream_t st);
size_t search_smem_bytes();
double measure_ffma_peak(int device, float* ms_out);

}  // namespace cvg
