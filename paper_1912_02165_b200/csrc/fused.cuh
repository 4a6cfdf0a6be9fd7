// fused.cuh -- the fused engine (conv_fused) entry points.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace wf {

size_t fused_scratch_bytes(const Geo& g, int r);
cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                      int passes, int r, int sm_count, cudaStream_t st);

}  // namespace wf
