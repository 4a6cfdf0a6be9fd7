// fused.cuh -- the fused engine (conv_fused) entry points.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace wf {

size_t fused_scratch_bytes(const Geo& g, int r);
// Persistent dataflow kernel (fused_persistent.cu), used when C'pad <= 128.
bool persistent_fits(const Geo& g);
size_t persistent_scratch_bytes(const Geo& g);
cudaError_t run_fused_persistent(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                                 int passes, int sm_count, cudaStream_t st);
// Warp-specialised persistent kernel (fused_ws.cu): F(4x4,3x3), C = C' = 64.
bool ws_fits(const Geo& g);
size_t ws_scratch_bytes(const Geo& g);
// counters_clean: the scratch's counters are known to be zero (the kernel
// leaves them zero when it finishes), so the memset is skipped
cudaError_t run_fused_ws(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g, int passes,
                         int sm_count, cudaStream_t st, bool counters_clean = false);
cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                      int passes, int r, int sm_count, cudaStream_t st, bool counters_clean = false);

}  // namespace wf
