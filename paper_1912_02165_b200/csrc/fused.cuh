// fused.cuh -- the fused engine (conv_fused) entry points.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace wf {

// Fused-engine variants (include/winofuse_b200.h WF_FUSED_*).
constexpr int kVarAuto = 0, kVarWS = 1, kVarItemQueue = 2, kVarWaves = 3, kVarWSRow = 4;
constexpr int kFusedCountersClean = 1, kFusedInstrument = 2;

// Per-call options of the fused engine (the C ABI's wf_fused_opts).  Every
// field has a measured default (0 = default); none changes the results.
struct FusedOpts {
  int variant = kVarAuto;   // which kernel runs (auto: the fastest that can hold the layer)
  int flags = 0;            // kFusedCountersClean | kFusedInstrument
  size_t ring_bytes = 0;    // L2 ring budget of the persistent kernels
  int lag = 0;              // steps between a block's producer and consumer units
  int gbatch = 0;           // G completions per publish (warp-specialised kernel)
};

// Tuning knobs read from the environment ONCE per process (capi.cu);
// developer aids with measured defaults -- the variant is never chosen by them.
int tuning_knob(const char* name, int dflt);

// The variant that runs for (g, o): o.variant if that kernel can hold the
// layer (else 0), or the automatic choice.
int fused_pick_variant(const Geo& g, const FusedOpts& o);
// Scratch for the picked variant and for the L2-wave fallback it takes when
// its CTAs cannot all be resident (the larger of the two).
size_t fused_scratch_bytes(const Geo& g, const FusedOpts& o);
// *ran = the variant that ran.
cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g, int passes,
                      int sm_count, cudaStream_t st, const FusedOpts& o, int* ran);

// Persistent item-queue dataflow kernel (fused_persistent.cu), C'pad <= 256.
bool persistent_fits(const Geo& g, const FusedOpts& o, bool automatic);
size_t persistent_scratch_bytes(const Geo& g, const FusedOpts& o);
cudaError_t run_fused_persistent(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                                 int passes, int sm_count, cudaStream_t st, const FusedOpts& o);
// Warp-specialised persistent kernel (fused_ws.cu).
bool ws_fits(const Geo& g, const FusedOpts& o);
size_t ws_scratch_bytes(const Geo& g, const FusedOpts& o);
cudaError_t run_fused_ws(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g, int passes,
                         int sm_count, cudaStream_t st, const FusedOpts& o);
cudaError_t ws_instrument_reset(int n_blk, cudaStream_t st);
// Copies the per-block ordering tickets (8 per block) and the summed per-role
// busy cycles (F units, G epilogue, I units) of the last instrumented launch;
// nu_nm = the ring slots of the plan.  Returns the number of blocks, -1 on error.
int ws_instrument_read(const Geo& g, const FusedOpts& o, unsigned long long* events, int n_events,
                       unsigned long long* role_cycles, int* nu_nm);
// L2-wave path (fused.cu): the three stage kernels per L2-sized wave of blocks.
size_t waves_scratch_bytes(const Geo& g);

}  // namespace wf
