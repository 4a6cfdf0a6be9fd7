// fused.cu -- conv_fused: L2-resident staged fusion, wave-pipelined.
//
// The layer is processed in waves of 128-tile blocks sized so that a wave's
// transformed tiles U (bf16 hi/lo) and transform-domain products M (f32)
// stay resident in the 126 MB L2; the three stage kernels (forward, position
// GEMM, inverse) run back to back for each wave.  The transformed data is
// written and re-read inside L2 and never makes an HBM round trip: HBM
// traffic = input + output + pack.  This is the GPU analogue of the
// reference's shared-cache fusion (engines.py:317-444; section 4:
// transformed tiles stay in the shared last-level cache).
//
// Waves alternate between the caller's stream and one auxiliary stream, each
// with its own U/M buffers, so wave w+1's forward transform runs on the SMs
// left idle by wave w's GEMM / inverse tails (stage overlap without a
// device-wide scheduler).  Fork/join through events keeps the call
// stream-ordered for the caller.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include "fused.cuh"
#include "staged.cuh"
#include "gemm.cuh"

namespace wf {

static constexpr int kMaxLanes = 4;
// concurrent wave pipelines and the L2 budget of their U + M (tuning knobs
// WF_WAVE_LANES, WF_WAVE_L2_MB)
// 3 lanes (measured): VGG 256->512 / 512->512 @28 130 -> 120 / 187 -> 177 us,
// the other wave layers (c1, c4, VGG @14) unchanged
static int lanes_cfg() { return std::max(1, std::min(kMaxLanes, tuning_knob("WF_WAVE_LANES", 3))); }
static size_t budget_cfg() { return static_cast<size_t>(tuning_knob("WF_WAVE_L2_MB", 56)) << 20; }

// Bytes of U + M for one 128-tile block.
static size_t block_bytes(const Geo& g) {
  const size_t P = static_cast<size_t>(g.P);
  return P * 2 * kBlockTiles * g.Cpad * 2 + P * g.Nout * kBlockTiles * 4;
}

// Blocks per wave: as many as keep a wave's U and M in its share of L2, but
// at least enough that the wave's GEMM has work for every SM twice over
// (position x block x N-chunk items) -- for wide layers (C' >= 256) one
// L2-sized block would leave most SMs idle and the wave loop would be
// launch-bound.
static int wave_blocks(const Geo& g) {
  if (const int k = tuning_knob("WF_WAVE_BLOCKS", 0)) return std::max(1, std::min(g.n_blk, k));
  size_t nb = budget_cfg() / lanes_cfg() / block_bytes(g);
  // CTA-pair GEMM layers whose single block already overflows a lane's L2
  // share (C' >= 512: 14-19 MB per block) gain nothing from waves; one wave
  // of all blocks keeps every pair GEMM full-width (VGG 512->512 @28: waves
  // of 6 + 6 + 1 blocks 0.155 ms, one wave 0.149 ms)
  if (nb == 0 && gemm_pair_layer(g) && !gemm_resident_fits(g)) return g.n_blk;
  const int n_nc = ceil_div(g.Cppad, gemm_nc(g.Cppad));
  // FFT-16 layers with a resident-V GEMM (C'pad <= 128): the forward and
  // inverse kernels (128 CTAs per block) want larger waves (measured c4
  // 64->64 @56: 3 -> 7 blocks per wave, 257 -> 244 us)
  const int par = (g.fft && gemm_resident_fits(g)) ? 6 : 2;
  const size_t nb_par = static_cast<size_t>(ceil_div(par * 148, g.P * n_nc));
  if (nb < nb_par) nb = nb_par;
  if (nb < 1) nb = 1;
  // CTA-pair GEMM (gemm_pair.cu): whole block pairs per wave
  if (gemm_pair_layer(g) && !gemm_resident_fits(g) && (nb & 1)) ++nb;
  if (nb > static_cast<size_t>(g.n_blk)) nb = g.n_blk;
  return static_cast<int>(nb);
}

size_t waves_scratch_bytes(const Geo& g) {
  const int wb = wave_blocks(g);
  const int lanes = std::min(ceil_div(g.n_blk, wb), lanes_cfg());
  return static_cast<size_t>(lanes) * wb * block_bytes(g);
}

int fused_pick_variant(const Geo& g, const FusedOpts& o) {
  switch (o.variant) {
    case kVarWS: return ws_fits(g, o) ? kVarWS : 0;
    case kVarWSRow: return ws_fits(g, o) ? kVarWSRow : 0;
    case kVarItemQueue: return persistent_fits(g, o, false) ? kVarItemQueue : 0;
    case kVarWaves: return kVarWaves;
    case kVarAuto: break;
    default: return 0;
  }
  if (ws_fits(g, o)) return kVarWS;
  if (persistent_fits(g, o, true)) return kVarItemQueue;
  return kVarWaves;
}

size_t fused_scratch_bytes(const Geo& g, const FusedOpts& o) {
  const int v = fused_pick_variant(g, o);
  size_t own = 0;
  if (v == kVarWS || v == kVarWSRow) own = ws_scratch_bytes(g, o);
  if (v == kVarItemQueue) own = persistent_scratch_bytes(g, o);
  return std::max(own, waves_scratch_bytes(g));
}

struct LaneResources {
  cudaStream_t aux[kMaxLanes - 1] = {};
  cudaEvent_t fork = nullptr, join[kMaxLanes - 1] = {};
};

static LaneResources& lane_resources() {
  static LaneResources res[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  LaneResources& r = res[dev & 63];
  if (!r.fork) {
    for (int i = 0; i < kMaxLanes - 1; ++i) {
      cudaStreamCreateWithFlags(&r.aux[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&r.join[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
  }
  return r;
}

static cudaError_t run_waves(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                             int passes, int sm_count, cudaStream_t st);

cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g, int passes,
                      int sm_count, cudaStream_t st, const FusedOpts& o, int* ran) {
  const int v = fused_pick_variant(g, o);
  if (v == 0) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  if (v == kVarWS || v == kVarWSRow) e = run_fused_ws(x, vpack, y, scratch, g, passes, sm_count, st, o);
  else if (v == kVarItemQueue) e = run_fused_persistent(x, vpack, y, scratch, g, passes, sm_count, st, o);
  if (v != kVarWaves && e != cudaErrorCooperativeLaunchTooLarge) {
    if (ran) *ran = v;
    return e;
  }
  // the persistent kernel's CTAs cannot all be resident on this device
  // (fewer SMs available): the L2 waves need no co-residency
  if (e == cudaErrorCooperativeLaunchTooLarge) (void)cudaGetLastError();
  if (ran) *ran = kVarWaves;
  e = run_waves(x, vpack, y, scratch, g, passes, sm_count, st);
  // the waves overwrite the warp-specialised kernel's dependency counters
  // (3 n_blk + 1 ints at the start of the scratch); a caller that keeps them
  // clean between calls gets them back zeroed
  if (e == cudaSuccess && (v == kVarWS || v == kVarWSRow) && (o.flags & kFusedCountersClean))
    e = cudaMemsetAsync(scratch, 0, static_cast<size_t>(3 * g.n_blk + 1) * sizeof(int), st);
  return e;
}

static cudaError_t run_waves(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                             int passes, int sm_count, cudaStream_t st) {
  const int wb = wave_blocks(g);
  const size_t P = static_cast<size_t>(g.P);
  const size_t lane_bytes = static_cast<size_t>(wb) * block_bytes(g);
  const int n_waves = ceil_div(g.n_blk, wb);
  const int lanes = std::min(n_waves, lanes_cfg());
  LaneResources& res = lane_resources();
  cudaStream_t streams[kMaxLanes] = {st, res.aux[0], res.aux[1], res.aux[2]};
  if (lanes > 1) {
    cudaError_t e = cudaEventRecord(res.fork, st);
    for (int l = 1; l < lanes && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(streams[l], res.fork, 0);
    if (e != cudaSuccess) return e;
  }
  for (int w = 0; w < n_waves; ++w) {
    const int lane = w % lanes;
    cudaStream_t s = streams[lane];
    uint8_t* U = scratch + lane * lane_bytes;
    float* M = reinterpret_cast<float*>(U + P * wb * 2 * kBlockTiles * g.Cpad * 2);
    const int b0 = w * wb;
    const int nb = (g.n_blk - b0) < wb ? (g.n_blk - b0) : wb;
    const int tile0 = b0 * kBlockTiles;
    const int nvalid = (g.n_tile - tile0) < nb * kBlockTiles ? (g.n_tile - tile0) : nb * kBlockTiles;
    const int ldm = nb * kBlockTiles;
    cudaError_t e = launch_forward_slab(x, U, g, b0, nb, passes, s);
    if (e != cudaSuccess) return e;
    e = launch_position_gemm(U, vpack, M, g, nb, ldm, nvalid, passes, sm_count, s);
    if (e != cudaSuccess) return e;
    e = launch_inverse(M, y, g, tile0, nvalid, ldm, s);
    if (e != cudaSuccess) return e;
  }
  for (int l = 1; l < lanes; ++l) {
    cudaError_t e = cudaEventRecord(res.join[l - 1], streams[l]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, res.join[l - 1], 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace wf
