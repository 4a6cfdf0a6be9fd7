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

namespace wf {

static constexpr int kMaxLanes = 4;
// concurrent wave pipelines and the L2 budget of their U + M (WF_WAVE_LANES,
// WF_WAVE_L2_MB override)
static int lanes_cfg() {
  const char* e = getenv("WF_WAVE_LANES");
  // 3 (measured): VGG 256->512 / 512->512 @28 130 -> 120 / 187 -> 177 us,
  // the other wave layers (c1, c4, VGG @14) unchanged
  return e ? std::max(1, std::min(kMaxLanes, atoi(e))) : 3;
}
static size_t budget_cfg() {
  const char* e = getenv("WF_WAVE_L2_MB");
  return (e ? static_cast<size_t>(atoi(e)) : 56) << 20;
}

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
  if (const char* e = getenv("WF_WAVE_BLOCKS")) return std::max(1, std::min(g.n_blk, atoi(e)));
  size_t nb = budget_cfg() / lanes_cfg() / block_bytes(g);
  const int n_nc = ceil_div(g.Cppad, gemm_nc(g.Cppad));
  // FFT-16 layers with a resident-V GEMM (C'pad <= 128): the forward and
  // inverse kernels (128 CTAs per block) want larger waves (measured c4
  // 64->64 @56: 3 -> 7 blocks per wave, 257 -> 244 us)
  const int par = (g.fft && gemm_resident_fits(g)) ? 6 : 2;
  const size_t nb_par = static_cast<size_t>(ceil_div(par * 148, g.P * n_nc));
  if (nb < nb_par) nb = nb_par;
  if (nb < 1) nb = 1;
  if (nb > static_cast<size_t>(g.n_blk)) nb = g.n_blk;
  return static_cast<int>(nb);
}

size_t fused_scratch_bytes(const Geo& g, int /*r*/) {
  if (ws_fits(g)) return ws_scratch_bytes(g);
  if (persistent_fits(g)) return persistent_scratch_bytes(g);
  return static_cast<size_t>(lanes_cfg()) * wave_blocks(g) * block_bytes(g);
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

// Scratch buffers whose last fused launch was a warp-specialised kernel of
// the same geometry (which leaves its counters zero).  A caller that owns its
// scratch (counters_clean) skips the counter reset only when this says the
// previous launch on that scratch left them clean -- a different kernel or
// layer in between (environment overrides, shared scratch) forces a reset.
struct CleanScratch {
  const void* ptr;
  size_t key;
};
static bool scratch_clean_then_mark(const void* ptr, size_t key, bool clean_after) {
  static CleanScratch slots[64] = {};
  static int next = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  bool was = false;
  int hit = -1;
  for (int i = 0; i < 64; ++i)
    if (slots[i].ptr == ptr) { hit = i; was = slots[i].key == key; break; }
  if (hit < 0) { hit = next; next = (next + 1) % 64; }
  slots[hit].ptr = ptr;
  slots[hit].key = clean_after ? key : 0;
  return was;
}

cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                      int passes, int /*r*/, int sm_count, cudaStream_t st, bool counters_clean) {
  const bool ws = ws_fits(g);
  // geometry key of the warp-specialised launch (its counters' extent)
  const size_t key = ws ? (static_cast<size_t>(g.n_blk) << 20) ^ (static_cast<size_t>(g.C) << 10) ^ g.Cp ^ 1 : 0;
  const bool clean = counters_clean && scratch_clean_then_mark(scratch, key, ws) && ws;
  if (ws) return run_fused_ws(x, vpack, y, scratch, g, passes, sm_count, st, clean);
  if (persistent_fits(g)) return run_fused_persistent(x, vpack, y, scratch, g, passes, sm_count, st);
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
    cudaError_t e = launch_forward_slab(x, U, g, b0, nb, s);
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
