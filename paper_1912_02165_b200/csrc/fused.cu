// fused.cu -- conv_fused, version 1: L2-resident staged fusion.
//
// The layer is processed in waves of 128-tile blocks sized so that a wave's
// transformed tiles U (bf16 hi/lo) and transform-domain products M (f32)
// stay resident in the 126 MB L2; the three stage kernels of staged.cu run
// back to back on the stream for each wave.  The transformed data is written
// and re-read inside L2 and never makes an HBM round trip, which is the
// GPU analogue of the reference's shared-cache fusion (engines.py:317-444,
// PAPER.md section 4: right-hand matrices and transformed tiles stay in the
// shared last-level cache).  HBM traffic is therefore input + output + pack.
#include "fused.cuh"
#include "staged.cuh"

namespace wf {

// Bytes of U + M for one 128-tile block.
static size_t block_bytes(const Geo& g) {
  const size_t P = static_cast<size_t>(g.T) * g.T;
  return P * 2 * kBlockTiles * g.Cpad * 2 + P * g.Cp * kBlockTiles * 4;
}

static int wave_blocks(const Geo& g) {
  const size_t budget = 48ull << 20;  // well inside the 126 MB L2 next to the x / y streams
  size_t nb = budget / block_bytes(g);
  if (nb < 1) nb = 1;
  if (nb > static_cast<size_t>(g.n_blk)) nb = g.n_blk;
  return static_cast<int>(nb);
}

size_t fused_scratch_bytes(const Geo& g, int /*r*/) {
  return static_cast<size_t>(wave_blocks(g)) * block_bytes(g);
}

cudaError_t run_fused(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                      int passes, int /*r*/, int sm_count, cudaStream_t st) {
  const int wb = wave_blocks(g);
  const size_t P = static_cast<size_t>(g.T) * g.T;
  uint8_t* U = scratch;
  float* M = reinterpret_cast<float*>(scratch + P * wb * 2 * kBlockTiles * g.Cpad * 2);
  for (int b0 = 0; b0 < g.n_blk; b0 += wb) {
    const int nb = (g.n_blk - b0) < wb ? (g.n_blk - b0) : wb;
    const int tile0 = b0 * kBlockTiles;
    const int nvalid = (g.n_tile - tile0) < nb * kBlockTiles ? (g.n_tile - tile0) : nb * kBlockTiles;
    const int ldm = nb * kBlockTiles;
    cudaError_t e = launch_forward_slab(x, U, g, b0, nb, st);
    if (e != cudaSuccess) return e;
    e = launch_position_gemm(U, vpack, M, g, nb, ldm, nvalid, passes, sm_count, st);
    if (e != cudaSuccess) return e;
    e = launch_inverse(M, y, g, tile0, nvalid, ldm, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace wf
