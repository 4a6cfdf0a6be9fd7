// gemm_pair.cu -- stage B on CTA pairs (tcgen05.mma.cta_group::2).
//
// The position GEMM M_p = U_p * V_p^T of the three-stage path and of the L2
// waves (staged.cu: position_gemm_kernel) streams, per 64-channel K block,
// A = 128 tiles x 64 (hi + lo, 32 KB) and B = NC x 64 (hi + lo, 64 KB at
// NC = 256) into every SM: 96 KB per 1536 tensor cycles, two stages in
// shared memory.  Measured (VGG 512->512 @28): tensor pipe 55 % of the
// elapsed cycles, the stage refill latency not covered by two stages.
//
// Here the two CTAs of a (2,1,1) cluster -- two SMs of one TPC -- own two
// consecutive 128-tile blocks of the same (position, N chunk) and issue ONE
// M = 256 MMA chain: each CTA stages its own A block and HALF of the B rows
// (NC / 2), so a K block costs 64 KB per SM instead of 96 KB and three
// stages fit.  Each CTA's TMEM holds the accumulator rows of its own block
// (M / 2 x NC), so the epilogue is the single-CTA one.
//
//   both CTAs, warp 0   : producer -- 2-D tensor copies (cta_group::2) into
//                         its own shared memory, completion bytes counted on
//                         the LEADER's full barrier
//   leader,   warp 1    : single-thread tcgen05.mma.cta_group::2 issuer;
//                         commits multicast to both CTAs' empty / tfull
//   both CTAs, warps 2-9: epilogue of their 128 rows; release the
//                         accumulator on the leader's tempty barrier
//   both CTAs, warp 1   : TMEM alloc / dealloc (cta_group::2)
//
// Used when C_pad is a multiple of 64 (whole K blocks: one box shape per
// operand); other shapes keep the single-CTA kernel.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"
#include "gemm.cuh"

namespace wf {

int tuning_knob(const char* name, int dflt);

namespace {

constexpr int kPairThreads = 320;
constexpr int kPairEpiWarps = 8;
constexpr int kPairMaxStages = 8;

// Operand buffers are addressed as 3-D tensors over the K-block layout
// (csrc/common.cuh): {64 x 16 bit = one 8-row x 8-channel core matrix row
// group's 128 bytes, 8 channel groups of a K block, 8-row groups}.  A box of
// {64, KS / 8, R / 8} gathers KS channels of R rows and lands in shared
// memory as the same layout with K block width KS (SBO = 16 KS): a stage
// holds KS channels, so KS = 32 doubles the stage count of KS = 64 for the
// same shared memory.
template <int KS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    position_gemm_pair_kernel(GemmParams P, int n_bp, const __grid_constant__ CUtensorMap tmA,
                              const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[kPairMaxStages], empty_bar[kPairMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  constexpr int kSub = kKBlock / KS;                       // stages per K block
  const int n_kb = P.Cpad / kKBlock;
  const int nh = prec_passes(P.passes) > 1 ? 2 : 1;        // hl halves streamed per operand
  const uint32_t a_bytes = kBlockTiles * KS * 2;           // one hl half of this CTA's A block
  const int bh = P.NC / 2;                                 // B rows staged by this CTA
  const uint32_t b_bytes = static_cast<uint32_t>(bh) * KS * 2;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  const int n_items = P.n_pos * n_bp * P.n_nc;
  const uint32_t tcols = P.NC * 2 <= 32 ? 32 : (P.NC * 2 <= 64 ? 64 : (P.NC * 2 <= 128 ? 128 : (P.NC * 2 <= 256 ? 256 : 512)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kPairEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if (tcols == 32) tmem_alloc_pair<32>(&tmem_slot);
    else if (tcols == 64) tmem_alloc_pair<64>(&tmem_slot);
    else if (tcols == 128) tmem_alloc_pair<128>(&tmem_slot);
    else if (tcols == 256) tmem_alloc_pair<256>(&tmem_slot);
    else tmem_alloc_pair<512>(&tmem_slot);
  }
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const size_t a_slab = static_cast<size_t>(kBlockTiles) * P.Cpad * 2;
  const int v_rows = P.cplx ? P.Cph : P.Cppad;
  const size_t v_slab = static_cast<size_t>(v_rows) * P.Cpad * 2;

  // item -> (position, block pair, N chunk): reuse the single-CTA order with
  // the pair count in place of the block count
  GemmParams Q = P;
  Q.n_blk = n_bp;

  if (warp == 0) {
    if (lane_id() == 0) {
      uint32_t full_c[kPairMaxStages];
      for (int s = 0; s < P.stages; ++s) full_c[s] = mapa_shared(&full_bar[s], 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = pair; it < n_items; it += n_pairs) {
        const GemmItem gi = gemm_item(Q, it);
        // an odd block count leaves the last pair's second block empty: it
        // re-reads the last block (its rows are never stored)
        const int blk = min(2 * gi.blk + static_cast<int>(rank), P.n_blk - 1);
        const size_t a_base = (static_cast<size_t>(gi.p) * P.n_blk + blk) * 2 * a_slab;
        const size_t b_base = static_cast<size_t>(gi.p) * 2 * v_slab;
        for (int jq = 0; jq < n_kb * kSub; ++jq) {
          const int j = jq / kSub, kq = (jq - j * kSub) * (KS / 8);   // K block, first channel group
          const int jb = gi.im ? (j + n_kb / 2) % n_kb : j;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * stage_bytes;
          if (rank == 0) mbar_expect_tx(&full_bar[stage], 2 * nh * (a_bytes + b_bytes));
          // 8-row group indices (1 KB each) of the A block / B half rows
          const size_t aoff = a_base + kblock_off(j, kBlockTiles);
          const size_t boff = b_base + kblock_off(jb, v_rows) +
                              static_cast<size_t>(gi.wrow0 + static_cast<int>(rank) * bh) / 8 * 16 * kKBlock;
          for (int h = 0; h < nh; ++h) {
            tma_load_3d_pair(st + h * a_bytes, &tmA, 0, kq, static_cast<int>((aoff + h * a_slab) >> 10), full_c[stage]);
            tma_load_3d_pair(st + 2 * a_bytes + h * b_bytes, &tmB, 0, kq, static_cast<int>((boff + h * v_slab) >> 10),
                             full_c[stage]);
          }
          if (++stage == P.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = idesc_bf16(2 * kBlockTiles, P.NC, false, false, prec_f16(P.passes));
      const uint32_t idesc_neg = idesc_bf16(2 * kBlockTiles, P.NC, false, true, prec_f16(P.passes));
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = pair; it < n_items; it += n_pairs) {
        const GemmItem gi = gemm_item(Q, it);
        mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc * P.NC;
        for (int jq = 0; jq < n_kb * kSub; ++jq) {
          const int j = jq / kSub;
          const uint32_t id = (P.cplx && !gi.im && j >= n_kb / 2) ? idesc_neg : idesc;
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t st = smem_u32(smem + stage * stage_bytes);
            constexpr uint32_t sbo = 16 * KS;
            for (uint32_t s = 0; s < KS / 16; ++s) {
              const uint64_t ahi = smem_desc(st + s * 256, 128, sbo);
              const uint64_t alo = smem_desc(st + a_bytes + s * 256, 128, sbo);
              const uint64_t bhi = smem_desc(st + 2 * a_bytes + s * 256, 128, sbo);
              const uint64_t blo = smem_desc(st + 2 * a_bytes + b_bytes + s * 256, 128, sbo);
              const uint32_t first = (jq == 0 && s == 0) ? 0u : 1u;
              if (nh > 1) {
                mma_bf16_ss_pair(dcol, alo, bhi, id, first);
                mma_bf16_ss_pair(dcol, ahi, blo, id, 1u);
                mma_bf16_ss_pair(dcol, ahi, bhi, id, 1u);
              } else {
                mma_bf16_ss_pair(dcol, ahi, bhi, id, first);
              }
            }
            mma_commit_pair(&empty_bar[stage]);
            if (jq == n_kb * kSub - 1) mma_commit_pair(&tfull_bar[acc]);
          }
          __syncwarp();
          if (++stage == P.stages) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // epilogue warps 2..9 -> TMEM lane quarter (warp % 4), column half
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane_id();
    const int split = (P.NC / 16 / 2) * 16;
    const int c_lo = half ? split : 0, c_hi = half ? P.NC : split;
    const uint32_t tempty_c0 = mapa_shared(&tempty_bar[0], 0), tempty_c1 = mapa_shared(&tempty_bar[1], 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = pair; it < n_items; it += n_pairs) {
      const GemmItem gi = gemm_item(Q, it);
      const int p = gi.p, blk = 2 * gi.blk + static_cast<int>(rank);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int tile = blk * kBlockTiles + row;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * P.NC;
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        tmem_ld16(taddr + c, v);
        tmem_ld_wait();
        if (tile < P.n_valid) {
          const int cp0 = gi.n0 + c;
          float* dst = P.M + (static_cast<size_t>(p) * P.Cp + cp0) * P.ldm + tile;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (cp0 + i < P.Cp) *dst = v[i];
            dst += P.ldm;
          }
        }
      }
      // the TMEM reads are complete (tcgen05.wait::ld); the global stores
      // need no ordering with the next MMAs, so the arrive is relaxed
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_cluster_relaxed(acc ? tempty_c1 : tempty_c0);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  cluster_sync();   // all pair MMAs consumed, no arrivals in flight to the peer
  tc_fence_after();
  if (warp == 1) {
    if (tcols == 32) tmem_dealloc_pair<32>(tmem);
    else if (tcols == 64) tmem_dealloc_pair<64>(tmem);
    else if (tcols == 128) tmem_dealloc_pair<128>(tmem);
    else if (tcols == 256) tmem_dealloc_pair<256>(tmem);
    else tmem_dealloc_pair<512>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// K-block operand bytes -> 3-D view {64 elements (128 B), 8 channel
// groups, 8-row groups}; box = KS / 8 channel groups of box_rows rows
bool encode_kblocks(CUtensorMap* m, const void* base, size_t bytes, int ks, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) || box_rows < 8 || box_rows > 2048 || box_rows % 8) return false;
  const cuuint64_t dims[3] = {64, 8, static_cast<cuuint64_t>(bytes / 1024)};
  const cuuint64_t strides[2] = {128, 1024};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(ks / 8), static_cast<cuuint32_t>(box_rows / 8)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Pair path applicable (else the caller runs the single-CTA kernel): whole
// K blocks, and enough blocks that an odd count's idle half-pair is cheap
// (one block: the pair would compute 128 dummy rows per MMA -- FFT-16
// 512->512 @7: GEMM 108 -> 155 us).
bool gemm_pair_layer(const Geo& g) {
  return tuning_knob("WF_GEMM_PAIR", 1) && g.Cpad % kKBlock == 0 && tensor_map_encoder() != nullptr;
}
bool gemm_pair_fits(const Geo& g, int nblk, int NC, int sm_count) {
  return gemm_pair_layer(g) && (nblk % 2 == 0 || nblk >= 7) && NC % 16 == 0 && NC <= 256 && sm_count >= 2;
}

cudaError_t launch_position_gemm_pair(const GemmParams& P0, const Geo& g, int sm_count, cudaStream_t st) {
  GemmParams P = P0;
  const int n_bp = (P.n_blk + 1) / 2;
  const int v_rows = P.cplx ? P.Cph : P.Cppad;
  const size_t u_bytes = static_cast<size_t>(P.n_pos) * P.n_blk * 2 * kBlockTiles * P.Cpad * 2;
  const size_t v_bytes = static_cast<size_t>(P.n_pos) * 2 * v_rows * P.Cpad * 2;
  const int ks = tuning_knob("WF_PAIR_KS", 32) == 64 ? 64 : 32;   // channels per stage
  CUtensorMap tmA, tmB;
  if (!encode_kblocks(&tmA, P.U, u_bytes, ks, kBlockTiles) || !encode_kblocks(&tmB, P.V, v_bytes, ks, P.NC / 2))
    return cudaErrorInvalidValue;
  const int stage_bytes = 2 * kBlockTiles * ks * 2 + 2 * (P.NC / 2) * ks * 2;
  P.stages = 200 * 1024 / stage_bytes;
  if (P.stages > kPairMaxStages) P.stages = kPairMaxStages;
  const int smem = P.stages * stage_bytes;
  const void* kern = ks == 64 ? reinterpret_cast<const void*>(position_gemm_pair_kernel<64>)
                              : reinterpret_cast<const void*>(position_gemm_pair_kernel<32>);
  cudaError_t e = set_smem_attr(kern, smem);
  if (e != cudaSuccess) return e;
  const int n_items = P.n_pos * n_bp * P.n_nc;
  int pairs = sm_count / 2;
  if (pairs > n_items) pairs = n_items;
  note_launch();
  if (ks == 64) position_gemm_pair_kernel<64><<<2 * pairs, kPairThreads, smem, st>>>(P, n_bp, tmA, tmB);
  else position_gemm_pair_kernel<32><<<2 * pairs, kPairThreads, smem, st>>>(P, n_bp, tmA, tmB);
  return cudaGetLastError();
}

}  // namespace wf
