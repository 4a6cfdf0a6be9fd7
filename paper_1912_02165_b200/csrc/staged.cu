// staged.cu -- the three stage kernels of the transformed convolution and
// the tcgen05 batched GEMM that is the transform-domain contraction.
//
//   stage A  forward_slab_kernel : x (NCHW f32) -> U (bf16 hi/lo UMMA slabs)
//   stage B  position_gemm_kernel: M[p] = U[p] * V[p]  on tcgen05 (3xBF16)
//   stage C  inverse_kernel      : M -> y (NCHW f32), clipped scatter
//
// They implement the reference's kernels.forward_tiles / matmul_rows /
// inverse_tiles (winofuse/kernels.py:52-166) in the shape of
// engines.conv_three_stage (engines.py:234-314).  The fused engine
// (fused.cu) reuses the device functions so the two engines agree.
#include <cstdio>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"
#include "gemm.cuh"

namespace wf {

// ---------------------------------------------------------------- stage A
// CTA = 32 tiles x 16 channels, 8 warps.  A warp owns 8 consecutive tiles x
// 8 channels: lane = (tile r8 = lane&7, channel pair q = lane>>3) so, for each
// transform position, the warp's 32 bf16x2 stores form exactly one 128-byte
// core matrix of the slab (coalesced).  Tiles past n_tile and channels past C
// are written as zeros (they are the MMA's padding rows / K columns).
template <int T, bool F16>
__global__ void __launch_bounds__(256) forward_slab_kernel(const float* __restrict__ x,
                                                           uint8_t* __restrict__ u, Geo g,
                                                           int tile0, int nblk_local) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = blockIdx.x * 32 + (warp & 3) * 8 + (lane & 7);  // local tile index
  const int c0 = blockIdx.y * 16 + (warp >> 2) * 8 + (lane >> 3) * 2;
  const int tile = tile0 + tl;
  const bool tvalid = tl < nblk_local * kBlockTiles && tile < g.n_tile;
  float ua[T][T], ub[T][T];
  {
    float w[T][T];
    int b = 0, ty = 0, tx = 0;
    if (tvalid) tile_coords(g, tile, b, ty, tx);
    const int oy = ty * g.m - g.pad_lo, ox = tx * g.m - g.pad_lo;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = c0 + h;
      if (tvalid && c < g.C) {
        load_window<T>(x + (static_cast<size_t>(b) * g.C + c) * g.H * g.W, g.H, g.W, oy, ox, w);
      } else {
#pragma unroll
        for (int r = 0; r < T; ++r)
#pragma unroll
          for (int s = 0; s < T; ++s) w[r][s] = 0.0f;
      }
      if (h == 0) forward_transform<T>(w, ua);
      else forward_transform<T>(w, ub);
    }
  }
  if (tl >= nblk_local * kBlockTiles) return;
  const int blk = tl / kBlockTiles, row = tl % kBlockTiles;
  const size_t slab = static_cast<size_t>(kBlockTiles) * g.Cpad * 2;
  const uint32_t off = slab_off(row, c0, kBlockTiles, g.Cpad);
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      const int p = r * T + s;
      uint32_t hi, lo;
      split2<F16>(u_operand<T, F16>(ua[r][s], r, s), u_operand<T, F16>(ub[r][s], r, s), hi, lo);
      uint8_t* base = u + ((static_cast<size_t>(p) * nblk_local + blk) * 2) * slab + off;
      *reinterpret_cast<uint32_t*>(base) = hi;
      *reinterpret_cast<uint32_t*>(base + slab) = lo;
    }
}

// ---------------------------------------------------------------- stage B
// Persistent warp-specialised tcgen05 GEMM, one work item = (position p,
// 128-tile block b, N chunk nc):  D[128 x NC] = U_p,b[128 x K] * V_p[NC x K]^T
// accumulated in TMEM, K streamed in 64-channel blocks by bulk copies.
//   warp 0      : bulk-copy producer (A hi/lo, B hi/lo K-block per stage)
//   warp 1      : TMEM allocator + single-thread MMA issuer
//   warps 2..9  : epilogue, TMEM -> registers -> M (f32, [p][c'][tile]);
//                 two warps per TMEM lane quarter, each half of the columns
// 3xBF16: D = Uhi*Vhi + Uhi*Vlo + Ulo*Vhi (f32 accumulate); 1 pass for bf16.
constexpr int kGemmThreads = 320;
constexpr int kGemmEpiWarps = 8;

__global__ void __launch_bounds__(kGemmThreads, 1) position_gemm_kernel(GemmParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[4], empty_bar[4], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5;
  const int n_kb = ceil_div(P.Cpad, kKBlock);
  const uint32_t a_bytes = kBlockTiles * kKBlock * 2;  // one hl half of A, full K block
  const uint32_t b_bytes = static_cast<uint32_t>(P.NC) * kKBlock * 2;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  const int n_items = P.n_pos * P.n_blk * P.n_nc;
  const uint32_t tcols = P.NC * 2 <= 32 ? 32 : (P.NC * 2 <= 64 ? 64 : (P.NC * 2 <= 128 ? 128 : (P.NC * 2 <= 256 ? 256 : 512)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kGemmEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if (tcols == 32) tmem_alloc<32>(&tmem_slot);
    else if (tcols == 64) tmem_alloc<64>(&tmem_slot);
    else if (tcols == 128) tmem_alloc<128>(&tmem_slot);
    else if (tcols == 256) tmem_alloc<256>(&tmem_slot);
    else tmem_alloc<512>(&tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const size_t a_slab = static_cast<size_t>(kBlockTiles) * P.Cpad * 2;
  const int v_rows = P.cplx ? P.Cph : P.Cppad;              // rows of one pack slab
  const size_t v_slab = static_cast<size_t>(v_rows) * P.Cpad * 2;

  if (warp == 0) {
    if (lane_id() == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const GemmItem gi = gemm_item(P, it);
        const uint8_t* a_src = P.U + (static_cast<size_t>(gi.p) * P.n_blk + gi.blk) * 2 * a_slab;
        const uint8_t* b_src = P.V + static_cast<size_t>(gi.p) * 2 * v_slab;
        for (int j = 0; j < n_kb; ++j) {
          const uint32_t kc = kblock_width(P.Cpad, j);
          // complex pack, Im half: the Re inputs (K blocks < n_kb / 2) meet
          // Im V and the Im inputs Re V -- the pack's K halves swapped
          const int jb = gi.im ? (j + n_kb / 2) % n_kb : j;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * stage_bytes;
          const uint32_t abytes = kBlockTiles * kc * 2, bbytes = P.NC * kc * 2;
          mbar_expect_tx(&full_bar[stage], 2 * abytes + (prec_passes(P.passes) > 1 ? 2 : 1) * bbytes);
          const size_t aoff = kblock_off(j, kBlockTiles);
          const size_t boff = kblock_off(jb, v_rows) + static_cast<size_t>(gi.wrow0) / 8 * 16 * kc;
          bulk_g2s(st, a_src + aoff, abytes, &full_bar[stage]);
          bulk_g2s(st + a_bytes, a_src + a_slab + aoff, abytes, &full_bar[stage]);
          bulk_g2s(st + 2 * a_bytes, b_src + boff, bbytes, &full_bar[stage]);
          if (prec_passes(P.passes) > 1) bulk_g2s(st + 2 * a_bytes + b_bytes, b_src + v_slab + boff, bbytes, &full_bar[stage]);
          if (++stage == P.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(kBlockTiles, P.NC, false, false, prec_f16(P.passes));
    // complex pack, Re half: the Im inputs meet -Im V (negated B operand)
    const uint32_t idesc_neg = idesc_bf16(kBlockTiles, P.NC, false, true, prec_f16(P.passes));
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const GemmItem gi = gemm_item(P, it);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem + acc * P.NC;
      for (int j = 0; j < n_kb; ++j) {
        const uint32_t kc = kblock_width(P.Cpad, j);
        const uint32_t id = (P.cplx && !gi.im && j >= n_kb / 2) ? idesc_neg : idesc;
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t st = smem_u32(smem + stage * stage_bytes);
          const uint32_t sbo = 16 * kc;
          for (uint32_t s = 0; s < kc / 16; ++s) {
            const uint64_t ahi = smem_desc(st + s * 256, 128, sbo);
            const uint64_t alo = smem_desc(st + a_bytes + s * 256, 128, sbo);
            const uint64_t bhi = smem_desc(st + 2 * a_bytes + s * 256, 128, sbo);
            const uint64_t blo = smem_desc(st + 2 * a_bytes + b_bytes + s * 256, 128, sbo);
            const uint32_t first = (j == 0 && s == 0) ? 0u : 1u;
            if (prec_passes(P.passes) > 1) {
              mma_bf16_ss(dcol, alo, bhi, id, first);
              mma_bf16_ss(dcol, ahi, blo, id, 1u);
              mma_bf16_ss(dcol, ahi, bhi, id, 1u);
            } else {
              mma_bf16_ss(dcol, ahi, bhi, id, first);
            }
          }
          mma_commit(&empty_bar[stage]);
          if (j == n_kb - 1) mma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == P.stages) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // epilogue warps 2..9 -> TMEM lane quarter (warp % 4), column half
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane_id();
    const int split = (P.NC / 16 / 2) * 16;
    const int c_lo = half ? split : 0, c_hi = half ? P.NC : split;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const GemmItem gi = gemm_item(P, it);
      const int p = gi.p, blk = gi.blk;
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
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    if (tcols == 32) tmem_dealloc<32>(tmem);
    else if (tcols == 64) tmem_dealloc<64>(tmem);
    else if (tcols == 128) tmem_dealloc<128>(tmem);
    else if (tcols == 256) tmem_dealloc<256>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- stage C
// Thread = (tile, c'); reads T^2 products M[p][c'][tile] (coalesced across the
// tiles of a warp), applies A^T m A and stores the clipped m x m block
// (reference kernels.py:103-141).
template <int T>
__global__ void __launch_bounds__(128) inverse_kernel(const float* __restrict__ M, float* __restrict__ y,
                                                      Geo g, int tile0, int ntile_local, int ldm) {
  const int tl = blockIdx.x * blockDim.x + threadIdx.x;
  const int cp = blockIdx.y;
  if (tl >= ntile_local) return;
  float mm[T][T];
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s)
      mm[r][s] = __ldg(M + (static_cast<size_t>(r * T + s) * g.Cp + cp) * ldm + tl);
  constexpr int MO = T - 2;
  float out[MO][MO];
  inverse_transform<T>(mm, out);
  int b, ty, tx;
  tile_coords(g, tile0 + tl, b, ty, tx);
  const int oy = ty * g.m, ox = tx * g.m;
  float* plane = y + (static_cast<size_t>(b) * g.Cp + cp) * g.Ho * g.Wo;
#pragma unroll
  for (int r = 0; r < MO; ++r) {
    if (oy + r >= g.Ho) break;
#pragma unroll
    for (int s = 0; s < MO; ++s)
      if (ox + s < g.Wo) plane[static_cast<size_t>(oy + r) * g.Wo + ox + s] = out[r][s];
  }
}

// ---------------------------------------------------------------- launchers
template <int T>
static cudaError_t launch_forward_t(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int prec,
                                    cudaStream_t st) {
  dim3 grid(ceil_div(nblk * kBlockTiles, 32), g.Cpad / 16);
  note_launch();
  if (prec_f16(prec)) forward_slab_kernel<T, true><<<grid, 256, 0, st>>>(x, u, g, blk0 * kBlockTiles, nblk);
  else forward_slab_kernel<T, false><<<grid, 256, 0, st>>>(x, u, g, blk0 * kBlockTiles, nblk);
  return cudaGetLastError();
}

cudaError_t launch_forward_slab(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int prec,
                                cudaStream_t st) {
  if (g.fft) return launch_fft_forward(x, u, g, blk0, nblk, prec, st);
  const int pcpc = forward_pipe_cpc(g);
  if (pcpc) return launch_forward_pipe(x, u, g, blk0, nblk, pcpc, prec, st);
  const int cpc = forward_staged_cpc(g);
  if (cpc) return launch_forward_staged(x, u, g, blk0, nblk, cpc, prec, st);
  switch (g.T) {
    case 4: return launch_forward_t<4>(x, u, g, blk0, nblk, prec, st);
    case 5: return launch_forward_t<5>(x, u, g, blk0, nblk, prec, st);
    case 6: return launch_forward_t<6>(x, u, g, blk0, nblk, prec, st);
    case 7: return launch_forward_t<7>(x, u, g, blk0, nblk, prec, st);
    case 8: return launch_forward_t<8>(x, u, g, blk0, nblk, prec, st);
  }
  return cudaErrorInvalidValue;
}

int gemm_nc(int Cppad) {
  if (Cppad <= 256) return Cppad;
  // Split into equal multiples of 16 not exceeding 256.
  const int n = ceil_div(Cppad, 256);
  return round_up(ceil_div(Cppad, n), 16);
}

cudaError_t launch_position_gemm(const uint8_t* U, const uint8_t* V, float* M, const Geo& g,
                                 int nblk, int ldm, int n_valid, int passes, int sm_count,
                                 cudaStream_t st) {
  if (gemm_resident_fits(g))
    return launch_gemm_resident(U, V, M, g, nblk, ldm, n_valid, passes, sm_count, st);
  GemmParams P;
  P.U = U; P.V = V; P.M = M;
  P.n_pos = g.P;
  P.n_blk = nblk;
  P.Cpad = g.Cpad; P.Cppad = g.Cppad; P.Cp = g.Nout;
  P.cplx = g.cplx;
  P.Cph = round_up(g.Cp, 16);
  if (g.cplx) {
    // chunks never straddle the Re / Im halves: NC divides C'
    P.NC = gemm_nc(g.Cp);
    P.n_nc = 2 * ceil_div(g.Cp, P.NC);
  } else {
    P.NC = gemm_nc(g.Cppad);
    P.n_nc = ceil_div(g.Cppad, P.NC);
  }
  P.ldm = ldm;
  P.n_valid = n_valid;
  P.passes = passes;
  if (gemm_pair_fits(g, nblk, P.NC, sm_count)) {
    const cudaError_t e = launch_position_gemm_pair(P, g, sm_count, st);
    if (e == cudaSuccess) return e;
    (void)cudaGetLastError();   // pair launch refused (tensor map / cluster resources): one CTA per block
  }
  const int stage_bytes = 2 * kBlockTiles * kKBlock * 2 + 2 * P.NC * kKBlock * 2;
  P.stages = 200 * 1024 / stage_bytes;
  if (P.stages > 4) P.stages = 4;
  if (P.stages < 2) P.stages = 2;
  const int smem = P.stages * stage_bytes;
  {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(position_gemm_kernel), 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int n_items = P.n_pos * P.n_blk * P.n_nc;
  const int grid = n_items < sm_count ? n_items : sm_count;
  note_launch();
  position_gemm_kernel<<<grid, kGemmThreads, smem, st>>>(P);
  return cudaGetLastError();
}

template <int T>
static cudaError_t launch_inverse_t(const float* M, float* y, const Geo& g, int tile0, int ntile,
                                    int ldm, cudaStream_t st) {
  dim3 grid(ceil_div(ntile, 128), g.Cp);
  note_launch();
  inverse_kernel<T><<<grid, 128, 0, st>>>(M, y, g, tile0, ntile, ldm);
  return cudaGetLastError();
}

cudaError_t launch_inverse(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                           cudaStream_t st) {
  if (g.fft) return launch_fft_inverse(M, y, g, tile0, ntile, ldm, st);
  return launch_inverse_vec(M, y, g, tile0, ntile, ldm, st);
  switch (g.T) {
    case 4: return launch_inverse_t<4>(M, y, g, tile0, ntile, ldm, st);
    case 5: return launch_inverse_t<5>(M, y, g, tile0, ntile, ldm, st);
    case 6: return launch_inverse_t<6>(M, y, g, tile0, ntile, ldm, st);
    case 7: return launch_inverse_t<7>(M, y, g, tile0, ntile, ldm, st);
    case 8: return launch_inverse_t<8>(M, y, g, tile0, ntile, ldm, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wf
