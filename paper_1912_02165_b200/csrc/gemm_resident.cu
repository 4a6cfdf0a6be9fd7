// gemm_resident.cu -- stage B when a whole transformed-kernel position fits
// in shared memory: position-major persistent tcgen05 GEMM.
//
// Work items (p, block) are ordered position-major and every CTA takes one
// contiguous run of them, so a CTA keeps V_p (hi + lo, all K blocks) resident
// in shared memory across all the blocks it multiplies for position p -- the
// GPU form of the paper's "right-hand matrix stays in cache" (PAPER.md
// section 4, reference engines.py:279-289 one position at a time).  Only the
// transformed tiles U stream in, through a 4-deep mbarrier pipeline of
// bulk async copies; accumulators rotate through 4 TMEM buffers so the
// epilogue of block k overlaps the MMAs of block k+1.
//   warp 0: producer, warp 1: TMEM alloc + MMA issuer, warps 2..9: epilogue
//   (two warps per TMEM lane quadrant, each draining half of the columns).
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace wf {

constexpr int kResThreads = 320;
constexpr int kResEpiWarps = 8;
constexpr int kResStages = 4;
constexpr int kResAcc = 4;

struct ResParams {
  const uint8_t* U;
  const uint8_t* V;
  float* M;
  int n_pos, n_blk, Cpad, Cppad, Cp;
  int ldm, n_valid, passes;
};

__global__ void __launch_bounds__(kResThreads, 1) gemm_resident_kernel(ResParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[kResStages], empty_bar[kResStages], tfull[kResAcc], tempty[kResAcc];
  __shared__ uint64_t vfull, vempty;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  const int n_kb = ceil_div(P.Cpad, kKBlock);
  const uint32_t v_half = static_cast<uint32_t>(P.Cppad) * P.Cpad * 2;    // one of hi / lo
  const uint32_t a_half = kBlockTiles * kKBlock * 2;
  uint8_t* vbuf = smem;
  uint8_t* abuf = smem + round_up(2 * v_half, 1024);
  const int NC = P.Cppad;
  const uint32_t tcols = NC * kResAcc <= 256 ? 256 : 512;
  const int n_items = P.n_pos * P.n_blk;
  const int lo_it = static_cast<int>((static_cast<long long>(n_items) * blockIdx.x) / gridDim.x);
  const int hi_it = static_cast<int>((static_cast<long long>(n_items) * (blockIdx.x + 1)) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kResStages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int a = 0; a < kResAcc; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], kResEpiWarps); }
    mbar_init(&vfull, 1);
    mbar_init(&vempty, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if (tcols == 256) tmem_alloc<256>(&tmem_slot);
    else tmem_alloc<512>(&tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const size_t a_slab = static_cast<size_t>(kBlockTiles) * P.Cpad * 2;
  if (warp == 0) {
    if (lane_id() == 0) {
      int stage = 0, cur_p = -1;
      uint32_t phase = 0, vphase = 0;
      for (int it = lo_it; it < hi_it; ++it) {
        const int p = it / P.n_blk, blk = it - p * P.n_blk;
        if (p != cur_p) {
          if (cur_p >= 0) { mbar_wait(&vempty, vphase); vphase ^= 1; }
          const uint8_t* vsrc = P.V + static_cast<size_t>(p) * 2 * v_half;
          mbar_expect_tx(&vfull, (prec_passes(P.passes) > 1 ? 2 : 1) * v_half);
          bulk_g2s(vbuf, vsrc, v_half, &vfull);
          if (prec_passes(P.passes) > 1) bulk_g2s(vbuf + v_half, vsrc + v_half, v_half, &vfull);
          cur_p = p;
        }
        const uint8_t* a_src = P.U + (static_cast<size_t>(p) * P.n_blk + blk) * 2 * a_slab;
        for (int j = 0; j < n_kb; ++j) {
          const uint32_t kc = kblock_width(P.Cpad, j);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = abuf + stage * 2 * a_half;
          const uint32_t bytes = kBlockTiles * kc * 2;
          mbar_expect_tx(&full_bar[stage], 2 * bytes);
          const size_t aoff = kblock_off(j, kBlockTiles);
          bulk_g2s(st, a_src + aoff, bytes, &full_bar[stage]);
          bulk_g2s(st + a_half, a_src + a_slab + aoff, bytes, &full_bar[stage]);
          if (++stage == kResStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(kBlockTiles, NC, false, false, prec_f16(P.passes));
    int stage = 0, acc = 0, cur_p = -1;
    uint32_t phase = 0, acc_phase = 0, vphase = 0;
    for (int it = lo_it; it < hi_it; ++it) {
      const int p = it / P.n_blk;
      if (p != cur_p) {
        mbar_wait(&vfull, vphase);
        vphase ^= 1;
        cur_p = p;
      }
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem + acc * NC;
      const bool last_of_p = (it + 1 == hi_it) || ((it + 1) / P.n_blk != p);
      for (int j = 0; j < n_kb; ++j) {
        const uint32_t kc = kblock_width(P.Cpad, j);
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t st = smem_u32(abuf + stage * 2 * a_half);
          const uint32_t vb = smem_u32(vbuf) + kblock_off(j, P.Cppad);
          const uint32_t sbo = 16 * kc;
          for (uint32_t s = 0; s < kc / 16; ++s) {
            const uint64_t ahi = smem_desc(st + s * 256, 128, sbo);
            const uint64_t alo = smem_desc(st + a_half + s * 256, 128, sbo);
            const uint64_t bhi = smem_desc(vb + s * 256, 128, sbo);
            const uint64_t blo = smem_desc(vb + v_half + s * 256, 128, sbo);
            const uint32_t first = (j == 0 && s == 0) ? 0u : 1u;
            if (prec_passes(P.passes) > 1) {
              mma_bf16_ss(dcol, alo, bhi, idesc, first);
              mma_bf16_ss(dcol, ahi, blo, idesc, 1u);
              mma_bf16_ss(dcol, ahi, bhi, idesc, 1u);
            } else {
              mma_bf16_ss(dcol, ahi, bhi, idesc, first);
            }
          }
          mma_commit(&empty_bar[stage]);
          if (j == n_kb - 1) {
            mma_commit(&tfull[acc]);
            if (last_of_p) mma_commit(&vempty);
          }
        }
        __syncwarp();
        if (++stage == kResStages) { stage = 0; phase ^= 1; }
      }
      if (++acc == kResAcc) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;               // which half of the columns
    const int row = q * 32 + lane_id();
    const int split = (NC / 16 / 2) * 16;           // 16-column chunks, first half to half 0
    const int c_lo = half ? split : 0, c_hi = half ? NC : split;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = lo_it; it < hi_it; ++it) {
      const int p = it / P.n_blk, blk = it - p * P.n_blk;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int tile = blk * kBlockTiles + row;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * NC;
      float* mrow = P.M + static_cast<size_t>(p) * P.Cp * P.ldm + tile;
      const bool live = tile < P.n_valid;
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        tmem_ld16(taddr + c, v);
        tmem_ld_wait();
        if (live) {
          float* dst = mrow + static_cast<size_t>(c) * P.ldm;
          if (c + 16 <= P.Cp) {
#pragma unroll
            for (int i = 0; i < 16; ++i) { *dst = v[i]; dst += P.ldm; }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (c + i < P.Cp) *dst = v[i];
              dst += P.ldm;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&tempty[acc]);
      if (++acc == kResAcc) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    if (tcols == 256) tmem_dealloc<256>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

static size_t resident_smem(int Cpad, int Cppad) {
  const size_t v = static_cast<size_t>(Cppad) * Cpad * 2 * 2;
  return round_up(static_cast<int>(v), 1024) + kResStages * 2 * kBlockTiles * kKBlock * 2;
}
size_t gemm_resident_smem(const Geo& g) { return resident_smem(g.Cpad, g.Cppad); }

static bool resident_fits(int Cpad, int Cppad) { return Cppad <= 128 && resident_smem(Cpad, Cppad) <= 200 * 1024; }
bool gemm_resident_fits(const Geo& g) { return resident_fits(g.Cpad, g.Cppad); }

// FFT-16 layers whose GEMM runs on position_gemm_kernel (V too large to stay
// resident) use the complex-structured pack: per bin only W = [Re V^T | Im V^T]
// (C' rows x 2C), the Re / Im output halves read it with the K halves in
// place (negated upper half) / swapped -- half the pack bytes of the real
// expansion, which is what those layers stream from DRAM.
// (C' <= 256 or a multiple of 256: the GEMM's N chunks then tile each half exactly)
bool fft_cplx_pack(int C, int Cp) {
  return C % 64 == 0 && Cp % 16 == 0 && (Cp <= 256 || Cp % 256 == 0) &&
         !resident_fits(round_up(2 * C, 16), round_up(2 * Cp, 16));
}

cudaError_t launch_gemm_resident(const uint8_t* U, const uint8_t* V, float* M, const Geo& g, int nblk,
                                 int ldm, int n_valid, int passes, int sm_count, cudaStream_t st) {
  ResParams P;
  P.U = U; P.V = V; P.M = M;
  P.n_pos = g.P; P.n_blk = nblk;
  P.Cpad = g.Cpad; P.Cppad = g.Cppad; P.Cp = g.Nout;
  P.ldm = ldm; P.n_valid = n_valid; P.passes = passes;
  {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(gemm_resident_kernel), 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int n_items = P.n_pos * nblk;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_items < sm_count ? n_items : sm_count);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = gemm_resident_smem(g);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, gemm_resident_kernel, P);
}

// ------------------------------------------------------------ stage C, v2
// A warp owns 32 * TPT consecutive tiles of one c'; thread (lane) takes the
// tiles lane, lane + 32, ...: every M load of a warp reads 128 contiguous
// bytes, and every output row store of a warp writes the rows of 32
// neighbouring tiles (one vector store per tile row segment, m = 4: float4,
// m = 6: float2 x 3), so the stores fill whole sectors.
template <int T, int TPT>
__global__ void __launch_bounds__(128) inverse_vec_kernel(const float* __restrict__ M, float* __restrict__ y,
                                                          Geo g, int tile0, int ntile_local, int ldm) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 * TPT);
  const int cp = blockIdx.y;
  if (base >= ntile_local) return;
  constexpr int MO = T - 2;
  const float* src = M + static_cast<size_t>(cp) * ldm + base + lane;
  const size_t pstride = static_cast<size_t>(g.Cp) * ldm;
  // vector row stores need aligned, complete m-wide segments
  const bool vec_ok = (MO == 4 && (g.Wo & 3) == 0) || (MO == 6 && (g.Wo & 1) == 0);
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int tl = base + lane + 32 * k;
    if (tl >= ntile_local) break;
    float mm[T][T];
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) mm[r][s] = __ldcg(src + (r * T + s) * pstride + 32 * k);
    float out[MO][MO];
    inverse_transform<T>(mm, out);
    int b, ty, tx;
    tile_coords(g, tile0 + tl, b, ty, tx);
    const int oy = ty * g.m, ox = tx * g.m;
    float* plane = y + (static_cast<size_t>(b) * g.Cp + cp) * g.Ho * g.Wo;
    const bool vec = vec_ok && ox + MO <= g.Wo;
#pragma unroll
    for (int r = 0; r < MO; ++r) {
      if (oy + r >= g.Ho) break;
      float* row = plane + static_cast<size_t>(oy + r) * g.Wo + ox;
      if (vec) {
        if constexpr (MO == 4) {
          *reinterpret_cast<float4*>(row) = make_float4(out[r][0], out[r][1], out[r][2], out[r][3]);
        } else if constexpr (MO == 6) {
#pragma unroll
          for (int s = 0; s < 6; s += 2) *reinterpret_cast<float2*>(row + s) = make_float2(out[r][s], out[r][s + 1]);
        }
      } else {
#pragma unroll
        for (int s = 0; s < MO; ++s)
          if (ox + s < g.Wo) row[s] = out[r][s];
      }
    }
  }
}

template <int T>
static cudaError_t launch_inv_vec_t(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                                    cudaStream_t st) {
  constexpr int TPT = T <= 6 ? 4 : 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(ntile, 128 * TPT), g.Cp);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, inverse_vec_kernel<T, TPT>, M, y, g, tile0, ntile, ldm);
}

cudaError_t launch_inverse_vec(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                               cudaStream_t st) {
  switch (g.T) {
    case 4: return launch_inv_vec_t<4>(M, y, g, tile0, ntile, ldm, st);
    case 5: return launch_inv_vec_t<5>(M, y, g, tile0, ntile, ldm, st);
    case 6: return launch_inv_vec_t<6>(M, y, g, tile0, ntile, ldm, st);
    case 7: return launch_inv_vec_t<7>(M, y, g, tile0, ntile, ldm, st);
    case 8: return launch_inv_vec_t<8>(M, y, g, tile0, ntile, ldm, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wf
