// fft16.cu -- stage kernels of the FFT-16 overlap-save transformed
// convolution (BASELINE config c4).  The reference has no FFT path
// (SURVEY.md 8(a) "FFT variant": SPEC.md:17 puts it out of scope); this
// follows the definition SURVEY.md 8(b) gives for the new framework:
//
//   * 16x16 input windows at stride 14 (the same OLA tile grid as
//     Winograd with m = 14), zero outside the padded input;
//   * rfft2 of each window: 16 x 9 = 144 Hermitian-half bins;
//   * per bin a complex GEMM  M[t][c'] = sum_c X[t][c] * conj(W[c'][c]),
//     run as a real GEMM with K = 2C ([Re | Im] of X) and N = 2C'
//     ([Re | Im] of M) on the same tcgen05 position GEMM as Winograd;
//   * irfft2 of each product window, keep the valid 14 x 14 block.
//
// Forward: one CTA = 8 tiles x 8 input channels, 16 half-warp groups.  A
// group computes one (tile, channel) 2-D FFT at a time: thread r does the
// real 16-point DFT of window row r, the row spectra go through a per-group
// shared scratch, then threads v = 0..8 run the complex 16-point FFT down
// column v.  The CTA's 144 x 16 x 8 spectrum is staged in shared memory and
// written as bf16 hi/lo operand slabs (coalesced 128-byte core matrices).
// Inverse mirrors it: load M for 16 tiles x 8 output channels, column
// inverse FFTs, then each row thread runs the inverse real DFT and keeps 14
// outputs.
#include "common.cuh"
#include "fft16.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace wf {
namespace {

constexpr int kFftTiles = 8;             // tiles per CTA (one 8-row core-matrix group of the slab)
constexpr int kFftCh = 8;                // channels per CTA
constexpr int kBins = 144;               // 16 x 9
constexpr int kBinPitch = 65;            // floats per bin in the staging arrays (odd: conflict-free columns)
constexpr int kGroupScratch = 2 * 144;   // per-group row spectra (re, im), pitch 9 per row
constexpr size_t kFftSmem = (2ull * kBins * kBinPitch + 16ull * kGroupScratch) * sizeof(float);

__device__ __forceinline__ int stage_idx(int p, int c, int t) { return p * kBinPitch + c * kFftTiles + t; }

template <bool F16>
__global__ void __launch_bounds__(256, 2) fft_forward_kernel(const float* __restrict__ x, uint8_t* __restrict__ u,
                                                             Geo g, int tile0, int nblk_local) {
  extern __shared__ float smem[];
  float* sre = smem;
  float* sim = smem + kBins * kBinPitch;
  const int grp = threadIdx.x >> 4, r = threadIdx.x & 15;
  float* gre = smem + 2 * kBins * kBinPitch + grp * kGroupScratch;
  float* gim = gre + 144;
  const unsigned gmask = 0xFFFFu << (threadIdx.x & 16);
  const int local_limit = nblk_local * kBlockTiles;
  const int tl0 = blockIdx.x * kFftTiles;   // first local tile of this CTA
  const int cg0 = blockIdx.y * kFftCh;      // first input channel

  // ---- 2-D FFTs: group grp owns tile grp & 7, channels 4 * (grp >> 3) + 0..3.
  {
    const int tg = grp & (kFftTiles - 1);
    const int tl = tl0 + tg, tile = tile0 + tl;
    const bool tvalid = tl < local_limit && tile < g.n_tile;
    int b = 0, ty = 0, tx = 0;
    if (tvalid) tile_coords(g, tile, b, ty, tx);
    const int iy = ty * g.m - g.pad_lo + r, ox = tx * g.m - g.pad_lo;
    const bool rvalid = tvalid && iy >= 0 && iy < g.H;
    // The group's 4 channel rows: with 16-byte aligned rows (W % 4 == 0)
    // all four are fetched up front as five aligned float4s each (a float4
    // lies wholly inside or outside the row; outside ones are not loaded),
    // so 20 independent loads per thread are in flight before the first FFT
    // (one row ahead measured load-latency bound); other widths load
    // per element, one channel at a time.
    const bool vec = (g.W & 3) == 0;
    const int sh = ox & 3, base = ox - sh;           // window start inside its 16-byte word
    float4 raw[kFftCh / 2][5];
    if (vec) {
#pragma unroll
      for (int ci4 = 0; ci4 < kFftCh / 2; ++ci4) {
        const int ch = cg0 + (grp >> 3) * (kFftCh / 2) + ci4;
        const float* src = x + ((static_cast<size_t>(b) * g.C + ch) * g.H + iy) * g.W;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const int c4 = base + 4 * i;
          raw[ci4][i] = (rvalid && ch < g.C && c4 >= 0 && c4 < g.W)
                            ? __ldg(reinterpret_cast<const float4*>(src + c4))
                            : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
      }
    }
    auto f4c = [](const float4& q, int c) { return c == 0 ? q.x : (c == 1 ? q.y : (c == 2 ? q.z : q.w)); };
    auto load_row = [&](int ci4, float (&row)[16]) {
      if (vec) {
        // columns [base, base + 20) -> window columns [ox, ox + 16)
        // (out-of-row float4s are zeros already; the in-row ones hold only
        // in-row columns)
        switch (sh) {
#define WF_FFT_PICK(SH)                                                            \
  case SH:                                                                         \
    _Pragma("unroll") for (int s2 = 0; s2 < 16; ++s2) row[s2] = f4c(raw[ci4][(s2 + SH) >> 2], (s2 + SH) & 3); \
    break;
          WF_FFT_PICK(0)
          WF_FFT_PICK(1)
          WF_FFT_PICK(2)
          WF_FFT_PICK(3)
#undef WF_FFT_PICK
        }
        return;
      }
      const int ch = cg0 + (grp >> 3) * (kFftCh / 2) + ci4;
      if (rvalid && ch < g.C) {
        const float* src = x + ((static_cast<size_t>(b) * g.C + ch) * g.H + iy) * g.W;
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) {
          const int ix = ox + s2;
          row[s2] = (ix >= 0 && ix < g.W) ? __ldg(src + ix) : 0.0f;
        }
      } else {
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) row[s2] = 0.0f;
      }
    };
#pragma unroll
    for (int ci4 = 0; ci4 < kFftCh / 2; ++ci4) {
      const int c = (grp >> 3) * (kFftCh / 2) + ci4;
      float row[16];
      load_row(ci4, row);
      float fr[9], fi[9];
      fft::rfft16(row, fr, fi);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        gre[r * 9 + k] = fr[k];
        gim[r * 9 + k] = fi[k];
      }
      __syncwarp(gmask);
      if (r < 9) {
        float cr[16], ci[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          cr[q] = gre[q * 9 + r];
          ci[q] = gim[q * 9 + r];
        }
        fft::fft16<-1>(cr, ci);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          sre[stage_idx(q * 9 + r, c, tg)] = cr[q];
          sim[stage_idx(q * 9 + r, c, tg)] = ci[q];
        }
      }
      __syncwarp(gmask);
    }
  }
  __syncthreads();

  // ---- write the bf16 hi/lo slabs: K index c (Re) and C + c (Im).
  const size_t slab = static_cast<size_t>(kBlockTiles) * g.Cpad * 2;
  const int tid = threadIdx.x;
  if ((g.C & 7) == 0) {
    // Re and Im 8-channel groups are both aligned core-matrix columns.
    const int q = tid & 3, t = (tid >> 2) & 7, part = (tid >> 5) & 1, pp = tid >> 6;
    const int tl = tl0 + t;
    if (tl < local_limit) {
      const int blk = tl / kBlockTiles, row = tl % kBlockTiles;
      const uint32_t off = slab_off(row, (part ? g.C : 0) + cg0 + 2 * q, kBlockTiles, g.Cpad);
      const float* sa = part ? sim : sre;
      // (running pointer: a 64-bit multiply per bin was most of this loop)
      uint8_t* base = u + ((static_cast<size_t>(pp) * nblk_local + blk) * 2) * slab + off;
      const size_t bstep = static_cast<size_t>(4) * nblk_local * 2 * slab;
#pragma unroll 4
      for (int p = pp; p < kBins; p += 4) {
        uint32_t hi, lo;
        split2<F16>(sa[stage_idx(p, 2 * q, t)], sa[stage_idx(p, 2 * q + 1, t)], hi, lo);
        *reinterpret_cast<uint32_t*>(base) = hi;
        *reinterpret_cast<uint32_t*>(base + slab) = lo;
        base += bstep;
      }
    }
  } else {
    // General channel counts: element-wise 16-bit stores.
    const int c = tid & 7, t = (tid >> 3) & 7, part = (tid >> 6) & 1, pp = tid >> 7;
    const int tl = tl0 + t;
    if (tl < local_limit && cg0 + c < g.C) {
      const int blk = tl / kBlockTiles, row = tl % kBlockTiles;
      const uint32_t off = slab_off(row, (part ? g.C : 0) + cg0 + c, kBlockTiles, g.Cpad);
      const float* sa = part ? sim : sre;
      for (int p = pp; p < kBins; p += 2) {
        const float v = sa[stage_idx(p, c, t)];
        uint32_t hv, lv;
        split2<F16>(v, 0.0f, hv, lv);
        uint8_t* base = u + ((static_cast<size_t>(p) * nblk_local + blk) * 2) * slab + off;
        *reinterpret_cast<uint16_t*>(base) = static_cast<uint16_t>(hv & 0xFFFFu);
        *reinterpret_cast<uint16_t*>(base + slab) = static_cast<uint16_t>(lv & 0xFFFFu);
      }
    }
    // K padding [2C, Cpad) must hold zeros: channel-group 0 writes it.
    const int npad = g.Cpad - 2 * g.C;
    if (blockIdx.y == 0 && npad > 0) {
      for (int i = tid; i < kBins * kFftTiles * npad; i += blockDim.x) {
        const int k = 2 * g.C + i % npad;
        const int t = (i / npad) % kFftTiles;
        const int p = i / (npad * kFftTiles);
        const int tl2 = tl0 + t;
        if (tl2 >= local_limit) continue;
        const int blk = tl2 / kBlockTiles, row = tl2 % kBlockTiles;
        uint8_t* base = u + ((static_cast<size_t>(p) * nblk_local + blk) * 2) * slab +
                        slab_off(row, k, kBlockTiles, g.Cpad);
        *reinterpret_cast<uint16_t*>(base) = 0;
        *reinterpret_cast<uint16_t*>(base + slab) = 0;
      }
    }
  }
}

// Inverse: CTA = 32 tiles x 2 output channels, 9 warps.  Pass 1: warp v
// runs the complex 16-point inverse FFT down spectrum column v for its 32
// tiles (lane = tile: every load of M is one coalesced 128-byte row) and
// keeps rows 0..13 in shared memory.  Pass 2: thread = (tile, c', output
// row r) runs the inverse real DFT over the 9 columns and stores its 14
// outputs (a warp covers whole output-row segments of adjacent tiles).
constexpr int kInvTiles = 32;
constexpr int kInvCh = 2;
constexpr int kInvThreads = 9 * 32;
constexpr size_t kInvSmem = static_cast<size_t>(kInvCh) * 14 * 9 * kInvTiles * sizeof(float2);

__global__ void __launch_bounds__(kInvThreads) fft_inverse_kernel(const float* __restrict__ M, float* __restrict__ y,
                                                                   Geo g, int tile0, int ntile, int ldm) {
  extern __shared__ float2 zs[];                 // [c][r][v][tile]
  const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
  const int tl0 = blockIdx.x * kInvTiles;
  const int cg0 = blockIdx.y * kInvCh;
  const int tl = tl0 + lane;
  const bool tvalid = tl < ntile;
  // both channels' spectrum columns are loaded before either FFT runs (64
  // independent coalesced loads in flight per thread)
  float rec[kInvCh][16], imc[kInvCh][16];
#pragma unroll
  for (int c = 0; c < kInvCh; ++c) {
    const int cp = cg0 + c;
    if (tvalid && cp < g.Cp) {
      // bins u * 9 + v, u = 0..15: a running pointer (stride 9 bins)
      const float* pr = M + (static_cast<size_t>(v) * g.Nout + cp) * ldm + tl;
      const size_t im_off = static_cast<size_t>(g.Cp) * ldm;
      const size_t ustep = static_cast<size_t>(9) * g.Nout * ldm;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        rec[c][u] = __ldcg(pr);
        imc[c][u] = __ldcg(pr + im_off);
        pr += ustep;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) rec[c][u] = imc[c][u] = 0.0f;
    }
  }
#pragma unroll
  for (int c = 0; c < kInvCh; ++c) {
    float (&re)[16] = rec[c];
    float (&im)[16] = imc[c];
    fft::fft16<1>(re, im);
#pragma unroll
    for (int r = 0; r < 14; ++r) zs[((c * 14 + r) * 9 + v) * kInvTiles + lane] = make_float2(re[r], im[r]);
  }
  __syncthreads();
  for (int u = threadIdx.x; u < kInvCh * 14 * kInvTiles; u += kInvThreads) {
    const int t = u % kInvTiles;
    const int r = (u / kInvTiles) % 14;
    const int c = u / (kInvTiles * 14);
    const int cp = cg0 + c;
    const int tli = tl0 + t;
    if (tli >= ntile || cp >= g.Cp) continue;
    int b = 0, ty = 0, tx = 0;
    tile_coords(g, tile0 + tli, b, ty, tx);
    const int oy = ty * g.m + r, ox = tx * g.m;
    if (oy >= g.Ho) continue;
    float zr[9], zi[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float2 z = zs[((c * 14 + r) * 9 + k) * kInvTiles + t];
      zr[k] = z.x;
      zi[k] = z.y;
    }
    float out[14];
    fft::irfft16<14>(zr, zi, out);
    float* dst = y + ((static_cast<size_t>(b) * g.Cp + cp) * g.Ho + oy) * g.Wo + ox;
    if ((g.Wo & 1) == 0 && ox + 14 <= g.Wo) {      // 8-byte aligned full row segment
#pragma unroll
      for (int s2 = 0; s2 < 14; s2 += 2)
        *reinterpret_cast<float2*>(dst + s2) = make_float2(out[s2] * (1.0f / 256.0f), out[s2 + 1] * (1.0f / 256.0f));
    } else {
#pragma unroll
      for (int s2 = 0; s2 < 14; ++s2)
        if (ox + s2 < g.Wo) dst[s2] = out[s2] * (1.0f / 256.0f);
    }
  }
}

}  // namespace

cudaError_t launch_fft_forward(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int prec,
                               cudaStream_t st) {
  auto kern = prec_f16(prec) ? fft_forward_kernel<true> : fft_forward_kernel<false>;
  {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(kFftSmem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(ceil_div(nblk * kBlockTiles, kFftTiles), ceil_div(g.C, kFftCh));
  note_launch();
  kern<<<grid, 256, kFftSmem, st>>>(x, u, g, blk0 * kBlockTiles, nblk);
  return cudaGetLastError();
}

cudaError_t launch_fft_inverse(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                               cudaStream_t st) {
  {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(fft_inverse_kernel), static_cast<int>(kInvSmem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(ceil_div(ntile, kInvTiles), ceil_div(g.Cp, kInvCh));
  note_launch();
  fft_inverse_kernel<<<grid, kInvThreads, kInvSmem, st>>>(M, y, g, tile0, ntile, ldm);
  return cudaGetLastError();
}

}  // namespace wf
