// forward.cu -- stage A, shared-memory-staged forward transform.
//
// One CTA = one 128-tile block x CPC channels.  The input rows the block's
// tile rows need are staged into shared memory with coalesced loads and
// explicit zero fill (implicit padding, reference kernels.py:73-86), so the
// per-thread window reads need no bounds checks.  Thread = (tile, channel
// pair); a warp covers 32/(CPC/2) consecutive tiles x CPC/2 pairs, so each
// store instruction writes whole rows of the UMMA core matrices of the U
// slab (csrc/common.cuh layout).  Launched with programmatic dependent
// launch: the prologue overlaps the previous kernel's tail.
#include <cstdlib>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace wf {

__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_dependents_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

struct FwdStage {
  int wreg;      // staged row width: (tiles_x - 1) * m + T (padded rows) or W (bulk path)
  int trows;     // max tile rows touched by one block
  int plane;     // floats per staged channel (padded)
  int bulk;      // 1: rows staged by bulk async copies, unpadded (W % 4 == 0)
};

template <int T, int CPC, bool F16>
__global__ void __launch_bounds__(64 * CPC, (T <= 6 && CPC <= 4) ? 2 : 1)
forward_staged_kernel(const float* __restrict__ x, uint8_t* __restrict__ u, Geo g, int blk0,
                      int nblk_local, FwdStage S) {
  extern __shared__ float xs[];
  __shared__ uint64_t stage_bar;
  constexpr int PAIRS = CPC / 2;
  constexpr int TPW = 32 / PAIRS;  // tiles per warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bl = blockIdx.x;
  const int t0 = (blk0 + bl) * kBlockTiles;
  const int cbase = blockIdx.y * CPC;
  const int per_img = g.tiles_y * g.tiles_x;
  const int gr0 = t0 / g.tiles_x;  // global tile-row index (b * tiles_y + ty)
  const int tlast = min(t0 + kBlockTiles, g.n_tile) - 1;
  const int nrows = tlast / g.tiles_x - gr0 + 1;

  grid_dependency_wait();

  const int row_elems = T * S.wreg;
  if (S.bulk) {
    // ---- the T window rows of a tile row are consecutive image rows: ONE
    // bulk async copy per (channel, tile row), all in flight at once,
    // unpadded (pitch W); rows outside the image are zeroed, border columns
    // are masked when the windows are read
    if (tid == 0) {
      mbar_init(&stage_bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    fence_proxy_async_smem();
    for (int u = tid; u < CPC * nrows; u += blockDim.x) {
      const int j = u % nrows, cl = u / nrows;
      const int gr = gr0 + j;
      const int b = gr / g.tiles_y, ty = gr - b * g.tiles_y;
      const int y0 = ty * g.m - g.pad_lo;
      const int ya = max(y0, 0), yb = min(y0 + T, g.H);
      const int c = cbase + cl;
      float* dst = xs + cl * S.plane + j * row_elems;
      const bool ok = c < g.C && b < g.B && yb > ya;
      if (ok) {
        const uint32_t bytes = static_cast<uint32_t>((yb - ya) * g.W * 4);
        mbar_add_tx(&stage_bar, bytes);
        bulk_g2s(dst + (ya - y0) * g.W, x + ((static_cast<size_t>(b) * g.C + c) * g.H + ya) * g.W, bytes,
                 &stage_bar);
      }
      const int z0 = ok ? ya - y0 : 0, z1 = ok ? yb - y0 : 0;
      for (int r = 0; r < T; ++r)
        if (r < z0 || r >= z1)
          for (int s2 = 0; s2 < g.W; ++s2) dst[r * g.W + s2] = 0.0f;
    }
    __syncthreads();
    if (tid == 0) mbar_arrive(&stage_bar);
    mbar_wait(&stage_bar, 0);
  } else {
  // ---- stage the input rows of this block's tile rows, zero padded.
  // (1) one descriptor per staged row -- global row offset (or -1 for a
  // zero row) and smem offset -- so the index divisions happen once per row;
  // (2) one warp per staged row, lanes along the row, ROWS rows per
  // iteration so every thread has ROWS independent loads in flight.
  constexpr int ROWS = 8;
  const int total_rows = CPC * nrows * T;
  long long* rsrc = reinterpret_cast<long long*>(xs + CPC * S.plane);
  int* rdst = reinterpret_cast<int*>(rsrc + total_rows);
  for (int row = tid; row < total_rows; row += blockDim.x) {
    const int r = row % T;
    const int j = (row / T) % nrows;
    const int cl = row / (T * nrows);
    const int gr = gr0 + j;
    const int b = gr / g.tiles_y, ty = gr - b * g.tiles_y;
    const int yy = ty * g.m - g.pad_lo + r;
    const int c = cbase + cl;
    const bool rok = c < g.C && yy >= 0 && yy < g.H && b < g.B;
    rsrc[row] = rok ? ((static_cast<long long>(b) * g.C + c) * g.H + yy) * g.W : -1;
    rdst[row] = cl * S.plane + j * row_elems + r * S.wreg;
  }
  __syncthreads();
  const int nw = blockDim.x / 32;
  for (int row0 = warp * ROWS; row0 < total_rows; row0 += nw * ROWS) {
    for (int s0 = 0; s0 < S.wreg; s0 += 32) {
      const int s = s0 + lane;
      const int xx = s - g.pad_lo;
      const bool col_ok = s < S.wreg && xx >= 0 && xx < g.W;
      float v[ROWS];
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        const int row = row0 + k;
        const long long src = row < total_rows ? rsrc[row] : -1;
        v[k] = (src >= 0 && col_ok) ? __ldg(x + src + xx) : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        const int row = row0 + k;
        if (row < total_rows && s < S.wreg) xs[rdst[row] + s] = v[k];
      }
    }
  }
  __syncthreads();
  }

  // ---- transform: thread = (tile tl, channel pair q)
  const int tl = (warp % (kBlockTiles / TPW)) * TPW + lane % TPW;
  const int q = (warp / (kBlockTiles / TPW)) * PAIRS + lane / TPW;  // always 0..PAIRS-1 here
  const int tile = t0 + tl;
  const int c0 = cbase + 2 * q;
  float2 u2[T][T];
  if (tile < g.n_tile) {
    const int b = tile / per_img;
    const int rem = tile - b * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int j = b * g.tiles_y + ty - gr0;
    // window column 0 = staged column tx*m (padded rows) or image column
    // tx*m - pad_lo (bulk rows, masked at the borders)
    const int x0 = tx * g.m - (S.bulk ? g.pad_lo : 0);
    const float* pa = xs + j * row_elems + x0 + (2 * q) * S.plane;
    const float* pb = pa + S.plane;
    float2 w[T][T];
    if (!S.bulk || (x0 >= 0 && x0 + T <= g.W)) {
#pragma unroll
      for (int r = 0; r < T; ++r)
#pragma unroll
        for (int s = 0; s < T; ++s) w[r][s] = make_float2(pa[r * S.wreg + s], pb[r * S.wreg + s]);
    } else {
#pragma unroll
      for (int r = 0; r < T; ++r)
#pragma unroll
        for (int s = 0; s < T; ++s) {
          const bool in = x0 + s >= 0 && x0 + s < g.W;
          w[r][s] = in ? make_float2(pa[r * S.wreg + s], pb[r * S.wreg + s]) : make_float2(0.0f, 0.0f);
        }
    }
    forward_transform2<T>(w, u2);          // channels 2q, 2q+1 (packed f32x2)
  } else {
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) u2[r][s] = make_float2(0.0f, 0.0f);
  }
  const size_t slab = static_cast<size_t>(kBlockTiles) * g.Cpad * 2;
  const size_t pstride = static_cast<size_t>(nblk_local) * 2 * slab;
  if constexpr (PAIRS >= 2) {
    // lanes q and q ^ 1 (same tile, neighbouring channel pairs, TPW lanes
    // apart) swap halves: the even one stores 4 channels of hi, the odd one
    // 4 channels of lo -- one 8-byte store per position
    const bool odd = q & 1;
    const uint32_t off = slab_off(tl, cbase + 2 * (q & ~1), kBlockTiles, g.Cpad);
    uint8_t* dst = u + static_cast<size_t>(bl) * 2 * slab + off + (odd ? slab : 0);
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        uint32_t hi, lo;
        split2<F16>(u_operand<T, F16>(u2[r][s], r, s), hi, lo);
        const uint32_t other = __shfl_xor_sync(0xffffffffu, odd ? hi : lo, TPW);
        *reinterpret_cast<uint2*>(dst + (r * T + s) * pstride) = odd ? make_uint2(other, lo) : make_uint2(hi, other);
      }
  } else {
    const uint32_t off = slab_off(tl, c0, kBlockTiles, g.Cpad);
    uint8_t* dst = u + static_cast<size_t>(bl) * 2 * slab + off;
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        uint32_t hi, lo;
        split2<F16>(u_operand<T, F16>(u2[r][s], r, s), hi, lo);
        uint8_t* p = dst + (r * T + s) * pstride;
        *reinterpret_cast<uint32_t*>(p) = hi;
        *reinterpret_cast<uint32_t*>(p + slab) = lo;
      }
  }
}

static FwdStage stage_geometry(const Geo& g) {
  FwdStage S;
  S.bulk = (g.W % 4 == 0) ? 1 : 0;
  S.wreg = S.bulk ? g.W : (g.tiles_x - 1) * g.m + g.T;
  S.trows = ceil_div(kBlockTiles - 1, g.tiles_x) + 1;
  if (S.trows > g.B * g.tiles_y) S.trows = g.B * g.tiles_y;
  S.plane = round_up(S.trows * g.T * S.wreg, 32) + 4;
  return S;
}

// Channels per CTA for the staged kernel (0 = does not fit: use the v1 kernel).
int forward_staged_cpc(const Geo& g) {
  const FwdStage S = stage_geometry(g);
  // 8 channels (512 threads, <= 128 registers) only while the two T x T
  // transforms of a thread fit; larger tiles use 256-thread CTAs.
  // 4 channels per CTA first: 256-thread CTAs, two per SM, finer work items
  // (better wave balance than 512-thread CTAs).
  const size_t desc = S.bulk ? 0 : static_cast<size_t>(S.trows) * g.T * 12;   // per channel
  if (const char* e = getenv("WF_FWD_CPC")) {
    const int cpc = atoi(e);
    if ((cpc == 2 || cpc == 4 || cpc == 8) && static_cast<size_t>(cpc) * (S.plane * 4 + desc) <= 200 * 1024 &&
        g.Cpad % cpc == 0)
      return cpc;
  }
  // Wide layers (C >= 256, many channel groups per block) take 8: a warp
  // then stores whole core-matrix rows of U (VGG 512->512 @28: L2 bytes of
  // the forward kernel 188 -> 116 MB per wave, layer 199 -> 187 us).
  const int first = g.Cpad >= 256 ? 8 : 4;
  // (8 channels: 512 threads, one CTA per SM, up to 200 KB of staging;
  // 4: two 256-thread CTAs per SM, 100 KB each)
  for (int cpc : {first, 12 - first, 2})
    if ((cpc < 8 || g.T <= 6) &&
        static_cast<size_t>(cpc) * (S.plane * 4 + desc) <= (cpc == 8 ? 200 : 100) * 1024 && g.Cpad % cpc == 0)
      return cpc;
  for (int cpc : {2})
    if (static_cast<size_t>(cpc) * (S.plane * 4 + desc) <= 200 * 1024) return cpc;
  return 0;
}

template <int T, int CPC, bool F16>
static cudaError_t launch_staged(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk,
                                 cudaStream_t st) {
  const FwdStage S = stage_geometry(g);
  // staging planes + (non-bulk path) one 12-byte descriptor per staged row
  const int smem = CPC * S.plane * 4 + (S.bulk ? 0 : CPC * S.trows * g.T * 12);
  auto kern = forward_staged_kernel<T, CPC, F16>;
  {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk, g.Cpad / CPC);
  cfg.blockDim = dim3(64 * CPC);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, x, u, g, blk0, nblk, S);
}

template <int T, bool F16>
static cudaError_t launch_staged_t(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc,
                                   cudaStream_t st) {
  switch (cpc) {
    case 8: return launch_staged<T, 8, F16>(x, u, g, blk0, nblk, st);
    case 4: return launch_staged<T, 4, F16>(x, u, g, blk0, nblk, st);
    case 2: return launch_staged<T, 2, F16>(x, u, g, blk0, nblk, st);
  }
  return cudaErrorInvalidValue;
}

template <bool F16>
static cudaError_t launch_forward_staged_f(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc,
                                           cudaStream_t st) {
  switch (g.T) {
    case 4: return launch_staged_t<4, F16>(x, u, g, blk0, nblk, cpc, st);
    case 5: return launch_staged_t<5, F16>(x, u, g, blk0, nblk, cpc, st);
    case 6: return launch_staged_t<6, F16>(x, u, g, blk0, nblk, cpc, st);
    case 7: return launch_staged_t<7, F16>(x, u, g, blk0, nblk, cpc, st);
    case 8: return launch_staged_t<8, F16>(x, u, g, blk0, nblk, cpc, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_forward_staged(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc, int prec,
                                  cudaStream_t st) {
  if (prec_f16(prec)) return launch_forward_staged_f<true>(x, u, g, blk0, nblk, cpc, st);
  return launch_forward_staged_f<false>(x, u, g, blk0, nblk, cpc, st);
}

}  // namespace wf
