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

// Window of one tile for the channel pair (2q, 2q+1) from shared memory:
// pa / pb = row 0, column 0 of the two channels; masked: the window crosses
// the image border (columns outside [0, W) read 0).
template <int T>
__device__ __forceinline__ void window_scalar(const float* pa, const float* pb, int pitch, bool masked, int x0, int W,
                                              float2 (&w)[T][T]) {
  if (!masked) {
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) w[r][s] = make_float2(pa[r * pitch + s], pb[r * pitch + s]);
  } else {
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        const bool in = x0 + s >= 0 && x0 + s < W;
        w[r][s] = in ? make_float2(pa[r * pitch + s], pb[r * pitch + s]) : make_float2(0.0f, 0.0f);
      }
  }
}

// Transform the window w of channels (2q, 2q+1) (valid: the tile exists;
// otherwise zeros are stored) and store the hi / lo operand halves.
template <int T, int CPC, bool F16>
__device__ __forceinline__ void transform_store(bool valid, const float2 (&w)[T][T], uint8_t* __restrict__ u, int bl,
                                                int nblk_local, int tl, int q, int cbase, int Cpad) {
  constexpr int PAIRS = CPC / 2;
  constexpr int TPW = 32 / PAIRS;  // tiles per warp
  float2 u2[T][T];
  if (valid) {
    forward_transform2<T>(w, u2);          // channels 2q, 2q+1 (packed f32x2)
  } else {
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) u2[r][s] = make_float2(0.0f, 0.0f);
  }
  const size_t slab = static_cast<size_t>(kBlockTiles) * Cpad * 2;
  const size_t pstride = static_cast<size_t>(nblk_local) * 2 * slab;
  if constexpr (PAIRS >= 2) {
    // lanes q and q ^ 1 (same tile, neighbouring channel pairs, TPW lanes
    // apart) swap halves: the even one stores 4 channels of hi, the odd one
    // 4 channels of lo -- one 8-byte store per position
    const bool odd = q & 1;
    const uint32_t off = slab_off(tl, cbase + 2 * (q & ~1), kBlockTiles, Cpad);
    // (the position stride is added to a running pointer: a 64-bit
    // multiply-add per store made address arithmetic a third of the
    // kernel's instructions)
    uint8_t* dst = u + static_cast<size_t>(bl) * 2 * slab + off + (odd ? slab : 0);
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        uint32_t hi, lo;
        split2<F16>(u_operand<T, F16>(u2[r][s], r, s), hi, lo);
        const uint32_t other = __shfl_xor_sync(0xffffffffu, odd ? hi : lo, TPW);
        *reinterpret_cast<uint2*>(dst) = odd ? make_uint2(other, lo) : make_uint2(hi, other);
        dst += pstride;
      }
  } else {
    const uint32_t off = slab_off(tl, cbase + 2 * q, kBlockTiles, Cpad);
    uint8_t* dst = u + static_cast<size_t>(bl) * 2 * slab + off;
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        uint32_t hi, lo;
        split2<F16>(u_operand<T, F16>(u2[r][s], r, s), hi, lo);
        *reinterpret_cast<uint32_t*>(dst) = hi;
        *reinterpret_cast<uint32_t*>(dst + slab) = lo;
        dst += pstride;
      }
  }
}

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
  const float* pa = nullptr;
  int x0 = 0;
  if (tile < g.n_tile) {
    const int b = tile / per_img;
    const int rem = tile - b * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int j = b * g.tiles_y + ty - gr0;
    // window column 0 = staged column tx*m (padded rows) or image column
    // tx*m - pad_lo (bulk rows, masked at the borders)
    x0 = tx * g.m - (S.bulk ? g.pad_lo : 0);
    pa = xs + j * row_elems + x0 + (2 * q) * S.plane;
  }
  float2 w[T][T];
  if (pa) window_scalar<T>(pa, pa + S.plane, S.wreg, S.bulk && (x0 < 0 || x0 + T > g.W), x0, g.W, w);
  transform_store<T, CPC, F16>(pa != nullptr, w, u, bl, nblk_local, tl, q, cbase, g.Cpad);
}

// ---------------------------------------------------------------------------
// Pipelined variant (bulk path, W % 4 == 0): a persistent CTA walks the
// (block, channel group) items with two staging buffers -- the bulk copies of
// item i+1 are in flight while item i is transformed and stored, so the HBM
// reads overlap the U stores instead of alternating with them (one 512-thread
// CTA per SM left the SM idle during every load).  Only the image rows the
// block's windows touch are staged, once each: per image a segment of
// (tile rows - 1) * m + T rows (consecutive tile rows share T - m rows);
// rows outside the image and padded channels are never written -- border
// windows mask them (rows, columns, channels) after the reads.  VGG
// 512->512 @28: 60 -> 47 us (issue-bound before: 64-bit store addressing,
// 4-way bank conflicts of the scalar window reads, zero fills).
// Window rows of the pipelined kernel read as aligned float4s: the staged
// rows are 16-byte aligned (W % 4 == 0), so a window of T columns starting at
// x0 lies in the (T + 6) / 4 float4s from x0 & ~3.  Scalar reads of windows
// m = 4 floats apart touch only 8 of the 32 banks (4-way conflicts); the
// float4 reads of 8 consecutive tiles are one conflict-free wavefront.
__device__ __forceinline__ float f4c(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}
// Window validity bits (masked path): bit r of rows = window row r inside
// the image, bit s of cols_a / cols_b = column s inside the image and the
// channel real (not K padding).
struct WinMask {
  uint32_t rows, cols_a, cols_b;
};
template <int T, int SH>
__device__ __forceinline__ void window_vec_sh(const float* pa, const float* pb, int pitch, bool masked,
                                              const WinMask& mk, float2 (&w)[T][T]) {
  constexpr int NV = (T + 6) / 4;
#pragma unroll
  for (int r = 0; r < T; ++r) {
    float4 va[NV], vb[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      va[i] = *reinterpret_cast<const float4*>(pa + r * pitch + 4 * i);
      vb[i] = *reinterpret_cast<const float4*>(pb + r * pitch + 4 * i);
    }
#pragma unroll
    for (int s = 0; s < T; ++s) {
      const int i = s + SH;
      w[r][s] = make_float2(f4c(va[i >> 2], i & 3), f4c(vb[i >> 2], i & 3));
    }
  }
  if (masked) {
    // selects, not products: rows outside the image are never staged
    // (uninitialised shared memory)
#pragma unroll
    for (int r = 0; r < T; ++r) {
      const uint32_t ra = (mk.rows >> r) & 1u ? mk.cols_a : 0u, rb = (mk.rows >> r) & 1u ? mk.cols_b : 0u;
#pragma unroll
      for (int s = 0; s < T; ++s) {
        if (!((ra >> s) & 1u)) w[r][s].x = 0.0f;
        if (!((rb >> s) & 1u)) w[r][s].y = 0.0f;
      }
    }
  }
}
// pa, pb: row 0 of the window's two channels at column x0 & ~3
template <int T>
__device__ __forceinline__ void window_vec(const float* pa, const float* pb, int pitch, int x0, bool masked,
                                           const WinMask& mk, float2 (&w)[T][T]) {
  switch (x0 & 3) {
    case 0: window_vec_sh<T, 0>(pa, pb, pitch, masked, mk, w); break;
    case 1: window_vec_sh<T, 1>(pa, pb, pitch, masked, mk, w); break;
    case 2: window_vec_sh<T, 2>(pa, pb, pitch, masked, mk, w); break;
    default: window_vec_sh<T, 3>(pa, pb, pitch, masked, mk, w); break;
  }
}

struct FwdPipe {
  int plane;     // floats per staged channel (multiple of 4)
  int n_cg;      // channel groups (Cpad / CPC)
  int n_items;   // nblk_local * n_cg
};

// Segment k (image b0 + k) of the item whose tile rows are gr0..grl:
// first tile row in the image, first staged row (smem) and row count.
struct FwdSeg {
  int tya, base, rows;
};
__device__ __forceinline__ FwdSeg fwd_seg(const Geo& g, int gr0, int grl, int k) {
  const int b0 = gr0 / g.tiles_y, b1 = grl / g.tiles_y, b = b0 + k;
  const int tya0 = gr0 - b0 * g.tiles_y;
  const int tyb0 = b0 == b1 ? grl - b0 * g.tiles_y : g.tiles_y - 1;
  const int rows0 = (tyb0 - tya0) * g.m + g.T;
  const int full = (g.tiles_y - 1) * g.m + g.T;
  FwdSeg sg;
  sg.tya = k == 0 ? tya0 : 0;
  const int tyb = b == b1 ? grl - b1 * g.tiles_y : g.tiles_y - 1;
  sg.rows = (tyb - sg.tya) * g.m + g.T;
  sg.base = k == 0 ? 0 : rows0 + (k - 1) * full;
  return sg;
}

template <int T, int CPC, bool F16>
__global__ void __launch_bounds__(64 * CPC, (T <= 6 && CPC <= 4) ? 2 : 1)
forward_pipe_kernel(const float* __restrict__ x, uint8_t* __restrict__ u, Geo g, int blk0, int nblk_local,
                    FwdPipe S) {
  extern __shared__ __align__(16) float xs_raw[];
  // 4 guard floats before the buffers, 12 after: the float4 window reads of
  // border tiles start up to 3 floats before a row and end past it (masked)
  float* xs = xs_raw + 4;
  __shared__ uint64_t full_bar[2];
  constexpr int PAIRS = CPC / 2;
  constexpr int TPW = 32 / PAIRS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per_img = g.tiles_y * g.tiles_x;
  const int buf_floats = CPC * S.plane;

  if (tid == 0) {
    mbar_init(&full_bar[0], 1);
    mbar_init(&full_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  grid_dependency_wait();

  // Stage item `it` into buffer `bi` (warp 0): one bulk copy per (channel,
  // image segment) of its in-image rows, then one arrival.  Rows outside the
  // image and padded channels are not staged at all: the window reads of
  // border tiles mask them.
  auto stage = [&](int it, int bi) {
    const int bl = it / S.n_cg, cbase = (it - bl * S.n_cg) * CPC;
    const int t0 = (blk0 + bl) * kBlockTiles;
    const int tlast = min(t0 + kBlockTiles, g.n_tile) - 1;
    const int gr0 = t0 / g.tiles_x, grl = tlast / g.tiles_x;
    const int nseg = grl / g.tiles_y - gr0 / g.tiles_y + 1;
    const int b0 = gr0 / g.tiles_y;
    float* buf = xs + bi * buf_floats;
    fence_proxy_async_smem();
    for (int v = lane; v < CPC * nseg; v += 32) {
      const int k = v / CPC, cl = v - k * CPC;
      const FwdSeg sg = fwd_seg(g, gr0, grl, k);
      const int y0 = sg.tya * g.m - g.pad_lo;
      const int ya = max(y0, 0), yb = min(y0 + sg.rows, g.H);
      const int c = cbase + cl;
      if (c < g.C && yb > ya) {
        const uint32_t bytes = static_cast<uint32_t>((yb - ya) * g.W * 4);
        mbar_add_tx(&full_bar[bi], bytes);
        bulk_g2s(buf + cl * S.plane + (sg.base + ya - y0) * g.W,
                 x + ((static_cast<size_t>(b0 + k) * g.C + c) * g.H + ya) * g.W, bytes, &full_bar[bi]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&full_bar[bi]);
  };

  // (one CTA barrier per item frees the buffer for the refill; per-warp
  // release through mbarriers measured the same)
  int it = blockIdx.x;
  if (warp == 0 && it < S.n_items) stage(it, 0);
  for (int i = 0; it < S.n_items; ++i, it += gridDim.x) {
    const int bi = i & 1;
    if (warp == 0 && it + static_cast<int>(gridDim.x) < S.n_items) {
      stage(it + gridDim.x, bi ^ 1);
    }
    mbar_wait(&full_bar[bi], (i >> 1) & 1);

    const int bl = it / S.n_cg, cbase = (it - bl * S.n_cg) * CPC;
    const int t0 = (blk0 + bl) * kBlockTiles;
    const int tlast = min(t0 + kBlockTiles, g.n_tile) - 1;
    const int gr0 = t0 / g.tiles_x, grl = tlast / g.tiles_x;
    const int b0 = gr0 / g.tiles_y;
    const int tl = (warp % (kBlockTiles / TPW)) * TPW + lane % TPW;
    const int q = (warp / (kBlockTiles / TPW)) * PAIRS + lane / TPW;
    const int tile = t0 + tl;
    const float* pa = nullptr;
    WinMask mk;
    bool masked = false;
    int x0 = 0;
    if (tile < g.n_tile) {
      const int b = tile / per_img;
      const int rem = tile - b * per_img;
      const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
      const FwdSeg sg = fwd_seg(g, gr0, grl, b - b0);
      x0 = tx * g.m - g.pad_lo;
      const int y0 = ty * g.m - g.pad_lo;
      const bool b_ok = cbase + 2 * q + 1 < g.C;
      masked = x0 < 0 || x0 + T > g.W || y0 < 0 || y0 + T > g.H || !b_ok;
      if (masked) {
        const uint32_t all = (1u << T) - 1u;
        const uint32_t cols = (x0 < 0 ? all << -x0 : all) & (all >> max(x0 + T - g.W, 0));
        mk.rows = (y0 < 0 ? all << -y0 : all) & (all >> max(y0 + T - g.H, 0));
        mk.cols_a = cbase + 2 * q < g.C ? cols : 0u;
        mk.cols_b = b_ok ? cols : 0u;
      }
      pa = xs + bi * buf_floats + (2 * q) * S.plane + (sg.base + (ty - sg.tya) * g.m) * g.W + (x0 & ~3);
    }
    float2 w[T][T];
    if (pa) window_vec<T>(pa, pa + S.plane, g.W, x0, masked, mk, w);
    transform_store<T, CPC, F16>(pa != nullptr, w, u, bl, nblk_local, tl, q, cbase, g.Cpad);
    __syncthreads();
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


// ---- pipelined launcher
int sm_count();
int tuning_knob(const char* name, int dflt);

// floats per staged channel of the pipelined kernel: at most trows tile rows
// spread over at most nseg images, (tile rows) * m + (images) * (T - m) rows
static int pipe_plane(const Geo& g) {
  const FwdStage S = stage_geometry(g);
  const int nseg = ceil_div(S.trows - 1, g.tiles_y) + 1;
  const int rows = S.trows * g.m + (nseg < S.trows ? nseg : S.trows) * (g.T - g.m);
  return round_up(rows * g.W, 32) + 4;
}

// Channels per CTA of the pipelined kernel (0 = not applicable): the two
// buffers of 8 channels in one 512-thread CTA per SM (T <= 6), or of 4 / 2
// channels in CTAs of which two fit per SM; wide layers first try 8 (a warp
// then stores whole core-matrix rows of U).
int forward_pipe_cpc(const Geo& g) {
  if (g.W % 4 != 0 || !tuning_knob("WF_FWD_PIPE", 1)) return 0;
  const size_t per_ch = 2 * static_cast<size_t>(pipe_plane(g)) * 4;
  const int first = g.Cpad >= 256 ? 8 : 4;
  // (2 channels -- 128-thread CTAs, 4-byte U stores -- measured slower than
  // the one-shot kernel: VGG 64->64 @224 three-stage 1.26 -> 1.45 ms)
  for (int cpc : {first, 12 - first}) {
    if (g.Cpad % cpc || (cpc == 8 && g.T > 6)) continue;
    if (cpc * per_ch + 64 <= static_cast<size_t>(cpc == 8 ? 200 : 110) * 1024) return cpc;
  }
  return 0;
}

template <int T, int CPC, bool F16>
static cudaError_t launch_pipe(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, cudaStream_t st) {
  FwdPipe S;
  S.plane = pipe_plane(g);
  S.n_cg = g.Cpad / CPC;
  S.n_items = nblk * S.n_cg;
  const int smem = (2 * CPC * S.plane + 16) * 4;
  auto kern = forward_pipe_kernel<T, CPC, F16>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  static int per_sm_cached = 0, smem_cached = -1;   // (per instantiation) CTAs per SM at the last smem size
  if (smem_cached != smem) {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 64 * CPC, smem);
    if (e != cudaSuccess) return e;
    per_sm_cached = per_sm > 0 ? per_sm : 1;
    smem_cached = smem;
  }
  int grid = sm_count() * per_sm_cached;
  if (grid > S.n_items) grid = S.n_items;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
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
static cudaError_t launch_pipe_t(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc,
                                 cudaStream_t st) {
  switch (cpc) {
    case 8: if constexpr (T <= 6) return launch_pipe<T, 8, F16>(x, u, g, blk0, nblk, st); break;
    case 4: return launch_pipe<T, 4, F16>(x, u, g, blk0, nblk, st);
  }
  return cudaErrorInvalidValue;
}

template <bool F16>
static cudaError_t launch_forward_pipe_f(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc,
                                         cudaStream_t st) {
  switch (g.T) {
    case 4: return launch_pipe_t<4, F16>(x, u, g, blk0, nblk, cpc, st);
    case 5: return launch_pipe_t<5, F16>(x, u, g, blk0, nblk, cpc, st);
    case 6: return launch_pipe_t<6, F16>(x, u, g, blk0, nblk, cpc, st);
    case 7: return launch_pipe_t<7, F16>(x, u, g, blk0, nblk, cpc, st);
    case 8: return launch_pipe_t<8, F16>(x, u, g, blk0, nblk, cpc, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_forward_pipe(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc, int prec,
                                cudaStream_t st) {
  if (prec_f16(prec)) return launch_forward_pipe_f<true>(x, u, g, blk0, nblk, cpc, st);
  return launch_forward_pipe_f<false>(x, u, g, blk0, nblk, cpc, st);
}

}  // namespace wf
