// common.cuh -- geometry, operand layouts and the unrolled tile transforms
// shared by every kernel of the library.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "basis_tables.cuh"

namespace wf {

constexpr int kBlockTiles = 128;  // MMA M: tiles per tensor-core block (lane = tile)
constexpr int kKBlock = 64;       // channels per K block of an operand slab

__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Host-side count of kernel launches issued by the library (capi.cu);
// exported as wf_kernel_launches() so benchmarks can report their launches.
void note_launch();

// Layer geometry for one (layer, tile) pair; tile order is batch-major, then
// tile row, then tile column (reference tiling.py:8-11, 66-75).
struct Geo {
  int B, C, Cp, H, W, pad_lo;
  int T, m;          // window side, output block side
  int Ho, Wo;        // output extents
  int tiles_y, tiles_x, n_tile;
  int Cpad, Cppad;   // GEMM K / N (channels, x2 for FFT re|im) rounded up to 16
  int n_blk;         // ceil(n_tile / 128)
  int P;             // transform positions: T*T (Winograd) or 16*9 bins (FFT-16)
  int Nout;          // product rows per position: C' (Winograd) or 2C' (FFT re|im)
  int fft;           // 1 for the FFT-16 overlap-save transform
};

// ------------------------------------------------------------------------
// Operand slab layout ("kblock" K-major interleaved UMMA layout).
// A slab holds `rows` rows x Kpad (multiple of 16) bf16.  Channels are cut
// into K blocks of 64 (the last one may be 16/32/48 wide); inside K block j
// of width kc the element (row, kk) lives at
//   (row/8)*(16*kc) + (kk/8)*128 + (row%8)*16 + (kk%8)*2
// so an 8-row x 8-channel core matrix is 128 contiguous bytes, K-adjacent
// core matrices are 128 B apart (LBO = 128) and 8-row groups 16*kc apart
// (SBO = 16*kc).  Every K block is one contiguous range (bulk-copyable), and
// any run of 8-aligned rows inside a K block is contiguous too.
__host__ __device__ inline uint32_t kblock_width(int Kpad, int j) {
  const int rest = Kpad - j * kKBlock;
  return static_cast<uint32_t>(rest < kKBlock ? rest : kKBlock);
}
__host__ __device__ inline uint32_t slab_off(uint32_t row, uint32_t k, uint32_t rows, int Kpad) {
  const uint32_t j = k >> 6, kk = k & 63u;
  const uint32_t kc = kblock_width(Kpad, static_cast<int>(j));
  return j * rows * 128u + (row >> 3) * (16u * kc) + (kk >> 3) * 128u + (row & 7u) * 16u +
         (kk & 7u) * 2u;
}
__host__ __device__ inline uint32_t kblock_off(int j, uint32_t rows) { return j * rows * 128u; }

// ------------------------------------------------------------------------
// Tile transforms with compile-time coefficients.  Sums run in ascending
// index order like the reference kernels (kernels.py:87-98, 130-141); zero
// coefficients vanish at compile time and +-1 become plain adds.
template <int T>
__device__ __forceinline__ void forward_transform(const float (&x)[T][T], float (&u)[T][T]) {
  float t[T][T];
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (bt<T>(r, q) != 0.0f) acc = fmaf(bt<T>(r, q), x[q][s], acc);
      t[r][s] = acc;
    }
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (bt<T>(s, q) != 0.0f) acc = fmaf(t[r][q], bt<T>(s, q), acc);
      u[r][s] = acc;
    }
}

// y = A^T mm A for one (tile, c'), m x m result.
template <int T>
__device__ __forceinline__ void inverse_transform(const float (&mm)[T][T], float (&y)[T - 2][T - 2]) {
  constexpr int M = T - 2;
  float t[M][T];
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (at<T>(r, q) != 0.0f) acc = fmaf(at<T>(r, q), mm[q][s], acc);
      t[r][s] = acc;
    }
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int s = 0; s < M; ++s) {
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (at<T>(s, q) != 0.0f) acc = fmaf(t[r][q], at<T>(s, q), acc);
      y[r][s] = acc;
    }
}

// Two independent transforms at once on packed f32x2 (FFMA2/FADD2 on
// sm_100): per element exactly the operations, order and rounding of the
// scalar versions above, so the results are bitwise identical to them.
__device__ __forceinline__ float2 f2_fma(float c, float2 x, float2 acc) {
  return __ffma2_rn(make_float2(c, c), x, acc);
}
template <int T>
__device__ __forceinline__ void forward_transform2(const float2 (&x)[T][T], float2 (&u)[T][T]) {
  float2 t[T][T];
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (bt<T>(r, q) != 0.0f) acc = f2_fma(bt<T>(r, q), x[q][s], acc);
      t[r][s] = acc;
    }
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (bt<T>(s, q) != 0.0f) acc = f2_fma(bt<T>(s, q), t[r][q], acc);
      u[r][s] = acc;
    }
}
template <int T>
__device__ __forceinline__ void inverse_transform2(const float2 (&mm)[T][T], float2 (&y)[T - 2][T - 2]) {
  constexpr int M = T - 2;
  float2 t[M][T];
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (at<T>(r, q) != 0.0f) acc = f2_fma(at<T>(r, q), mm[q][s], acc);
      t[r][s] = acc;
    }
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int s = 0; s < M; ++s) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < T; ++q)
        if (at<T>(s, q) != 0.0f) acc = f2_fma(at<T>(s, q), t[r][q], acc);
      y[r][s] = acc;
    }
}

// Zero-filled T x T input window for one (tile, channel) (reference
// kernels.py:73-86: origin (ty*m - pad_lo, tx*m - pad_lo), implicit padding).
template <int T>
__device__ __forceinline__ void load_window(const float* __restrict__ plane, int H, int W, int oy,
                                            int ox, float (&x)[T][T]) {
#pragma unroll
  for (int r = 0; r < T; ++r) {
    const int yy = oy + r;
    const bool rok = (yy >= 0) && (yy < H);
#pragma unroll
    for (int s = 0; s < T; ++s) {
      const int xx = ox + s;
      x[r][s] = (rok && xx >= 0 && xx < W) ? __ldg(plane + static_cast<size_t>(yy) * W + xx) : 0.0f;
    }
  }
}

__device__ __forceinline__ void tile_coords(const Geo& g, int tile, int& b, int& ty, int& tx) {
  const int per_img = g.tiles_y * g.tiles_x;
  b = tile / per_img;
  const int rem = tile - b * per_img;
  ty = rem / g.tiles_x;
  tx = rem - ty * g.tiles_x;
}

}  // namespace wf
