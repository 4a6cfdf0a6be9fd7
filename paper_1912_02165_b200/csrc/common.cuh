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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the CURRENT device,
// remembered per (kernel, device): the attribute is per device, so a
// process-wide "done" flag would launch without it on a second GPU.
cudaError_t set_smem_attr(const void* kernel, int bytes);

// Launch a kernel whose CTAs wait on one another (the persistent dataflow
// kernels): checks that `grid` CTAs fit on the device at once (occupancy x
// SMs) and launches cooperatively, so the driver schedules every CTA
// together or fails the launch -- never a partly resident grid spinning on
// CTAs that cannot start.  cudaErrorCooperativeLaunchTooLarge when they do
// not fit (the caller falls back to the non-persistent path).
cudaError_t launch_coresident(const void* kernel, int grid, int threads, size_t smem, cudaStream_t st, void** args);
// Whether `grid` CTAs of `kernel` (threads, smem) fit on the current device at once.
bool coresident_fits(const void* kernel, int grid, int threads, size_t smem);

// Tensor-core precision of a launch: passes (1 or 3) in the low bits, the
// operand format (bf16 / fp16 hi-lo split) in bit 4.
constexpr int kPrecF16 = 16;
__host__ __device__ constexpr int prec_passes(int prec) { return prec & 15; }
__host__ __device__ constexpr bool prec_f16(int prec) { return (prec & kPrecF16) != 0; }

// 3xfp16 operand balancing.  fp16 has 11-bit significands but a narrow
// exponent range: the transformed kernels of large tiles are tiny (T = 8:
// rows of G with L1 norm 0.078, so V ~ 1e-4 and its lo parts subnormal) while
// the transformed tiles are large.  Position (r, s) therefore runs on
// U' = U * 2^(e_r + e_s - K) and V' = V * 2^-(e_r + e_s - K), e_r = the
// rounded log2 of G row r's L1 norm: an exact power-of-two rebalancing
// (U' V' == U V) that keeps both operands (and their lo parts) in the normal
// fp16 range for inputs of magnitude up to ~2^10.  FFT-16 runs unscaled.
constexpr int kF16Shift = 4;
template <int T>
__host__ __device__ constexpr int g_row_exp(int r) {
  double s = (gd<T>(r, 0) < 0 ? -gd<T>(r, 0) : gd<T>(r, 0)) + (gd<T>(r, 1) < 0 ? -gd<T>(r, 1) : gd<T>(r, 1)) +
             (gd<T>(r, 2) < 0 ? -gd<T>(r, 2) : gd<T>(r, 2));
  int e = 0;
  while (s >= 1.5) { s *= 0.5; ++e; }
  while (s < 0.75) { s *= 2.0; --e; }
  return e;
}
template <int T>
__host__ __device__ constexpr float f16_u_scale(int r, int s) {
  int e = g_row_exp<T>(r) + g_row_exp<T>(s) - kF16Shift;
  float v = 1.0f;
  while (e > 0) { v *= 2.0f; --e; }
  while (e < 0) { v *= 0.5f; ++e; }
  return v;
}
// U operand value of position (r, s) as the MMA sees it (scaled for 3xfp16)
template <int T, bool F16>
__device__ __forceinline__ float2 u_operand(float2 v, int r, int s) {
  if constexpr (F16) return make_float2(v.x * f16_u_scale<T>(r, s), v.y * f16_u_scale<T>(r, s));
  else return v;
}
template <int T, bool F16>
__device__ __forceinline__ float u_operand(float v, int r, int s) {
  if constexpr (F16) return v * f16_u_scale<T>(r, s);
  else return v;
}

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
  int cplx;          // FFT-16 with the complex-structured pack (fft_cplx_pack): V read once per bin
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

// ------------------------------------------------------------------------
// F(4x4, 3x3) (T = 6) specialisations: the 1-D transforms factored into
// shared sums (14 adds/FMAs instead of 22 for B^T, 10 instead of 18 for A^T)
// with the coefficients of the reference basis (basis_tables.cuh: bt<6>,
// at<6>).  Every path (fused, three-stage, reference-layout stage kernels)
// uses these, scalar or packed f32x2 with per element the same operations,
// so fused and three-stage results stay bitwise equal.
struct ScalarOps {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float fma(float c, float x, float acc) { return __fmaf_rn(c, x, acc); }
};
struct PairOps {
  static __device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
  // a - b == fma(b, -1, a) exactly (one rounding, like the scalar subtraction)
  static __device__ __forceinline__ float2 sub(float2 a, float2 b) {
    return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a);
  }
  static __device__ __forceinline__ float2 fma(float c, float2 x, float2 acc) {
    return __ffma2_rn(make_float2(c, c), x, acc);
  }
};
// u = B^T x for one line of 6 (in place):
//   u0 = 4x0 - 5x2 + x4        = 4(x0 - x2) + (x4 - x2)
//   u1 = -4x1 - 4x2 + x3 + x4  = (x3 + x4) - 4(x1 + x2)
//   u2 = 4x1 - 4x2 - x3 + x4   = (x4 - x3) + 4(x1 - x2)
//   u3 = -2x1 - x2 + 2x3 + x4  = (x4 - x2) + 2(x3 - x1)
//   u4 = 2x1 - x2 - 2x3 + x4   = (x4 - x2) - 2(x3 - x1)
//   u5 = -4x1 + 5x3 - x5       = 4(x3 - x1) + (x3 - x5)
template <class O, class V>
__device__ __forceinline__ void bt6_line(V& x0, V& x1, V& x2, V& x3, V& x4, V& x5) {
  const V a = O::add(x3, x4), b = O::add(x1, x2);
  const V c = O::sub(x4, x3), d = O::sub(x1, x2);
  const V e = O::sub(x4, x2), f = O::sub(x3, x1);
  const V g = O::sub(x0, x2), h = O::sub(x3, x5);
  x0 = O::fma(4.0f, g, e);
  x1 = O::fma(-4.0f, b, a);
  x2 = O::fma(4.0f, d, c);
  x3 = O::fma(2.0f, f, e);
  x4 = O::fma(-2.0f, f, e);
  x5 = O::fma(4.0f, f, h);
}
// y = A^T m for one line of 6 -> 4:
//   y0 = m0 + m1 + m2 + m3 + m4     = (m0 + p) + r
//   y1 = m1 - m2 + 2m3 - 2m4        = q + 2s
//   y2 = m1 + m2 + 4m3 + 4m4        = p + 4r
//   y3 = m1 - m2 + 8m3 - 8m4 - m5   = (q - m5) + 8s
// with p = m1 + m2, q = m1 - m2, r = m3 + m4, s = m3 - m4
template <class O, class V>
__device__ __forceinline__ void at6_line(V m0, V m1, V m2, V m3, V m4, V m5, V& y0, V& y1, V& y2, V& y3) {
  const V p = O::add(m1, m2), q = O::sub(m1, m2), r = O::add(m3, m4), s = O::sub(m3, m4);
  y0 = O::add(O::add(m0, p), r);
  y1 = O::fma(2.0f, s, q);
  y2 = O::fma(4.0f, r, p);
  y3 = O::fma(8.0f, s, O::sub(q, m5));
}
// Order: every window row first (B^T along the row), then every column --
// the streaming order of the fused kernel, which transforms each staged row
// as it is loaded and emits one column of positions at a time.
template <class O, class V>
__device__ __forceinline__ void forward6_inplace(V (&u)[6][6]) {
#pragma unroll
  for (int r = 0; r < 6; ++r) bt6_line<O>(u[r][0], u[r][1], u[r][2], u[r][3], u[r][4], u[r][5]);
#pragma unroll
  for (int s = 0; s < 6; ++s) bt6_line<O>(u[0][s], u[1][s], u[2][s], u[3][s], u[4][s], u[5][s]);
}
template <class O, class V>
__device__ __forceinline__ void forward6(const V (&x)[6][6], V (&u)[6][6]) {
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int s = 0; s < 6; ++s) u[r][s] = x[r][s];
  forward6_inplace<O>(u);
}
// Inverse order: every row of products first (A^T along the row: 6 -> 4
// values), then every column of the 6 x 4 result.  The row pass of a
// position row needs only that row's six products -- the warp-specialised
// kernel's row-unit instance runs it in the GEMM epilogue -- so every T = 6
// path uses this order and stays bitwise equal to it.
// (same operations as inverse6, with the row pass written over mm)
template <class O, class V>
__device__ __forceinline__ void inverse6_inplace(V (&mm)[6][6], V (&y)[4][4]) {
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    V t0, t1, t2, t3;
    at6_line<O>(mm[r][0], mm[r][1], mm[r][2], mm[r][3], mm[r][4], mm[r][5], t0, t1, t2, t3);
    mm[r][0] = t0; mm[r][1] = t1; mm[r][2] = t2; mm[r][3] = t3;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) at6_line<O>(mm[0][j], mm[1][j], mm[2][j], mm[3][j], mm[4][j], mm[5][j], y[0][j], y[1][j], y[2][j], y[3][j]);
}
template <class O, class V>
__device__ __forceinline__ void inverse6(const V (&mm)[6][6], V (&y)[4][4]) {
  V z[6][4];
#pragma unroll
  for (int r = 0; r < 6; ++r)
    at6_line<O>(mm[r][0], mm[r][1], mm[r][2], mm[r][3], mm[r][4], mm[r][5], z[r][0], z[r][1], z[r][2], z[r][3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) at6_line<O>(z[0][j], z[1][j], z[2][j], z[3][j], z[4][j], z[5][j], y[0][j], y[1][j], y[2][j], y[3][j]);
}
template <>
__device__ __forceinline__ void forward_transform<6>(const float (&x)[6][6], float (&u)[6][6]) {
  forward6<ScalarOps>(x, u);
}
template <>
__device__ __forceinline__ void forward_transform2<6>(const float2 (&x)[6][6], float2 (&u)[6][6]) {
  forward6<PairOps>(x, u);
}
template <>
__device__ __forceinline__ void inverse_transform<6>(const float (&mm)[6][6], float (&y)[4][4]) {
  inverse6<ScalarOps>(mm, y);
}
template <>
__device__ __forceinline__ void inverse_transform2<6>(const float2 (&mm)[6][6], float2 (&y)[4][4]) {
  inverse6<PairOps>(mm, y);
}

// ------------------------------------------------------------------------
// F(6x6, 3x3) (T = 8) specialisations, factored the same way (26 adds/FMAs
// instead of 44 for B^T, 20 instead of 38 for A^T), coefficients of the
// reference basis (basis_tables.cuh: bt<8>, at<8>).
// u = B^T x for one line of 8 (in place):
//   u0 = x0 - 21/4 x2 + 21/4 x4 - x6                 = (x0 - x6) + 21/4 (x4 - x2)
//   u1, u2 = a1 +- b1, a1 = x2 + x6 - 17/4 x4,       b1 = x1 + x5 - 17/4 x3
//   u3, u4 = a3 +- b3, a3 = x2 / 4 - 5/4 x4 + x6,    b3 = x1 / 2 - 5/2 x3 + 2 x5
//   u5, u6 = a5 +- b5, a5 = 4 x2 - 5 x4 + x6,        b5 = 2 x1 - 5/2 x3 + x5 / 2
//   u7 = x1 - 21/4 x3 + 21/4 x5 - x7                 = (x1 - x7) + 21/4 (x5 - x3)
template <class O, class V>
__device__ __forceinline__ void bt8_line(V& x0, V& x1, V& x2, V& x3, V& x4, V& x5, V& x6, V& x7) {
  const V a1 = O::fma(-4.25f, x4, O::add(x2, x6)), b1 = O::fma(-4.25f, x3, O::add(x1, x5));
  const V a3 = O::fma(0.25f, x2, O::fma(-1.25f, x4, x6)), b3 = O::fma(0.5f, x1, O::fma(-2.5f, x3, O::add(x5, x5)));
  const V a5 = O::fma(4.0f, x2, O::fma(-5.0f, x4, x6)), b5 = O::fma(0.5f, x5, O::fma(-2.5f, x3, O::add(x1, x1)));
  const V u0 = O::fma(5.25f, O::sub(x4, x2), O::sub(x0, x6));
  const V u7 = O::fma(5.25f, O::sub(x5, x3), O::sub(x1, x7));
  x0 = u0;
  x1 = O::add(a1, b1);
  x2 = O::sub(a1, b1);
  x3 = O::add(a3, b3);
  x4 = O::sub(a3, b3);
  x5 = O::add(a5, b5);
  x6 = O::sub(a5, b5);
  x7 = u7;
}
// y = A^T m for one line of 8 -> 6, with s = m1 + m2, d = m1 - m2 (and 34, 56):
//   y0 = m0 + s12 + s34 + s56
//   y1 = d12 +  2 d34 + d56 / 2      y2 = s12 +  4 s34 + s56 / 4
//   y3 = d12 +  8 d34 + d56 / 8      y4 = s12 + 16 s34 + s56 / 16
//   y5 = d12 + 32 d34 + d56 / 32 - m7
template <class O, class V>
__device__ __forceinline__ void at8_line(V m0, V m1, V m2, V m3, V m4, V m5, V m6, V m7, V& y0, V& y1, V& y2, V& y3,
                                         V& y4, V& y5) {
  const V s12 = O::add(m1, m2), d12 = O::sub(m1, m2);
  const V s34 = O::add(m3, m4), d34 = O::sub(m3, m4);
  const V s56 = O::add(m5, m6), d56 = O::sub(m5, m6);
  y0 = O::add(O::add(O::add(m0, s12), s34), s56);
  y1 = O::fma(2.0f, d34, O::fma(0.5f, d56, d12));
  y2 = O::fma(4.0f, s34, O::fma(0.25f, s56, s12));
  y3 = O::fma(8.0f, d34, O::fma(0.125f, d56, d12));
  y4 = O::fma(16.0f, s34, O::fma(0.0625f, s56, s12));
  y5 = O::fma(32.0f, d34, O::fma(0.03125f, d56, O::sub(d12, m7)));
}
// Order as for T = 6: rows, then columns (forward); columns, then rows (inverse).
template <class O, class V>
__device__ __forceinline__ void forward8(const V (&x)[8][8], V (&u)[8][8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int s = 0; s < 8; ++s) u[r][s] = x[r][s];
#pragma unroll
  for (int r = 0; r < 8; ++r) bt8_line<O>(u[r][0], u[r][1], u[r][2], u[r][3], u[r][4], u[r][5], u[r][6], u[r][7]);
#pragma unroll
  for (int s = 0; s < 8; ++s) bt8_line<O>(u[0][s], u[1][s], u[2][s], u[3][s], u[4][s], u[5][s], u[6][s], u[7][s]);
}
template <class O, class V>
__device__ __forceinline__ void inverse8(const V (&mm)[8][8], V (&y)[6][6]) {
  V t[6][8];
#pragma unroll
  for (int s = 0; s < 8; ++s)
    at8_line<O>(mm[0][s], mm[1][s], mm[2][s], mm[3][s], mm[4][s], mm[5][s], mm[6][s], mm[7][s], t[0][s], t[1][s],
                t[2][s], t[3][s], t[4][s], t[5][s]);
#pragma unroll
  for (int r = 0; r < 6; ++r)
    at8_line<O>(t[r][0], t[r][1], t[r][2], t[r][3], t[r][4], t[r][5], t[r][6], t[r][7], y[r][0], y[r][1], y[r][2],
                y[r][3], y[r][4], y[r][5]);
}
template <>
__device__ __forceinline__ void forward_transform<8>(const float (&x)[8][8], float (&u)[8][8]) {
  forward8<ScalarOps>(x, u);
}
template <>
__device__ __forceinline__ void forward_transform2<8>(const float2 (&x)[8][8], float2 (&u)[8][8]) {
  forward8<PairOps>(x, u);
}
template <>
__device__ __forceinline__ void inverse_transform<8>(const float (&mm)[8][8], float (&y)[6][6]) {
  inverse8<ScalarOps>(mm, y);
}
template <>
__device__ __forceinline__ void inverse_transform2<8>(const float2 (&mm)[8][8], float2 (&y)[6][6]) {
  inverse8<PairOps>(mm, y);
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
