// fft16.cuh -- 16-point FFT building blocks for the FFT-16 overlap-save
// transformed convolution (BASELINE config c4; no reference implementation,
// SURVEY.md 8(a) "FFT variant").
//
// Conventions (match numpy.fft): X[k] = sum_n x[n] exp(-2 pi i k n / 16),
// rfft keeps k = 0..8; the inverse carries no 1/N (the caller scales).
#pragma once

namespace wf {
namespace fft {

// cos / sin of 2*pi*k/16, k = 0..15
// (a switch, not a table: a constexpr array would be materialised in local
// memory; the switch folds to an immediate once k is a compile-time value)
__host__ __device__ constexpr float kc(int k) {
  switch (k & 15) {
    case 0: return 1.0f;
    case 1: case 15: return 0.92387953251128674f;
    case 2: case 14: return 0.70710678118654752f;
    case 3: case 13: return 0.38268343236508977f;
    case 4: case 12: return 0.0f;
    case 5: case 11: return -0.38268343236508977f;
    case 6: case 10: return -0.70710678118654752f;
    case 7: case 9: return -0.92387953251128674f;
    default: return -1.0f;
  }
}
__host__ __device__ constexpr float ks(int k) { return kc((k + 12) & 15); }  // sin(x) = cos(x - pi/2)

__device__ __forceinline__ int bitrev4(int i) {
  return ((i & 1) << 3) | ((i & 2) << 1) | ((i & 4) >> 1) | ((i & 8) >> 3);
}

// In-place radix-2 DIT complex FFT of 16 points held in registers.
// sign = -1: forward (exp(-i...)), +1: inverse (no scaling).
template <int SIGN>
__device__ __forceinline__ void fft16(float (&re)[16], float (&im)[16]) {
  float r[16], q[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int j = (((i & 1) << 3) | ((i & 2) << 1) | ((i & 4) >> 1) | ((i & 8) >> 3));
    r[i] = re[j];
    q[i] = im[j];
  }
#pragma unroll
  for (int len = 2; len <= 16; len <<= 1) {
    const int half = len >> 1;
    const int step = 16 / len;
#pragma unroll
    for (int base = 0; base < 16; base += len)
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const float wr = kc(k * step);
        const float wi = SIGN * ks(k * step);
        const int a = base + k, b = a + half;
        const float tr = r[b] * wr - q[b] * wi;
        const float ti = r[b] * wi + q[b] * wr;
        r[b] = r[a] - tr;
        q[b] = q[a] - ti;
        r[a] = r[a] + tr;
        q[a] = q[a] + ti;
      }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    re[i] = r[i];
    im[i] = q[i];
  }
}

// Real 16-point forward DFT, bins 0..8 (direct form; constant twiddles fold).
__device__ __forceinline__ void rfft16(const float (&x)[16], float (&re)[9], float (&im)[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    float sr = 0.0f, si = 0.0f;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      const int t = (k * n) & 15;
      if (kc(t) != 0.0f) sr = fmaf(x[n], kc(t), sr);
      if (ks(t) != 0.0f) si = fmaf(-x[n], ks(t), si);
    }
    re[k] = sr;
    im[k] = si;
  }
}

// Inverse of rfft16 for a Hermitian spectrum given by bins 0..8 (imag parts
// of bins 0 and 8 ignored); first NOUT outputs, no 1/16 scaling.
template <int NOUT>
__device__ __forceinline__ void irfft16(const float (&re)[9], const float (&im)[9], float (&x)[NOUT]) {
#pragma unroll
  for (int n = 0; n < NOUT; ++n) {
    float s = re[0] + ((n & 1) ? -re[8] : re[8]);
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const int t = (k * n) & 15;
      // 2 * Re(X[k] e^{+i 2pi kn/16}) = 2 (re cos - im sin)
      if (kc(t) != 0.0f) s = fmaf(2.0f * re[k], kc(t), s);
      if (ks(t) != 0.0f) s = fmaf(-2.0f * im[k], ks(t), s);
    }
    x[n] = s;
  }
}

}  // namespace fft
}  // namespace wf
