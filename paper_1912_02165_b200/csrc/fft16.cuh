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

// t = w * z for a compile-time twiddle w = (wr, wi) (after unrolling):
// IEEE semantics keep x * 0 from folding away (NaN, -0), so the trivial
// twiddles -- (+-1, 0) and (0, +-1) -- take the multiplication-free forms
// explicitly (in fft16 they are 17 of the 32 butterflies).
__device__ __forceinline__ void twiddle(float wr, float wi, float zr, float zi, float& tr, float& ti) {
  if (wi == 0.0f) {
    tr = zr * wr;              // wr = +-1: a (negated) copy
    ti = zi * wr;
  } else if (wr == 0.0f) {
    tr = -zi * wi;             // wi = +-1
    ti = zr * wi;
  } else {
    tr = zr * wr - zi * wi;
    ti = zr * wi + zi * wr;
  }
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
        float tr, ti;
        twiddle(wr, wi, r[b], q[b], tr, ti);
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

// In-place radix-2 DIT complex FFT of 8 points (sign -1 forward, +1 inverse,
// no scaling); twiddles are the even 16th roots (compile-time constants).
template <int SIGN>
__device__ __forceinline__ void fft8(float (&r)[8], float (&q)[8]) {
  float a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = ((i & 1) << 2) | (i & 2) | ((i & 4) >> 2);
    a[i] = r[j];
    b[i] = q[j];
  }
#pragma unroll
  for (int len = 2; len <= 8; len <<= 1) {
    const int half = len >> 1;
    const int step = 16 / len;
#pragma unroll
    for (int base = 0; base < 8; base += len)
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const float wr = kc(k * step);
        const float wi = SIGN * ks(k * step);
        const int u = base + k, v = u + half;
        float tr, ti;
        twiddle(wr, wi, a[v], b[v], tr, ti);
        a[v] = a[u] - tr;
        b[v] = b[u] - ti;
        a[u] = a[u] + tr;
        b[u] = b[u] + ti;
      }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[i] = a[i];
    q[i] = b[i];
  }
}

// Real 16-point forward DFT, bins 0..8: the even / odd samples as one
// 8-point complex FFT (z[n] = x[2n] + i x[2n+1]), then the split
// X[k] = E[k] + W16^k O[k] with E, O recovered from Z[k] and conj(Z[8-k])
// (about half the operations of the direct 16 x 9 form).
__device__ __forceinline__ void rfft16(const float (&x)[16], float (&re)[9], float (&im)[9]) {
  float zr[8], zi[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    zr[n] = x[2 * n];
    zi[n] = x[2 * n + 1];
  }
  fft8<-1>(zr, zi);
  re[0] = zr[0] + zi[0];
  im[0] = 0.0f;
  re[8] = zr[0] - zi[0];
  im[8] = 0.0f;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const int j = 8 - k;
    const float er = 0.5f * (zr[k] + zr[j]), ei = 0.5f * (zi[k] - zi[j]);
    const float orr = 0.5f * (zi[k] + zi[j]), oi = 0.5f * (zr[j] - zr[k]);
    const float c = kc(k), s = ks(k);
    if (c == 0.0f) {           // k = 4: W16^4 = -i
      re[k] = fmaf(s, oi, er);
      im[k] = fmaf(-s, orr, ei);
    } else {
      re[k] = fmaf(s, oi, fmaf(c, orr, er));
      im[k] = fmaf(-s, orr, fmaf(c, oi, ei));
    }
  }
}

// Inverse of rfft16 for a Hermitian spectrum given by bins 0..8 (imag parts
// of bins 0 and 8 ignored); first NOUT outputs, no 1/16 scaling.  The 16
// outputs come out of one 8-point complex inverse FFT of
// Z[k] = (X[k] + conj(X[8-k])) + i (X[k] - conj(X[8-k])) e^{+2 pi i k/16}:
// x[2n] = Re z[n], x[2n+1] = Im z[n].
template <int NOUT>
__device__ __forceinline__ void irfft16(const float (&re)[9], const float (&im)[9], float (&x)[NOUT]) {
  static_assert(NOUT <= 16, "irfft16 outputs");
  float zr[8], zi[8];
  zr[0] = re[0] + re[8];
  zi[0] = re[0] - re[8];
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const int j = 8 - k;
    const float sr = re[k] + re[j], si = im[k] - im[j];
    const float dr = re[k] - re[j], di = im[k] + im[j];
    const float c = kc(k), s = ks(k);
    if (c == 0.0f) {           // k = 4
      zr[k] = sr - dr * s;
      zi[k] = si - di * s;
    } else {
      zr[k] = sr - fmaf(dr, s, di * c);
      zi[k] = si + fmaf(dr, c, -di * s);
    }
  }
  fft8<1>(zr, zi);
#pragma unroll
  for (int n = 0; n < NOUT; ++n) x[n] = (n & 1) ? zi[n >> 1] : zr[n >> 1];
}

}  // namespace fft
}  // namespace wf
