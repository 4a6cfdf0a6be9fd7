// gemm.cuh -- parameters and item order of the position GEMM kernels
// (staged.cu: one CTA per 128-tile block; gemm_pair.cu: CTA pairs).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace wf {

struct GemmParams {
  const uint8_t* U;  // [p][blk][hl] slabs of 128 x Cpad
  const uint8_t* V;  // [p][hl] slabs of Cppad x Cpad
  float* M;          // [p][c'][tile], tile stride ldm
  int n_pos, n_blk, Cpad, Cppad, Cp;
  int NC, n_nc;      // N chunk width (multiple of 16, <= 256) and count
  int ldm;           // tiles per (p, c') row of M
  int n_valid;       // valid tiles (rows beyond are not stored)
  int passes;        // precision (common.cuh prec_*): passes 3 or 1, bf16 or fp16 operands
  int stages;        // smem pipeline depth
  int cplx;          // FFT-16 complex-structured pack: V = [Re V^T | Im V^T], Cph rows per bin
  int Cph;           // rows of the complex-structured pack (C' rounded to 16)
};

// Item -> (position, block, N chunk); for the complex-structured pack the
// chunks alternate Re / Im halves of the same pack rows (adjacent items read
// the same rows, so the second read hits L2).  n0 = first output column,
// wrow0 = first pack row, im = Im half.
struct GemmItem {
  int p, blk, n0, wrow0, im;
};
__device__ __forceinline__ GemmItem gemm_item(const GemmParams& P, int it) {
  GemmItem r;
  r.p = it / (P.n_blk * P.n_nc);
  const int rem = it - r.p * P.n_blk * P.n_nc;
  r.blk = rem / P.n_nc;
  const int nc = rem - r.blk * P.n_nc;
  if (P.cplx) {
    r.im = nc & 1;
    r.wrow0 = (nc >> 1) * P.NC;
    r.n0 = r.im * (P.Cp / 2) + r.wrow0;
  } else {
    r.im = 0;
    r.wrow0 = r.n0 = nc * P.NC;
  }
  return r;
}

// CTA-pair variant (gemm_pair.cu): whole K blocks only (C_pad % 64 == 0)
bool gemm_pair_layer(const Geo& g);
bool gemm_pair_fits(const Geo& g, int nblk, int NC, int sm_count);
cudaError_t launch_position_gemm_pair(const GemmParams& P, const Geo& g, int sm_count, cudaStream_t st);

}  // namespace wf
