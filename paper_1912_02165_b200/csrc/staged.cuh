// staged.cuh -- launchers of the stage kernels (staged.cu) used by the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace wf {

// U slabs for blocks [blk0, blk0 + nblk) -> u (local block index 0..nblk-1).
cudaError_t launch_forward_slab(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int prec,
                                cudaStream_t st);
// M[p][c'][t] (t < n_valid, stride ldm) = U_p * V_p for nblk local blocks.
cudaError_t launch_position_gemm(const uint8_t* U, const uint8_t* V, float* M, const Geo& g,
                                 int nblk, int ldm, int n_valid, int passes, int sm_count,
                                 cudaStream_t st);
// y <- inverse transform of M for tiles [tile0, tile0 + ntile).
cudaError_t launch_inverse(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                           cudaStream_t st);
int gemm_nc(int Cppad);
// Shared-memory-staged forward transform (forward.cu); 0 = geometry too wide.
int forward_staged_cpc(const Geo& g);
int forward_pipe_cpc(const Geo& g);
cudaError_t launch_forward_pipe(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc, int prec,
                                cudaStream_t st);
cudaError_t launch_forward_staged(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int cpc,
                                  int prec, cudaStream_t st);

}  // namespace wf

namespace wf {
// Position-major GEMM with the transformed kernels of one position resident
// in shared memory (gemm_resident.cu); used whenever C'pad <= 128 and V_p fits.
bool gemm_resident_fits(const Geo& g);
bool fft_cplx_pack(int C, int Cp);
cudaError_t launch_gemm_resident(const uint8_t* U, const uint8_t* V, float* M, const Geo& g, int nblk,
                                 int ldm, int n_valid, int passes, int sm_count, cudaStream_t st);
cudaError_t launch_inverse_vec(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                               cudaStream_t st);
// FFT-16 overlap-save stage kernels (fft16.cu)
cudaError_t launch_fft_forward(const float* x, uint8_t* u, const Geo& g, int blk0, int nblk, int prec,
                               cudaStream_t st);
cudaError_t launch_fft_inverse(const float* M, float* y, const Geo& g, int tile0, int ntile, int ldm,
                               cudaStream_t st);
}  // namespace wf
