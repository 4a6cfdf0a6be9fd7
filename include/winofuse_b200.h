/* winofuse_b200.h -- C ABI of the sm_100a transformed-convolution library.
 *
 * This is the drop-in boundary that replaces the reference's numba kernel
 * layer (winofuse/kernels.py) and the compute bodies of its engines
 * (winofuse/engines.py).  Every entry point takes plain device pointers,
 * sizes and a cudaStream_t passed as void*; nothing here allocates, frees
 * or synchronises (the caller owns all memory, the call is stream-ordered).
 * Python binds it with ctypes (paper_1912_02165_b200/_lib.py); any other
 * host language binds the same symbols.
 *
 * Tensors: activations float32 NCHW, kernels float32 (C', C, K, K), the
 * reference KernelPack float32 (T*T, C, C') -- exactly the reference layouts
 * (winofuse/tensor.py:1-5, transforms.py:22-41).
 *
 * Return value: 0 on success, otherwise a WF_ERR_* code; wf_last_error()
 * returns a thread-local description of the most recent failure.
 */
#ifndef WINOFUSE_B200_H
#define WINOFUSE_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WF_OK 0
#define WF_ERR_PARAM 1       /* InvalidParameterError  (engines.py:63-72)   */
#define WF_ERR_SHAPE 2       /* ShapeMismatchError     (engines.py:183-197) */
#define WF_ERR_UNSUPPORTED 3 /* valid for the reference, not on sm_100a      */
#define WF_ERR_CUDA 4        /* launch / runtime failure                     */
#define WF_ERR_SCRATCH 5     /* caller-provided scratch too small            */

/* transform family */
#define WF_WINOGRAD 0
#define WF_FFT16 1

/* tensor-core precision mode */
#define WF_PREC_3XBF16 0 /* x = hi + lo (bf16), hi*hi + hi*lo + lo*hi, f32 accumulate */
#define WF_PREC_BF16 1   /* single bf16 pass (fast, loose)                         */

/* Mirrors LayerSpec (reference winofuse/tensor.py:36-78). */
typedef struct wf_layer {
  int batch;
  int in_channels;
  int out_channels;
  int height;
  int width;
  int kernel;
  int pad_lo;
  int pad_hi;
} wf_layer;

/* Library / device introspection. */
int wf_version(void);
const char* wf_last_error(void);
int wf_device_sm_count(void);
/* Number of kernels this library has launched in the process so far
 * (diagnostic; benchmarks difference it around a timed region). */
unsigned long long wf_kernel_launches(void);

/* ---------------------------------------------------------------- packs --
 * Replaces transforms.transform_kernels (winofuse/transforms.py:63-80):
 * pack[p][c][c'] = f32( (G w[c'][c] G^T)[p] ) computed in float64 with one
 * final rounding.  w and pack are device pointers. */
int wf_filter_transform(const float* w, float* pack, int c_in, int c_out, int tile, void* stream);

/* Bytes of the MMA-ready packed kernels (bf16 hi/lo, UMMA K-major tiles). */
size_t wf_mma_pack_bytes(int tile, int c_in, int c_out, int transform);
/* Reference-layout f32 pack (T*T, C, C') -> MMA-ready device pack. */
int wf_mma_pack(const float* pack, void* mma_pack, int tile, int c_in, int c_out, int transform,
                void* stream);

/* ---------------------------------------------------------------- engines --
 * conv_three_stage (winofuse/engines.py:234-314): forward-transform every
 * tile, one batched GEMM per transform position, inverse-transform every
 * tile, with full-size intermediates in caller-provided scratch. */
size_t wf_three_stage_scratch_bytes(const wf_layer* layer, int tile, int transform);
int wf_conv_three_stage(const float* x, const void* mma_pack, float* y, void* scratch,
                        size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                        int precision, void* stream);

/* conv_fused (winofuse/engines.py:317-444): the transformed tiles never make
 * an HBM round trip.  `r` is the tile-task size (tiles per CTA task, the
 * reference's R, engines.py:57); 0 picks the kernel's native size. */
size_t wf_fused_scratch_bytes(const wf_layer* layer, int tile, int transform, int r);
int wf_conv_fused(const float* x, const void* mma_pack, float* y, void* scratch,
                  size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                  int precision, int r, void* stream);

/* wf_conv_fused for a caller that owns `scratch` for this one layer (a
 * planned layer, engines.LayerPlan): with WF_FUSED_COUNTERS_CLEAN the caller
 * asserts that the scratch's dependency counters are zero -- it zeroed the
 * scratch once and only calls this layer's fused engine on it -- and the
 * per-call counter reset is skipped (the kernel leaves them zero again).
 * Same results as wf_conv_fused. */
#define WF_FUSED_COUNTERS_CLEAN 1
int wf_conv_fused_planned(const float* x, const void* mma_pack, float* y, void* scratch,
                          size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                          int precision, int flags, void* stream);

/* conv_direct (winofuse/engines.py:213-231, kernels.py:22-49): 7-loop
 * cross-correlation with float64 accumulation, one f32 store. */
int wf_conv_direct(const float* x, const float* w, float* y, const wf_layer* layer, void* stream);

/* ------------------------------------------------------- stage functions --
 * Reference-layout stage kernels (winofuse/transforms.py:94-152, kernels.py:
 * 52-195).  left/dst: (T*T, rows, C) f32, res: (T*T, rows, C') f32. */
int wf_forward_tiles(const float* x, float* dst, const wf_layer* layer, int tile, int t0, int t1,
                     int row0, int dst_rows, void* stream);
int wf_multiply_positions(const float* left, const float* pack, float* res, int positions,
                          int rows, int r_eff, int c_in, int c_out, void* stream);
int wf_inverse_tiles(const float* res, float* y, const wf_layer* layer, int tile, int t0, int t1,
                     int row0, int res_rows, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WINOFUSE_B200_H */
