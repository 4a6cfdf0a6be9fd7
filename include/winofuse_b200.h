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
#define WF_PREC_3XBF16 0 /* x = hi + lo (bf16), hi*hi + hi*lo + lo*hi, f32 accumulate  */
#define WF_PREC_BF16 1   /* single bf16 pass (fast, loose)                          */
#define WF_PREC_3XFP16 2 /* x = hi + lo (fp16, 11-bit significands), three passes:  */
                         /* ~22-bit products at the bf16 rate; needs the transformed */
                         /* values inside the fp16 range (|u| < 65504)               */

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
/* Reference-layout f32 pack (T*T, C, C') -> MMA-ready device pack (3xbf16 /
 * bf16 operand format). */
int wf_mma_pack(const float* pack, void* mma_pack, int tile, int c_in, int c_out, int transform,
                void* stream);
/* The same for a precision mode (WF_PREC_*): the operand format (bf16 or fp16
 * hi/lo) of the pack must match the precision the engines run with. */
int wf_mma_pack_ex(const float* pack, void* mma_pack, int tile, int c_in, int c_out, int transform, int precision,
                   void* stream);

/* ---------------------------------------------------------------- engines --
 * conv_three_stage (winofuse/engines.py:234-314): forward-transform every
 * tile, one batched GEMM per transform position, inverse-transform every
 * tile, with full-size intermediates in caller-provided scratch. */
size_t wf_three_stage_scratch_bytes(const wf_layer* layer, int tile, int transform);
int wf_conv_three_stage(const float* x, const void* mma_pack, float* y, void* scratch,
                        size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                        int precision, void* stream);

/* The three stages as separate launches (phases: WF_PHASE_* bits), so a
 * caller can time each with events -- the reference's per-stage phase_s
 * (engines.py:263-302).  Run in order on one stream over the same scratch. */
#define WF_PHASE_FORWARD 1
#define WF_PHASE_MULTIPLY 2
#define WF_PHASE_INVERSE 4
int wf_conv_three_stage_phases(const float* x, const void* mma_pack, float* y, void* scratch,
                               size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                               int precision, int phases, void* stream);

/* conv_fused (winofuse/engines.py:317-444): the transformed tiles never make
 * an HBM round trip.  `r` is the reference's tiles-per-task knob
 * (engines.py:57); the sm_100a kernels use 128-tile blocks (the MMA M) and
 * ignore it. */
size_t wf_fused_scratch_bytes(const wf_layer* layer, int tile, int transform, int r);
int wf_conv_fused(const float* x, const void* mma_pack, float* y, void* scratch,
                  size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                  int precision, int r, void* stream);

/* Fused-engine variants: which kernel runs the layer. */
#define WF_FUSED_AUTO 0  /* the fastest variant that can hold the layer               */
#define WF_FUSED_WS 1    /* warp-specialised persistent dataflow kernel (fused_ws.cu)  */
#define WF_FUSED_ITEMQ 2 /* item-queue persistent dataflow kernel (fused_persistent.cu)*/
#define WF_FUSED_WAVES 3 /* the stage kernels per L2-resident wave of blocks (fused.cu) */
#define WF_FUSED_WS_ROW 4 /* warp-specialised kernel, row units: a CTA owns a row of      */
                          /* transform positions and runs the inverse transform's row    */
                          /* pass in the GEMM epilogue (F(4x4,3x3), C = C' = 64, inputs   */
                          /* whose F units stage in 48 KB); never picked by AUTO (slower) */

/* Flags.  COUNTERS_CLEAN: the caller asserts that the scratch's dependency
 * counters are zero -- it zero-filled the scratch once and only runs this
 * layer's fused engine on it -- so the per-call counter reset is skipped
 * (the warp-specialised kernel leaves them zero again).  INSTRUMENT: run the
 * instrumented kernel (ordering tickets + per-role busy cycles, read back
 * with wf_fused_instrument_read); warp-specialised variant only. */
#define WF_FUSED_COUNTERS_CLEAN 1
#define WF_FUSED_INSTRUMENT 2

/* Per-call options; zero-initialise for the defaults. */
typedef struct wf_fused_opts {
  int variant;       /* WF_FUSED_*                                                    */
  int flags;         /* WF_FUSED_COUNTERS_CLEAN | WF_FUSED_INSTRUMENT                 */
  size_t ring_bytes; /* L2 ring budget of the persistent kernels (EngineConfig.l2_budget_bytes), 0 = default */
  int lag;           /* steps between a block's producer and consumer units, 0 = default; any value is safe (clamped to the rings) */
  int gbatch;        /* G completions per publish (warp-specialised), 0 = default    */
} wf_fused_opts;

/* The variant that runs (> 0), or -WF_ERR_* (e.g. -WF_ERR_UNSUPPORTED when
 * the requested variant cannot hold the layer). */
int wf_fused_variant(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts);
size_t wf_fused_scratch_bytes_ex(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts);
/* *variant_ran (may be NULL) = the variant that ran: the requested or picked
 * one, or WF_FUSED_WAVES when a persistent kernel's CTAs cannot all be
 * resident on the device (the waves need no co-residency). */
int wf_conv_fused_ex(const float* x, const void* mma_pack, float* y, void* scratch, size_t scratch_bytes,
                     const wf_layer* layer, int tile, int transform, int precision, const wf_fused_opts* opts,
                     int* variant_ran, void* stream);
/* wf_conv_fused_ex with opts = {WF_FUSED_AUTO, flags}. */
int wf_conv_fused_planned(const float* x, const void* mma_pack, float* y, void* scratch,
                          size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                          int precision, int flags, void* stream);
/* After an instrumented launch (synchronises the device): events = 8 words
 * per 128-tile block (ordering tickets: 0 F start << 12 | CTA, 1 ~F end,
 * 2 G start, 3 ~G end, 4 I start, 5 ~I end), role_cycles[4] = SM cycles summed
 * over CTAs of the F units, the G epilogue and the I units, then the SM clock
 * in kHz, ring_slots = the
 * U and M ring slots of the plan.  Returns the number of blocks or -WF_ERR_*. */
int wf_fused_instrument_read(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts,
                             unsigned long long* events, int n_events, unsigned long long* role_cycles,
                             int* ring_slots);

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
