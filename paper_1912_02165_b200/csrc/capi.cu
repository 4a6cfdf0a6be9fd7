// capi.cu -- the extern "C" boundary (include/winofuse_b200.h) plus the small
// utility kernels: device filter transform, MMA pack, FP64 direct
// convolution and the reference-layout stage kernels.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <cuda_bf16.h>
#include "../../include/winofuse_b200.h"
#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"
#include "fused.cuh"

namespace wf {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

int tuning_knob(const char* name, int dflt);

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t set_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({kernel, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{kernel, dev}] = bytes;
  return e;
}

bool coresident_fits(const void* kernel, int grid, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return false;
  if (set_smem_attr(kernel, static_cast<int>(smem)) != cudaSuccess) return false;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) return false;
  if (tuning_knob("WF_DEBUG_LAUNCH", 0))
    fprintf(stderr, "[wf] coresident: grid %d threads %d smem %zu -> %d CTAs/SM x %d SMs\n", grid, threads, smem,
            per_sm, sms);
  return per_sm * sms >= grid;
}

cudaError_t launch_coresident(const void* kernel, int grid, int threads, size_t smem, cudaStream_t st, void** args) {
  if (!coresident_fits(kernel, grid, threads, smem)) return cudaErrorCooperativeLaunchTooLarge;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelExC(&cfg, kernel, args);
}

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(WF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int tuning_knob(const char* name, int dflt) {
  static std::mutex mu;
  static std::map<std::string, int> cache;   // name -> value (dflt when unset)
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(name);
  if (it != cache.end()) return it->second;
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  cache[name] = v;
  return v;
}

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cache[64] = {0};
  if (dev < 64 && cache[dev]) return cache[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cache[dev] = n;
  return n;
}

// Validate (layer, tile, transform) and fill the geometry.  Mirrors the
// reference checks: LayerSpec (tensor.py:54-64), EngineConfig tile range
// (engines.py:66-68), tile > kernel (tiling.py:66-70).
static int make_geo(const wf_layer* L, int tile, int transform, Geo& g) {
  if (!L) return fail(WF_ERR_PARAM, "layer is NULL");
  if (L->batch < 1 || L->in_channels < 1 || L->out_channels < 1 || L->height < 1 || L->width < 1 ||
      L->kernel < 1 || L->pad_lo < 0 || L->pad_hi < 0)
    return fail(WF_ERR_SHAPE, "invalid layer dimensions");
  if (L->height + L->pad_lo + L->pad_hi < L->kernel || L->width + L->pad_lo + L->pad_hi < L->kernel)
    return fail(WF_ERR_SHAPE, "padded input smaller than kernel");
  if (transform == WF_WINOGRAD) {
    if (tile < 4 || tile > 8) return fail(WF_ERR_PARAM, "tile side must be in [4, 8], got %d", tile);
    if (L->kernel != 3)
      return fail(WF_ERR_UNSUPPORTED, "sm_100a Winograd kernels implement K=3 only (got K=%d)", L->kernel);
  } else if (transform == WF_FFT16) {
    if (tile != 16) return fail(WF_ERR_PARAM, "the FFT transform uses tile 16, got %d", tile);
    if (L->kernel != 3) return fail(WF_ERR_UNSUPPORTED, "FFT-16 kernels implement K=3 only (got K=%d)", L->kernel);
  } else {
    return fail(WF_ERR_PARAM, "unknown transform %d", transform);
  }
  g.B = L->batch; g.C = L->in_channels; g.Cp = L->out_channels;
  g.H = L->height; g.W = L->width; g.pad_lo = L->pad_lo;
  g.T = tile; g.m = tile - L->kernel + 1;
  g.Ho = L->height + L->pad_lo + L->pad_hi - L->kernel + 1;
  g.Wo = L->width + L->pad_lo + L->pad_hi - L->kernel + 1;
  g.tiles_y = ceil_div(g.Ho, g.m);
  g.tiles_x = ceil_div(g.Wo, g.m);
  const long long nt = 1LL * g.B * g.tiles_y * g.tiles_x;
  if (nt > (1LL << 30)) return fail(WF_ERR_UNSUPPORTED, "layer too large (%lld tiles)", nt);
  g.n_tile = static_cast<int>(nt);
  g.fft = transform == WF_FFT16 ? 1 : 0;
  g.Cpad = round_up(g.fft ? 2 * g.C : g.C, 16);
  g.Cppad = round_up(g.fft ? 2 * g.Cp : g.Cp, 16);
  g.P = g.fft ? 16 * 9 : g.T * g.T;
  g.Nout = g.fft ? 2 * g.Cp : g.Cp;
  g.n_blk = ceil_div(g.n_tile, kBlockTiles);
  g.cplx = g.fft && fft_cplx_pack(g.C, g.Cp) ? 1 : 0;
  return WF_OK;
}

// Tensor-core passes of a precision mode (0 = unknown mode).
static int precision_passes(int precision) {
  switch (precision) {
    case WF_PREC_3XBF16: return 3;
    case WF_PREC_BF16: return 1;
    case WF_PREC_3XFP16: return 3 | kPrecF16;
  }
  return 0;
}

int make_geo_public(const wf_layer* L, int tile, int transform, Geo& g) {
  return make_geo(L, tile, transform, g);
}

// -------------------------------------------------------- filter transform
// pack[p][c][c'] = f32( sum G[r][a] w[c'][c][a][b] G[s][b] ), f64 arithmetic,
// one rounding (reference transforms.py:63-80).
template <int T>
__global__ void filter_transform_kernel(const float* __restrict__ w, float* __restrict__ pack,
                                        int C, int Cp) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= C * Cp) return;
  const int cp = idx / C, c = idx - cp * C;
  const float* k = w + (static_cast<size_t>(cp) * C + c) * 9;
  double tmp[T][3];
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) acc = __dadd_rn(acc, __dmul_rn(gd<T>(r, a), static_cast<double>(k[a * 3 + b])));
      tmp[r][b] = acc;
    }
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) acc = __dadd_rn(acc, __dmul_rn(tmp[r][b], gd<T>(s, b)));
      pack[(static_cast<size_t>(r * T + s) * C + c) * Cp + cp] = static_cast<float>(acc);
    }
}

// ----------------------------------------------------------------- MMA pack
// V slab (p, hl): rows = c' (Cppad), K = c (Cpad), bf16 hi/lo split of the f32 pack.
struct PosScale {
  float v[64];   // per-position factor of the V operand (3xfp16 balancing, common.cuh)
};
__global__ void mma_pack_kernel(const float* __restrict__ pack, uint8_t* __restrict__ out, int P,
                                int C, int Cp, int Cpad, int Cppad, int f16, PosScale sc, int cplx) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long per_p = static_cast<long long>(Cppad) * (Cpad / 2);
  if (idx >= per_p * P) return;
  const int p = static_cast<int>(idx / per_p);
  const long long rem = idx - p * per_p;
  const int n = static_cast<int>(rem / (Cpad / 2));
  const int c = static_cast<int>(rem - static_cast<long long>(n) * (Cpad / 2)) * 2;
  float a = 0.0f, b = 0.0f;
  if (cplx) {
    // W[n][k] for output column n < C'/2 of the real expansion P (2C x C'
    // here, C and Cp being 2C_in and 2C'_out): P[k][n] for the Re inputs
    // (k < C/2), -P[k][n] (= +Im V) for the Im inputs
    const int half = C / 2;
    if (n < Cp / 2) {
      if (c < C) a = pack[(static_cast<size_t>(p) * C + c) * Cp + n] * (c < half ? 1.0f : -1.0f);
      if (c + 1 < C) b = pack[(static_cast<size_t>(p) * C + c + 1) * Cp + n] * (c + 1 < half ? 1.0f : -1.0f);
    }
  } else if (n < Cp) {
    if (c < C) a = pack[(static_cast<size_t>(p) * C + c) * Cp + n];
    if (c + 1 < C) b = pack[(static_cast<size_t>(p) * C + c + 1) * Cp + n];
  }
  uint32_t hi, lo;
  if (f16) {
    const float f = p < 64 ? sc.v[p] : 1.0f;
    split_f16x2(a * f, b * f, hi, lo);
  }
  else split_bf16x2(a, b, hi, lo);
  const size_t slab = static_cast<size_t>(Cppad) * Cpad * 2;
  uint8_t* base = out + static_cast<size_t>(p) * 2 * slab + slab_off(n, c, Cppad, Cpad);
  *reinterpret_cast<uint32_t*>(base) = hi;
  *reinterpret_cast<uint32_t*>(base + slab) = lo;
}

// --------------------------------------------------------- direct (FP64)
__global__ void direct_conv_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                   float* __restrict__ y, wf_layer L, int Ho, int Wo) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = 1LL * L.batch * L.out_channels * Ho * Wo;
  if (idx >= total) return;
  const int xo = static_cast<int>(idx % Wo);
  long long r = idx / Wo;
  const int yo = static_cast<int>(r % Ho);
  r /= Ho;
  const int cp = static_cast<int>(r % L.out_channels);
  const int b = static_cast<int>(r / L.out_channels);
  const int K = L.kernel;
  double acc = 0.0;
  for (int c = 0; c < L.in_channels; ++c) {
    const float* plane = x + (static_cast<size_t>(b) * L.in_channels + c) * L.height * L.width;
    const float* ker = w + (static_cast<size_t>(cp) * L.in_channels + c) * K * K;
    for (int ky = 0; ky < K; ++ky) {
      const int yy = yo + ky - L.pad_lo;
      if (yy < 0 || yy >= L.height) continue;
      for (int kx = 0; kx < K; ++kx) {
        const int xx = xo + kx - L.pad_lo;
        if (xx < 0 || xx >= L.width) continue;
        // separate multiply and add (no DFMA): the reference's numba loop
        // accumulates exactly like this (kernels.py:47-48, fastmath off)
        acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(plane[static_cast<size_t>(yy) * L.width + xx]),
                                       static_cast<double>(ker[ky * K + kx])));
      }
    }
  }
  y[idx] = static_cast<float>(acc);
}

// ------------------------------------------- reference-layout stage kernels
// forward_tiles (kernels.py:52-100): dst[p][row0 + i - t0][c] f32.
template <int T>
__global__ void forward_tiles_kernel(const float* __restrict__ x, float* __restrict__ dst, Geo g,
                                     int t0, int t1, int row0, int dst_rows) {
  const int i = t0 + blockIdx.x * blockDim.y + threadIdx.y;
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= t1 || c >= g.C) return;
  int b, ty, tx;
  tile_coords(g, i, b, ty, tx);
  float w[T][T], u[T][T];
  load_window<T>(x + (static_cast<size_t>(b) * g.C + c) * g.H * g.W, g.H, g.W, ty * g.m - g.pad_lo,
                 tx * g.m - g.pad_lo, w);
  forward_transform<T>(w, u);
  const int row = row0 + (i - t0);
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s)
      dst[(static_cast<size_t>(r * T + s) * dst_rows + row) * g.C + c] = u[r][s];
}

// multiply_positions (kernels.py:169-195): res[p][r][:] = left[p][r][:] @ pack[p]
// in f32, ascending c.  Utility path (CUDA cores); the engines use tcgen05.
__global__ void multiply_positions_kernel(const float* __restrict__ left, const float* __restrict__ pack,
                                          float* __restrict__ res, int rows, int r_eff, int C, int Cp) {
  const int p = blockIdx.z;
  const int r = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r_eff || j >= Cp) return;
  const float* a = left + (static_cast<size_t>(p) * rows + r) * C;
  const float* bcol = pack + static_cast<size_t>(p) * C * Cp + j;
  float acc = 0.0f;
  for (int c = 0; c < C; ++c) acc = __fadd_rn(acc, __fmul_rn(a[c], bcol[static_cast<size_t>(c) * Cp]));
  res[(static_cast<size_t>(p) * rows + r) * Cp + j] = acc;
}

// inverse_tiles (kernels.py:103-141): res[p][row0 + i - t0][c'] -> y.
template <int T>
__global__ void inverse_tiles_kernel(const float* __restrict__ res, float* __restrict__ y, Geo g, int t0,
                                     int t1, int row0, int res_rows) {
  const int i = t0 + blockIdx.x * blockDim.y + threadIdx.y;
  const int cp = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= t1 || cp >= g.Cp) return;
  const int row = row0 + (i - t0);
  float mm[T][T];
#pragma unroll
  for (int r = 0; r < T; ++r)
#pragma unroll
    for (int s = 0; s < T; ++s) mm[r][s] = res[(static_cast<size_t>(r * T + s) * res_rows + row) * g.Cp + cp];
  float out[T - 2][T - 2];
  inverse_transform<T>(mm, out);
  int b, ty, tx;
  tile_coords(g, i, b, ty, tx);
  const int oy = ty * g.m, ox = tx * g.m;
  float* plane = y + (static_cast<size_t>(b) * g.Cp + cp) * g.Ho * g.Wo;
  for (int r = 0; r < T - 2 && oy + r < g.Ho; ++r)
    for (int s = 0; s < T - 2 && ox + s < g.Wo; ++s) plane[static_cast<size_t>(oy + r) * g.Wo + ox + s] = out[r][s];
}

}  // namespace wf

using namespace wf;

#define WF_TDISPATCH(T_, CALL)        \
  switch (T_) {                      \
    case 4: { constexpr int TT = 4; CALL; } break; \
    case 5: { constexpr int TT = 5; CALL; } break; \
    case 6: { constexpr int TT = 6; CALL; } break; \
    case 7: { constexpr int TT = 7; CALL; } break; \
    case 8: { constexpr int TT = 8; CALL; } break; \
    default: return fail(WF_ERR_PARAM, "tile %d", T_); \
  }

extern "C" {

int wf_version(void) { return 100; }

const char* wf_last_error(void) { return g_last_error.c_str(); }

int wf_device_sm_count(void) { return sm_count(); }

unsigned long long wf_kernel_launches(void) { return wf::g_launches.load(); }

int wf_filter_transform(const float* w, float* pack, int c_in, int c_out, int tile, void* stream) {
  if (!w || !pack) return fail(WF_ERR_PARAM, "null pointer");
  if (c_in < 1 || c_out < 1) return fail(WF_ERR_SHAPE, "channels must be >= 1");
  if (tile < 4 || tile > 8) return fail(WF_ERR_PARAM, "tile side must be in [4, 8], got %d", tile);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n = c_in * c_out;
  note_launch();
  WF_TDISPATCH(tile, (filter_transform_kernel<TT><<<ceil_div(n, 128), 128, 0, st>>>(w, pack, c_in, c_out)));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "filter_transform");
}

size_t wf_mma_pack_bytes(int tile, int c_in, int c_out, int transform) {
  if (c_in < 1 || c_out < 1) return 0;
  if (transform == WF_FFT16 && tile == 16) {  // 144 bins, real-expanded (2C x 2C') complex GEMM
    if (fft_cplx_pack(c_in, c_out))           // or [Re V^T | Im V^T] (C' x 2C) per bin
      return static_cast<size_t>(144) * 2 * round_up(c_out, 16) * round_up(2 * c_in, 16) * 2;
    return static_cast<size_t>(144) * 2 * round_up(2 * c_out, 16) * round_up(2 * c_in, 16) * 2;
  }
  if (transform != WF_WINOGRAD || tile < 4 || tile > 8) return 0;
  return static_cast<size_t>(tile) * tile * 2 * round_up(c_out, 16) * round_up(c_in, 16) * 2;
}

int wf_mma_pack(const float* pack, void* mma_pack, int tile, int c_in, int c_out, int transform,
                void* stream) {
  return wf_mma_pack_ex(pack, mma_pack, tile, c_in, c_out, transform, WF_PREC_3XBF16, stream);
}

int wf_mma_pack_ex(const float* pack, void* mma_pack, int tile, int c_in, int c_out, int transform, int precision,
                   void* stream) {
  if (!pack || !mma_pack) return fail(WF_ERR_PARAM, "null pointer");
  if (c_in < 1 || c_out < 1) return fail(WF_ERR_SHAPE, "channels must be >= 1");
  const int prec = precision_passes(precision);
  if (prec == 0) return fail(WF_ERR_PARAM, "precision %d", precision);
  int P;
  int cplx = 0;
  if (transform == WF_FFT16) {
    // pack holds the real expansion (144, 2C, 2C') of the complex bins
    if (tile != 16) return fail(WF_ERR_PARAM, "the FFT transform uses tile 16, got %d", tile);
    P = 144;
    cplx = fft_cplx_pack(c_in, c_out) ? 1 : 0;
    c_in *= 2;
    c_out *= 2;
  } else if (transform == WF_WINOGRAD) {
    if (tile < 4 || tile > 8) return fail(WF_ERR_PARAM, "tile side must be in [4, 8], got %d", tile);
    P = tile * tile;
  } else {
    return fail(WF_ERR_PARAM, "unknown transform %d", transform);
  }
  const int Cpad = round_up(c_in, 16), Cppad = cplx ? round_up(c_out / 2, 16) : round_up(c_out, 16);
  const long long total = 1LL * P * Cppad * (Cpad / 2);
  // 3xfp16: V' = V / u_scale(r, s) so that U' V' == U V (common.cuh f16_u_scale)
  PosScale sc;
  for (int p = 0; p < 64; ++p) sc.v[p] = 1.0f;
  if (prec_f16(prec) && transform == WF_WINOGRAD) {
    for (int p = 0; p < P; ++p) {
      const int r = p / tile, s = p % tile;
      float u = 1.0f;
      switch (tile) {
        case 4: u = f16_u_scale<4>(r, s); break;
        case 5: u = f16_u_scale<5>(r, s); break;
        case 6: u = f16_u_scale<6>(r, s); break;
        case 7: u = f16_u_scale<7>(r, s); break;
        case 8: u = f16_u_scale<8>(r, s); break;
      }
      sc.v[p] = 1.0f / u;
    }
  }
  note_launch();
  mma_pack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pack, static_cast<uint8_t*>(mma_pack), P, c_in, c_out, Cpad, Cppad, prec_f16(prec) ? 1 : 0, sc, cplx);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "mma_pack");
}

size_t wf_three_stage_scratch_bytes(const wf_layer* layer, int tile, int transform) {
  Geo g;
  if (make_geo(layer, tile, transform, g) != WF_OK) return 0;
  const size_t P = static_cast<size_t>(g.P);
  const size_t u = P * g.n_blk * 2 * kBlockTiles * g.Cpad * 2;
  const size_t m = P * g.Nout * static_cast<size_t>(g.n_blk) * kBlockTiles * 4;
  return u + m;
}

int wf_conv_three_stage_phases(const float* x, const void* mma_pack, float* y, void* scratch,
                               size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                               int precision, int phases, void* stream) {
  Geo g;
  int rc = make_geo(layer, tile, transform, g);
  if (rc != WF_OK) return rc;
  if (!scratch) return fail(WF_ERR_PARAM, "null pointer");
  if ((phases & WF_PHASE_FORWARD) && !x) return fail(WF_ERR_PARAM, "null pointer");
  if ((phases & WF_PHASE_MULTIPLY) && !mma_pack) return fail(WF_ERR_PARAM, "null pointer");
  if ((phases & WF_PHASE_INVERSE) && !y) return fail(WF_ERR_PARAM, "null pointer");
  if (phases < 1 || phases > 7) return fail(WF_ERR_PARAM, "phases %d", phases);
  const int passes = precision_passes(precision);
  if (passes == 0) return fail(WF_ERR_PARAM, "precision %d", precision);
  const size_t need = wf_three_stage_scratch_bytes(layer, tile, transform);
  if (scratch_bytes < need) return fail(WF_ERR_SCRATCH, "scratch %zu < %zu bytes", scratch_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t P = static_cast<size_t>(g.P);
  uint8_t* U = static_cast<uint8_t*>(scratch);
  float* M = reinterpret_cast<float*>(U + P * g.n_blk * 2 * kBlockTiles * g.Cpad * 2);
  const int ldm = g.n_blk * kBlockTiles;
  cudaError_t e = cudaSuccess;
  if (phases & WF_PHASE_FORWARD) {
    e = launch_forward_slab(x, U, g, 0, g.n_blk, passes, st);
    if (e != cudaSuccess) return cuda_fail(e, "forward");
  }
  if (phases & WF_PHASE_MULTIPLY) {
    e = launch_position_gemm(U, static_cast<const uint8_t*>(mma_pack), M, g, g.n_blk, ldm, g.n_tile, passes,
                             sm_count(), st);
    if (e != cudaSuccess) return cuda_fail(e, "gemm");
  }
  if (phases & WF_PHASE_INVERSE) {
    e = launch_inverse(M, y, g, 0, g.n_tile, ldm, st);
    if (e != cudaSuccess) return cuda_fail(e, "inverse");
  }
  return WF_OK;
}

int wf_conv_three_stage(const float* x, const void* mma_pack, float* y, void* scratch,
                        size_t scratch_bytes, const wf_layer* layer, int tile, int transform,
                        int precision, void* stream) {
  return wf_conv_three_stage_phases(x, mma_pack, y, scratch, scratch_bytes, layer, tile, transform, precision,
                                    WF_PHASE_FORWARD | WF_PHASE_MULTIPLY | WF_PHASE_INVERSE, stream);
}

static int fused_opts(const wf_fused_opts* in, FusedOpts& o) {
  o = FusedOpts();
  if (!in) return WF_OK;
  if (in->variant < WF_FUSED_AUTO || in->variant > WF_FUSED_WS_ROW) return fail(WF_ERR_PARAM, "variant %d", in->variant);
  if (in->flags & ~(WF_FUSED_COUNTERS_CLEAN | WF_FUSED_INSTRUMENT)) return fail(WF_ERR_PARAM, "flags %d", in->flags);
  if (in->lag < 0 || in->gbatch < 0) return fail(WF_ERR_PARAM, "negative lag / gbatch");
  o.variant = in->variant;
  o.flags = in->flags;
  o.ring_bytes = in->ring_bytes;
  o.lag = in->lag;
  o.gbatch = in->gbatch;
  return WF_OK;
}

size_t wf_fused_scratch_bytes(const wf_layer* layer, int tile, int transform, int r) {
  (void)r;
  return wf_fused_scratch_bytes_ex(layer, tile, transform, nullptr);
}

size_t wf_fused_scratch_bytes_ex(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts) {
  Geo g;
  FusedOpts o;
  if (make_geo(layer, tile, transform, g) != WF_OK || fused_opts(opts, o) != WF_OK) return 0;
  if (fused_pick_variant(g, o) == 0) return 0;
  return fused_scratch_bytes(g, o);
}

int wf_fused_variant(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts) {
  Geo g;
  FusedOpts o;
  int rc = make_geo(layer, tile, transform, g);
  if (rc != WF_OK) return -rc;
  rc = fused_opts(opts, o);
  if (rc != WF_OK) return -rc;
  const int v = fused_pick_variant(g, o);
  if (v == 0) return -fail(WF_ERR_UNSUPPORTED, "fused variant %d cannot run this layer", o.variant);
  return v;
}

int wf_conv_fused_ex(const float* x, const void* mma_pack, float* y, void* scratch, size_t scratch_bytes,
                     const wf_layer* layer, int tile, int transform, int precision, const wf_fused_opts* opts,
                     int* variant_ran, void* stream) {
  Geo g;
  FusedOpts o;
  int rc = make_geo(layer, tile, transform, g);
  if (rc != WF_OK) return rc;
  rc = fused_opts(opts, o);
  if (rc != WF_OK) return rc;
  if (!x || !mma_pack || !y) return fail(WF_ERR_PARAM, "null pointer");
  const int passes = precision_passes(precision);
  if (passes == 0) return fail(WF_ERR_PARAM, "precision %d", precision);
  if (fused_pick_variant(g, o) == 0)
    return fail(WF_ERR_UNSUPPORTED, "fused variant %d cannot run this layer", o.variant);
  if ((o.flags & WF_FUSED_INSTRUMENT) && fused_pick_variant(g, o) != kVarWS && fused_pick_variant(g, o) != kVarWSRow)
    return fail(WF_ERR_UNSUPPORTED, "instrumentation is implemented by the warp-specialised variant only");
  const size_t need = fused_scratch_bytes(g, o);
  if (need && (!scratch || scratch_bytes < need))
    return fail(WF_ERR_SCRATCH, "scratch %zu < %zu bytes", scratch_bytes, need);
  int ran = 0;
  cudaError_t e = run_fused(x, static_cast<const uint8_t*>(mma_pack), y, static_cast<uint8_t*>(scratch), g, passes,
                            sm_count(), static_cast<cudaStream_t>(stream), o, &ran);
  if (variant_ran) *variant_ran = ran;
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "fused");
}

int wf_conv_fused(const float* x, const void* mma_pack, float* y, void* scratch, size_t scratch_bytes,
                  const wf_layer* layer, int tile, int transform, int precision, int r, void* stream) {
  if (r < 0) return fail(WF_ERR_PARAM, "tiles per task (r) must be >= 0");
  return wf_conv_fused_ex(x, mma_pack, y, scratch, scratch_bytes, layer, tile, transform, precision, nullptr, nullptr,
                          stream);
}

int wf_conv_fused_planned(const float* x, const void* mma_pack, float* y, void* scratch, size_t scratch_bytes,
                          const wf_layer* layer, int tile, int transform, int precision, int flags, void* stream) {
  if (flags & ~WF_FUSED_COUNTERS_CLEAN) return fail(WF_ERR_PARAM, "flags %d", flags);
  wf_fused_opts o = {};
  o.flags = flags;
  return wf_conv_fused_ex(x, mma_pack, y, scratch, scratch_bytes, layer, tile, transform, precision, &o, nullptr,
                          stream);
}

int wf_fused_instrument_read(const wf_layer* layer, int tile, int transform, const wf_fused_opts* opts,
                             unsigned long long* events, int n_events, unsigned long long* role_cycles,
                             int* ring_slots) {
  Geo g;
  FusedOpts o;
  int rc = make_geo(layer, tile, transform, g);
  if (rc != WF_OK) return -rc;
  rc = fused_opts(opts, o);
  if (rc != WF_OK) return -rc;
  if (!events || !role_cycles || !ring_slots) return -fail(WF_ERR_PARAM, "null pointer");
  if (cudaDeviceSynchronize() != cudaSuccess) return -fail(WF_ERR_CUDA, "synchronize");
  const int n = ws_instrument_read(g, o, events, n_events, role_cycles, ring_slots);
  if (n < 0) return -fail(WF_ERR_UNSUPPORTED, "no instrumented warp-specialised plan for this layer");
  return n;
}

int wf_conv_direct(const float* x, const float* w, float* y, const wf_layer* layer, void* stream) {
  if (!layer || !x || !w || !y) return fail(WF_ERR_PARAM, "null pointer");
  const wf_layer L = *layer;
  if (L.batch < 1 || L.in_channels < 1 || L.out_channels < 1 || L.height < 1 || L.width < 1 || L.kernel < 1 ||
      L.pad_lo < 0 || L.pad_hi < 0)
    return fail(WF_ERR_SHAPE, "invalid layer dimensions");
  const int Ho = L.height + L.pad_lo + L.pad_hi - L.kernel + 1;
  const int Wo = L.width + L.pad_lo + L.pad_hi - L.kernel + 1;
  if (Ho < 1 || Wo < 1) return fail(WF_ERR_SHAPE, "padded input smaller than kernel");
  const long long total = 1LL * L.batch * L.out_channels * Ho * Wo;
  note_launch();
  direct_conv_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, w, y, L, Ho, Wo);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "direct_conv");
}

int wf_forward_tiles(const float* x, float* dst, const wf_layer* layer, int tile, int t0, int t1, int row0,
                     int dst_rows, void* stream) {
  Geo g;
  int rc = make_geo(layer, tile, WF_WINOGRAD, g);
  if (rc != WF_OK) return rc;
  if (!x || !dst) return fail(WF_ERR_PARAM, "null pointer");
  if (t0 < 0 || t1 > g.n_tile || t0 >= t1) return fail(WF_ERR_SHAPE, "tile range [%d, %d) invalid", t0, t1);
  if (row0 < 0 || row0 + (t1 - t0) > dst_rows) return fail(WF_ERR_SHAPE, "destination rows too small");
  dim3 blk(32, 4), grid(ceil_div(t1 - t0, 4), ceil_div(g.C, 32));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  note_launch();
  WF_TDISPATCH(tile, (forward_tiles_kernel<TT><<<grid, blk, 0, st>>>(x, dst, g, t0, t1, row0, dst_rows)));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "forward_tiles");
}

int wf_multiply_positions(const float* left, const float* pack, float* res, int positions, int rows, int r_eff,
                          int c_in, int c_out, void* stream) {
  if (!left || !pack || !res) return fail(WF_ERR_PARAM, "null pointer");
  if (positions < 1 || rows < 1 || c_in < 1 || c_out < 1 || r_eff < 0 || r_eff > rows)
    return fail(WF_ERR_SHAPE, "bad multiply shape");
  if (r_eff == 0) return WF_OK;
  dim3 grid(ceil_div(c_out, 128), r_eff, positions);
  note_launch();
  multiply_positions_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(left, pack, res, rows, r_eff,
                                                                                 c_in, c_out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "multiply_positions");
}

int wf_inverse_tiles(const float* res, float* y, const wf_layer* layer, int tile, int t0, int t1, int row0,
                     int res_rows, void* stream) {
  Geo g;
  int rc = make_geo(layer, tile, WF_WINOGRAD, g);
  if (rc != WF_OK) return rc;
  if (!res || !y) return fail(WF_ERR_PARAM, "null pointer");
  if (t0 < 0 || t1 > g.n_tile || t0 >= t1) return fail(WF_ERR_SHAPE, "tile range [%d, %d) invalid", t0, t1);
  if (row0 < 0 || row0 + (t1 - t0) > res_rows) return fail(WF_ERR_SHAPE, "result rows too small");
  dim3 blk(32, 4), grid(ceil_div(t1 - t0, 4), ceil_div(g.Cp, 32));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  note_launch();
  WF_TDISPATCH(tile, (inverse_tiles_kernel<TT><<<grid, blk, 0, st>>>(res, y, g, t0, t1, row0, res_rows)));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WF_OK : cuda_fail(e, "inverse_tiles");
}

}  // extern "C"
