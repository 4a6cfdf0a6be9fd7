/* winofuse_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the parity tests, the
 * driver smoke check and bench.py's CPU baseline compare the sm_100a kernels
 * against; the product never links or calls it.
 *
 * It restates, in plain C, the reference's numba kernels and engines
 * (/root/reference/pkg/src/winofuse):
 *   oracle_direct_conv        <- kernels.direct_conv        (kernels.py:22-49)
 *   oracle_forward_tiles      <- kernels.forward_tiles      (kernels.py:52-100)
 *   oracle_inverse_tiles      <- kernels.inverse_tiles      (kernels.py:103-141)
 *   oracle_matmul_rows        <- kernels.matmul_rows        (kernels.py:144-166)
 *   oracle_multiply_positions <- kernels.multiply_positions (kernels.py:169-195)
 *   oracle_conv_fused         <- engines.conv_fused task loop (engines.py:317-444)
 *   oracle_conv_three_stage   <- engines.conv_three_stage   (engines.py:234-314)
 * with the same float32 contract (kernels.py:1-11): channel reductions in
 * ascending order, no FMA contraction (build with -ffp-contract=off), every
 * output stored once.  The transform matrices are inputs (bt32 T x T, at32
 * (T-K+1) x T, the reference's WinogradBasis.bt32 / at32).  Pinned against the
 * reference's own outputs by tests/test_oracle.py (tests/golden/).
 *
 * Build: make -C oracle   (-> oracle/liboracle.so, OpenMP worker pool)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int batch, c_in, c_out, height, width, kernel, pad_lo, pad_hi;
} oracle_layer;

static int out_h(const oracle_layer* L) { return L->height + L->pad_lo + L->pad_hi - L->kernel + 1; }
static int out_w(const oracle_layer* L) { return L->width + L->pad_lo + L->pad_hi - L->kernel + 1; }

/* kernels.py:22-49 -- seven loops, f64 accumulation, one f32 store. */
void oracle_direct_conv(const float* inp, const float* ker, float* out, const oracle_layer* L) {
  const int ho = out_h(L), wo = out_w(L), k = L->kernel;
  for (int b = 0; b < L->batch; ++b)
    for (int o = 0; o < L->c_out; ++o)
      for (int y = 0; y < ho; ++y)
        for (int x = 0; x < wo; ++x) {
          double acc = 0.0;
          for (int c = 0; c < L->c_in; ++c)
            for (int ky = 0; ky < k; ++ky) {
              const int yy = y + ky - L->pad_lo;
              if (yy < 0 || yy >= L->height) continue;
              for (int kx = 0; kx < k; ++kx) {
                const int xx = x + kx - L->pad_lo;
                if (xx < 0 || xx >= L->width) continue;
                acc += (double)inp[(((size_t)b * L->c_in + c) * L->height + yy) * L->width + xx] *
                       (double)ker[(((size_t)o * L->c_in + c) * k + ky) * k + kx];
              }
            }
          out[(((size_t)b * L->c_out + o) * ho + y) * wo + x] = (float)acc;
        }
}

/* kernels.py:52-100 -- gather (zero fill) + u = bt @ win @ bt^T for tiles
 * [t0, t1), all channels, into dst[p][row0 + i - t0][c] with dst rows `rows`. */
void oracle_forward_tiles(const float* inp, const float* bt, int t0, int t1, int row0, float* dst,
                          int rows, const oracle_layer* L, int tile) {
  const int t = tile, m = tile - L->kernel + 1;
  const int ty_n = (out_h(L) + m - 1) / m, tx_n = (out_w(L) + m - 1) / m;
  float win[64], tmp[64], u[64];
  for (int i = t0; i < t1; ++i) {
    const int tx = i % tx_n, rest = i / tx_n, ty = rest % ty_n, b = rest / ty_n;
    const int oy = ty * m - L->pad_lo, ox = tx * m - L->pad_lo;
    const int row = row0 + (i - t0);
    for (int c = 0; c < L->c_in; ++c) {
      const float* plane = inp + ((size_t)b * L->c_in + c) * L->height * L->width;
      for (int r = 0; r < t; ++r)
        for (int s = 0; s < t; ++s) {
          const int yy = oy + r, xx = ox + s;
          win[r * t + s] = (yy >= 0 && yy < L->height && xx >= 0 && xx < L->width)
                               ? plane[(size_t)yy * L->width + xx] : 0.0f;
        }
      for (int r = 0; r < t; ++r)
        for (int s = 0; s < t; ++s) {
          float acc = 0.0f;
          for (int q = 0; q < t; ++q) acc += bt[r * t + q] * win[q * t + s];
          tmp[r * t + s] = acc;
        }
      for (int r = 0; r < t; ++r)
        for (int s = 0; s < t; ++s) {
          float acc = 0.0f;
          for (int q = 0; q < t; ++q) acc += tmp[r * t + q] * bt[s * t + q];
          u[r * t + s] = acc;
        }
      for (int p = 0; p < t * t; ++p) dst[((size_t)p * rows + row) * L->c_in + c] = u[p];
    }
  }
}

/* kernels.py:103-141 -- v = at @ m @ at^T, clipped scatter. */
void oracle_inverse_tiles(const float* res, const float* at, int t0, int t1, int row0, int rows,
                          float* out, const oracle_layer* L, int tile) {
  const int t = tile, m = tile - L->kernel + 1, ho = out_h(L), wo = out_w(L);
  const int ty_n = (ho + m - 1) / m, tx_n = (wo + m - 1) / m;
  float mm[64], tmp[64];
  for (int i = t0; i < t1; ++i) {
    const int tx = i % tx_n, rest = i / tx_n, ty = rest % ty_n, b = rest / ty_n;
    const int oy = ty * m, ox = tx * m;
    const int ny = m < ho - oy ? m : ho - oy, nx = m < wo - ox ? m : wo - ox;
    const int row = row0 + (i - t0);
    for (int o = 0; o < L->c_out; ++o) {
      for (int p = 0; p < t * t; ++p) mm[p] = res[((size_t)p * rows + row) * L->c_out + o];
      for (int r = 0; r < m; ++r)
        for (int s = 0; s < t; ++s) {
          float acc = 0.0f;
          for (int q = 0; q < t; ++q) acc += at[r * t + q] * mm[q * t + s];
          tmp[r * t + s] = acc;
        }
      float* plane = out + ((size_t)b * L->c_out + o) * ho * wo;
      for (int r = 0; r < ny; ++r)
        for (int s = 0; s < nx; ++s) {
          float acc = 0.0f;
          for (int q = 0; q < t; ++q) acc += tmp[r * t + q] * at[s * t + q];
          plane[(size_t)(oy + r) * wo + ox + s] = acc;
        }
    }
  }
}

/* kernels.py:144-166 -- dst[r] = lhs[r] @ rhs, ascending k, f32. */
void oracle_matmul_rows(const float* lhs, const float* rhs, float* dst, int m_rows, int n_c, int n) {
  float stack_acc[1024];
  float* acc = n <= 1024 ? stack_acc : (float*)malloc(sizeof(float) * (size_t)n);
  for (int r = 0; r < m_rows; ++r) {
    for (int j = 0; j < n; ++j) acc[j] = 0.0f;
    for (int c = 0; c < n_c; ++c) {
      const float a = lhs[(size_t)r * n_c + c];
      for (int j = 0; j < n; ++j) acc[j] += a * rhs[(size_t)c * n + j];
    }
    for (int j = 0; j < n; ++j) dst[(size_t)r * n + j] = acc[j];
  }
  if (acc != stack_acc) free(acc);
}

/* kernels.py:169-195 -- res[p] = left[p] @ pack[p] for the first r_eff rows. */
void oracle_multiply_positions(const float* left, const float* pack, float* res, int n_pos, int rows,
                               int r_eff, int n_c, int n) {
  for (int p = 0; p < n_pos; ++p)
    oracle_matmul_rows(left + (size_t)p * rows * n_c, pack + (size_t)p * n_c * n,
                       res + (size_t)p * rows * n, r_eff, n_c, n);
}

/* engines.py:317-444 -- fused engine: tasks of r consecutive tiles, each
 * forward -> multiply -> inverse in a private scratch; tasks are handed out
 * by an OpenMP dynamic schedule (the reference's locked cursor).  Outputs
 * are bit-identical for any thread count (disjoint output tiles). */
int oracle_conv_fused(const float* inp, const float* pack, float* out, const float* bt,
                      const float* at, const oracle_layer* L, int tile, int r, int threads) {
  const int m = tile - L->kernel + 1;
  const int ty_n = (out_h(L) + m - 1) / m, tx_n = (out_w(L) + m - 1) / m;
  const int n_tile = L->batch * ty_n * tx_n, n_task = (n_tile + r - 1) / r, t2 = tile * tile;
  if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    float* left = (float*)malloc(sizeof(float) * (size_t)t2 * r * L->c_in);
    float* res = (float*)malloc(sizeof(float) * (size_t)t2 * r * L->c_out);
#pragma omp for schedule(dynamic, 1)
    for (int task = 0; task < n_task; ++task) {
      const int lo = task * r, hi = lo + r < n_tile ? lo + r : n_tile;
      oracle_forward_tiles(inp, bt, lo, hi, 0, left, r, L, tile);
      oracle_multiply_positions(left, pack, res, t2, r, hi - lo, L->c_in, L->c_out);
      oracle_inverse_tiles(res, at, lo, hi, 0, r, out, L, tile);
    }
    free(left);
    free(res);
  }
  return n_task;
}

/* engines.py:234-314 -- staged engine with full-size intermediates. */
int oracle_conv_three_stage(const float* inp, const float* pack, float* out, const float* bt,
                            const float* at, const oracle_layer* L, int tile, int threads) {
  const int m = tile - L->kernel + 1;
  const int ty_n = (out_h(L) + m - 1) / m, tx_n = (out_w(L) + m - 1) / m;
  const int n_tile = L->batch * ty_n * tx_n, t2 = tile * tile;
  float* lhs = (float*)malloc(sizeof(float) * (size_t)t2 * n_tile * L->c_in);
  float* res = (float*)malloc(sizeof(float) * (size_t)t2 * n_tile * L->c_out);
  if (!lhs || !res) {
    free(lhs);
    free(res);
    return -1;
  }
  if (threads < 1) threads = 1;
  const int chunk = (n_tile + threads - 1) / threads;
#pragma omp parallel for num_threads(threads) schedule(static, 1)
  for (int w = 0; w < threads; ++w) {
    const int a = w * chunk, b = a + chunk < n_tile ? a + chunk : n_tile;
    if (a < b) oracle_forward_tiles(inp, bt, a, b, a, lhs, n_tile, L, tile);
  }
  for (int p = 0; p < t2; ++p) {
#pragma omp parallel for num_threads(threads) schedule(static, 1)
    for (int w = 0; w < threads; ++w) {
      const int a = w * chunk, b = a + chunk < n_tile ? a + chunk : n_tile;
      if (a < b)
        oracle_matmul_rows(lhs + ((size_t)p * n_tile + a) * L->c_in, pack + (size_t)p * L->c_in * L->c_out,
                           res + ((size_t)p * n_tile + a) * L->c_out, b - a, L->c_in, L->c_out);
    }
  }
#pragma omp parallel for num_threads(threads) schedule(static, 1)
  for (int w = 0; w < threads; ++w) {
    const int a = w * chunk, b = a + chunk < n_tile ? a + chunk : n_tile;
    if (a < b) oracle_inverse_tiles(res, at, a, b, a, n_tile, out, L, tile);
  }
  free(lhs);
  free(res);
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
