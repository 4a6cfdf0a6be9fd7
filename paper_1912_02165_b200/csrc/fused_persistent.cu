// fused_persistent.cu -- conv_fused as ONE persistent dataflow kernel.
//
// The reference's fused engine (engines.py:317-444) hands tasks of R tiles
// to worker threads from a locked cursor; each task runs forward ->
// multiply -> inverse while its transformed tiles stay in cache.  Here one
// CTA per SM pulls work items from a global atomic queue.  Three item kinds
// per 128-tile block b:
//   F(b, cg)  forward transform of CPC channels -> U ring slot (bf16 hi/lo
//             UMMA slabs); input rows staged in smem with cp.async zero-fill
//   G(b, gg)  tcgen05 GEMM for GP transform positions: M[p] = U[p] * V[p]
//             (3xBF16, f32 accumulation in TMEM) -> M ring slot (f32)
//   I(b, ig)  inverse transform + clipped store of a group of output channels
// Items are dispensed in a lagged order -- F for block s, G for block s-L1,
// I for block s-L2 at "step" s -- and each item waits (acquire on a
// per-block counter) only on items dispensed earlier, so the queue can
// never deadlock (an unscheduled CTA holds no item).  The rings (U: NU
// slots, M: NM slots) are sized to stay resident in the 126 MB L2, so the
// transformed tiles and products never make an HBM round trip, and all
// three stages of different blocks run concurrently on different SMs with
// no per-stage launch or tail.
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "fused.cuh"
#include "staged.cuh"

namespace wf {

struct PersistParams {
  const float* x;
  float* y;
  const uint8_t* vpack;   // MMA pack: per position hi / lo slabs of Cppad x Cpad
  uint8_t* uring;         // NU slots x T^2 x (hi, lo) x 128 x Cpad bf16
  float* mring;           // NM slots x T^2 x Cp x 128 f32
  int* counters;          // [0] queue head, then doneF, doneG, doneI (n_blk each)
  Geo g;
  int n_cg, n_gg, n_ig;   // items per block of each kind
  int cpc, gp, igc;       // channels per F item, positions per G item, c' per I item
  int ftiles;             // tiles per F item (a 128-tile block is split into 128 / ftiles parts)
  int NU, NM, L1, L2;
  int passes;
  int n_steps, n_items;
  int discard;                 // drop consumed ring lines from L2 (WF_DISCARD=0 disables)
  int split_f;                 // >0: CTAs [0, split_f) run only F items, the rest G and I items
  int only;                    // tuning aid: 1/2/3 = execute only F / G / I items (results invalid)
  int wreg, trows, plane; // F staging geometry
  int f_desc_off, f_max_rows;  // F row-descriptor table (bytes into smem, capacity)
  int stages;                  // G smem pipeline depth
  int f_bulk, f_shift;         // F staging by bulk copies; staged column of x = 0
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Poll with relaxed loads (an acquire load also invalidates the SM's L1 on
// every iteration), then one acquire load once the target is reached.
__device__ __forceinline__ void spin_until(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  while (ld_relaxed_gpu(p) < target) __nanosleep(128);
  (void)ld_acquire(p);
}
// Invalidate one 128-byte L2 line without writing it back (its data is dead).
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Optional per-CTA item accounting (wait / run cycles per item kind) for
// tuning; off unless WF_PROFILE is set.  Read with wf_debug_fused_profile().
constexpr int kProfCtas = 512, kProfSlots = 16;
__device__ unsigned long long g_prof[kProfCtas * kProfSlots];
__constant__ int g_prof_on;
// Optional item trace (WF_PROFILE=2): per item {cta, kind<<24 | block, start ns, end ns}.
constexpr int kTraceMax = 16384;
__device__ unsigned long long g_trace[kTraceMax * 2];
__device__ int g_trace_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// sub-phase marks (thread 0): slot 9 F staging, 10 F transform+store,
// 11 I loads, 12 I transform+smem, 13 I write-back
__device__ __forceinline__ void prof_mark(int slot, long long& t) {
  if (g_prof_on && threadIdx.x == 0) {
    const long long now = clock64();
    g_prof[(blockIdx.x % kProfCtas) * kProfSlots + slot] += now - t;
    t = now;
  }
}

// Items active in step s, and the item -> (step, kind, sub) decode.
__device__ __forceinline__ int items_in_step(const PersistParams& P, int s, int& nf, int& ng) {
  const int nb = P.g.n_blk;
  nf = (s < nb) ? P.n_cg : 0;
  ng = (s >= P.L1 && s - P.L1 < nb) ? P.n_gg : 0;
  const int ni = (s >= P.L2 && s - P.L2 < nb) ? P.n_ig : 0;
  return nf + ng + ni;
}

struct GemmSync {
  uint64_t full[3], empty[3], tfull[8];
  uint64_t fbar;            // F-item staging (bulk copies)
};

// ------------------------------------------------------------------ F item
// Returns whether the staging mbarrier was used (one phase consumed).
template <int T, int NT, int KC, bool F16>
__device__ bool run_forward_item(const PersistParams& P, int b, int cg, uint8_t* smem, GemmSync& sy,
                                 int fparity) {
  const Geo& g = P.g;
  float* xs = reinterpret_cast<float*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int CPC = P.cpc;
  // item cg = (part of the block) x (channel group)
  const int n_cgrp = g.Cpad / CPC;
  const int part = cg / n_cgrp;
  cg -= part * n_cgrp;
  const int tb0 = part * P.ftiles;                 // first tile of this part inside the block
  const int t0 = b * kBlockTiles + tb0;
  const int cbase = cg * CPC;
  const int gr0 = t0 / g.tiles_x;
  const int tlast = min(t0 + P.ftiles, g.n_tile) - 1;
  const int nrows = tlast >= t0 ? tlast / g.tiles_x - gr0 + 1 : 0;
  const int row_elems = T * P.wreg;
  const int total_rows = CPC * nrows * T;
  if (cbase >= g.C) {
    // a channel group made only of K padding (C < Cpad): its U entries are
    // zeros -- no staging, no transform
    const int pairs = CPC / 2, tpw = 32 / pairs;
    const int tl = (warp % (P.ftiles / tpw)) * tpw + lane % tpw;
    const int q = lane / tpw;
    if (warp < P.ftiles / tpw) {
      const size_t slab = static_cast<size_t>(kBlockTiles) * g.Cpad * 2;
      uint8_t* dst = P.uring + static_cast<size_t>(b % P.NU) * T * T * 2 * slab +
                     slab_off(tb0 + tl, cbase + 2 * q, kBlockTiles, g.Cpad);
#pragma unroll 4
      for (int p = 0; p < T * T; ++p) {
        *reinterpret_cast<uint32_t*>(dst + static_cast<size_t>(p) * 2 * slab) = 0u;
        *reinterpret_cast<uint32_t*>(dst + static_cast<size_t>(p) * 2 * slab + slab) = 0u;
      }
    }
    return false;
  }
  long long tprof = 0;
  if (g_prof_on && tid == 0) tprof = clock64();
  if (P.f_bulk) {
    // Rows are 16-byte aligned in global memory (W % 4 == 0) and the T
    // window rows of a tile row are consecutive image rows, i.e. one
    // contiguous global range: ONE bulk async copy per (channel, tile row),
    // landing unpadded (pitch W) in shared memory; rows outside the image
    // are zeroed with plain stores and the left/right padding columns are
    // masked when the windows are read.  All copies complete on one mbarrier.
    fence_proxy_async_smem();
    const int units = CPC * nrows;
    for (int u = tid; u < units; u += NT) {
      const int j = u % nrows;
      const int cl = u / nrows;
      const int gr = gr0 + j;
      const int bi = gr / g.tiles_y, ty = gr - bi * g.tiles_y;
      const int y0 = ty * g.m - g.pad_lo;
      const int ya = max(y0, 0), yb = min(y0 + T, g.H);
      const int c = cbase + cl;
      float* dst = xs + cl * P.plane + j * row_elems;
      const bool ok = c < g.C && bi < g.B && yb > ya;
      if (ok) {
        const uint32_t bytes = static_cast<uint32_t>((yb - ya) * g.W * 4);
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sy.fbar)),
                     "r"(bytes) : "memory");
        bulk_g2s(dst + (ya - y0) * g.W, P.x + ((static_cast<size_t>(bi) * g.C + c) * g.H + ya) * g.W, bytes,
                 &sy.fbar);
      }
      const int z0 = ok ? ya - y0 : 0, z1 = ok ? yb - y0 : 0;   // rows [z0, z1) come from the copy
      for (int r = 0; r < T; ++r)
        if (r < z0 || r >= z1)
          for (int s2 = 0; s2 < g.W; ++s2) dst[r * g.W + s2] = 0.0f;
    }
    // only the warps that issued copies synchronise before the single
    // arrival (the others go straight to the mbarrier wait), so a warp that
    // is still publishing the previous item's completion delays nobody
    const int nw_issue = min(NT / 32, (units + 31) / 32);
    if (warp < nw_issue) {
      if (nw_issue > 1) asm volatile("bar.sync 1, %0;" ::"r"(nw_issue * 32) : "memory");
      if (tid == 0) mbar_arrive(&sy.fbar);
    }
    if (units == 0 && tid == 0) mbar_arrive(&sy.fbar);
    mbar_wait(&sy.fbar, fparity);
  } else {
  // stage input rows (zero padded): one warp per row, lanes along the row
  // (coalesced); ROWS rows per iteration so every thread has several
  // independent loads in flight before it stores to shared memory
  // (1) one descriptor per staged row (global row offset or -1 for a zero
  // row, smem offset): the index divisions happen once per row, in parallel
  long long* rsrc = reinterpret_cast<long long*>(smem + P.f_desc_off);
  int* rdst = reinterpret_cast<int*>(rsrc + P.f_max_rows);
  for (int row = tid; row < total_rows; row += NT) {
    const int r = row % T;
    const int rest = row / T;
    const int j = rest % nrows;
    const int cl = rest / nrows;
    const int gr = gr0 + j;
    const int bi = gr / g.tiles_y, ty = gr - bi * g.tiles_y;
    const int yy = ty * g.m - g.pad_lo + r;
    const int c = cbase + cl;
    const bool rok = c < g.C && yy >= 0 && yy < g.H && bi < g.B;
    rsrc[row] = rok ? ((static_cast<long long>(bi) * g.C + c) * g.H + yy) * g.W : -1;
    rdst[row] = cl * P.plane + j * row_elems + r * P.wreg;
  }
  __syncthreads();
  // (2) one warp per row, lanes along the row (coalesced), ROWS rows per
  // iteration so each thread has several independent loads in flight
  constexpr int ROWS = 4;
  constexpr int NW = NT / 32;
  const int lo_ok = g.pad_lo, hi_ok = g.pad_lo + g.W;       // staged column s holds x = s - pad_lo
  for (int row0 = warp * ROWS; row0 < total_rows; row0 += NW * ROWS) {
    for (int s0 = 0; s0 < P.wreg; s0 += 64) {
      float v[ROWS][2];
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        const int row = row0 + k;
        const long long src = row < total_rows ? rsrc[row] : -1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int s = s0 + lane + 32 * h;
          v[k][h] = (src >= 0 && s >= lo_ok && s < hi_ok) ? __ldg(P.x + src + (s - g.pad_lo)) : 0.0f;
        }
      }
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        const int row = row0 + k;
        if (row >= total_rows) break;
        float* d = xs + rdst[row];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int s = s0 + lane + 32 * h;
          if (s < P.wreg) d[s] = v[k][h];
        }
      }
    }
  }
  }  // staging path
  __syncthreads();
  prof_mark(9, tprof);

  // thread = (tile, channel pair); a warp = 32 / pairs tiles x all pairs, so
  // each store instruction writes whole 16-byte core-matrix rows (CPC = 8)
  const int pairs = CPC / 2;
  const int tpw = 32 / pairs;
  const int nwarps_used = P.ftiles / tpw;
  const int tl = (warp % nwarps_used) * tpw + lane % tpw;   // tile inside the part
  const int q = lane / tpw;
  const int tile = t0 + tl;
  const int c0 = cbase + 2 * q;
  float2 u2[T][T];
  if (P.only == 6) return true;          // tuning aid: staging only
  if (tile < g.n_tile && warp < nwarps_used) {
    const int per_img = g.tiles_y * g.tiles_x;
    const int bi = tile / per_img;
    const int rem = tile - bi * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int j = bi * g.tiles_y + ty - gr0;
    const int x0 = tx * g.m - g.pad_lo;          // image column of window column 0
    const float* pa = xs + j * row_elems + x0 + P.f_shift + (2 * q) * P.plane;
    const float* pb = pa + P.plane;
    float2 w[T][T];
    if constexpr (T == 6) {
      // F(4,3) interior windows start at column 4 tx - 1 of an unpadded,
      // 16-byte aligned row: read columns [4 tx - 4, 4 tx + 4) as two
      // conflict-free 16-byte loads plus one scalar (instead of six scalar
      // loads with 4-way bank conflicts)
      if (P.f_bulk && g.m == 4 && g.pad_lo == 1 && x0 >= 3 && x0 + T <= g.W && (P.wreg & 3) == 0) {
#pragma unroll
        for (int r = 0; r < T; ++r) {
          const float* ra = pa + r * P.wreg - 3;
          const float* rb = pb + r * P.wreg - 3;
          const float4 a0 = *reinterpret_cast<const float4*>(ra), a1 = *reinterpret_cast<const float4*>(ra + 4);
          const float4 b0 = *reinterpret_cast<const float4*>(rb), b1 = *reinterpret_cast<const float4*>(rb + 4);
          w[r][0] = make_float2(a0.w, b0.w);
          w[r][1] = make_float2(a1.x, b1.x);
          w[r][2] = make_float2(a1.y, b1.y);
          w[r][3] = make_float2(a1.z, b1.z);
          w[r][4] = make_float2(a1.w, b1.w);
          w[r][5] = make_float2(ra[8], rb[8]);
        }
        goto have_window;
      }
    }
    if (!P.f_bulk || (x0 >= 0 && x0 + T <= g.W)) {
#pragma unroll
      for (int r = 0; r < T; ++r)
#pragma unroll
        for (int s = 0; s < T; ++s) w[r][s] = make_float2(pa[r * P.wreg + s], pb[r * P.wreg + s]);
    } else {                                      // unpadded staging: mask the border columns
#pragma unroll
      for (int r = 0; r < T; ++r)
#pragma unroll
        for (int s = 0; s < T; ++s) {
          const bool in = x0 + s >= 0 && x0 + s < g.W;
          w[r][s] = in ? make_float2(pa[r * P.wreg + s], pb[r * P.wreg + s]) : make_float2(0.0f, 0.0f);
        }
    }
  have_window:
    forward_transform2<T>(w, u2);     // channels 2q, 2q+1 of the pair (packed f32x2)
  } else {
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) u2[r][s] = make_float2(0.0f, 0.0f);
  }
  if (warp < nwarps_used) {
    const int cpad = KC ? KC : g.Cpad;
    const size_t slab = static_cast<size_t>(kBlockTiles) * cpad * 2;
    uint8_t* slot = P.uring + static_cast<size_t>(b % P.NU) * T * T * 2 * slab;
    uint8_t* dst = slot + slab_off(tb0 + tl, c0, kBlockTiles, cpad);
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) {
        uint32_t hi, lo;
        split2<F16>(u_operand<T, F16>(u2[r][s], r, s), hi, lo);
        uint8_t* p = dst + static_cast<size_t>(r * T + s) * 2 * slab;
        if (P.only == 5) {                 // tuning aid: no stores (keep the values live)
          if ((hi ^ lo) == 0x12345678u) *reinterpret_cast<uint32_t*>(p) = hi;
          continue;
        }
        *reinterpret_cast<uint32_t*>(p) = hi;
        *reinterpret_cast<uint32_t*>(p + slab) = lo;
      }
  }
  prof_mark(10, tprof);
  return true;
}

// ------------------------------------------------------------------ G item
// Pipeline over (position p of the group, K block j): stage = A K-block
// (hi, lo) + V_p K-block (hi, lo).  Accumulator for position p = TMEM
// columns [p_local * Cppad, +Cppad).


// Barrier parities are derived from CTA-uniform counters (every thread keeps
// identical copies): pipeline step K (over all G items of this CTA) uses
// stage K % 3 with parity (K / 3) & 1; accumulator pl has been completed
// tuse[pl] times before this item.
template <int NT, int KC>
__device__ void run_gemm_item(const PersistParams& P, int b, int gg, uint8_t* smem, GemmSync& sy,
                              uint32_t tmem, int gbase, const int (&tuse)[8]) {
  const Geo& g = P.g;
  const int warp = threadIdx.x >> 5;
  const int n_kb = ceil_div(g.Cpad, kKBlock);
  const int p0 = gg * P.gp;
  const int np = min(P.gp, g.T * g.T - p0);
  const uint32_t a_half = kBlockTiles * kKBlock * 2;
  const uint32_t b_half = static_cast<uint32_t>(g.Cppad) * kKBlock * 2;
  const uint32_t stage_bytes = 2 * a_half + 2 * b_half;
  const size_t a_slab = static_cast<size_t>(kBlockTiles) * g.Cpad * 2;
  const size_t v_slab = static_cast<size_t>(g.Cppad) * g.Cpad * 2;
  const uint8_t* uslot = P.uring + static_cast<size_t>(b % P.NU) * g.T * g.T * 2 * a_slab;
  const int n_steps = np * n_kb;
  if (warp == 0) {
    if (lane_id() == 0) {
      fence_proxy_async_smem();          // smem last written by generic stores (F items)
      for (int k = 0; k < n_steps; ++k) {
        const int K = gbase + k;
        const int pl = k / n_kb, j = k - pl * n_kb;
        const int p = p0 + pl;
        const int st = K % P.stages;
        mbar_wait(&sy.empty[st], ((K / P.stages) & 1) ^ 1);
        const uint32_t kc = kblock_width(g.Cpad, j);
        uint8_t* sb = smem + st * stage_bytes;
        const uint32_t abytes = kBlockTiles * kc * 2, bbytes = g.Cppad * kc * 2;
        mbar_expect_tx(&sy.full[st], 2 * abytes + (prec_passes(P.passes) > 1 ? 2 : 1) * bbytes);
        const uint8_t* a_src = uslot + static_cast<size_t>(p) * 2 * a_slab + kblock_off(j, kBlockTiles);
        const uint8_t* b_src = P.vpack + static_cast<size_t>(p) * 2 * v_slab + kblock_off(j, g.Cppad);
        bulk_g2s(sb, a_src, abytes, &sy.full[st]);
        bulk_g2s(sb + a_half, a_src + a_slab, abytes, &sy.full[st]);
        bulk_g2s(sb + 2 * a_half, b_src, bbytes, &sy.full[st]);
        if (prec_passes(P.passes) > 1) bulk_g2s(sb + 2 * a_half + b_half, b_src + v_slab, bbytes, &sy.full[st]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(kBlockTiles, g.Cppad, false, false, prec_f16(P.passes));
    for (int k = 0; k < n_steps; ++k) {
      const int K = gbase + k;
      const int pl = k / n_kb, j = k - pl * n_kb;
      const int st = K % P.stages;
      mbar_wait(&sy.full[st], (K / P.stages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t kc = kblock_width(g.Cpad, j);
        const uint32_t sa = smem_u32(smem + st * stage_bytes);
        const uint32_t sbb = sa + 2 * a_half;
        const uint32_t sbo = 16 * kc;
        const uint32_t dcol = tmem + pl * g.Cppad;
        for (uint32_t s = 0; s < kc / 16; ++s) {
          const uint64_t ahi = smem_desc(sa + s * 256, 128, sbo);
          const uint64_t alo = smem_desc(sa + a_half + s * 256, 128, sbo);
          const uint64_t bhi = smem_desc(sbb + s * 256, 128, sbo);
          const uint64_t blo = smem_desc(sbb + b_half + s * 256, 128, sbo);
          const uint32_t first = (j == 0 && s == 0) ? 0u : 1u;
          if (prec_passes(P.passes) > 1) {
            mma_bf16_ss(dcol, alo, bhi, idesc, first);
            mma_bf16_ss(dcol, ahi, blo, idesc, 1u);
            mma_bf16_ss(dcol, ahi, bhi, idesc, 1u);
          } else {
            mma_bf16_ss(dcol, ahi, bhi, idesc, first);
          }
        }
        mma_commit(&sy.empty[st]);
        if (j == n_kb - 1) mma_commit(&sy.tfull[pl]);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    const int qd = warp & 3;
    const int row = qd * 32 + lane_id();
    const int tile = b * kBlockTiles + row;
    // M ring layout: [p][c' pair][tile][2] -- a lane stores 8 bytes (two c'),
    // a warp 256 contiguous bytes; the I items load the same pairs
    const int cpo2 = KC ? KC : round_up(g.Cp, 2);
    float* mslot = P.mring + static_cast<size_t>(b % P.NM) * g.T * g.T * cpo2 * kBlockTiles;
    const bool live = tile < g.n_tile;
    for (int pl = 0; pl < np; ++pl) {
      mbar_wait(&sy.tfull[pl], tuse[pl] & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(qd * 32) << 16) + pl * (KC ? KC : g.Cppad);
      float2* mrow = reinterpret_cast<float2*>(mslot + static_cast<size_t>(p0 + pl) * cpo2 * kBlockTiles) + row;
      if constexpr (KC != 0) {
#pragma unroll
        for (int c = 0; c < KC; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          tmem_ld_wait();
          if (live) {
#pragma unroll
            for (int i = 0; i < 8; ++i) __stcg(mrow + (c / 2 + i) * kBlockTiles, make_float2(v[2 * i], v[2 * i + 1]));
          }
        }
      } else {
        for (int c = 0; c < g.Cppad; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          tmem_ld_wait();
          if (live) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + 2 * i < g.Cp)
                __stcg(mrow + static_cast<size_t>(c / 2 + i) * kBlockTiles, make_float2(v[2 * i], v[2 * i + 1]));
          }
        }
      }
    }
    tc_fence_before();
  }
}

// ------------------------------------------------------------------ I item
// Thread = (tile, c' sub-lane): the T*T products of one (tile, c') are read
// with one coalesced load per position (lanes = consecutive tiles), inverse
// transformed, and the m x m block is stored row by row -- vector stores
// when the rows are 16-byte (8-byte) aligned, so a warp writes contiguous
// output-row segments with no shared-memory staging.
template <int T, int NT, int KC>
__device__ void run_inverse_item(const PersistParams& P, int b, int ig) {
  const Geo& g = P.g;
  constexpr int MO = T - 2;
  constexpr int SUB = NT / kBlockTiles;      // c' handled concurrently
  const int cpo2 = KC ? KC : round_up(g.Cp, 2);   // M ring rows per position
  const int tid = threadIdx.x;
  const int tl = tid % kBlockTiles, cs = tid / kBlockTiles;
  const int tile = b * kBlockTiles + tl;
  if (tile >= g.n_tile) return;
  const int per_img = g.tiles_y * g.tiles_x;
  const int bi = tile / per_img;
  const int rem = tile - bi * per_img;
  const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
  const int oy = ty * MO, ox = tx * MO;
  const bool full = oy + MO <= g.Ho && ox + MO <= g.Wo;
  const bool vec = full && ((MO == 4 && (g.Wo & 3) == 0) || (MO == 2 && (g.Wo & 1) == 0));
  const float2* mbase =
      reinterpret_cast<const float2*>(P.mring + static_cast<size_t>(b % P.NM) * g.T * g.T * cpo2 * kBlockTiles) + tl;
  const size_t plane = static_cast<size_t>(g.Ho) * g.Wo;
  float* ybase = P.y + static_cast<size_t>(bi) * g.Cp * plane + static_cast<size_t>(oy) * g.Wo + ox;
  const int c_end = min(g.Cp, (ig + 1) * P.igc);
  // one c' pair (2k, 2k+1) per pass: one 8-byte load per position, packed
  // f32x2 inverse; the odd member may be past the end
  for (int cp = ig * P.igc + 2 * cs; cp < c_end; cp += 2 * SUB) {
    const bool two = cp + 1 < c_end;
    const float2* src = mbase + static_cast<size_t>(cp / 2) * kBlockTiles;
    float2 mm[T][T];
#pragma unroll
    for (int r = 0; r < T; ++r)
#pragma unroll
      for (int s = 0; s < T; ++s) mm[r][s] = __ldcg(src + static_cast<size_t>(r * T + s) * (cpo2 / 2) * kBlockTiles);
    float2 out[MO][MO];
    inverse_transform2<T>(mm, out);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
      float* dst = ybase + static_cast<size_t>(cp + h) * plane;
      if (vec) {
#pragma unroll
        for (int r = 0; r < MO; ++r) {
          if constexpr (MO == 4) {
            *reinterpret_cast<float4*>(dst + r * g.Wo) =
                h ? make_float4(out[r][0].y, out[r][1].y, out[r][2].y, out[r][3].y)
                  : make_float4(out[r][0].x, out[r][1].x, out[r][2].x, out[r][3].x);
          } else if constexpr (MO == 2) {
            *reinterpret_cast<float2*>(dst + r * g.Wo) =
                h ? make_float2(out[r][0].y, out[r][1].y) : make_float2(out[r][0].x, out[r][1].x);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < MO; ++r)
#pragma unroll
          for (int s = 0; s < MO; ++s)
            if (oy + r < g.Ho && ox + s < g.Wo) dst[r * g.Wo + s] = h ? out[r][s].y : out[r][s].x;
      }
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int T, int NT, int CPS, int KC, bool F16>
__global__ void __launch_bounds__(NT, CPS) fused_persistent_kernel(PersistParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ GemmSync sy;
  __shared__ uint32_t tmem_slot;
  __shared__ int item_s[2][4];       // double-buffered: kind, block, sub-index (or -1: done), deps ready
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = P.g.n_blk;
  int* head = P.counters;
  int* doneF = P.counters + 1;
  int* doneG = doneF + nb;
  int* doneI = doneG + nb;
  if (tid == 0) {
    for (int s = 0; s < 3; ++s) { mbar_init(&sy.full[s], 1); mbar_init(&sy.empty[s], 1); }
    for (int a = 0; a < 8; ++a) mbar_init(&sy.tfull[a], 1);
    mbar_init(&sy.fbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512 / CPS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  int fcount = 0;             // F items so far (staging-barrier parity)
  int gsteps = 0;              // pipeline steps of all G items so far (CTA-uniform)
  int tuse[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int n_kb = ceil_div(P.g.Cpad, kKBlock);

  // Item decode (thread kDecodeTid only; items are handed out in increasing
  // order, so the step walk is amortised).  The decode of item k+1 -- from
  // a queue index fetched one item earlier, hiding the atomic's round trip --
  // runs at the start of item k and lands in the other half of item_s, so
  // the loop has a single barrier per item.  Dependencies only point
  // backwards, so holding prefetched items cannot deadlock the queue.
  constexpr int kDecodeTid = 64;
  int step = 0, step_base = 0, nf = 0, ng = 0;
  int next_item = 0;
  int step_items = 0;
  // role split (P.split_f > 0): forward-only CTAs take F items from their
  // own queue in block order; the others take G and I items (step s: G of
  // block s, then I of block s - (L2 - L1)) from a second queue
  const bool split = P.split_f > 0;
  const bool role_f = split && static_cast<int>(blockIdx.x) < P.split_f;
  if (split && !role_f) head = P.counters + 1 + 3 * nb;
  auto decode = [&](int* dst) {
    const int item = next_item;
    next_item = atomicAdd(head, 1);
    dst[3] = 0;
    if (split) {
      if (role_f) {
        if (item >= nb * P.n_cg) { dst[0] = -1; return; }
        dst[0] = 0; dst[1] = item / P.n_cg; dst[2] = item - dst[1] * P.n_cg;
        return;
      }
      if (item >= nb * (P.n_gg + P.n_ig)) { dst[0] = -1; return; }
      const int lag2 = P.L2 - P.L1;
      while (item >= step_base + step_items) {
        step_base += step_items;
        ++step;
        step_items = (step < nb ? P.n_gg : 0) + (step >= lag2 && step - lag2 < nb ? P.n_ig : 0);
      }
      const int k = item - step_base;
      const int ngs = step < nb ? P.n_gg : 0;
      if (k < ngs) { dst[0] = 1; dst[1] = step; dst[2] = k; }
      else { dst[0] = 2; dst[1] = step - lag2; dst[2] = k - ngs; }
      return;
    }
    if (item >= P.n_items) {
      dst[0] = -1;
      return;
    }
    while (item >= step_base + step_items) {
      step_base += step_items;
      ++step;
      step_items = items_in_step(P, step, nf, ng);
    }
    const int k = item - step_base;
    if (k < nf) { dst[0] = 0; dst[1] = step; dst[2] = k; }
    else if (k < nf + ng) { dst[0] = 1; dst[1] = step - P.L1; dst[2] = k - nf; }
    else { dst[0] = 2; dst[1] = step - P.L2; dst[2] = k - nf - ng; }
  };
  if (tid == kDecodeTid) {
    next_item = atomicAdd(head, 1);
    if (split) step_items = (0 < nb ? P.n_gg : 0) + (0 >= P.L2 - P.L1 ? P.n_ig : 0);
    else step_items = items_in_step(P, 0, nf, ng);
    decode(item_s[0]);
  }
  __syncthreads();
  for (int it = 0;; ++it) {
    const int* cur = item_s[it & 1];
    const int kind = cur[0], b = cur[1], sub = cur[2];
    if (kind < 0) break;
    if (tid == kDecodeTid) {
      // decode the next item and check its dependencies now, one item
      // ahead: when they are already complete its warps skip the polling
      int* nx = item_s[(it + 1) & 1];
      decode(nx);
      const int nk = nx[0], nbk = nx[1];
      bool ready = false;
      if (nk == 0) ready = nbk < P.NU || ld_acquire(doneG + (nbk - P.NU)) >= P.n_gg;
      else if (nk == 1) ready = ld_acquire(doneF + nbk) >= P.n_cg &&
                                (nbk < P.NM || ld_acquire(doneI + (nbk - P.NM)) >= P.n_ig);
      else if (nk == 2) ready = ld_acquire(doneG + nbk) >= P.n_gg;
      nx[3] = ready ? 1 : 0;
    }
    long long t_a = 0, t_b = 0;
    unsigned long long g_a = 0;
    if (g_prof_on && tid == 0) { t_a = clock64(); g_a = gtimer(); }
    // Dependency wait, per warp (lane 0 acquires, __syncwarp orders the
    // lanes after it): no CTA barrier at the start of an item.
    if (cur[3]) {
      if (kind == 1 && tid == 0) fence_proxy_async_global();          // U read by bulk copies
    } else if ((tid & 31) == 0) {
      if (kind == 0) {
        if (b >= P.NU) spin_until(doneG + (b - P.NU), P.n_gg);          // U slot free
      } else if (kind == 1) {
        spin_until(doneF + b, P.n_cg);                                   // U complete
        if (b >= P.NM) spin_until(doneI + (b - P.NM), P.n_ig);           // M slot free
        fence_proxy_async_global();
      } else {
        spin_until(doneG + b, P.n_gg);                                   // M complete
      }
    }
    __syncwarp();
    if (g_prof_on && tid == 0) t_b = clock64();
    if (P.only && P.only != kind + 1 && !((P.only == 5 || P.only == 6) && kind == 0)) {
      // tuning aid (WF_ONLY=1/2/3): items of the other kinds are skipped
    } else if (kind == 0) {                                // ---- F(b, sub)
      if (run_forward_item<T, NT, KC, F16>(P, b, sub, smem, sy, fcount & 1)) ++fcount;
    } else if (kind == 1) {                                // ---- G(b, sub)
      tc_fence_after();
      run_gemm_item<NT, KC>(P, b, sub, smem, sy, tmem, gsteps, tuse);
      const int np = min(P.gp, P.g.T * P.g.T - sub * P.gp);
      gsteps += np * n_kb;
#pragma unroll
      for (int i = 0; i < 8; ++i) tuse[i] += (i < np) ? 1 : 0;
      tc_fence_before();
    } else {                                               // ---- I(b, sub)
      run_inverse_item<T, NT, KC>(P, b, sub);
    }
    __syncthreads();                                       // item done: smem free, next item decoded
    if (P.discard) {
      // Ring data this item consumed is dead (each region has exactly one
      // reader): drop its L2 lines without write-back, so dead U / M never
      // costs DRAM write bandwidth and live ring data keeps the L2.
      if (kind == 1) {
        const int np = min(P.gp, P.g.T * P.g.T - sub * P.gp);
        const size_t a2 = 2ull * kBlockTiles * P.g.Cpad * 2;           // hi + lo slab of one position
        const uint8_t* base = P.uring + (static_cast<size_t>(b % P.NU) * P.g.T * P.g.T + sub * P.gp) * a2;
        const int lines = static_cast<int>(np * a2 / 128);
        for (int i = tid; i < lines; i += NT) discard_l2(base + static_cast<size_t>(i) * 128);
      } else if (kind == 2) {
        const int cpo2 = KC ? KC : round_up(P.g.Cp, 2);
        const int pair0 = sub * P.igc / 2;
        const int npair = (min(P.g.Cp, (sub + 1) * P.igc) - sub * P.igc + 1) / 2;
        const size_t pstride = static_cast<size_t>(cpo2 / 2) * kBlockTiles * 8;    // bytes per position
        const uint8_t* base = reinterpret_cast<const uint8_t*>(P.mring) +
                              static_cast<size_t>(b % P.NM) * P.g.T * P.g.T * cpo2 * kBlockTiles * 4 +
                              static_cast<size_t>(pair0) * kBlockTiles * 8;
        const int per_pos = npair * kBlockTiles * 8 / 128;               // lines per position
        const int lines = P.g.T * P.g.T * per_pos;
        for (int i = tid; i < lines; i += NT)
          discard_l2(base + static_cast<size_t>(i / per_pos) * pstride + static_cast<size_t>(i % per_pos) * 128);
      }
    }
    {
      // Completion is published by a thread whose warp has slack at the start
      // of the next item (warp 3 is idle in G items; warp 7 waits for the
      // staging issue of F items), so its fence does not delay the item.
      const int publisher = item_s[(it + 1) & 1][0] == 1 ? 96 : 224;
      if (tid == publisher) {
        long long tp = 0;
        if (g_prof_on) tp = clock64();
        __threadfence();
        atomicAdd((kind == 0 ? doneF : kind == 1 ? doneG : doneI) + b, 1);
        if (g_prof_on) g_prof[(blockIdx.x % kProfCtas) * kProfSlots + 14] += clock64() - tp;
      }
    }
    if (g_prof_on > 1 && tid == 0) {
      const int kk = atomicAdd(&g_trace_n, 1);
      if (kk < kTraceMax) {
        g_trace[2 * kk] = (static_cast<unsigned long long>(blockIdx.x) << 32) | (static_cast<unsigned>(kind) << 24) | b;
        g_trace[2 * kk + 1] = ((gtimer() - g_a) << 40) | (g_a & ((1ull << 40) - 1));
      }
    }
    if (g_prof_on && tid == 0) {
      unsigned long long* pr = g_prof + (blockIdx.x % kProfCtas) * kProfSlots + kind * 3;
      pr[0] += t_b - t_a;
      pr[1] += clock64() - t_b;
      pr[2] += 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512 / CPS>(tmem);
}

// ------------------------------------------------------------------ host
struct PersistPlan {
  bool ok;
  int cpc, ftiles, gp, igc, n_cg, n_gg, n_ig, NU, NM, L1, L2, wreg, trows, plane, nt, f_desc_off, f_max_rows, cps, stages;
  int f_bulk, f_shift;
  size_t u_slot, m_slot, counters_bytes, smem;
};

static PersistPlan persist_plan_cpc(const Geo& g, int cps, int cpc, const FusedOpts& o);

// Two CTAs per SM (they overlap each other's latency) when T <= 6 and the
// shared memory fits, else one; forward items of 64 tiles x 8 channels
// (whole 16-byte core-matrix rows per store) when their input staging fits,
// else 128 tiles x 4 channels (fewer staged rows per channel, for wide images).
static PersistPlan persist_plan(const Geo& g, const FusedOpts& o) {
  PersistPlan pl = {};
  for (int cps = (g.T <= 6 ? 2 : 1); cps >= 1 && !pl.ok; --cps)
    for (int cpc = 8; cpc >= 4 && !pl.ok; cpc /= 2) pl = persist_plan_cpc(g, cps, cpc, o);
  return pl;
}

static PersistPlan persist_plan_cpc(const Geo& g, int cps, int cpc, const FusedOpts& o) {
  PersistPlan pl = {};
  if (g.fft) return pl;                    // FFT-16 runs the staged L2 waves
  pl.nt = 256;
  pl.cps = cps;
  pl.stages = pl.cps == 2 ? 2 : 3;
  pl.cpc = cpc;
  pl.ftiles = pl.nt / (pl.cpc / 2);        // ftiles x cpc/2 pairs = nt threads
  if (pl.ftiles > kBlockTiles) return pl;
  // up to C' = 256 (one CTA per SM, two GEMM stages; measured VGG 256->256@56
  // 332 -> 313 us against the L2 waves); WF_PERSIST_MAX_CP overrides
  const int max_cppad = tuning_knob("WF_PERSIST_MAX_CP", 256);
  if (g.Cpad % pl.cpc != 0 || g.Cppad > max_cppad) return pl;
  pl.gp = (512 / pl.cps) / g.Cppad;
  if (pl.gp > 8) pl.gp = 8;
  if (const int gp = tuning_knob("WF_GP", 0)) pl.gp = std::max(1, std::min(pl.gp, gp));
  if (pl.gp > g.T * g.T) pl.gp = g.T * g.T;
  pl.igc = tuning_knob("WF_IGC", 8);   // c' per I item (thread = tile x c' sub-lane)
  pl.n_cg = (kBlockTiles / pl.ftiles) * (g.Cpad / pl.cpc);
  pl.n_gg = ceil_div(g.T * g.T, pl.gp);
  pl.n_ig = ceil_div(g.Cp, pl.igc);
  pl.wreg = (g.tiles_x - 1) * g.m + g.T;
  // bulk-copy staging needs 16-byte aligned input rows; staged column 4 = x 0
  pl.f_bulk = (g.W % 4 == 0) ? 1 : 0;
  pl.f_shift = pl.f_bulk ? 0 : g.pad_lo;
  if (pl.f_bulk) pl.wreg = g.W;             // unpadded rows, one bulk copy per (channel, tile row)
  pl.trows = ceil_div(pl.ftiles - 1, g.tiles_x) + 1;
  if (pl.trows > g.B * g.tiles_y) pl.trows = g.B * g.tiles_y;
  // plane pitch = 1 (mod 32) words: the 4 channel pairs of a warp land on
  // different banks (2-way instead of 4-way conflicts on the window reads)
  // (bulk-copy staging needs 16-byte aligned rows: pitch = 4 mod 32 instead)
  pl.plane = round_up(pl.trows * g.T * pl.wreg, 32) + (pl.f_bulk ? 16 : 1);
  pl.f_max_rows = pl.cpc * pl.trows * g.T;
  pl.f_desc_off = round_up(pl.cpc * pl.plane * 4, 16);
  const size_t f_smem = pl.f_desc_off + static_cast<size_t>(pl.f_max_rows) * 12;
  size_t g_smem = pl.stages * (2 * kBlockTiles * kKBlock * 2 + 2 * static_cast<size_t>(g.Cppad) * kKBlock * 2);
  if (pl.cps == 1 && g_smem > 200u * 1024) {           // wide C': two stages
    pl.stages = 2;
    g_smem = pl.stages * (2 * kBlockTiles * kKBlock * 2 + 2 * static_cast<size_t>(g.Cppad) * kKBlock * 2);
  }
  pl.smem = f_smem > g_smem ? f_smem : g_smem;
  if (pl.smem > (pl.cps == 2 ? 108u : 200u) * 1024) return pl;
  pl.u_slot = static_cast<size_t>(g.T) * g.T * 2 * kBlockTiles * g.Cpad * 2;
  pl.m_slot = static_cast<size_t>(g.T) * g.T * round_up(g.Cp, 2) * kBlockTiles * 4;
  // lags and ring sizes: ~a machine-full of items in flight between stages,
  // rings within an L2 budget
  // A "window" = the blocks whose items occupy all CTAs at once.  Producers
  // run `lag` steps ahead of consumers; a ring slot is reused only after
  // lag + window more steps, so neither side normally waits.
  // measured on B200 (c2, tools/lag_sweep.py): rings below ~64 MB starve the
  // pipeline and larger rings with longer lags keep helping, beyond the
  // 126 MB L2 (the spilled part of the rings costs little HBM time here):
  // 100 MB / lag 8: 178 us, 124 / 12: 150 us, 220 / 24: 121 us, 300 / 32: 117 us
  size_t budget = o.ring_bytes ? o.ring_bytes : static_cast<size_t>(tuning_knob("WF_L2_BUDGET_MB", 300)) << 20;
  const int items_per_block = pl.n_cg + pl.n_gg + pl.n_ig;
  const int window = ceil_div(148 * pl.cps, items_per_block) + 1;
  // the lag is a number of blocks; what matters is the work between a
  // producer and its consumer, ~800 items (measured: c2 32 blocks of 33
  // items, c5 (T = 8) 16-24 of 32, VGG 128->128@112 8-20 of 57 -- the old
  // fixed 32 left that layer 822 us instead of 520), and the rings need
  // slack beyond lag + window or the producers stall on ring slots
  int lag = std::max(4, std::min(32, (800 + items_per_block / 2) / items_per_block));
  if (o.lag > 0) lag = o.lag;
  else if (const int k = tuning_knob("WF_LAG", 0)) lag = k;
  const int slots = static_cast<int>(budget / (pl.u_slot + pl.m_slot));
  if (slots < 4) return pl;
  if (2 * (lag + window + 2) > slots) lag = slots / 2 - window - 2;
  if (lag < 1) lag = 1;
  int lag2 = lag;                          // inverse items trail the GEMM items by lag2 steps
  if (const int k = tuning_knob("WF_LAG2", 0)) lag2 = k;
  if (lag2 < 1) lag2 = 1;
  pl.L1 = lag;
  pl.L2 = lag + lag2;
  pl.NU = slots / 2;
  pl.NM = slots - pl.NU;
  if (pl.NU < pl.L1 + 1) pl.NU = pl.L1 + 1;
  if (pl.NM < pl.L2 - pl.L1 + 1) pl.NM = pl.L2 - pl.L1 + 1;
  if (pl.NU > g.n_blk) pl.NU = g.n_blk;
  if (pl.NM > g.n_blk) pl.NM = g.n_blk;
  if (pl.NU <= pl.L1 && pl.NU < g.n_blk) return pl;
  pl.counters_bytes = static_cast<size_t>(2 + 3 * g.n_blk) * sizeof(int);
  pl.ok = true;
  return pl;
}

// Small layers (a few 128-tile blocks) have no stage overlap to exploit and
// pay the persistent pipeline's fill and drain: they run as a single L2 wave
// (three back-to-back kernels on L2-resident intermediates) instead.
// (The automatic dispatch applies the threshold; an explicit WF_FUSED_ITEMQ
// request runs the kernel on any layer it can hold -- the tests do.)
// Very narrow layers (Cpad = 16) have too little work per item for the
// persistent pipeline unless they are large (measured on c5).
bool persistent_fits(const Geo& g, const FusedOpts& o, bool automatic) {
  if (automatic) {
    const int min_blocks = tuning_knob("WF_PERSIST_MIN_BLOCKS", 16);
    if (g.n_blk < min_blocks) return false;
    if (g.Cpad < 32 && g.n_blk < 4 * min_blocks) return false;
  }
  return persist_plan(g, o).ok;
}

size_t persistent_scratch_bytes(const Geo& g, const FusedOpts& o) {
  const PersistPlan pl = persist_plan(g, o);
  if (!pl.ok) return 0;
  return round_up(static_cast<int>(pl.counters_bytes), 1024) + pl.NU * pl.u_slot + pl.NM * pl.m_slot;
}

template <int T, int NT, int CPS, int KC>
static cudaError_t launch_persist_t(const PersistParams& P, size_t smem, int grid, cudaStream_t st) {
  auto kern = prec_f16(P.passes) ? fused_persistent_kernel<T, NT, CPS, KC, true>
                                 : fused_persistent_kernel<T, NT, CPS, KC, false>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), 200 * 1024);
  if (e != cudaSuccess) return e;
  // No co-residency needed: items are claimed through one atomic counter in
  // dependency order by CTAs that are already running, so every item a CTA
  // waits on was claimed earlier by a resident CTA; CTAs that cannot be
  // resident yet simply start later (and find the queue drained).  The grid
  // is still sized to what fits at once.
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) == cudaSuccess && per_sm >= 1 &&
      per_sm * sms < grid)
    grid = per_sm * sms;
  note_launch();
  kern<<<grid, NT, smem, st>>>(P);
  return cudaGetLastError();
}

cudaError_t run_fused_persistent(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g,
                                 int passes, int sm_count, cudaStream_t st, const FusedOpts& o) {
  const PersistPlan pl = persist_plan(g, o);
  if (!pl.ok) return cudaErrorInvalidValue;
  PersistParams P;
  P.x = x; P.y = y; P.vpack = vpack;
  P.counters = reinterpret_cast<int*>(scratch);
  P.uring = scratch + round_up(static_cast<int>(pl.counters_bytes), 1024);
  P.mring = reinterpret_cast<float*>(P.uring + pl.NU * pl.u_slot);
  P.g = g;
  P.n_cg = pl.n_cg; P.n_gg = pl.n_gg; P.n_ig = pl.n_ig;
  P.cpc = pl.cpc; P.gp = pl.gp; P.igc = pl.igc; P.ftiles = pl.ftiles;
  P.NU = pl.NU; P.NM = pl.NM; P.L1 = pl.L1; P.L2 = pl.L2;
  P.passes = passes;
  P.n_steps = g.n_blk + pl.L2;
  P.n_items = g.n_blk * (pl.n_cg + pl.n_gg + pl.n_ig);
  P.only = 0;
#ifdef WF_TUNING_AIDS
  P.only = tuning_knob("WF_ONLY", 0);      // cost one item kind in isolation (results invalid)
#endif
  P.split_f = tuning_knob("WF_SPLIT", 0) * sm_count * pl.cps / 100;
  P.discard = tuning_knob("WF_DISCARD", 0);   // measured neutral-to-slower on c2 (DRAM is not the limiter)
  P.wreg = pl.wreg; P.trows = pl.trows; P.plane = pl.plane;
  P.f_desc_off = pl.f_desc_off; P.f_max_rows = pl.f_max_rows;
  P.f_bulk = pl.f_bulk; P.f_shift = pl.f_shift;
  cudaError_t e = cudaMemsetAsync(P.counters, 0, pl.counters_bytes, st);
  if (e != cudaSuccess) return e;
  {
    static int prof_state = -1;
    if (prof_state < 0) {
      prof_state = tuning_knob("WF_PROFILE", 0);
      cudaMemcpyToSymbol(g_prof_on, &prof_state, sizeof(int));
    }
  }
  const int grid = sm_count * pl.cps;
  P.stages = pl.stages;
  // square channel counts that are multiples of 16 get compile-time strides
  const int kc = (g.Cpad == g.Cppad && g.Cppad == g.Cp && g.C == g.Cp) ? g.Cp : 0;
  switch (g.T) {
    case 4:
      if (pl.cps == 1) return launch_persist_t<4, 256, 1, 0>(P, pl.smem, grid, st);
      return launch_persist_t<4, 256, 2, 0>(P, pl.smem, grid, st);
    case 5:
      if (pl.cps == 1) return launch_persist_t<5, 256, 1, 0>(P, pl.smem, grid, st);
      return launch_persist_t<5, 256, 2, 0>(P, pl.smem, grid, st);
    case 6:
      if (pl.cps == 1) return launch_persist_t<6, 256, 1, 0>(P, pl.smem, grid, st);
      if (kc == 64) return launch_persist_t<6, 256, 2, 64>(P, pl.smem, grid, st);
      if (kc == 32) return launch_persist_t<6, 256, 2, 32>(P, pl.smem, grid, st);
      return launch_persist_t<6, 256, 2, 0>(P, pl.smem, grid, st);
    case 7: return launch_persist_t<7, 256, 1, 0>(P, pl.smem, grid, st);
    case 8:
      if (kc == 64) return launch_persist_t<8, 256, 1, 64>(P, pl.smem, grid, st);
      return launch_persist_t<8, 256, 1, 0>(P, pl.smem, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wf

// Debug/tuning hook (not part of the public ABI): copy the per-CTA item
// accounting [cta][kind F,G,I][wait cycles, run cycles, count] and reset it.
extern "C" int wf_debug_fused_profile(unsigned long long* host, int n) {
  using namespace wf;
  const int cnt = n < kProfCtas * kProfSlots ? n : kProfCtas * kProfSlots;
  cudaError_t e = cudaMemcpyFromSymbol(host, wf::g_prof, cnt * sizeof(unsigned long long));
  static unsigned long long zeros[kProfCtas * kProfSlots] = {0};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(wf::g_prof, zeros, sizeof(zeros));
  return e == cudaSuccess ? 0 : 4;
}

// Debug/tuning hook: copy the item trace (2 words per item) and reset it;
// returns the number of items recorded.
extern "C" int wf_debug_fused_trace(unsigned long long* host, int max_items) {
  using namespace wf;
  int n = 0;
  cudaMemcpyFromSymbol(&n, wf::g_trace_n, sizeof(int));
  if (n > kTraceMax) n = kTraceMax;
  if (n > max_items) n = max_items;
  cudaMemcpyFromSymbol(host, wf::g_trace, static_cast<size_t>(n) * 2 * sizeof(unsigned long long));
  const int zero = 0;
  cudaMemcpyToSymbol(wf::g_trace_n, &zero, sizeof(int));
  return n;
}
