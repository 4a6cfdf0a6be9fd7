// fused_ws.cu -- conv_fused as ONE warp-specialised persistent kernel
// (F(4x4,3x3), C = C' = 64: the c2 benchmark layer and the 64-channel
// ResNet / VGG layers).
//
// The reference's fused engine (engines.py:317-444) keeps a task's
// transformed tiles in the shared last-level cache between its three
// stages.  Here every SM runs all three stages at once, each on its own
// warps, and the transformed tiles U and the products M live in L2-resident
// rings between them:
//   warp 0      G producer: bulk copies of U (half-K blocks) and V into smem
//   warp 1      G issuer: tcgen05.mma 3xBF16, f32 accumulators in TMEM
//               (2 x 4 positions x 64 columns, double buffered)
//   warps 4-7   G epilogue: tcgen05.ld -> M ring (f32, c' pairs interleaved)
//   warp 2      F/I producer: bulk copies of input rows (F) or M (I) into a
//               2-slot smem ring
//   warps 8-15  F/I workers: forward transform + bf16 hi/lo split -> U ring
//               (F units) or inverse transform -> output (I units)
//   warp 3      publisher: per-unit completion (fence + atomic) to the
//               per-block counters other SMs wait on
// Work is assigned statically (CTA k takes every grid-th unit of each
// queue).  Every queue walks the total order "step s: F(s), G(s - L1),
// I(s - L2)" with L1 < NU and L2 - L1 < NM, so every dependency points to
// an earlier step and, with all CTAs co-resident, the lowest unfinished
// unit is always runnable: no deadlock, and no role ever waits on another
// role of its own CTA except through its pipeline.
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "fused.cuh"

namespace wf {
namespace ws {

constexpr int NT = 512;
#ifndef WF_WS_REGS
#define WF_WS_REGS 1
#endif
constexpr uint32_t kRegsLight = WF_WS_REGS ? 40 : 128;
constexpr uint32_t kRegsEpi = WF_WS_REGS ? 64 : 128;
constexpr uint32_t kRegsFI = WF_WS_REGS ? 200 : 128;
static_assert(4 * 32 * kRegsLight + 4 * 32 * kRegsEpi + 8 * 32 * kRegsFI <= 65536, "register file");
constexpr int kNAcc = 8;                                 // TMEM accumulator buffers (units in flight), at most
constexpr int kMaxGP = 6;                                // positions per G unit, at most
constexpr int kMaxAStages = 4;

// Layer shape: window T (6: F(4x4,3x3), 8: F(6x6,3x3)), C input channels
// (GEMM K, 32-channel K blocks), CP output channels (GEMM N, 64-wide G
// units).  Shared memory: A stages + the V slab of the CTA's (position, c'
// group) + two 72 KB F/I slots <= 227 KB.
// GP_ = positions per G unit: 1 (a CTA owns one position) or T (the "row
// unit" instance, T = 6 with C, C' <= 64: a CTA owns one ROW of positions
// (r, 0..5), keeps their six V slabs resident, accumulates the row's six
// products of a block in TMEM and runs the inverse transform's row pass in
// the GEMM epilogue, so the M ring carries 4 instead of 6 values per row
// and the I units only run the column pass).
template <int T_, int C_, int CP_, int SL_ = 2, int GP_ = 1>
struct Shape {
  // (other GP_ > 1: a G unit covers GP_ consecutive positions with the
  // one-position M layout -- fewer, larger units for the narrow layers,
  // whose G roles are bound by the per-unit latency)
  static constexpr int kGP = GP_;
  static constexpr bool kRow = T_ == 6 && GP_ == 6;
  static constexpr int kNcols = GP_ * (CP_ < 64 ? CP_ : 64);     // TMEM columns of one unit
  // TMEM buffers in flight (row units: 6 x 64 columns, one buffer)
  static constexpr int kAcc = kRow ? 1 : (512 / kNcols < kNAcc ? 512 / kNcols : kNAcc);
  static_assert(!kRow || (C_ <= 64 && CP_ == 64 && SL_ == 2), "row units");
  static_assert((T_ * T_) % GP_ == 0 && kAcc >= 1 && kAcc * kNcols <= 512, "positions per G unit");
  // F/I staging slots: 2 x 72 KB.  (3 x 48 KB with 2-channel I units was
  // measured on c2: 98 vs 80 us -- twice the I units and a shorter lag)
  static constexpr int kSlots = SL_;
  static constexpr int kT = T_, kP = T_ * T_;
  static constexpr int C = C_, CP = CP_;               // C = Cpad (input channels may be fewer)
  static constexpr int kN = CP < 64 ? CP : 64;           // output channels per G unit (MMA N)
  static constexpr int kTmemColsUsed = kAcc * kGP * kN;
  static constexpr int kTmemCols = kTmemColsUsed <= 128 ? 128 : kTmemColsUsed <= 256 ? 256 : 512;
  // F unit: kFT tiles x 8 channels (one core-matrix k group, so that a
  // warp's U stores fill whole 32-byte sectors): 64 tiles with a thread per
  // (tile, channel pair) for T = 6, 32 tiles with a thread per (tile,
  // channel) for T = 8, whose larger windows need more staging per tile
  static constexpr int kCPC = 8;
  static constexpr int kFT = T_ == 6 ? 64 : 32;
  // F staging or I staging slot (two of them)
  // (C = 256, T = 6: 48 KB, room for the 64 KB V slab; 2-channel I units)
  static constexpr uint32_t kFISlot = (SL_ == 3 || kRow ? 48 : T_ == 6 ? (C_ >= 256 ? 48 : 72) : 73) * 1024;
  // I unit: kIPairs c' pairs.  M ring slot layout: [I unit][position][c' pair
  // in unit][tile][2]: the products one I unit needs are one contiguous
  // range (72 KB for T = 6, 64 KB for T = 8) -- one bulk copy
  // (row units: [I unit][row r][output column j][c' pair][tile][2], 6 x 4
  // values per (tile, c'): 48 KB)
  static constexpr int kIPairs = (T_ == 6 && C_ < 256 && SL_ == 2) ? 2 : 1;
  static constexpr uint32_t kIPos = kIPairs * kBlockTiles * 8;
  static constexpr uint32_t kMUnit = (kRow ? T_ * (T_ - 2) : kP) * kIPos;
  static constexpr int kKBW = C < 32 ? C : 32;           // K block width (channels per A stage)
  static constexpr int kKB = C / kKBW;                   // K blocks
  static constexpr uint32_t kAHalf = kBlockTiles * kKBW * 2;   // hi or lo of one K block
  static constexpr uint32_t kAStage = 2 * kAHalf;
  static constexpr int kVKW = C < 64 ? C : 64;           // K block width of the MMA pack (kblock layout)
  static constexpr uint32_t kVChunk = kN * kVKW * 2;     // one c' group's rows of one pack K block
  static constexpr int kNG = CP / kN;                    // c' groups (G units per position)
  static constexpr int kNGG = kP / kGP * kNG;            // G units per block
  static constexpr int kNCG = (kBlockTiles / kFT) * (C / kCPC);   // F units per block
  static constexpr int kNIG = CP / (2 * kIPairs);                 // I units per block
  // (2 stages measured equal to 4 on c2: the G units wait for their inputs, not for stage space)
  // (every extra resident V slab of a multi-position unit takes one stage's room)
  static constexpr int kAStages = kRow ? 2 : (C >= 128 ? 3 : 4) - (C == 64 ? GP_ - 1 : 0);
  static constexpr uint32_t kVHalf = kN * C * 2;         // V hi (or lo) of one (position, c' group)
  static constexpr uint32_t kVGroup = 2 * kVHalf;
  static constexpr size_t kUPos = 2 * kKB * kAHalf;      // U of one position: [hl][K block]
  static constexpr size_t kUSlot = kP * kUPos;
  static constexpr size_t kMPos = static_cast<size_t>(CP) * kBlockTiles * 4;
  static constexpr size_t kMSlot = kRow ? static_cast<size_t>(CP / (2 * kIPairs)) * kMUnit : kP * kMPos;
  static constexpr uint32_t kOffB = kAStages * kAStage;
  static constexpr uint32_t kOffFI = kOffB + kGP * kVGroup;
  static constexpr uint32_t kSmem = kOffFI + kSlots * kFISlot;
  static_assert(kSmem <= 227 * 1024 && kAStages <= kMaxAStages && C % 16 == 0 && CP % kN == 0, "shape");
  static_assert((T_ == 6 || T_ == 8) && kMUnit <= kFISlot, "window");
};

struct Params {
  const float* x;
  float* y;
  const uint8_t* vpack;   // standard MMA pack: per position hi / lo slabs of 64 x 64 (kblock, kc = 64)
  uint8_t* uring;         // NU slots x S::kUSlot
  float* mring;           // NM slots x S::kMSlot
  int* counters;          // doneF, doneG, doneI (n_blk each)
  Geo g;
  int NU, NM, L2;
  int gbatch;             // G units per completion publish (one fence per batch)
  int passes;
  int discard;            // drop consumed ring lines from L2 (WF_WS_DISCARD bits: 1 U, 2 M)
  int dbg;                // tuning aid (WF_WS_DBG=3: no GEMM work, results invalid)
  int plane;              // floats per staged channel of an F unit
  int n_fi;               // F/I queue length
  int grid;
  int prof;
};

// Stores with the kernel's L2 eviction priorities (Params::hints).
// Stores with the kernel's L2 eviction priorities, per window size (compile
// time: a runtime switch in the store paths measured 12-16% slower even when
// off): layer input and output evict-first, U ring stores evict-last (WF_WS_RING_HINTS bit 1; bit 2 = the M ring stores, measured neutral, off).
#ifndef WF_WS_L2_HINTS_T6
#define WF_WS_L2_HINTS_T6 1
#endif
#ifndef WF_WS_L2_HINTS_T8
#define WF_WS_L2_HINTS_T8 1
#endif
template <class S>
struct Hints {
  static constexpr bool on = S::kT == 6 ? WF_WS_L2_HINTS_T6 : WF_WS_L2_HINTS_T8;
};
template <class S, class T>
__device__ __forceinline__ void out_store(T* p, T v) {
  if constexpr (Hints<S>::on) st_hint(p, v, l2_policy_evict_first());
  else *p = v;
}
#ifndef WF_WS_RING_HINTS
#define WF_WS_RING_HINTS 1
#endif
template <class S>
__device__ __forceinline__ void ring_store(uint2* p, uint2 v) {
  if constexpr (Hints<S>::on && (WF_WS_RING_HINTS & 1)) st_hint(p, v, l2_policy_evict_last());
  else *p = v;
}
template <class S>
__device__ __forceinline__ void ring_store(float2* p, float2 v) {
  if constexpr (Hints<S>::on && (WF_WS_RING_HINTS & 2)) st_hint(p, v, l2_policy_evict_last());
  else __stcg(p, v);
}

// Optional per-CTA role accounting (WF_WS_PROF=1; tools/ws_prof.py):
// clock64 cycles per slot, globaltimer ns for the role end times.
constexpr int kProfSlots = 32;
__device__ unsigned long long g_wsprof[1024 * kProfSlots];
enum ProfSlot {
  kGPDep, kGPStage, kGIFull, kGITempty, kGEWait, kGEBusy, kFPDep, kFPSlot, kFWWait, kFWF, kFWI, kPubFence,
  kStart, kEndGP, kEndGI, kEndGE, kEndFP, kEndFW, kEndPub, kNF, kNI, kFWLoop, kFPBusy, kFPBusyI, kFPTx, kFPCopy
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__shared__ unsigned long long s_prof[kProfSlots];
// Instrumented instance: per-block ordering tickets.  Every unit takes a
// ticket from one global counter when it starts (after acquiring its
// dependencies) and when it ends (before its completion is released), so
// ticket order is consistent with the release/acquire chains of the
// dependency protocol; a consumer that started before its producer ended,
// or a producer that rewrote a ring slot before the slot's previous
// consumer ended, shows up as an inverted ticket pair (the GPU analogue of
// the reference's operand-overlap check, engines.py:382-396).
// Events per block (all kept as a minimum, "end" events as ~ticket so the
// minimum of ~t is the maximum of t): 0 F start (ticket << 12 | CTA of the
// first F unit), 1 ~F end, 2 G start, 3 ~G end, 4 I start, 5 ~I end.
constexpr int kTraceBlocks = 4096;
__device__ unsigned long long g_wstrace[kTraceBlocks * 8];
__device__ unsigned long long g_wsticket;
template <bool ON>
__device__ __forceinline__ void trace(int b, int ev, bool is_min) {
  if (!ON || b >= kTraceBlocks) return;
  const unsigned long long t = atomicAdd(&g_wsticket, 1ull);
  const unsigned long long v = ev == 0 ? (t << 12) | blockIdx.x : (is_min ? t : ~t);
  atomicMin(&g_wstrace[b * 8 + ev], v);
}
// Compiled in only for the profiling instantiation of the kernel.
template <bool ON>
struct ProfT {
  bool on;
  __device__ ProfT(bool flag) : on(ON && flag) {}
  __device__ long long now() const { return (ON && on) ? clock64() : 0; }
  __device__ void add(int slot, long long t0) const { if (ON && on) s_prof[slot] += clock64() - t0; }
  __device__ void inc(int slot) const { if (ON && on) s_prof[slot] += 1; }
  __device__ void end(int slot) const { if (ON && on) g_wsprof[blockIdx.x * kProfSlots + slot] = gtimer(); }
};

struct Sync {
  uint64_t a_full[kMaxAStages], a_empty[kMaxAStages];
  uint64_t b_full[2], b_empty[2];
  uint64_t tfull[kNAcc][kMaxGP], tempty[kNAcc];
  uint64_t fi_full[3], fi_empty[3];
  // completion counts: F/I unit k adds 8 (one per worker warp) to fi_cnt[k % 4],
  // G unit k adds 4 (one per epilogue warp) to g_cnt[k % kNAcc].  A warp can
  // not get a full counter ring ahead of another (the F/I slot ring and the
  // TMEM buffer ring block it first), so each count is attributed to its unit.
  int fi_cnt[4], g_cnt[kNAcc];
  uint32_t tmem;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const int* p, int target) {
  if (ld_acquire_gpu(p) >= target) return;
  while (ld_relaxed_gpu(p) < target) __nanosleep(64);
  (void)ld_acquire_gpu(p);
}
__device__ __forceinline__ int ld_acquire_cta_smem(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_cta_smem(int* p, int v) {
  asm volatile("red.release.cta.shared::cta.add.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// Publish one completed unit: release at gpu scope (orders every write this
// thread performed or observed -- the other warps' stores, through the CTA
// scope acquire that preceded it -- before the counter increment).
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_gpu(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acqrel_cta_smem(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.s32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
// Invalidate one 128-byte L2 line without write-back: ring data whose single
// consumer has copied it into shared memory is dead, so it should neither
// cost a DRAM write-back nor push live ring lines out of L2.
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
// Register re-distribution between warpgroups (all 4 warps of a group run it).
template <uint32_t N> __device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N> __device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
// Pin a pointer in registers: without it ptxas re-derives "kernel parameter
// + lane offset" (LDC.64 + two adds) in front of every store of an unrolled
// store sequence -- 36 constant-bank loads on the F units' critical path --
// instead of keeping the 64-bit base and using the stores' immediate offsets.
template <class T>
__device__ __forceinline__ void keep_in_regs(T*& p) {
  asm volatile("" : "+l"(p));
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// The F/I queue: step s holds the S::kNCG F units of block s (s < n_blk) and
// then the S::kNIG I units of block s - L2.  Closed-form decode (no state
// carried across units: nothing to keep live through the transforms).
template <class S>
struct FIWalker {
  __device__ void init(const Params&) {}
  // -> kind (0 = F, 2 = I), block, sub
  __device__ void decode(const Params& P, int u, int& kind, int& b, int& sub) const {
    const int nb = P.g.n_blk, L = P.L2;
    constexpr int nf = S::kNCG, ni = S::kNIG;
    if (L >= nb) {                       // all F steps come before the first I step
      if (u < nf * nb) { kind = 0; b = u / nf; sub = u - b * nf; }
      else { kind = 2; b = (u - nf * nb) / ni; sub = (u - nf * nb) - b * ni; }
      return;
    }
    if (u < nf * L) { kind = 0; b = u / nf; sub = u - b * nf; return; }
    const int u2 = u - nf * L;
    if (u2 < (nf + ni) * (nb - L)) {     // steps L .. nb-1: F(s) then I(s - L)
      const int st = u2 / (nf + ni), k = u2 - st * (nf + ni);
      if (k < nf) { kind = 0; b = L + st; sub = k; }
      else { kind = 2; b = st; sub = k - nf; }
      return;
    }
    const int u3 = u2 - (nf + ni) * (nb - L);  // steps nb ..: I only
    kind = 2; b = nb - L + u3 / ni; sub = u3 - (u3 / ni) * ni;
  }
};

// Input staging of one F unit (64 tiles x 8 channels): every image row the
// unit's windows touch is staged once per channel ("segments": the unit's
// tile rows of one image, at most 3 or so images for small images), one bulk
// copy per (channel, segment); rows outside the image are not staged, the
// workers zero them.
struct FGeo {
  int gr0, bi0, ya0, rows0, nseg, rows_full, rows_last;
  __device__ __host__ FGeo(const Geo& g, int t0, int tlast) {
    const int gr1 = tlast / g.tiles_x;
    gr0 = t0 / g.tiles_x;
    bi0 = gr0 / g.tiles_y;
    const int bi1 = gr1 / g.tiles_y;
    const int ty0 = gr0 - bi0 * g.tiles_y, ty1 = gr1 - bi1 * g.tiles_y;
    ya0 = ty0 * g.m - g.pad_lo > 0 ? ty0 * g.m - g.pad_lo : 0;
    rows_full = min(g.H, (g.tiles_y - 1) * g.m - g.pad_lo + g.T);
    nseg = bi1 - bi0 + 1;
    rows0 = (nseg == 1 ? min(g.H, ty1 * g.m - g.pad_lo + g.T) : rows_full) - ya0;
    rows_last = nseg == 1 ? 0 : min(g.H, ty1 * g.m - g.pad_lo + g.T);
  }
  __device__ __host__ int rowoff(int k) const { return k == 0 ? 0 : rows0 + (k - 1) * rows_full; }
  __device__ __host__ int rows(int k) const { return k == 0 ? rows0 : (k == nseg - 1 ? rows_last : rows_full); }
  __device__ __host__ int total() const { return nseg == 1 ? rows0 : rows0 + (nseg - 2) * rows_full + rows_last; }
  // staged row holding image row y of segment k
  __device__ __host__ int srow(int k, int y) const { return k == 0 ? y - ya0 : rowoff(k) + y; }
};

// ------------------------------------------------------------ F/I producer
template <class S, bool PROF>
__device__ void fi_producer(const Params& P, uint8_t* smem, Sync& sy) {
  const Geo& g = P.g;
  const int lane = threadIdx.x & 31;
  const int* doneG = P.counters + g.n_blk;
  const ProfT<PROF> pf(P.prof && lane == 0);
  FIWalker<S> wk;
  wk.init(P);

  int it = 0;
  for (int u = blockIdx.x; u < P.n_fi; u += P.grid, ++it) {
    int kind, b, sub;
    wk.decode(P, u, kind, b, sub);
    const int slot = it % S::kSlots;
    uint8_t* dstbase = smem + S::kOffFI + slot * S::kFISlot;
    // every lane waits (warp-uniform spins: a lane-0 spin with the other 31
    // lanes parked in __syncwarp made the parked lanes re-issue WARPSYNC and
    // took issue slots from the transform warps on the same SMSP)
    {
      long long t0 = pf.now();
      if (kind == 0) {
        if (b >= P.NU) spin_until(doneG + (b - P.NU), S::kNGG);     // U slot free
      } else {
        spin_until(doneG + b, S::kNGG);                               // M complete
        fence_proxy_async_global();
      }
      pf.add(kFPDep, t0);
      t0 = pf.now();
      mbar_wait(&sy.fi_empty[slot], ((it / S::kSlots) & 1) ^ 1);
      pf.add(kFPSlot, t0);
    }

    const long long tb = pf.now();
    // (no proxy fence: the slot is only ever written by bulk copies; the
    // workers' generic reads of its previous contents are ordered before
    // these writes by the fi_empty barrier)
    if (kind == 0) {
      constexpr int kCPC = S::kCPC;
      const int part = sub / (S::C / kCPC), cg = sub % (S::C / kCPC);
      const int t0 = b * kBlockTiles + part * S::kFT;
      const int tlast = min(t0 + S::kFT, g.n_tile) - 1;
      float* xs = reinterpret_cast<float*>(dstbase);
      // the single arrival carries the whole unit's byte count and comes
      // first: the phase cannot complete before every copy has landed
      // (copies that land earlier only drive the tx-count negative)
      // channels at or past C (K padding of a 16-channel layer) are not staged
      const int real = min(max(g.C - cg * kCPC, 0), kCPC);
      if (tlast < t0 || real == 0) {
        if (lane == 0) mbar_arrive(&sy.fi_full[slot]);
      } else {
        const FGeo fg(g, t0, tlast);
        if (lane == 0) mbar_expect_tx(&sy.fi_full[slot], static_cast<uint32_t>(fg.total() * g.W * 4 * real));
        for (int cu = lane; cu < kCPC * fg.nseg; cu += 32) {
          const int k = cu / kCPC, cl = cu - k * kCPC;
          const int c = cg * kCPC + cl;
          const int y0 = k == 0 ? fg.ya0 : 0;
          const uint32_t bytes = static_cast<uint32_t>(fg.rows(k) * g.W * 4);
          if (bytes && cl < real)
          {
            float* sdst = xs + cl * P.plane + fg.rowoff(k) * g.W;
            const float* gsrc = P.x + ((static_cast<size_t>(fg.bi0 + k) * g.C + c) * g.H + y0) * g.W;
            if constexpr (Hints<S>::on) bulk_g2s_hint(sdst, gsrc, bytes, &sy.fi_full[slot], l2_policy_evict_first());
            else bulk_g2s(sdst, gsrc, bytes, &sy.fi_full[slot]);
          }
        }
      }
    } else {
      // the unit's products are one contiguous range: two copies
      const uint8_t* msrc = reinterpret_cast<const uint8_t*>(P.mring) + static_cast<size_t>(b % P.NM) * S::kMSlot +
                            static_cast<size_t>(sub) * S::kMUnit;
      if (lane == 0) {
        constexpr uint32_t half = S::kMUnit / 2;
        mbar_expect_tx(&sy.fi_full[slot], S::kMUnit);    // the arrival, with the byte count
        bulk_g2s(dstbase, msrc, half, &sy.fi_full[slot]);
        bulk_g2s(dstbase + half, msrc + half, half, &sy.fi_full[slot]);
      }
    }
    __syncwarp();
    pf.add(kind == 0 ? kFPBusy : kFPBusyI, tb);
  }
  pf.end(kEndFP);
}

// ------------------------------------------------------------- F/I workers
// F(6x6,3x3) units (T = 8).  Per element the operations of forward8 /
// inverse8 (common.cuh), which every other path of the library uses for
// T = 8, so the results stay bitwise equal to them; rows are transformed as
// they are loaded and positions stored one column at a time.
//
// F(b, sub): thread = (tile tl, channel cl); a warp = 4 tiles x 8 channels
// (half of the rows of a core matrix), so that a warp writes 64 contiguous
// bytes of each core matrix it stores to.
template <class S, bool F16>
__device__ __forceinline__ void f_unit8(const Params& P, const uint8_t* src, Sync& sy, int slot, int b, int sub,
                                        int wl, int lane) {
  static_assert(S::kT == 8 && S::kCPC == 8, "T = 8 F unit");
  const Geo& g = P.g;
  constexpr int kCPC = S::kCPC;
  const int part = sub / (S::C / kCPC), cg = sub % (S::C / kCPC);
  constexpr int kFT = S::kFT;
  const int tb0 = part * kFT;
  const int t0 = b * kBlockTiles + tb0;
  const int tl = wl * 4 + (lane & 3), cl = lane >> 2, cq = cl & 3;
  const int tile = t0 + tl;
  const bool live = tile < g.n_tile;
  float x[8][8];
  if (live) {
    const FGeo fg(g, t0, min(t0 + kFT, g.n_tile) - 1);
    const int per_img = g.tiles_y * g.tiles_x;
    const int bi = tile / per_img;
    const int rem = tile - bi * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int y0 = ty * g.m - g.pad_lo;
    const int x0 = tx * g.m - g.pad_lo;
    const float* pa = reinterpret_cast<const float*>(src) + cl * P.plane + fg.srow(bi - fg.bi0, y0) * g.W + x0;
    // window columns [x0, x0 + 8), x0 = 6 tx - 1: three 8-byte loads
    // [x0 + 1, x0 + 7) and two scalars per row.  W is even, so every pair
    // lies wholly inside or wholly outside the image; the padding columns
    // and rows are zeros (their loads are predicated off)
    const bool v0 = x0 >= 0, v3 = x0 + 3 < g.W, v5 = x0 + 5 < g.W, v7 = x0 + 7 < g.W;
    const bool cv = S::C >= 64 || cg * kCPC + cl < g.C;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float* ra = pa + r * g.W;
      float a0 = 0.0f, a7 = 0.0f;
      float2 p1 = make_float2(0.0f, 0.0f), p3 = p1, p5 = p1;
      if (cv && y0 + r >= 0 && y0 + r < g.H) {
        if (v0) a0 = ra[0];
        p1 = *reinterpret_cast<const float2*>(ra + 1);
        if (v3) p3 = *reinterpret_cast<const float2*>(ra + 3);
        if (v5) p5 = *reinterpret_cast<const float2*>(ra + 5);
        if (v7) a7 = ra[7];
      }
      x[r][0] = a0;
      x[r][1] = p1.x; x[r][2] = p1.y;
      x[r][3] = p3.x; x[r][4] = p3.y;
      x[r][5] = p5.x; x[r][6] = p5.y;
      x[r][7] = a7;
      bt8_line<ScalarOps>(x[r][0], x[r][1], x[r][2], x[r][3], x[r][4], x[r][5], x[r][6], x[r][7]);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) x[r][c] = 0.0f;
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&sy.fi_empty[slot]);     // window consumed: slot free
  // Two positions (r, s), (r + 1, s) at a time, a 4-lane transpose of the
  // bf16 halves of channels c0 .. c0 + 3 of a tile (lanes cq = 0..3 hold
  // channel c0 + cq, c0 = 8 cg or 8 cg + 4): after it, lane cq stores the 4
  // channels of [hi, lo][cq & 1] of position r + (cq >> 1) as one 8-byte store.
  const int row = tb0 + tl, c0 = cg * kCPC + (cl & 4);
  uint8_t* dst = P.uring + static_cast<size_t>(b % P.NU) * S::kUSlot + (c0 / S::kKBW) * S::kAHalf +
                 (row >> 3) * (16 * S::kKBW) + ((c0 % S::kKBW) >> 3) * 128 + (row & 7) * 16 + (c0 & 7) * 2 +
                 (cq & 1) * (S::kKB * S::kAHalf) + (cq >> 1) * 8 * S::kUPos;
  keep_in_regs(dst);
  const bool odd = cq & 1, upper = cq & 2;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    bt8_line<ScalarOps>(x[0][s], x[1][s], x[2][s], x[3][s], x[4][s], x[5][s], x[6][s], x[7][s]);
#pragma unroll
    for (int r = 0; r < 8; r += 2) {
      uint32_t hi, lo;                                    // (position r, position r + 1) of channel c0 + cq
      split2<F16>(u_operand<8, F16>(x[r][s], r, s), u_operand<8, F16>(x[r + 1][s], r + 1, s), hi, lo);
      // step 1 (lanes cq ^ 1): the even lane gathers the hi halves of its
      // channel pair, the odd one the lo halves: A = position r, B = r + 1
      const uint32_t got = __shfl_xor_sync(0xffffffffu, odd ? hi : lo, 4);
      const uint32_t mine = odd ? lo : hi;
      const uint32_t lo_ch = odd ? got : mine, hi_ch = odd ? mine : got;
      const uint32_t A = __byte_perm(lo_ch, hi_ch, 0x5410), B = __byte_perm(lo_ch, hi_ch, 0x7632);
      // step 2 (lanes cq ^ 2): channels c0 + 2, c0 + 3 join c0, c0 + 1
      const uint32_t got2 = __shfl_xor_sync(0xffffffffu, upper ? A : B, 8);
      if (live)
        ring_store<S>(reinterpret_cast<uint2*>(dst + (r * 8 + s) * S::kUPos), upper ? make_uint2(got2, B) : make_uint2(A, got2));
    }
  }
}

// I(b, sub), T = 6 with 2-channel I units (C = 256): thread = (tile, c');
// per element the operations of inverse6 (== the f32x2 path of the wider
// I units).
template <class S>
__device__ __forceinline__ void i_unit6s(const Params& P, const uint8_t* src, Sync& sy, int slot, int b, int sub,
                                         int wtid, int lane) {
  static_assert(S::kT == 6 && S::kIPairs == 1, "T = 6 scalar I unit");
  const Geo& g = P.g;
  const int tl = wtid & (kBlockTiles - 1), cq = wtid >> 7;
  const int tile = b * kBlockTiles + tl;
  const float* ms = reinterpret_cast<const float*>(src) + tl * 2 + cq;
  // row pass as the staged products are read (A^T along each row), then
  // the column pass one output column at a time (== inverse6)
  float z[6][4];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    float m[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) m[s] = ms[(r * 6 + s) * (S::kIPos / 4)];
    at6_line<ScalarOps>(m[0], m[1], m[2], m[3], m[4], m[5], z[r][0], z[r][1], z[r][2], z[r][3]);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&sy.fi_empty[slot]);
  float t[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    at6_line<ScalarOps>(z[0][j], z[1][j], z[2][j], z[3][j], z[4][j], z[5][j], t[0][j], t[1][j], t[2][j], t[3][j]);
  if (tile < g.n_tile) {
    const int per_img = g.tiles_y * g.tiles_x;
    const int bi = tile / per_img;
    const int rem = tile - bi * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int oy = ty * 4, ox = tx * 4;
    const bool vec = oy + 4 <= g.Ho && ox + 4 <= g.Wo && (g.Wo & 3) == 0;
    const int cp = 2 * sub + cq;
    float* ybase = P.y + ((static_cast<size_t>(bi) * g.Cp + cp) * g.Ho + oy) * g.Wo + ox;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float o[4] = {t[r][0], t[r][1], t[r][2], t[r][3]};
      if (vec) {
        out_store<S>(reinterpret_cast<float4*>(ybase + r * g.Wo), make_float4(o[0], o[1], o[2], o[3]));
      } else if (oy + r < g.Ho) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (ox + c < g.Wo) ybase[r * g.Wo + c] = o[c];
      }
    }
  }
}

// I(b, sub), T = 8: thread = (tile, c' of the unit's pair); 64 staged
// products per thread, inverse transform, clipped 6 x 6 output block.
template <class S>
__device__ __forceinline__ void i_unit8(const Params& P, const uint8_t* src, Sync& sy, int slot, int b, int sub,
                                        int wtid, int lane) {
  static_assert(S::kT == 8 && S::kIPairs == 1, "T = 8 I unit");
  const Geo& g = P.g;
  const int tl = wtid & (kBlockTiles - 1), cq = wtid >> 7;
  const int tile = b * kBlockTiles + tl;
  const float* ms = reinterpret_cast<const float*>(src) + tl * 2 + cq;
  // column pass (A^T down each column) as the products are read
  float t[6][8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    float m[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) m[r] = ms[(r * 8 + s) * (S::kIPos / 4)];
    at8_line<ScalarOps>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], t[0][s], t[1][s], t[2][s], t[3][s], t[4][s],
                        t[5][s]);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&sy.fi_empty[slot]);
  if (tile < g.n_tile) {
    const int per_img = g.tiles_y * g.tiles_x;
    const int bi = tile / per_img;
    const int rem = tile - bi * per_img;
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    const int oy = ty * 6, ox = tx * 6;
    const bool vec = oy + 6 <= g.Ho && ox + 6 <= g.Wo && (g.Wo & 1) == 0;
    const int cp = 2 * sub + cq;
    float* ybase = P.y + ((static_cast<size_t>(bi) * g.Cp + cp) * g.Ho + oy) * g.Wo + ox;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      float out[6];
      at8_line<ScalarOps>(t[r][0], t[r][1], t[r][2], t[r][3], t[r][4], t[r][5], t[r][6], t[r][7], out[0], out[1], out[2],
                          out[3], out[4], out[5]);
      if (vec) {
#pragma unroll
        for (int c = 0; c < 6; c += 2)
          out_store<S>(reinterpret_cast<float2*>(ybase + r * g.Wo + c), make_float2(out[c], out[c + 1]));
      } else if (oy + r < g.Ho) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
          if (ox + c < g.Wo) ybase[r * g.Wo + c] = out[c];
      }
    }
  }
}

template <class S, bool PROF, bool F16>
__device__ void fi_workers(const Params& P, uint8_t* smem, Sync& sy) {
  const Geo& g = P.g;
  const int wtid = threadIdx.x - 256, lane = threadIdx.x & 31, wl = wtid >> 5;
  const ProfT<PROF> pf(P.prof && wtid == 0);
  const long long tloop = pf.now();
  constexpr int kT = S::kT, kCPC = S::kCPC;
  constexpr uint32_t kIPos = S::kIPos;
  FIWalker<S> wk;
  wk.init(P);
  int it = 0;
  for (int u = blockIdx.x; u < P.n_fi; u += P.grid, ++it) {
    int kind, b, sub;
    wk.decode(P, u, kind, b, sub);
    const int slot = it % S::kSlots;
    const uint8_t* src = smem + S::kOffFI + slot * S::kFISlot;
    long long t0 = pf.now();
    mbar_wait(&sy.fi_full[slot], (it / S::kSlots) & 1);
    pf.add(kFWWait, t0);
    t0 = pf.now();
    if (kind == 2 && (P.discard & 2)) {
      // the I unit's products are in shared memory now: drop their L2 lines
      // (dead; a write-back would cost DRAM bandwidth), 2-3 lines per worker
      // thread, ordered before the unit's release like a write
      const uint8_t* m = reinterpret_cast<const uint8_t*>(P.mring) + static_cast<size_t>(b % P.NM) * S::kMSlot +
                         static_cast<size_t>(sub) * S::kMUnit;
      for (int i = wtid; i < static_cast<int>(S::kMUnit / 128); i += 256) discard_l2(m + static_cast<size_t>(i) * 128);
    }
    if (PROF && lane == 0) trace<PROF>(b, kind == 0 ? 0 : 4, true);
#ifdef WF_TUNING_AIDS
    if (P.dbg == 4 || P.dbg == 7 || (P.dbg == 5 && kind == 0) || (P.dbg == 6 && kind == 2)) {
      // tuning aid: no transform work (4, 7: none, 5: no F, 6: no I); results invalid
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sy.fi_empty[slot]);
        red_release_cta_smem(&sy.fi_cnt[it & 3], 1);
      }
      continue;
    }
#endif

    if constexpr (S::kT == 8) {
      if (kind == 0) f_unit8<S, F16>(P, src, sy, slot, b, sub, wl, lane);
      else i_unit8<S>(P, src, sy, slot, b, sub, wtid, lane);
    } else if (kind == 0) {
      // ---- F(b, sub): thread = (tile tl, channel pair q); a warp = 8 tiles
      // (one core-matrix row group) x 4 pairs (one 8-channel k group), so
      // every store instruction writes one contiguous 128-byte core matrix
      const int part = sub / (S::C / kCPC), cg = sub % (S::C / kCPC);
      constexpr int kFT = S::kFT;
      const int tb0 = part * kFT;
      const int t0 = b * kBlockTiles + tb0;
      const int tl = wl * 8 + (lane & 7), q = lane >> 3;
      const int tile = t0 + tl;
      const bool live = tile < g.n_tile;
      float2 w[kT][kT];
      if (live) {
        const FGeo fg(g, t0, min(t0 + kFT, g.n_tile) - 1);
        const int per_img = g.tiles_y * g.tiles_x;
        const int bi = tile / per_img;
        const int rem = tile - bi * per_img;
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        const int y0 = ty * g.m - g.pad_lo;
        const int x0 = tx * g.m - g.pad_lo;
        const float* pa = reinterpret_cast<const float*>(src) + (2 * q) * P.plane + fg.srow(bi - fg.bi0, y0) * g.W + x0;
        const float* pb = pa + P.plane;
        // window columns [x0, x0 + 6) with x0 = 4 tx - 1: one aligned 16-byte
        // load [x0 + 1, x0 + 5) and two scalars per row, branch free; the
        // image's padding columns and rows are zeros (their loads are
        // predicated off or read neighbouring staged data inside the slot)
        const bool lo_ok = x0 >= 0, hi_ok = x0 + kT <= g.W;
        // K padding channels (only in 16-channel layers) are zeros, never loaded
        const int c0 = cg * kCPC + 2 * q;
        const bool ca = S::C >= 64 || c0 < g.C, cb = S::C >= 64 || c0 + 1 < g.C;
#pragma unroll
        for (int r = 0; r < kT; ++r) {
          const bool rv = y0 + r >= 0 && y0 + r < g.H;
          const float* ra = pa + r * g.W - 3;
          const float* rb = pb + r * g.W - 3;
          float4 a1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f), b1 = a1;
          float a0 = 0.0f, b0 = 0.0f, a5 = 0.0f, b5 = 0.0f;
          if (rv && ca) {
            a1 = *reinterpret_cast<const float4*>(ra + 4);
            if (lo_ok) a0 = ra[3];
            if (hi_ok) a5 = ra[8];
          }
          if (rv && cb) {
            b1 = *reinterpret_cast<const float4*>(rb + 4);
            if (lo_ok) b0 = rb[3];
            if (hi_ok) b5 = rb[8];
          }
          w[r][0] = make_float2(a0, b0);
          w[r][1] = make_float2(a1.x, b1.x);
          w[r][2] = make_float2(a1.y, b1.y);
          w[r][3] = make_float2(a1.z, b1.z);
          w[r][4] = make_float2(a1.w, b1.w);
          w[r][5] = make_float2(a5, b5);
          bt6_line<PairOps>(w[r][0], w[r][1], w[r][2], w[r][3], w[r][4], w[r][5]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy.fi_empty[slot]);     // window consumed: slot free
      {
        // columns: B^T down each column, then one column of positions
        // (r, s), r = 0..5, split (== forward_transform2<6>) and stored.
        // Lanes q and q^1 (same tile, neighbouring channel pairs) swap
        // halves so that the even one stores 4 channels of hi and the odd
        // one 4 channels of lo: one 8-byte store per position instead of
        // two 4-byte ones (a warp still writes whole core-matrix rows).
        const bool odd = q & 1;
        const int row = tb0 + tl, c0 = cg * kCPC + 2 * (q & ~1);
        uint8_t* dst = P.uring + static_cast<size_t>(b % P.NU) * S::kUSlot + (c0 / S::kKBW) * S::kAHalf +
                       (row >> 3) * (16 * S::kKBW) + ((c0 % S::kKBW) >> 3) * 128 + (row & 7) * 16 + (c0 & 7) * 2 +
                       (odd ? S::kKB * S::kAHalf : 0);
        keep_in_regs(dst);
#pragma unroll
        for (int s = 0; s < kT; ++s) {
          bt6_line<PairOps>(w[0][s], w[1][s], w[2][s], w[3][s], w[4][s], w[5][s]);
#pragma unroll
          for (int r = 0; r < kT; ++r) {
            uint32_t hi, lo;
            split2<F16>(u_operand<kT, F16>(w[r][s], r, s), hi, lo);
            const uint32_t other = __shfl_xor_sync(0xffffffffu, odd ? hi : lo, 8);
            if (live)
              ring_store<S>(reinterpret_cast<uint2*>(dst + (r * kT + s) * S::kUPos),
                         odd ? make_uint2(other, lo) : make_uint2(hi, other));
          }
        }
      }
    } else if constexpr (S::kIPairs == 1) {
      i_unit6s<S>(P, src, sy, slot, b, sub, wtid, lane);
    } else {
      // ---- I(b, sub): thread = (tile, c' pair); 36 staged float2 per thread
      const int tl = wtid & (kBlockTiles - 1), pr = wtid >> 7;
      const int tile = b * kBlockTiles + tl;
      // row pass as the staged products are read (A^T along each row; the
      // row-unit instance stages its result, computed in the GEMM epilogue),
      // then the column pass (== inverse_transform2<6>)
      constexpr int MO = kT - 2;
      float2 z[kT][MO];
      const float2* ms = reinterpret_cast<const float2*>(src + pr * kBlockTiles * 8) + tl;
      if constexpr (S::kRow) {
#pragma unroll
        for (int r = 0; r < kT; ++r)
#pragma unroll
          for (int j = 0; j < MO; ++j) z[r][j] = ms[(r * MO + j) * (kIPos / 8)];
      } else {
#pragma unroll
        for (int r = 0; r < kT; ++r) {
          float2 m[kT];
#pragma unroll
          for (int s = 0; s < kT; ++s) m[s] = ms[(r * kT + s) * (kIPos / 8)];
          at6_line<PairOps>(m[0], m[1], m[2], m[3], m[4], m[5], z[r][0], z[r][1], z[r][2], z[r][3]);
        }
      }
      // (the slot is released after the column pass has consumed every
      // staged value: the row-unit instance's loads feed no arithmetic
      // before it)
      float2 t[MO][MO];
#pragma unroll
      for (int j = 0; j < MO; ++j)
        at6_line<PairOps>(z[0][j], z[1][j], z[2][j], z[3][j], z[4][j], z[5][j], t[0][j], t[1][j], t[2][j], t[3][j]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy.fi_empty[slot]);
      if (tile < g.n_tile) {
        const int per_img = g.tiles_y * g.tiles_x;
        const int bi = tile / per_img;
        const int rem = tile - bi * per_img;
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        const int oy = ty * MO, ox = tx * MO;
        const bool vec = oy + MO <= g.Ho && ox + MO <= g.Wo && (g.Wo & 3) == 0;
        const size_t plane = static_cast<size_t>(g.Ho) * g.Wo;
        const int cp = 4 * sub + 2 * pr;
        float* ybase = P.y + (static_cast<size_t>(bi) * g.Cp + cp) * plane + static_cast<size_t>(oy) * g.Wo + ox;
#pragma unroll
        for (int r = 0; r < MO; ++r) {
          const float2 o[MO] = {t[r][0], t[r][1], t[r][2], t[r][3]};
          if (vec) {
            out_store<S>(reinterpret_cast<float4*>(ybase + r * g.Wo), make_float4(o[0].x, o[1].x, o[2].x, o[3].x));
            out_store<S>(reinterpret_cast<float4*>(ybase + plane + r * g.Wo),
                      make_float4(o[0].y, o[1].y, o[2].y, o[3].y));
          } else if (oy + r < g.Ho) {
#pragma unroll
            for (int c = 0; c < MO; ++c)
              if (ox + c < g.Wo) {
                ybase[r * g.Wo + c] = o[c].x;
                ybase[plane + r * g.Wo + c] = o[c].y;
              }
          }
        }
      }
    }
    __syncwarp();
    if (PROF && lane == 0) trace<PROF>(b, kind == 0 ? 1 : 5, false);   // before this warp's release
    if (lane == 0) red_release_cta_smem(&sy.fi_cnt[it & 3], 1);
    pf.add(kind == 0 ? kFWF : kFWI, t0);
    pf.inc(kind == 0 ? kNF : kNI);
  }
  pf.add(kFWLoop, tloop);
  pf.end(kEndFW);
}

// G units of this CTA, in block order.  A G unit is one (position, group of
// 64 output channels) of one block; CTA k owns the pair k % (36 * groups)
// for the blocks b = k / (36 * groups), + grid / (36 * groups), ... -- its V
// slab (64 x C, hi + lo) is loaded once and stays in shared memory (grid >=
// 36 * groups; the remaining CTAs have no G work).
template <class S>
struct GUnits {
  int p, ng, b0, step;
  __device__ GUnits(const Params& P) {
    constexpr int combos = S::kNGG;                      // (position or position row, c' group) pairs
    step = P.grid / combos;
    const int c = blockIdx.x % combos;
    p = c % (S::kP / S::kGP);
    ng = c / (S::kP / S::kGP);
    b0 = static_cast<int>(blockIdx.x) < step * combos ? blockIdx.x / combos : P.g.n_blk;
  }
};

// -------------------------------------------------------------- G producer
template <class S, bool PROF>
__device__ void g_producer(const Params& P, uint8_t* smem, Sync& sy, int n_g) {
  // the whole warp runs the loop (warp-uniform waits); lane 0 issues the copies
  const Geo& g = P.g;
  const int lane = threadIdx.x & 31;
  const int* doneF = P.counters;
  const int* doneI = P.counters + 2 * g.n_blk;
  const ProfT<PROF> pf(P.prof && lane == 0);
  const GUnits<S> gu(P);
  if (gu.b0 < g.n_blk && lane == 0) {
    // V of this CTA's (position, c' group), once: in the MMA pack (per
    // position a hi and a lo slab of CP x C, K blocks of 64) the group's 64
    // rows of one K block are 8 KB contiguous; smem holds [hl][K block of 64]
    mbar_expect_tx(&sy.b_full[0], S::kGP * S::kVGroup);
    const size_t slab = static_cast<size_t>(S::CP) * S::C * 2;
    for (int pl = 0; pl < S::kGP; ++pl)
      for (int hl = 0; hl < 2; ++hl)
        for (int j = 0; j < S::C / S::kVKW; ++j)
          bulk_g2s(smem + S::kOffB + pl * S::kVGroup + (hl * (S::C / S::kVKW) + j) * S::kVChunk,
                   P.vpack + (static_cast<size_t>(gu.p * S::kGP + pl) * 2 + hl) * slab +
                       static_cast<size_t>(j) * S::CP * S::kVKW * 2 + static_cast<size_t>(gu.ng) * S::kVChunk,
                   S::kVChunk, &sy.b_full[0]);
  }
  __syncwarp();
  int a_it = 0;
  for (int b = gu.b0; b < g.n_blk; b += gu.step) {
    long long t0 = pf.now();
    spin_until(doneF + b, S::kNCG);                                   // U complete
    if (b >= P.NM) spin_until(doneI + (b - P.NM), S::kNIG);           // M slot free
    pf.add(kGPDep, t0);
    if (lane == 0) trace<PROF>(b, 2, true);
    fence_proxy_async_global();
    const uint8_t* uslot = P.uring + static_cast<size_t>(b % P.NU) * S::kUSlot;
    for (int pl = 0; pl < S::kGP; ++pl) {
      const int p = gu.p * S::kGP + pl;
      for (int kb = 0; kb < S::kKB; ++kb) {
        const int st = a_it % S::kAStages;
        long long t2 = pf.now();
        mbar_wait(&sy.a_empty[st], ((a_it / S::kAStages) & 1) ^ 1);
        pf.add(kGPStage, t2);
        if (lane == 0) {
          uint8_t* adst = smem + st * S::kAStage;
          mbar_expect_tx(&sy.a_full[st], S::kAStage);
          const uint8_t* asrc = uslot + p * S::kUPos + kb * S::kAHalf;
          bulk_g2s(adst, asrc, S::kAHalf, &sy.a_full[st]);                          // hi
          bulk_g2s(adst + S::kAHalf, asrc + S::kKB * S::kAHalf, S::kAHalf, &sy.a_full[st]);    // lo
        }
        __syncwarp();
        ++a_it;
      }
    }
  }
  pf.end(kEndGP);
}

// ---------------------------------------------------------------- G issuer
template <class S, bool PROF>
__device__ void g_issuer(const Params& P, uint8_t* smem, Sync& sy, int n_g) {
  // the whole warp runs the loop; lane 0 issues the MMAs
  const int lane = threadIdx.x & 31;
  constexpr int kN = S::kN;
  const uint32_t idesc = idesc_bf16(kBlockTiles, kN, false, false, prec_f16(P.passes));
  const ProfT<PROF> pf(P.prof);
  const GUnits<S> gu(P);
  if (gu.b0 < P.g.n_blk) mbar_wait(&sy.b_full[0], 0);            // the resident V slab
  const uint32_t sb = smem_u32(smem + S::kOffB);
  int a_it = 0, k = 0;
  for (int b = gu.b0; b < P.g.n_blk; b += gu.step, ++k) {
    const int buf = k % S::kAcc;
    long long t0 = pf.now();
    mbar_wait(&sy.tempty[buf], ((k / S::kAcc) & 1) ^ 1);
    pf.add(kGITempty, t0);
    tc_fence_after();
   for (int pl = 0; pl < S::kGP; ++pl) {
    const uint32_t dcol = sy.tmem + (buf * S::kGP + pl) * kN;
    const uint32_t sbp = sb + pl * S::kVGroup;             // the unit's pl-th position
    for (int kb = 0; kb < S::kKB; ++kb) {
      const int st = a_it % S::kAStages;
      long long t2 = pf.now();
      mbar_wait(&sy.a_full[st], (a_it / S::kAStages) & 1);
      pf.add(kGIFull, t2);
      tc_fence_after();
      __syncwarp();
      if (lane == 0) {
        const uint32_t sa = smem_u32(smem + st * S::kAStage);
#pragma unroll
        for (int s = 0; s < S::kKBW / 16; ++s) {
          const uint64_t ahi = smem_desc(sa + s * 256, 128, 16 * S::kKBW);
          const uint64_t alo = smem_desc(sa + S::kAHalf + s * 256, 128, 16 * S::kKBW);
          // V: [hl][pack K block][64 rows x kVKW k]; channel k0 of this K step
          const int k0 = kb * S::kKBW + s * 16;
          const uint32_t voff = (k0 / S::kVKW) * S::kVChunk + ((k0 % S::kVKW) >> 3) * 128;
          const uint64_t bhi = smem_desc(sbp + voff, 128, 16 * S::kVKW);
          const uint64_t blo = smem_desc(sbp + S::kVHalf + voff, 128, 16 * S::kVKW);
          const uint32_t first = (kb == 0 && s == 0) ? 0u : 1u;
          if (prec_passes(P.passes) > 1) {
            mma_bf16_ss(dcol, alo, bhi, idesc, first);
            mma_bf16_ss(dcol, ahi, blo, idesc, 1u);
            mma_bf16_ss(dcol, ahi, bhi, idesc, 1u);
          } else {
            mma_bf16_ss(dcol, ahi, bhi, idesc, first);
          }
        }
        mma_commit(&sy.a_empty[st]);
        if (kb == S::kKB - 1) mma_commit(&sy.tfull[buf][pl]);
      }
      __syncwarp();
      ++a_it;
    }
   }
  }
  pf.end(kEndGI);
}

// -------------------------------------------------------------- G epilogue
template <class S, bool PROF>
__device__ void g_epilogue(const Params& P, Sync& sy, int n_g) {
  const int lane = threadIdx.x & 31, qd = (threadIdx.x >> 5) & 3;
  const int row = qd * 32 + lane;
  const ProfT<PROF> pf(P.prof && qd == 0 && lane == 0);
  const GUnits<S> gu(P);
  const int gg = gu.p;
  constexpr int kN = S::kN;
  int k = 0;
  for (int b = gu.b0; b < P.g.n_blk; b += gu.step, ++k) {
    const int buf = k % S::kAcc;
    const bool live = b * kBlockTiles + row < P.g.n_tile;
    float* mslot = P.mring + static_cast<size_t>(b % P.NM) * (S::kMSlot / 4);
    if constexpr (S::kRow) {
      // ---- row unit: the six products (r, 0..5) of this thread's tile, 4
      // output channels at a time -> row pass of the inverse transform
      // (A^T along the row, == the first pass of inverse6) -> M ring, 4
      // values per (tile, c'): [I unit c' / 4][r][j][pair][tile][2]
      long long t0 = pf.now();
      for (int pl = 0; pl < S::kGP; ++pl) mbar_wait(&sy.tfull[buf][pl], (k / S::kAcc) & 1);
      pf.add(kGEWait, t0);
      t0 = pf.now();
      tc_fence_after();
      const uint32_t taddr = sy.tmem + (static_cast<uint32_t>(qd * 32) << 16) + buf * (S::kGP * kN);
      float2* mrow = reinterpret_cast<float2*>(mslot) + row;
#pragma unroll 2
      for (int c = 0; c < kN; c += 4) {
        float m[6][4];
#pragma unroll
        for (int pl = 0; pl < 6; ++pl) tmem_ld4(taddr + pl * kN + c, m[pl]);
        tmem_ld_wait();
        float z[4][4];                                   // [c' in chunk][j]
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          at6_line<ScalarOps>(m[0][cc], m[1][cc], m[2][cc], m[3][cc], m[4][cc], m[5][cc], z[cc][0], z[cc][1], z[cc][2],
                              z[cc][3]);
        if (live) {
          // I unit c / 4 (C' = 64: one c' group), pairs (c, c + 1) and (c + 2, c + 3)
          float2* mu = mrow + static_cast<size_t>(c / 4) * (S::kMUnit / 8) + static_cast<size_t>(gg) * (4 * S::kIPos / 8);
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int pr = 0; pr < 2; ++pr)
              ring_store<S>(mu + (j * 2 + pr) * kBlockTiles, make_float2(z[2 * pr][j], z[2 * pr + 1][j]));
        }
      }
      pf.add(kGEBusy, t0);
    } else
    for (int pl = 0; pl < S::kGP; ++pl) {
      long long t0 = pf.now();
      mbar_wait(&sy.tfull[buf][pl], (k / S::kAcc) & 1);
      pf.add(kGEWait, t0);
      t0 = pf.now();
      tc_fence_after();
      const uint32_t taddr = sy.tmem + (static_cast<uint32_t>(qd * 32) << 16) + buf * (S::kGP * kN) + pl * kN;
      // pair k of position p: [k / kIPairs][p][k % kIPairs][tile][2] (see
      // Shape::kMUnit); this unit's 64 outputs are the pairs 32 ng .. 32 ng + 31
      float2* mrow = reinterpret_cast<float2*>(mslot + static_cast<size_t>(gg * S::kGP + pl) * (S::kIPos / 4)) + row;
#pragma unroll
      for (int c = 0; c < kN; c += 16) {
        float vv[16];
        tmem_ld16(taddr + c, vv);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int k = gu.ng * (kN / 2) + c / 2 + i;
            ring_store<S>(mrow + (k / S::kIPairs) * (S::kMUnit / 8) + (k % S::kIPairs) * kBlockTiles,
                   make_float2(vv[2 * i], vv[2 * i + 1]));
          }
        }
      }
      pf.add(kGEBusy, t0);
    }
    tc_fence_before();
    if ((P.discard & 1) && S::kNG == 1) {
      // the unit's U (one position, read by this unit only when C' = 64) is
      // dead: drop its L2 lines before the unit is published (publishing
      // lets the next F units of the ring slot write it again).
      // Row units: every epilogue warp fences (gpu scope) between its M
      // stores and its burst of discards (12 per thread).  Without the
      // fence about one call in 500 produced wrong values in one warp's
      // stores of one 4-channel chunk (DESIGN.md 5.5 lists what was
      // measured; the mechanism is not pinned down); with it 0 in 20000
      // calls.  The one-position units (2 discards per thread) show 0
      // mismatches in 60000 calls and keep the cheaper chain (a fence per
      // warp costs them 80 -> 92 us on c2).
      if constexpr (S::kRow) {
        __syncwarp();
        if (lane == 0) fence_acq_rel_gpu();
        __syncwarp();
      }
      const uint8_t* u = P.uring + static_cast<size_t>(b % P.NU) * S::kUSlot + gg * S::kGP * S::kUPos;
      constexpr int lines = static_cast<int>(S::kGP * S::kUPos / 128);
      for (int i = qd * 32 + lane; i < lines; i += 128) discard_l2(u + static_cast<size_t>(i) * 128);
    }
    __syncwarp();
    if (lane == 0) {
      // the last of the 4 epilogue warps to finish publishes the unit (counted
      // before the buffer is released, so no warp can count a later use of
      // this buffer first)
      if (atom_acqrel_cta_smem(&sy.g_cnt[buf], 1) == 4 * (k / S::kAcc) + 3) {
        const long long t1 = pf.now();
        trace<PROF>(b, 3, false);    // before the release that publishes it
        if (P.gbatch == 1) {
          red_release_gpu(P.counters + P.g.n_blk + b, 1);
        } else if (k % P.gbatch == P.gbatch - 1 || b + gu.step >= P.g.n_blk) {
          // batched publish (narrow C': the fence, not the GEMM, bounds the
          // G roles): acquire the batch's earlier units through their
          // completion counts, one fence, then the counts of every unit
          const int k0 = k - k % P.gbatch;
          for (int j = k0; j < k; ++j) (void)ld_acquire_cta_smem(&sy.g_cnt[j % S::kAcc]);
          fence_acq_rel_gpu();
          for (int j = k0; j <= k; ++j) red_relaxed_gpu(P.counters + P.g.n_blk + gu.b0 + j * gu.step, 1);
        }
        pf.add(kPubFence, t1);
      }
      mbar_arrive(&sy.tempty[buf]);
    }
  }
  pf.end(kEndGE);
}

// --------------------------------------------------------------- publisher
template <class S, bool PROF>
__device__ void publisher(const Params& P, Sync& sy, int n_g) {
  // lane 0 polls the per-unit worker counts and publishes the unit
  const int lane = threadIdx.x & 31;
  const ProfT<PROF> pf(P.prof && lane == 0);
  int* doneF = P.counters;
  int* doneI = doneF + 2 * P.g.n_blk;
  FIWalker<S> wk;
  wk.init(P);
  int kf = 0;
  for (int uf = blockIdx.x; uf < P.n_fi; uf += P.grid, ++kf) {
    while (ld_acquire_cta_smem(&sy.fi_cnt[kf & 3]) < 8 * ((kf >> 2) + 1)) __nanosleep(32);   // warp-uniform
    int kind, b, sub;
    wk.decode(P, uf, kind, b, sub);
    if (lane == 0) {
      const long long t0 = pf.now();
      red_release_gpu((kind == 0 ? doneF : doneI) + b, 1);
      pf.add(kPubFence, t0);
    }
  }
  (void)n_g;
  pf.end(kEndPub);
}

template <class S, bool PROF, bool F16>
__global__ void __launch_bounds__(NT, 1) fused_ws_kernel(Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Sync sy;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S::kAStages; ++s) { mbar_init(&sy.a_full[s], 1); mbar_init(&sy.a_empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sy.b_full[s], 1);
      mbar_init(&sy.b_empty[s], 1);
    }
    for (int s = 0; s < S::kSlots; ++s) {
      mbar_init(&sy.fi_full[s], 1);
      mbar_init(&sy.fi_empty[s], 8);
    }
    for (int s = 0; s < kNAcc; ++s) {
      for (int p = 0; p < kMaxGP; ++p) mbar_init(&sy.tfull[s][p], 1);
      mbar_init(&sy.tempty[s], 4);
    }
    for (int i = 0; i < 4; ++i) sy.fi_cnt[i] = 0;
    for (int i = 0; i < kNAcc; ++i) sy.g_cnt[i] = 0;
    for (int i = 0; i < kProfSlots; ++i) s_prof[i] = 0;
    if (PROF) g_wsprof[blockIdx.x * kProfSlots + kStart] = gtimer();
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<S::kTmemCols>(&sy.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // 512 threads x 128 registers fill the register file at launch; the
  // single-lane roles (warps 0-3) and the epilogue (4-7) hand registers to
  // the transform warps (8-15): 4*32*40 + 4*32*64 + 8*32*200 <= 64K.  Each
  // warpgroup re-sizes inside its own branch so ptxas allocates every
  // role's code under its own limit.
  const int n_g = P.g.n_blk * S::kNGG;
  if (warp < 4) {
    regs_dec<kRegsLight>();
    if (P.dbg == 3 || P.dbg == 7) {
      // tuning aid: no GEMM work, every G unit is published at once (results invalid)
      if (warp == 0) {
        if (lane_id() == 0)
          for (int v = blockIdx.x; v < n_g; v += P.grid) red_release_gpu(P.counters + P.g.n_blk + v / S::kNGG, 1);
      } else if (warp == 2) {
        fi_producer<S, PROF>(P, smem, sy);
      } else if (warp == 3) {
        publisher<S, PROF>(P, sy, n_g);
      }
    } else if (warp == 0) {
      g_producer<S, PROF>(P, smem, sy, n_g);
    } else if (warp == 1) {
      g_issuer<S, PROF>(P, smem, sy, n_g);
    } else if (warp == 2) {
      fi_producer<S, PROF>(P, smem, sy);
    } else {
      publisher<S, PROF>(P, sy, n_g);
    }
  } else if (warp < 8) {
    regs_dec<kRegsEpi>();
    if (P.dbg != 3 && P.dbg != 7) g_epilogue<S, PROF>(P, sy, n_g);
  } else {
    regs_inc<kRegsFI>();
    fi_workers<S, PROF, F16>(P, smem, sy);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<S::kTmemCols>(sy.tmem);
  }
  // The last CTA to finish zeroes the dependency counters, so a caller that
  // owns this scratch can skip the memset before the next launch
  // (wf_conv_fused_planned).  Every CTA finished all its counter accesses
  // before its release increment; the last one acquires them all.
  {
    __shared__ int last;
    int* done = P.counters + 3 * P.g.n_blk;
    if (tid == 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(done) : "memory");
      last = old == P.grid - 1;
    }
    __syncthreads();
    if (last)
      for (int i = tid; i <= 3 * P.g.n_blk; i += NT) P.counters[i] = 0;
  }
  if (PROF && tid < kProfSlots && (tid < kStart || tid > kEndPub)) g_wsprof[blockIdx.x * kProfSlots + tid] += s_prof[tid];
}

struct Plan {
  bool ok;
  int NU, NM, L2, plane;
  size_t counters_bytes, u_slot, m_slot;
};

// floats per staged channel of an F unit of kft tiles: the largest unit's rows
static int fi_plane(const Geo& g, int kft) {
  int max_rows = 0;
  for (int t0 = 0; t0 < g.n_tile; t0 += kft) {
    const FGeo fg(g, t0, std::min(t0 + kft, g.n_tile) - 1);
    max_rows = std::max(max_rows, fg.total());
  }
  return round_up(max_rows * g.W, 32) + 16;
}
// The row-unit instance (F(4x4,3x3), C = C' = 64) has 48 KB F/I slots next to
// its six resident V slabs: it runs where an F unit's input rows fit them
// (W = 56: yes; W = 224: no) and the device has a CTA per position row.
static bool row_units_fit(const Geo& g) {
  if (g.T != 6 || g.fft || g.Cpad != 64 || g.C != 64 || g.Cp != 64 || g.Cppad != 64) return false;
  if (g.W % 4 != 0 || g.pad_lo != 1 || g.W < 8) return false;
  return static_cast<size_t>(8) * fi_plane(g, 64) * 4 <= 48 * 1024;
}

template <class S>
static Plan plan_t(const Geo& g, const FusedOpts& o) {
  Plan pl = {};
  // the bulk-copied input rows must be 16-byte aligned (W % 4 == 0); the
  // branch-free window loads assume pad_lo = 1
  if (g.W % 4 != 0 || g.m != S::kT - 2 || g.pad_lo != 1 || g.W < 8) return pl;
  pl.plane = fi_plane(g, S::kFT);
  if (static_cast<size_t>(S::kCPC) * pl.plane * 4 > S::kFISlot) return pl;
  // ring budget 140 MB (the U + M rings of c2 take 70 MB: inside the 126 MB
  // L2 next to the streamed input and output).  Measured (tools/ring_sweep.py,
  // c2): budget 100 / 120 / 140 / 200 / 300 MB -> 103 / 87 / 82 / 81 / 82 us;
  // smaller rings starve the lagged pipeline
  size_t budget = o.ring_bytes ? o.ring_bytes : static_cast<size_t>(tuning_knob("WF_WS_BUDGET_MB", 140)) << 20;
  int slots = static_cast<int>(budget / (S::kUSlot + S::kMSlot));
  if (slots < 4) slots = 4;
  pl.NU = std::min(slots / 2, g.n_blk);
  pl.NM = std::min(slots - slots / 2, g.n_blk);
  // the lag counts steps; a step is one block's F and I units, so the lag
  // that keeps a fixed number of units between a block's F and I units
  // shrinks with the units per step (measured best: c2, 32 units per step,
  // 32 steps; VGG 64->128 / 128->128 / 128->256 / 256->256, 48 / 64 / 96 /
  // 192 units, 16 / 12 / 8 / 4 steps; c5 64->64 and 128->128 about the same;
  // c5 16->16, 16 units, 64 steps with 8-unit G publish batches)
  const int units = S::kNCG + S::kNIG;
  // (VGG 3 -> 64 with two-position G units, 20 units per step: 40 .. 56 steps
  // measured 316 us, 32 steps 334 us)
  int lag = units <= 16 ? 64 : units <= 24 ? 48 : units <= 32 ? 32 : std::max(4, std::min(32, 768 / units));
  if (o.lag > 0) lag = o.lag;
  else if (const int k = tuning_knob("WF_WS_LAG", 0)) lag = k;
  // deadlock freedom: some L1 with 1 <= L1 < NU (when F waits on G) and L2 - L1 < NM
  const int lmax = (pl.NU >= g.n_blk ? g.n_blk + pl.NM : pl.NU + pl.NM - 2);
  if (lag > lmax) lag = lmax;
  if (lag < 2) lag = 2;
  pl.L2 = lag;
  if (pl.NU < 2 && pl.NU < g.n_blk) return pl;
  pl.counters_bytes = static_cast<size_t>(3 * g.n_blk + 1) * sizeof(int);   // + finished-CTA count
  pl.u_slot = S::kUSlot;
  pl.m_slot = S::kMSlot;
  pl.ok = true;
  return pl;
}

// Shapes with a kernel instance: T = 6 with Cpad in {64, 128} (= C) and 16
// (C <= 16), C' (= C'pad) in {64, 128, 256}; T = 8 with C = C' in {64, 128}
// -- every (position, c' group) pair gets a CTA of its own (T^2 x C'/64 <=
// 148), and A stages + V + two F/I slots fit smem.
template <class F>
static auto with_shape(const Geo& g, const FusedOpts& o, F&& f) -> decltype(f(Shape<6, 64, 64>())) {
  using R = decltype(f(Shape<6, 64, 64>()));
  if (o.variant == kVarWSRow) return row_units_fit(g) ? f(Shape<6, 64, 64, 2, 6>()) : R();
  // C = Cpad except for the 16-channel instance, which zero-pads C <= 16
  // (VGG's RGB layer); C' = C'pad
  if (g.fft || g.Cp != g.Cppad || (g.C != g.Cpad && g.Cpad != 16)) return R();
  switch (g.T * 1000000 + g.Cpad * 1000 + g.Cp) {
#ifdef WF_WS_ONLY   // tuning builds (tools/build_alt.sh): one instance, compiles in 40 s
#ifndef WF_WS_ONLY_GP
#define WF_WS_ONLY_GP 1
#endif
    case WF_WS_ONLY: return f(Shape<WF_WS_ONLY / 1000000, (WF_WS_ONLY / 1000) % 1000, WF_WS_ONLY % 1000, 2, WF_WS_ONLY_GP>());
#else
    // (two positions per G unit where it measured faster and the V slabs
    // fit: VGG 3 -> 64 @224 359 -> 332 us, 64 -> 128 @112 224 -> 211 us;
    // 64 -> 64 and F(6x6,3x3) 32 -> 32 / 64 -> 64 measured equal or slower)
    case 6016064: return f(Shape<6, 16, 64, 2, 2>());
    case 6064064: return f(Shape<6, 64, 64>());
    case 6064128: return f(Shape<6, 64, 128, 2, 2>());
    case 6064256: return f(Shape<6, 64, 256>());
    case 6128064: return f(Shape<6, 128, 64>());
    case 6128128: return f(Shape<6, 128, 128>());
    case 6128256: return f(Shape<6, 128, 256>());
    case 6256256: return f(Shape<6, 256, 256>());   // VGG conv3_2/3_3 (36 x 4 = 144 CTAs)
    // F(6x6,3x3): the c5 sweep's layers (64 x C'/64 <= 148); C' < 64 runs
    // G units of N = C'
    // positions per G unit of the narrow instances: the 16-channel layers'
    // G roles are bound by the per-unit latency (dependency poll, 8 KB of
    // U, 3 MMAs, publish); two positions per unit measured 15-21% faster
    // on the c5 16 -> 16 layers (419 -> 331 us @112), four slower; the
    // 32-channel layers show no difference
#ifndef WF_WS_GP16
#define WF_WS_GP16 2
#endif
#ifndef WF_WS_GP32
#define WF_WS_GP32 1
#endif
    case 8016016: return f(Shape<8, 16, 16, 2, WF_WS_GP16>());
    case 8032032: return f(Shape<8, 32, 32, 2, WF_WS_GP32>());
    case 8064064: return f(Shape<8, 64, 64>());
    case 8128128: return f(Shape<8, 128, 128>());
#endif
  }
  return R();
}

static Plan plan(const Geo& g, const FusedOpts& o) {
  return with_shape(g, o, [&](auto s) { return plan_t<decltype(s)>(g, o); });
}

template <class S>
static cudaError_t launch_t(const Params& P, int sm_count, cudaStream_t st) {
  // units of a CTA wait on units of other CTAs: every CTA must be resident
  const bool f16 = prec_f16(P.passes);
  const void* kern = P.prof ? (f16 ? reinterpret_cast<const void*>(fused_ws_kernel<S, true, true>)
                                   : reinterpret_cast<const void*>(fused_ws_kernel<S, true, false>))
                            : (f16 ? reinterpret_cast<const void*>(fused_ws_kernel<S, false, true>)
                                   : reinterpret_cast<const void*>(fused_ws_kernel<S, false, false>));
  Params p = P;
  void* args[] = {&p};
  return launch_coresident(kern, sm_count, NT, S::kSmem, st, args);
}

}  // namespace ws

bool ws_fits(const Geo& g, const FusedOpts& o) {
  const ws::Plan pl = ws::plan(g, o);
  if (!pl.ok) return false;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a CTA per (position, c' group)
  return ws::with_shape(g, o, [&](auto s) { return sms >= decltype(s)::kNGG; });
}

size_t ws_scratch_bytes(const Geo& g, const FusedOpts& o) {
  const ws::Plan pl = ws::plan(g, o);
  if (!pl.ok) return 0;
  return round_up(static_cast<int>(pl.counters_bytes), 1024) + pl.NU * pl.u_slot + pl.NM * pl.m_slot;
}

cudaError_t run_fused_ws(const float* x, const uint8_t* vpack, float* y, uint8_t* scratch, const Geo& g, int passes,
                         int sm_count, cudaStream_t st, const FusedOpts& o) {
  const ws::Plan pl = ws::plan(g, o);
  const bool counters_clean = (o.flags & kFusedCountersClean) != 0;
  if (!pl.ok) return cudaErrorInvalidValue;
  ws::Params P;
  P.x = x; P.y = y; P.vpack = vpack;
  P.counters = reinterpret_cast<int*>(scratch);
  P.uring = scratch + round_up(static_cast<int>(pl.counters_bytes), 1024);
  P.mring = reinterpret_cast<float*>(P.uring + pl.NU * pl.u_slot);
  P.g = g;
  P.NU = pl.NU; P.NM = pl.NM; P.L2 = pl.L2;
  P.passes = passes;
  // Dead ring lines dropped from L2 (discard.global.L2) instead of being
  // written back (bit 1: U, by the G epilogue; bit 2: M, by the I workers).
  // Measured with the L2 eviction priorities (Hints) and 70 MB rings
  // (tools/ring_sweep.py under ncu, L2 cleaned before the call): c2 without
  // discards 170 MB of DRAM per call at 79.9 us, with the U discards 97 MB
  // (0.94 x Q_fused) at 81.9 us; c5 64->64 @56 866 MB without, 554 MB with
  // U, 449 MB (1.09 x Q_fused) with M discards at +2.5% (128->128 @112 +7%),
  // 385 MB with both at +6%.  The 16-channel (RGB) instance runs without.
  P.discard = tuning_knob("WF_WS_DISCARD", g.T == 8 ? 2 : (g.Cpad > 16 ? 1 : 0));
  P.dbg = 0;
#ifdef WF_TUNING_AIDS
  // ablations (results invalid): 3 no GEMM work, 4 no transform work, 5 no F, 6 no I, 7 = 3 + 4
  P.dbg = tuning_knob("WF_WS_DBG", 0);
#endif
  P.plane = pl.plane;
  P.grid = sm_count;
  // the instrumented instance: per-role busy cycles and per-block ordering
  // tickets (wf_fused_instrument_read)
  P.prof = (o.flags & kFusedInstrument) ? 1 : 0;
  if (P.prof) {
    cudaError_t e = ws_instrument_reset(g.n_blk, st);
    if (e != cudaSuccess) return e;
  }
  if (!counters_clean) {
    cudaError_t e = cudaMemsetAsync(P.counters, 0, pl.counters_bytes, st);
    if (e != cudaSuccess) return e;
  }
  return ws::with_shape(g, o, [&](auto s) {
    using S = decltype(s);
    P.n_fi = g.n_blk * (S::kNCG + S::kNIG);
    // G publishes batched for C' <= 32 (4 units per fence).  A batch delays
    // the publish of its first unit until its last unit (step * (batch - 1)
    // blocks later) is done, which must stay inside the ring and lag slack
    // the deadlock-freedom argument uses.
    const int step = std::max(1, sm_count / S::kNGG);
    int gb = S::CP <= 16 ? 8 : S::CP <= 32 ? 4 : 1;
    if (o.gbatch > 0) gb = std::min(S::kAcc, o.gbatch);
    else if (const int k = tuning_knob("WF_WS_GBATCH", 0)) gb = std::max(1, std::min(S::kAcc, k));
    while (gb > 1 && (gb - 1) * step >= std::min(P.L2, std::min(P.NU, P.NM))) --gb;
    // ... and a batch makes G(b)'s publish wait for F(b + (batch - 1) * step):
    // the largest deadlock-free lag (plan_t: NU + NM - 2 when F waits on G)
    // shrinks by that many blocks.  A requested lag beyond it (wf_fused_opts.
    // lag, WF_WS_LAG) shrinks the batch, not the other way round.
    if (P.NU < g.n_blk)
      while (gb > 1 && P.L2 > P.NU + P.NM - 2 - (gb - 1) * step) --gb;
    P.gbatch = gb;
    return ws::launch_t<S>(P, sm_count, st);
  });
}


}  // namespace wf

// Debug/tuning hook (not part of the public ABI): copy the per-CTA role
// accounting of the warp-specialised kernel ([cta][32] u64) and reset it.
extern "C" int wf_debug_ws_profile(unsigned long long* host, int n) {
  const int cnt = n < 1024 * wf::ws::kProfSlots ? n : 1024 * wf::ws::kProfSlots;
  cudaError_t e = cudaMemcpyFromSymbol(host, wf::ws::g_wsprof, cnt * sizeof(unsigned long long));
  static unsigned long long zeros[1024 * wf::ws::kProfSlots] = {0};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(wf::ws::g_wsprof, zeros, sizeof(zeros));
  return e == cudaSuccess ? 0 : 4;
}

namespace wf {
cudaError_t ws_instrument_reset(int n_blk, cudaStream_t st) {
  (void)n_blk;
  void* p = nullptr;
  cudaError_t e = cudaGetSymbolAddress(&p, ws::g_wstrace);
  if (e == cudaSuccess) e = cudaMemsetAsync(p, 0xff, sizeof(ws::g_wstrace), st);
  if (e == cudaSuccess) e = cudaGetSymbolAddress(&p, ws::g_wsticket);
  if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaGetSymbolAddress(&p, ws::g_wsprof);
  if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(ws::g_wsprof), st);
  return e;
}

int ws_instrument_read(const Geo& g, const FusedOpts& o, unsigned long long* events, int n_events,
                       unsigned long long* role_cycles, int* nu_nm) {
  const ws::Plan pl = ws::plan(g, o);
  if (!pl.ok) return -1;
  nu_nm[0] = pl.NU;
  nu_nm[1] = pl.NM;
  const int nb = g.n_blk < ws::kTraceBlocks ? g.n_blk : ws::kTraceBlocks;
  const int cnt = (n_events < nb * 8 ? n_events : nb * 8);
  if (cudaMemcpyFromSymbol(events, ws::g_wstrace, cnt * sizeof(unsigned long long)) != cudaSuccess) return -1;
  static unsigned long long prof[1024 * ws::kProfSlots];
  if (cudaMemcpyFromSymbol(prof, ws::g_wsprof, sizeof(prof)) != cudaSuccess) return -1;
  unsigned long long f = 0, gg = 0, i = 0;
  for (int c = 0; c < 1024; ++c) {
    f += prof[c * ws::kProfSlots + ws::kFWF];
    gg += prof[c * ws::kProfSlots + ws::kGEBusy];
    i += prof[c * ws::kProfSlots + ws::kFWI];
  }
  role_cycles[0] = f;
  role_cycles[1] = gg;
  role_cycles[2] = i;
  int dev = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  role_cycles[3] = static_cast<unsigned long long>(khz);
  return nb;
}
}  // namespace wf
