// Microbenchmarks + layout checks for the sm_100a primitives the fused
// transformed-convolution kernel is built on.  Not part of the product; the
// numbers it prints drive the design choices recorded in DESIGN.md.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_1912_02165_b200/csrc ubench.cu -o ubench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include <cuda_bf16.h>
#include "sm100.cuh"

using namespace wf;

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

// byte offset of (r, k) in the interleaved K-major layout with K total cols
__host__ __device__ inline uint32_t il_off(uint32_t r, uint32_t k, uint32_t K) {
  return (r / 8) * (16 * K) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
}

// ---------------------------------------------------------------- check GEMM
// D[M x N] = A[M x K] * B[N x K]^T, one CTA, 128 threads.  mode 0 = SS, 1 = TS
template <int M, int N, int K>
__global__ void gemm_check(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 2;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < M * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + il_off(r, k, K)) = __float2bfloat16(A[i]);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sB + il_off(r, k, K)) = __float2bfloat16(B[i]);
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t dcol = tbase;          // D at column 0
  const uint32_t acol = tbase + 256;    // A (TS mode) at column 256
  if (mode == 1) {
    // write A into TMEM: lane = row, column = k/2, packed (k even -> low half)
    const int row = tid;  // 128 threads, M = 128
    if (row < M) {
      for (int kc = 0; kc < K / 16; ++kc) {
        uint32_t w[8];
        for (int j = 0; j < 8; ++j) {
          float a0 = A[row * K + kc * 16 + 2 * j];
          float a1 = A[row * K + kc * 16 + 2 * j + 1];
          w[j] = pack_bf16x2(a0, a1);
        }
        tmem_st8(acol + ((uint32_t)(warp * 32) << 16) + kc * 8, w);
      }
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16(M, N);
      for (int kc = 0; kc < K / 16; ++kc) {
        uint64_t bd = smem_desc(smem_u32(sB) + kc * 256, 128, 16 * K);
        if (mode == 0) {
          uint64_t ad = smem_desc(smem_u32(sA) + kc * 256, 128, 16 * K);
          mma_bf16_ss(dcol, ad, bd, idesc, kc > 0);
        } else {
          mma_bf16_ts(dcol, acol + kc * 8, bd, idesc, kc > 0);
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // read back: thread = row
  const int row = tid;
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(dcol + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int M, int N, int K>
bool run_check(int mode) {
  std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 17 - 8);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  size_t sm = (M + N) * K * 2;
  CK(cudaFuncSetAttribute(gemm_check<M, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  gemm_check<M, N, K><<<1, 128, sm>>>(dA, dB, dD, mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M * N; ++i)
    if (D[i] != R[i]) {
      if (bad < 5) printf("  mismatch %d (m=%d n=%d): got %f want %f\n", i, i / N, i % N, D[i], R[i]);
      ++bad;
    }
  printf("gemm_check M=%d N=%d K=%d mode=%s : %s (%d bad)\n", M, N, K, mode ? "TS" : "SS",
         bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

// ------------------------------------------------------------ MMA rate
// Each CTA issues `iters` x (K/16) MMAs on resident smem; one commit per group.
template <int M, int N, int K, int MODE>
__global__ void mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 2;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (M + N) * K * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    unsigned long long t0 = clock64();
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16(M, N);
      for (int it = 0; it < iters; ++it) {
        for (int kc = 0; kc < K / 16; ++kc) {
          uint64_t bd = smem_desc(smem_u32(sB) + kc * 256, 128, 16 * K);
          const uint32_t d = tbase + (it & 1) * N;
          if (MODE == 0) {
            uint64_t ad = smem_desc(smem_u32(sA) + kc * 256, 128, 16 * K);
            mma_bf16_ss(d, ad, bd, idesc, kc > 0);
          } else {
            mma_bf16_ts(d, tbase + 256 + kc * 8, bd, idesc, kc > 0);
          }
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane_id() == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int M, int N, int K, int MODE>
void run_rate(int nsm) {
  const int iters = 4000;
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  size_t sm = (M + N) * K * 2;
  CK(cudaFuncSetAttribute(mma_rate<M, N, K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  mma_rate<M, N, K, MODE><<<nsm, 128, sm>>>(10, dc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<M, N, K, MODE><<<nsm, 128, sm>>>(iters, dc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> c(nsm);
  CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (auto x : c) avg += x; avg /= nsm;
  double macs = (double)iters * M * N * K;
  printf("mma_rate %s M=%3d N=%3d K=%d: %.1f cyc/mma(K16)  %.0f MAC/clk/SM  chip %.1f TFLOP/s (%.3f ms)\n",
         MODE ? "TS" : "SS", M, N, K, avg / (iters * (K / 16)), macs / avg,
         2.0 * macs * nsm / (ms * 1e-3) / 1e12, ms);
  cudaFree(dc);
}

// ------------------------------------------------------------ L2 broadcast read
// Every CTA streams the same `bytes` buffer `reps` times with 16B loads.
__global__ void l2_read(const uint4* __restrict__ buf, size_t n16, int reps, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r) {
    size_t start = (size_t)(blockIdx.x * 37 + r * 101) % n16;  // de-synchronise CTAs a bit
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
      size_t j = i + start; if (j >= n16) j -= n16;
      uint4 v = __ldcg(buf + j);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678) sink[blockIdx.x] = acc;
}

// Same, but with 1-D bulk copies into a smem ring (the TMA path).
__global__ void l2_bulk(const uint8_t* __restrict__ buf, size_t bytes, int reps, int chunk,
                        int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    size_t nch = bytes / chunk;
    uint32_t phase[4] = {0, 0, 0, 0};
    size_t issued = 0, total = nch * reps;
    size_t off0 = (size_t)blockIdx.x * 7 % nch;
    for (; issued < total && issued < 4; ++issued) {
      mbar_expect_tx(&bars[issued], chunk);
      bulk_g2s(smem + issued * chunk, buf + ((issued + off0) % nch) * chunk, chunk, &bars[issued]);
    }
    for (size_t done = 0; done < total; ++done) {
      int s = done % 4;
      mbar_wait(&bars[s], phase[s]);
      phase[s] ^= 1;
      if (issued < total) {
        mbar_expect_tx(&bars[s], chunk);
        bulk_g2s(smem + s * chunk, buf + ((issued + off0) % nch) * chunk, chunk, &bars[s]);
        ++issued;
      }
    }
    sink[blockIdx.x] = smem[5];
  }
}

// ------------------------------------------------------------ DSMEM push
__global__ void __cluster_dims__(2, 1, 1) dsmem_push(int reps, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int bytes = 64 * 1024;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  uint32_t local = smem_u32(smem), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1));
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
      asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(remote + i), "r"(r), "r"(i), "r"(r), "r"(i) : "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[7];
}


// ------------------------------------------------------------ DSMEM bulk copy (TMA engine)
// CTA r copies a 32 KB smem block into CTA r^1's smem with cp.async.bulk.shared::cluster.shared::cta
__global__ void __cluster_dims__(2, 1, 1) dsmem_bulk(int reps, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  const int bytes = 32 * 1024;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t dst_local = smem_u32(smem + bytes), dst_remote, bar_remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst_remote) : "r"(dst_local), "r"(rank ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar_remote) : "r"(smem_u32(&bar)), "r"(rank ^ 1));
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      mbar_expect_tx(&bar, bytes);   // expect the peer's copy into my smem
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst_remote), "r"(smem_u32(smem)), "r"(bytes), "r"(bar_remote) : "memory");
      mbar_wait(&bar, r & 1);
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[bytes + 7];
}

// ------------------------------------------------------------ multicast bulk load
// cluster of 4: each CTA loads 1/4 of a 64 KB chunk and multicasts it to all 4.
template <int CS>
__global__ void mcast_load(const uint8_t* __restrict__ buf, size_t bytes, int reps, int mc, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  const int chunk = 64 * 1024;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const size_t nch = bytes / chunk;
  const size_t cl = blockIdx.x / CS, ncl = gridDim.x / CS;
  for (int r = 0; r < reps; ++r) {
    const size_t c = (cl + r * ncl) % nch;
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, chunk);
      if (mc) {
        const int part = chunk / CS;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                     :: "r"(smem_u32(smem) + rank * part), "l"(buf + c * chunk + rank * part), "r"(part),
                        "r"(smem_u32(&bar)), "h"((uint16_t)((1u << CS) - 1)) : "memory");
      } else {
        bulk_g2s(smem, buf + c * chunk, chunk, &bar);
      }
    }
    mbar_wait(&bar, r & 1);
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[11];
}

// ------------------------------------------------------------ multicast ring bandwidth
// CS CTAs per cluster stream the same sequence of CHUNK-byte chunks through a
// NST-deep smem ring.  mc=1: each CTA issues 1/CS of every chunk with
// .multicast::cluster to all CTAs; mc=0: every CTA issues the whole chunk
// itself (same data, unicast).  A cluster barrier every 8 chunks keeps the
// CTAs within one ring of each other.  distinct=1: clusters read disjoint data.
template <int CS, int NST, int CHUNK>
__global__ void mc_ring(const uint8_t* __restrict__ buf, size_t bytes, int nchunks, int mc, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[NST];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&bars[i], 1); fence_mbar_init(); }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const size_t nch_buf = bytes / CHUNK;
  const size_t cl = blockIdx.x / CS;
  const size_t base = (cl * 977) % nch_buf;
  for (int c0 = 0; c0 < nchunks; c0 += 8) {
    if (threadIdx.x == 0) {
      for (int c = c0; c < c0 + 8 && c < nchunks; ++c) {
        const int s = c % NST;
        if (c >= NST) mbar_wait(&bars[s], ((c / NST) - 1) & 1);
        mbar_expect_tx(&bars[s], CHUNK);
        const uint8_t* src = buf + ((base + c) % nch_buf) * CHUNK;
        if (mc) {
          const int part = CHUNK / CS;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                       :: "r"(smem_u32(smem + s * CHUNK) + rank * part), "l"(src + rank * part), "r"(part),
                          "r"(smem_u32(&bars[s])), "h"((uint16_t)((1u << CS) - 1)) : "memory");
        } else {
          bulk_g2s(smem + s * CHUNK, src, CHUNK, &bars[s]);
        }
      }
      // drain this group
      for (int c = c0; c < c0 + 8 && c < nchunks; ++c) {
        const int s = c % NST;
        if (c + NST >= c0 + 8 || c + NST >= nchunks) mbar_wait(&bars[s], (c / NST) & 1);
      }
    }
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[13];
}

template <int CS>
void run_mc(int nsm, uint8_t* buf, size_t bytes, int* sink) {
  constexpr int NST = 8, CHUNK = 16384;
  auto kern = mc_ring<CS, NST, CHUNK>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * CHUNK));
  int grid = (nsm / CS) * CS;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = NST * CHUNK;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mc = 0; mc < 2; ++mc) {
    int nchunks = 16;
    CK(cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, bytes, nchunks, mc, sink));
    CK(cudaDeviceSynchronize());
    nchunks = 2048;
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, bytes, nchunks, mc, sink));
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double delivered = (double)CHUNK * nchunks * grid;
    double l2_unique = delivered / CS;
    printf("cluster%d %s: delivered to SMEM %.2f TB/s (%.1f GB/s/SM), unique-data rate %.2f TB/s\n", CS,
           mc ? "MULTICAST" : "unicast  ", delivered / (ms * 1e-3) / 1e12, delivered / grid / (ms * 1e-3) / 1e9,
           l2_unique / (ms * 1e-3) / 1e12);
  }
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  printf("device %s  SMs %d  L2 %d MB  smem/block optin %zu KB  clock %d MHz\n", p.name, nsm,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin >> 10, p.clockRate / 1000);

  bool ok = true;
  ok &= run_check<128, 64, 64>(0);
  ok &= run_check<128, 16, 64>(0);
  ok &= run_check<128, 8, 32>(0);
  ok &= run_check<128, 256, 32>(0);
  ok &= run_check<128, 64, 64>(1);
  ok &= run_check<128, 16, 32>(1);
  ok &= run_check<128, 8, 32>(1);
  ok &= run_check<128, 24, 32>(0);
  printf("LAYOUT CHECKS: %s\n", ok ? "PASS" : "FAIL");

  if (argc > 1) {
  run_rate<128, 256, 64, 0>(nsm);
  run_rate<128, 128, 64, 0>(nsm);
  run_rate<128, 64, 64, 0>(nsm);
  run_rate<128, 32, 64, 0>(nsm);
  run_rate<128, 16, 64, 0>(nsm);
  run_rate<128, 8, 64, 0>(nsm);
  run_rate<64, 64, 64, 0>(nsm);
  run_rate<64, 32, 64, 0>(nsm);
  run_rate<128, 64, 64, 1>(nsm);
  run_rate<128, 32, 64, 1>(nsm);
  run_rate<128, 16, 64, 1>(nsm);
  }

  if (argc > 1) {
  // L2 broadcast read bandwidth
  for (size_t kb : {64, 600, 4096, 32768}) {
    size_t bytes = kb * 1024;
    uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
    uint4* sink; CK(cudaMalloc(&sink, nsm * 4 * 16));
    int reps = (int)std::max<size_t>(1, (size_t)(256ull << 20) / (bytes * nsm) + 1);
    l2_read<<<nsm * 2, 512>>>((const uint4*)buf, bytes / 16, 1, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    l2_read<<<nsm * 2, 512>>>((const uint4*)buf, bytes / 16, reps, sink);
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tot = (double)bytes * reps * nsm * 2;
    printf("l2_read  shared buffer %6zu KB: %.2f TB/s aggregate\n", kb, tot / (ms * 1e-3) / 1e12);
    // bulk path
    int chunk = 16384;
    CK(cudaFuncSetAttribute(l2_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * chunk));
    l2_bulk<<<nsm, 32, 4 * chunk>>>(buf, bytes, 1, chunk, (int*)sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    l2_bulk<<<nsm, 32, 4 * chunk>>>(buf, bytes, reps * 2, chunk, (int*)sink);
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
    tot = (double)bytes * reps * 2 * nsm;
    printf("l2_bulk  shared buffer %6zu KB: %.2f TB/s aggregate\n", kb, tot / (ms * 1e-3) / 1e12);
    cudaFree(buf); cudaFree(sink);
  }
  }
  // DSMEM push bandwidth
  {
    int* sink; CK(cudaMalloc(&sink, 4096));
    CK(cudaFuncSetAttribute(dsmem_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    dsmem_push<<<nsm, 256, 64 * 1024>>>(2, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = 200;
    cudaEventRecord(e0);
    dsmem_push<<<nsm, 256, 64 * 1024>>>(reps, sink);
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tot = 64.0 * 1024 * reps * nsm;
    printf("dsmem_push: %.2f TB/s aggregate, %.1f GB/s per SM\n", tot / (ms * 1e-3) / 1e12,
           tot / nsm / (ms * 1e-3) / 1e9);
    cudaFree(sink);
  }

  {
    int* sink; CK(cudaMalloc(&sink, 4096));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    size_t bytes = 256ull << 20;
    uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
    for (int mc = 0; mc < 2; ++mc) {
      CK(cudaFuncSetAttribute(mcast_load<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      int grid = (nsm / 4) * 4;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = 64 * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, mcast_load<4>, (const uint8_t*)buf, bytes, 4, mc, sink));
      CK(cudaDeviceSynchronize());
      int reps2 = 400;
      cudaEventRecord(e0);
      CK(cudaLaunchKernelEx(&cfg, mcast_load<4>, (const uint8_t*)buf, bytes, reps2, mc, sink));
      cudaEventRecord(e1); CK(cudaDeviceSynchronize());
      cudaEventElapsedTime(&ms, e0, e1);
      double delivered = 64.0 * 1024 * reps2 * grid;
      printf("cluster4 %s load of shared 64KB chunks: delivered %.2f TB/s to SMEM (%.1f GB/s per SM)\n",
             mc ? "MULTICAST" : "unicast  ", delivered / (ms * 1e-3) / 1e12, delivered / grid / (ms * 1e-3) / 1e9);
    }
    run_mc<1>(nsm, buf, bytes, sink);
    run_mc<2>(nsm, buf, bytes, sink);
    run_mc<4>(nsm, buf, bytes, sink);
    run_mc<8>(nsm, buf, bytes, sink);
    cudaFree(buf);
    cudaFree(sink);
  }
  return ok ? 0 : 1;
}
