// DSMEM (distributed shared memory) bandwidth between the CTAs of a cluster,
// measured three ways, for cluster sizes 2, 4, 6 and 8 (one CTA per SM, all
// SMs):
//   bulk   cp.async.bulk.shared::cluster.shared::cta (the TMA engine copies a
//          local smem range into a peer CTA's smem, completion on the peer's
//          mbarrier), NIF copies of CHUNK bytes in flight per round
//   st     st.shared::cluster.v4 from every thread (512 threads)
//   ld     ld.shared::cluster.v4 from every thread (512 threads)
// Not part of the product: the numbers decide the cluster design.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_1912_02165_b200/csrc dsmem.cu -o dsmem
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace wf;

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_n() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

// smem: [0, NIF*CHUNK) source, [NIF*CHUNK, 2*NIF*CHUNK) receive
template <int NIF, int CHUNK>
__global__ void bulk_push(int rounds, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  const uint32_t rank = cta_rank(), n = cluster_n();
  const uint32_t peer = (rank + 1) % n;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  cluster_sync();
  const uint32_t dst = mapa(smem_u32(smem + NIF * CHUNK), peer);
  const uint32_t pbar = mapa(smem_u32(&bar), peer);
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) mbar_expect_tx(&bar, NIF * CHUNK);
    cluster_sync();   // every CTA armed its barrier for this round
    if (threadIdx.x == 0) {
      for (int i = 0; i < NIF; ++i)
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dst + i * CHUNK),
            "r"(smem_u32(smem + i * CHUNK)), "r"(CHUNK), "r"(pbar)
            : "memory");
      mbar_wait(&bar, r & 1);
    }
    __syncthreads();
  }
  cluster_sync();
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[NIF * CHUNK + 5];
}

__global__ void st_push(int reps, int bytes, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t rank = cta_rank(), n = cluster_n();
  cluster_sync();
  const uint32_t remote = mapa(smem_u32(smem), (rank + 1) % n);
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
      asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(remote + i), "r"(r), "r"(i), "r"(r), "r"(i)
                   : "memory");
  cluster_sync();
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[7];
}

__global__ void ld_pull(int reps, int bytes, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t rank = cta_rank(), n = cluster_n();
  for (int i = threadIdx.x * 4; i < bytes; i += blockDim.x * 4) *reinterpret_cast<int*>(smem + i) = i;
  cluster_sync();
  const uint32_t remote = mapa(smem_u32(smem), (rank + 1) % n);
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16) {
      uint32_t a, b, c, d;
      asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(remote + i));
      acc += a ^ b ^ c ^ d;
    }
  cluster_sync();
  if (acc == 0x12345) sink[blockIdx.x] = acc;
}

template <class K, class... A>
static float timed(K kern, int cs, int grid, int threads, size_t smem, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, args...));   // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int NIF, int CHUNK>
static void run_bulk(int nsm, int cs, int* sink) {
  auto k = bulk_push<NIF, CHUNK>;
  const size_t smem = 2 * NIF * CHUNK;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int ncl = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
  }
  const int grid = std::min(nsm / cs, ncl) * cs;
  const int rounds = 400;
  const float ms = timed(k, cs, grid, 128, smem, rounds, sink);
  const double per_sm = double(NIF) * CHUNK * rounds / (ms * 1e-3) / 1e9;
  printf("bulk cs=%d NIF=%d chunk=%5d: %7.1f GB/s per SM sent (%d CTAs, max active clusters %d), %.2f us per round\n",
         cs, NIF, CHUNK, per_sm, grid, ncl, ms * 1e3 / rounds);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, nsm);
  int* sink;
  CK(cudaMalloc(&sink, 1 << 16));
  for (int cs : {2, 4, 6, 8}) {
    run_bulk<1, 16384>(nsm, cs, sink);
    run_bulk<4, 16384>(nsm, cs, sink);
    run_bulk<8, 8192>(nsm, cs, sink);
    run_bulk<6, 16384>(nsm, cs, sink);
  }
  const int bytes = 64 * 1024;
  CK(cudaFuncSetAttribute(st_push, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(ld_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(st_push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(ld_pull, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {2, 4, 6, 8}) {
    for (int th : {256, 512, 1024}) {
      const int grid = (nsm / cs) * cs, reps = 100;
      float ms = timed(st_push, cs, grid, th, bytes, reps, bytes, sink);
      printf("st.shared::cluster.v4 cs=%d threads=%4d: %7.1f GB/s per SM\n", cs, th,
             double(bytes) * reps / (ms * 1e-3) / 1e9);
      ms = timed(ld_pull, cs, grid, th, bytes, reps, bytes, sink);
      printf("ld.shared::cluster.v4 cs=%d threads=%4d: %7.1f GB/s per SM\n", cs, th,
             double(bytes) * reps / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
