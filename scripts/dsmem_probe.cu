// Probe (not part of the product): can a thread-block cluster serve the
// walker's random 4-byte leaf-index gathers from distributed shared memory
// faster than L2 does?  Each CTA of a C-CTA cluster holds a 128 KiB slice of
// a C x 128 KiB table; every lane reads a u32 index, gathers one random word
// of the table from the owning CTA's shared memory (ld.shared::cluster), and
// writes the walker's 12 B.  Compared against the same gathers from global
// memory (L2-resident table of the same size) and from a table 16x larger.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem_probe scripts/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr uint32_t kSliceWords = 32768;  // 128 KiB per CTA

__device__ __forceinline__ uint32_t ld_idx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t ld_dsmem(uint32_t local_addr, uint32_t rank) {
  uint32_t remote, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote));
  return v;
}

template <int C, int L>
__global__ void __launch_bounds__(512, 1) dsm(const uint32_t* __restrict__ idx, uint64_t n,
                                              uint64_t* __restrict__ o64, uint32_t* __restrict__ o32) {
  extern __shared__ __align__(16) uint32_t slice[];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t me = cluster.block_rank();
  for (uint32_t i = threadIdx.x; i < kSliceWords; i += blockDim.x) slice[i] = (me * kSliceWords + i) * 2654435761u;
  cluster.sync();
  const uint32_t base_addr = (uint32_t)__cvta_generic_to_shared(slice);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * L;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x) * L + threadIdx.x; b < n; b += stride) {
    uint32_t v[L], r[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = b + j * blockDim.x < n ? ld_idx(idx + b + j * blockDim.x) : 0;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const uint32_t a = v[j] & (C * kSliceWords - 1);
      r[j] = ld_dsmem(base_addr + (a % kSliceWords) * 4, a / kSliceWords);
    }
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const uint64_t i = b + j * blockDim.x;
      if (i < n) {
        o64[i] = ((uint64_t)r[j] << 12) | (v[j] & 0xFFF);
        o32[i] = r[j] & 3;
      }
    }
  }
  cluster.sync();
}

template <int L>
__global__ void __launch_bounds__(512, 2) gl(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                             uint32_t mask, uint64_t n, uint64_t* __restrict__ o64,
                                             uint32_t* __restrict__ o32) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * L;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x) * L + threadIdx.x; b < n; b += stride) {
    uint32_t v[L], r[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = ld_idx(idx + b + j * blockDim.x);
#pragma unroll
    for (int j = 0; j < L; ++j) r[j] = __ldg(tab + (v[j] & mask));
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const uint64_t i = b + j * blockDim.x;
      o64[i] = ((uint64_t)r[j] << 12) | (v[j] & 0xFFF);
      o32[i] = r[j] & 3;
    }
  }
}

template <int C, int L>
static void run_dsm(const uint32_t* idx, uint64_t n, uint64_t* o64, uint32_t* o32) {
  auto k = dsm<C, L>;
  const int smem = kSliceWords * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int nclusters = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k, &cfg);
  if (e != cudaSuccess || nclusters == 0) {
    printf("dsmem C=%d: no clusters (%s)\n", C, cudaGetErrorString(e));
    cudaGetLastError();
    return;
  }
  cfg.gridDim = dim3(C * nclusters);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, k, idx, n, o64, o32);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k, idx, n, o64, o32);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("dsmem C=%2d L=%d (%d clusters, %d CTAs, table %u KiB): %.3f ms  %.1f G lanes/s  [%s]\n", C, L, nclusters,
         C * nclusters, C * kSliceWords * 4 / 1024, ms, n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int L>
static void run_gl(const uint32_t* idx, const uint32_t* tab, uint32_t words, uint64_t n, uint64_t* o64,
                   uint32_t* o32, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gl<L><<<sms * 2, 512>>>(idx, tab, words - 1, n, o64, o32);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) gl<L><<<sms * 2, 512>>>(idx, tab, words - 1, n, o64, o32);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("global  L=%d table %8u KiB: %.3f ms  %.1f G lanes/s\n", L, words * 4 / 1024, ms, n / ms / 1e6);
}

int main() {
  const uint64_t n = 128ull << 20;
  const uint32_t big = 16u << 20;  // 64 MiB
  uint32_t *idx, *tab, *o32;
  uint64_t* o64;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&tab, (uint64_t)big * 4);
  cudaMalloc(&o32, n * 4);
  cudaMalloc(&o64, n * 8);
  uint32_t* h = (uint32_t*)malloc(n * 4);
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (uint32_t)s;
  }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(tab, 1, (uint64_t)big * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint32_t words : {8u * kSliceWords, 16u * kSliceWords, 1u << 20, big}) {
    run_gl<8>(idx, tab, words, n, o64, o32, sms);
    run_gl<4>(idx, tab, words, n, o64, o32, sms);
  }
  run_dsm<1, 8>(idx, n, o64, o32);
  run_dsm<2, 8>(idx, n, o64, o32);
  run_dsm<4, 8>(idx, n, o64, o32);
  run_dsm<8, 8>(idx, n, o64, o32);
  run_dsm<8, 16>(idx, n, o64, o32);
  run_dsm<16, 8>(idx, n, o64, o32);
  run_dsm<16, 16>(idx, n, o64, o32);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
