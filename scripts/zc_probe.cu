// Probe (not part of the product): SM-driven zero-copy reads of pinned host
// memory over the host link vs the copy engine (cudaMemcpyAsync H2D), for
// copy_to_user from a pinned host payload: (1) DMA H2D, (2) LSU 16-byte
// loads from mapped pinned memory stored to HBM, (3) TMA bulk copies
// (cp.async.bulk global->shared with a host-mapped source, then shared->global).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/zc_probe.bin scripts/zc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) lsu_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n) {
  constexpr int U = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) dst[i + u * stride] = v[u];
  }
}

constexpr int kStages = 4;
constexpr int kChunk = 16384;
__global__ void __launch_bounds__(32, 1) tma_copy(const uint8_t* src, uint8_t* dst, uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bar[kStages];
  const uint64_t nchunks = bytes / kChunk;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t parity = 0;
  auto load = [&](uint64_t c, int s) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(ring + (size_t)s * kChunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
                 "l"(src + c * kChunk), "r"(kChunk), "r"(b)
                 : "memory");
  };
  uint64_t first = blockIdx.x, step = gridDim.x;
  int k = 0;
  for (uint64_t c = first; c < nchunks && k < kStages - 1; c += step, ++k) load(c, k % kStages);
  k = 0;
  for (uint64_t c = first; c < nchunks; c += step, ++k) {
    const int s = k % kStages;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    const uint32_t ph = (parity >> s) & 1u;
    asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(b),
                 "r"(ph)
                 : "memory");
    parity ^= 1u << s;
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(ring + (size_t)s * kChunk);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * kChunk), "r"(sm),
                 "r"(kChunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    const uint64_t cn = c + (uint64_t)(kStages - 1) * step;
    if (cn < nchunks) load(cn, (k + kStages - 1) % kStages);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t bytes = 256ull << 20;
  uint8_t *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  for (uint64_t i = 0; i < bytes; i += 4096) h[i] = (uint8_t)i;
  cudaMalloc(&d, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %.3f ms  %.1f GB/s  [%s]\n", name, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("DMA cudaMemcpyAsync H2D", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); });
  for (int per : {1, 2, 4}) {
    char nm[64];
    snprintf(nm, sizeof nm, "LSU zero-copy, %d x 512 thr/SM", per);
    timeit(nm, [&] { lsu_copy<<<sms * per, 512>>>((const uint4*)h, (uint4*)d, bytes / 16); });
  }
  for (int per : {1, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "TMA zero-copy, %d CTAs/SM x 4 x 16K", per);
    timeit(nm, [&] { tma_copy<<<sms * per, 32, kStages * kChunk>>>(h, d, bytes); });
  }
  return 0;
}
