// Probe (not part of the product): copy 8 GiB of 4 KiB page chunks from a
// contiguous source into randomly permuted destination pages (the C5
// copy_to_user pattern), (a) with warp-wide 16-byte LSU copies, 8 vectors in
// flight per lane (the exec kernel's scheme), (b) with TMA bulk copies
// (cp.async.bulk global->shared with an mbarrier, then shared->global bulk
// stores) driven by one lane per warp over an R-stage ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_copy_probe.bin scripts/tma_copy_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__global__ void __launch_bounds__(256, 2) lsu_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                   const uint32_t* __restrict__ perm, uint64_t n_pages) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = pol_first();
  for (uint64_t p = warp; p < n_pages; p += nwarps) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (p << 12));
    uint4* d = reinterpret_cast<uint4*>(dst + ((uint64_t)perm[p] << 12));
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                   : "l"(s + j * 32 + lane), "l"(pol));
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(d + j * 32 + lane),
                   "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w), "l"(pol)
                   : "memory");
  }
}

template <int R, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tma_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                          const uint32_t* __restrict__ perm, uint64_t n_pages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[WARPS][R];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* ring = smem + (size_t)wid * R * 4096;
  if (lane == 0) {
    for (int s = 0; s < R; ++s) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[wid][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane != 0) return;
  const uint64_t warp = (uint64_t)blockIdx.x * WARPS + wid;
  const uint64_t nwarps = (uint64_t)gridDim.x * WARPS;
  auto issue = [&](uint64_t p, int s) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[wid][s]);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + s * 4096);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(d),
                 "l"(src + (p << 12)), "r"(b)
                 : "memory");
  };
  uint32_t phase[R];
  for (int s = 0; s < R; ++s) phase[s] = 0;
  // prologue: R - 1 loads in flight
  uint64_t next = warp;
  for (int s = 0; s < R - 1 && next < n_pages; ++s, next += nwarps) issue(next, s);
  int s = 0;
  for (uint64_t p = warp; p < n_pages; p += nwarps) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[wid][s]);
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(b),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(ring + s * 4096);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(dst + ((uint64_t)perm[p] << 12)),
                 "r"(a)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the stage the next load goes to was stored from one iteration ago
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    const int sn = (s + R - 1) % R;
    if (next < n_pages) {
      issue(next, sn);
      next += nwarps;
    }
    s = (s + 1) % R;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int R, int WARPS>
static void run_tma(uint8_t* dst, const uint8_t* src, const uint32_t* perm, uint64_t n_pages, int sms, int per_sm) {
  auto k = tma_copy<R, WARPS>;
  const int smem = R * WARPS * 4096;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) k<<<sms * per_sm, WARPS * 32, smem>>>(dst, src, perm, n_pages);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k<<<sms * per_sm, WARPS * 32, smem>>>(dst, src, perm, n_pages);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("tma R=%d warps=%2d x%d/SM (smem %3d KiB): %.3f ms  %.0f GB/s  [%s]\n", R, WARPS, per_sm, smem / 1024, ms,
         2.0 * n_pages * 4096 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t n_pages = 2ull << 20;  // 8 GiB
  uint8_t *src, *dst;
  uint32_t* perm;
  cudaMalloc(&src, n_pages << 12);
  cudaMalloc(&dst, n_pages << 12);
  cudaMalloc(&perm, n_pages * 4);
  uint32_t* h = (uint32_t*)malloc(n_pages * 4);
  for (uint64_t i = 0; i < n_pages; ++i) h[i] = (uint32_t)i;
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = n_pages - 1; i > 0; --i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const uint64_t j = s % (i + 1);
    const uint32_t t = h[i]; h[i] = h[j]; h[j] = t;
  }
  cudaMemcpy(perm, h, n_pages * 4, cudaMemcpyHostToDevice);
  cudaMemset(src, 7, n_pages << 12);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) lsu_copy<<<sms * 2, 256>>>(dst, src, perm, n_pages);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) lsu_copy<<<sms * 2, 256>>>(dst, src, perm, n_pages);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("lsu 16B x8/lane, 2x256/SM:           %.3f ms  %.0f GB/s\n", ms, 2.0 * n_pages * 4096 / ms / 1e6);
    cudaMemcpy(dst, src, n_pages << 12, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) cudaMemcpyAsync(dst, src, n_pages << 12, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("cudaMemcpy D2D (contiguous):          %.3f ms  %.0f GB/s\n", ms, 2.0 * n_pages * 4096 / ms / 1e6);
  }
  run_tma<4, 8>(dst, src, perm, n_pages, sms, 1);
  run_tma<6, 8>(dst, src, perm, n_pages, sms, 1);
  run_tma<8, 4>(dst, src, perm, n_pages, sms, 1);
  run_tma<4, 4>(dst, src, perm, n_pages, sms, 2);
  run_tma<6, 4>(dst, src, perm, n_pages, sms, 2);
  run_tma<12, 4>(dst, src, perm, n_pages, sms, 1);
  run_tma<3, 16>(dst, src, perm, n_pages, sms, 1);
  // check
  uint8_t* hb = (uint8_t*)malloc(4096);
  cudaMemcpy(hb, dst + ((uint64_t)h[12345] << 12), 4096, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 4096; ++i) bad += hb[i] != 7;
  printf("check: %d bad bytes, err %s\n", bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
