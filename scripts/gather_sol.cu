// Speed-of-light probe for the walker's access pattern (not part of the
// product): n independent random 4-byte gathers from a table of `tab_bytes`
// (the C5 leaf-index footprint), with the walker's stream around them
// (u32 index in, u64 + u32 out per lane), 8 lanes in flight per thread.
// Prints G gathers/s for: gather only (4 B out), gather + walker-shaped
// output (12 B out), and pure streaming of the same 16 B/lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_sol scripts/gather_sol.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 2) k(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                            uint32_t mask, uint64_t n, uint64_t* __restrict__ o64,
                                            uint32_t* __restrict__ o32) {
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
  for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x) * 8 + threadIdx.x; base < n; base += stride) {
    uint32_t v[8], r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ld32(idx + base + j * blockDim.x, pf);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = MODE == 2 ? v[j] : ld32(tab + (v[j] & mask), pl);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t i = base + j * blockDim.x;
      if (MODE == 0) {
        o32[i] = r[j];
      } else {
        o64[i] = ((uint64_t)r[j] << 12) | (v[j] & 0xFFF);
        o32[i] = r[j] & 3;
      }
    }
  }
}

int main() {
  const uint64_t n = 128ull << 20;
  const uint64_t tab_words = 16ull << 20;  // 64 MiB
  uint32_t *idx, *tab, *o32;
  uint64_t* o64;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&tab, tab_words * 4);
  cudaMalloc(&o32, n * 4);
  cudaMalloc(&o64, n * 8);
  // random indices: a cheap LCG on the host would take long; fill on device
  uint32_t* h = (uint32_t*)malloc(n * 4);
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (uint32_t)s;
  }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(tab, 1, tab_words * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[3] = {"gather, 4 B out", "gather, walker-shaped 12 B out", "stream only, 16 B/lane"};
  for (int mode = 0; mode < 3; ++mode) {
    auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    for (int grid_mul = 2; grid_mul <= 4; grid_mul += 2) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) fn<<<sms * grid_mul, 512>>>(idx, tab, (uint32_t)tab_words - 1, n, o64, o32);
      cudaEventRecord(a);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) fn<<<sms * grid_mul, 512>>>(idx, tab, (uint32_t)tab_words - 1, n, o64, o32);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      ms /= reps;
      printf("%-34s grid %3dx%d: %.3f ms  %.1f G lanes/s\n", names[mode], sms * grid_mul, 512, ms, n / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
