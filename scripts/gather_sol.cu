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

// MODE 0: 4 B out; 1: walker-shaped 12 B out; 2: stream only.
// SMEM: resolve the upper levels through an 8 KiB shared-memory code table
// first (the walker's staged codes), L lanes per thread.
template <int MODE, bool SMEM, int L>
__global__ void __launch_bounds__(512, 2) k(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                            uint32_t mask, uint64_t n, uint64_t* __restrict__ o64,
                                            uint32_t* __restrict__ o32) {
  __shared__ uint32_t codes[2048];
  if (SMEM) {
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) codes[i] = ((uint32_t)i * 2654435761u) | 1u;
    __syncthreads();
  }
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * L;
  for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x) * L + threadIdx.x; base < n; base += stride) {
    uint32_t v[L], r[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = ld32(idx + base + j * blockDim.x, pf);
#pragma unroll
    for (int j = 0; j < L; ++j) {
      uint32_t a = v[j] & mask;
      if (SMEM) a = (codes[(v[j] >> 9) & 2047] ^ v[j]) & mask;  // dependent, still uniform over the table
      r[j] = MODE == 2 ? v[j] : ld32(tab + a, pl);
    }
#pragma unroll
    for (int j = 0; j < L; ++j) {
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
  struct Case {
    const char* name;
    void (*fn)(const uint32_t*, const uint32_t*, uint32_t, uint64_t, uint64_t*, uint32_t*);
  };
  const Case cases[] = {
      {"gather, 4 B out, 8/thr", k<0, false, 8>},
      {"gather, walker 12 B out, 8/thr", k<1, false, 8>},
      {"stream only, 16 B/lane, 8/thr", k<2, false, 8>},
      {"gather+smem codes, walker, 8/thr", k<1, true, 8>},
      {"gather, walker, 4/thr", k<1, false, 4>},
      {"gather+smem codes, walker, 4/thr", k<1, true, 4>},
  };
  for (const Case& c : cases) {
    for (int grid_mul = 2; grid_mul <= 4; grid_mul += 2) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) c.fn<<<sms * grid_mul, 512>>>(idx, tab, (uint32_t)tab_words - 1, n, o64, o32);
      cudaEventRecord(a);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) c.fn<<<sms * grid_mul, 512>>>(idx, tab, (uint32_t)tab_words - 1, n, o64, o32);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      ms /= reps;
      printf("%-36s grid %3dx%d: %.3f ms  %.1f G lanes/s\n", c.name, sms * grid_mul, 512, ms, n / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
