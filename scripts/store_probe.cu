// Probe (not part of the product): does routing the walker's 12 B/lane of
// results through shared memory + TMA bulk stores (cp.async.bulk.global.
// shared::cta) relieve the L1->XBAR request port that bounds the walk
// (ncu: l1tex__m_l1tex2xbar_req_cycles_active ~86 %)?  Each warp owns 128
// consecutive lanes per step: u32 index in, one random 4-byte gather from a
// 2 MiB table, u64 + u32 out.  Mode 0 stores from registers (the walker
// today); mode 1 stages the warp's 1 KiB + 512 B of results in shared memory
// and one lane bulk-stores them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/store_probe.bin scripts/store_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_idx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 2) k(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                            uint32_t mask, uint64_t n, uint64_t* __restrict__ o64,
                                            uint32_t* __restrict__ o32) {
  constexpr int L = 4;
  __shared__ __align__(128) uint64_t s64[2][16][128];
  __shared__ __align__(128) uint32_t s32[2][16][128];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nwarps = (uint64_t)gridDim.x * 16;
  int buf = 0;
  for (uint64_t wb = ((uint64_t)blockIdx.x * 16 + warp) * 128; wb < n; wb += nwarps * 128) {
    uint32_t v[L], r[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = ld_idx(idx + wb + j * 32 + lane);
#pragma unroll
    for (int j = 0; j < L; ++j) r[j] = __ldg(tab + (v[j] & mask));
    if (MODE == 3) {  // pv_translate_words: one 4-byte frame word out per lane
#pragma unroll
      for (int j = 0; j < L; ++j) o32[wb + j * 32 + lane] = r[j];
    } else if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int j = 0; j < L; ++j) {
        const uint64_t i = wb + j * 32 + lane;
        o64[i] = ((uint64_t)r[j] << 12) | (v[j] & 0xFFF);
        if (MODE == 0) o32[i] = r[j] & 3;  // MODE 2: the PV_OUT_PACKED form, 8 B out per lane
      }
    } else {
      // the buffer written two steps ago must have been read out by its bulk store
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int j = 0; j < L; ++j) {
        s64[buf][warp][j * 32 + lane] = ((uint64_t)r[j] << 12) | (v[j] & 0xFFF);
        s32[buf][warp][j * 32 + lane] = r[j] & 3;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const uint32_t a64 = (uint32_t)__cvta_generic_to_shared(&s64[buf][warp][0]);
        const uint32_t a32 = (uint32_t)__cvta_generic_to_shared(&s32[buf][warp][0]);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(o64 + wb), "r"(a64)
                     : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(o32 + wb), "r"(a32)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      buf ^= 1;
    }
  }
  if (MODE == 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Mode 2: each thread owns 4 consecutive lanes: one 16-byte VA load, 4
// gathers, two 16-byte stores of u64 results and one 16-byte store of u32
// statuses (3 store instructions per 4 lanes instead of 8, same bytes).
__global__ void __launch_bounds__(512, 2) kvec(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                               uint32_t mask, uint64_t n, uint64_t* __restrict__ o64,
                                               uint32_t* __restrict__ o32) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; b < n; b += stride) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(idx + b));
    const uint32_t r0 = __ldg(tab + (v.x & mask)), r1 = __ldg(tab + (v.y & mask)), r2 = __ldg(tab + (v.z & mask)),
                   r3 = __ldg(tab + (v.w & mask));
    ulonglong2 a, c;
    a.x = ((uint64_t)r0 << 12) | (v.x & 0xFFF);
    a.y = ((uint64_t)r1 << 12) | (v.y & 0xFFF);
    c.x = ((uint64_t)r2 << 12) | (v.z & 0xFFF);
    c.y = ((uint64_t)r3 << 12) | (v.w & 0xFFF);
    reinterpret_cast<ulonglong2*>(o64 + b)[0] = a;
    reinterpret_cast<ulonglong2*>(o64 + b)[1] = c;
    uint4 st;
    st.x = r0 & 3; st.y = r1 & 3; st.z = r2 & 3; st.w = r3 & 3;
    *reinterpret_cast<uint4*>(o32 + b) = st;
  }
}

int main(int argc, char** argv) {
  const uint64_t n = 128ull << 20;
  const uint32_t words = argc > 1 ? (1u << atoi(argv[1])) : (1u << 19);  // 2 MiB by default (argv[1]: log2 words)
  printf("table %u KiB\n", words / 256);
  uint32_t *idx, *tab, *o32;
  uint64_t* o64;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&tab, (uint64_t)words * 4);
  cudaMalloc(&o32, n * 4);
  cudaMalloc(&o64, n * 8);
  uint32_t* h = (uint32_t*)malloc(n * 4);
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (uint32_t)s;
  }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(tab, 1, (uint64_t)words * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void (*fns[5])(const uint32_t*, const uint32_t*, uint32_t, uint64_t, uint64_t*, uint32_t*) = {k<0>, k<1>, kvec,
                                                                                              k<2>, k<3>};
  const char* names[5] = {"register stores", "smem + bulk stores", "4 lanes/thread, v4 io",
                          "register stores, 8 B out (packed)", "register stores, 4 B out (words)"};
  uint64_t* check = (uint64_t*)malloc(1 << 20);
  for (int m = 0; m < 5; ++m) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemset(o64, 0, n * 8);
    for (int w = 0; w < 3; ++w) fns[m]<<<sms * 2, 512>>>(idx, tab, words - 1, n, o64, o32);
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) fns[m]<<<sms * 2, 512>>>(idx, tab, words - 1, n, o64, o32);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    uint64_t bad = 0;
    if (m == 4) {
      cudaMemcpy(check, o32 + (n - 131072), 131072 * 4, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 131072; ++i) bad += ((const uint32_t*)check)[i] != 0x01010101u;
    } else {
      cudaMemcpy(check, o64 + (n - 131072), 1 << 20, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 131072; ++i) bad += check[i] != ((0x01010101ull << 12) | (h[n - 131072 + i] & 0xFFF));
    }
    printf("%-22s %.3f ms  %.1f G lanes/s  mismatches %llu  [%s]\n", names[m], ms, n / ms / 1e6,
           (unsigned long long)bad, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
