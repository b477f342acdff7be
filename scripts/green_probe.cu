// Probe (not part of the product): can the C5 step's walk and copy run side
// by side on disjoint SM sets (green contexts, cuDevSmResourceSplitByCount)?
//  1. do runtime-API launches on green-context streams work on memory from
//     cudaMalloc, and stay on their partition's SMs (%smid)?
//  2. HBM copy bandwidth (16-byte loads/stores, 2 x 4 GiB) vs SM count, and
//     the walker's access pattern (u32 in, random 4-byte gather from 2 MiB,
//     u32 out; scripts/store_probe.cu mode 3) vs SM count;
//  3. both at once on a walk / copy split.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/green_probe.bin scripts/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    CUresult r_ = (x);                                                               \
    if (r_ != CUDA_SUCCESS) {                                                        \
      const char* s_ = nullptr;                                                      \
      cuGetErrorString(r_, &s_);                                                     \
      printf("%s failed: %s\n", #x, s_ ? s_ : "?");                                  \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__global__ void smid_kernel(uint32_t* out) {
  if (threadIdx.x == 0) {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    out[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(512) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void __launch_bounds__(512, 2) gather_kernel(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ tab,
                                                        uint32_t mask, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(idx + i));
    out[i] = __ldg(tab + (v & mask));
  }
}

struct Part {
  CUgreenCtx g;
  cudaStream_t s;
  unsigned sms;
};

static float time_ms(cudaStream_t s, void (*fn)(cudaStream_t, void*), void* arg, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fn(s, arg);
  cudaEventRecord(a, s);
  for (int r = 0; r < reps; ++r) fn(s, arg);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

struct Bufs {
  uint4 *src, *dst;
  uint64_t n16;
  uint32_t *idx, *tab, *out;
  uint64_t lanes;
  unsigned grid_copy, grid_gather;
};

static void run_copy(cudaStream_t s, void* p) {
  Bufs* b = (Bufs*)p;
  copy_kernel<<<b->grid_copy, 512, 0, s>>>(b->src, b->dst, b->n16);
}
static void run_gather(cudaStream_t s, void* p) {
  Bufs* b = (Bufs*)p;
  gather_kernel<<<b->grid_gather, 512, 0, s>>>(b->idx, b->tab, (1u << 19) - 1, b->lanes, b->out);
}

int main() {
  CK(cuInit(0));
  cudaFree(0);
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  Bufs b;
  b.n16 = (4ull << 30) / 16;
  b.lanes = 128ull << 20;
  cudaMalloc(&b.src, b.n16 * 16);
  cudaMalloc(&b.dst, b.n16 * 16);
  cudaMalloc(&b.idx, b.lanes * 4);
  cudaMalloc(&b.tab, (1u << 19) * 4);
  cudaMalloc(&b.out, b.lanes * 4);
  cudaMemset(b.src, 1, b.n16 * 16);
  cudaMemset(b.tab, 1, (1u << 19) * 4);
  {
    std::vector<uint32_t> h(b.lanes);
    uint64_t s = 88172645463325252ull;
    for (auto& x : h) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      x = (uint32_t)s;
    }
    cudaMemcpy(b.idx, h.data(), b.lanes * 4, cudaMemcpyHostToDevice);
  }
  uint32_t* smids;
  cudaMallocManaged(&smids, 4096 * 4);
  for (unsigned want : {16u, 32u, 48u, 64u, 74u}) {
    CUdevResource grp[1], rem;
    unsigned nb = 1;
    CK(cuDevSmResourceSplitByCount(grp, &nb, &all, &rem, 0, want));
    Part P[2];
    CUdevResource* rs[2] = {&grp[0], &rem};
    for (int i = 0; i < 2; ++i) {
      CUdevResourceDesc d;
      CK(cuDevResourceGenerateDesc(&d, rs[i], 1));
      CK(cuGreenCtxCreate(&P[i].g, d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
      CUstream cs;
      CK(cuGreenCtxStreamCreate(&cs, P[i].g, CU_STREAM_NON_BLOCKING, 0));
      P[i].s = (cudaStream_t)cs;
      P[i].sms = rs[i]->sm.smCount;
    }
    std::set<uint32_t> ids[2];
    for (int i = 0; i < 2; ++i) {
      smid_kernel<<<2048, 32, 0, P[i].s>>>(smids);
      cudaError_t e = cudaStreamSynchronize(P[i].s);
      if (e != cudaSuccess) {
        printf("launch on green stream %d: %s\n", i, cudaGetErrorString(e));
        return 1;
      }
      for (int k = 0; k < 2048; ++k) ids[i].insert(smids[k]);
    }
    int overlap = 0;
    for (auto x : ids[0]) overlap += ids[1].count(x);
    printf("split %u: walk part %u SMs (used %zu), copy part %u SMs (used %zu), overlap %d\n", want, P[0].sms,
           ids[0].size(), P[1].sms, ids[1].size(), overlap);
    // alone
    b.grid_gather = P[0].sms * 2;
    b.grid_copy = P[1].sms * 4;
    const float tg = time_ms(P[0].s, run_gather, &b), tc = time_ms(P[1].s, run_copy, &b);
    // together: K of each, one stream each
    cudaEvent_t a, z, ga, gz;
    cudaEventCreate(&a); cudaEventCreate(&z); cudaEventCreate(&ga); cudaEventCreate(&gz);
    cudaDeviceSynchronize();
    cudaEventRecord(a, P[1].s);
    cudaStreamWaitEvent(P[0].s, a, 0);
    cudaEventRecord(ga, P[0].s);
    for (int r = 0; r < 5; ++r) run_gather(P[0].s, &b);
    cudaEventRecord(gz, P[0].s);
    for (int r = 0; r < 5; ++r) run_copy(P[1].s, &b);
    cudaStreamWaitEvent(P[1].s, gz, 0);
    cudaEventRecord(z, P[1].s);
    cudaEventSynchronize(z);
    float both = 0, gonly = 0;
    cudaEventElapsedTime(&both, a, z);
    cudaEventElapsedTime(&gonly, ga, gz);
    printf("   gather alone %.3f ms (%.1f G lanes/s) | copy alone %.3f ms (%.0f GB/s) | both %.3f ms/iter "
           "(gather %.3f) [%s]\n",
           tg, b.lanes / tg / 1e6, tc, 2.0 * b.n16 * 16 / tc / 1e6, both / 5, gonly / 5,
           cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 2; ++i) {
      cuStreamDestroy((CUstream)P[i].s);
      cuGreenCtxDestroy(P[i].g);
    }
  }
  // the full device for reference
  b.grid_gather = 296;
  b.grid_copy = 148 * 4;
  const float tg = time_ms(0, run_gather, &b), tc = time_ms(0, run_copy, &b);
  printf("full device: gather %.3f ms (%.1f G lanes/s) | copy %.3f ms (%.0f GB/s)\n", tg, b.lanes / tg / 1e6, tc,
         2.0 * b.n16 * 16 / tc / 1e6);
  return 0;
}
