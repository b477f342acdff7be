// Probe (not part of the product): the per-call round trip of a persistent
// device server vs one kernel launch per call.  The host writes a request
// (sequence number + argument) into mapped pinned memory and spins on the
// reply; the device side either is a resident 1-warp kernel polling the
// request word (ld.acquire.sys) or a fresh launch per call that writes the
// reply.  The reply carries one dependent HBM read (a walk-sized access).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/poll_probe.bin scripts/poll_probe.cu
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct Req { volatile uint64_t seq; volatile uint64_t arg; uint64_t pad[6]; };
struct Rep { volatile uint64_t seq; volatile uint64_t val; uint64_t pad[6]; };

__device__ __forceinline__ uint64_t ld_acquire_sys(const volatile uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(volatile uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void server(Req* req, Rep* rep, const uint64_t* table, uint64_t n_calls) {
  if (threadIdx.x != 0) return;
  uint64_t want = 1;
  while (want <= n_calls) {
    const uint64_t s = ld_acquire_sys(&req->seq);
    if (s != want) continue;
    const uint64_t a = req->arg;
    const uint64_t v = table[a & ((1u << 20) - 1)];  // one dependent HBM read
    rep->val = v;
    st_release_sys(&rep->seq, s);
    ++want;
  }
}

__global__ void one(uint64_t seq, uint64_t arg, Rep* rep, const uint64_t* table) {
  const uint64_t v = table[arg & ((1u << 20) - 1)];
  rep->val = v;
  st_release_sys(&rep->seq, seq);
}

int main() {
  Req* req;
  Rep* rep;
  cudaHostAlloc(&req, sizeof(Req), cudaHostAllocMapped);
  cudaHostAlloc(&rep, sizeof(Rep), cudaHostAllocMapped);
  req->seq = 0;
  rep->seq = 0;
  uint64_t* table;
  cudaMalloc(&table, (1u << 20) * 8);
  cudaMemset(table, 7, (1u << 20) * 8);
  cudaStream_t st, st2;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
  const int N = 20000;
  // launch per call
  for (int r = 0; r < 2; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 1; i <= N; ++i) {
      one<<<1, 32, 0, st>>>(i + r * N, i * 2654435761u, rep, table);
      while (rep->seq != (uint64_t)(i + r * N)) {}
    }
    auto t1 = std::chrono::steady_clock::now();
    printf("launch per call      %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  }
  cudaStreamSynchronize(st);
  rep->seq = 0;
  // persistent server
  server<<<1, 32, 0, st2>>>(req, rep, table, N);
  for (int i = 1; i <= 200; ++i) {  // warm
    req->arg = i;
    __atomic_store_n(&req->seq, (uint64_t)i, __ATOMIC_RELEASE);
    while (rep->seq != (uint64_t)i) {}
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 201; i <= N; ++i) {
    req->arg = i * 2654435761u;
    __atomic_store_n(&req->seq, (uint64_t)i, __ATOMIC_RELEASE);
    while (rep->seq != (uint64_t)i) {}
  }
  auto t1 = std::chrono::steady_clock::now();
  printf("persistent server    %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / (N - 200));
  cudaStreamSynchronize(st2);
  printf("[%s]\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
