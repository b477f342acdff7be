// pv_copy.cu — K2/K3: batched copy_to_user / copy_from_user.
//
// Restates copy_user_buffer (memvirt.py:604-628) for a batch of operations:
//   * the translation is performed once per page touched; the first chunk
//     keeps the unaligned start, chunk = min(remaining, 4096 - (cur & 0xFFF));
//   * a page whose translation fails stops its op: every page before it is
//     copied, nothing after it; `copied` is the completed prefix
//     (PageFault.bytes_copied, memvirt.py:618-622);
//   * the data access is bounds-checked against host memory and raises
//     OutOfRange (memvirt.py:156-168) -- also a stopping point.
//
// B200 design: two launches over one flat page list of the batch.
//   plan  : one thread per 4 pages walks each page (L1-cached upper levels,
//           one dependent load per level) and records the op's first failing
//           page with a u64 atomicMin;
//   exec  : one warp per page chunk moves up to 4 KiB with 16-byte vector
//           loads/stores (8 x 16 B in flight per lane, all loads issued
//           before the stores), realigning with funnel shifts when source and
//           destination disagree modulo 4, byte loops only for heads/tails.
// A separate stamp pass detects two pages of one to_guest batch landing on
// the same hpa page (order-dependent last-writer-wins), which the host then
// re-plans sequentially.
#include "pv_common.cuh"

namespace pv {

constexpr int kPlanTpb = 256;
constexpr int kPlanPpt = 4;  // pages per plan thread
constexpr int kExecTpb = 256;
constexpr int kExecWarps = kExecTpb / 32;
constexpr int kExecPpw = 4;  // pages per exec warp

__global__ void __launch_bounds__(kPlanTpb)
plan_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_space* __restrict__ spaces,
            const pv_op* __restrict__ ops, uint64_t n_ops, const uint64_t* __restrict__ page_off, uint64_t n_pages,
            uint64_t* __restrict__ page_hpa, uint32_t* __restrict__ page_status, uint64_t* __restrict__ page_aux,
            unsigned long long* __restrict__ op_first_bad) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * kPlanPpt < n_pages; t += nthreads) {
    const uint64_t p0 = t * kPlanPpt;
    uint64_t op = upper_search(page_off, 0, n_ops, p0);
    uint64_t op_end = __ldg(page_off + op + 1);
    pv_op o = ops[op];
    pv_space sp = spaces[o.space];
#pragma unroll 1
    for (uint64_t p = p0; p < p0 + kPlanPpt && p < n_pages; ++p) {
      while (p >= op_end) {
        ++op;
        op_end = __ldg(page_off + op + 1);
        o = ops[op];
        sp = spaces[o.space];
      }
      const uint64_t k = p - __ldg(page_off + op);
      const uint64_t cur = op_page_va(o.gva, k);
      const uint64_t done = cur - o.gva;
      const uint64_t chunk = min(o.len - done, kPageSize - (cur & kPageMask));
      uint64_t value = 0, aux = 0;
      uint32_t st = translate_global(image, image_bytes, sp, cur, &value, &aux);
      if (st == PV_ST_OK) {
        value = (value << kPageShift) | (cur & kPageMask);
        // host_mem.write / read bounds check (memvirt.py:156-158).
        if (value + chunk > image_bytes || value + chunk < value) st = PV_ST_DATA_OOR;
      }
      page_hpa[p] = value;
      page_status[p] = st;
      if (page_aux != nullptr) page_aux[p] = aux;
      if (st != PV_ST_OK) atomicMin(op_first_bad + op, (unsigned long long)k);
    }
  }
}

// Stamp destination hpa pages of a to_guest batch; flag conflicts.
__global__ void __launch_bounds__(kPlanTpb)
stamp_kernel(const uint64_t* __restrict__ page_off, uint64_t n_ops, uint64_t n_pages,
             const uint64_t* __restrict__ page_hpa, const unsigned long long* __restrict__ op_first_bad,
             unsigned long long* __restrict__ owner, uint64_t owner_pages, uint32_t epoch, uint32_t* conflict) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * kPlanPpt < n_pages; t += nthreads) {
    // one detected conflict decides the batch (the exec kernel stands down):
    // stop stamping, so heavily overlapping batches do not serialise on atomics
    if (*reinterpret_cast<volatile const uint32_t*>(conflict)) return;
    const uint64_t p0 = t * kPlanPpt;
    uint64_t op = upper_search(page_off, 0, n_ops, p0);
    uint64_t op_end = __ldg(page_off + op + 1);
    for (uint64_t p = p0; p < p0 + kPlanPpt && p < n_pages; ++p) {
      while (p >= op_end) {
        ++op;
        op_end = __ldg(page_off + op + 1);
      }
      const uint64_t k = p - __ldg(page_off + op);
      if (k >= op_first_bad[op]) continue;
      const uint64_t hp = page_hpa[p] >> kPageShift;
      if (hp >= owner_pages) continue;
      const unsigned long long mine = ((unsigned long long)epoch << 40) | (p + 1);
      const unsigned long long seen = *reinterpret_cast<volatile const unsigned long long*>(owner + hp);
      if ((seen >> 40) == epoch && seen != mine) {  // already stamped by another chunk of this batch
        atomicOr(conflict, 1u);
        return;
      }
      const unsigned long long old = atomicMax(owner + hp, mine);
      if ((old >> 40) == epoch && old != mine) atomicOr(conflict, 1u);
    }
  }
}

// ---- warp copy of one chunk (<= 4096 bytes) -------------------------------

__device__ __forceinline__ uint4 ld_v4_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_v4_stream(uint4* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void warp_copy_bytes(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, uint32_t n,
                                                uint32_t lane) {
  for (uint32_t i = lane; i < n; i += 32) d[i] = s[i];
}

// Copy n bytes (n <= 4096) from s to d with the whole warp.
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, uint32_t n,
                                          uint32_t lane, uint64_t pol) {
  const uintptr_t da = reinterpret_cast<uintptr_t>(d), sa = reinterpret_cast<uintptr_t>(s);
  if (((da ^ sa) & 15) == 0) {
    const uint32_t head = min(n, (uint32_t)((16 - (da & 15)) & 15));
    if (lane < head) d[lane] = s[lane];
    const uint32_t nv = (n - head) >> 4;
    const uint4* sv = reinterpret_cast<const uint4*>(s + head);
    uint4* dv = reinterpret_cast<uint4*>(d + head);
    uint4 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t i = lane + 32 * j;
      if (i < nv) r[j] = ld_v4_stream(sv + i, pol);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t i = lane + 32 * j;
      if (i < nv) st_v4_stream(dv + i, r[j], pol);
    }
    const uint32_t done = head + (nv << 4), tail = n - done;
    if (lane < tail) d[done + lane] = s[done + lane];
    return;
  }
  // Destination-aligned 4-byte words; the source is realigned with funnel
  // shifts from aligned words (never reading past the word holding the last
  // source byte).
  const uint32_t head = min(n, (uint32_t)((4 - (da & 3)) & 3));
  if (lane < head) d[lane] = s[lane];
  const uint32_t nw = (n - head) >> 2;
  const uint8_t* s1 = s + head;
  uint32_t* dw = reinterpret_cast<uint32_t*>(d + head);
  const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(s1) & 3);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(s1) & ~uintptr_t(3));
  if (sh == 0) {
    for (uint32_t i = lane; i < nw; i += 32) dw[i] = __ldg(sw + i);
  } else {
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < nw; i0 += 32 * 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t i = i0 + lane + 32 * j;
        if (i < nw) {
          const uint32_t lo = __ldg(sw + i), hi = __ldg(sw + i + 1);
          v[j] = __funnelshift_r(lo, hi, 8 * sh);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t i = i0 + lane + 32 * j;
        if (i < nw) dw[i] = v[j];
      }
    }
  }
  const uint32_t done = head + (nw << 2), tail = n - done;
  if (lane < tail) d[done + lane] = s[done + lane];
}

// Copy with 16-byte vectors only, for chunks whose source and destination
// agree modulo 16 (the host proves it per batch: (gva - src) mod 16 is an op
// constant); a chunk that does not qualify still copies correctly byte-wise.
__device__ __forceinline__ void warp_copy_aligned(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, uint32_t n,
                                                  uint32_t lane, uint64_t pol) {
  const uintptr_t da = reinterpret_cast<uintptr_t>(d), sa = reinterpret_cast<uintptr_t>(s);
  if (((da ^ sa) & 15) != 0) {
    warp_copy_bytes(d, s, n, lane);
    return;
  }
  const uint32_t head = min(n, (uint32_t)((16 - (da & 15)) & 15));
  if (lane < head) d[lane] = s[lane];
  const uint32_t nv = (n - head) >> 4;
  const uint4* sv = reinterpret_cast<const uint4*>(s + head);
  uint4* dv = reinterpret_cast<uint4*>(d + head);
  uint4 r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t i = lane + 32 * j;
    if (i < nv) r[j] = ld_v4_stream(sv + i, pol);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t i = lane + 32 * j;
    if (i < nv) st_v4_stream(dv + i, r[j], pol);
  }
  const uint32_t done = head + (nv << 4), tail = n - done;
  if (lane < tail) d[done + lane] = s[done + lane];
}

template <bool kAligned>
__global__ void __launch_bounds__(kExecTpb, kAligned ? 4 : 2)
exec_kernel(uint8_t* __restrict__ image, uint64_t image_bytes, const pv_op* __restrict__ ops, uint64_t n_ops,
            const uint64_t* __restrict__ page_off, uint64_t n_pages, uint32_t direction,
            const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ page_status,
            const uint64_t* __restrict__ page_aux, const unsigned long long* __restrict__ op_first_bad,
            uint8_t* __restrict__ buf, pv_op_result* __restrict__ results, uint8_t* __restrict__ dirty,
            const uint32_t* __restrict__ abort_flag) {
  // A conflicted batch (stamp pass) is left untouched for the host to re-plan.
  if (abort_flag != nullptr && *abort_flag != 0) return;
  const uint64_t pol = policy_evict_first();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = warp; w * kExecPpw < n_pages; w += nwarps) {
    const uint64_t p0 = w * kExecPpw;
    uint64_t op = upper_search(page_off, 0, n_ops, p0);
    uint64_t op_begin = __ldg(page_off + op), op_end = __ldg(page_off + op + 1);
#pragma unroll 1
    for (uint64_t p = p0; p < p0 + kExecPpw && p < n_pages; ++p) {
      while (p >= op_end) {
        ++op;
        op_begin = op_end;
        op_end = __ldg(page_off + op + 1);
      }
      const pv_op o = ops[op];
      const uint64_t k = p - op_begin;
      const uint64_t bad = op_first_bad[op];
      const uint64_t cur = op_page_va(o.gva, k);
      const uint64_t done = cur - o.gva;
      if (lane == 0) {
        // Exactly one page writes each op's result.
        if (bad == kNone ? k == 0 : k == bad) {
          pv_op_result r;
          if (bad == kNone) {
            r.copied = o.len;
            r.value = 0;
            r.aux = 0;
            r.status = PV_ST_OK;
            r.fail_page = 0;
          } else {
            r.copied = done;
            r.value = page_hpa[p];
            r.aux = page_aux != nullptr ? page_aux[p] : 0;
            r.status = page_status[p];
            r.fail_page = (uint32_t)k;
          }
          results[op] = r;
        }
      }
      if (k >= bad) continue;
      const uint64_t hpa = page_hpa[p];
      const uint32_t chunk = (uint32_t)min(o.len - done, kPageSize - (cur & kPageMask));
      uint8_t* bp = buf + o.buf_off + done;
      uint8_t* dst = direction == PV_TO_GUEST ? image + hpa : bp;
      const uint8_t* src = direction == PV_TO_GUEST ? bp : image + hpa;
      if (kAligned) warp_copy_aligned(dst, src, chunk, lane, pol);
      else warp_copy(dst, src, chunk, lane, pol);
      if (direction == PV_TO_GUEST && dirty != nullptr && lane == 0) dirty[hpa >> kPageShift] = 1;
    }
  }
}

cudaError_t launch_copy_plan(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_op* ops,
                             uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages, uint64_t* page_hpa,
                             uint32_t* page_status, uint64_t* page_aux, uint64_t* op_first_bad, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const uint64_t threads = (n_pages + kPlanPpt - 1) / kPlanPpt;
  uint64_t grid = (threads + kPlanTpb - 1) / kPlanTpb;
  const uint64_t cap = resident_grid((const void*)plan_kernel, kPlanTpb, 0);
  if (grid > cap) grid = cap;
  plan_kernel<<<(unsigned)grid, kPlanTpb, 0, stream>>>(image, image_bytes, spaces, ops, n_ops, page_off, n_pages,
                                                       page_hpa, page_status, page_aux,
                                                       reinterpret_cast<unsigned long long*>(op_first_bad));
  return cudaGetLastError();
}

cudaError_t launch_copy_stamp(const uint64_t* page_off, uint64_t n_ops, uint64_t n_pages, const uint64_t* page_hpa,
                              const uint64_t* op_first_bad, uint64_t* owner, uint64_t owner_pages, uint32_t epoch,
                              uint32_t* conflict, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const uint64_t threads = (n_pages + kPlanPpt - 1) / kPlanPpt;
  uint64_t grid = (threads + kPlanTpb - 1) / kPlanTpb;
  const uint64_t cap = resident_grid((const void*)stamp_kernel, kPlanTpb, 0);
  if (grid > cap) grid = cap;
  stamp_kernel<<<(unsigned)grid, kPlanTpb, 0, stream>>>(
      page_off, n_ops, n_pages, page_hpa, reinterpret_cast<const unsigned long long*>(op_first_bad),
      reinterpret_cast<unsigned long long*>(owner), owner_pages, epoch, conflict);
  return cudaGetLastError();
}

cudaError_t launch_copy_exec(uint8_t* image, uint64_t image_bytes, const pv_op* ops, uint64_t n_ops,
                             const uint64_t* page_off, uint64_t n_pages, uint32_t direction, const uint64_t* page_hpa,
                             const uint32_t* page_status, const uint64_t* page_aux, const uint64_t* op_first_bad,
                             uint8_t* buf, pv_op_result* results, uint8_t* dirty, const uint32_t* abort_flag,
                             cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const bool aligned = direction & PV_COPY_ALIGNED16;
  direction &= ~PV_COPY_ALIGNED16;
  auto k = aligned ? exec_kernel<true> : exec_kernel<false>;
  const uint64_t warps = (n_pages + kExecPpw - 1) / kExecPpw;
  uint64_t grid = (warps + kExecWarps - 1) / kExecWarps;
  const uint64_t cap = resident_grid((const void*)k, kExecTpb, 0);
  if (grid > cap) grid = cap;
  k<<<(unsigned)grid, kExecTpb, 0, stream>>>(image, image_bytes, ops, n_ops, page_off, n_pages, direction, page_hpa,
                                             page_status, page_aux,
                                             reinterpret_cast<const unsigned long long*>(op_first_bad), buf, results,
                                             dirty, abort_flag);
  return cudaGetLastError();
}

}  // namespace pv
