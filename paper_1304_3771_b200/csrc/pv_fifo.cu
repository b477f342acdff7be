// pv_fifo.cu — K4: exact replay of the per-process FIFO translation cache.
//
// The reference's TranslationCache (memvirt.py:336-374) is a per-process
// FIFO of (gva page, hpa page) pairs: capacity 10, linear lookup, insert only
// on a miss that resolved, oldest-first eviction independent of hits, hit /
// miss counters.  ProcessTranslator.translate (memvirt.py:585-594) consults
// it before walking.  Results may differ from a fresh walk when an entry is
// stale (tables edited without flush_page, e.g. backend.py:164-174 or the
// trap shim backend.py:288-296), and the counters are pinned metrics
// (harness.py:180-184), so the replay is exact and order-preserving.
//
// B200 design: one warp per process.  Lane i holds ring slot i of the cache
// (key, value); a lookup is a broadcast key, one __ballot_sync compare over
// the live slots and a shuffle of the hit value.  Lookup inputs are fetched
// 32 at a time (one per lane, coalesced) and results written back 32 at a
// time, so the sequential part is only the compare/insert chain.
#include "pv_common.cuh"

namespace pv {

struct WarpFifo {
  uint64_t key, val;  // this lane's slot
  uint32_t cap, len, head;
  uint64_t hits, misses;

  __device__ void load(const pv_fifo& f, uint32_t lane) {
    cap = f.capacity;
    len = f.len;
    head = f.head;
    hits = f.hits;
    misses = f.misses;
    key = lane < PV_FIFO_MAX ? f.key[lane] : 0;
    val = lane < PV_FIFO_MAX ? f.val[lane] : 0;
  }
  __device__ void store(pv_fifo& f, uint32_t lane) const {
    f.key[lane] = key;
    f.val[lane] = val;
    if (lane == 0) {
      f.len = len;
      f.head = head;
      f.hits = hits;
      f.misses = misses;
    }
  }
  // Is lane's slot live?  Live slots are head .. head+len-1 (mod cap).
  __device__ __forceinline__ bool live(uint32_t lane) const {
    if (lane >= cap) return false;
    const uint32_t rel = lane >= head ? lane - head : lane + cap - head;
    return rel < len;
  }
  // Returns true on a hit with *v = cached value (broadcast to all lanes).
  __device__ __forceinline__ bool lookup(uint64_t k, uint32_t lane, uint64_t* v) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, live(lane) && key == k);
    if (m) {
      *v = __shfl_sync(0xFFFFFFFFu, val, __ffs(m) - 1);
      ++hits;
      return true;
    }
    ++misses;
    return false;
  }
  __device__ __forceinline__ void insert(uint64_t k, uint64_t v, uint32_t lane) {
    uint32_t slot;
    if (len >= cap) {
      slot = head;
      head = head + 1 == cap ? 0 : head + 1;
    } else {
      slot = head + len;
      if (slot >= cap) slot -= cap;
      ++len;
    }
    if (lane == slot) {
      key = k;
      val = v;
    }
  }
};

// Translate-lane replay: lookups are whole lanes of a pv_translate batch.
template <bool kVa32>
__global__ void fifo_lanes_kernel(const void* __restrict__ vas, const uint64_t* __restrict__ lane_idx,
                                  const uint64_t* __restrict__ proc_off, uint32_t n_procs, pv_fifo* __restrict__ fifo,
                                  uint64_t* __restrict__ value, uint32_t* __restrict__ status) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t proc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (proc >= n_procs) return;
  WarpFifo c;
  c.load(fifo[proc], lane);
  const uint64_t b = proc_off[proc], e = proc_off[proc + 1];
  for (uint64_t base = b; base < e; base += 32) {
    const uint64_t mine = base + lane;
    uint64_t li = 0, va = 0, v = 0;
    uint32_t st = 0;
    if (mine < e) {
      li = lane_idx[mine];
      va = kVa32 ? (uint64_t)((const uint32_t*)vas)[li] : ((const uint64_t*)vas)[li];
      v = value[li];
      st = status[li];
    }
    bool changed = false;
    const uint32_t n = (uint32_t)(e - base < 32 ? e - base : 32);
    for (uint32_t j = 0; j < n; ++j) {
      const uint64_t vj = __shfl_sync(0xFFFFFFFFu, va, j);
      const uint64_t fresh = __shfl_sync(0xFFFFFFFFu, v, j);
      const uint32_t sj = __shfl_sync(0xFFFFFFFFu, st, j);
      uint64_t hv;
      if (c.lookup(vj >> kPageShift, lane, &hv)) {
        if (lane == j) {
          v = (hv << kPageShift) | (vj & kPageMask);
          st = PV_ST_OK;
          changed = true;
        }
      } else if (sj == PV_ST_OK) {
        c.insert(vj >> kPageShift, fresh >> kPageShift, lane);
      }
    }
    if (changed) {
      value[li] = v;
      status[li] = st;
    }
  }
  c.store(fifo[proc], lane);
}

// Copy-plan replay: lookups are the pages of each op of the process, in op
// order and page order; an op stops at its first page that misses and fails
// to resolve, or whose data access is out of range.
__global__ void fifo_copy_kernel(const pv_op* __restrict__ ops, const uint64_t* __restrict__ page_off,
                                 const uint64_t* __restrict__ op_idx, const uint64_t* __restrict__ proc_off,
                                 uint32_t n_procs, pv_fifo* __restrict__ fifo, uint64_t image_bytes,
                                 uint64_t* __restrict__ page_hpa, uint32_t* __restrict__ page_status,
                                 unsigned long long* __restrict__ op_first_bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t proc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (proc >= n_procs) return;
  WarpFifo c;
  c.load(fifo[proc], lane);
  for (uint64_t q = proc_off[proc]; q < proc_off[proc + 1]; ++q) {
    const uint64_t op = op_idx[q];
    const pv_op o = ops[op];
    const uint64_t p_begin = page_off[op], p_end = page_off[op + 1];
    uint64_t bad = kNone;
    for (uint64_t base = p_begin; base < p_end && bad == kNone; base += 32) {
      const uint64_t mine = base + lane;
      uint64_t v = 0;
      uint32_t st = 0;
      if (mine < p_end) {
        v = page_hpa[mine];
        st = page_status[mine];
      }
      bool changed = false;
      const uint32_t n = (uint32_t)(p_end - base < 32 ? p_end - base : 32);
      for (uint32_t j = 0; j < n; ++j) {
        const uint64_t k = base + j - p_begin;
        const uint64_t cur = op_page_va(o.gva, k);
        const uint64_t chunk = min(o.len - (cur - o.gva), kPageSize - (cur & kPageMask));
        const uint64_t fresh = __shfl_sync(0xFFFFFFFFu, v, j);
        const uint32_t sj = __shfl_sync(0xFFFFFFFFu, st, j);
        uint64_t hv;
        if (c.lookup(cur >> kPageShift, lane, &hv)) {
          const uint64_t hpa = (hv << kPageShift) | (cur & kPageMask);
          const bool oor = hpa + chunk > image_bytes || hpa + chunk < hpa;
          if (lane == j) {
            v = hpa;
            st = oor ? PV_ST_DATA_OOR : PV_ST_OK;
            changed = true;
          }
          if (oor) {
            bad = k;
            break;
          }
        } else {
          // A resolved walk is cached even when the data access then fails.
          if (sj == PV_ST_OK || sj == PV_ST_DATA_OOR) c.insert(cur >> kPageShift, fresh >> kPageShift, lane);
          if (sj != PV_ST_OK) {
            bad = k;
            break;
          }
        }
      }
      if (changed && mine < p_end) {
        page_hpa[mine] = v;
        page_status[mine] = st;
      }
    }
    if (lane == 0) op_first_bad[op] = bad;
  }
  c.store(fifo[proc], lane);
}

cudaError_t launch_fifo_lanes(const void* vas, uint32_t flags, const uint64_t* lane_idx, const uint64_t* proc_off,
                              uint32_t n_procs, pv_fifo* fifo, uint64_t* value, uint32_t* status,
                              cudaStream_t stream) {
  if (n_procs == 0) return cudaSuccess;
  const uint32_t warps = 4;
  const uint32_t grid = (n_procs + warps - 1) / warps;
  if (flags & PV_VA32)
    fifo_lanes_kernel<true><<<grid, warps * 32, 0, stream>>>(vas, lane_idx, proc_off, n_procs, fifo, value, status);
  else
    fifo_lanes_kernel<false><<<grid, warps * 32, 0, stream>>>(vas, lane_idx, proc_off, n_procs, fifo, value, status);
  return cudaGetLastError();
}

cudaError_t launch_fifo_copy(const pv_op* ops, const uint64_t* page_off, const uint64_t* op_idx,
                             const uint64_t* proc_off, uint32_t n_procs, pv_fifo* fifo, uint64_t image_bytes,
                             uint64_t* page_hpa, uint32_t* page_status, uint64_t* op_first_bad, cudaStream_t stream) {
  if (n_procs == 0) return cudaSuccess;
  const uint32_t warps = 4;
  const uint32_t grid = (n_procs + warps - 1) / warps;
  fifo_copy_kernel<<<grid, warps * 32, 0, stream>>>(ops, page_off, op_idx, proc_off, n_procs, fifo, image_bytes,
                                                   page_hpa, page_status,
                                                   reinterpret_cast<unsigned long long*>(op_first_bad));
  return cudaGetLastError();
}

}  // namespace pv
