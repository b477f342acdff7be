// pv_copy.cu — K2/K3: batched copy_to_user / copy_from_user.
//
// Restates copy_user_buffer (memvirt.py:604-628) for a batch of operations:
//   * the translation is performed once per page touched; the first chunk
//     keeps the unaligned start, chunk = min(remaining, 4096 - (cur & 0xFFF));
//   * a page whose translation fails stops its op: every page before it is
//     copied, nothing after it; `copied` is the completed prefix
//     (PageFault.bytes_copied, memvirt.py:618-622);
//   * the data access is bounds-checked against host memory and raises
//     OutOfRange (memvirt.py:156-168) -- also a stopping point;
//   * the op buffer side is clamped at buf_bytes: a chunk reaching past the
//     buffer moves only the bytes the buffer holds, like the reference's
//     slices of a short host_buf (host_buf[copied:copied + chunk],
//     memvirt.py:624) -- the page is still translated and counted.
//
// B200 design: two launches over one flat page list of the batch.
//   plan  : one thread per 4 pages walks each page (L1-cached upper levels,
//           one dependent load per level) and records the op's first failing
//           page with a u64 atomicMin;
//   exec  : batches whose buffer and guest addresses agree modulo 16 (the
//           host proves it) move through TMA bulk copies (exec_bulk_kernel);
//           the rest: one warp per page chunk moves up to 4 KiB with 16-byte
//           vector loads/stores (8 x 16 B in flight per lane, all loads
//           issued before the stores), realigning with funnel shifts when
//           source and destination disagree modulo 4, byte loops only for
//           heads/tails.
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

template <bool kMark>
__global__ void __launch_bounds__(kPlanTpb)
plan_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_space* __restrict__ spaces,
            const pv_op* __restrict__ ops, uint64_t n_ops, const uint64_t* __restrict__ page_off, uint64_t n_pages,
            uint64_t* __restrict__ page_hpa, uint32_t* __restrict__ page_status, uint64_t* __restrict__ page_aux,
            unsigned long long* __restrict__ op_first_bad, NodeMarks marks) {
  const NodeMarks* nm = kMark ? &marks : nullptr;
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
      uint32_t st = translate_global(image, image_bytes, sp, cur, &value, &aux, nm);
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
             unsigned long long* __restrict__ owner, uint64_t owner_pages, uint32_t epoch, uint32_t* conflict,
             const uint32_t* __restrict__ node_map) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * kPlanPpt < n_pages; t += nthreads) {
    // a table hazard decides the batch (the host runs it page by page);
    // an overlap only stops the stamping (heavily overlapping batches do
    // not serialise on atomics) while the hazard check goes on
    const uint32_t seen_conflict = *reinterpret_cast<volatile const uint32_t*>(conflict);
    if (seen_conflict & PV_CONFLICT_TABLE) return;
    if (seen_conflict && node_map == nullptr) return;
    bool overlap = seen_conflict & PV_CONFLICT_OVERLAP;  // stamping is over; the hazard check goes on
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
      if (node_map != nullptr && __ldg(node_map + hp) == epoch) {  // writes a node the batch walks
        atomicOr(conflict, PV_CONFLICT_TABLE);
        return;
      }
      if (overlap) continue;
      const unsigned long long mine = ((unsigned long long)epoch << 40) | (p + 1);
      const unsigned long long seen = *reinterpret_cast<volatile const unsigned long long*>(owner + hp);
      if ((seen >> 40) == epoch && seen != mine) {  // already stamped by another chunk of this batch
        atomicOr(conflict, PV_CONFLICT_OVERLAP);
        if (node_map == nullptr) return;
        overlap = true;
        continue;
      }
      const unsigned long long old = atomicMax(owner + hp, mine);
      if ((old >> 40) == epoch && old != mine) {
        atomicOr(conflict, PV_CONFLICT_OVERLAP);
        if (node_map == nullptr) return;
        overlap = true;
      }
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

__global__ void __launch_bounds__(kExecTpb, 2)
exec_kernel(uint8_t* __restrict__ image, uint64_t image_bytes, const pv_op* __restrict__ ops, uint64_t n_ops,
            const uint64_t* __restrict__ page_off, uint64_t n_pages, uint32_t direction,
            const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ page_status,
            const uint64_t* __restrict__ page_aux, const unsigned long long* __restrict__ op_first_bad,
            uint8_t* __restrict__ buf, uint64_t buf_bytes, pv_op_result* __restrict__ results,
            uint8_t* __restrict__ dirty, const uint32_t* __restrict__ abort_flag) {
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
      const uint32_t chunk = buf_clamp(o.buf_off + done, (uint32_t)min(o.len - done, kPageSize - (cur & kPageMask)),
                                       buf_bytes);
      uint8_t* bp = buf + o.buf_off + done;
      uint8_t* dst = direction == PV_TO_GUEST ? image + hpa : bp;
      const uint8_t* src = direction == PV_TO_GUEST ? bp : image + hpa;
      warp_copy(dst, src, chunk, lane, pol);
      if (direction == PV_TO_GUEST && dirty != nullptr && lane == 0) dirty[hpa >> kPageShift] = 1;
    }
  }
}

// ---- TMA bulk exec (batches proven 16-byte co-aligned by the host) -----------
//
// Same semantics as exec_kernel; the data moves through the Tensor Memory
// Accelerator instead of the LSU: each warp owns a contiguous run of pages and
// one lane drives a kBulkStages-deep ring of 4 KiB shared-memory stages
// (cp.async.bulk global -> shared, completion on a per-stage mbarrier; then
// cp.async.bulk shared -> global, one bulk group per page), keeping
// kBulkStages - 1 page loads in flight.  The whole warp computes the page
// metadata 32 pages at a time (one page per lane, a batch ahead of the ring)
// and copies the < 16-byte head / tail of a chunk with the LSU.  Measured on
// the C5 pattern (scripts/tma_copy_probe.cu): 6.36 TB/s vs 6.16 TB/s for
// the best LSU copy.
#ifndef PV_BULK_WARPS
#define PV_BULK_WARPS 8
#endif
#ifndef PV_BULK_STAGES
#define PV_BULK_STAGES 6
#endif
#ifndef PV_BULK_EVICT_FIRST
#define PV_BULK_EVICT_FIRST 0  // evict-first bulk copies measured slower (exec 2.79 vs 2.75 ms, scripts/ab_evict.sh)
#endif
constexpr int kBulkWarps = PV_BULK_WARPS;
constexpr int kBulkStages = PV_BULK_STAGES;
constexpr size_t kBulkSmem = (size_t)kBulkWarps * kBulkStages * kPageSize;

struct BulkMeta {
  uint64_t src, dst;  // chunk start
  uint32_t head, mid, tail;  // LSU head bytes, TMA middle (16-byte multiple), LSU tail bytes
};

__device__ __forceinline__ uint64_t bulk_shfl64(uint64_t v, int j) {
  return ((uint64_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)(v >> 32), j) << 32) |
         __shfl_sync(0xFFFFFFFFu, (uint32_t)v, j);
}

__global__ void __launch_bounds__(kBulkWarps * 32, 1)
exec_bulk_kernel(uint8_t* __restrict__ image, uint64_t image_bytes, const pv_op* __restrict__ ops, uint64_t n_ops,
                 const uint64_t* __restrict__ page_off, uint64_t n_pages, uint32_t direction,
                 const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ page_status,
                 const uint64_t* __restrict__ page_aux, const unsigned long long* __restrict__ op_first_bad,
                 uint8_t* __restrict__ buf, uint64_t buf_bytes, pv_op_result* __restrict__ results,
                 uint8_t* __restrict__ dirty, const uint32_t* __restrict__ abort_flag) {
  extern __shared__ __align__(128) uint8_t bulk_ring[];
  __shared__ __align__(8) uint64_t bars[kBulkWarps][kBulkStages];
  if (abort_flag != nullptr && *abort_flag != 0) return;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* ring = bulk_ring + (size_t)wid * kBulkStages * kPageSize;
  if (lane == 0) {
    for (int st = 0; st < kBulkStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[wid][st])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t warp = (uint64_t)blockIdx.x * kBulkWarps + wid, nwarps = (uint64_t)gridDim.x * kBulkWarps;
  const uint64_t per = (n_pages + nwarps - 1) / nwarps;
  const uint64_t pb = min(warp * per, n_pages), pe = min(pb + per, n_pages);
  if (pb >= pe) return;
  const bool to_guest = direction == PV_TO_GUEST;
  const uint64_t pol = policy_evict_first();
  uint64_t op_hint = upper_search(page_off, 0, n_ops, pb);

  // Metadata of pages q .. q + 31 (one per lane); writes each op's result and
  // the dirty marks on the way.  Warp-collective.
  auto meta = [&](uint64_t q) {
    BulkMeta m;
    m.src = m.dst = 0;
    m.head = m.mid = m.tail = 0;
    const uint64_t p = q + lane;
    uint64_t oi = op_hint;
    if (p < pe) {
      while (__ldg(page_off + oi + 1) <= p) ++oi;
      const pv_op o = ops[oi];
      const uint64_t k = p - __ldg(page_off + oi);
      const uint64_t bad = op_first_bad[oi];
      const uint64_t cur = op_page_va(o.gva, k);
      const uint64_t done = cur - o.gva;
      if (bad == kNone ? k == 0 : k == bad) {  // exactly one page writes each op's result
        pv_op_result r;
        if (bad == kNone) {
          r.copied = o.len;
          r.value = r.aux = 0;
          r.status = PV_ST_OK;
          r.fail_page = 0;
        } else {
          r.copied = done;
          r.value = page_hpa[p];
          r.aux = page_aux != nullptr ? page_aux[p] : 0;
          r.status = page_status[p];
          r.fail_page = (uint32_t)k;
        }
        results[oi] = r;
      }
      if (k < bad) {
        const uint64_t hpa = page_hpa[p];
        const uint32_t len =
            buf_clamp(o.buf_off + done, (uint32_t)min(o.len - done, kPageSize - (cur & kPageMask)), buf_bytes);
        uint8_t* bp = buf + o.buf_off + done;
        m.dst = reinterpret_cast<uint64_t>(to_guest ? image + hpa : bp);
        m.src = reinterpret_cast<uint64_t>(to_guest ? bp : image + hpa);
        if ((m.src ^ m.dst) & 15) {
          m.head = len;  // not co-aligned: the whole chunk through the LSU
        } else {
          m.head = min(len, (uint32_t)((16 - (m.dst & 15)) & 15));
          const uint32_t rest = len - m.head;
          m.mid = rest & ~15u;
          m.tail = rest - m.mid;
        }
        if (to_guest && dirty != nullptr) dirty[hpa >> kPageShift] = 1;
      }
    }
    op_hint = __shfl_sync(0xFFFFFFFFu, oi, 31);
    return m;
  };
  const uint64_t n = pe - pb;
  BulkMeta cur = meta(pb), nxt = meta(pb + 32);
  uint64_t base = 0;  // slot of cur's lane 0
  auto slot_src = [&](uint64_t j) { return j - base < 32 ? bulk_shfl64(cur.src, (int)(j - base)) : bulk_shfl64(nxt.src, (int)(j - base - 32)); };
  auto slot_dst = [&](uint64_t j) { return j - base < 32 ? bulk_shfl64(cur.dst, (int)(j - base)) : bulk_shfl64(nxt.dst, (int)(j - base - 32)); };
  auto slot_u32 = [&](uint64_t j, uint32_t a, uint32_t b) {
    const uint32_t va = __shfl_sync(0xFFFFFFFFu, a, (int)((j - base) & 31));
    const uint32_t vb = __shfl_sync(0xFFFFFFFFu, b, (int)((j - base) & 31));
    return j - base < 32 ? va : vb;
  };
  auto issue_load = [&](uint64_t j) {  // all lanes call (shuffles); lane 0 issues
    const uint64_t src = slot_src(j), dst = slot_dst(j);
    const uint32_t head = slot_u32(j, cur.head, nxt.head), mid = slot_u32(j, cur.mid, nxt.mid);
    (void)dst;
    if (lane == 0 && mid != 0) {
      const int st = (int)(j % kBulkStages);
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[wid][st]);
      const uint32_t sm = (uint32_t)__cvta_generic_to_shared(ring + (size_t)st * kPageSize);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(mid) : "memory");
#if PV_BULK_EVICT_FIRST
      // streamed payload: evict-first in L2, so it does not push out what a walk beside it keeps there
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              sm),
          "l"(src + head), "r"(mid), "r"(bar), "l"(pol)
          : "memory");
#else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
                   "l"(src + head), "r"(mid), "r"(bar)
                   : "memory");
#endif
    }
  };
  for (uint64_t j = 0; j + 1 < (uint64_t)kBulkStages && j < n; ++j) issue_load(j);
  uint32_t parity = 0;  // lane 0: per-stage mbarrier phase bits
  for (uint64_t i = 0; i < n; ++i) {
    if (i - base == 32) {  // advance the metadata window (warp-uniform)
      cur = nxt;
      base += 32;
      nxt = meta(pb + base + 32);
    }
    const uint64_t src = slot_src(i), dst = slot_dst(i);
    const uint32_t head = slot_u32(i, cur.head, nxt.head), mid = slot_u32(i, cur.mid, nxt.mid),
                   tail = slot_u32(i, cur.tail, nxt.tail);
    if (lane == 0) {
      const int st = (int)(i % kBulkStages);
      if (mid != 0) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[wid][st]);
        const uint32_t ph = (parity >> st) & 1u;
        asm volatile(
            "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(bar),
            "r"(ph)
            : "memory");
        parity ^= 1u << st;
        const uint32_t sm = (uint32_t)__cvta_generic_to_shared(ring + (size_t)st * kPageSize);
#if PV_BULK_EVICT_FIRST
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst + head),
                     "r"(sm), "r"(mid), "l"(pol)
                     : "memory");
#else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head), "r"(sm), "r"(mid)
                     : "memory");
#endif
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // one group per slot, empty or not
    }
    if (head) warp_copy(reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), head, lane, pol);
    if (tail)
      warp_copy(reinterpret_cast<uint8_t*>(dst + head + mid), reinterpret_cast<const uint8_t*>(src + head + mid), tail,
                lane, pol);
    // the next load reuses the stage of slot i - 1, whose store must have read it out
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    if (i + kBulkStages - 1 < n) issue_load(i + kBulkStages - 1);
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- per-call path: one op per launch, request in the parameters -----------

__global__ void walk_one_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, pv_space sp, uint64_t va,
                                uint32_t flags, pv_one_result* out, uint64_t seq) {
  uint64_t value = 0, aux = 0;
  const uint32_t st = translate_global(image, image_bytes, sp, va, &value, &aux);
  if (st == PV_ST_OK && !(flags & PV_OUT_PFN)) value = (value << kPageShift) | (va & kPageMask);
  out->value = value;
  out->aux = aux;
  out->status = st;
  __threadfence_system();
  *reinterpret_cast<volatile uint64_t*>(&out->seq) = seq;
}

constexpr int kSmallTpb = 256;
static_assert(PV_SMALL_PAGES <= kSmallTpb, "one plan thread per page");

// Translation of page k of a small op: the caller's FIFO hit, or a walk
// (kCoherent: L2 loads that see this kernel's earlier writes).
template <bool kCoherent, class M>
__device__ __forceinline__ uint32_t small_page(const uint8_t* __restrict__ image, uint64_t image_bytes,
                                               const pv_small_op& op, uint32_t k, uint64_t* value, uint64_t* aux,
                                               M nodes) {
  const uint64_t cur = op_page_va(op.gva, k);
  const uint64_t done = cur - op.gva;
  const uint64_t chunk = min(op.len - done, kPageSize - (cur & kPageMask));
  const uint64_t hit = op.pre_hpa[k];
  uint32_t st = PV_ST_OK;
  if (hit != 0) {
    *value = hit - 1;  // the caller's translation (a FIFO hit): the byte hpa
  } else {
    st = translate_global<kCoherent>(image, image_bytes, op.space, cur, value, aux, nodes);
    if (st == PV_ST_OK) *value = (*value << kPageShift) | (cur & kPageMask);
  }
  if (st == PV_ST_OK && (*value + chunk > image_bytes || *value + chunk < *value))
    st = PV_ST_DATA_OOR;  // memvirt.py:156-158
  return st;
}

// The table-hazard form of copy_small_kernel, on one warp: page k is
// translated (coherent walk) and its chunk written before page k + 1 is
// translated (memvirt.py:615-627).
__device__ __noinline__ void small_sequential(uint8_t* __restrict__ image, uint64_t image_bytes,
                                              const pv_small_op& op, uint8_t* __restrict__ buf, uint64_t buf_bytes,
                                              pv_small_result* out, uint8_t* __restrict__ dirty, uint32_t n_pages,
                                              uint32_t lane) {
  const uint64_t pol = policy_evict_first();
  pv_op_result r;
  r.copied = op.len;
  r.value = r.aux = 0;
  r.status = PV_ST_OK;
  r.fail_page = 0;
  for (uint32_t k = 0; k < n_pages; ++k) {
    uint64_t value = 0, aux = 0;
    uint32_t st = 0;
    if (lane == 0) st = small_page<true>(image, image_bytes, op, k, &value, &aux, (NodeList*)nullptr);
    st = __shfl_sync(0xffffffffu, st, 0);
    value = __shfl_sync(0xffffffffu, value, 0);
    aux = __shfl_sync(0xffffffffu, aux, 0);
    if (lane == 0) {
      out->page_hpa[k] = value;
      out->page_status[k] = st;
    }
    const uint64_t cur = op_page_va(op.gva, k);
    const uint64_t done = cur - op.gva;
    if (st != PV_ST_OK) {
      r.copied = done;
      r.value = value;
      r.aux = aux;
      r.status = st;
      r.fail_page = k;
      break;
    }
    const uint32_t chunk = buf_clamp(done, (uint32_t)min(op.len - done, kPageSize - (cur & kPageMask)), buf_bytes);
    warp_copy(image + value, buf + done, chunk, lane, pol);
    if (dirty != nullptr && lane == 0) dirty[value >> kPageShift] = 1;
    __threadfence();  // the chunk is in L2 before the next page's walk reads it
    __syncwarp();
  }
  if (lane == 0) out->op = r;
}

// One CTA: thread k translates page k (or takes the caller's FIFO hit), the
// op's first failing page is a shared atomicMin, then warp w copies pages
// w, w + 8, ... below it (memvirt.py:615-627 prefix semantics).  A to_guest
// op whose chunk k lands on a table node the walk of a later page reads (a
// table hazard) runs page by page instead -- walk k, write k, walk k + 1
// through coherent loads -- exactly like copy_user_buffer.
// The op's body on one CTA of kSmallTpb threads (all threads call it; it ends
// with a barrier).  out->op, page_hpa, page_status are written; the caller
// publishes the completion.
__device__ __noinline__ void copy_small_body(uint8_t* __restrict__ image, uint64_t image_bytes, const pv_small_op& op,
                                             uint8_t* __restrict__ buf, uint64_t buf_bytes, pv_small_result* out,
                                             uint8_t* __restrict__ dirty, uint32_t n_pages) {
  __shared__ uint64_t s_hpa[PV_SMALL_PAGES];
  __shared__ NodeList s_nodes[PV_SMALL_PAGES];
  __shared__ uint32_t s_bad, s_hazard;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool to_guest = op.direction == PV_TO_GUEST;
  if (tid == 0) {
    s_bad = n_pages;
    s_hazard = 0;
  }
  __syncthreads();
  uint64_t value = 0, aux = 0;
  uint32_t st = PV_ST_OK;
  if (tid < n_pages) {
    s_nodes[tid].n = 0;
    st = small_page<false>(image, image_bytes, op, tid, &value, &aux, to_guest ? &s_nodes[tid] : nullptr);
    s_hpa[tid] = value;
    out->page_hpa[tid] = value;
    out->page_status[tid] = st;
    if (st != PV_ST_OK) atomicMin(&s_bad, tid);
  }
  __syncthreads();
  if (to_guest && tid < s_bad) {  // chunk tid is written: does a later page walk its page?
    const uint64_t dst = s_hpa[tid] >> kPageShift;
    for (uint32_t j = tid + 1; j < n_pages; ++j)
      for (uint32_t i = 0; i < s_nodes[j].n; ++i)
        if (s_nodes[j].page[i] == dst) s_hazard = 1;
  }
  __syncthreads();
  if (s_hazard) {
    if (warp == 0) small_sequential(image, image_bytes, op, buf, buf_bytes, out, dirty, n_pages, lane);
    __syncthreads();
    return;
  }
  const uint32_t bad = s_bad;
  if (tid == bad) {
    pv_op_result r;
    r.copied = op_page_va(op.gva, tid) - op.gva;
    r.value = value;
    r.aux = aux;
    r.status = st;
    r.fail_page = tid;
    out->op = r;
  } else if (tid == 0 && bad == n_pages) {
    pv_op_result r;
    r.copied = op.len;
    r.value = r.aux = 0;
    r.status = PV_ST_OK;
    r.fail_page = 0;
    out->op = r;
  }
  const uint64_t pol = policy_evict_first();
  for (uint32_t k = warp; k < bad; k += kSmallTpb / 32) {
    const uint64_t cur = op_page_va(op.gva, k);
    const uint64_t done = cur - op.gva;
    const uint32_t chunk = buf_clamp(done, (uint32_t)min(op.len - done, kPageSize - (cur & kPageMask)), buf_bytes);
    const uint64_t hpa = s_hpa[k];
    uint8_t* bp = buf + done;
    if (op.direction == PV_TO_GUEST) {
      warp_copy(image + hpa, bp, chunk, lane, pol);
      if (dirty != nullptr && lane == 0) dirty[hpa >> kPageShift] = 1;
    } else {
      warp_copy(bp, image + hpa, chunk, lane, pol);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallTpb)
copy_small_kernel(uint8_t* __restrict__ image, uint64_t image_bytes, pv_small_op op, uint8_t* __restrict__ buf,
                  uint64_t buf_bytes, pv_small_result* out, uint8_t* __restrict__ dirty, uint32_t n_pages,
                  uint64_t seq) {
  copy_small_body(image, image_bytes, op, buf, buf_bytes, out, dirty, n_pages);
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile uint64_t*>(&out->seq) = seq;
  }
}

// ---- per-call server: one resident CTA serving walk_one / copy_small requests
// posted in mapped pinned host memory (no launch per call).  Thread 0 polls
// the request sequence word with system-scope acquire loads; a request is
// pulled into shared memory by every thread at once (one link round trip),
// served by the same device code as walk_one_kernel / copy_small_kernel, and
// completed by a system-scope release of the reply sequence.  After idle_ns
// without a request the server marks itself exited, looks once more (a request
// posted meanwhile is served) and returns, so a device-wide synchronisation
// waits at most that long.

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const volatile uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(volatile uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kSmallTpb) server_kernel(ServerBox* box, uint64_t idle_ns) {
  __shared__ __align__(16) ServerReq s_req;
  __shared__ uint64_t s_seq;
  __shared__ uint32_t s_stop;
  const uint32_t tid = threadIdx.x;
  uint64_t last = 0;
  if (tid == 0) last = ld_acquire_sys_u64(&box->rep_seq);
  for (;;) {
    if (tid == 0) {
      const uint64_t t0 = globaltimer_ns();
      uint32_t stop = 0;
      uint64_t sq;
      for (;;) {
        sq = ld_acquire_sys_u64(&box->req_seq);
        if (sq != last) break;
        if (globaltimer_ns() - t0 > idle_ns) {
          st_release_sys_u64(&box->state, kServerExited);
          __threadfence_system();
          sq = ld_acquire_sys_u64(&box->req_seq);
          if (sq != last) {
            st_release_sys_u64(&box->state, kServerRunning);
            break;
          }
          stop = 1;
          break;
        }
      }
      s_seq = sq;
      s_stop = stop;
    }
    __syncthreads();
    if (s_stop) return;
    {  // pull the request (one round trip: every thread loads 8 bytes)
      const volatile uint64_t* src = reinterpret_cast<const volatile uint64_t*>(&box->req);
      uint64_t* dst = reinterpret_cast<uint64_t*>(&s_req);
      for (uint32_t i = tid; i < sizeof(ServerReq) / 8; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const uint32_t kind = s_req.kind;
    if (kind == kServerWalk) {
      if (tid == 0) {
        uint64_t value = 0, aux = 0;
        const uint64_t va = s_req.va;
        const uint32_t st = translate_global(reinterpret_cast<const uint8_t*>(s_req.image), s_req.image_bytes,
                                             s_req.op.space, va, &value, &aux);
        if (st == PV_ST_OK && !(s_req.flags & PV_OUT_PFN)) value = (value << kPageShift) | (va & kPageMask);
        box->one.value = value;
        box->one.aux = aux;
        box->one.status = st;
      }
    } else if (kind == kServerCopy) {
      copy_small_body(reinterpret_cast<uint8_t*>(s_req.image), s_req.image_bytes, s_req.op,
                      reinterpret_cast<uint8_t*>(s_req.buf), s_req.buf_bytes, &box->small,
                      reinterpret_cast<uint8_t*>(s_req.dirty), s_req.n_pages);
    }
    __syncthreads();
    if (tid == 0) {
      if (kind == kServerStop) st_release_sys_u64(&box->state, kServerExited);
      // the CTA's reply writes are ordered before this release by the barrier
      // above (cumulativity): no separate system fence
      st_release_sys_u64(&box->rep_seq, s_seq);
      last = s_seq;
    }
    if (kind == kServerStop) return;
  }
}

cudaError_t launch_server(ServerBox* box, uint64_t idle_ns, cudaStream_t stream) {
  server_kernel<<<1, kSmallTpb, 0, stream>>>(box, idle_ns);
  return cudaGetLastError();
}

cudaError_t launch_walk_one(const uint8_t* image, uint64_t image_bytes, const pv_space& sp, uint64_t va,
                            uint32_t flags, pv_one_result* out, uint64_t seq, cudaStream_t stream) {
  walk_one_kernel<<<1, 1, 0, stream>>>(image, image_bytes, sp, va, flags, out, seq);
  return cudaGetLastError();
}

cudaError_t launch_copy_small(uint8_t* image, uint64_t image_bytes, const pv_small_op& op, uint8_t* buf,
                              uint64_t buf_bytes, pv_small_result* out, uint8_t* dirty, uint32_t n_pages,
                              uint64_t seq, cudaStream_t stream) {
  copy_small_kernel<<<1, kSmallTpb, 0, stream>>>(image, image_bytes, op, buf, buf_bytes, out, dirty, n_pages, seq);
  return cudaGetLastError();
}

cudaError_t launch_copy_plan(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_op* ops,
                             uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages, uint64_t* page_hpa,
                             uint32_t* page_status, uint64_t* page_aux, uint64_t* op_first_bad, uint32_t* node_map,
                             uint32_t epoch, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const uint64_t threads = (n_pages + kPlanPpt - 1) / kPlanPpt;
  uint64_t grid = (threads + kPlanTpb - 1) / kPlanTpb;
  const NodeMarks marks{node_map, epoch};
  auto* fb = reinterpret_cast<unsigned long long*>(op_first_bad);
  void* tk = timing_begin("plan", stream);
  if (node_map != nullptr) {
    const uint64_t cap = resident_grid((const void*)plan_kernel<true>, kPlanTpb, 0);
    if (grid > cap) grid = cap;
    plan_kernel<true><<<(unsigned)grid, kPlanTpb, 0, stream>>>(image, image_bytes, spaces, ops, n_ops, page_off,
                                                               n_pages, page_hpa, page_status, page_aux, fb, marks);
  } else {
    const uint64_t cap = resident_grid((const void*)plan_kernel<false>, kPlanTpb, 0);
    if (grid > cap) grid = cap;
    plan_kernel<false><<<(unsigned)grid, kPlanTpb, 0, stream>>>(image, image_bytes, spaces, ops, n_ops, page_off,
                                                                n_pages, page_hpa, page_status, page_aux, fb, marks);
  }
  timing_end(tk, stream);
  return cudaGetLastError();
}

cudaError_t launch_copy_stamp(const uint64_t* page_off, uint64_t n_ops, uint64_t n_pages, const uint64_t* page_hpa,
                              const uint64_t* op_first_bad, uint64_t* owner, uint64_t owner_pages, uint32_t epoch,
                              uint32_t* conflict, const uint32_t* node_map, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const uint64_t threads = (n_pages + kPlanPpt - 1) / kPlanPpt;
  uint64_t grid = (threads + kPlanTpb - 1) / kPlanTpb;
  const uint64_t cap = resident_grid((const void*)stamp_kernel, kPlanTpb, 0);
  if (grid > cap) grid = cap;
  void* tk = timing_begin("stamp", stream);
  stamp_kernel<<<(unsigned)grid, kPlanTpb, 0, stream>>>(
      page_off, n_ops, n_pages, page_hpa, reinterpret_cast<const unsigned long long*>(op_first_bad),
      reinterpret_cast<unsigned long long*>(owner), owner_pages, epoch, conflict, node_map);
  timing_end(tk, stream);
  return cudaGetLastError();
}

cudaError_t launch_copy_exec(uint8_t* image, uint64_t image_bytes, const pv_op* ops, uint64_t n_ops,
                             const uint64_t* page_off, uint64_t n_pages, uint32_t direction, const uint64_t* page_hpa,
                             const uint32_t* page_status, const uint64_t* page_aux, const uint64_t* op_first_bad,
                             uint8_t* buf, uint64_t buf_bytes, pv_op_result* results, uint8_t* dirty,
                             const uint32_t* abort_flag, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  const bool aligned = direction & PV_COPY_ALIGNED16;
  direction &= ~PV_COPY_ALIGNED16;
  if (aligned) {
    // host-proven 16-byte co-alignment: the TMA bulk path (1 CTA of 8 warps per SM)
    const cudaError_t e = ensure_dynamic_smem((const void*)exec_bulk_kernel, kBulkSmem);
    if (e != cudaSuccess) return e;
    uint64_t grid = resident_grid((const void*)exec_bulk_kernel, kBulkWarps * 32, kBulkSmem);
    const uint64_t want = (n_pages + kBulkWarps - 1) / kBulkWarps;
    if (grid > want) grid = want;
    exec_bulk_kernel<<<(unsigned)grid, kBulkWarps * 32, kBulkSmem, stream>>>(
        image, image_bytes, ops, n_ops, page_off, n_pages, direction, page_hpa, page_status, page_aux,
        reinterpret_cast<const unsigned long long*>(op_first_bad), buf, buf_bytes, results, dirty, abort_flag);
    return cudaGetLastError();
  }
  auto k = exec_kernel;
  const uint64_t warps = (n_pages + kExecPpw - 1) / kExecPpw;
  uint64_t grid = (warps + kExecWarps - 1) / kExecWarps;
  const uint64_t cap = resident_grid((const void*)k, kExecTpb, 0);
  if (grid > cap) grid = cap;
  k<<<(unsigned)grid, kExecTpb, 0, stream>>>(image, image_bytes, ops, n_ops, page_off, n_pages, direction, page_hpa,
                                             page_status, page_aux,
                                             reinterpret_cast<const unsigned long long*>(op_first_bad), buf, buf_bytes,
                                             results, dirty, abort_flag);
  return cudaGetLastError();
}

}  // namespace pv
