// pv_common.cuh — shared device helpers of the HAS data plane.
//
// PTE codec and the three-level walk of the reference (memvirt.py:51-66,
// 99-121, 244-259), restated for sm_100a: one u64 load per level, trapping
// wins over present (memvirt.py:111-116), the writable bit is never
// consulted (memvirt.py:244-259), bits 3-11 are ignored, the VA top index is
// masked to 2 bits so VA bits >= 32 alias (memvirt.py:121).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/pv.h"

namespace pv {

// Measurement hook (pv_timing): event pair around a named launch when enabled.
void* timing_begin(const char* name, cudaStream_t stream);
void timing_end(void* token, cudaStream_t stream);

constexpr uint32_t kPageShift = 12;
constexpr uint64_t kPageSize = 4096;
constexpr uint64_t kPageMask = kPageSize - 1;
constexpr uint64_t kFlagPresent = 0x1;
constexpr uint64_t kFlagTrapping = 0x4;
constexpr uint64_t kNone = ~0ull;

__host__ __device__ __forceinline__ uint32_t top_index(uint64_t va) { return (uint32_t)(va >> 30) & 0x3u; }
__host__ __device__ __forceinline__ uint32_t mid_index(uint64_t va) { return (uint32_t)(va >> 21) & 0x1FFu; }
__host__ __device__ __forceinline__ uint32_t leaf_index(uint64_t va) { return (uint32_t)(va >> 12) & 0x1FFu; }

// Number of whole nodes addressable in a window with byte base `base`.
__host__ __device__ __forceinline__ uint64_t node_limit(uint64_t image_bytes, uint64_t base) {
  return base >= image_bytes ? 0 : (image_bytes - base) >> kPageShift;
}

template <bool kCoherent = false>
__device__ __forceinline__ uint64_t ld_word(const uint8_t* image, uint64_t base, uint64_t pfn, uint32_t idx) {
  const auto* p = reinterpret_cast<const unsigned long long*>(image + base + (pfn << kPageShift)) + idx;
  // coherent (L2) loads for walks that must see this kernel's own writes
  return kCoherent ? __ldcg(p) : __ldg(p);
}

// L2 cache-policy descriptors: streamed data (VAs, results, payload) is
// evict-first so it does not push the page tables out of the 126 MB L2;
// page-table gathers are evict-last.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_u64_hint(const void* p, uint64_t pol) {
  unsigned long long v;
  asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_u64_stream(void* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_u32_stream(void* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// Classify one entry word at `level`.  Returns PV_ST_OK and advances *node,
// or a status word (fault / trap) for the walk's stage.
__device__ __forceinline__ uint32_t classify(uint64_t w, uint32_t level, uint32_t index, uint32_t stage2,
                                             uint64_t* node, uint64_t* trap_node) {
  if (w & kFlagTrapping) {
    *trap_node = *node;
    return (stage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | level | (index << 16);
  }
  if (!(w & kFlagPresent)) return (stage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | level;
  *node = w >> kPageShift;
  return PV_ST_OK;
}

// Table-node marks (the to_guest table-hazard check, pv_copy_plan_nodes):
// node_map[absolute image page] = epoch for every node a walk reads.  Most
// walks share their upper nodes, so the mark is a read (an L1 hit) and a
// store only when the page is not marked yet.
struct NodeMarks {
  uint32_t* map;  // one u32 per image page, or nullptr (no marking)
  uint32_t epoch;
};

// The node pages one walk reads, in order (a copy_small table-hazard check).
struct NodeList {
  static constexpr uint32_t kCap = 16;  // 6 levels (two stages), 2 pages each when a window is unaligned
  uint64_t page[kCap];
  uint32_t n;
};

__device__ __forceinline__ void mark_node(NodeList* nl, uint64_t base, uint64_t node) {
  if (nl == nullptr) return;
  const uint64_t at = base + (node << kPageShift);
  if (nl->n < NodeList::kCap) nl->page[nl->n++] = at >> kPageShift;
  if ((at & kPageMask) && nl->n < NodeList::kCap) nl->page[nl->n++] = (at >> kPageShift) + 1;
}

__device__ __forceinline__ void mark_node(const NodeMarks* nm, uint64_t base, uint64_t node) {
  if (nm == nullptr) return;
  const uint64_t at = base + (node << kPageShift);  // a window base need not be page aligned
  uint32_t* p = nm->map + (at >> kPageShift);
  // a plain (L1-cached) read: a stale value only costs a redundant store
  if (*p != nm->epoch) *p = nm->epoch;
  if ((at & kPageMask) && p[1] != nm->epoch) p[1] = nm->epoch;
}

// Full three-level walk through global memory (L1/L2 cached).  On success
// returns PV_ST_OK with *out = leaf target pfn.  On a trap *out = node pfn.
// With nm != nullptr every node read is marked (mark_node).
template <bool kCoherent = false, class M = const NodeMarks*>
__device__ __forceinline__ uint32_t walk_global(const uint8_t* __restrict__ image, uint64_t image_bytes,
                                                uint64_t base, uint64_t root, uint64_t va, uint32_t stage2,
                                                uint64_t* out, M nm = nullptr) {
  const uint64_t lim = node_limit(image_bytes, base);
  uint64_t node = root, trap_node = 0;
  const uint32_t idx[3] = {top_index(va), mid_index(va), leaf_index(va)};
#pragma unroll
  for (uint32_t l = 0; l < 3; ++l) {
    if (node >= lim) return (stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | (l + 1);
    mark_node(nm, base, node);
    const uint64_t w = ld_word<kCoherent>(image, base, node, idx[l]);
    const uint32_t st = classify(w, l + 1, idx[l], stage2, &node, &trap_node);
    if (st != PV_ST_OK) {
      *out = trap_node;
      return st;
    }
  }
  *out = node;
  return PV_ST_OK;
}

// Extension geometry PV_ONE_STAGE_4L: 4 levels of 512 entries over 48-bit
// VAs, 2 MiB leaves at level 3 (PV_FLAG_PS).  Returns the 4 KiB frame of
// va (for a 2 MiB leaf: its pfn + va's 4 KiB index inside it).
template <bool kCoherent = false, class M = const NodeMarks*>
__device__ __forceinline__ uint32_t walk4_global(const uint8_t* __restrict__ image, uint64_t image_bytes,
                                                 uint64_t base, uint64_t root, uint64_t va, uint64_t* out,
                                                 M nm = nullptr) {
  const uint64_t lim = node_limit(image_bytes, base);
  const uint32_t idx[4] = {(uint32_t)(va >> 39) & 511u, (uint32_t)(va >> 30) & 511u, (uint32_t)(va >> 21) & 511u,
                           (uint32_t)(va >> 12) & 511u};
  uint64_t node = root;
#pragma unroll
  for (uint32_t l = 0; l < 4; ++l) {
    if (node >= lim) return PV_ST_NODE_OOR | (l + 1);
    mark_node(nm, base, node);
    const uint64_t w = ld_word<kCoherent>(image, base, node, idx[l]);
    if (w & kFlagTrapping) {
      *out = node;
      return PV_ST_TRAP | (l + 1) | (idx[l] << 16);
    }
    if (!(w & kFlagPresent)) return PV_ST_FAULT | (l + 1);
    if (l == 2 && (w & PV_FLAG_PS)) {
      *out = (w >> kPageShift) + idx[3];
      return PV_ST_OK;
    }
    node = w >> kPageShift;
  }
  *out = node;
  return PV_ST_OK;
}

// Translate `va` through a space with global-memory walks.  On success
// *value = leaf pfn of the final stage.  On failure *value / *aux follow the
// pv.h status conventions (va or gpa for faults, node pfn for traps).
template <bool kCoherent = false, class M = const NodeMarks*>
__device__ __forceinline__ uint32_t translate_global(const uint8_t* __restrict__ image, uint64_t image_bytes,
                                                     const pv_space& sp, uint64_t va, uint64_t* value,
                                                     uint64_t* aux, M nm = nullptr) {
  uint64_t r = 0;
  if (sp.mode == PV_ONE_STAGE_4L) {
    const uint32_t st4 = walk4_global<kCoherent>(image, image_bytes, sp.s1_base, sp.s1_root_pfn, va, &r, nm);
    *value = (st4 == PV_ST_OK || PV_ST_KIND(st4) == PV_ST_TRAP) ? r : va;
    return st4;
  }
  uint32_t st = walk_global<kCoherent>(image, image_bytes, sp.s1_base, sp.s1_root_pfn, va, 0, &r, nm);
  if (st != PV_ST_OK) {
    *value = (PV_ST_KIND(st) == PV_ST_TRAP) ? r : va;
    return st;
  }
  if (sp.mode != PV_TWO_STAGE) {
    *value = r;
    return PV_ST_OK;
  }
  const uint64_t gpa = (r << kPageShift) | (va & kPageMask);
  st = walk_global<kCoherent>(image, image_bytes, 0, sp.s2_root_pfn, gpa, 1, &r, nm);
  if (st != PV_ST_OK) {
    if (PV_ST_KIND(st) == PV_ST_TRAP2) {
      *value = r;
      *aux = gpa;
    } else {
      *value = gpa;
    }
    return st;
  }
  *value = r;
  return PV_ST_OK;
}

// PV_OUT_PACKED lane word (pv.h): the value when the lane translated, else
// PV_PACKED_ERR | compact status << 42 | value (a value wider than 42 bits
// spills: *spill is set and the low bits read PV_PACKED_SPILL_VALUE).
__device__ __forceinline__ uint64_t pack_lane(uint32_t st, uint64_t v, bool* spill) {
  *spill = false;
  if (st == PV_ST_OK) return v;
  const uint64_t compact = (uint64_t)((st & 0xFFFu) | (((st >> 16) & 0x1FFu) << 12));
  uint64_t low = v;
  if (v >> PV_PACKED_VALUE_BITS) {
    *spill = true;
    low = PV_PACKED_SPILL_VALUE;
  }
  return PV_PACKED_ERR | (compact << PV_PACKED_VALUE_BITS) | low;
}

// Output forms of a translate launch (pv_translate / pv_translate_words).
constexpr uint32_t kOutSplit = 0;   // u64 value + u32 status (+ aux)
constexpr uint32_t kOutPacked = 1;  // PV_OUT_PACKED u64 lane words
constexpr uint32_t kOutWord = 2;    // pv_translate_words: u32 lane words + exception records

// Exception list of a kOutWord launch (pv.h pv_translate_words).
struct ExcSink {
  pv_exc* rec;
  uint64_t per;               // records per stripe (exc_cap / PV_EXC_STRIPES)
  unsigned long long* count;  // PV_EXC_STRIPES counters
  uint64_t lane_base;
};

// 4-byte lane word (pv.h pv_translate_words) of lane i; appends the lane's
// exception record when the word alone cannot carry its value.  v: the frame
// number of a lane that translated, else the exception's value.
// The 4-byte word of a lane (v: its frame number, or its exception's value)
// and whether the lane needs an exception record (its value is not its own
// va, or it carries a TDP-stage gpa: `has_aux`).
__device__ __forceinline__ uint32_t word_code(uint32_t st, uint64_t v, uint64_t va, bool has_aux, bool* need) {
  *need = false;
  if (st == PV_ST_OK) return (uint32_t)v;
  const uint32_t compact = (st & 0xFFFu) | (((st >> 16) & 0x1FFu) << 12);
  if (v == va && !has_aux) return PV_W32_ERR | PV_W32_VA | compact;
  *need = true;
  return PV_W32_ERR | compact;
}

// Every thread of the warp that reaches the call takes part (the slots of a
// warp's records are reserved with one atomic: a fault-heavy batch -- C4: a
// trap on one lane in ten -- would otherwise serialise on the counter).
__device__ __forceinline__ uint32_t word_lane(uint32_t st, uint64_t v, uint64_t va, uint64_t aux, uint64_t i,
                                              const ExcSink& x) {
  const uint32_t compact = (st & 0xFFFu) | (((st >> 16) & 0x1FFu) << 12);
  const bool ok = st == PV_ST_OK;
  const bool va_valued = !ok && v == va && PV_ST_KIND(st) != PV_ST_TRAP2;
  const bool need = !ok && !va_valued;
  const unsigned mask = __activemask();
  const unsigned b = __ballot_sync(mask, need);
  if (ok) return (uint32_t)v;
  if (va_valued) return PV_W32_ERR | PV_W32_VA | compact;
  const int me = (int)(threadIdx.x & 31u);
  const int leader = __ffs(b) - 1;
  const uint32_t stripe = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % PV_EXC_STRIPES;
  unsigned long long base = 0;
  if (me == leader) base = atomicAdd(x.count + stripe, (unsigned long long)__popc(b));
  base = __shfl_sync(b, base, leader);
  const unsigned long long k = base + (unsigned long long)__popc(b & ((1u << me) - 1u));
  if (k < x.per) {
    pv_exc r;
    r.lane = x.lane_base + i;
    r.value = v;
    r.aux = aux;
    r.status = st;
    r.reserved = 0;
    x.rec[stripe * x.per + k] = r;
  }
  return PV_W32_ERR | compact;
}

__host__ __device__ __forceinline__ uint64_t page_span(uint64_t gva, uint64_t len) {
  return len == 0 ? 0 : ((gva + len - 1) >> kPageShift) - (gva >> kPageShift) + 1;
}

// VA of page k of an op (the first chunk keeps the unaligned start;
// memvirt.py:615-619).
__host__ __device__ __forceinline__ uint64_t op_page_va(uint64_t gva, uint64_t k) {
  return k == 0 ? gva : ((gva >> kPageShift) + k) << kPageShift;
}

// Bytes of a `len`-byte chunk at buffer offset `at` that lie inside a
// `buf_bytes`-byte op buffer (a short host_buf slice, memvirt.py:624).
__host__ __device__ __forceinline__ uint32_t buf_clamp(uint64_t at, uint32_t len, uint64_t buf_bytes) {
  return at >= buf_bytes ? 0u : (buf_bytes - at < len ? (uint32_t)(buf_bytes - at) : len);
}

// Largest i with off[i] <= p, searching [lo, hi).
__device__ __forceinline__ uint64_t upper_search(const uint64_t* __restrict__ off, uint64_t lo, uint64_t hi,
                                                 uint64_t p) {
  while (hi - lo > 1) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(off + mid) <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// Per-call server mailbox (pv_copy.cu server_kernel, pv_abi.cu pv_server_*):
// mapped pinned host memory, one per device.
constexpr uint32_t kServerWalk = 1, kServerCopy = 2, kServerStop = 3;
constexpr uint64_t kServerRunning = 1, kServerExited = 2, kServerLaunched = 3;
struct ServerReq {
  uint32_t kind;
  uint32_t flags;
  uint64_t image, image_bytes, buf, buf_bytes, dirty, va;
  uint32_t n_pages;
  uint32_t reserved;
  pv_small_op op;  // op.space is the walk's space
};
static_assert(sizeof(ServerReq) % 8 == 0, "the server pulls requests in 8-byte words");
struct ServerBox {
  volatile uint64_t req_seq;  // written by the host after the request
  uint64_t pad0[15];
  ServerReq req;
  alignas(128) volatile uint64_t rep_seq;  // written by the server after the reply
  volatile uint64_t state;                 // kServer* (host: launched; server: running / exited)
  pv_one_result one;
  pv_small_result small;
};
cudaError_t launch_server(ServerBox* box, uint64_t idle_ns, cudaStream_t stream);

// Grid size that fills every SM with resident CTAs of `func` (cached per
// function and device; defined in pv_abi.cu).
uint64_t resident_grid(const void* func, int tpb, size_t smem);

// Stream-ordered device scratch for one call (cudaMallocAsync from the
// device's default pool, which is told once to keep up to 256 MiB cached so
// repeated calls do not go back to the driver); release with cudaFreeAsync
// on the same stream.
cudaError_t stream_scratch(void** p, size_t bytes, cudaStream_t stream);

// Raise a kernel's dynamic shared-memory limit once per (kernel, device),
// thread-safe.
cudaError_t ensure_dynamic_smem(const void* func, size_t bytes);

}  // namespace pv
