// pv_translate.cu — K1: batched gva -> (gpa ->) hpa translation.
//
// Restates, for a whole batch of lanes at once, the reference's per-address
// walk (memvirt.py:244-259), walk_guest (memvirt.py:262-267), the uncached
// ProcessTranslator resolve (memvirt.py:596-601) and resolve_hybrid
// (memvirt.py:677-682).
//
// B200 design.  A CTA owns a contiguous run of 2048-lane chunks of one
// segment (one address space).  On entering a space it stages the space's
// top-level words and every present mid-level node (<= 4 x 4 KiB per stage)
// in shared memory, so the two upper levels of every walk are shared-memory
// lookups and each stage costs exactly one dependent global load: the leaf
// PTE (L1-allocating, since leaf tables are small and reused across lanes).
// Each thread walks 8 lanes at once (8 independent leaf loads in flight),
// VAs stream in with L1::no_allocate loads and results stream out with
// evict-first stores.
#include "pv_common.cuh"

namespace pv {

constexpr int kTpb = 256;
constexpr int kVpt = 8;
constexpr uint64_t kChunk = (uint64_t)kTpb * kVpt;  // lanes per chunk

struct StageSmem {
  uint64_t root;          // root pfn
  uint64_t lim;           // node limit of the window
  uint64_t base;          // window base
  uint64_t top_word[4];
  uint32_t top_status[4]; // PV_ST_OK if the mid node is staged, else final status
  uint64_t top_node[4];   // trap node (root) for level-1 traps / mid node pfn
};

__device__ __forceinline__ uint64_t ld_stream_va(const void* vas, uint64_t i, bool va32) {
  if (va32) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"((const uint32_t*)vas + i));
    return v;
  }
  unsigned long long v;
  asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"((const uint64_t*)vas + i));
  return v;
}

// Stage one walk stage: top words and present mid nodes.  Called by all
// threads of the CTA; ends with __syncthreads().
__device__ void stage_space(const uint8_t* __restrict__ image, uint64_t image_bytes, uint64_t base,
                            uint64_t root, uint32_t stage2, StageSmem& s, uint64_t* mid /*[4][512]*/) {
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    s.root = root;
    s.base = base;
    s.lim = node_limit(image_bytes, base);
  }
  if (tid < 4) {
    const uint64_t lim = node_limit(image_bytes, base);
    if (root >= lim) {
      s.top_word[tid] = 0;
      s.top_status[tid] = (stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 1u;
      s.top_node[tid] = 0;
    } else {
      const uint64_t w = ld_word(image, base, root, tid);
      s.top_word[tid] = w;
      if (w & kFlagTrapping) {
        s.top_status[tid] = (stage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | 1u | (tid << 16);
        s.top_node[tid] = root;
      } else if (!(w & kFlagPresent)) {
        s.top_status[tid] = (stage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | 1u;
        s.top_node[tid] = 0;
      } else if ((w >> kPageShift) >= lim) {
        s.top_status[tid] = (stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 2u;
        s.top_node[tid] = w >> kPageShift;
      } else {
        s.top_status[tid] = PV_ST_OK;
        s.top_node[tid] = w >> kPageShift;
      }
    }
  }
  __syncthreads();
  // 4 nodes x 4 KiB, 16 B per thread per step.
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (s.top_status[t] != PV_ST_OK) continue;
    const uint4* src = reinterpret_cast<const uint4*>(image + base + (s.top_node[t] << kPageShift));
    uint4* dst = reinterpret_cast<uint4*>(mid + t * 512);
    for (uint32_t i = tid; i < 256; i += kTpb) dst[i] = __ldg(src + i);
  }
  __syncthreads();
}

// Upper two levels from shared memory.  Returns PV_ST_OK with *leaf_node set
// (already bounds-checked), or a final status with *value.
__device__ __forceinline__ uint32_t walk_upper(const StageSmem& s, const uint64_t* mid, uint64_t va,
                                               uint32_t stage2, uint64_t* leaf_node, uint64_t* value) {
  const uint32_t t = top_index(va);
  const uint32_t ts = s.top_status[t];
  if (ts != PV_ST_OK) {
    *value = (PV_ST_KIND(ts) == PV_ST_TRAP || PV_ST_KIND(ts) == PV_ST_TRAP2) ? s.top_node[t] : va;
    return ts;
  }
  const uint32_t m = mid_index(va);
  const uint64_t w = mid[t * 512 + m];
  if (w & kFlagTrapping) {
    *value = s.top_node[t];
    return (stage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | 2u | (m << 16);
  }
  if (!(w & kFlagPresent)) {
    *value = va;
    return (stage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | 2u;
  }
  const uint64_t node = w >> kPageShift;
  if (node >= s.lim) {
    *value = va;
    return (stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 3u;
  }
  *leaf_node = node;
  return PV_ST_OK;
}

template <bool kTwo, bool kVa32, bool kPfn>
__global__ void __launch_bounds__(kTpb)
translate_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_space* __restrict__ spaces,
                 const pv_seg* __restrict__ segs, uint32_t n_segs, uint64_t n_chunks, const void* __restrict__ vas,
                 uint64_t* __restrict__ out_value, uint32_t* __restrict__ out_status, uint64_t* __restrict__ out_aux) {
  extern __shared__ __align__(16) uint64_t smem_mid[];  // [kTwo ? 2 : 1][4][512]
  __shared__ StageSmem st1, st2;
  uint64_t* mid1 = smem_mid;
  uint64_t* mid2 = smem_mid + 4 * 512;

  const uint64_t c_begin = (n_chunks * blockIdx.x) / gridDim.x;
  const uint64_t c_end = (n_chunks * (blockIdx.x + 1)) / gridDim.x;
  // Every thread tracks the segment and the staged space in registers; the
  // values are CTA-uniform, so the staging branch is uniform too.
  pv_seg seg;
  seg.begin = seg.end = seg.chunk0 = 0;
  uint64_t seg_chunks = 0;
  uint32_t staged_space = 0xFFFFFFFFu;
  bool two = false;

  for (uint64_t c = c_begin; c < c_end; ++c) {
    if (c < seg.chunk0 || c >= seg.chunk0 + seg_chunks) {
      uint32_t lo = 0, hi = n_segs;
      while (hi - lo > 1) {
        const uint32_t m = (lo + hi) >> 1;
        if (segs[m].chunk0 <= c) lo = m; else hi = m;
      }
      seg = segs[lo];
      seg_chunks = (seg.end - seg.begin + kChunk - 1) / kChunk;
    }
    if (seg.space != staged_space) {
      const pv_space sp = spaces[seg.space];
      staged_space = seg.space;
      two = kTwo && sp.mode == PV_TWO_STAGE;
      __syncthreads();  // everyone is done with the previous staging
      stage_space(image, image_bytes, sp.s1_base, sp.s1_root_pfn, 0, st1, mid1);
      if (two) stage_space(image, image_bytes, 0, sp.s2_root_pfn, 1, st2, mid2);
    }
    const uint64_t lane0 = seg.begin + (c - seg.chunk0) * kChunk;

    uint64_t va[kVpt], node[kVpt], val[kVpt], aux[kVpt];
    uint32_t status[kVpt];
    bool live[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
      const uint64_t i = lane0 + (uint64_t)j * kTpb + threadIdx.x;
      live[j] = i < seg.end;
      va[j] = live[j] ? ld_stream_va(vas, i, kVa32) : 0;
      aux[j] = 0;
    }
    // Stage 1: upper levels from smem.
#pragma unroll
    for (int j = 0; j < kVpt; ++j) status[j] = walk_upper(st1, mid1, va[j], 0, &node[j], &val[j]);
    // Stage 1 leaf: one independent global load per lane.
    uint64_t w[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j)
      w[j] = (live[j] && status[j] == PV_ST_OK) ? ld_word(image, st1.base, node[j], leaf_index(va[j])) : 0;
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
      if (status[j] != PV_ST_OK) continue;
      const uint32_t li = leaf_index(va[j]);
      if (w[j] & kFlagTrapping) {
        status[j] = PV_ST_TRAP | 3u | (li << 16);
        val[j] = node[j];
      } else if (!(w[j] & kFlagPresent)) {
        status[j] = PV_ST_FAULT | 3u;
        val[j] = va[j];
      } else {
        val[j] = w[j] >> kPageShift;  // leaf target pfn
      }
    }
    if (kTwo && two) {
      uint64_t gpa[kVpt];
#pragma unroll
      for (int j = 0; j < kVpt; ++j) {
        gpa[j] = (val[j] << kPageShift) | (va[j] & kPageMask);
        if (status[j] == PV_ST_OK) status[j] = walk_upper(st2, mid2, gpa[j], 1, &node[j], &val[j]) | 0x80000000u;
      }
#pragma unroll
      for (int j = 0; j < kVpt; ++j)
        w[j] = (live[j] && status[j] == 0x80000000u) ? ld_word(image, 0, node[j], leaf_index(gpa[j])) : 0;
#pragma unroll
      for (int j = 0; j < kVpt; ++j) {
        if (!(status[j] & 0x80000000u)) continue;
        status[j] &= 0x7FFFFFFFu;
        if (status[j] != PV_ST_OK) {
          if (PV_ST_KIND(status[j]) == PV_ST_TRAP2) aux[j] = gpa[j];
          continue;
        }
        const uint32_t li = leaf_index(gpa[j]);
        if (w[j] & kFlagTrapping) {
          status[j] = PV_ST_TRAP2 | 3u | (li << 16);
          val[j] = node[j];
          aux[j] = gpa[j];
        } else if (!(w[j] & kFlagPresent)) {
          status[j] = PV_ST_FAULT2 | 3u;
          val[j] = gpa[j];
        } else {
          val[j] = w[j] >> kPageShift;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
      if (!live[j]) continue;
      const uint64_t i = lane0 + (uint64_t)j * kTpb + threadIdx.x;
      uint64_t v = val[j];
      if (!kPfn && status[j] == PV_ST_OK) v = (v << kPageShift) | (va[j] & kPageMask);
      __stcs(reinterpret_cast<unsigned long long*>(out_value) + i, (unsigned long long)v);
      __stcs(out_status + i, status[j]);
      if (out_aux != nullptr && PV_ST_KIND(status[j]) == PV_ST_TRAP2) out_aux[i] = aux[j];
    }
  }
}

template <bool kTwo, bool kVa32, bool kPfn>
static cudaError_t launch_t(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                            uint32_t n_segs, uint64_t n_chunks, const void* vas, uint64_t* out_value,
                            uint32_t* out_status, uint64_t* out_aux, cudaStream_t stream) {
  const size_t smem = (kTwo ? 2 : 1) * 4 * 512 * sizeof(uint64_t);
  auto k = translate_kernel<kTwo, kVa32, kPfn>;
  uint64_t grid = resident_grid((const void*)k, kTpb, smem);
  if (grid > n_chunks) grid = n_chunks;
  if (grid == 0) return cudaSuccess;
  k<<<(unsigned)grid, kTpb, smem, stream>>>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, out_value,
                                            out_status, out_aux);
  return cudaGetLastError();
}

cudaError_t launch_translate(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                             uint32_t n_segs, uint64_t n_chunks, const void* vas, uint32_t flags, bool two_stage,
                             uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux, cudaStream_t stream) {
  const bool va32 = flags & PV_VA32, pfn = flags & PV_OUT_PFN;
#define PV_DISPATCH(T, V, P)                                                                                    \
  if (two_stage == T && va32 == V && pfn == P)                                                                  \
    return launch_t<T, V, P>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, out_value, out_status, \
                             out_aux, stream);
  PV_DISPATCH(false, false, false)
  PV_DISPATCH(false, false, true)
  PV_DISPATCH(false, true, false)
  PV_DISPATCH(false, true, true)
  PV_DISPATCH(true, false, false)
  PV_DISPATCH(true, false, true)
  PV_DISPATCH(true, true, false)
  PV_DISPATCH(true, true, true)
#undef PV_DISPATCH
  return cudaErrorInvalidValue;
}

uint64_t translate_chunk() { return kChunk; }

}  // namespace pv
