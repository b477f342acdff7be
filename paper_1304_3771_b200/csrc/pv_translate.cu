// pv_translate.cu — K1: batched gva -> (gpa ->) hpa translation.
//
// Restates, for a whole batch of lanes at once, the reference's per-address
// walk (memvirt.py:244-259), walk_guest (memvirt.py:262-267), the uncached
// ProcessTranslator resolve (memvirt.py:596-601) and resolve_hybrid
// (memvirt.py:677-682).
//
// B200 design.  CTAs take 2048-lane chunks in grid-stride order, so at any
// moment the whole GPU walks one narrow band of the lane array -- one or two
// address spaces -- and the random leaf gathers hit a few MiB of leaf index
// that stays L2-resident (contiguous per-CTA ranges kept every space's index,
// 65 MB at C5, live at once and re-fetched ~10 % of the gathers from HBM).
// A pre-pass (stage_table_kernel, one CTA per segment) resolves the two
// upper levels of each walk stage into 4-byte codes, one per mid-level entry
// of every present top entry (4 x 512 codes = 8 KiB per stage); a CTA
// entering a segment copies that table into shared memory with 512 16-byte
// loads instead of re-walking the upper levels:
//     bits 0-1  kind: 0 not present (fault at level 2), 1 present,
//               2 trapping (trap at level 2), 3 the walk already stopped at
//               level 1 / 2 (status precomputed per top entry)
//     bit  2    the leaf node lies past the image (struct.error at level 3)
//     bit  3    the leaf node is in the leaf index (pv.h pv_index)
//     bits 4-31 leaf-index slot (bit 3 set) or leaf-node pfn
// so resolving the two upper levels of a lane is ONE 4-byte shared-memory
// read, and every stage costs exactly one dependent global load: a 4-byte
// leaf-index code (L2-resident: half the bytes of the reference's 8-byte
// PTEs) or, for leaf nodes outside the index, the raw leaf PTE.  Each thread walks 8 lanes at once with predicated (branch-free) code
// (8 independent leaf loads in flight) and prefetches the next chunk's VAs
// before gathering the current chunk's leaves; VAs stream in with
// L1::no_allocate loads and results stream out with evict-first stores.
#include <cstdlib>
#include <type_traits>

#include "pv_common.cuh"

namespace pv {

#ifndef PV_TR_WARP_BALLOT
#define PV_TR_WARP_BALLOT 1  // warp-uniform fast-path decision: C5 -2 %, C4 -6 % walk time (profiles/r02_smem_lookup_ab.md)
#endif
#ifndef PV_TR_DEDUP
#define PV_TR_DEDUP 0  // A/B option: explicit warp dedup of leaf-code gathers (profiles/r02_smem_lookup_ab.md)
#endif
constexpr int kTpb = 256;
constexpr int kVpt = 8;
constexpr uint64_t kChunk = (uint64_t)kTpb * kVpt;  // lanes per chunk
constexpr uint32_t kCodeStop = 3u;
constexpr uint32_t kCodeOor = 4u;      // leaf node past the image
constexpr uint32_t kCodeIndexed = 8u;  // payload is a leaf-index slot, not a pfn
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

struct Stage {
  uint64_t base;          // window base (bytes)
  uint64_t lim;           // node limit of the window (pages)
  uint64_t top_node[4];   // root (level-1 traps) / mid node pfn (level-2 traps)
  uint32_t top_status[4]; // status when the walk stops at level 1 or 2 (code kind 3)
};

__device__ __forceinline__ uint64_t ld_stream_va(const void* vas, uint64_t i, bool va32, uint64_t pol) {
  if (va32) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(v)
        : "l"((const uint32_t*)vas + i), "l"(pol));
    return v;
  }
  unsigned long long v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
      : "=l"(v)
      : "l"((const uint64_t*)vas + i), "l"(pol));
  return v;
}

// Stage the upper two levels of one walk stage (all threads; ends with a
// barrier): the Stage record and the 512 codes of each top entry t_sel ..
// t_sel + t_cnt - 1, written to codes[t * 512 ...].  Leaf pfns take 28 bits of a
// code (pfn << 4), so images must be below 2^40 bytes (pv_translate checks).
__device__ void stage_codes(const uint8_t* __restrict__ image, uint64_t image_bytes, uint64_t base, uint64_t root,
                            uint32_t stage2, Stage& s, uint32_t* codes /*[4*512]*/,
                            const uint32_t* __restrict__ slot_of, uint32_t t_sel, uint32_t t_cnt) {
  const uint32_t tid = threadIdx.x;
  const uint64_t lim = node_limit(image_bytes, base);
  if (tid < 4) {
    uint32_t st;
    uint64_t node = 0;
    if (root >= lim) {
      st = (stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 1u;
    } else {
      const uint64_t w = ld_word(image, base, root, tid);
      if (w & kFlagTrapping) {
        st = (stage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | 1u | (tid << 16);
        node = root;
      } else if (!(w & kFlagPresent)) {
        st = (stage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | 1u;
      } else {
        node = w >> kPageShift;
        st = node >= lim ? ((stage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 2u) : PV_ST_OK;
      }
    }
    s.top_status[tid] = st;
    s.top_node[tid] = node;
    if (tid == 0) {
      s.base = base;
      s.lim = lim;
    }
  }
  __syncthreads();
  for (uint32_t i = t_sel * 512 + tid; i < (t_sel + t_cnt) * 512; i += blockDim.x) {
    const uint32_t t = i >> 9;
    uint32_t code = kCodeStop;
    if (s.top_status[t] == PV_ST_OK) {
      const uint64_t w = ld_word(image, base, s.top_node[t], i & 511);
      const uint64_t leaf = w >> kPageShift;
      if (w & kFlagTrapping) {
        code = 2u;
      } else if (!(w & kFlagPresent)) {
        code = 0u;
      } else if (leaf >= lim) {
        code = 1u | kCodeOor;
      } else {
        const uint32_t slot = slot_of != nullptr ? slot_of[(base >> kPageShift) + leaf] : kNoSlot;
        code = slot != kNoSlot ? (1u | kCodeIndexed | (slot << 4)) : (1u | ((uint32_t)leaf << 4));
      }
    }
    codes[i] = code;
  }
  __syncthreads();
}

// Per-segment stage tables, computed once per launch: for segment i,
// codes[(2 i + k) * 2048 ...] and stages[2 i + k] of walk stage k (k = 1 only
// for two-stage spaces).
constexpr uint32_t kStageCodes = 4 * 512;

__global__ void __launch_bounds__(512)
stage_table_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_space* __restrict__ spaces,
                   const pv_seg* __restrict__ segs, bool kTwoAllowed, const uint32_t* __restrict__ slot_of,
                   uint32_t* __restrict__ codes_out, Stage* __restrict__ stages_out) {
  // grid (n_segs, 4 top entries, 2 stages): 512 codes per CTA, one per thread
  __shared__ __align__(16) uint32_t codes[kStageCodes];
  __shared__ Stage st;
  const uint32_t i = blockIdx.x, t = blockIdx.y, k = blockIdx.z;
  const pv_space sp = spaces[segs[i].space];
  const bool two = kTwoAllowed && sp.mode == PV_TWO_STAGE;
  if (k == 1 && !two) return;
  if (k == 0) stage_codes(image, image_bytes, sp.s1_base, sp.s1_root_pfn, 0, st, codes, slot_of, t, 1);
  else stage_codes(image, image_bytes, 0, sp.s2_root_pfn, 1, st, codes, slot_of, t, 1);
  uint4* dst = reinterpret_cast<uint4*>(codes_out + (2ull * i + k) * kStageCodes + t * 512);
  for (uint32_t j = threadIdx.x; j < 512 / 4; j += blockDim.x) dst[j] = reinterpret_cast<const uint4*>(codes + t * 512)[j];
  if (threadIdx.x == 0 && t == 0) stages_out[2 * i + k] = st;
}

// Copy a segment's stage table into shared memory (all threads; CTA-uniform
// call site; the caller brackets it with barriers).
__device__ __forceinline__ void load_stage(const uint32_t* __restrict__ g_codes, const Stage* __restrict__ g_stages,
                                           uint64_t t, uint32_t* codes, Stage& st) {
  const uint4* src = reinterpret_cast<const uint4*>(g_codes + t * kStageCodes);
  for (uint32_t j = threadIdx.x; j < kStageCodes / 4; j += blockDim.x) reinterpret_cast<uint4*>(codes)[j] = src[j];
  if (threadIdx.x == 0) st = g_stages[t];
}

// Upper two levels of one stage for one lane from the code table.  `x` is
// the address walked (va, or gpa in the TDP stage).  Returns PV_ST_OK when
// the leaf PTE must be read (leaf node in *code_out >> 3), else the status.
template <bool kStage2>
__device__ __forceinline__ uint32_t upper(const Stage& s, const uint32_t* codes, uint64_t x, uint32_t* code_out) {
  const uint32_t t = top_index(x), m = mid_index(x);
  const uint32_t code = codes[(t << 9) | m];
  *code_out = code;
  const uint32_t kind = code & 3u;
  const uint32_t st_present = (code & kCodeOor) ? ((kStage2 ? PV_ST_NODE_OOR2 : PV_ST_NODE_OOR) | 3u) : PV_ST_OK;
  const uint32_t st_np = (kStage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | 2u;
  const uint32_t st_trap = (kStage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | 2u | (m << 16);
  return kind == 1u ? st_present : kind == 0u ? st_np : kind == 2u ? st_trap : s.top_status[t];
}

template <bool kStage2>
__device__ __forceinline__ uint32_t leaf_status(uint64_t w, uint32_t st, uint64_t x) {
  if (st != PV_ST_OK) return st;
  if (w & kFlagTrapping) return (kStage2 ? PV_ST_TRAP2 : PV_ST_TRAP) | 3u | (leaf_index(x) << 16);
  if (!(w & kFlagPresent)) return (kStage2 ? PV_ST_FAULT2 : PV_ST_FAULT) | 3u;
  return PV_ST_OK;
}

// Window-relative pfn of the leaf node a staged code points at.
__device__ __forceinline__ uint64_t leaf_node_pfn(const Stage& s, uint32_t code,
                                                  const uint64_t* __restrict__ slot_page) {
  return (code & kCodeIndexed) ? slot_page[code >> 4] - (s.base >> kPageShift) : (uint64_t)(code >> 4);
}

// Node pfn a trap reports: level 3 -> the leaf node, level 1/2 -> top_node.
__device__ __forceinline__ uint64_t trap_node(const Stage& s, uint32_t st, uint32_t code, uint64_t x,
                                              const uint64_t* __restrict__ slot_page) {
  return PV_ST_LEVEL(st) == 3u ? leaf_node_pfn(s, code, slot_page) : s.top_node[top_index(x)];
}

__device__ __forceinline__ uint64_t raw_leaf(const uint8_t* image, const Stage& s, uint64_t node, uint64_t x,
                                             uint64_t pol) {
  return ld_u64_hint(reinterpret_cast<const unsigned long long*>(image + s.base + (node << kPageShift)) +
                         leaf_index(x),
                     pol);
}

// Leaf PTE word of a lane whose upper levels resolved: from the leaf index
// (decoded back into an equivalent word) or the raw table.
__device__ __forceinline__ uint64_t leaf_word(const uint8_t* image, const Stage& s, uint32_t code, uint64_t x,
                                              const uint32_t* __restrict__ leaf_codes,
                                              const uint64_t* __restrict__ slot_page, uint64_t pol) {
  if (code & kCodeIndexed) {
    uint32_t lc;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(lc)
        : "l"(leaf_codes + ((uint64_t)(code >> 4) << 9) + leaf_index(x)), "l"(pol));
    const uint32_t k = lc & 3u;
    if (k == 1u) return ((uint64_t)(lc >> 2) << kPageShift) | kFlagPresent;
    if (k == 0u) return 0;
    if (k == 2u) return kFlagTrapping;
    return raw_leaf(image, s, leaf_node_pfn(s, code, slot_page), x, pol);  // escape
  }
  return raw_leaf(image, s, code >> 4, x, pol);
}

template <bool kTwo, bool kVa32, bool kPfn, int TPB = kTpb, int MINB = (kTwo ? 3 : 4)>
__global__ void __launch_bounds__(TPB, MINB)
translate_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_space* __restrict__ spaces,
                 const pv_seg* __restrict__ segs, uint32_t n_segs, uint64_t n_chunks, const void* __restrict__ vas,
                 const uint32_t* __restrict__ g_codes, const Stage* __restrict__ g_stages,
                 const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ leaf_codes,
                 const uint64_t* __restrict__ slot_page,
                 uint64_t* __restrict__ out_value, uint32_t* __restrict__ out_status, uint64_t* __restrict__ out_aux,
                 uint32_t mode, ExcSink sink) {
  constexpr int VPT = (int)(kChunk / TPB);
  __shared__ __align__(16) uint32_t codes1[4 * 512];
  __shared__ __align__(16) uint32_t codes2[kTwo ? 4 * 512 : 1];
  __shared__ Stage st1, st2;

  // Segment and staged segment live in registers; they are CTA-uniform, so
  // every branch on them is uniform.
  pv_seg seg;
  seg.begin = seg.end = seg.chunk0 = 0;
  seg.space = 0xFFFFFFFFu;
  uint64_t seg_chunks = 0;
  uint32_t seg_idx = 0xFFFFFFFFu, staged_seg = 0xFFFFFFFFu;
  bool two = false;
  const uint64_t pol_stream = policy_evict_first(), pol_table = policy_evict_last();

  auto find_seg = [&](uint64_t c) {
    if (c < seg.chunk0 || c >= seg.chunk0 + seg_chunks) {
      uint32_t lo = 0, hi = n_segs;
      while (hi - lo > 1) {
        const uint32_t m = (lo + hi) >> 1;
        if (segs[m].chunk0 <= c) lo = m; else hi = m;
      }
      seg = segs[lo];
      seg_idx = lo;
      seg_chunks = (seg.end - seg.begin + kChunk - 1) / kChunk;
    }
  };
  using VaT = typename std::conditional<kVa32, uint32_t, uint64_t>::type;
  auto load_vas = [&](uint64_t c, VaT (&va)[VPT]) {
    const uint64_t lane0 = seg.begin + (c - seg.chunk0) * kChunk;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const uint64_t i = lane0 + (uint64_t)j * TPB + threadIdx.x;
      va[j] = i < seg.end ? (VaT)ld_stream_va(vas, i, kVa32, pol_stream) : 0;
    }
  };

  VaT va[VPT], nva[VPT];
  bool have_next = false;
  // Large batches (stage tables precomputed, g_codes != nullptr): grid-stride
  // chunk order.  Small batches (a few chunks per CTA): contiguous chunk
  // ranges and in-kernel staging -- no pre-pass launch, no scratch.
  const bool pre = g_codes != nullptr;
  const uint64_t c_first = pre ? blockIdx.x : (n_chunks * blockIdx.x) / gridDim.x;
  const uint64_t c_last = pre ? n_chunks : (n_chunks * (blockIdx.x + 1)) / gridDim.x;
  const uint64_t c_step = pre ? gridDim.x : 1;
  for (uint64_t c = c_first; c < c_last; c += c_step) {
    find_seg(c);
    if (seg_idx != staged_seg) {
      staged_seg = seg_idx;
      const pv_space sp = spaces[seg.space];
      two = kTwo && sp.mode == PV_TWO_STAGE;
      __syncthreads();  // everyone is done with the previous table
      if (pre) {
        load_stage(g_codes, g_stages, 2ull * seg_idx, codes1, st1);
        if (two) load_stage(g_codes, g_stages, 2ull * seg_idx + 1, codes2, st2);
      } else {
        stage_codes(image, image_bytes, sp.s1_base, sp.s1_root_pfn, 0, st1, codes1, slot_of, 0, 4);
        if (two) stage_codes(image, image_bytes, 0, sp.s2_root_pfn, 1, st2, codes2, slot_of, 0, 4);
      }
      __syncthreads();
    }
    if (have_next) {
#pragma unroll
      for (int j = 0; j < VPT; ++j) va[j] = nva[j];
    } else {
      load_vas(c, va);
    }
    const uint64_t lane0 = seg.begin + (c - seg.chunk0) * kChunk;
    const uint64_t seg_end = seg.end;
    // Prefetch the next chunk's VAs when it is in the same segment.
    const uint64_t cn = c + c_step;
#ifndef PV_TR_PREFETCH
#define PV_TR_PREFETCH 0  // next-chunk VA prefetch: measured slower once chunks went grid-stride (162 vs 158 G/s)
#endif
    have_next = PV_TR_PREFETCH && cn < c_last && cn < seg.chunk0 + seg_chunks;
    if (have_next) load_vas(cn, nva);

    // Fast path (one-stage walks): when every lane of this thread resolves
    // its upper levels to an indexed, in-image leaf node and its leaf code is
    // PRESENT, the translation is (code >> 2) << 12 | offset and the status
    // OK -- no status logic, no branches per lane.  Anything else (faults,
    // traps, escapes, unindexed nodes, two-stage spaces) takes the general
    // path below, which re-reads the same (now L1-resident) codes.
    // (Two-stage walks take the same path twice: the stage-1 leaf code gives
    // the gpa, whose TDP upper levels come from codes2 and leaf code from the
    // index -- a TDP fault or trap anywhere sends the thread to the general
    // path.)
    if (leaf_codes != nullptr) {
      uint32_t fc[VPT];
      bool simple = true;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
#ifdef PV_PROBE_FAKE_CODES
        // probe build only (wrong results): the code of a hashed (top, mid) computed in registers
        // instead of the shared-memory table read -- the same spread of leaf-index gathers without the
        // SMEM lookup and its bank conflicts (scripts/ab_smem_lookup.sh)
        if (j == 0) {
          fc[0] = codes1[(top_index(va[0]) << 9) | mid_index(va[0])];  // one real lookup per thread and chunk
        } else {
          const uint32_t h = (((top_index(va[j]) << 9) | mid_index(va[j])) * 2654435761u) >> 21;
          fc[j] = (fc[0] & 0xFu) | (((fc[0] >> 4) + h % 1300u) << 4);
        }
#else
        fc[j] = codes1[(top_index(va[j]) << 9) | mid_index(va[j])];
#endif
        const bool valid = lane0 + (uint64_t)j * TPB + threadIdx.x < seg_end;
        simple &= !valid || (fc[j] & 0xFu) == (1u | kCodeIndexed);
      }
#if PV_TR_WARP_BALLOT
      // warp-ballot fault handling (north star): the warp takes the fast path only when every lane of it
      // can, so the branch is warp-uniform -- measured faster than a per-thread decision on both the
      // fault-free C5 walk and the fault-heavy C4 one
      simple = __all_sync(0xFFFFFFFFu, simple);
#endif
      if (simple) {
        uint32_t lc[VPT];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          const bool valid = lane0 + (uint64_t)j * TPB + threadIdx.x < seg_end;
          lc[j] = 1u;
#if PV_TR_DEDUP
          // A/B option (north star: "a coalesced TLB-style dedup of repeated pages"): lanes of the warp
          // that want the same leaf code elect one loader and receive the code by shuffle; default: the
          // LSU merges same-sector requests of one warp instruction by itself
          {
            const uint32_t* a = leaf_codes + ((uint64_t)(fc[j] >> 4) << 9) + leaf_index(va[j]);
            const unsigned peers = __match_any_sync(0xFFFFFFFFu, valid ? (unsigned long long)a : ~0ull);
            const int leader = __ffs(peers) - 1;
            uint32_t v = 1u;
            if (valid && (int)(threadIdx.x & 31u) == leader)
              asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol_table));
            v = __shfl_sync(0xFFFFFFFFu, v, leader);
            if (valid) lc[j] = v;
          }
#else
          if (valid)
            asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
                : "=r"(lc[j])
                : "l"(leaf_codes + ((uint64_t)(fc[j] >> 4) << 9) + leaf_index(va[j])), "l"(pol_table));
#endif
        }
        bool present = true;
#pragma unroll
        for (int j = 0; j < VPT; ++j) present &= (lc[j] & 3u) == 1u;
#if PV_TR_WARP_BALLOT
        present = __all_sync(0xFFFFFFFFu, present);
#endif
        if (present && kTwo && two) {
          // stage 2 over the gpa: lc[] becomes the TDP leaf code (same shape)
          uint64_t gpa[VPT];
          bool simple2 = true;
#pragma unroll
          for (int j = 0; j < VPT; ++j) {
            gpa[j] = ((uint64_t)(lc[j] >> 2) << kPageShift) | (va[j] & kPageMask);
            fc[j] = codes2[(top_index(gpa[j]) << 9) | mid_index(gpa[j])];
            const bool valid = lane0 + (uint64_t)j * TPB + threadIdx.x < seg_end;
            simple2 &= !valid || (fc[j] & 0xFu) == (1u | kCodeIndexed);
          }
#if PV_TR_WARP_BALLOT
          simple2 = __all_sync(0xFFFFFFFFu, simple2);
#endif
          present = simple2;
          if (simple2) {
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
              const bool valid = lane0 + (uint64_t)j * TPB + threadIdx.x < seg_end;
              lc[j] = 1u;
              if (valid)
                asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
                    : "=r"(lc[j])
                    : "l"(leaf_codes + ((uint64_t)(fc[j] >> 4) << 9) + leaf_index(gpa[j])), "l"(pol_table));
            }
#pragma unroll
            for (int j = 0; j < VPT; ++j) present &= (lc[j] & 3u) == 1u;
#if PV_TR_WARP_BALLOT
            present = __all_sync(0xFFFFFFFFu, present);
#endif
          }
        }
        if (present) {
#pragma unroll
          for (int j = 0; j < VPT; ++j) {
            const uint64_t i = lane0 + (uint64_t)j * TPB + threadIdx.x;
            if (i >= seg_end) continue;
            const uint64_t pfn = lc[j] >> 2;
            if (mode == kOutWord) {
              st_u32_stream(reinterpret_cast<uint32_t*>(out_value) + i, (uint32_t)pfn, pol_stream);
              continue;
            }
            st_u64_stream(out_value + i, kPfn ? pfn : ((pfn << kPageShift) | (va[j] & kPageMask)), pol_stream);
            if (mode == kOutSplit) st_u32_stream(out_status + i, PV_ST_OK, pol_stream);
          }
          continue;
        }
      }
    }
    uint32_t st[VPT], code[VPT];
    uint64_t w[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) st[j] = upper<false>(st1, codes1, va[j], &code[j]);
#pragma unroll
    for (int j = 0; j < VPT; ++j) w[j] = st[j] == PV_ST_OK ? leaf_word(image, st1, code[j], va[j], leaf_codes, slot_page, pol_table) : 0;
    uint64_t val[VPT], aux[VPT];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      st[j] = leaf_status<false>(w[j], st[j], va[j]);
      const uint32_t k = PV_ST_KIND(st[j]);
      val[j] = k == PV_ST_OK ? (w[j] >> kPageShift) : k == PV_ST_TRAP ? trap_node(st1, st[j], code[j], va[j], slot_page) : va[j];
      aux[j] = 0;
    }
    if (kTwo && two) {
      uint64_t gpa[VPT];
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        gpa[j] = (val[j] << kPageShift) | (va[j] & kPageMask);
        if (st[j] == PV_ST_OK) st[j] = upper<true>(st2, codes2, gpa[j], &code[j]) | 0x80000000u;
      }
#pragma unroll
      for (int j = 0; j < VPT; ++j) w[j] = st[j] == 0x80000000u ? leaf_word(image, st2, code[j], gpa[j], leaf_codes, slot_page, pol_table) : 0;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        if (!(st[j] & 0x80000000u)) continue;
        st[j] = leaf_status<true>(w[j], st[j] & 0x7FFFFFFFu, gpa[j]);
        const uint32_t k = PV_ST_KIND(st[j]);
        if (k == PV_ST_OK) {
          val[j] = w[j] >> kPageShift;
        } else if (k == PV_ST_TRAP2) {
          val[j] = trap_node(st2, st[j], code[j], gpa[j], slot_page);
          aux[j] = gpa[j];
        } else {
          val[j] = gpa[j];
        }
      }
    }
    if (mode == kOutWord) {
      // 4-byte words: the thread's lanes that need an exception record are
      // counted first, so the warp reserves all its records of this chunk
      // with ONE atomic (a per-lane or per-j atomic would put an L2 round
      // trip per lane group on the critical path of a fault-heavy walk)
      uint32_t word[VPT];
      unsigned bal[VPT];
      const unsigned mask = __activemask();
      uint32_t total = 0;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const bool valid = lane0 + (uint64_t)j * TPB + threadIdx.x < seg_end;
        bool need = false;
        word[j] = word_code(st[j], val[j], (uint64_t)va[j], kTwo && PV_ST_KIND(st[j]) == PV_ST_TRAP2, &need);
        bal[j] = __ballot_sync(mask, valid && need);
        total += __popc(bal[j]);
      }
      if (total) {
        const int me = (int)(threadIdx.x & 31u), leader = __ffs(mask) - 1;
        const uint32_t stripe = (blockIdx.x * (TPB >> 5) + (threadIdx.x >> 5)) % PV_EXC_STRIPES;
        unsigned long long base = 0;
        if (me == leader) base = atomicAdd(sink.count + stripe, (unsigned long long)total);
        base = __shfl_sync(mask, base, leader);
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          if (bal[j] >> me & 1u) {
            const unsigned long long k = base + __popc(bal[j] & ((1u << me) - 1u));
            if (k < sink.per) {
              pv_exc r;
              r.lane = sink.lane_base + lane0 + (uint64_t)j * TPB + threadIdx.x;
              r.value = val[j];
              r.aux = kTwo ? aux[j] : 0;
              r.status = st[j];
              r.reserved = 0;
              sink.rec[stripe * sink.per + k] = r;
            }
          }
          base += __popc(bal[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const uint64_t i = lane0 + (uint64_t)j * TPB + threadIdx.x;
        if (i < seg_end) st_u32_stream(reinterpret_cast<uint32_t*>(out_value) + i, word[j], pol_stream);
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const uint64_t i = lane0 + (uint64_t)j * TPB + threadIdx.x;
      if (i >= seg_end) continue;
      uint64_t v = val[j];
      if (!kPfn && st[j] == PV_ST_OK) v = (v << kPageShift) | (va[j] & kPageMask);
      if (mode == kOutPacked) {
        bool spill;
        st_u64_stream(out_value + i, pack_lane(st[j], v, &spill), pol_stream);
        if (spill && out_aux != nullptr) out_aux[i] = v;
      } else {
        st_u64_stream(out_value + i, v, pol_stream);
        st_u32_stream(out_status + i, st[j], pol_stream);
      }
      if (kTwo && out_aux != nullptr && PV_ST_KIND(st[j]) == PV_ST_TRAP2) out_aux[i] = aux[j];
    }
  }
}

// Generic form for batches that contain extension-geometry spaces
// (PV_ONE_STAGE_4L), 8 lanes per thread, each lane walked through
// translate_global.  PV_GEN_LEVELSYNC=1 (A/B option) walks a 4-level chunk's
// 8 lanes level by level instead (walk4_global's checks in the same order, the
// 8 loads of a level in flight together): C3 -5 %, C1 4-level +19 % walk time
// (profiles/r02_generic_ab.md), so lane-by-lane stays the default.
#ifndef PV_GEN_TPB
#define PV_GEN_TPB 256
#endif
#ifndef PV_GEN_LEVELSYNC
#define PV_GEN_LEVELSYNC 0
#endif
#ifndef PV_GEN_MINB
#define PV_GEN_MINB 0  // A/B option: minimum resident CTAs per SM for the register budget
#endif
constexpr int kGenTpb = PV_GEN_TPB;
constexpr int kGenVpt = (int)(kChunk / kGenTpb);

template <bool kVa32, bool kPfn>
__device__ __forceinline__ void emit_lane(uint64_t i, uint32_t st, uint64_t v, uint64_t a, uint64_t va,
                                          uint64_t* __restrict__ out_value, uint32_t* __restrict__ out_status,
                                          uint64_t* __restrict__ out_aux, uint32_t mode, const ExcSink& sink) {
  if (mode == kOutWord) {
    reinterpret_cast<uint32_t*>(out_value)[i] = word_lane(st, v, va, PV_ST_KIND(st) == PV_ST_TRAP2 ? a : 0, i, sink);
    return;
  }
  if (!kPfn && st == PV_ST_OK) v = (v << kPageShift) | (va & kPageMask);
  if (mode == kOutPacked) {
    bool spill;
    out_value[i] = pack_lane(st, v, &spill);
    if (spill && out_aux != nullptr) out_aux[i] = v;
  } else {
    out_value[i] = v;
    out_status[i] = st;
  }
  if (out_aux != nullptr && PV_ST_KIND(st) == PV_ST_TRAP2) out_aux[i] = a;
}

template <bool kVa32, bool kPfn>
#if PV_GEN_MINB > 1
__global__ void __launch_bounds__(kGenTpb, PV_GEN_MINB)
#else
__global__ void __launch_bounds__(kGenTpb)
#endif
translate_generic_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes,
                         const pv_space* __restrict__ spaces, const pv_seg* __restrict__ segs, uint32_t n_segs,
                         uint64_t n_chunks, const void* __restrict__ vas, uint64_t* __restrict__ out_value,
                         uint32_t* __restrict__ out_status, uint64_t* __restrict__ out_aux, uint32_t mode,
                         ExcSink sink) {
  for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    uint32_t lo = 0, hi = n_segs;
    while (hi - lo > 1) {
      const uint32_t m = (lo + hi) >> 1;
      if (segs[m].chunk0 <= c) lo = m; else hi = m;
    }
    const pv_seg seg = segs[lo];
    const pv_space sp = spaces[seg.space];
    const uint64_t lane0 = seg.begin + (c - seg.chunk0) * kChunk;
    if (PV_GEN_LEVELSYNC && sp.mode == PV_ONE_STAGE_4L) {
      const uint64_t base = sp.s1_base, lim = node_limit(image_bytes, base);
      uint64_t va[kGenVpt], node[kGenVpt];
      uint32_t st[kGenVpt];
      uint32_t live = 0;
#pragma unroll
      for (int j = 0; j < kGenVpt; ++j) {
        const uint64_t i = lane0 + (uint64_t)j * kGenTpb + threadIdx.x;
        va[j] = 0;
        node[j] = sp.s1_root_pfn;
        st[j] = PV_ST_OK;
        if (i < seg.end) {
          va[j] = kVa32 ? (uint64_t)((const uint32_t*)vas)[i] : ((const uint64_t*)vas)[i];
          live |= 1u << j;
        }
      }
#pragma unroll
      for (uint32_t l = 0; l < 4; ++l) {
        uint64_t w[kGenVpt];
#pragma unroll
        for (int j = 0; j < kGenVpt; ++j) {  // this level's loads, all in flight
          w[j] = 0;
          if (!((live >> j) & 1u)) continue;
          if (node[j] >= lim) {
            st[j] = PV_ST_NODE_OOR | (l + 1);
            node[j] = va[j];
            live &= ~(1u << j);
          } else {
            w[j] = ld_word(image, base, node[j], (uint32_t)(va[j] >> (39 - 9 * l)) & 511u);
          }
        }
#pragma unroll
        for (int j = 0; j < kGenVpt; ++j) {
          if (!((live >> j) & 1u)) continue;
          if (w[j] & kFlagTrapping) {  // value: the node holding the trapping entry
            st[j] = PV_ST_TRAP | (l + 1) | ((((uint32_t)(va[j] >> (39 - 9 * l))) & 511u) << 16);
            live &= ~(1u << j);
          } else if (!(w[j] & kFlagPresent)) {
            st[j] = PV_ST_FAULT | (l + 1);
            node[j] = va[j];
            live &= ~(1u << j);
          } else if (l == 2 && (w[j] & PV_FLAG_PS)) {  // 2 MiB leaf: its 4 KiB frame of va
            node[j] = (w[j] >> kPageShift) + ((va[j] >> kPageShift) & 511u);
            live &= ~(1u << j);
          } else {
            node[j] = w[j] >> kPageShift;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kGenVpt; ++j) {
        const uint64_t i = lane0 + (uint64_t)j * kGenTpb + threadIdx.x;
        if (i < seg.end) emit_lane<kVa32, kPfn>(i, st[j], node[j], 0, va[j], out_value, out_status, out_aux, mode,
                                                sink);
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < kGenVpt; ++j) {
      const uint64_t i = lane0 + (uint64_t)j * kGenTpb + threadIdx.x;
      if (i >= seg.end) continue;
      const uint64_t va = kVa32 ? (uint64_t)((const uint32_t*)vas)[i] : ((const uint64_t*)vas)[i];
      uint64_t v = 0, a = 0;
      const uint32_t st = translate_global(image, image_bytes, sp, va, &v, &a);
      if (mode == kOutWord) {
        reinterpret_cast<uint32_t*>(out_value)[i] =
            word_lane(st, v, va, PV_ST_KIND(st) == PV_ST_TRAP2 ? a : 0, i, sink);
        continue;
      }
      if (!kPfn && st == PV_ST_OK) v = (v << kPageShift) | (va & kPageMask);
      if (mode == kOutPacked) {
        bool spill;
        out_value[i] = pack_lane(st, v, &spill);
        if (spill && out_aux != nullptr) out_aux[i] = v;
      } else {
        out_value[i] = v;
        out_status[i] = st;
      }
      if (out_aux != nullptr && PV_ST_KIND(st) == PV_ST_TRAP2) out_aux[i] = a;
    }
  }
}

template <bool kVa32, bool kPfn>
static cudaError_t launch_generic(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces,
                                  const pv_seg* segs, uint32_t n_segs, uint64_t n_chunks, const void* vas,
                                  uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux, uint32_t mode,
                                  const ExcSink& sink, cudaStream_t stream) {
  auto k = translate_generic_kernel<kVa32, kPfn>;
  uint64_t grid = resident_grid((const void*)k, kGenTpb, 0);
  if (grid > n_chunks) grid = n_chunks;
  if (grid == 0) return cudaSuccess;
  k<<<(unsigned)grid, kGenTpb, 0, stream>>>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, out_value,
                                         out_status, out_aux, mode, sink);
  return cudaGetLastError();
}

template <bool kTwo, bool kVa32, bool kPfn>
static cudaError_t launch_t(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                            uint32_t n_segs, uint64_t n_chunks, const void* vas, const pv_index* idx,
                            uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux, bool concurrent,
                            uint32_t mode, const ExcSink& sink, cudaStream_t stream) {
  // one-stage walks: 512-thread CTAs x 4 lanes (2 CTAs/SM) measured best on
  // C5 (scripts/ab_walk.sh: 0.848 ms vs 0.858 at 1024 x 2 and 0.923 at 128 x 16)
#ifndef PV_TR_MINB
#define PV_TR_MINB 2
#endif
#ifndef PV_TR2_TPB
#define PV_TR2_TPB 512  // two-stage walks: 512 x 4 lanes, 2 CTAs/SM (C1 TDP 37.5 vs 28.2 G/s at 256 x 8)
#endif
#ifndef PV_TR1_TPB
#define PV_TR1_TPB 512
#endif
#ifndef PV_CONC_TPB
#define PV_CONC_TPB 256  // PV_CONCURRENT one-stage walks: 256 x 8 lanes, <= 64 registers
#endif
  auto k = kTwo ? translate_kernel<kTwo, kVa32, kPfn, PV_TR2_TPB, (PV_TR2_TPB == 256 ? 3 : 1024 / PV_TR2_TPB)>
                : translate_kernel<kTwo, kVa32, kPfn, PV_TR1_TPB, PV_TR_MINB * 512 / PV_TR1_TPB>;
  int tpb = kTwo ? PV_TR2_TPB : PV_TR1_TPB;
  if (concurrent && !kTwo) {
    // PV_CONCURRENT: a small CTA (256 threads x <= 64 registers, 8 KiB of
    // SMEM) per SM, so it fits beside the copy exec's CTA (256 threads x 166
    // registers, 192 KiB of SMEM) on every SM: the two kernels co-reside
    k = translate_kernel<kTwo, kVa32, kPfn, PV_CONC_TPB, 1024 / PV_CONC_TPB>;
    tpb = PV_CONC_TPB;
  }
  uint64_t grid = resident_grid((const void*)k, tpb, 0);
  if (concurrent) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms > 0 && grid > (uint64_t)sms) grid = (uint64_t)sms;
  }
  if (grid > n_chunks) grid = n_chunks;
  if (grid == 0) return cudaSuccess;
  const uint32_t* slot_of = idx != nullptr ? idx->slot_of : nullptr;
  const uint32_t* leaf_codes = idx != nullptr ? idx->leaf_codes : nullptr;
  const uint64_t* slot_page = idx != nullptr ? idx->slot_page : nullptr;
  if (n_chunks < 8 * grid) {
    // few chunks per CTA: each CTA stages its (usually one) segment itself
    k<<<(unsigned)grid, tpb, 0, stream>>>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, nullptr, nullptr,
                                          slot_of, leaf_codes, slot_page, out_value, out_status, out_aux, mode, sink);
    return cudaGetLastError();
  }
  // per-segment stage tables: stream-ordered scratch (per call, so calls on
  // distinct streams never share it)
  const size_t codes_bytes = 2ull * n_segs * kStageCodes * sizeof(uint32_t);
  void* tab = nullptr;
  cudaError_t e = stream_scratch(&tab, codes_bytes + 2ull * n_segs * sizeof(Stage), stream);
  if (e != cudaSuccess) return e;
  uint32_t* g_codes = static_cast<uint32_t*>(tab);
  Stage* g_stages = reinterpret_cast<Stage*>(static_cast<uint8_t*>(tab) + codes_bytes);
  stage_table_kernel<<<dim3(n_segs, 4, kTwo ? 2 : 1), 512, 0, stream>>>(image, image_bytes, spaces, segs, kTwo,
                                                                         slot_of, g_codes, g_stages);
  k<<<(unsigned)grid, tpb, 0, stream>>>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, g_codes, g_stages,
                                        slot_of, leaf_codes, slot_page, out_value, out_status, out_aux, mode, sink);
  e = cudaGetLastError();
  cudaFreeAsync(tab, stream);
  return e;
}

cudaError_t launch_translate(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                             uint32_t n_segs, uint64_t n_chunks, const void* vas, uint32_t flags, bool two_stage,
                             const pv_index* idx, uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux,
                             const ExcSink* words, cudaStream_t stream) {
  const bool va32 = flags & PV_VA32, pfn = flags & PV_OUT_PFN;
  // words != nullptr: pv_translate_words (out_value holds u32 lane words)
  const uint32_t mode = words != nullptr ? kOutWord : (flags & PV_OUT_PACKED) ? kOutPacked : kOutSplit;
  const ExcSink sink = words != nullptr ? *words : ExcSink{nullptr, 0, nullptr, 0};
  if (flags & PV_HAS_4L) {
    if (va32) return pfn ? launch_generic<true, true>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas,
                                                      out_value, out_status, out_aux, mode, sink, stream)
                         : launch_generic<true, false>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas,
                                                       out_value, out_status, out_aux, mode, sink, stream);
    return pfn ? launch_generic<false, true>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, out_value,
                                             out_status, out_aux, mode, sink, stream)
               : launch_generic<false, false>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, out_value,
                                              out_status, out_aux, mode, sink, stream);
  }
  if (image_bytes >= (1ull << 40)) return cudaErrorInvalidValue;  // leaf pfns / slots must fit 28-bit codes
#define PV_DISPATCH(T, V, P)                                                                                    \
  if (two_stage == T && va32 == V && pfn == P)                                                                  \
    return launch_t<T, V, P>(image, image_bytes, spaces, segs, n_segs, n_chunks, vas, idx, out_value, \
                             out_status, out_aux, flags & PV_CONCURRENT, mode, sink, stream);
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
