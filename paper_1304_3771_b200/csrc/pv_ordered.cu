// pv_ordered.cu — ordered execution of a to_guest copy batch whose chunks
// overlap on destination pages (last-writer-wins in op order, exactly as the
// reference's sequential copy_user_buffer calls, memvirt.py:604-628).
//
// B200 design: every live chunk (page k of op o with k < first_bad[o]) is
// keyed by its destination hpa page; a stable radix sort (CUB, only the bits
// the image needs) groups chunks by page while preserving the global chunk
// order (= op order, then page order), carrying the 16-byte chunk
// descriptors along as values.  A producer/consumer WARP PAIR then owns one
// destination page: the consumer stages the page in shared memory; the
// producer streams the page's chunk payloads in with TMA bulk copies
// (cp.async.bulk issued by one lane, completion counted on a per-slot
// mbarrier) into a circular byte ring, up to kK chunks ahead, LAST CHUNK
// FIRST; the consumer lets each byte take the value of the first arrival that
// covers it (a per-block coverage map skips bytes a later writer already
// set), which is exactly the state the in-order copies leave.  Chunks that
// later writers overwrite completely never move: both warps walk the page's
// descriptors last-first and only the chunks that still reach an uncovered
// byte are streamed (NeedIter, metadata only); the page is never read --
// bytes no chunk covers are merged from the image at write-back, once.  The
// pipeline is warp-private: no CTA-wide barriers on the per-chunk path.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "pv_common.cuh"

#ifndef PV_ORDERED_BACKOFF_NS
#define PV_ORDERED_BACKOFF_NS 64
#endif

namespace pv {

// A chunk descriptor: the 16-byte aligned source start, and
// meta = shift (4 bits) | dst offset in page (12 bits) << 4 | len (13 bits) << 16.
struct __align__(16) ChunkDesc {
  uint64_t src;
  uint32_t meta;
  uint32_t pad;
};

__device__ __forceinline__ void write_result(const pv_op& o, uint64_t p0, uint64_t p1, uint64_t bad,
                                             const uint64_t* __restrict__ page_hpa,
                                             const uint32_t* __restrict__ page_status,
                                             const uint64_t* __restrict__ page_aux, pv_op_result* __restrict__ out) {
  pv_op_result r;
  if (bad == kNone || p1 == p0) {
    r.copied = o.len;
    r.value = r.aux = 0;
    r.status = PV_ST_OK;
    r.fail_page = 0;
  } else {
    const uint64_t p = p0 + bad;
    r.copied = op_page_va(o.gva, bad) - o.gva;
    r.value = page_hpa[p];
    r.aux = page_aux != nullptr ? page_aux[p] : 0;
    r.status = page_status[p];
    r.fail_page = (uint32_t)bad;
  }
  *out = r;
}

// One thread per op: the op's result (copied prefix / first failure), and
// per page keys[p] = destination page of live page p (else the dead key,
// which sorts last), desc[p] = p's chunk descriptor and iota[p] = p (the
// sort's values; with PV_ORD_INDEX=0 the descriptors are the values).
__global__ void ordered_keys_kernel(const pv_op* __restrict__ ops, uint64_t n_ops, const uint64_t* __restrict__ page_off,
                                    const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ page_status,
                                    const uint64_t* __restrict__ page_aux,
                                    const unsigned long long* __restrict__ first_bad, const uint8_t* __restrict__ buf,
                                    uint64_t buf_bytes, uint32_t dead_key, uint32_t* __restrict__ keys,
                                    ChunkDesc* __restrict__ desc, uint32_t* __restrict__ iota,
                                    pv_op_result* __restrict__ results) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += stride) {
    const pv_op o = ops[i];
    const uint64_t p0 = page_off[i], p1 = page_off[i + 1];
    const uint64_t bad = first_bad[i];
    write_result(o, p0, p1, bad, page_hpa, page_status, page_aux, results + i);
    for (uint64_t p = p0; p < p1; ++p) {
      const uint64_t k = p - p0;
      const uint64_t hpa = page_hpa[p];
      const bool live = k < bad;
      keys[p] = live ? (uint32_t)(hpa >> kPageShift) : dead_key;
      const uint64_t cur = op_page_va(o.gva, k);
      const uint64_t done = cur - o.gva;
      const uint32_t len =
          live ? buf_clamp(o.buf_off + done, (uint32_t)min(o.len - done, kPageSize - (cur & kPageMask)), buf_bytes) : 0;
      const uint64_t src = reinterpret_cast<uint64_t>(buf + o.buf_off + done);
      ChunkDesc d;
      d.src = src & ~15ull;
      d.meta = (uint32_t)(src & 15) | ((uint32_t)(hpa & kPageMask) << 4) | (len << 16);
      d.pad = 0;
      desc[p] = d;
      if (iota != nullptr) iota[p] = (uint32_t)p;
    }
  }
}


// ---- warp-per-page apply ------------------------------------------------------------

#ifndef PV_AP_PAGES
#define PV_AP_PAGES 4
#endif
#ifndef PV_AP_RING
#define PV_AP_RING 8192
#endif
#ifndef PV_AP_K
#define PV_AP_K 16
#endif
#ifndef PV_AP_WINDOW
#define PV_AP_WINDOW 6144  // measured: 3.66 ms vs 6.56 ms at the full ring (C2), see DESIGN.md
#endif
// The sort carries u32 chunk indices, not the 16-byte descriptors: the
// apply gathers the descriptors it scans by index.  C2: sort 0.533 -> 0.317
// ms, apply 0.144 -> 0.244 ms, apply phase 0.939 -> 0.836 ms
// (profiles/r02_ord_index_ab.md; PV_ORD_INDEX=0 sorts the descriptors).
#ifndef PV_ORD_INDEX
#define PV_ORD_INDEX 1
#endif
constexpr int kApPages = PV_AP_PAGES;                    // page slots (producer + consumer warp each) per CTA
constexpr int kK = PV_AP_K;                         // chunks in flight per page slot (mbarrier pairs)
constexpr uint32_t kRB = PV_AP_RING;                 // circular byte ring per page slot (power of two)
constexpr uint32_t kRB16 = kRB / 16;
constexpr uint32_t kWin = PV_AP_WINDOW;  // ring bytes a slot keeps in flight (<= kRB)
static_assert(kRB >= kPageSize + 32 && kWin <= kRB, "a chunk span (<= 4112 bytes) must fit the ring");

struct __align__(16) PageSmem {
  uint8_t page[kPageSize];
  uint8_t ring[kRB];
  uint16_t cov[kPageSize / 16];  // bytes of each 16-byte block already final (bit x = byte x)
  uint64_t full[kK];
  uint64_t empty[kK];
  uint32_t meta[kK];
  uint32_t vstart[kK];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// Producer-side wait for a ring slot: back off between polls so the spinning
// warp does not take issue slots from the consumer it is waiting for.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  while (!ok) {
    __nanosleep(PV_ORDERED_BACKOFF_NS);
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, uint64_t src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// Destination block j of a chunk from the ring, realigned: D is the
// (warp-uniform) word part of the realignment, so the word selection is
// static -- two 16-byte SMEM loads and four funnel shifts.
template <int D>
__device__ __forceinline__ uint4 realign(const uint4* ring16, int32_t j, int32_t dq, uint32_t sb) {
  const uint4 U = ring16[(uint32_t)(j + dq) & (kRB16 - 1)];
  const uint4 V = ring16[(uint32_t)(j + dq + 1) & (kRB16 - 1)];
  uint32_t y0, y1, y2, y3, y4;
  if constexpr (D == 0) { y0 = U.x; y1 = U.y; y2 = U.z; y3 = U.w; y4 = V.x; }
  if constexpr (D == 1) { y0 = U.y; y1 = U.z; y2 = U.w; y3 = V.x; y4 = V.y; }
  if constexpr (D == 2) { y0 = U.z; y1 = U.w; y2 = V.x; y3 = V.y; y4 = V.z; }
  if constexpr (D == 3) { y0 = U.w; y1 = V.x; y2 = V.y; y3 = V.z; y4 = V.w; }
  uint4 out;
  out.x = __funnelshift_r(y0, y1, sb);
  out.y = __funnelshift_r(y1, y2, sb);
  out.z = __funnelshift_r(y2, y3, sb);
  out.w = __funnelshift_r(y3, y4, sb);
  return out;
}

// Byte mask of the set bits of a nibble (bit b -> byte b), no table.
__device__ __forceinline__ uint32_t nibble_bytes(uint32_t x) { return ((x * 0x00204081u) & 0x01010101u) * 0xFFu; }

// Apply one chunk LAST-FIRST: the page's chunks arrive in reverse program
// order, so a byte takes the value of the first chunk (in arrival order) that
// covers it and later arrivals only fill bytes no later writer has covered --
// the same final bytes as applying every chunk in order.  cov[] tracks the
// final bytes per 16-byte block; blocks already final are skipped.  Returns
// the number of blocks this lane made fully final.
template <int D>
__device__ __forceinline__ uint32_t apply_chunk_rev(PageSmem& W, uint32_t lane, int32_t off, int32_t len, int32_t dq,
                                                    uint32_t sb) {
  const uint4* ring16 = reinterpret_cast<const uint4*>(W.ring);
  uint4* page16 = reinterpret_cast<uint4*>(W.page);
  const int32_t end = off + len;
  const int32_t jh = off >> 4, jt = (end - 1) >> 4;
  uint32_t made_full = 0;
  for (int32_t j = jh + (int32_t)lane; j <= jt; j += 32) {
    const int32_t lo = max(off - 16 * j, 0), hi = min(end - 16 * j, 16);
    const uint32_t rmask = (0xFFFFu >> (16 - hi)) & (0xFFFFu << lo);
    const uint32_t c = W.cov[j];
    const uint32_t need = rmask & ~c;
    if (need == 0) continue;
    const uint4 v = realign<D>(ring16, j, dq, sb);
    if (need == 0xFFFFu) {
      page16[j] = v;
    } else {
      const uint32_t m0 = nibble_bytes(need & 15), m1 = nibble_bytes((need >> 4) & 15),
                     m2 = nibble_bytes((need >> 8) & 15), m3 = nibble_bytes(need >> 12);
      const uint4 old = page16[j];
      page16[j] = make_uint4((old.x & ~m0) | (v.x & m0), (old.y & ~m1) | (v.y & m1), (old.z & ~m2) | (v.z & m2),
                             (old.w & ~m3) | (v.w & m3));
    }
    const uint32_t nc = c | rmask;
    W.cov[j] = (uint16_t)nc;
    made_full += nc == 0xFFFFu;
  }
  return made_full;
}
// The chunks of one page that can still change it, last-first.  Walking the
// page's chunk descriptors from the LAST one (program order) backwards, a
// chunk matters only if it covers a byte no later chunk covers; every other
// chunk is overwritten entirely and its payload never has to move.  Coverage
// depends on (offset, len) only -- the metadata -- so the producer and the
// consumer warp of a page slot each run this iterator and see the same
// sequence without talking (their ring accounting, G / vhead, stays in
// step).  Lane l tracks bytes [128 l, 128 l + 128) of the page (c[4]);
// fullreg (warp-uniform) has bit l set once lane l's bytes are all covered,
// which lets a window of 32 candidates be filtered in one step (a chunk whose
// 128-byte regions are all covered is dead) before the exact per-chunk test.
// Pages the batch covers completely stop after a few dozen chunks; pages it
// never covers (e.g. an arena's first byte) still scan every descriptor but
// move only the few chunks that reach their uncovered bytes.
struct NeedIter {
  const ChunkDesc* rd;  // candidate k (0 = last chunk in program order) at rd - k, or at desc[ix[last - k]]
  const ChunkDesc* desc;
  const uint32_t* ix;   // PV_ORD_INDEX: sorted chunk indices (nullptr: rd holds sorted descriptors)
  uint32_t last;
  uint32_t n, k0;       // candidates, current window start
  uint32_t cand;        // window lanes not yet rejected (warp-uniform)
  uint32_t meta_l;      // this lane's window candidate
  uint64_t src_l;
  uint32_t c[4];        // this lane's 128 coverage bits
  uint32_t fullreg;     // bit l: lane l's bytes are all covered (warp-uniform)
};

__device__ __forceinline__ void need_window(NeedIter& it, uint32_t lane) {
  const uint32_t k = it.k0 + lane;
  bool maybe = false;
  it.meta_l = 0;
  it.src_l = 0;
  if (k < it.n) {
    const ChunkDesc d = it.ix != nullptr ? it.desc[it.ix[it.last - k]] : *(it.rd - k);
    it.meta_l = d.meta;
    it.src_l = d.src;
    const uint32_t off = (d.meta >> 4) & 0xFFF, len = d.meta >> 16;
    if (len != 0) {
      const uint32_t r0 = off >> 7, r1 = (off + len - 1) >> 7;
      const uint32_t regions = (r1 == 31 ? 0xFFFFFFFFu : ((2u << r1) - 1u)) & ~((1u << r0) - 1u);
      maybe = (regions & ~it.fullreg) != 0;
    }
  }
  it.cand = __ballot_sync(0xFFFFFFFFu, maybe);
}

__device__ __forceinline__ void need_init(NeedIter& it, const ChunkDesc* __restrict__ desc,
                                          const uint32_t* __restrict__ ix, uint32_t b, uint32_t n, uint32_t lane) {
  it.rd = desc + b + n - 1;
  it.desc = desc;
  it.ix = ix;
  it.last = b + n - 1;
  it.n = n;
  it.k0 = 0;
  it.c[0] = it.c[1] = it.c[2] = it.c[3] = 0u;
  it.fullreg = 0u;
  need_window(it, lane);
}

// Next chunk that matters (its meta, and its source for the producer);
// false when none is left.  Warp-collective.
__device__ __forceinline__ bool need_next(NeedIter& it, uint32_t lane, uint32_t& meta, uint64_t& src) {
  const int32_t mine = 128 * (int32_t)lane;
  while (it.fullreg != 0xFFFFFFFFu) {
    while (it.cand == 0u) {
      it.k0 += 32;
      if (it.k0 >= it.n) return false;
      need_window(it, lane);
    }
    const int j = __ffs(it.cand) - 1;
    it.cand &= it.cand - 1u;
    const uint32_t mj = __shfl_sync(0xFFFFFFFFu, it.meta_l, j);
    const int32_t off = (int32_t)((mj >> 4) & 0xFFF), len = (int32_t)(mj >> 16);
    const int32_t lo = max(off - mine, 0), hi = min(off + len - mine, 128);
    uint32_t m[4], fresh = 0u;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int32_t wl = max(lo - 32 * w, 0), wh = min(hi - 32 * w, 32);
      m[w] = wl < wh ? ((wh == 32 ? 0xFFFFFFFFu : ((1u << wh) - 1u)) & ~((1u << wl) - 1u)) : 0u;
      fresh |= m[w] & ~it.c[w];
    }
    const uint64_t s = ((uint64_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)(it.src_l >> 32), j) << 32) |
                       __shfl_sync(0xFFFFFFFFu, (uint32_t)it.src_l, j);
    if (__any_sync(0xFFFFFFFFu, fresh != 0u)) {
#pragma unroll
      for (int w = 0; w < 4; ++w) it.c[w] |= m[w];
      it.fullreg = __ballot_sync(0xFFFFFFFFu, (it.c[0] & it.c[1] & it.c[2] & it.c[3]) == 0xFFFFFFFFu);
      meta = mj;
      src = s;
      return true;
    }
  }
  return false;
}

// One page slot per producer/consumer warp pair.  The producer warp walks
// the page's chunks that matter (NeedIter) and keeps the ring full (TMA
// bulk copies, completion on full[slot]); the consumer warp applies them in
// the same order and releases each ring slot on empty[slot].  Ring bytes are
// packed back to back in virtual byte order; before reusing bytes the
// producer waits for the release of the newest chunk that still occupies
// them (releases are in order).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void produce(PageSmem& P, const ChunkDesc* __restrict__ desc,
                                        const uint32_t* __restrict__ ix, uint32_t b, uint32_t n,
                                        uint32_t lane, uint64_t pol, uint32_t& G, uint32_t& vhead, uint32_t& hptr,
                                        int64_t& released) {
  NeedIter it;
  need_init(it, desc, ix, b, n, lane);
  uint32_t meta;
  uint64_t src;
  while (need_next(it, lane, meta, src)) {
    const uint32_t span = (((meta & 15) + (meta >> 16) + 15) >> 4) << 4;
    const uint32_t ve = vhead + span;
    // chunk G reuses slot G % kK (last held by chunk G - kK) and the ring
    // bytes of every chunk whose virtual start is below ve - kWin
    if (G >= (uint32_t)kK && hptr < G - kK + 1) hptr = G - kK + 1;
    while (hptr < G && (int32_t)(P.vstart[hptr % kK] - (ve - kWin)) < 0) ++hptr;
    int64_t r = (int64_t)hptr - 1;
    if (G >= (uint32_t)kK && (int64_t)(G - kK) > r) r = G - kK;
    if (r > released) {
      mbar_wait_backoff(&P.empty[r % kK], (uint32_t)(r / kK) & 1);
      released = r;
    }
    const uint32_t slot = G % kK;
    P.vstart[slot] = vhead;  // producer-private history (every lane stores the same value)
    if (lane == 0) {
      P.meta[slot] = meta;
      const uint32_t p = vhead % kRB;
      const uint32_t first = span < kRB - p ? span : kRB - p;  // split at the ring's end
      mbar_expect_tx(&P.full[slot], span);
      if (span != 0) bulk_g2s(P.ring + p, src, first, &P.full[slot], pol);
      if (first < span) bulk_g2s(P.ring, src + first, span - first, &P.full[slot], pol);
    }
    vhead = ve;
    ++G;
  }
}

__global__ void __launch_bounds__(kApPages * 64)
ordered_apply_kernel(uint8_t* __restrict__ image, const ChunkDesc* __restrict__ desc,
                     const uint32_t* __restrict__ ix, const uint32_t* __restrict__ seg_key, const uint32_t* __restrict__ seg_len,
                     const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ n_segs_dev,
                     uint32_t dead_key, uint8_t* __restrict__ dirty) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t pslot = warp >> 1;
  const bool producer = (warp & 1) == 0;
  PageSmem& P = reinterpret_cast<PageSmem*>(smem_raw)[pslot];
  if (producer && lane == 0) {
    for (int k = 0; k < kK; ++k) {
      mbar_init(&P.full[k], 1);
      mbar_init(&P.empty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint32_t n_segs = *n_segs_dev;
  uint32_t G = 0, vhead = 0, hptr = 0;  // chunks so far / virtual ring bytes so far (both roles)
  int64_t released = -1;                 // producer: newest chunk known released
  for (uint32_t s = blockIdx.x * kApPages + pslot; s < n_segs; s += gridDim.x * kApPages) {
    const uint32_t key = seg_key[s];
    if (key == dead_key) continue;
    const uint32_t b = seg_start[s], n = seg_len[s];
    if (producer) {
      produce(P, desc, ix, b, n, lane, pol, G, vhead, hptr, released);
      continue;
    }
    // The page is assembled in SMEM from the chunks that matter only; bytes
    // no chunk covers keep the image's contents, merged in at write-back.
    reinterpret_cast<uint4*>(P.cov)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    NeedIter it;
    need_init(it, desc, ix, b, n, lane);
    uint32_t meta_it;
    uint64_t src_it;
    while (need_next(it, lane, meta_it, src_it)) {
      const uint32_t slot = G % kK;
      mbar_wait(&P.full[slot], (G / kK) & 1);
      const uint32_t meta = P.meta[slot];
      const uint32_t shift = meta & 15, len = meta >> 16;
      const int32_t off = (int32_t)((meta >> 4) & 0xFFF);
      // dest byte 16j + x  <->  ring byte 16j + delta + x
      const int32_t delta = (int32_t)(vhead % kRB + shift) - off;
      const int32_t dq = delta >> 4;
      const uint32_t dr = (uint32_t)delta & 15, sb = (dr & 3) * 8;
      switch (dr >> 2) {
        case 0: apply_chunk_rev<0>(P, lane, off, (int32_t)len, dq, sb); break;
        case 1: apply_chunk_rev<1>(P, lane, off, (int32_t)len, dq, sb); break;
        case 2: apply_chunk_rev<2>(P, lane, off, (int32_t)len, dq, sb); break;
        default: apply_chunk_rev<3>(P, lane, off, (int32_t)len, dq, sb); break;
      }
      vhead += ((shift + len + 15) >> 4) << 4;
      ++G;
      __syncwarp();  // every lane's ring reads and page writes of this chunk are done
      if (lane == 0) mbar_arrive(&P.empty[slot]);
    }
    __syncwarp();
    const uint64_t dst = (uint64_t)key << kPageShift;
    uint4* out = reinterpret_cast<uint4*>(image + dst);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t j = lane + 32 * k;
      const uint32_t c = P.cov[j];
      if (c == 0u) continue;  // no writer: the image keeps these bytes
      const uint4 v = reinterpret_cast<const uint4*>(P.page)[j];
      if (c == 0xFFFFu) {
        out[j] = v;
      } else {
        const uint32_t m0 = nibble_bytes(c & 15), m1 = nibble_bytes((c >> 4) & 15), m2 = nibble_bytes((c >> 8) & 15),
                       m3 = nibble_bytes(c >> 12);
        const uint4 old = out[j];
        out[j] = make_uint4((old.x & ~m0) | (v.x & m0), (old.y & ~m1) | (v.y & m1), (old.z & ~m2) | (v.z & m2),
                            (old.w & ~m3) | (v.w & m3));
      }
    }
    if (dirty != nullptr && lane == 0) dirty[key] = 1;
    __syncwarp();
  }
}

// Per-op results (the exec kernel's result rule, for ops run in order).
// Results only (a batch without pages: nothing to sort or apply).
__global__ void ordered_results_kernel(const pv_op* __restrict__ ops, uint64_t n_ops,
                                       const uint64_t* __restrict__ page_off, const uint64_t* __restrict__ page_hpa,
                                       const uint32_t* __restrict__ page_status, const uint64_t* __restrict__ page_aux,
                                       const unsigned long long* __restrict__ first_bad,
                                       pv_op_result* __restrict__ results) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += stride)
    write_result(ops[i], page_off[i], page_off[i + 1], first_bad[i], page_hpa, page_status, page_aux, results + i);
}

struct OrderedScratch {
  uint32_t *keys_in, *keys_out, *seg_key, *seg_len, *seg_start, *n_segs;
  ChunkDesc *desc, *desc_sorted;
  uint32_t *idx_in, *idx_out;  // PV_ORD_INDEX
  void* cub_tmp;
  size_t cub_bytes;
};

static size_t cub_need(uint64_t n, int end_bit) {
  size_t a = 0, b = 0, c = 0;
  if (PV_ORD_INDEX)
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n, 0, end_bit);
  else
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (ChunkDesc*)nullptr,
                                    (ChunkDesc*)nullptr, (int)n, 0, end_bit);
  cub::DeviceRunLengthEncode::Encode(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                     (uint32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return std::max(a, std::max(b, c));
}

// Keys are destination page numbers < image_pages and the dead key is
// image_pages itself, so sorting the low bits_for(image_pages) bits suffices.
static int bits_for(uint64_t image_pages) {
  int b = 1;
  while (b < 32 && (image_pages >> b) != 0) ++b;
  return b;
}

static uint64_t arr_bytes(uint64_t n, uint64_t elt) { return ((n + 1) * elt + 255) / 256 * 256; }

size_t ordered_scratch_bytes(uint64_t n_pages, uint64_t image_pages) {
  return (PV_ORD_INDEX ? 7 : 5) * arr_bytes(n_pages, 4) + 2 * arr_bytes(n_pages, sizeof(ChunkDesc)) + 256 +
         cub_need(n_pages, bits_for(image_pages)) + 256;
}

static OrderedScratch carve(void* base, uint64_t n, size_t cub_bytes) {
  uint8_t* p = static_cast<uint8_t*>(base);
  OrderedScratch s;
  uint32_t** arrs[] = {&s.keys_in, &s.keys_out, &s.seg_key, &s.seg_len, &s.seg_start};
  for (auto a : arrs) {
    *a = reinterpret_cast<uint32_t*>(p);
    p += arr_bytes(n, 4);
  }
  s.desc = reinterpret_cast<ChunkDesc*>(p);
  p += arr_bytes(n, sizeof(ChunkDesc));
  s.desc_sorted = reinterpret_cast<ChunkDesc*>(p);
  p += arr_bytes(n, sizeof(ChunkDesc));
  s.idx_in = s.idx_out = nullptr;
  if (PV_ORD_INDEX) {
    s.idx_in = reinterpret_cast<uint32_t*>(p);
    p += arr_bytes(n, 4);
    s.idx_out = reinterpret_cast<uint32_t*>(p);
    p += arr_bytes(n, 4);
  }
  s.n_segs = reinterpret_cast<uint32_t*>(p);
  p += 256;
  s.cub_tmp = p;
  s.cub_bytes = cub_bytes;
  return s;
}

cudaError_t launch_copy_ordered(uint8_t* image, uint64_t image_bytes, const pv_op* ops, uint64_t n_ops,
                                const uint64_t* page_off, uint64_t n_pages, const uint64_t* page_hpa,
                                const uint32_t* page_status, const uint64_t* page_aux, const uint64_t* op_first_bad,
                                const uint8_t* buf, uint64_t buf_bytes, pv_op_result* results, uint8_t* dirty,
                                void* scratch, uint64_t scratch_bytes, cudaStream_t stream) {
  if (n_pages == 0) {
    uint64_t g = (n_ops + 255) / 256;
    if (g > 4096) g = 4096;
    if (g) ordered_results_kernel<<<(unsigned)g, 256, 0, stream>>>(
        ops, n_ops, page_off, page_hpa, page_status, page_aux,
        reinterpret_cast<const unsigned long long*>(op_first_bad), results);
    return cudaGetLastError();
  }
  const uint64_t image_pages = image_bytes >> kPageShift;
  if (n_pages >= 0xFFFFFFFFull || image_pages >= 0xFFFFFFFFull) return cudaErrorInvalidValue;
  const uint32_t dead_key = (uint32_t)image_pages;
  const int end_bit = bits_for(image_pages);
  const size_t need = cub_need(n_pages, end_bit);
  if (scratch_bytes < ordered_scratch_bytes(n_pages, image_pages)) return cudaErrorInvalidValue;
  OrderedScratch s = carve(scratch, n_pages, need);
  {
    uint64_t g = (n_ops + 255) / 256;
    if (g > 8192) g = 8192;
    void* tk = timing_begin("ordered_keys", stream);
    ordered_keys_kernel<<<(unsigned)g, 256, 0, stream>>>(ops, n_ops, page_off, page_hpa, page_status, page_aux,
                                                         reinterpret_cast<const unsigned long long*>(op_first_bad),
                                                         buf, buf_bytes, dead_key, s.keys_in, s.desc, s.idx_in,
                                                         results);
    timing_end(tk, stream);
  }
  size_t tb = s.cub_bytes;
  // the 16-byte descriptors ride along as the sort's values (no index gather afterwards)
  void* tks = timing_begin("ordered_sort", stream);
  cudaError_t e = PV_ORD_INDEX
                      ? cub::DeviceRadixSort::SortPairs(s.cub_tmp, tb, s.keys_in, s.keys_out, s.idx_in, s.idx_out,
                                                        (int)n_pages, 0, end_bit, stream)
                      : cub::DeviceRadixSort::SortPairs(s.cub_tmp, tb, s.keys_in, s.keys_out, s.desc, s.desc_sorted,
                                                        (int)n_pages, 0, end_bit, stream);
  timing_end(tks, stream);
  if (e != cudaSuccess) return e;
  tb = s.cub_bytes;
  e = cub::DeviceRunLengthEncode::Encode(s.cub_tmp, tb, s.keys_out, s.seg_key, s.seg_len, s.n_segs, (int)n_pages,
                                         stream);
  if (e != cudaSuccess) return e;
  tb = s.cub_bytes;
  e = cub::DeviceScan::ExclusiveSum(s.cub_tmp, tb, s.seg_len, s.seg_start, (int)n_pages, stream);
  if (e != cudaSuccess) return e;
  constexpr size_t smem = sizeof(PageSmem) * kApPages;
  e = ensure_dynamic_smem((const void*)ordered_apply_kernel, smem);
  if (e != cudaSuccess) return e;
  uint64_t g2 = resident_grid((const void*)ordered_apply_kernel, kApPages * 64, smem);
  const uint64_t want = (n_pages + kApPages - 1) / kApPages;
  if (g2 > want) g2 = want;
  void* tk = timing_begin("ordered_apply", stream);
  ordered_apply_kernel<<<(unsigned)g2, kApPages * 64, smem, stream>>>(image, PV_ORD_INDEX ? s.desc : s.desc_sorted,
                                                                      s.idx_out, s.seg_key, s.seg_len,
                                                                      s.seg_start, s.n_segs, dead_key, dirty);
  timing_end(tk, stream);
  return cudaGetLastError();
}

}  // namespace pv
