// pv_ordered.cu — ordered execution of a to_guest copy batch whose chunks
// overlap on destination pages (last-writer-wins in op order, exactly as the
// reference's sequential copy_user_buffer calls, memvirt.py:604-628).
//
// B200 design: every live chunk (page k of op o with k < first_bad[o]) is
// keyed by its destination hpa page; a stable radix sort (CUB, 32-bit keys,
// only the bits the image needs) groups chunks by page while preserving the
// global chunk order (= op order, then page order); one CTA then owns one
// destination page: it stages the page in shared memory, applies every chunk
// of that page in order (all source bytes really move; the successive
// overwrites land in SMEM instead of HBM, the way a write-back cache would
// absorb them), and writes the page back once.  Chunk payloads stream in
// through a cp.async ring ahead of the ordered applies, so the per-chunk
// barrier only orders the shared-memory writes.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "pv_common.cuh"

namespace pv {

constexpr int kOrdTpb = 256;
constexpr uint32_t kDeadKey = 0xFFFFFFFFu;

// keys[p] = destination page of live page p, else kDeadKey; vals[p] = p;
// page_op[p] = the op page p belongs to.
__global__ void ordered_keys_kernel(const uint64_t* __restrict__ page_off, uint64_t n_ops, uint64_t n_pages,
                                    const uint64_t* __restrict__ page_hpa, const unsigned long long* __restrict__ first_bad,
                                    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                    uint32_t* __restrict__ page_op) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pages; p += stride) {
    const uint64_t op = upper_search(page_off, 0, n_ops, p);
    const uint64_t k = p - page_off[op];
    keys[p] = k < first_bad[op] ? (uint32_t)(page_hpa[p] >> kPageShift) : kDeadKey;
    vals[p] = (uint32_t)p;
    page_op[p] = (uint32_t)op;
  }
}

constexpr int kRing = 8;                       // chunks in flight per CTA
constexpr uint32_t kSlotPad = 16;              // headroom so word reads at offset -3.. stay in the slot
constexpr uint32_t kSlot = kSlotPad + kPageSize + 32;  // aligned superset of a <= 4 KiB chunk
constexpr uint32_t kBatch = kOrdTpb;           // chunk descriptors resolved per round

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One CTA per destination page: stage the page in SMEM, then apply its
// chunks in order.  Chunk descriptors are resolved 256 at a time (one per
// thread, independent loads); chunk payloads stream in with 16-byte
// cp.async (LDGSTS) into an 8-deep SMEM ring, so global-memory latency
// overlaps the ordered SMEM applies.  The buffer must be readable up to the
// next 16-byte boundary after each chunk (true of any 512-byte-granular
// device allocation).
__global__ void __launch_bounds__(kOrdTpb)
ordered_apply_kernel(uint8_t* __restrict__ image, const pv_op* __restrict__ ops, const uint64_t* __restrict__ page_off,
                     const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ page_op,
                     const uint32_t* __restrict__ sorted_pages, const uint32_t* __restrict__ seg_key,
                     const uint32_t* __restrict__ seg_len, const uint32_t* __restrict__ seg_start,
                     const uint32_t* __restrict__ n_segs_dev, const uint8_t* __restrict__ buf,
                     uint8_t* __restrict__ dirty) {
  __shared__ __align__(16) uint8_t page[kPageSize];
  __shared__ __align__(16) uint8_t ring[kRing][kSlot];
  __shared__ uint64_t d_src[kBatch];   // 16-byte aligned source start
  __shared__ uint32_t d_meta[kBatch];  // shift (4 bits) | off (12 bits) << 4 | len (13 bits) << 16
  const uint32_t n_segs = *n_segs_dev;
  const uint32_t t = threadIdx.x;
  for (uint32_t s = blockIdx.x; s < n_segs; s += gridDim.x) {
    const uint32_t key = seg_key[s];
    if (key == kDeadKey) continue;
    const uint64_t dst = (uint64_t)key << kPageShift;
    reinterpret_cast<uint4*>(page)[t] = reinterpret_cast<const uint4*>(image + dst)[t];
    const uint32_t b = seg_start[s], n = seg_len[s];
    for (uint32_t base = 0; base < n; base += kBatch) {
      const uint32_t m = min(kBatch, n - base);
      __syncthreads();  // previous round's descriptors / ring slots are free
      if (t < m) {
        const uint32_t p = sorted_pages[b + base + t];
        const uint32_t op = page_op[p];
        const pv_op o = ops[op];
        const uint64_t k = p - page_off[op];
        const uint64_t cur = op_page_va(o.gva, k);
        const uint64_t done = cur - o.gva;
        const uint32_t len = (uint32_t)min(o.len - done, kPageSize - (cur & kPageMask));
        const uint32_t off = (uint32_t)(page_hpa[p] & kPageMask);
        const uint64_t src = reinterpret_cast<uint64_t>(buf + o.buf_off + done);
        d_src[t] = src & ~15ull;
        d_meta[t] = (uint32_t)(src & 15) | (off << 4) | (len << 16);
      }
      __syncthreads();
      auto issue = [&](uint32_t c) {
        const uint32_t meta = d_meta[c];
        const uint32_t shift = meta & 15, len = meta >> 16;
        const uint32_t blocks = (shift + len + 15) >> 4;  // <= 257
        const uint8_t* src = reinterpret_cast<const uint8_t*>(d_src[c]);
        uint8_t* slot = ring[c % kRing] + kSlotPad;
        for (uint32_t i = t; i < blocks; i += kOrdTpb) cp_async16(slot + 16 * i, src + 16 * i);
      };
#pragma unroll
      for (int c = 0; c < kRing - 1; ++c) {
        if ((uint32_t)c < m) issue(c);
        cp_async_commit();
      }
      for (uint32_t c = 0; c < m; ++c) {
        if (c + kRing - 1 < m) issue(c + kRing - 1);
        cp_async_commit();
        cp_async_wait<kRing - 1>();  // chunk c's group (this thread's part) landed
        __syncthreads();             // ... and every thread's part
        const uint32_t meta = d_meta[c];
        const uint32_t shift = meta & 15, off = (meta >> 4) & 0xFFF, len = meta >> 16;
        // destination-aligned 4-byte words; each word is owned by one thread
        // (no read-modify-write races), the source is realigned with a funnel
        // shift from two aligned slot words; conflict-free SMEM banks.
        const uint32_t* slot32 = reinterpret_cast<const uint32_t*>(ring[c % kRing]);
        uint32_t* page32 = reinterpret_cast<uint32_t*>(page);
        const uint32_t w_first = off >> 2, w_last = (off + len - 1) >> 2;
        for (uint32_t w = w_first + t; w <= w_last; w += kOrdTpb) {
          const int32_t s0 = (int32_t)(kSlotPad + shift + 4 * w) - (int32_t)off;  // slot byte of word byte 0
          const uint32_t lo = slot32[s0 >> 2], hi = slot32[(s0 >> 2) + 1];
          const uint32_t v = __funnelshift_r(lo, hi, (s0 & 3) * 8);
          const uint32_t b0 = 4 * w < off ? off - 4 * w : 0;                      // first byte of the word in chunk
          const uint32_t b1 = 4 * w + 4 > off + len ? off + len - 4 * w : 4;      // one past the last
          if (b0 == 0 && b1 == 4) {
            page32[w] = v;
          } else {
            const uint32_t m = (b1 == 4 ? 0xFFFFFFFFu : ((1u << (8 * b1)) - 1u)) & ~((1u << (8 * b0)) - 1u);
            page32[w] = (page32[w] & ~m) | (v & m);
          }
        }
        __syncthreads();  // chunk c applied before c+1; its slot may be refilled
      }
      cp_async_wait<0>();
    }
    __syncthreads();
    reinterpret_cast<uint4*>(image + dst)[t] = reinterpret_cast<const uint4*>(page)[t];
    if (dirty != nullptr && t == 0) dirty[key] = 1;
    __syncthreads();
  }
}

// Per-op results (the exec kernel's result rule, for ops run in order).
__global__ void ordered_results_kernel(const pv_op* __restrict__ ops, uint64_t n_ops,
                                       const uint64_t* __restrict__ page_off, const uint64_t* __restrict__ page_hpa,
                                       const uint32_t* __restrict__ page_status, const uint64_t* __restrict__ page_aux,
                                       const unsigned long long* __restrict__ first_bad,
                                       pv_op_result* __restrict__ results) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += stride) {
    const pv_op o = ops[i];
    const uint64_t bad = first_bad[i];
    pv_op_result r;
    if (bad == kNone || page_off[i + 1] == page_off[i]) {
      r.copied = o.len;
      r.value = r.aux = 0;
      r.status = PV_ST_OK;
      r.fail_page = 0;
    } else {
      const uint64_t p = page_off[i] + bad;
      r.copied = op_page_va(o.gva, bad) - o.gva;
      r.value = page_hpa[p];
      r.aux = page_aux != nullptr ? page_aux[p] : 0;
      r.status = page_status[p];
      r.fail_page = (uint32_t)bad;
    }
    results[i] = r;
  }
}

struct OrderedScratch {
  uint32_t *keys_in, *vals_in, *keys_out, *vals_out, *seg_key, *seg_len, *seg_start, *page_op, *n_segs;
  void* cub_tmp;
  size_t cub_bytes;
};

static size_t cub_need(uint64_t n, int end_bit) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, end_bit);
  cub::DeviceRunLengthEncode::Encode(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                     (uint32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return std::max(a, std::max(b, c));
}

static int bits_for(uint64_t) {
  return 32;  // dead keys (0xFFFFFFFF) must sort last: sort on every bit
}

size_t ordered_scratch_bytes(uint64_t n_pages, uint64_t image_pages) {
  const uint64_t arr = ((n_pages + 1) * 4 + 255) / 256 * 256;
  return 8 * arr + 256 + cub_need(n_pages, bits_for(image_pages)) + 256;
}

static OrderedScratch carve(void* base, uint64_t n, size_t cub_bytes) {
  uint8_t* p = static_cast<uint8_t*>(base);
  OrderedScratch s;
  uint32_t** arrs[] = {&s.keys_in, &s.vals_in, &s.keys_out, &s.vals_out, &s.seg_key, &s.seg_len, &s.seg_start,
                       &s.page_op};
  for (auto a : arrs) {
    *a = reinterpret_cast<uint32_t*>(p);
    p += ((n + 1) * 4 + 255) / 256 * 256;
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
                                const uint8_t* buf, pv_op_result* results, uint8_t* dirty, void* scratch,
                                uint64_t scratch_bytes, cudaStream_t stream) {
  {
    uint64_t g = (n_ops + 255) / 256;
    if (g > 4096) g = 4096;
    if (g) ordered_results_kernel<<<(unsigned)g, 256, 0, stream>>>(
        ops, n_ops, page_off, page_hpa, page_status, page_aux,
        reinterpret_cast<const unsigned long long*>(op_first_bad), results);
  }
  if (n_pages == 0) return cudaGetLastError();
  if (n_pages >= 0xFFFFFFFFull || (image_bytes >> kPageShift) >= 0xFFFFFFFFull) return cudaErrorInvalidValue;
  const int end_bit = bits_for(image_bytes >> kPageShift);
  const size_t need = cub_need(n_pages, end_bit);
  if (scratch_bytes < ordered_scratch_bytes(n_pages, image_bytes >> kPageShift)) return cudaErrorInvalidValue;
  OrderedScratch s = carve(scratch, n_pages, need);
  uint64_t grid = (n_pages + 255) / 256;
  if (grid > 4096) grid = 4096;
  ordered_keys_kernel<<<(unsigned)grid, 256, 0, stream>>>(page_off, n_ops, n_pages, page_hpa,
                                                          reinterpret_cast<const unsigned long long*>(op_first_bad),
                                                          s.keys_in, s.vals_in, s.page_op);
  size_t tb = s.cub_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(s.cub_tmp, tb, s.keys_in, s.keys_out, s.vals_in, s.vals_out,
                                                  (int)n_pages, 0, end_bit, stream);
  if (e != cudaSuccess) return e;
  tb = s.cub_bytes;
  e = cub::DeviceRunLengthEncode::Encode(s.cub_tmp, tb, s.keys_out, s.seg_key, s.seg_len, s.n_segs, (int)n_pages,
                                         stream);
  if (e != cudaSuccess) return e;
  tb = s.cub_bytes;
  e = cub::DeviceScan::ExclusiveSum(s.cub_tmp, tb, s.seg_len, s.seg_start, (int)n_pages, stream);
  if (e != cudaSuccess) return e;
  uint64_t g2 = resident_grid((const void*)ordered_apply_kernel, kOrdTpb, 0);
  if (g2 > n_pages) g2 = n_pages;
  ordered_apply_kernel<<<(unsigned)g2, kOrdTpb, 0, stream>>>(image, ops, page_off, page_hpa, s.page_op, s.vals_out,
                                                             s.seg_key, s.seg_len, s.seg_start, s.n_segs, buf, dirty);
  return cudaGetLastError();
}

}  // namespace pv
