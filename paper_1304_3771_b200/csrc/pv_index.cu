// pv_index.cu — leaf index: a derived 4-byte image of the leaf-level
// page-table nodes a batch walks (see pv.h, pv_index).
//
// Why: at the C5 scale (24 processes x 2.6 GiB mapped) the reference's
// 8-byte leaf PTEs occupy 130 MB, more than the 126 MB L2, so random walks
// miss L2 ~70 % of the time and each miss costs a 64-byte DRAM burst for an
// 8-byte word.  Encoded as 4-byte codes the same leaves take 65 MB and stay
// L2-resident under the walker's evict-last policy.
//
// Exactness: a code is a pure function of its PTE word (state = the
// reference's decode_entry precedence, memvirt.py:110-117, pfn = word >> 12);
// PTEs whose pfn does not fit 30 bits encode as "escape" and the walker reads
// the raw word.  The host runtime re-encodes a slot whenever its page is
// written (host writes at push time; device writes through the dirty map).
#include "pv_common.cuh"

namespace pv {

constexpr int kEncTpb = 256;

__device__ __forceinline__ uint32_t encode_leaf(uint64_t w) {
  if (w & kFlagTrapping) return 2u;
  if (!(w & kFlagPresent)) return 0u;
  const uint64_t pfn = w >> kPageShift;
  return pfn < (1ull << 30) ? (1u | ((uint32_t)pfn << 2)) : 3u;
}

// A CTA takes 256 slots at a time: every thread checks one slot (its page
// in the image and, for device-write syncs, dirty), the slots that need it
// are compacted in shared memory, then the CTA encodes them one by one with
// 256 threads x 2 entries (16-byte loads).  A sync where nothing indexed was
// written costs one parallel pass over the dirty bytes.
__global__ void __launch_bounds__(kEncTpb)
encode_kernel(const uint8_t* __restrict__ image, uint64_t image_pages, const uint64_t* __restrict__ slot_page,
              const uint64_t* __restrict__ slots, uint64_t first_slot, uint64_t n, uint32_t* __restrict__ leaf_codes,
              const uint8_t* __restrict__ dirty) {
  __shared__ uint64_t todo[kEncTpb];
  __shared__ uint32_t n_todo;
  for (uint64_t t0 = (uint64_t)blockIdx.x * kEncTpb; t0 < n; t0 += (uint64_t)gridDim.x * kEncTpb) {
    if (threadIdx.x == 0) n_todo = 0;
    __syncthreads();
    const uint64_t i = t0 + threadIdx.x;
    if (i < n) {
      const uint64_t slot = slots != nullptr ? slots[i] : first_slot + i;
      const uint64_t page = slot_page[slot];
      if (page < image_pages && (dirty == nullptr || dirty[page] != 0)) todo[atomicAdd(&n_todo, 1u)] = slot;
    }
    __syncthreads();
    const uint32_t m = n_todo;
    for (uint32_t k = 0; k < m; ++k) {
      const uint64_t slot = todo[k];
      const uint64_t page = slot_page[slot];
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(image + (page << kPageShift)) + threadIdx.x);
      const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
      uint2 out;
      out.x = encode_leaf(w0);
      out.y = encode_leaf(w1);
      reinterpret_cast<uint2*>(leaf_codes + (slot << 9))[threadIdx.x] = out;
    }
    __syncthreads();  // todo / n_todo reused by the next tile
  }
}

cudaError_t launch_index_encode(const uint8_t* image, uint64_t image_bytes, const uint64_t* slot_page,
                                const uint64_t* slots, uint64_t first_slot, uint64_t n, uint32_t* leaf_codes,
                                const uint8_t* dirty, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n + kEncTpb - 1) / kEncTpb;
  const uint64_t cap = resident_grid((const void*)encode_kernel, kEncTpb, 0);
  if (grid > cap) grid = cap;
  encode_kernel<<<(unsigned)grid, kEncTpb, 0, stream>>>(image, image_bytes >> kPageShift, slot_page, slots,
                                                        first_slot, n, leaf_codes, dirty);
  return cudaGetLastError();
}

}  // namespace pv
