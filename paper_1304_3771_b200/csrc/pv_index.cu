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

// One CTA per slot (grid-stride); 256 threads x 2 entries; 16-byte loads.
__global__ void __launch_bounds__(kEncTpb)
encode_kernel(const uint8_t* __restrict__ image, uint64_t image_pages, const uint64_t* __restrict__ slot_page,
              const uint64_t* __restrict__ slots, uint64_t first_slot, uint64_t n, uint32_t* __restrict__ leaf_codes,
              const uint8_t* __restrict__ dirty) {
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t slot = slots != nullptr ? slots[i] : first_slot + i;
    const uint64_t page = slot_page[slot];
    if (page >= image_pages) continue;
    if (dirty != nullptr && dirty[page] == 0) continue;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(image + (page << kPageShift)) + threadIdx.x);
    const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
    uint2 out;
    out.x = encode_leaf(w0);
    out.y = encode_leaf(w1);
    reinterpret_cast<uint2*>(leaf_codes + (slot << 9))[threadIdx.x] = out;
  }
}

cudaError_t launch_index_encode(const uint8_t* image, uint64_t image_bytes, const uint64_t* slot_page,
                                const uint64_t* slots, uint64_t first_slot, uint64_t n, uint32_t* leaf_codes,
                                const uint8_t* dirty, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = n;
  const uint64_t cap = resident_grid((const void*)encode_kernel, kEncTpb, 0);
  if (grid > cap) grid = cap;
  encode_kernel<<<(unsigned)grid, kEncTpb, 0, stream>>>(image, image_bytes >> kPageShift, slot_page, slots,
                                                        first_slot, n, leaf_codes, dirty);
  return cudaGetLastError();
}

}  // namespace pv
