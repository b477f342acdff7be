// pv_map.cu — batched table construction on the device.
//
// Reference (memvirt.py:270-313 TableEditor.map / _descend, 508-526
// map_process_page / map_region, 191-213 FrameAllocator): pages are mapped
// one after another; a page whose top entry is NOT_PRESENT allocates a mid
// node, a page whose (top, mid) entry is NOT_PRESENT allocates a leaf node
// (each from the table's FIFO allocator, zeroed on allocation, installed as
// PRESENT | writable), and the leaf entry is written last.  map_process_page
// first draws the page's data frame from the guest allocator, so its frame
// order per page is [data][mid?][leaf?].
//
// Device form, exact for a batch in which every page maps a currently free
// leaf slot exactly once:
//   plan   : per page, read the existing top / mid entries; the first page (in
//            batch order) of each top index that lacks a mid node and of each
//            (top, mid) that lacks a leaf node is marked -- those are exactly
//            the pages that allocate, in the reference's order -- and any page
//            the batch cannot build exactly (leaf already present or trapping
//            = AlreadyMapped, existing node past the image = struct.error, a
//            repeated (top, mid, leaf) slot) lowers *bad;
//   commit : the caller draws the frames from its allocator in order and
//            passes their per-page offsets (exclusive scan of the counts);
//            frames that may hold bytes are zeroed, then the new top entries,
//            the new mid entries and the leaf entries are written in three
//            dependent passes (each pass reads the entries the previous one
//            installed).
// Every written page is marked in the dirty map (host coherence, leaf index).
#include "pv_common.cuh"

namespace pv {

constexpr int kMapTpb = 256;
constexpr uint32_t kTops = 4, kMids = 512;
constexpr uint64_t kWordPW = kFlagPresent | 0x2ull;  // encode_entry(PRESENT, pfn, writable=True) flags

struct MapScratch {
  uint32_t* first_top;  // [4]   first page lacking the mid node of its top
  uint32_t* first_tm;   // [2048] first page lacking the leaf node of its (top, mid)
  uint32_t* first_key;  // [2^20] first page of each (top, mid, leaf) slot
};

static MapScratch carve_map(void* scratch) {
  MapScratch s;
  s.first_top = reinterpret_cast<uint32_t*>(scratch);
  s.first_tm = s.first_top + kTops;
  s.first_key = s.first_tm + kTops * kMids;
  return s;
}

size_t map_scratch_bytes() { return (kTops + kTops * kMids + (1u << 20)) * sizeof(uint32_t); }

__device__ __forceinline__ uint64_t* word_ptr(uint8_t* image, uint64_t base, uint64_t node, uint32_t idx) {
  return reinterpret_cast<uint64_t*>(image + base + (node << kPageShift)) + idx;
}

__global__ void __launch_bounds__(kMapTpb)
map_plan_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, uint64_t base, uint64_t root,
                const uint64_t* __restrict__ vas, uint64_t n, MapScratch sc, uint8_t* __restrict__ need,
                unsigned long long* __restrict__ bad) {
  const uint64_t lim = node_limit(image_bytes, base);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t va = vas[i];
    const uint32_t t = top_index(va), m = mid_index(va), l = leaf_index(va);
    atomicMin(sc.first_key + ((t << 18) | (m << 9) | l), (uint32_t)i);
    uint8_t st = 0;  // bit 0: top lacks a mid node, bit 1: (top, mid) lacks a leaf node
    if (root >= lim) {
      atomicMin(bad, (unsigned long long)i);
    } else {
      const uint64_t tw = ld_word(image, base, root, t);
      if (!(tw & (kFlagPresent | kFlagTrapping))) {
        st = 3;
      } else {
        const uint64_t mnode = tw >> kPageShift;  // _descend follows any entry that is not NOT_PRESENT
        if (mnode >= lim) {
          atomicMin(bad, (unsigned long long)i);
        } else {
          const uint64_t mw = ld_word(image, base, mnode, m);
          if (!(mw & (kFlagPresent | kFlagTrapping))) {
            st = 2;
          } else {
            const uint64_t lnode = mw >> kPageShift;
            if (lnode >= lim || (ld_word(image, base, lnode, l) & (kFlagPresent | kFlagTrapping)))
              atomicMin(bad, (unsigned long long)i);  // struct.error / AlreadyMapped
          }
        }
      }
    }
    if (st & 1) atomicMin(sc.first_top + t, (uint32_t)i);
    if (st & 2) atomicMin(sc.first_tm + t * kMids + m, (uint32_t)i);
    need[i] = st;  // provisional: presence bits, resolved to "allocates" by map_need_kernel
  }
}

__global__ void __launch_bounds__(kMapTpb)
map_need_kernel(const uint64_t* __restrict__ vas, uint64_t n, MapScratch sc, uint8_t* __restrict__ need,
                unsigned long long* __restrict__ bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t va = vas[i];
    const uint32_t t = top_index(va), m = mid_index(va), l = leaf_index(va);
    if (sc.first_key[(t << 18) | (m << 9) | l] != (uint32_t)i) atomicMin(bad, (unsigned long long)i);
    const uint8_t st = need[i];
    uint8_t r = 0;
    if ((st & 1) && sc.first_top[t] == (uint32_t)i) r |= 1;
    if ((st & 2) && sc.first_tm[t * kMids + m] == (uint32_t)i) r |= 2;
    need[i] = r;
  }
}

// Zero allocated frames that may hold bytes (host-known hot[j], or written
// on the device since the host last looked: dirty[page]).
__global__ void __launch_bounds__(kMapTpb)
map_zero_kernel(uint8_t* __restrict__ image, uint64_t base, const uint64_t* __restrict__ frames, uint64_t n_frames,
                const uint8_t* __restrict__ hot, uint8_t* __restrict__ dirty) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (kMapTpb / 32);
  for (uint64_t j = (uint64_t)blockIdx.x * (kMapTpb / 32) + warp; j < n_frames; j += nw) {
    const uint64_t page = (base >> kPageShift) + frames[j];
    const bool z = (hot != nullptr && hot[j]) || (dirty != nullptr && dirty[page]);
    if (!z) continue;
    uint4* p = reinterpret_cast<uint4*>(image + (page << kPageShift));
#pragma unroll
    for (int k = 0; k < 8; ++k) p[lane + 32 * k] = make_uint4(0, 0, 0, 0);
    if (dirty != nullptr && lane == 0) dirty[page] = 1;
  }
}

// Frame of page i at position `pos` of its allocation group.
__device__ __forceinline__ uint64_t frame_at(const uint64_t* frames, const uint64_t* frame_off, uint64_t i,
                                             uint32_t pos) {
  return frames[frame_off[i] + pos];
}

__global__ void __launch_bounds__(kMapTpb)
map_top_kernel(uint8_t* __restrict__ image, uint64_t base, uint64_t root, const uint64_t* __restrict__ vas, uint64_t n,
               const uint8_t* __restrict__ need, const uint64_t* __restrict__ frames,
               const uint64_t* __restrict__ frame_off, uint32_t data_first, uint8_t* __restrict__ dirty) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (!(need[i] & 1)) continue;
    const uint64_t mid = frame_at(frames, frame_off, i, data_first);
    *word_ptr(image, base, root, top_index(vas[i])) = (mid << kPageShift) | kWordPW;
    if (dirty != nullptr) dirty[(base >> kPageShift) + root] = 1;
  }
}

__global__ void __launch_bounds__(kMapTpb)
map_mid_kernel(uint8_t* __restrict__ image, uint64_t base, uint64_t root, const uint64_t* __restrict__ vas, uint64_t n,
               const uint8_t* __restrict__ need, const uint64_t* __restrict__ frames,
               const uint64_t* __restrict__ frame_off, uint32_t data_first, uint8_t* __restrict__ dirty) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint8_t nd = need[i];
    if (!(nd & 2)) continue;
    const uint64_t va = vas[i];
    const uint64_t leaf = frame_at(frames, frame_off, i, data_first + (nd & 1));
    const uint64_t mnode = *word_ptr(image, base, root, top_index(va)) >> kPageShift;
    *word_ptr(image, base, mnode, mid_index(va)) = (leaf << kPageShift) | kWordPW;
    if (dirty != nullptr) dirty[(base >> kPageShift) + mnode] = 1;
  }
}

__global__ void __launch_bounds__(kMapTpb)
map_leaf_kernel(uint8_t* __restrict__ image, uint64_t base, uint64_t root, const uint64_t* __restrict__ vas, uint64_t n,
                const uint64_t* __restrict__ frames, const uint64_t* __restrict__ frame_off, uint32_t data_first,
                const uint64_t* __restrict__ targets, uint64_t target_add, uint64_t leaf_flags,
                uint64_t* __restrict__ out_data, uint8_t* __restrict__ dirty) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t va = vas[i];
    uint64_t target;
    if (data_first) {
      const uint64_t data = frame_at(frames, frame_off, i, 0);
      if (out_data != nullptr) out_data[i] = data;
      target = data + target_add;
    } else {
      target = targets[i] + target_add;
    }
    const uint64_t mnode = *word_ptr(image, base, root, top_index(va)) >> kPageShift;
    const uint64_t lnode = *word_ptr(image, base, mnode, mid_index(va)) >> kPageShift;
    *word_ptr(image, base, lnode, leaf_index(va)) = (target << kPageShift) | leaf_flags;
    if (dirty != nullptr) dirty[(base >> kPageShift) + lnode] = 1;
  }
}

template <typename K>
static unsigned grid_of(K k, uint64_t work) {
  uint64_t g = (work + kMapTpb - 1) / kMapTpb;
  const uint64_t cap = resident_grid((const void*)k, kMapTpb, 0);
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

cudaError_t launch_map_plan(const uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root,
                            const uint64_t* vas, uint64_t n, uint8_t* need, uint64_t* bad, void* scratch,
                            cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(scratch, 0xFF, map_scratch_bytes(), stream);
  if (e != cudaSuccess) return e;
  MapScratch sc = carve_map(scratch);
  auto* b = reinterpret_cast<unsigned long long*>(bad);
  map_plan_kernel<<<grid_of(map_plan_kernel, n), kMapTpb, 0, stream>>>(image, image_bytes, base, root, vas, n, sc,
                                                                       need, b);
  map_need_kernel<<<grid_of(map_need_kernel, n), kMapTpb, 0, stream>>>(vas, n, sc, need, b);
  return cudaGetLastError();
}

cudaError_t launch_map_commit(uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root, const uint64_t* vas,
                              uint64_t n, const uint8_t* need, const uint64_t* frames, uint64_t n_frames,
                              const uint64_t* frame_off, const uint8_t* hot, uint32_t data_first,
                              const uint64_t* targets, uint64_t target_add, uint64_t leaf_flags, uint64_t* out_data,
                              uint8_t* dirty, cudaStream_t stream) {
  (void)image_bytes;
  if (n == 0) return cudaSuccess;
  if (n_frames) {
    const uint64_t warps_per_cta = kMapTpb / 32;
    uint64_t g = (n_frames + warps_per_cta - 1) / warps_per_cta;
    const uint64_t cap = resident_grid((const void*)map_zero_kernel, kMapTpb, 0);
    if (g > cap) g = cap;
    map_zero_kernel<<<(unsigned)g, kMapTpb, 0, stream>>>(image, base, frames, n_frames, hot, dirty);
  }
  map_top_kernel<<<grid_of(map_top_kernel, n), kMapTpb, 0, stream>>>(image, base, root, vas, n, need, frames,
                                                                     frame_off, data_first, dirty);
  map_mid_kernel<<<grid_of(map_mid_kernel, n), kMapTpb, 0, stream>>>(image, base, root, vas, n, need, frames,
                                                                     frame_off, data_first, dirty);
  map_leaf_kernel<<<grid_of(map_leaf_kernel, n), kMapTpb, 0, stream>>>(image, base, root, vas, n, frames, frame_off,
                                                                       data_first, targets, target_add, leaf_flags,
                                                                       out_data, dirty);
  return cudaGetLastError();
}

}  // namespace pv
