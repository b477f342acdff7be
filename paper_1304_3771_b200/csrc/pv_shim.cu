// pv_shim.cu — the hybrid resolver's trap shim on the device.
//
// Reference semantics (backend.py:117-128, 288-296; memvirt.py:685-696): a
// copy through HardwareHasAccess resolves each page through the merged
// (hybrid) top level; a trapping entry exits to the default shim, which
//   1. walks the guest's own table for the page (walk_guest of va & ~0xFFF),
//   2. converts the gpa linearly (gpa_to_hpa: 0 <= gpa < slot size),
//   3. rewrites the process's shadow leaf for the page through
//      TableEditor.map(..., replace=True): word = (hpa >> 12) << 12 | P | W,
// and the walk is retried once (a second trap is TrapFixupFailed).  Pages and
// ops run in order, so the first page that reaches a trapping slot fixes it
// and every later page that reaches the slot reads the fixed word.
//
// Device form, after pv_copy_plan over the hybrid spaces of a batch:
//   eval    : every trapped page whose shim is "simple" -- the trap is at the
//             leaf, the shadow descend for the page ends on exactly the
//             trapping slot (no node allocation, no divergence between the
//             merged and the shadow table), the guest walk succeeds and the
//             gpa is inside the slot -- is marked and appended to a list with
//             the word its shim would write.  Every other trap is left to
//             the host's per-op shim (it may allocate nodes, raise, or fail).
//   firstbad: each op's first failing page, not counting simple traps;
//   cut     : the first op whose first failure is a (non-simple) trap -- the
//             host finishes that op through its per-op shim and re-plans the
//             ops after it, so no shim of a later op may take effect here;
//   claim   : per slot, the earliest reached simple trap in (op, page) order
//             wins (open-addressing table, atomicMax of ~page);
//   apply   : winners write their word into the image (marking the dirty map);
//   rewalk  : reached simple traps re-walk the hybrid table (the retry) and
//             become ordinary translations; unreached ones get their trap
//             status back and re-enter the first-failure minimum;
//   stop    : every op after the cut moves nothing (first failing page 0):
//             the host re-plans those ops once its per-op shim has run, so
//             no byte may move through the pre-shim tables.  With a shim row
//             of guest_bytes 0 (a replaced trap_shim) nothing is simple and
//             the first trapping op is the cut.
// The passes after eval run as one cooperative kernel that returns at once
// when eval found no trap at all, so a trap-free batch pays two launches.  The scratch area is left
// zeroed after each call (the claim table cleans up after itself).
#include <cooperative_groups.h>

#include "pv_common.cuh"

namespace pv {

constexpr uint32_t kShimmed = 0x800u;  // internal page-status mark (never returned)
constexpr int kShimTpb = 256;

struct ShimScratch {
  unsigned long long* count;  // [0] simple traps listed
  unsigned long long* cut;    // [1] ~(first cut op), 0 = none
  unsigned long long* traps;  // [2] trapping pages seen by eval (simple or not)
  unsigned long long* list_p; // page index (bit 63: reached, bit 62: winner)
  unsigned long long* list_w; // shim word
  unsigned long long* list_op;
  unsigned long long* keys;   // slot word index + 1, 0 = empty
  unsigned long long* vals;   // ~winning page, 0 = none
  uint64_t mask;              // table capacity - 1
};

static uint64_t table_cap(uint64_t n_pages) {
  uint64_t c = 1024;
  while (c < 2 * n_pages) c <<= 1;
  return c;
}

static ShimScratch carve(void* scratch, uint64_t n_pages) {
  ShimScratch s;
  auto* w = reinterpret_cast<unsigned long long*>(scratch);
  const uint64_t cap = table_cap(n_pages);
  s.count = w;
  s.cut = w + 1;
  s.traps = w + 2;
  s.list_p = w + 3;
  s.list_w = s.list_p + n_pages;
  s.list_op = s.list_w + n_pages;
  s.keys = s.list_op + n_pages;
  s.vals = s.keys + cap;
  s.mask = cap - 1;
  return s;
}

size_t shim_scratch_bytes(uint64_t n_pages) { return (3 + 3 * n_pages + 2 * table_cap(n_pages)) * 8; }

__device__ __forceinline__ uint64_t hash_slot(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  return k;
}

// Op of page p and the page's index within it.
__device__ __forceinline__ void op_of(const uint64_t* __restrict__ page_off, uint64_t n_ops, uint64_t p, uint64_t* op,
                                      uint64_t* k) {
  *op = upper_search(page_off, 0, n_ops, p);
  *k = p - __ldg(page_off + *op);
}

// TableEditor._descend(create=False-like) over the shadow table (memvirt.py:
// 282-298): anything but NOT_PRESENT is followed (a trapping upper entry is
// descended through).  Returns false where the reference would allocate a
// node or read past memory.
__device__ __forceinline__ bool shadow_descend(const uint8_t* __restrict__ image, uint64_t image_bytes, uint64_t root,
                                               uint64_t va, uint64_t* leaf_node) {
  const uint64_t lim = node_limit(image_bytes, 0);
  uint64_t node = root;
  const uint32_t idx[2] = {top_index(va), mid_index(va)};
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    if (node >= lim) return false;
    const uint64_t w = *reinterpret_cast<const volatile unsigned long long*>(image + (node << kPageShift) + 8 * idx[l]);
    if (!(w & (kFlagPresent | kFlagTrapping))) return false;  // NOT_PRESENT: the reference allocates
    node = w >> kPageShift;
  }
  if (node >= lim) return false;
  *leaf_node = node;
  return true;
}

__global__ void __launch_bounds__(kShimTpb)
shim_eval_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes, const pv_op* __restrict__ ops, uint64_t n_ops,
                 const uint64_t* __restrict__ page_off, uint64_t n_pages, const pv_shim* __restrict__ shims,
                 const uint64_t* __restrict__ page_hpa, uint32_t* __restrict__ page_status, ShimScratch sc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pages; p += stride) {
    const uint32_t st = page_status[p];
    if (PV_ST_KIND(st) == PV_ST_TRAP2) atomicAdd(sc.traps, 1ull);
    if (PV_ST_KIND(st) != PV_ST_TRAP) continue;
    atomicAdd(sc.traps, 1ull);
    if (PV_ST_LEVEL(st) != 3) continue;
    uint64_t op, k;
    op_of(page_off, n_ops, p, &op, &k);
    const pv_op o = ops[op];
    const pv_shim sh = shims[o.space];
    if (sh.guest_bytes == 0) continue;
    const uint64_t page_va = op_page_va(o.gva, k) & ~kPageMask;
    // walk_guest(page_va) in the guest window (memvirt.py:262-267)
    uint64_t gpfn = 0;
    if (walk_global(image, image_bytes, sh.guest_base, sh.guest_root_pfn, page_va, 0, &gpfn) != PV_ST_OK) continue;
    const uint64_t gpa = gpfn << kPageShift;
    if ((gpa >> kPageShift) != gpfn || gpa >= sh.guest_bytes) continue;  // gpa_to_hpa: OutOfRange
    uint64_t leaf = 0;
    if (!shadow_descend(image, image_bytes, sh.shadow_root_pfn, page_va, &leaf)) continue;
    if (leaf != page_hpa[p] || leaf_index(page_va) != PV_ST_INDEX(st)) continue;  // not the trapping slot
    const uint64_t hpa = sh.guest_base + gpa;
    const uint64_t word = ((hpa >> kPageShift) << kPageShift) | kFlagPresent | 0x2ull;  // PRESENT, writable
    page_status[p] = st | kShimmed;
    const unsigned long long i = atomicAdd(sc.count, 1ull);
    sc.list_p[i] = p;
    sc.list_w[i] = word;
    sc.list_op[i] = op;
  }
}

// The passes after eval, in ONE cooperative launch (grid-wide barriers
// between them): a trap-free batch costs one more launch, not seven.
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t find_slot(const ShimScratch& sc, uint64_t key) {
  uint64_t h = hash_slot(key) & sc.mask;
  while (sc.keys[h] != key) h = (h + 1) & sc.mask;
  return h;
}

// Steps 1-5 (only when eval listed simple traps).
__device__ __noinline__ void shim_fix(cg::grid_group& grid, uint64_t tid, uint64_t nthr, uint64_t n,
                                      const ShimScratch& sc, uint8_t* __restrict__ image, uint64_t image_bytes,
                                      const pv_space* __restrict__ spaces, const pv_op* __restrict__ ops,
                                      uint64_t n_ops, const uint64_t* __restrict__ page_off, uint64_t n_pages,
                                      uint64_t* __restrict__ page_hpa, uint32_t* __restrict__ page_status,
                                      unsigned long long* __restrict__ op_first_bad, uint8_t* __restrict__ dirty,
                                      unsigned long long* __restrict__ n_written) {
  // 1. the first failing page of every op holding a simple trap is recomputed
  for (uint64_t i = tid; i < n; i += nthr) op_first_bad[sc.list_op[i]] = kNone;
  grid.sync();
  for (uint64_t p = tid; p < n_pages; p += nthr) {
    const uint32_t st = page_status[p];
    if (st == PV_ST_OK || (st & kShimmed)) continue;
    uint64_t op, k;
    op_of(page_off, n_ops, p, &op, &k);
    atomicMin(op_first_bad + op, (unsigned long long)k);
  }
  grid.sync();
  // 2. the cut: the first op whose first failure is a trap the device cannot fix
  for (uint64_t p = tid; p < n_pages; p += nthr) {
    const uint32_t st = page_status[p];
    const uint32_t kd = PV_ST_KIND(st);
    if ((kd != PV_ST_TRAP && kd != PV_ST_TRAP2) || (st & kShimmed)) continue;
    uint64_t op, k;
    op_of(page_off, n_ops, p, &op, &k);
    if (op_first_bad[op] == k) atomicMax(sc.cut, ~(unsigned long long)op);
  }
  grid.sync();
  // 3. claim: per slot, the earliest reached page wins
  const unsigned long long cut = ~*sc.cut;  // kNone when no op is cut
  for (uint64_t i = tid; i < n; i += nthr) {
    const uint64_t p = sc.list_p[i], op = sc.list_op[i];
    const uint64_t k = p - __ldg(page_off + op);
    if (op > cut || k >= op_first_bad[op]) continue;  // never reached in program order
    sc.list_p[i] = p | (1ull << 63);
    const uint64_t key = page_hpa[p] * 512 + PV_ST_INDEX(page_status[p]) + 1;
    uint64_t h = hash_slot(key) & sc.mask;
    while (true) {
      const unsigned long long prev = atomicCAS(sc.keys + h, 0ull, (unsigned long long)key);
      if (prev == 0 || prev == key) break;
      h = (h + 1) & sc.mask;
    }
    atomicMax(sc.vals + h, ~(unsigned long long)p);
  }
  grid.sync();
  // 4. winners write their word
  for (uint64_t i = tid; i < n; i += nthr) {
    const uint64_t tagged = sc.list_p[i];
    if (!(tagged >> 63)) continue;
    const uint64_t p = tagged & ~(3ull << 62);
    const uint64_t node = page_hpa[p];
    const uint64_t key = node * 512 + PV_ST_INDEX(page_status[p]) + 1;
    const uint64_t h = find_slot(sc, key);
    if (~sc.vals[h] != p) continue;
    sc.list_p[i] = tagged | (1ull << 62);
    const uint64_t word = sc.list_w[i];
    sc.list_w[i] = h;  // for the cleanup
    *reinterpret_cast<unsigned long long*>(image + (node << kPageShift) + 8 * PV_ST_INDEX(page_status[p])) = word;
    if (dirty != nullptr) dirty[node] = 1;
    if (n_written != nullptr) atomicAdd(n_written, 1ull);
  }
  grid.sync();
  // 5. the retry walk of every reached page; unreached ones get their trap
  //    status back; winners clear their claim-table entry
  for (uint64_t i = tid; i < n; i += nthr) {
    const uint64_t tagged = sc.list_p[i];
    const uint64_t p = tagged & ~(3ull << 62), op = sc.list_op[i];
    const uint64_t k = p - __ldg(page_off + op);
    if ((tagged >> 62) & 1) {
      const uint64_t h = sc.list_w[i];
      sc.keys[h] = 0;
      sc.vals[h] = 0;
    }
    if (!(tagged >> 63)) {
      page_status[p] &= ~kShimmed;
      atomicMin(op_first_bad + op, (unsigned long long)k);
      continue;
    }
    // the retry of resolve_hybrid_with_fixup (memvirt.py:693-696)
    const pv_op o = ops[op];
    const uint64_t cur = op_page_va(o.gva, k);
    const uint64_t chunk = min(o.len - (cur - o.gva), kPageSize - (cur & kPageMask));
    uint64_t value = 0, aux = 0;
    uint32_t st = translate_global(image, image_bytes, spaces[o.space], cur, &value, &aux);
    if (st == PV_ST_OK) {
      value = (value << kPageShift) | (cur & kPageMask);
      if (value + chunk > image_bytes || value + chunk < value) st = PV_ST_DATA_OOR;
    }
    page_hpa[p] = value;
    page_status[p] = st;
    if (st != PV_ST_OK) atomicMin(op_first_bad + op, (unsigned long long)k);
  }
  grid.sync();
  if (tid == 0) *sc.cut = 0;  // step 6 computes the cut after the shim
  grid.sync();
}

__global__ void __launch_bounds__(kShimTpb)
shim_resolve_kernel(ShimScratch sc, uint8_t* __restrict__ image, uint64_t image_bytes,
                    const pv_space* __restrict__ spaces, const pv_op* __restrict__ ops, uint64_t n_ops,
                    const uint64_t* __restrict__ page_off, uint64_t n_pages, uint64_t* __restrict__ page_hpa,
                    uint32_t* __restrict__ page_status, unsigned long long* __restrict__ op_first_bad,
                    uint8_t* __restrict__ dirty, unsigned long long* __restrict__ n_written) {
  if (*sc.traps == 0) return;  // uniform across the grid: nothing trapped
  const uint64_t n = *sc.count;
  cg::grid_group grid = cg::this_grid();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  if (n != 0) shim_fix(grid, tid, nthr, n, sc, image, image_bytes, spaces, ops, n_ops, page_off, n_pages, page_hpa,
                       page_status, op_first_bad, dirty, n_written);
  // 6. stop: the cut after the shim is the first op whose first failing page
  //    still traps; the ops after it move nothing
  for (uint64_t op = tid; op < n_ops; op += nthr) {
    const unsigned long long fb = op_first_bad[op];
    if (fb == kNone) continue;
    const uint32_t kd = PV_ST_KIND(page_status[__ldg(page_off + op) + fb]);
    if (kd == PV_ST_TRAP || kd == PV_ST_TRAP2) atomicMax(sc.cut, ~(unsigned long long)op);
  }
  grid.sync();
  const unsigned long long cut = ~*sc.cut;
  if (cut != kNone)
    for (uint64_t op = cut + 1 + tid; op < n_ops; op += nthr) op_first_bad[op] = 0;
  grid.sync();
  if (tid == 0) {  // leave the scratch zero-filled
    *sc.count = 0;
    *sc.cut = 0;
    *sc.traps = 0;
  }
}

cudaError_t launch_copy_shim(uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_shim* shims,
                             const pv_op* ops, uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages,
                             uint64_t* page_hpa, uint32_t* page_status, uint64_t* op_first_bad, uint8_t* dirty,
                             uint64_t* n_written, void* scratch, cudaStream_t stream) {
  if (n_pages == 0) return cudaSuccess;
  ShimScratch sc = carve(scratch, n_pages);
  auto* fb = reinterpret_cast<unsigned long long*>(op_first_bad);
  auto grid_for = [](const void* f, uint64_t work) {
    uint64_t g = (work + kShimTpb - 1) / kShimTpb;
    const uint64_t cap = resident_grid(f, kShimTpb, 0);
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
  };
  const unsigned gp = grid_for((const void*)shim_eval_kernel, n_pages);
  shim_eval_kernel<<<gp, kShimTpb, 0, stream>>>(image, image_bytes, ops, n_ops, page_off, n_pages, shims, page_hpa,
                                                 page_status, sc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // every CTA of a cooperative launch must be resident at once
  unsigned gr = (unsigned)resident_grid((const void*)shim_resolve_kernel, kShimTpb, 0);
  unsigned long long* nw = reinterpret_cast<unsigned long long*>(n_written);
  void* args[] = {&sc, &image, &image_bytes, &spaces, &ops, &n_ops, &page_off, &n_pages,
                  &page_hpa, &page_status, &fb, &dirty, &nw};
  return cudaLaunchCooperativeKernel((const void*)shim_resolve_kernel, dim3(gr), dim3(kShimTpb), args, 0, stream);
}

}  // namespace pv
