// pv_image.cu — a physical-memory image that keeps only some byte ranges in
// HBM (per-rank residency).
//
// The reference's host memory is one flat bytearray: the host-private region
// followed by one slot per guest (memvirt.py:433-480), and every hpa is a
// byte offset into it.  A rank of a guest-sharded job serves only its own
// guests, so it needs the host-private region (all table nodes of the
// shadow / TDP / hybrid walks live there) and its guests' slots -- not the
// other 7/8 of a 64 GiB world.  The image is one reserved virtual range of
// the full size (so every hpa keeps its offset and no kernel changes), with
// physical HBM mapped only under the resident ranges (CUDA virtual memory
// management: cuMemAddressReserve / cuMemCreate / cuMemMap).  The gaps are
// backed by one small zero-filled "hole" allocation mapped again and again:
// a stray access (a corrupted table pointing into another guest's slot)
// reads junk instead of faulting the context; the host control plane never
// relies on non-resident bytes (image.py keeps them host-side).
//
// Driver entry points come from cudaGetDriverEntryPoint, so libpv has no
// link-time dependency on libcuda (it still loads on a GPU-less host).
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "pv_common.cuh"

namespace pv {
namespace {

struct Driver {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) free_va = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      p == nullptr)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuMemGetAllocationGranularity", &d.granularity) && entry("cuMemAddressReserve", &d.reserve) &&
           entry("cuMemAddressFree", &d.free_va) && entry("cuMemCreate", &d.create) &&
           entry("cuMemRelease", &d.release) && entry("cuMemMap", &d.map) && entry("cuMemUnmap", &d.unmap) &&
           entry("cuMemSetAccess", &d.access);
  });
  return d;
}

struct Image {
  CUdeviceptr base = 0;
  size_t reserved = 0;
  std::vector<std::pair<size_t, size_t>> mapped;  // (offset, size) of every mapping
  std::vector<CUmemGenericAllocationHandle> handles;
  uint64_t resident_bytes = 0;
  uint64_t hole_bytes = 0;
};

void destroy(const Driver& d, Image* im) {
  for (auto& m : im->mapped) d.unmap(im->base + m.first, m.second);
  for (auto h : im->handles) d.release(h);
  if (im->base) d.free_va(im->base, im->reserved);
  delete im;
}

}  // namespace
}  // namespace pv

using namespace pv;

extern "C" int pv_image_create(uint64_t image_bytes, const uint64_t* ranges, uint32_t n_ranges, uint64_t hole_bytes,
                               uint8_t** out_ptr, void** out_handle, uint64_t* out_device_bytes) {
  if (!out_ptr || !out_handle || image_bytes == 0 || (n_ranges && !ranges)) return PV_EINVAL;
  const Driver& d = driver();
  if (!d.ok) return PV_ECUDA - (int)cudaErrorNotSupported;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PV_ECUDA - (int)cudaErrorNoDevice;
  CUmemAllocationProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gran = 0;
  if (d.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || gran == 0)
    return PV_ECUDA - (int)cudaErrorInvalidValue;
  auto up = [gran](uint64_t x) { return (x + gran - 1) / gran * gran; };
  auto down = [gran](uint64_t x) { return x / gran * gran; };
  const size_t total = up(image_bytes);
  // resident ranges, widened to the granularity and merged
  std::vector<std::pair<uint64_t, uint64_t>> res;
  for (uint32_t i = 0; i < n_ranges; ++i) {
    const uint64_t a = ranges[2 * i], b = ranges[2 * i + 1];
    if (a > b || b > image_bytes) return PV_EINVAL;
    if (a < b) res.emplace_back(down(a), std::min<uint64_t>(up(b), total));
  }
  std::sort(res.begin(), res.end());
  std::vector<std::pair<uint64_t, uint64_t>> merged;
  for (auto& r : res) {
    if (!merged.empty() && r.first <= merged.back().second)
      merged.back().second = std::max(merged.back().second, r.second);
    else
      merged.push_back(r);
  }
  auto* im = new Image();
  im->reserved = total;
  if (d.reserve(&im->base, total, gran, 0, 0) != CUDA_SUCCESS) {
    delete im;
    return PV_ENOMEM;
  }
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  auto map_one = [&](size_t off, size_t size, CUmemGenericAllocationHandle h) -> bool {
    if (d.map(im->base + off, size, 0, h, 0) != CUDA_SUCCESS) return false;
    im->mapped.emplace_back(off, size);
    return d.access(im->base + off, size, &acc, 1) == CUDA_SUCCESS;
  };
  bool ok = true;
  for (auto& r : merged) {
    CUmemGenericAllocationHandle h;
    if (d.create(&h, r.second - r.first, &prop, 0) != CUDA_SUCCESS) {
      ok = false;
      break;
    }
    im->handles.push_back(h);
    ok = map_one(r.first, r.second - r.first, h);
    if (!ok) break;
    im->resident_bytes += r.second - r.first;
  }
  // the gaps: one hole allocation mapped repeatedly
  std::vector<std::pair<uint64_t, uint64_t>> gaps;
  uint64_t at = 0;
  for (auto& r : merged) {
    if (r.first > at) gaps.emplace_back(at, r.first);
    at = r.second;
  }
  if (at < total) gaps.emplace_back(at, total);
  if (ok && !gaps.empty()) {
    const size_t hole = std::max<size_t>(gran, up(hole_bytes ? hole_bytes : (256ull << 20)));
    CUmemGenericAllocationHandle h;
    ok = d.create(&h, hole, &prop, 0) == CUDA_SUCCESS;
    if (ok) {
      im->handles.push_back(h);
      im->hole_bytes = hole;
      for (auto& g : gaps) {
        for (uint64_t off = g.first; ok && off < g.second; off += hole)
          ok = map_one(off, std::min<uint64_t>(hole, g.second - off), h);
        if (!ok) break;
      }
    }
  }
  if (ok) {
    // a fresh image is zero-filled, like the reference's bytearray
    for (auto& r : merged)
      if (cudaMemset(reinterpret_cast<void*>(im->base + r.first), 0, r.second - r.first) != cudaSuccess) ok = false;
    if (ok && im->hole_bytes) {
      // every hole mapping starts at byte 0 of the hole: zeroing the longest
      // one zeroes every byte of the hole that is mapped anywhere
      size_t best = 0, best_off = 0;
      for (auto& g : gaps) {
        const size_t len = std::min<uint64_t>(im->hole_bytes, g.second - g.first);
        if (len > best) best = len, best_off = g.first;
      }
      if (best) ok = cudaMemset(reinterpret_cast<void*>(im->base + best_off), 0, best) == cudaSuccess;
    }
    ok = ok && cudaDeviceSynchronize() == cudaSuccess;
  }
  if (!ok) {
    destroy(d, im);
    return PV_ENOMEM;
  }
  *out_ptr = reinterpret_cast<uint8_t*>(im->base);
  *out_handle = im;
  if (out_device_bytes) *out_device_bytes = im->resident_bytes + im->hole_bytes;
  return PV_SUCCESS;
}

extern "C" int pv_image_destroy(void* handle) {
  if (!handle) return PV_EINVAL;
  const Driver& d = driver();
  if (!d.ok) return PV_ECUDA - (int)cudaErrorNotSupported;
  cudaDeviceSynchronize();
  destroy(d, static_cast<Image*>(handle));
  return PV_SUCCESS;
}
