// pv_abi.cu — extern "C" entry points of libpv (declared in include/pv.h).
//
// Thin validation + launch layer: no allocation of user-visible memory, no
// exceptions across the boundary, CUDA errors returned as PV_ECUDA - err.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <unordered_map>

#include <cuda.h>

#include "pv_common.cuh"

namespace pv {
cudaError_t launch_translate(const uint8_t*, uint64_t, const pv_space*, const pv_seg*, uint32_t, uint64_t,
                             const void*, uint32_t, bool, const pv_index*, uint64_t*, uint32_t*, uint64_t*,
                             const ExcSink*, cudaStream_t);
cudaError_t launch_index_encode(const uint8_t*, uint64_t, const uint64_t*, const uint64_t*, uint64_t, uint64_t,
                                uint32_t*, const uint8_t*, cudaStream_t);
uint64_t translate_chunk();
cudaError_t launch_copy_plan(const uint8_t*, uint64_t, const pv_space*, const pv_op*, uint64_t, const uint64_t*,
                             uint64_t, uint64_t*, uint32_t*, uint64_t*, uint64_t*, uint32_t*, uint32_t, cudaStream_t);
cudaError_t launch_copy_stamp(const uint64_t*, uint64_t, uint64_t, const uint64_t*, const uint64_t*, uint64_t*,
                              uint64_t, uint32_t, uint32_t*, const uint32_t*, cudaStream_t);
cudaError_t launch_walk_one(const uint8_t*, uint64_t, const pv_space&, uint64_t, uint32_t, pv_one_result*, uint64_t,
                            cudaStream_t);
cudaError_t launch_copy_small(uint8_t*, uint64_t, const pv_small_op&, uint8_t*, uint64_t, pv_small_result*, uint8_t*,
                              uint32_t, uint64_t, cudaStream_t);
cudaError_t launch_copy_exec(uint8_t*, uint64_t, const pv_op*, uint64_t, const uint64_t*, uint64_t, uint32_t,
                             const uint64_t*, const uint32_t*, const uint64_t*, const uint64_t*, uint8_t*,
                             uint64_t, pv_op_result*, uint8_t*, const uint32_t*, cudaStream_t);
size_t fifo_scratch_bytes(uint64_t, uint64_t, uint32_t);
size_t shim_scratch_bytes(uint64_t);
size_t map_scratch_bytes();
size_t frame_scratch_bytes(uint64_t);
cudaError_t launch_frame_pack(const uint64_t*, uint64_t, const uint64_t*, const uint64_t*, const uint64_t*,
                              const uint64_t*, pv_frame*, uint32_t*, cudaStream_t);
cudaError_t launch_frame_identify(const pv_frame*, uint64_t, const int32_t*, uint32_t, const uint64_t*,
                                  const uint64_t*, uint32_t, uint32_t*, uint32_t*, cudaStream_t);
cudaError_t launch_frame_assemble(const pv_frame*, uint64_t, const uint32_t*, uint64_t*, uint32_t*, void*, uint64_t,
                                  cudaStream_t);
cudaError_t launch_map_plan(const uint8_t*, uint64_t, uint64_t, uint64_t, const uint64_t*, uint64_t, uint8_t*,
                            uint64_t*, void*, cudaStream_t);
cudaError_t launch_map_commit(uint8_t*, uint64_t, uint64_t, uint64_t, const uint64_t*, uint64_t, const uint8_t*,
                              const uint64_t*, uint64_t, const uint64_t*, const uint8_t*, uint32_t, const uint64_t*,
                              uint64_t, uint64_t, uint64_t*, uint8_t*, cudaStream_t);
cudaError_t launch_copy_shim(uint8_t*, uint64_t, const pv_space*, const pv_shim*, const pv_op*, uint64_t,
                             const uint64_t*, uint64_t, uint64_t*, uint32_t*, uint64_t*, uint8_t*, uint64_t*,
                             void*, cudaStream_t);
size_t ordered_scratch_bytes(uint64_t, uint64_t);
cudaError_t launch_result_encode(uint8_t*, uint64_t, const uint64_t*, const uint32_t*, const uint8_t*, const uint64_t*,
                                 uint64_t, uint32_t*, uint8_t*, cudaStream_t);
cudaError_t launch_result_decode(const uint8_t*, uint64_t, const uint64_t*, uint64_t, uint32_t*, uint32_t*,
                                 cudaStream_t);
cudaError_t launch_copy_ordered(uint8_t*, uint64_t, const pv_op*, uint64_t, const uint64_t*, uint64_t, const uint64_t*,
                                const uint32_t*, const uint64_t*, const uint64_t*, const uint8_t*, uint64_t,
                                pv_op_result*, uint8_t*, void*, uint64_t, cudaStream_t);
cudaError_t launch_fifo_lanes_abi(const void*, uint32_t, const uint64_t*, const uint64_t*, const uint64_t*, uint32_t,
                                  uint64_t, uint64_t, uint32_t, pv_fifo*, uint64_t*, uint32_t*, void*, uint64_t,
                                  cudaStream_t);
cudaError_t launch_fifo_copy_abi(const pv_op*, const uint64_t*, const uint64_t*, const uint32_t*, const uint64_t*,
                                 const uint64_t*, uint32_t, uint64_t, uint64_t, uint32_t, pv_fifo*, uint64_t, uint64_t*,
                                 uint32_t*, uint64_t*, void*, uint64_t, cudaStream_t);

namespace {
struct TimedLaunch {
  std::string name;
  cudaEvent_t ev[2];
};
std::mutex timing_mu;
bool timing_on = false;
std::vector<TimedLaunch> timing_log;
}  // namespace

cudaError_t timing_enable(bool on) {
  std::lock_guard<std::mutex> g(timing_mu);
  for (auto& t : timing_log) {
    cudaEventDestroy(t.ev[0]);
    cudaEventDestroy(t.ev[1]);
  }
  timing_log.clear();
  timing_on = on;
  return cudaSuccess;
}

void* timing_begin(const char* name, cudaStream_t stream) {
  std::lock_guard<std::mutex> g(timing_mu);
  if (!timing_on) return nullptr;
  TimedLaunch t{name, {nullptr, nullptr}};
  if (cudaEventCreate(&t.ev[0]) != cudaSuccess || cudaEventCreate(&t.ev[1]) != cudaSuccess) return nullptr;
  cudaEventRecord(t.ev[0], stream);
  timing_log.push_back(t);
  return reinterpret_cast<void*>(timing_log.size());
}

void timing_end(void* token, cudaStream_t stream) {
  if (token == nullptr) return;
  std::lock_guard<std::mutex> g(timing_mu);
  const size_t i = reinterpret_cast<size_t>(token) - 1;
  if (i < timing_log.size()) cudaEventRecord(timing_log[i].ev[1], stream);
}

double timing_ms(const char* name, uint64_t* launches) {
  std::lock_guard<std::mutex> g(timing_mu);
  double ms = 0;
  uint64_t n = 0;
  for (auto& t : timing_log) {
    if (name != nullptr && t.name != name) continue;
    float f = 0;
    cudaEventSynchronize(t.ev[1]);
    if (cudaEventElapsedTime(&f, t.ev[0], t.ev[1]) == cudaSuccess) {
      ms += f;
      ++n;
    }
  }
  if (launches != nullptr) *launches = n;
  return ms;
}

// SMs the calling thread's launches size their grids for (0: the device's);
// set by pv_set_sm_budget while the thread launches into an SM partition.
static thread_local uint32_t t_sm_budget = 0;

uint64_t resident_grid(const void* func, int tpb, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::pair<uint64_t, uint64_t>> cache;  // -> (sms, per_sm)
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(func) << 8) ^ (uint64_t)dev ^ ((uint64_t)smem << 48);
  uint64_t sms_dev = 0, per = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      sms_dev = it->second.first;
      per = it->second.second;
    }
  }
  if (per == 0) {
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, tpb, smem);
    if (per_sm < 1) per_sm = 1;
    sms_dev = (uint64_t)sms;
    per = (uint64_t)per_sm;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = {sms_dev, per};
  }
  const uint64_t sms = (t_sm_budget != 0 && t_sm_budget < sms_dev) ? t_sm_budget : sms_dev;
  return sms * per;
}

cudaError_t ensure_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, size_t> done;  // (func, device) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(func) << 8) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

cudaError_t stream_scratch(void** p, size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static bool configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> g(mu);
    if (!configured[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = 256ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      configured[dev] = true;
    }
  }
  return cudaMallocAsync(p, bytes < 256 ? 256 : bytes, stream);
}

// Host -> device copy done by SMs reading host-mapped pinned memory over the
// link (16 bytes per load), so it never queues behind copy-engine transfers
// already in flight (pv_upload).
__global__ void __launch_bounds__(256) upload_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                     uint64_t n16, uint8_t* __restrict__ dst_tail,
                                                     const uint8_t* __restrict__ src_tail, uint32_t tail) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
}

__global__ void scatter_pages_kernel(uint8_t* __restrict__ image, uint64_t image_pages,
                                     const uint64_t* __restrict__ pfns, uint64_t n, const uint8_t* __restrict__ src) {
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t pfn = pfns[i];
    if (pfn >= image_pages) continue;
    const uint4* s = reinterpret_cast<const uint4*>(src + i * kPageSize);
    uint4* d = reinterpret_cast<uint4*>(image + pfn * kPageSize);
    for (uint32_t j = threadIdx.x; j < kPageSize / 16; j += blockDim.x) d[j] = s[j];
  }
}

__global__ void gather_pages_kernel(const uint8_t* __restrict__ image, uint64_t image_pages,
                                    const uint64_t* __restrict__ pfns, uint64_t n, uint8_t* __restrict__ dst) {
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t pfn = pfns[i];
    if (pfn >= image_pages) continue;
    const uint4* s = reinterpret_cast<const uint4*>(image + pfn * kPageSize);
    uint4* d = reinterpret_cast<uint4*>(dst + i * kPageSize);
    for (uint32_t j = threadIdx.x; j < kPageSize / 16; j += blockDim.x) d[j] = s[j];
  }
}

static inline int rc(cudaError_t e) { return e == cudaSuccess ? PV_SUCCESS : PV_ECUDA - (int)e; }

}  // namespace pv

using namespace pv;

extern "C" {

int pv_abi_version(void) { return PV_ABI_VERSION; }

uint64_t pv_translate_chunk(void) { return translate_chunk(); }

const char* pv_status_name(uint32_t status) {
  switch (PV_ST_KIND(status)) {
    case PV_ST_OK: return "ok";
    case PV_ST_FAULT: return "page_fault";
    case PV_ST_FAULT2: return "page_fault_tdp";
    case PV_ST_TRAP: return "trap_exit";
    case PV_ST_TRAP2: return "trap_exit_tdp";
    case PV_ST_NODE_OOR: return "node_out_of_range";
    case PV_ST_NODE_OOR2: return "node_out_of_range_tdp";
    case PV_ST_DATA_OOR: return "out_of_range";
    case PV_ST_CONFLICT: return "conflict";
    default: return "unknown";
  }
}

int pv_translate(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                 uint32_t n_segs, uint64_t n_chunks, const void* vas, uint32_t flags, const pv_index* index,
                 uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux, void* stream) {
  if (n_chunks == 0) return PV_SUCCESS;
  const bool packed = flags & PV_OUT_PACKED;
  if (!image || !spaces || !segs || !vas || !out_value || (!out_status && !packed) || n_segs == 0) return PV_EINVAL;
  if (image_bytes % kPageSize) return PV_EINVAL;
  // 4-byte walk codes carry leaf pfns in 28 bits (pv_translate.cu stage_codes)
  if (image_bytes >= (1ull << 40)) return PV_EINVAL;
  if (flags & ~(uint32_t)(PV_VA32 | PV_OUT_PFN | PV_OUT_PACKED | PV_CONCURRENT | PV_HAS_TWO_STAGE | PV_HAS_4L))
    return PV_EINVAL;
  const bool two = flags & PV_HAS_TWO_STAGE;
  // packed lanes spill wide values into out_aux (only u64 VAs, TDP stages and 4-level walks can)
  if (packed && !out_aux && (!(flags & PV_VA32) || two || (flags & PV_HAS_4L))) return PV_EINVAL;
  if (index != nullptr && (!index->slot_of || !index->leaf_codes || !index->slot_page)) return PV_EINVAL;
  return rc(launch_translate(image, image_bytes, spaces, segs, n_segs, n_chunks, vas,
                             flags & (PV_VA32 | PV_OUT_PFN | PV_OUT_PACKED | PV_CONCURRENT | PV_HAS_4L), two, index,
                             out_value, out_status, out_aux, nullptr, (cudaStream_t)stream));
}

int pv_translate_words(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_seg* segs,
                       uint32_t n_segs, uint64_t n_chunks, const void* vas, uint32_t flags, const pv_index* index,
                       uint32_t* out_word, pv_exc* exc, uint64_t exc_cap, unsigned long long* exc_count,
                       uint64_t lane_base, void* stream) {
  if (n_chunks == 0) return PV_SUCCESS;
  if (!image || !spaces || !segs || !vas || !out_word || !exc_count || (!exc && exc_cap) || n_segs == 0)
    return PV_EINVAL;
  if (image_bytes % kPageSize) return PV_EINVAL;
  // frame numbers fill 28 bits of a word (and of the walk codes)
  if (image_bytes >= (1ull << 40)) return PV_EINVAL;
  if (flags & ~(uint32_t)(PV_VA32 | PV_OUT_PFN | PV_CONCURRENT | PV_HAS_TWO_STAGE | PV_HAS_4L)) return PV_EINVAL;
  if (index != nullptr && (!index->slot_of || !index->leaf_codes || !index->slot_page)) return PV_EINVAL;
  const ExcSink sink{exc, exc_cap / PV_EXC_STRIPES, exc_count, lane_base};
  return rc(launch_translate(image, image_bytes, spaces, segs, n_segs, n_chunks, vas,
                             flags & (PV_VA32 | PV_OUT_PFN | PV_CONCURRENT | PV_HAS_4L), flags & PV_HAS_TWO_STAGE,
                             index, reinterpret_cast<uint64_t*>(out_word), nullptr, nullptr, &sink,
                             (cudaStream_t)stream));
}

int pv_index_encode(const uint8_t* image, uint64_t image_bytes, const uint64_t* slot_page, const uint64_t* slots,
                    uint64_t first_slot, uint64_t n, uint32_t* leaf_codes, const uint8_t* dirty, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !slot_page || !leaf_codes || image_bytes % kPageSize) return PV_EINVAL;
  return rc(launch_index_encode(image, image_bytes, slot_page, slots, first_slot, n, leaf_codes, dirty,
                                (cudaStream_t)stream));
}

uint64_t pv_fifo_scratch_bytes(uint64_t n_lookups, uint64_t n_windows, uint32_t capacity) {
  return fifo_scratch_bytes(n_lookups, n_windows, capacity);
}

int pv_fifo_replay(const void* vas, uint32_t flags, const uint64_t* lane_idx, const uint64_t* proc_off,
                   const uint64_t* win_off, uint32_t n_procs, uint64_t n_lookups, uint64_t n_windows,
                   uint32_t capacity, pv_fifo* fifo, uint64_t* value, uint32_t* status, void* scratch,
                   uint64_t scratch_bytes, void* stream) {
  if (n_procs == 0) return PV_SUCCESS;
  if (!vas || !lane_idx || !proc_off || !win_off || !fifo || !value || !status || !scratch) return PV_EINVAL;
  if (capacity < 1 || capacity > PV_FIFO_MAX) return PV_EINVAL;
  return rc(launch_fifo_lanes_abi(vas, flags, lane_idx, proc_off, win_off, n_procs, n_lookups, n_windows, capacity,
                                  fifo, value, status, scratch, scratch_bytes, (cudaStream_t)stream));
}

int pv_copy_plan(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_op* ops,
                 uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages, uint32_t direction, uint64_t* page_hpa,
                 uint32_t* page_status, uint64_t* page_aux, uint64_t* op_first_bad, uint64_t* page_owner,
                 uint32_t epoch, uint32_t* conflict, void* stream) {
  if (n_pages == 0) return PV_SUCCESS;
  if (!image || !spaces || !ops || !page_off || !page_hpa || !page_status || !op_first_bad || n_ops == 0)
    return PV_EINVAL;
  if (direction != PV_TO_GUEST && direction != PV_FROM_GUEST) return PV_EINVAL;
  if (image_bytes % kPageSize) return PV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_copy_plan(image, image_bytes, spaces, ops, n_ops, page_off, n_pages, page_hpa, page_status,
                                   page_aux, op_first_bad, nullptr, 0, s);
  if (e != cudaSuccess) return rc(e);
  if (direction == PV_TO_GUEST && page_owner != nullptr) {
    if (!conflict) return PV_EINVAL;
    e = launch_copy_stamp(page_off, n_ops, n_pages, page_hpa, op_first_bad, page_owner, image_bytes / kPageSize,
                          epoch, conflict, nullptr, s);
  }
  return rc(e);
}

int pv_copy_plan_nodes(const uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_op* ops,
                       uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages, uint64_t* page_hpa,
                       uint32_t* page_status, uint64_t* page_aux, uint64_t* op_first_bad, uint32_t* node_map,
                       uint64_t node_pages, uint32_t epoch, void* stream) {
  if (n_pages == 0) return PV_SUCCESS;
  if (!image || !spaces || !ops || !page_off || !page_hpa || !page_status || !op_first_bad || !node_map ||
      n_ops == 0)
    return PV_EINVAL;
  if (image_bytes % kPageSize || node_pages < image_bytes / kPageSize || epoch == 0) return PV_EINVAL;
  return rc(launch_copy_plan(image, image_bytes, spaces, ops, n_ops, page_off, n_pages, page_hpa, page_status,
                             page_aux, op_first_bad, node_map, epoch, (cudaStream_t)stream));
}

int pv_copy_stamp(const uint64_t* page_off, uint64_t n_ops, uint64_t n_pages, const uint64_t* page_hpa,
                  const uint64_t* op_first_bad, uint64_t* page_owner, uint64_t owner_pages, uint32_t epoch,
                  uint32_t* conflict, const uint32_t* node_map, void* stream) {
  if (n_pages == 0) return PV_SUCCESS;
  if (!page_off || !page_hpa || !op_first_bad || !page_owner || !conflict) return PV_EINVAL;
  return rc(launch_copy_stamp(page_off, n_ops, n_pages, page_hpa, op_first_bad, page_owner, owner_pages, epoch,
                              conflict, node_map, (cudaStream_t)stream));
}

int pv_copy_exec(uint8_t* image, uint64_t image_bytes, const pv_op* ops, uint64_t n_ops, const uint64_t* page_off,
                 uint64_t n_pages, uint32_t direction, const uint64_t* page_hpa, const uint32_t* page_status,
                 const uint64_t* page_aux, const uint64_t* op_first_bad, uint8_t* buf, uint64_t buf_bytes,
                 pv_op_result* results, uint8_t* dirty, const uint32_t* abort_flag, void* stream) {
  if (n_pages == 0) return PV_SUCCESS;
  if (!image || !ops || !page_off || !page_hpa || !page_status || !op_first_bad || !buf || !results)
    return PV_EINVAL;
  if ((direction & ~PV_COPY_ALIGNED16) != PV_TO_GUEST && (direction & ~PV_COPY_ALIGNED16) != PV_FROM_GUEST)
    return PV_EINVAL;
  return rc(launch_copy_exec(image, image_bytes, ops, n_ops, page_off, n_pages, direction, page_hpa, page_status,
                             page_aux, op_first_bad, buf, buf_bytes, results, dirty, abort_flag,
                             (cudaStream_t)stream));
}

int pv_copy_fifo_replay(const pv_op* ops, const uint64_t* page_off, const uint64_t* look_page, const uint32_t* look_op,
                        const uint64_t* proc_off, const uint64_t* win_off, uint32_t n_procs, uint64_t n_lookups,
                        uint64_t n_windows, uint32_t capacity, pv_fifo* fifo, uint64_t image_bytes,
                        uint64_t* page_hpa, uint32_t* page_status, uint64_t* op_first_bad, void* scratch,
                        uint64_t scratch_bytes, void* stream) {
  if (n_procs == 0) return PV_SUCCESS;
  if (!ops || !page_off || !look_page || !look_op || !proc_off || !win_off || !fifo || !page_hpa || !page_status ||
      !op_first_bad || !scratch)
    return PV_EINVAL;
  if (capacity < 1 || capacity > PV_FIFO_MAX) return PV_EINVAL;
  return rc(launch_fifo_copy_abi(ops, page_off, look_page, look_op, proc_off, win_off, n_procs, n_lookups, n_windows,
                                 capacity, fifo, image_bytes, page_hpa, page_status, op_first_bad, scratch,
                                 scratch_bytes, (cudaStream_t)stream));
}

uint64_t pv_copy_shim_scratch_bytes(uint64_t n_pages) { return shim_scratch_bytes(n_pages); }

int pv_copy_shim(uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_shim* shims, const pv_op* ops,
                 uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages, uint64_t* page_hpa,
                 uint32_t* page_status, uint64_t* op_first_bad, uint8_t* dirty, uint64_t* n_written,
                 void* scratch, uint64_t scratch_bytes, void* stream) {
  if (n_pages == 0) return PV_SUCCESS;
  if (!image || !spaces || !shims || !ops || !page_off || !page_hpa || !page_status || !op_first_bad || !scratch ||
      n_ops == 0)
    return PV_EINVAL;
  if (image_bytes % kPageSize || scratch_bytes < shim_scratch_bytes(n_pages)) return PV_EINVAL;
  return rc(launch_copy_shim(image, image_bytes, spaces, shims, ops, n_ops, page_off, n_pages, page_hpa, page_status,
                             op_first_bad, dirty, n_written, scratch, (cudaStream_t)stream));
}

int pv_frame_pack(const uint64_t* ops, uint64_t n, const uint64_t* vcpu, const uint64_t* cr3, const uint64_t* tag,
                  const uint64_t* frame_off, pv_frame* frames, uint32_t* status, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!ops || !vcpu || !cr3 || !tag || !frame_off || !frames || !status) return PV_EINVAL;
  return rc(launch_frame_pack(ops, n, vcpu, cr3, tag, frame_off, frames, status, (cudaStream_t)stream));
}

int pv_frame_identify(const pv_frame* frames, uint64_t n, const int32_t* vcpu_guest, uint32_t n_vcpus,
                      const uint64_t* reg_guest, const uint64_t* reg_cr3, uint32_t n_reg, uint32_t* record,
                      uint32_t* status, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!frames || !record || !status || (n_vcpus && !vcpu_guest) || (n_reg && (!reg_guest || !reg_cr3)))
    return PV_EINVAL;
  return rc(launch_frame_identify(frames, n, vcpu_guest, n_vcpus, reg_guest, reg_cr3, n_reg, record, status,
                                  (cudaStream_t)stream));
}

uint64_t pv_frame_assemble_scratch_bytes(uint64_t n) { return frame_scratch_bytes(n); }

int pv_frame_assemble(const pv_frame* frames, uint64_t n, const uint32_t* record, uint64_t* ops_out, uint32_t* status,
                      void* scratch, uint64_t scratch_bytes, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!frames || !record || !ops_out || !status || !scratch || n >= 0xFFFFFFFFull) return PV_EINVAL;
  if (scratch_bytes < frame_scratch_bytes(n)) return PV_EINVAL;
  return rc(launch_frame_assemble(frames, n, record, ops_out, status, scratch, scratch_bytes, (cudaStream_t)stream));
}

uint64_t pv_map_scratch_bytes(void) { return map_scratch_bytes(); }

int pv_map_plan(const uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root_pfn, const uint64_t* vas,
                uint64_t n, uint8_t* need, uint64_t* bad, void* scratch, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !vas || !need || !bad || !scratch || image_bytes % kPageSize || base % kPageSize) return PV_EINVAL;
  if (n >= 0xFFFFFFFFull) return PV_EINVAL;
  return rc(launch_map_plan(image, image_bytes, base, root_pfn, vas, n, need, bad, scratch, (cudaStream_t)stream));
}

int pv_map_commit(uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root_pfn, const uint64_t* vas,
                  uint64_t n, const uint8_t* need, const uint64_t* frames, uint64_t n_frames,
                  const uint64_t* frame_off, const uint8_t* hot, uint32_t data_first, const uint64_t* targets,
                  uint64_t target_add, uint64_t leaf_flags, uint64_t* out_data, uint8_t* dirty, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !vas || !need || !frame_off || image_bytes % kPageSize || base % kPageSize) return PV_EINVAL;
  if (n_frames && !frames) return PV_EINVAL;
  if (!data_first && !targets) return PV_EINVAL;
  return rc(launch_map_commit(image, image_bytes, base, root_pfn, vas, n, need, frames, n_frames, frame_off, hot,
                              data_first ? 1u : 0u, targets, target_add, leaf_flags, out_data, dirty,
                              (cudaStream_t)stream));
}

int pv_walk_one(const uint8_t* image, uint64_t image_bytes, const pv_space* space, uint64_t va, uint32_t flags,
                pv_one_result* out, uint64_t seq, void* stream) {
  if (!image || !space || !out || image_bytes % kPageSize) return PV_EINVAL;
  if (flags & ~(uint32_t)PV_OUT_PFN) return PV_EINVAL;
  return rc(launch_walk_one(image, image_bytes, *space, va, flags, out, seq, (cudaStream_t)stream));
}

int pv_copy_small(uint8_t* image, uint64_t image_bytes, const pv_small_op* op, uint8_t* buf, uint64_t buf_bytes,
                  pv_small_result* out, uint8_t* dirty, uint64_t seq, void* stream) {
  if (!image || !op || !out || image_bytes % kPageSize) return PV_EINVAL;
  if (op->direction != PV_TO_GUEST && op->direction != PV_FROM_GUEST) return PV_EINVAL;
  const uint64_t n = page_span(op->gva, op->len);
  if (n > PV_SMALL_PAGES) return PV_EINVAL;
  if (n != 0 && !buf) return PV_EINVAL;
  return rc(launch_copy_small(image, image_bytes, *op, buf, buf_bytes, out, dirty, (uint32_t)n, seq,
                              (cudaStream_t)stream));
}

}  // extern "C"

namespace {
// One per-call server per device (pv_copy.cu server_kernel): its mailbox,
// private non-blocking stream and request counter; requests of all host
// threads are serialised by the mutex.
struct ServerSlot {
  std::mutex mu;
  ServerBox* box = nullptr;
  cudaStream_t stream = nullptr;
  uint64_t seq = 0;
};
constexpr int kMaxDevices = 64;
ServerSlot g_server[kMaxDevices];

uint64_t server_idle_ns() {
  static const uint64_t v = [] {
    const char* e = std::getenv("PV_SERVER_IDLE_US");
    const long us = e ? std::atol(e) : 200;
    return (uint64_t)(us > 0 ? us : 200) * 1000ull;
  }();
  return v;
}

// Post the request `fill` writes into the mailbox and wait for its reply
// (slot lock held by the caller).  Launches the server when it is not
// resident; returns a PV_ code.
int server_box(ServerSlot& S) {
  if (S.box != nullptr) return PV_SUCCESS;
  cudaStream_t st = nullptr;
  const cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return PV_ECUDA - (int)e;
  void* p = nullptr;
  if (cudaHostAlloc(&p, sizeof(ServerBox), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaStreamDestroy(st);
    return PV_ENOMEM;
  }
  std::memset(p, 0, sizeof(ServerBox));
  S.stream = st;
  S.box = static_cast<ServerBox*>(p);
  S.box->state = kServerExited;
  return PV_SUCCESS;
}

template <class Fill>
int server_roundtrip(ServerSlot& S, Fill fill) {
  const int rb = server_box(S);
  if (rb != PV_SUCCESS) return rb;
  ServerBox* box = S.box;
  fill(box->req);
  const uint64_t sq = ++S.seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  box->req_seq = sq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  auto launch = [&]() -> int {
    box->state = kServerLaunched;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    const cudaError_t e = launch_server(box, server_idle_ns(), S.stream);
    return e == cudaSuccess ? PV_SUCCESS : PV_ECUDA - (int)e;
  };
  if (box->state == kServerExited) {
    const int r = launch();
    if (r != PV_SUCCESS) return r;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t it = 1; box->rep_seq != sq; ++it) {
    if ((it & 1023) == 0) {
      // the server may have idled out just before the request landed
      if (box->state == kServerExited && box->rep_seq != sq) {
        const int r = launch();
        if (r != PV_SUCCESS) return r;
      }
      const cudaError_t e = cudaStreamQuery(S.stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return PV_ECUDA - (int)e;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        return PV_ECUDA - (int)cudaErrorLaunchTimeout;
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return PV_SUCCESS;
}

ServerSlot* server_slot() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  return &g_server[dev];
}
}  // namespace

extern "C" {

// Spin until *seq_word == sq (a stream-ordered per-call launch publishing
// into the mailbox), checking `stream` for errors now and then.
static int wait_published(const volatile uint64_t* seq_word, uint64_t sq, cudaStream_t stream) {
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t it = 1; *seq_word != sq; ++it) {
    if ((it & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return PV_ECUDA - (int)e;
      if (e == cudaSuccess && *seq_word != sq) return PV_ECUDA - (int)cudaErrorUnknown;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        return PV_ECUDA - (int)cudaErrorLaunchTimeout;
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return PV_SUCCESS;
}

int pv_server_walk(const uint8_t* image, uint64_t image_bytes, const pv_space* space, uint64_t va, uint32_t flags,
                   pv_one_result* out, void* stream) {
  if (!image || !space || !out || image_bytes % kPageSize) return PV_EINVAL;
  if (flags & ~(uint32_t)(PV_OUT_PFN | PV_SERVER_IDLE)) return PV_EINVAL;
  ServerSlot* S = server_slot();
  if (!S) return PV_EINVAL;
  std::lock_guard<std::mutex> lk(S->mu);
  int r;
  const cudaError_t q = (flags & PV_SERVER_IDLE) ? cudaSuccess : cudaStreamQuery((cudaStream_t)stream);
  flags &= PV_OUT_PFN;
  if (q == cudaSuccess) {
    r = server_roundtrip(*S, [&](ServerReq& req) {
      req.kind = kServerWalk;
      req.flags = flags;
      req.image = (uint64_t)image;
      req.image_bytes = image_bytes;
      req.va = va;
      req.op.space = *space;
    });
  } else if (q == cudaErrorNotReady) {  // queued work first: the stream-ordered launch
    r = server_box(*S);
    if (r != PV_SUCCESS) return r;
    const uint64_t sq = ++S->seq;
    const cudaError_t e = launch_walk_one(image, image_bytes, *space, va, flags, &S->box->one, sq,
                                          (cudaStream_t)stream);
    if (e != cudaSuccess) return PV_ECUDA - (int)e;
    r = wait_published(&S->box->one.seq, sq, (cudaStream_t)stream);
  } else {
    return PV_ECUDA - (int)q;
  }
  if (r != PV_SUCCESS) return r;
  out->value = S->box->one.value;
  out->aux = S->box->one.aux;
  out->status = S->box->one.status;
  out->seq = S->seq;
  return PV_SUCCESS;
}

int pv_server_copy_small(uint8_t* image, uint64_t image_bytes, const pv_small_op* op, uint8_t* buf,
                         uint64_t buf_bytes, pv_small_result* out, uint8_t* dirty, uint32_t flags,
                         void* stream) {
  if (!image || !op || !out || image_bytes % kPageSize) return PV_EINVAL;
  if (op->direction != PV_TO_GUEST && op->direction != PV_FROM_GUEST) return PV_EINVAL;
  const uint64_t n = page_span(op->gva, op->len);
  if (n > PV_SMALL_PAGES) return PV_EINVAL;
  if (n != 0 && !buf) return PV_EINVAL;
  if (flags & ~(uint32_t)PV_SERVER_IDLE) return PV_EINVAL;
  ServerSlot* S = server_slot();
  if (!S) return PV_EINVAL;
  std::lock_guard<std::mutex> lk(S->mu);
  int r;
  const cudaError_t q = (flags & PV_SERVER_IDLE) ? cudaSuccess : cudaStreamQuery((cudaStream_t)stream);
  if (q == cudaSuccess) {
    r = server_roundtrip(*S, [&](ServerReq& req) {
      req.kind = kServerCopy;
      req.flags = 0;
      req.image = (uint64_t)image;
      req.image_bytes = image_bytes;
      req.buf = (uint64_t)buf;
      req.buf_bytes = buf_bytes;
      req.dirty = (uint64_t)dirty;
      req.n_pages = (uint32_t)n;
      std::memcpy(&req.op, op, sizeof(pv_small_op) - sizeof(uint64_t) * (PV_SMALL_PAGES - n));
    });
  } else if (q == cudaErrorNotReady) {
    r = server_box(*S);
    if (r != PV_SUCCESS) return r;
    const uint64_t sq = ++S->seq;
    const cudaError_t e = launch_copy_small(image, image_bytes, *op, buf, buf_bytes, &S->box->small, dirty,
                                            (uint32_t)n, sq, (cudaStream_t)stream);
    if (e != cudaSuccess) return PV_ECUDA - (int)e;
    r = wait_published(&S->box->small.seq, sq, (cudaStream_t)stream);
  } else {
    return PV_ECUDA - (int)q;
  }
  if (r != PV_SUCCESS) return r;
  const pv_small_result& res = S->box->small;
  out->op = res.op;
  std::memcpy(out->page_hpa, res.page_hpa, n * sizeof(uint64_t));
  std::memcpy(out->page_status, res.page_status, n * sizeof(uint32_t));
  out->seq = S->seq;
  return PV_SUCCESS;
}

int pv_server_stop(void) {
  ServerSlot* S = server_slot();
  if (!S) return PV_EINVAL;
  std::lock_guard<std::mutex> lk(S->mu);
  if (S->box == nullptr || S->box->state == kServerExited) return PV_SUCCESS;
  const int r = server_roundtrip(*S, [&](ServerReq& q) { q.kind = kServerStop; });
  if (r != PV_SUCCESS) return r;
  const cudaError_t e = cudaStreamSynchronize(S->stream);
  return e == cudaSuccess ? PV_SUCCESS : PV_ECUDA - (int)e;
}

int pv_server_resident(void) {
  ServerSlot* S = server_slot();
  if (!S) return 0;
  std::lock_guard<std::mutex> lk(S->mu);
  return S->box != nullptr && S->box->state != kServerExited;
}

void* pv_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return p;
}

void pv_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

uint64_t pv_copy_ordered_scratch_bytes(uint64_t n_pages, uint64_t image_bytes) {
  return ordered_scratch_bytes(n_pages, image_bytes >> kPageShift);
}

int pv_copy_ordered(uint8_t* image, uint64_t image_bytes, const pv_op* ops, uint64_t n_ops, const uint64_t* page_off,
                    uint64_t n_pages, const uint64_t* page_hpa, const uint32_t* page_status,
                    const uint64_t* page_aux, const uint64_t* op_first_bad, const uint8_t* buf, uint64_t buf_bytes,
                    pv_op_result* results, uint8_t* dirty, void* scratch, uint64_t scratch_bytes, void* stream) {
  if (n_ops == 0) return PV_SUCCESS;
  if (!image || !ops || !page_off || !page_hpa || !page_status || !op_first_bad || !buf || !results || !scratch)
    return PV_EINVAL;
  if (image_bytes % kPageSize) return PV_EINVAL;
  return rc(launch_copy_ordered(image, image_bytes, ops, n_ops, page_off, n_pages, page_hpa, page_status, page_aux,
                                op_first_bad, buf, buf_bytes, results, dirty, scratch, scratch_bytes,
                                (cudaStream_t)stream));
}

int pv_result_encode(uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa, const uint32_t* header,
                     const uint8_t* blob_buf, const uint64_t* blob_off, uint64_t n, uint32_t* status, uint8_t* dirty,
                     void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !page_hpa || !header || !blob_off || !status) return PV_EINVAL;
  return rc(launch_result_encode(image, image_bytes, page_hpa, header, blob_buf, blob_off, n, status, dirty,
                                 (cudaStream_t)stream));
}

int pv_result_decode(const uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa, uint64_t n,
                     uint32_t* header, uint32_t* status, void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !page_hpa || !header || !status) return PV_EINVAL;
  return rc(launch_result_decode(image, image_bytes, page_hpa, n, header, status, (cudaStream_t)stream));
}

int pv_scatter_pages(uint8_t* image, uint64_t image_bytes, const uint64_t* pfns, uint64_t n, const uint8_t* src,
                     void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !pfns || !src || image_bytes % kPageSize) return PV_EINVAL;
  const uint64_t grid = n < 4096 ? n : 4096;
  scatter_pages_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(image, image_bytes / kPageSize, pfns, n, src);
  return rc(cudaGetLastError());
}

int pv_upload(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return PV_SUCCESS;
  if (!dst || !src || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15))
    return PV_EINVAL;
  const uint64_t n16 = bytes / 16;
  uint64_t grid = (n16 + 255) / 256;
  if (grid > 148) grid = 148;
  if (grid == 0) grid = 1;
  upload_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16, static_cast<uint8_t*>(dst) + n16 * 16,
      static_cast<const uint8_t*>(src) + n16 * 16, (uint32_t)(bytes & 15));
  return rc(cudaGetLastError());
}

int pv_gather_pages(const uint8_t* image, uint64_t image_bytes, const uint64_t* pfns, uint64_t n, uint8_t* dst,
                    void* stream) {
  if (n == 0) return PV_SUCCESS;
  if (!image || !pfns || !dst || image_bytes % kPageSize) return PV_EINVAL;
  const uint64_t grid = n < 4096 ? n : 4096;
  gather_pages_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(image, image_bytes / kPageSize, pfns, n, dst);
  return rc(cudaGetLastError());
}

int pv_timing(int enable) { return rc(timing_enable(enable != 0)); }

double pv_timing_ms(const char* kernel, uint64_t* launches) { return timing_ms(kernel, launches); }

}  // extern "C"

// ---- SM partitions (green contexts through driver entry points: no libcuda link)
namespace {
struct SmSplit {
  uint32_t want = 0;
  void* green[2] = {nullptr, nullptr};
  cudaStream_t stream[2] = {nullptr, nullptr};
  uint32_t sms[2] = {0, 0};
};
std::mutex g_split_mu;
std::unordered_map<uint64_t, SmSplit> g_splits;  // (device << 32 | want) -> partition

template <class F>
bool driver_fn(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      p == nullptr)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}
}  // namespace

extern "C" {

int pv_sm_split(uint32_t first_sms, uint32_t flags, void** stream_first, void** stream_rest, uint32_t* sms_first,
                uint32_t* sms_rest) {
  if (!stream_first || !stream_rest || first_sms == 0 ||
      (flags & ~(uint32_t)(PV_SM_SPLIT_FINE | PV_SM_SPLIT_INTERLEAVE)))
    return PV_EINVAL;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return rc(e);
  std::lock_guard<std::mutex> lk(g_split_mu);
  SmSplit& P = g_splits[((uint64_t)dev << 34) | ((uint64_t)(flags & 3u) << 32) | first_sms];
  if (P.stream[0] == nullptr) {
    CUresult (*getres)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned) = nullptr;
    CUresult (*gendesc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
    CUresult (*gcreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
    CUresult (*gstream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
    CUresult (*getdev)(CUdevice*, int) = nullptr;
    if (!driver_fn("cuDeviceGetDevResource", &getres) || !driver_fn("cuDevSmResourceSplitByCount", &split) ||
        !driver_fn("cuDevResourceGenerateDesc", &gendesc) || !driver_fn("cuGreenCtxCreate", &gcreate) ||
        !driver_fn("cuGreenCtxStreamCreate", &gstream) || !driver_fn("cuDeviceGet", &getdev))
      return PV_ECUDA - (int)cudaErrorNotSupported;
    CUdevice cd;
    CUdevResource all, rem;
    // PV_SM_SPLIT_FINE: single-SM granularity (CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING) instead of
    // the driver's co-scheduled 8-SM groups; PV_SM_SPLIT_INTERLEAVE: the device is cut into groups of that
    // granularity and the first set takes every other group.  Each is a different placement of the two
    // sets over the GPCs; which is fastest depends on the box (profiles/r02_split_ab.md)
    const unsigned use = (flags & PV_SM_SPLIT_FINE) ? CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING : 0u;
    if (getdev(&cd, dev) != CUDA_SUCCESS || getres(cd, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
        first_sms >= all.sm.smCount)
      return PV_EINVAL;
    std::vector<CUdevResource> groups;
    std::vector<CUdevResource> sets[2];
    if (flags & PV_SM_SPLIT_INTERLEAVE) {
      const unsigned g = (flags & PV_SM_SPLIT_FINE) ? 1u : 8u;
      unsigned nb = 0;
      if (split(nullptr, &nb, &all, nullptr, use, g) != CUDA_SUCCESS || nb == 0) return PV_EINVAL;
      groups.resize(nb);
      if (split(groups.data(), &nb, &all, &rem, use, g) != CUDA_SUCCESS) return PV_EINVAL;
      groups.resize(nb);
      unsigned have = 0;
      std::vector<bool> taken(nb, false);
      for (unsigned pass = 0; pass < 2 && have < first_sms; ++pass)  // even groups first, then odd ones
        for (unsigned k = pass; k < nb && have < first_sms; k += 2) {
          taken[k] = true;
          have += groups[k].sm.smCount;
        }
      for (unsigned k = 0; k < nb; ++k) sets[taken[k] ? 0 : 1].push_back(groups[k]);
      if (rem.sm.smCount) sets[1].push_back(rem);
    } else {
      CUdevResource grp[1];
      unsigned nb = 1;
      if (split(grp, &nb, &all, &rem, use, first_sms) != CUDA_SUCCESS || nb != 1) return PV_EINVAL;
      sets[0].push_back(grp[0]);
      sets[1].push_back(rem);
    }
    if (sets[0].empty() || sets[1].empty()) return PV_EINVAL;
    for (int i = 0; i < 2; ++i) {
      CUdevResourceDesc d;
      CUgreenCtx g;
      CUstream cs;
      if (gendesc(&d, sets[i].data(), (unsigned)sets[i].size()) != CUDA_SUCCESS ||
          gcreate(&g, d, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
          gstream(&cs, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
        return PV_ECUDA - (int)cudaErrorNotSupported;
      P.green[i] = g;
      P.stream[i] = (cudaStream_t)cs;
      uint32_t n = 0;
      for (const auto& r : sets[i]) n += r.sm.smCount;
      P.sms[i] = n;
    }
  }
  *stream_first = P.stream[0];
  *stream_rest = P.stream[1];
  if (sms_first) *sms_first = P.sms[0];
  if (sms_rest) *sms_rest = P.sms[1];
  return PV_SUCCESS;
}

int pv_peer_alloc(uint64_t bytes, void** dev_ptr, uint8_t* handle) {
  if (!dev_ptr || !handle || bytes == 0) return PV_EINVAL;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? PV_ENOMEM : rc(e);
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return rc(e);
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == PV_PEER_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *dev_ptr = p;
  return PV_SUCCESS;
}

int pv_peer_open(const uint8_t* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return PV_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return rc(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int pv_peer_close(void* dev_ptr) { return dev_ptr ? rc(cudaIpcCloseMemHandle(dev_ptr)) : PV_EINVAL; }

int pv_peer_free(void* dev_ptr) { return dev_ptr ? rc(cudaFree(dev_ptr)) : PV_EINVAL; }

int pv_memcpy(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return PV_SUCCESS;
  if (!dst || !src) return PV_EINVAL;
  return rc(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
}

uint32_t pv_set_sm_budget(uint32_t sms) {
  const uint32_t old = t_sm_budget;
  t_sm_budget = sms;
  return old;
}

int pv_stream_idle(void* stream) {
  const cudaError_t e = cudaStreamQuery((cudaStream_t)stream);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) return 0;
  return rc(e);
}

int pv_stream_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  return rc(e);
}

}  // extern "C"
