// pv_wire.cu — batched result-page codec.
//
// The reference's non-blocking path writes each completed operation's
// record into the issuing thread's result page (resultpage.py:44-51,
// backend.py:352-355): little-endian header {status u32, flags u32,
// values 6 x u32, blob_len u32} (36 bytes) followed by an inline blob of up
// to 4060 bytes; the guest decodes it (resultpage.py:54-61,
// frontend.py:182-184).  Here a batch of records is encoded into / decoded
// from the HBM image in one launch: one warp per record, the 36-byte header
// written by 9 lanes, the <= 4060-byte blob moved by all 32 lanes.  A batch
// holds at most one record per result page (one operation in flight per
// guest thread, frontend.py:151-154), so records never overlap.
#include "pv_common.cuh"

namespace pv {

constexpr uint32_t kHeaderBytes = 36;
constexpr uint32_t kBlobCapacity = kPageSize - kHeaderBytes;  // 4060

__global__ void result_encode_kernel(uint8_t* __restrict__ image, uint64_t image_bytes,
                                     const uint64_t* __restrict__ page_hpa, const uint32_t* __restrict__ header,
                                     const uint8_t* __restrict__ blob_buf, const uint64_t* __restrict__ blob_off,
                                     uint64_t n, uint32_t* __restrict__ out_status, uint8_t* __restrict__ dirty) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nwarps) {
    const uint32_t* h = header + r * 9;  // status, flags, values[6], blob_len
    const uint32_t blob_len = h[8];
    const uint64_t hpa = page_hpa[r];
    const uint64_t total = kHeaderBytes + (uint64_t)blob_len;
    // PhysMem.write bounds check (memvirt.py:156-158); the codec itself
    // rejects oversized blobs (resultpage.py:46-47).
    uint32_t st = PV_ST_OK;
    if (blob_len > kBlobCapacity) st = PV_ST_CONFLICT;  // reported as ValueError by the host
    else if (hpa + total > image_bytes || hpa + total < hpa) st = PV_ST_DATA_OOR;
    if (lane == 0) out_status[r] = st;
    if (st != PV_ST_OK) continue;
    uint8_t* dst = image + hpa;
    if (lane < 9) {
      const uint32_t v = h[lane];
      // header words may be unaligned if hpa is: store bytes
      dst[lane * 4 + 0] = (uint8_t)v;
      dst[lane * 4 + 1] = (uint8_t)(v >> 8);
      dst[lane * 4 + 2] = (uint8_t)(v >> 16);
      dst[lane * 4 + 3] = (uint8_t)(v >> 24);
    }
    const uint8_t* src = blob_buf + blob_off[r];
    for (uint32_t i = lane; i < blob_len; i += 32) dst[kHeaderBytes + i] = src[i];
    if (dirty != nullptr && lane == 0) {
      dirty[hpa >> kPageShift] = 1;
      dirty[(hpa + total - 1) >> kPageShift] = 1;
    }
  }
}

__global__ void result_decode_kernel(const uint8_t* __restrict__ image, uint64_t image_bytes,
                                     const uint64_t* __restrict__ page_hpa, uint64_t n,
                                     uint32_t* __restrict__ header_out, uint32_t* __restrict__ out_status) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * 9; i += stride) {
    const uint64_t r = i / 9;
    const uint32_t w = (uint32_t)(i % 9);
    const uint64_t hpa = page_hpa[r];
    const bool ok = hpa + kHeaderBytes <= image_bytes && hpa + kHeaderBytes > hpa;
    if (w == 0) out_status[r] = ok ? PV_ST_OK : PV_ST_DATA_OOR;
    if (!ok) continue;
    const uint8_t* p = image + hpa + 4 * w;
    header_out[i] = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
  }
}

cudaError_t launch_result_encode(uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa,
                                 const uint32_t* header, const uint8_t* blob_buf, const uint64_t* blob_off, uint64_t n,
                                 uint32_t* out_status, uint8_t* dirty, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n + 7) / 8;
  if (grid > 4096) grid = 4096;
  result_encode_kernel<<<(unsigned)grid, 256, 0, stream>>>(image, image_bytes, page_hpa, header, blob_buf, blob_off,
                                                           n, out_status, dirty);
  return cudaGetLastError();
}

cudaError_t launch_result_decode(const uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa, uint64_t n,
                                 uint32_t* header_out, uint32_t* out_status, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n * 9 + 255) / 256;
  if (grid > 4096) grid = 4096;
  result_decode_kernel<<<(unsigned)grid, 256, 0, stream>>>(image, image_bytes, page_hpa, n, header_out, out_status);
  return cudaGetLastError();
}

}  // namespace pv
