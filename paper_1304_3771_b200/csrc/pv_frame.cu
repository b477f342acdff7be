// pv_frame.cu — the forwarding wire format on the device.
//
// Reference (hypercall.py): a file operation travels as frames of one opcode
// plus exactly six 32-bit argument slots (ARG_LAYOUT, hypercall.py:46-58);
// page_fault needs seven words and travels as a first frame [tag, w0..w4]
// and a continuation frame (opcode 0x7F) [tag, w5, w6] (pack, :125-137).
// The receiver identifies the issuer from the vCPU and the virtual CR3
// (VcpuRegistry.identify, :178-211) and reassembles operations with a
// FrameAssembler whose pending first frames are keyed by (guest, process,
// tag) (:145-175).
//
// Device form, for batches of frames:
//   pack     : one thread per operation (frame slots at an exclusive scan of
//              1 / 2 frames per op), Unpackable for a layout word >= 2^32;
//   identify : per frame, vcpu -> guest from a dense table, (guest, cr3) ->
//              process record by binary search over the sorted registry;
//   assemble : single-frame operations decode in place; page-fault first and
//              continuation frames are compacted in order (CUB select),
//              stably sorted by (record, tag) (CUB radix sort) and every run
//              of one key replays the reference's pending-frame automaton
//              sequentially (runs are short).  An error never changes the
//              automaton's state in the reference (it raises before storing),
//              so per-frame outcomes of a batch equal feeding the frames one by
//              one and catching each error.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "pv_common.cuh"

namespace pv {

constexpr uint32_t kCont = 0x7F;
constexpr uint32_t kPageFault = 7;
constexpr int kFrTpb = 256;

// ARG_LAYOUT (hypercall.py:46-58) as indices into the FileOp field order
// (device_id 0, handle 1, gva 2, length 3, offset 4, flags 5, cmd 6,
// arg_gva 7, arg_len 8, prot 9, event_mask 10, timeout_ms 11, pid 12,
// access 13, vma_start 14, vma_length 15).
__constant__ int8_t kLayout[10][8] = {
    {-1},                         // 0: not a kind
    {0, 5, -1},                   // OPEN: device_id, flags
    {1, -1},                      // RELEASE: handle
    {1, 2, 3, 4, -1},             // READ: handle, gva, length, offset
    {1, 2, 3, 4, -1},             // WRITE
    {1, 6, 7, 8, 2, 5, -1},       // IOCTL: handle, cmd, arg_gva, arg_len, gva, flags
    {1, 2, 3, 9, 4, 5, -1},       // MMAP: handle, gva, length, prot, offset, flags
    {1, 2, 13, 14, 15, 4, 5, -1}, // PAGE_FAULT: handle, gva, access, vma_start, vma_length, offset, flags
    {1, 10, 11, -1},              // POLL: handle, event_mask, timeout_ms
    {1, 12, -1},                  // NOTIFY_SUBSCRIBE: handle, pid
};

__device__ __forceinline__ uint32_t layout_len(uint32_t kind) {
  uint32_t n = 0;
  while (n < 8 && kLayout[kind][n] >= 0) ++n;
  return n;
}

__global__ void __launch_bounds__(kFrTpb)
frame_pack_kernel(const uint64_t* __restrict__ ops, uint64_t n, const uint64_t* __restrict__ vcpu,
                  const uint64_t* __restrict__ cr3, const uint64_t* __restrict__ tag,
                  const uint64_t* __restrict__ frame_off, pv_frame* __restrict__ frames, uint32_t* __restrict__ status) {
  __shared__ uint64_t rows[kFrTpb * PV_FOP_WORDS];  // the tile's op rows, loaded with coalesced words
  const uint64_t n_tiles = (n + kFrTpb - 1) / kFrTpb;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i0 = tile * kFrTpb, i = i0 + threadIdx.x;
    const uint64_t words = (min((uint64_t)kFrTpb, n - i0)) * PV_FOP_WORDS;
    const uint64_t* src = ops + i0 * PV_FOP_WORDS;
    __syncthreads();
    for (uint64_t w = threadIdx.x; w < words; w += kFrTpb) rows[w] = src[w];
    __syncthreads();
    if (i >= n) continue;
    const uint64_t* op = rows + threadIdx.x * PV_FOP_WORDS;
    const uint32_t kind = (uint32_t)op[0];
    uint32_t st = PV_FRAME_OK;
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (kind < 1 || kind > 9 || op[0] > 9) {
      st = PV_FRAME_BAD_KIND;
    } else {
      // the layout's words, in layout order (unrolled over the 7 slots so w stays in registers)
#pragma unroll
      for (uint32_t k = 0; k < 7; ++k) {
        const int f = kLayout[kind][k];
        if (f < 0) break;
        const uint64_t v = op[1 + f];
        if (v > 0xFFFFFFFFull) {  // `0 <= value <= WORD_MASK` (hypercall.py:114-116)
          st = PV_FRAME_UNPACKABLE | ((uint32_t)f << 8);
          break;
        }
        w[k] = (uint32_t)v;
      }
    }
    status[i] = st;
    if (st != PV_FRAME_OK) continue;
    pv_frame* fo = frames + frame_off[i];
    const uint32_t vc = (uint32_t)vcpu[i];
    const uint64_t c3 = cr3[i];
    if (kind == kPageFault) {
      const uint32_t t = (uint32_t)tag[i];
      pv_frame a, b;
      a.opcode = kind;
      b.opcode = kCont;
      a.args[0] = b.args[0] = t;
      a.args[1] = w[0];
      a.args[2] = w[1];
      a.args[3] = w[2];
      a.args[4] = w[3];
      a.args[5] = w[4];
      b.args[1] = w[5];
      b.args[2] = w[6];
      b.args[3] = b.args[4] = b.args[5] = 0;
      a.vcpu = b.vcpu = vc;
      a.virtual_cr3 = b.virtual_cr3 = c3;
      fo[0] = a;
      fo[1] = b;
    } else {
      pv_frame a;
      a.opcode = kind;
      a.args[0] = w[0];
      a.args[1] = w[1];
      a.args[2] = w[2];
      a.args[3] = w[3];
      a.args[4] = w[4];
      a.args[5] = w[5];
      a.vcpu = vc;
      a.virtual_cr3 = c3;
      fo[0] = a;
    }
  }
}

__global__ void __launch_bounds__(kFrTpb)
frame_identify_kernel(const pv_frame* __restrict__ frames, uint64_t n, const int32_t* __restrict__ vcpu_guest,
                      uint32_t n_vcpus, const uint64_t* __restrict__ reg_guest, const uint64_t* __restrict__ reg_cr3,
                      uint32_t n_reg, uint32_t* __restrict__ record, uint32_t* __restrict__ status) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t vc = frames[i].vcpu;
    const int32_t g = vc < n_vcpus ? vcpu_guest[vc] : -1;
    if (g < 0) {
      status[i] = PV_FRAME_UNKNOWN_VCPU;
      record[i] = 0xFFFFFFFFu;
      continue;
    }
    const uint64_t c3 = frames[i].virtual_cr3;
    uint32_t lo = 0, hi = n_reg;  // first entry >= (g, c3)
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      const bool less = reg_guest[m] < (uint64_t)g || (reg_guest[m] == (uint64_t)g && reg_cr3[m] < c3);
      if (less) lo = m + 1; else hi = m;
    }
    const bool hit = lo < n_reg && reg_guest[lo] == (uint64_t)g && reg_cr3[lo] == c3;
    status[i] = hit ? PV_FRAME_OK : PV_FRAME_UNKNOWN_PROCESS;
    record[i] = hit ? lo : 0xFFFFFFFFu;
  }
}

// kInv[kind][field] = position of FileOp field `field` in the kind's layout
// (-1: not carried), the inverse of kLayout.
__constant__ int8_t kInv[10][16] = {
    {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
    {0, -1, -1, -1, -1, 1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},  // OPEN
    {-1, 0, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}, // RELEASE
    {-1, 0, 1, 2, 3, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},    // READ
    {-1, 0, 1, 2, 3, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},    // WRITE
    {-1, 0, 4, -1, -1, 5, 1, 2, 3, -1, -1, -1, -1, -1, -1, -1},      // IOCTL
    {-1, 0, 1, 2, 4, 5, -1, -1, -1, 3, -1, -1, -1, -1, -1, -1},      // MMAP
    {-1, 0, 1, -1, 5, 6, -1, -1, -1, -1, -1, -1, -1, 2, 3, 4},       // PAGE_FAULT
    {-1, 0, -1, -1, -1, -1, -1, -1, -1, -1, 1, 2, -1, -1, -1, -1},   // POLL
    {-1, 0, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 1, -1, -1, -1},      // NOTIFY_SUBSCRIBE
};

// One FileOp row {kind, 16 fields} from the kind's layout words w0..w6,
// built in registers (selects, no indexed register arrays) and stored once.
__device__ __forceinline__ void store_op(uint64_t* __restrict__ row, uint32_t kind, uint32_t w0, uint32_t w1,
                                         uint32_t w2, uint32_t w3, uint32_t w4, uint32_t w5, uint32_t w6) {
  row[0] = kind;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int p = kInv[kind][j];
    const uint32_t v = p == 0 ? w0 : p == 1 ? w1 : p == 2 ? w2 : p == 3 ? w3 : p == 4 ? w4 : p == 5 ? w5 :
                       p == 6 ? w6 : 0u;
    row[1 + j] = v;
  }
}

// Per frame: decode single-frame operations, flag page-fault first /
// continuation frames for the pairing pass.  A CTA builds the 136-byte op
// rows of 256 consecutive frames in shared memory and stores them as
// coalesced 8-byte words (row stores straight from registers would scatter
// every warp store over 32 rows).
__global__ void __launch_bounds__(kFrTpb)
frame_classify_kernel(const pv_frame* __restrict__ frames, uint64_t n, const uint32_t* __restrict__ record,
                      uint64_t* __restrict__ ops_out, uint32_t* __restrict__ status, uint8_t* __restrict__ pair_flag,
                      uint64_t* __restrict__ keys, uint32_t* __restrict__ iota) {
  __shared__ uint64_t rows[kFrTpb * PV_FOP_WORDS];
  const uint64_t n_tiles = (n + kFrTpb - 1) / kFrTpb;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i0 = tile * kFrTpb, i = i0 + threadIdx.x;
    if (i < n) {
      pair_flag[i] = 0;
      iota[i] = (uint32_t)i;
      if (status[i] == PV_FRAME_OK) {  // identify failed: the reference raises before feed
        const pv_frame f = frames[i];
        if (f.opcode == kCont || f.opcode == kPageFault) {
          pair_flag[i] = 1;
          keys[i] = ((uint64_t)record[i] << 32) | f.args[0];
        } else if (f.opcode < 1 || f.opcode > 9) {  // FileOpKind(opcode): ValueError
          status[i] = PV_FRAME_BAD_KIND;
        } else {
          store_op(rows + threadIdx.x * PV_FOP_WORDS, f.opcode, f.args[0], f.args[1], f.args[2], f.args[3],
                   f.args[4], f.args[5], 0);
        }
      }
    }
    __syncthreads();
    const uint64_t words = (min((uint64_t)kFrTpb, n - i0)) * PV_FOP_WORDS;
    uint64_t* dst = ops_out + i0 * PV_FOP_WORDS;
    for (uint64_t w = threadIdx.x; w < words; w += kFrTpb) dst[w] = rows[w];  // rows of other frames: undefined
    __syncthreads();
  }
}

// One thread per run of equal keys in the sorted pairing list: the
// reference's automaton (hypercall.py:155-175) in frame order.
__global__ void __launch_bounds__(kFrTpb)
frame_pair_kernel(const pv_frame* __restrict__ frames, const uint64_t* __restrict__ skeys,
                  const uint32_t* __restrict__ sidx, const uint32_t* __restrict__ n_sel, uint64_t* __restrict__ ops_out,
                  uint32_t* __restrict__ status) {
  const uint32_t n = *n_sel;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    if (r > 0 && skeys[r - 1] == skeys[r]) continue;  // not a run head
    uint32_t pending = 0xFFFFFFFFu;
    for (uint32_t j = r; j < n && skeys[j] == skeys[r]; ++j) {
      const uint32_t i = sidx[j];
      const pv_frame f = frames[i];
      if (f.opcode == kPageFault) {
        if (pending != 0xFFFFFFFFu) {
          status[i] = PV_FRAME_DUP_FIRST;  // "second first-frame before continuation"
        } else {
          pending = i;
          status[i] = PV_FRAME_PENDING;
        }
        continue;
      }
      if (pending == 0xFFFFFFFFu) {
        status[i] = PV_FRAME_ORPHAN;  // "continuation frame without a matching first frame"
        continue;
      }
      const pv_frame h = frames[pending];
      // words = head.args[1:] + frame.args[1 : 1 + n_tail]
      store_op(ops_out + (uint64_t)i * PV_FOP_WORDS, kPageFault, h.args[1], h.args[2], h.args[3], h.args[4],
               h.args[5], f.args[1], f.args[2]);
      status[pending] = PV_FRAME_CONSUMED;
      status[i] = PV_FRAME_OK;
      pending = 0xFFFFFFFFu;
    }
  }
}

static unsigned grid_for(const void* k, uint64_t n) {
  uint64_t g = (n + kFrTpb - 1) / kFrTpb;
  const uint64_t cap = resident_grid(k, kFrTpb, 0);
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

cudaError_t launch_frame_pack(const uint64_t* ops, uint64_t n, const uint64_t* vcpu, const uint64_t* cr3,
                              const uint64_t* tag, const uint64_t* frame_off, pv_frame* frames, uint32_t* status,
                              cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  void* tk = timing_begin("frame_pack", stream);
  frame_pack_kernel<<<grid_for((const void*)frame_pack_kernel, n), kFrTpb, 0, stream>>>(ops, n, vcpu, cr3, tag,
                                                                                       frame_off, frames, status);
  timing_end(tk, stream);
  return cudaGetLastError();
}

cudaError_t launch_frame_identify(const pv_frame* frames, uint64_t n, const int32_t* vcpu_guest, uint32_t n_vcpus,
                                  const uint64_t* reg_guest, const uint64_t* reg_cr3, uint32_t n_reg,
                                  uint32_t* record, uint32_t* status, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  frame_identify_kernel<<<grid_for((const void*)frame_identify_kernel, n), kFrTpb, 0, stream>>>(
      frames, n, vcpu_guest, n_vcpus, reg_guest, reg_cr3, n_reg, record, status);
  return cudaGetLastError();
}

size_t frame_scratch_bytes(uint64_t n) {
  // flags, keys, selected keys/idx (2 copies each for the sort), count, CUB temp
  size_t temp_select = 0, temp_sort = 0;
  cub::DeviceSelect::Flagged((void*)nullptr, temp_select, (const uint64_t*)nullptr, (const uint8_t*)nullptr,
                             (uint64_t*)nullptr, (uint32_t*)nullptr, (int64_t)n);
  cub::DeviceRadixSort::SortPairs((void*)nullptr, temp_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n);
  const size_t temp = temp_select > temp_sort ? temp_select : temp_sort;
  return 16 * 256 + n * (1 + 8 + 8 + 8 + 4 + 4 + 4) + temp;  // 9 regions, each 256-aligned
}

static inline size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }

cudaError_t launch_frame_assemble(const pv_frame* frames, uint64_t n, const uint32_t* record, uint64_t* ops_out,
                                  uint32_t* status, void* scratch, uint64_t scratch_bytes, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  size_t off = 0;
  auto take = [&](size_t b) {
    void* r = p + off;
    off = up256(off + b);
    return r;
  };
  uint32_t* n_sel = (uint32_t*)take(sizeof(uint32_t));
  uint8_t* flag = (uint8_t*)take(n);
  uint64_t* keys = (uint64_t*)take(n * 8);
  uint64_t* sel_keys = (uint64_t*)take(n * 8);
  uint64_t* sorted_keys = (uint64_t*)take(n * 8);
  uint32_t* iota = (uint32_t*)take(n * 4);
  uint32_t* sel_idx = (uint32_t*)take(n * 4);
  uint32_t* sorted_idx = (uint32_t*)take(n * 4);
  void* temp = p + off;
  size_t temp_bytes = scratch_bytes > off ? scratch_bytes - off : 0;

  void* tk = timing_begin("frame_classify", stream);
  frame_classify_kernel<<<grid_for((const void*)frame_classify_kernel, n), kFrTpb, 0, stream>>>(
      frames, n, record, ops_out, status, flag, keys, iota);
  timing_end(tk, stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // compact the pairing frames in order
  size_t need = temp_bytes;
  e = cub::DeviceSelect::Flagged(temp, need, keys, flag, sel_keys, n_sel, (int64_t)n, stream);
  if (e != cudaSuccess) return e;
  e = cub::DeviceSelect::Flagged(temp, need = temp_bytes, iota, flag, sel_idx, n_sel, (int64_t)n, stream);
  if (e != cudaSuccess) return e;
  uint32_t h_sel = 0;
  e = cudaMemcpyAsync(&h_sel, n_sel, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess || h_sel == 0) return e;
  need = temp_bytes;
  e = cub::DeviceRadixSort::SortPairs(temp, need, sel_keys, sorted_keys, sel_idx, sorted_idx, (int64_t)h_sel, 0, 64,
                                      stream);
  if (e != cudaSuccess) return e;
  frame_pair_kernel<<<grid_for((const void*)frame_pair_kernel, h_sel), kFrTpb, 0, stream>>>(
      frames, sorted_keys, sorted_idx, n_sel, ops_out, status);
  return cudaGetLastError();
}

}  // namespace pv
