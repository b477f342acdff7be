/*
 * pv.h — C ABI of the B200 hybrid-address-space (HAS) data plane.
 *
 * This is the drop-in boundary for the hot path of the devfsim reference
 * (arXiv 1304.3771, "Paradice"): batched gva -> (gpa ->) hpa translation
 * through guest / shadow / TDP / hybrid page tables and the page-chunked
 * copy_to_user / copy_from_user gather/scatter between an operation buffer
 * and guest pages.  Every entry point cites the reference interface it
 * replaces (paths relative to the reference's pkg/src/devfsim/).
 *
 * Conventions
 *   - plain pointers and sizes only; no exceptions cross the ABI.
 *   - "device pointer" arguments are CUDA device memory owned by the caller;
 *     "host pointer" arguments are host memory (pinned or pageable).
 *   - every call is asynchronous on `stream` unless its comment says it
 *     synchronises; a NULL stream is the legacy default stream.
 *   - return value: 0 on success, negative on API / launch error
 *     (PV_EINVAL, PV_ENOMEM, PV_ECUDA).  Per-lane / per-op outcomes are
 *     reported through status arrays (PV_ST_* below), never as return codes.
 *
 * Memory image
 *   The image is the reference's host physical memory (memvirt.py:124-188,
 *   `PhysMem` over one flat bytearray): host-private region first, then the
 *   guest slots (memvirt.py:433-480).  It lives in HBM as one flat byte array
 *   of `image_bytes` bytes (a multiple of 4096).  A page-table node at pfn P
 *   of a memory window with byte base B is at image offset B + P*4096; entry
 *   i of it is the little-endian u64 at B + P*4096 + i*8 (memvirt.py:170-172).
 *   Like the reference, node reads are bounded only by the image, not by the
 *   window; a read past the image is reported as PV_ST_NODE_OOR (the
 *   reference raises struct.error there).
 */
#ifndef PV_H_
#define PV_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PV_ABI_VERSION 5

/* ---- return codes ------------------------------------------------------ */
#define PV_SUCCESS 0
#define PV_EINVAL (-22)
#define PV_ENOMEM (-12)
#define PV_ECUDA (-1000) /* PV_ECUDA - cudaError_t value */

/* ---- per-lane / per-op status word --------------------------------------
 * bits 0-3  : level (1 top, 2 mid, 3 leaf)            (memvirt.py:60-62)
 * bits 4-11 : kind
 * bits 16-24: entry index within the node (traps only; TrapExit.index)
 * Rebuilt into the reference exception types by the Python layer
 * (errors.py:15-45).
 */
#define PV_ST_OK 0x000u
#define PV_ST_FAULT 0x010u     /* PageFault(va, level); value = va            */
#define PV_ST_FAULT2 0x020u    /* PageFault in the TDP stage; value = gpa     */
#define PV_ST_TRAP 0x040u      /* TrapExit(va, level, node, index); value=node */
#define PV_ST_TRAP2 0x060u     /* TrapExit in the TDP stage; value = node,
                                  aux = gpa (the TrapExit.va of that walk)     */
#define PV_ST_NODE_OOR 0x080u  /* node read past the image; value = va        */
#define PV_ST_NODE_OOR2 0x0A0u /* same, TDP stage; value = gpa                */
#define PV_ST_DATA_OOR 0x100u  /* OutOfRange on the data access; value = hpa  */
#define PV_ST_CONFLICT 0x400u  /* batch-level: two ops of one to_guest batch
                                  write the same hpa page (host re-plans)      */
#define PV_ST_KIND(s) ((s) & 0xFF0u)
#define PV_ST_LEVEL(s) ((s) & 0xFu)
#define PV_ST_INDEX(s) (((s) >> 16) & 0x1FFu)

/* ---- translator description ----------------------------------------------
 * One process address space as the reference's ProcessTranslator /
 * _HybridResolver see it (memvirt.py:568-601, 677-696; backend.py:117-128).
 *   PV_ONE_STAGE : walk(s1_base window, s1_root_pfn, va) -> hpa.  Shadow
 *                  translation (memvirt.py:598-599), hybrid resolve
 *                  (memvirt.py:677-682), host tables, and walk_guest
 *                  (memvirt.py:262-267; s1_base = guest slot base, result is
 *                  the gpa).
 *   PV_TWO_STAGE : gpa = walk_guest(gva) in the guest window, then
 *                  walk(host, s2_root_pfn, gpa) (memvirt.py:600-601).
 */
#define PV_ONE_STAGE 1u
#define PV_TWO_STAGE 2u
/* Extension (BASELINE config 3; no reference semantics, parity pinned only
 * by the oracle restatement): a single-stage 4-level table over 48-bit VAs
 * (9/9/9/9/12; VA bits >= 48 ignored) whose level-3 entries may map 2 MiB
 * pages (PV_FLAG_PS).  Same entry codec otherwise (T before P, W ignored);
 * a 2 MiB leaf translates to (pfn << 12) + (va & 0x1FFFFF).  Fault / trap
 * levels run 1..4. */
#define PV_ONE_STAGE_4L 3u
#define PV_FLAG_PS 0x80u

typedef struct pv_space {
  uint64_t s1_base;     /* byte base of the stage-1 memory window          */
  uint64_t s1_root_pfn; /* stage-1 root node pfn (window relative)          */
  uint64_t s2_root_pfn; /* TDP root node pfn (host memory, base 0)          */
  uint32_t mode;        /* PV_ONE_STAGE | PV_TWO_STAGE                      */
  uint32_t reserved;
} pv_space;

/* A contiguous run of lanes translated through one space. */
typedef struct pv_seg {
  uint64_t begin;       /* first lane                                      */
  uint64_t end;         /* one past the last lane                          */
  uint64_t chunk0;      /* first global chunk id of this segment (exclusive
                           prefix sum of ceil((end-begin)/pv_translate_chunk())) */
  uint32_t space;       /* index into the spaces array                     */
  uint32_t reserved;
} pv_seg;

/* ---- leaf index ------------------------------------------------------------
 * A derived, L2-resident 4-byte copy of the leaf-level page-table nodes a
 * batch walks (the reference's 8-byte leaf PTEs of a large world do not fit
 * the 126 MB L2).  Slot s caches image page slot_page[s] (absolute page
 * number) as 512 codes:  bits 0-1 state (0 not present, 1 present,
 * 2 trapping, 3 escape: read the raw PTE), bits 2-31 target pfn (present).
 * slot_of[page] maps an image page to its slot (0xFFFFFFFF = not indexed).
 * It is a cache keyed by page contents: pv_index_encode must re-run for a
 * slot whenever its page changes (the host runtime does this for host writes
 * and, via the device dirty map, for device writes).  Walks that reach a
 * page that is not indexed read the raw PTE, so results never depend on
 * what is indexed.
 */
typedef struct pv_index {
  const uint32_t* slot_of;    /* device, one per image page                  */
  const uint32_t* leaf_codes; /* device, 512 per slot                        */
  const uint64_t* slot_page;  /* device, absolute image page of each slot    */
  uint64_t n_slots;
} pv_index;

/* (Re)build leaf codes.  slots (device, may be NULL): encode slots[i] for
 * i < n; NULL: encode slots first_slot .. first_slot+n-1.  dirty (device,
 * one byte per image page, may be NULL): only slots whose page is marked. */
int pv_index_encode(const uint8_t* image, uint64_t image_bytes,
                    const uint64_t* slot_page, const uint64_t* slots,
                    uint64_t first_slot, uint64_t n, uint32_t* leaf_codes,
                    const uint8_t* dirty, void* stream);

/* ---- translate flags ---------------------------------------------------- */
#define PV_VA32 0x1u    /* vas is uint32_t[] (else uint64_t[])             */
#define PV_OUT_PFN 0x2u /* value = leaf pfn (walk); else address with the
                           page offset of the va (translate / resolve)     */
#define PV_OUT_PACKED 0x8u /* one u64 per lane in out_value (out_status may be
                              NULL): see pv_translate */
#define PV_CONCURRENT 0x4u /* size the walk for a kernel running beside it:
                              one CTA per SM (the rest of each SM's
                              registers and shared memory stay free) */
#define PV_HAS_4L 0x40000000u        /* some space of the batch is
                           PV_ONE_STAGE_4L (selects the generic kernel)    */
#define PV_HAS_TWO_STAGE 0x80000000u /* some space of the batch is
                           PV_TWO_STAGE (selects the two-stage kernel)     */

/* One user-buffer copy operation (memvirt.py:604-628). */
typedef struct pv_op {
  uint64_t gva;     /* first guest virtual address                         */
  uint64_t len;     /* bytes                                               */
  uint64_t buf_off; /* byte offset of this op's payload in the op buffer   */
  uint32_t space;   /* index into the spaces array                         */
  uint32_t reserved;
} pv_op;

/* Per-op outcome of a copy batch. */
typedef struct pv_op_result {
  uint64_t copied; /* bytes copied before the failing page (PageFault.bytes_copied) */
  uint64_t value;  /* fault va / gpa, trap node pfn, or OOR hpa (per status)        */
  uint64_t aux;    /* gpa of a TDP-stage trap                                       */
  uint32_t status; /* PV_ST_*                                                        */
  uint32_t fail_page; /* page index within the op of the failing page               */
} pv_op_result;

/* FIFO translation cache state of one process (memvirt.py:336-374). */
#define PV_FIFO_MAX 32
typedef struct pv_fifo {
  uint64_t key[PV_FIFO_MAX]; /* gva >> 12 (unmasked)                        */
  uint64_t val[PV_FIFO_MAX]; /* hpa >> 12                                   */
  uint64_t hits;
  uint64_t misses;
  uint32_t capacity;         /* 1..PV_FIFO_MAX (reference default 10)       */
  uint32_t len;              /* live entries                                */
  uint32_t head;             /* ring index of the oldest entry              */
  uint32_t reserved;
} pv_fifo;

#define PV_TO_GUEST 0u   /* copy_to_user  : buffer -> guest pages           */
#define PV_FROM_GUEST 1u /* copy_from_user: guest pages -> buffer           */
/* pv_copy_exec direction hint (or-ed in): for every op,
 * (gva - (buf + buf_off)) % 16 == 0, so every chunk's 16-byte-aligned middle
 * moves through the Tensor Memory Accelerator (cp.async.bulk global -> shared
 * -> global, a 6-stage ring per warp) and only its < 16-byte head / tail
 * through the LSU.  Chunks that do not satisfy it are still copied correctly,
 * through the LSU. */
#define PV_COPY_ALIGNED16 0x100u

/* ---- library ------------------------------------------------------------ */
int pv_abi_version(void);
/* Lanes per translate chunk (for pv_seg.chunk0). */
uint64_t pv_translate_chunk(void);
/* Static name of a status kind ("ok", "page_fault", ...). */
const char* pv_status_name(uint32_t status);

/* ---- K1: batched translation ----------------------------------------------
 * Replaces per-lane calls of walk (memvirt.py:244-259), walk_guest
 * (memvirt.py:262-267), ProcessTranslator.translate with use_cache=False /
 * _resolve_page (memvirt.py:585-601) and resolve_hybrid (memvirt.py:677-682).
 * spaces / segs / vas / out_* are device pointers.  out_aux may be NULL
 * (then TDP-stage trap gpas are not reported).  Lanes not covered by any
 * segment are not written.  index (HOST pointer to a struct of device
 * pointers, may be NULL): leaf index consulted instead of the raw leaf PTEs
 * for indexed leaf nodes.  Batches of at least 8 chunks per resident CTA
 * build per-segment stage tables in library-internal scratch taken from the
 * device's default stream-ordered pool (cudaMallocAsync / cudaFreeAsync on
 * `stream`, 16.5 KiB per segment; the pool keeps up to 256 MiB cached).
 *
 * PV_OUT_PACKED: out_value[i] carries the whole lane result (8 bytes instead
 * of 12 to store and to move to the host): a lane that translated is its
 * value (an hpa / pfn, below 2^40), any other lane is PV_PACKED_ERR | compact
 * status << 42 | value, compact status = (status & 0xFFF) | index << 12
 * (21 bits; index = status >> 16).  A value that needs more than 42 bits (a
 * TDP-stage fault gpa from a wild guest PTE, a u64 VA) is written to
 * out_aux[i] and the lane's low 42 bits read PV_PACKED_SPILL_VALUE; out_aux
 * must then be non-NULL unless the batch is PV_VA32 and one-stage (those
 * never spill).  out_status is not written and may be NULL.
 */
#define PV_PACKED_ERR (1ull << 63)
#define PV_PACKED_VALUE_BITS 42
#define PV_PACKED_SPILL_VALUE ((1ull << 42) - 1)
int pv_translate(const uint8_t* image, uint64_t image_bytes,
                 const pv_space* spaces, const pv_seg* segs, uint32_t n_segs,
                 uint64_t n_chunks, const void* vas, uint32_t flags,
                 const pv_index* index,
                 uint64_t* out_value, uint32_t* out_status, uint64_t* out_aux,
                 void* stream);

/* ---- K1, 4-byte lane words -------------------------------------------------
 * The same batch walk as pv_translate (same replacements, spaces, segs,
 * vas, flags except PV_OUT_PACKED, index), with one 4-byte word per lane in
 * out_word -- half the bytes of PV_OUT_PACKED to store and to move to the
 * host, which bounds a host-fed batch (the VAs go in at 4 bytes per lane):
 *   bit 31 clear   the lane translated: the word is its frame number (the
 *                  hpa / gpa >> 12; the value is word << 12 | (va & 0xFFF),
 *                  or the word itself under PV_OUT_PFN);
 *   PV_W32_ERR     the lane raises: bits 0-20 hold the compact status (as
 *                  PV_OUT_PACKED: (status & 0xFFF) | index << 12), and
 *     | PV_W32_VA  the exception's value is the lane's own va (page faults
 *                  and out-of-range nodes of a one-stage walk), or
 *     otherwise    the value (and the TDP-stage trap gpa, aux) is in an
 *                  exception record with .lane = lane_base + lane.
 * The records are striped over PV_EXC_STRIPES counters so a fault-heavy
 * batch does not serialise on one atomic: exc_count (device) holds
 * PV_EXC_STRIPES counters, stripe s owns records exc[s * per .. (s+1) * per)
 * with per = exc_cap / PV_EXC_STRIPES, and its counter is advanced by one
 * atomic per warp; counters are never reset here (zero them before the first
 * call of a series that shares them); a stripe's records past `per` are
 * counted but not written -- the caller re-runs with a larger list.  Record
 * order within a stripe is unspecified (one record per lane). */
#define PV_EXC_STRIPES 32
#define PV_W32_ERR 0x80000000u
#define PV_W32_VA 0x40000000u
#define PV_W32_COMPACT_MASK 0x1FFFFFu
typedef struct pv_exc {
  uint64_t lane;   /* lane_base + lane index of the batch                   */
  uint64_t value;  /* the exception's value (trap node, gpa, ...)          */
  uint64_t aux;    /* TDP-stage trap gpa (0 otherwise)                      */
  uint32_t status; /* full status word                                      */
  uint32_t reserved;
} pv_exc;
int pv_translate_words(const uint8_t* image, uint64_t image_bytes,
                       const pv_space* spaces, const pv_seg* segs, uint32_t n_segs,
                       uint64_t n_chunks, const void* vas, uint32_t flags,
                       const pv_index* index, uint32_t* out_word,
                       pv_exc* exc, uint64_t exc_cap, unsigned long long* exc_count,
                       uint64_t lane_base, void* stream);

/* ---- K4: FIFO cache replay --------------------------------------------------
 * Applies the per-process FIFO translation cache (memvirt.py:336-374,
 * 585-594) to lookups that pv_translate / pv_copy_plan resolved fresh.
 * Lookups of process p are positions proc_off[p] .. proc_off[p+1]) of a
 * lookup stream in program order; win_off[p] = sum over q < p of
 * ceil(lookups_q / 32) (n_procs + 1 entries).  Every process uses the same
 * `capacity` (1..PV_FIFO_MAX).  A hit replaces the lookup's value/status with
 * the cached translation; a miss that resolved inserts (oldest-first
 * eviction); a miss that faulted keeps the fault and inserts nothing.
 * fifo[] (device) is updated in place (entries rewritten oldest-first with
 * head 0, counters advanced).  Exact; parallel over 32-lookup windows with
 * sequential verification (see pv_fifo.cu).  scratch: device memory of
 * pv_fifo_scratch_bytes(lookups, windows, capacity) bytes.  At most 65536
 * processes per call (PV_EINVAL / CUDA invalid-value beyond).  n_lookups and
 * n_windows must equal proc_off[n_procs] and win_off[n_procs] (the device
 * arrays are not read back: the call never synchronises the stream).
 */
uint64_t pv_fifo_scratch_bytes(uint64_t n_lookups, uint64_t n_windows, uint32_t capacity);

/* Lanes of a pv_translate batch: lookup l is lane lane_idx[l] (device);
 * key = vas[lane] >> 12.  flags: PV_VA32 as for pv_translate. */
int pv_fifo_replay(const void* vas, uint32_t flags, const uint64_t* lane_idx,
                   const uint64_t* proc_off, const uint64_t* win_off,
                   uint32_t n_procs, uint64_t n_lookups, uint64_t n_windows,
                   uint32_t capacity, pv_fifo* fifo,
                   uint64_t* value, uint32_t* status, void* scratch,
                   uint64_t scratch_bytes, void* stream);

/* ---- K2/K3: batched user-buffer copy -------------------------------------
 * Replaces copy_user_buffer (memvirt.py:604-628) as used by
 * SoftwareHasAccess / HardwareHasAccess copy_to_user / copy_from_user
 * (backend.py:92-104, 152-162).  Ops run with the reference's per-op
 * semantics: one translation per page touched, chunk = min(remaining,
 * 4096 - (cur & 0xFFF)), pages before the first failing page are copied and
 * nothing after it, `copied` reports the completed prefix.
 *
 * pv_copy_plan translates every page of every op (page_off[] = exclusive
 * prefix sum of page spans, n_ops+1 entries, device) into page_hpa[] /
 * page_status[] (device, page_off[n_ops] entries each) and records each op's
 * first failing page in op_first_bad[] (device, n_ops; the caller sets it to
 * all-ones first).  For PV_TO_GUEST it also stamps destination pages in
 * page_owner[] (device, one u64 per image page; NULL disables) with
 * (epoch << 40 | page + 1), one stamp per live chunk, and sets *conflict
 * (device u32) to PV_CONFLICT_OVERLAP when two chunks of the batch write
 * one hpa page.
 *
 * pv_copy_exec moves the bytes for every page below its op's first failing
 * page and fills results[] (device, n_ops).  dirty[] (device, one byte per
 * image page; may be NULL) is set to 1 for every image page written.
 * buf is the op buffer (device) of buf_bytes bytes: a chunk reaching past
 * it moves only the bytes the buffer holds (the reference's slice of a
 * short host_buf, memvirt.py:624), never reading or writing beyond it.
 * abort_flag (device, may be NULL): when
 * *abort_flag != 0 at launch (the conflict word of the stamp pass) the
 * kernel writes nothing, so the host can re-plan the batch in order.
 */
int pv_copy_plan(const uint8_t* image, uint64_t image_bytes,
                 const pv_space* spaces, const pv_op* ops, uint64_t n_ops,
                 const uint64_t* page_off, uint64_t n_pages, uint32_t direction,
                 uint64_t* page_hpa, uint32_t* page_status, uint64_t* page_aux,
                 uint64_t* op_first_bad, uint64_t* page_owner, uint32_t epoch,
                 uint32_t* conflict, void* stream);

int pv_copy_exec(uint8_t* image, uint64_t image_bytes, const pv_op* ops,
                 uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages,
                 uint32_t direction, const uint64_t* page_hpa,
                 const uint32_t* page_status, const uint64_t* page_aux,
                 const uint64_t* op_first_bad, uint8_t* buf, uint64_t buf_bytes,
                 pv_op_result* results, uint8_t* dirty,
                 const uint32_t* abort_flag, void* stream);

/* pv_copy_plan (without the stamp) that also marks, in node_map[] (device,
 * one u32 per image page, node_pages >= image_bytes / 4096 entries), every
 * page-table node page any page's walk reads with `epoch` (non-zero; the
 * same epoch as the stamp pass that follows).  The table-hazard check of a
 * to_guest batch: a copy in program order translates page k, then writes
 * chunk k, so a chunk that lands on a table node changes the walks of the
 * pages after it (memvirt.py:615-627); a batch cannot reproduce that and
 * must run page by page instead. */
int pv_copy_plan_nodes(const uint8_t* image, uint64_t image_bytes,
                       const pv_space* spaces, const pv_op* ops, uint64_t n_ops,
                       const uint64_t* page_off, uint64_t n_pages,
                       uint64_t* page_hpa, uint32_t* page_status, uint64_t* page_aux,
                       uint64_t* op_first_bad, uint32_t* node_map, uint64_t node_pages,
                       uint32_t epoch, void* stream);

/* *conflict bits (device u32) set by the stamp pass; the exec stands down
 * on any. */
#define PV_CONFLICT_OVERLAP 0x1u /* two chunks write one hpa page: ordered apply */
#define PV_CONFLICT_TABLE 0x2u   /* a chunk writes a node page marked in node_map: page by page */

/* The conflict pass of pv_copy_plan on its own (run it after
 * pv_copy_fifo_replay when the cache may have changed destinations).
 * owner_pages = number of u64 entries in page_owner.  node_map (device,
 * may be NULL): the marks of pv_copy_plan_nodes with the same epoch; a live
 * chunk whose destination page is marked sets PV_CONFLICT_TABLE. */
int pv_copy_stamp(const uint64_t* page_off, uint64_t n_ops, uint64_t n_pages,
                  const uint64_t* page_hpa, const uint64_t* op_first_bad,
                  uint64_t* page_owner, uint64_t owner_pages, uint32_t epoch,
                  uint32_t* conflict, const uint32_t* node_map, void* stream);

/* Replays the FIFO cache over a copy plan: lookup l is page look_page[l]
 * of op look_op[l] (pages of an op consecutive and in order, ops of a
 * process in program order).  Each op stops at its first page that misses
 * and fails to resolve or whose data access is out of range; page_hpa /
 * page_status are rewritten for cache hits and op_first_bad recomputed for
 * every op in the stream, so pv_copy_exec sees the cached translations. */
int pv_copy_fifo_replay(const pv_op* ops, const uint64_t* page_off,
                        const uint64_t* look_page, const uint32_t* look_op,
                        const uint64_t* proc_off, const uint64_t* win_off,
                        uint32_t n_procs, uint64_t n_lookups, uint64_t n_windows,
                        uint32_t capacity, pv_fifo* fifo,
                        uint64_t image_bytes, uint64_t* page_hpa,
                        uint32_t* page_status, uint64_t* op_first_bad,
                        void* scratch, uint64_t scratch_bytes, void* stream);

/* Ordered execution of a PV_TO_GUEST batch whose chunks share destination
 * pages (the stamp pass reported a conflict): runs after pv_copy_plan (and
 * pv_copy_fifo_replay) instead of pv_copy_exec and gives exactly the bytes
 * the reference's sequential copy_user_buffer calls leave (last writer wins
 * in op order, pages of an op in order); fills results[] like pv_copy_exec.
 * Chunks are grouped by destination page with a stable radix sort and each
 * page is rebuilt in shared memory by one CTA.  scratch: device memory of
 * pv_copy_ordered_scratch_bytes(n_pages, image_bytes) bytes. */
uint64_t pv_copy_ordered_scratch_bytes(uint64_t n_pages, uint64_t image_bytes);
int pv_copy_ordered(uint8_t* image, uint64_t image_bytes, const pv_op* ops,
                    uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages,
                    const uint64_t* page_hpa, const uint32_t* page_status,
                    const uint64_t* page_aux, const uint64_t* op_first_bad,
                    const uint8_t* buf, uint64_t buf_bytes, pv_op_result* results,
                    uint8_t* dirty, void* scratch, uint64_t scratch_bytes,
                    void* stream);

/* ---- per-call path (one walk or one small copy per launch) -----------------
 * The reference's drivers call ctx.mem.copy_to_user / copy_from_user once per
 * op and ProcessTranslator.translate once per page (devices.py:148, 254, 316;
 * backend.py:92-104; memvirt.py:585-628).  These entry points serve one such
 * call in ONE launch with no memcpy: the request travels in the kernel's
 * parameters (by value), results are written straight into host-mapped
 * pinned memory (pv_host_alloc) and published last with `seq`, so the caller
 * can spin on out->seq instead of synchronising the stream.
 *
 * pv_walk_one: walk / walk_guest / translate (uncached) / resolve_hybrid of
 * one address (memvirt.py:244-267, 596-601, 677-682).  flags: PV_OUT_PFN.
 * out->value / aux / status follow the pv_translate conventions. */
typedef struct pv_one_result {
  uint64_t value;
  uint64_t aux;
  uint64_t status;
  uint64_t seq; /* written last (after a system-scope fence) */
} pv_one_result;
int pv_walk_one(const uint8_t* image, uint64_t image_bytes, const pv_space* space /* host */,
                uint64_t va, uint32_t flags, pv_one_result* out, uint64_t seq, void* stream);

/* pv_copy_small: one copy_user_buffer op of at most PV_SMALL_PAGES pages
 * (memvirt.py:604-628): every page translated (pre_hpa[k] != 0: the caller
 * resolved page k itself -- a FIFO cache hit -- to byte hpa pre_hpa[k] - 1;
 * still bounds-checked), the op stops at its first failing
 * page, the chunks before it move between `buf` (device memory or
 * host-mapped pinned memory, buf_bytes bytes, clamped like pv_copy_exec) and
 * the image, dirty[] marks written image pages.  out->page_hpa /
 * page_status hold every page's translation (for the caller's FIFO inserts). */
#define PV_SMALL_PAGES 64
typedef struct pv_small_op {
  pv_space space;
  uint64_t gva;
  uint64_t len;
  uint32_t direction; /* PV_TO_GUEST / PV_FROM_GUEST */
  uint32_t reserved;
  uint64_t pre_hpa[PV_SMALL_PAGES];
} pv_small_op;
typedef struct pv_small_result {
  pv_op_result op;
  uint64_t page_hpa[PV_SMALL_PAGES];
  uint32_t page_status[PV_SMALL_PAGES];
  uint64_t seq; /* written last (after a system-scope fence) */
} pv_small_result;
int pv_copy_small(uint8_t* image, uint64_t image_bytes, const pv_small_op* op /* host */, uint8_t* buf,
                  uint64_t buf_bytes, pv_small_result* out, uint8_t* dirty, uint64_t seq, void* stream);

/* ---- per-call server ---------------------------------------------------------
 * The same two per-call operations without a kernel launch per call: a
 * resident one-CTA server kernel on a library-private non-blocking stream of
 * the current device polls a request mailbox in mapped pinned host memory,
 * serves the request with the device code of pv_walk_one / pv_copy_small and
 * publishes the reply there; the call returns when the reply is in *out.
 * Ordered after the work queued on `stream`: when the stream is idle
 * (cudaStreamQuery) the server serves the request, otherwise it is launched
 * on the stream (pv_walk_one / pv_copy_small into the mailbox) and the call
 * waits for it.  The first served call -- and the first after
 * PV_SERVER_IDLE_US (default 200) microseconds without a request, after which
 * the server exits by itself so device-wide synchronisation never waits
 * longer -- launches the server.  Work queued on OTHER streams is not waited
 * for (as with the launches above).  Calls from several host threads are
 * serialised.  While resident the server holds one CTA slot of one SM;
 * pv_server_stop parks it (synchronous) before batch kernels that size their
 * grids to fill every SM.  out->seq is the call's request number.
 * PV_SERVER_IDLE in flags: the caller asserts that nothing queued on `stream`
 * is still pending that the request depends on, so the stream is not queried
 * (a cudaStreamQuery costs about as much as a PCIe round trip). */
#define PV_SERVER_IDLE 0x100u
int pv_server_walk(const uint8_t* image, uint64_t image_bytes, const pv_space* space /* host */,
                   uint64_t va, uint32_t flags, pv_one_result* out /* host */, void* stream);
int pv_server_copy_small(uint8_t* image, uint64_t image_bytes, const pv_small_op* op /* host */,
                         uint8_t* buf, uint64_t buf_bytes, pv_small_result* out /* host */,
                         uint8_t* dirty, uint32_t flags, void* stream);
int pv_server_stop(void);
/* 1 while the server of the current device may be resident. */
int pv_server_resident(void);

/* ---- per-rank residency ------------------------------------
 * A zero-filled device image of image_bytes whose byte offsets are the
 * reference's hpas (memvirt.py:433-480 slot carving), with HBM behind only
 * the byte ranges [ranges[2i], ranges[2i+1]) (host array; widened to the
 * VMM granularity, 2 MiB).  Every other page is backed by one shared
 * zero-filled hole of hole_bytes (0: 256 MiB) mapped repeatedly, so a stray
 * access reads junk instead of faulting.  One reserved virtual range: every
 * kernel addresses it like a flat allocation.  *out_device_bytes = HBM
 * actually allocated (resident ranges + hole).  Replaces the flat image
 * allocation of a guest-sharded rank (each GPU holds the host-private region
 * and its own guests' slots). */
int pv_image_create(uint64_t image_bytes, const uint64_t* ranges, uint32_t n_ranges, uint64_t hole_bytes,
                    uint8_t** out_ptr, void** out_handle, uint64_t* out_device_bytes);
int pv_image_destroy(void* handle);

/* Host-mapped pinned memory (cudaHostAllocMapped | Portable): the device
 * reads and writes it through the same pointer (UVA). */
void* pv_host_alloc(uint64_t bytes);
void pv_host_free(void* p);

/* ---- trap shim on the device -----------------------
 * The default hypervisor shim of the hybrid resolver (backend.py:117-128,
 * 288-296; resolve_hybrid_with_fixup, memvirt.py:685-696) for a planned copy
 * batch over hybrid spaces: run after pv_copy_plan, before the stamp / exec.
 * shims[s] (device, one per space of the batch) names the guest process
 * behind hybrid space s; guest_bytes == 0 disables the shim for that space.
 *
 * Every trapped page whose shim the device can run exactly is resolved: a
 * leaf-level trap whose shadow descend (TableEditor._descend, memvirt.py:
 * 282-298) ends on the trapping slot, whose guest walk succeeds and whose
 * gpa lies inside the slot.  Per slot, the earliest such page in (op, page)
 * order writes word = (hpa >> 12) << 12 | P | W into the image (dirty set for
 * the node page); the page then re-walks the hybrid table (the retry) and
 * gets an ordinary translation.  op_first_bad is recomputed.  Every other
 * trap keeps its PV_ST_TRAP status; the first op whose first failure is such
 * a trap is the cut -- shims of pages after it are not applied (their traps
 * stand), so the host can finish that op with its own shim and re-plan the
 * rest in order.  n_written (device u64, may be NULL) is incremented by the
 * number of table words written.  scratch: device memory of pv_copy_shim_scratch_bytes
 * (n_pages) bytes, zero-filled before its first use; every call leaves it
 * zero-filled again. */
typedef struct pv_shim {
  uint64_t guest_base;      /* byte base of the guest slot (gpa 0)                */
  uint64_t guest_bytes;     /* slot size: gpa_to_hpa bound (memvirt.py:491-497)   */
  uint64_t guest_root_pfn;  /* the process's guest table root (window relative)  */
  uint64_t shadow_root_pfn; /* the process's shadow table root (host memory)     */
} pv_shim;

uint64_t pv_copy_shim_scratch_bytes(uint64_t n_pages);
int pv_copy_shim(uint8_t* image, uint64_t image_bytes, const pv_space* spaces, const pv_shim* shims,
                 const pv_op* ops, uint64_t n_ops, const uint64_t* page_off, uint64_t n_pages,
                 uint64_t* page_hpa, uint32_t* page_status, uint64_t* op_first_bad,
                 uint8_t* dirty, uint64_t* n_written, void* scratch, uint64_t scratch_bytes,
                 void* stream);

/* ---- batched table construction --------------------
 * n calls of TableEditor(mem, root, alloc).map(vas[i], target_i) in order
 * (memvirt.py:270-313) on the image window at byte `base` (host memory: 0;
 * a guest memory: its slot base), node frames drawn from a FIFO frame
 * allocator (memvirt.py:191-213); with data_first, every page first draws its
 * own data frame from the same allocator and maps it (map_process_page /
 * map_region, memvirt.py:508-526: frame order per page [data][mid?][leaf?]).
 *
 * pv_map_plan: need[i] (device u8) = bit 0 "page i allocates the mid node of
 * its top entry", bit 1 "page i allocates the leaf node of its (top, mid)
 * entry".  *bad (device u64; the caller sets it to all-ones) is lowered to
 * the first page the batch cannot build exactly -- its leaf entry is not
 * NOT_PRESENT (AlreadyMapped), an existing node lies past the image
 * (struct.error), or it repeats the (top, mid, leaf) slot of an earlier page
 * -- in which case the caller runs the reference's per-page loop instead.
 * vas (device u64) must be page aligned.  scratch: pv_map_scratch_bytes().
 *
 * pv_map_commit: frames (device u64, n_frames) = the allocator's frames in
 * allocation order, frame_off[i] (device u64) = exclusive prefix sum over
 * pages of (data_first + popcount(need[i])).  Frames j with hot[j] != 0
 * (device u8, may be NULL) or whose page is marked in dirty are zeroed
 * (FrameAllocator.alloc zeroes; never-written frames are already zero).  The
 * leaf entry of page i becomes (target << 12) | leaf_flags with target =
 * frames[frame_off[i]] + target_add (data_first; the data frame is also
 * stored to out_data[i] when out_data != NULL) or targets[i] + target_add;
 * new nodes are installed PRESENT | writable.  dirty (device, one byte per
 * image page, may be NULL) is set for every page written. */
uint64_t pv_map_scratch_bytes(void);
int pv_map_plan(const uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root_pfn,
                const uint64_t* vas, uint64_t n, uint8_t* need, uint64_t* bad,
                void* scratch, void* stream);
int pv_map_commit(uint8_t* image, uint64_t image_bytes, uint64_t base, uint64_t root_pfn,
                  const uint64_t* vas, uint64_t n, const uint8_t* need,
                  const uint64_t* frames, uint64_t n_frames, const uint64_t* frame_off,
                  const uint8_t* hot, uint32_t data_first, const uint64_t* targets,
                  uint64_t target_add, uint64_t leaf_flags, uint64_t* out_data,
                  uint8_t* dirty, void* stream);

/* ---- hypercall frame codec ---------------------------
 * The forwarding wire format (hypercall.py): a FileOp is PV_FOP_WORDS u64
 * words {kind, device_id, handle, gva, length, offset, flags, cmd, arg_gva,
 * arg_len, prot, event_mask, timeout_ms, pid, access, vma_start, vma_length}
 * (hypercall.py:62-79, field order); a frame is one opcode, six 32-bit slots,
 * the issuing vCPU and the virtual CR3 (HypercallFrame, :92-101). */
#define PV_FOP_WORDS 17
typedef struct pv_frame {
  uint32_t opcode;      /* FileOpKind, or 0x7F = continuation                 */
  uint32_t args[6];     /* the six argument slots                              */
  uint32_t vcpu;
  uint64_t virtual_cr3;
} pv_frame;

/* per-op / per-frame outcome */
#define PV_FRAME_OK 0u               /* packed / identified / op decoded here    */
#define PV_FRAME_PENDING 1u          /* page-fault first frame still waiting     */
#define PV_FRAME_CONSUMED 2u         /* first frame completed by a later frame   */
#define PV_FRAME_UNPACKABLE 3u       /* Unpackable: layout word >= 2^32; bits
                                        8-15 = FileOp field index (pack)          */
#define PV_FRAME_BAD_KIND 4u         /* not a FileOpKind (ValueError)            */
#define PV_FRAME_ORPHAN 5u           /* Unpackable: continuation without a first */
#define PV_FRAME_DUP_FIRST 6u        /* Unpackable: second first-frame           */
#define PV_FRAME_UNKNOWN_VCPU 7u     /* UnknownVcpu (identify)                   */
#define PV_FRAME_UNKNOWN_PROCESS 8u  /* UnknownProcess (identify)                */

/* pack (hypercall.py:125-137) for n ops (device, n x PV_FOP_WORDS u64):
 * op i writes its frames at frames[frame_off[i]] (frame_off = exclusive scan
 * of 2 for PAGE_FAULT, else 1); vcpu / cr3 / tag are per-op device u64
 * arrays (tag: page faults only).  status[i] (device u32) per op; a failing
 * op writes no frame. */
int pv_frame_pack(const uint64_t* ops, uint64_t n, const uint64_t* vcpu, const uint64_t* cr3,
                  const uint64_t* tag, const uint64_t* frame_off, pv_frame* frames,
                  uint32_t* status, void* stream);
/* VcpuRegistry.identify (hypercall.py:178-211) per frame: vcpu_guest[v]
 * (device i32, n_vcpus entries, -1 = unregistered) and the registry of
 * processes sorted by (reg_guest, reg_cr3) (device u64 arrays, n_reg
 * entries).  record[i] = index of the frame's process in the registry;
 * status[i] = PV_FRAME_OK / UNKNOWN_VCPU / UNKNOWN_PROCESS. */
int pv_frame_identify(const pv_frame* frames, uint64_t n, const int32_t* vcpu_guest,
                      uint32_t n_vcpus, const uint64_t* reg_guest, const uint64_t* reg_cr3,
                      uint32_t n_reg, uint32_t* record, uint32_t* status, void* stream);
/* FrameAssembler.feed (hypercall.py:155-175) over a batch in frame order,
 * after pv_frame_identify (frames whose status is not PV_FRAME_OK are
 * skipped, as the reference raises before feeding them).  Frame i that
 * completes an operation gets PV_FRAME_OK and the op at ops_out[i *
 * PV_FOP_WORDS]; pending frames are keyed by (record, tag).  Equal to
 * feeding the frames one by one, each error caught.  SYNCHRONISES `stream`
 * once (the size of the pairing set).  scratch: device memory of
 * pv_frame_assemble_scratch_bytes(n) bytes. */
uint64_t pv_frame_assemble_scratch_bytes(uint64_t n);
int pv_frame_assemble(const pv_frame* frames, uint64_t n, const uint32_t* record,
                      uint64_t* ops_out, uint32_t* status, void* scratch,
                      uint64_t scratch_bytes, void* stream);

/* ---- result-page codec ------------------------------
 * Batched resultpage.encode + the backend's host_mem.write of the record
 * (resultpage.py:44-51, backend.py:352-355): record r is header[9*r ..
 * 9*r+8] = {status, flags, values[6], blob_len} followed by blob_len bytes
 * of blob_buf at blob_off[r], written at image offset page_hpa[r].  At most
 * one record per page per batch.  status[r]: PV_ST_OK, PV_ST_DATA_OOR
 * (record past the image: OutOfRange), PV_ST_CONFLICT (blob_len > 4060:
 * the codec's ValueError).  dirty as for pv_copy_exec. */
int pv_result_encode(uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa,
                     const uint32_t* header, const uint8_t* blob_buf,
                     const uint64_t* blob_off, uint64_t n, uint32_t* status,
                     uint8_t* dirty, void* stream);
/* Batched resultpage.decode of the header words (resultpage.py:54-61);
 * blobs stay in the image at page_hpa[r] + 36. */
int pv_result_decode(const uint8_t* image, uint64_t image_bytes, const uint64_t* page_hpa,
                     uint64_t n, uint32_t* header, uint32_t* status, void* stream);

/* ---- utility kernels used by the host runtime ---------------------------- */
/* Copy `bytes` from pinned (device-mapped) host memory to device memory with
 * SM loads over the host link instead of a copy engine, so small descriptor
 * uploads do not queue behind a large host-to-device transfer already in
 * flight on another stream (a copy batch whose payload is still arriving).
 * dst and src 16-byte aligned. */
int pv_upload(void* dst, const void* src, uint64_t bytes, void* stream);

/* Scatter `n` whole pages from a (pinned) host staging area into the image:
 * page i of src goes to image page pfns[i].  pfns device, src device. */
int pv_scatter_pages(uint8_t* image, uint64_t image_bytes, const uint64_t* pfns,
                     uint64_t n, const uint8_t* src, void* stream);
/* Gather whole pages out of the image (inverse of pv_scatter_pages). */
int pv_gather_pages(const uint8_t* image, uint64_t image_bytes,
                    const uint64_t* pfns, uint64_t n, uint8_t* dst, void* stream);

/* Synchronises `stream` and reports the first CUDA error seen (0 if none). */
int pv_stream_sync(void* stream);
/* 1 when everything queued on `stream` has completed, 0 while work is
 * pending, negative on a CUDA error (does not synchronise). */
int pv_stream_idle(void* stream);

/* ---- SM partitions ------------------------------------------------------------
 * Two disjoint SM sets of the current device (green contexts): a group of at
 * least first_sms SMs and the rest, one non-blocking stream on each (created
 * once per (device, first_sms, flags) and kept).  flags: PV_SM_SPLIT_FINE
 * splits at single-SM granularity instead of the driver's co-scheduled groups
 * of 8 SMs (another placement of the two sets over the GPCs; which one is
 * faster depends on the box -- bench.py times both and keeps the faster).  Kernels launched on a stream run
 * only on its SMs, so a walk (bound by the SM->L2 request rate) and a page
 * copy (bound by HBM) can share the device side by side without competing
 * for the same SMs.  *sms_first / *sms_rest: the SM counts (may be NULL).
 * PV_EINVAL when the split is impossible, PV_ECUDA - cudaErrorNotSupported
 * when the driver has no green contexts. */
#define PV_SM_SPLIT_FINE 0x1u
/* the device is cut into groups (8 SMs, or 1 with PV_SM_SPLIT_FINE) and the
 * first set takes every other group: both sets interleave over the GPCs */
#define PV_SM_SPLIT_INTERLEAVE 0x2u
int pv_sm_split(uint32_t first_sms, uint32_t flags, void** stream_first, void** stream_rest,
                uint32_t* sms_first, uint32_t* sms_rest);
/* Grids of the calling thread's subsequent launches are sized for `sms` SMs
 * (0: the whole device) -- set it to the partition's count while launching
 * into a pv_sm_split stream.  Returns the previous value. */
uint32_t pv_set_sm_budget(uint32_t sms);

/* ---- results straight into rank 0's HBM --------------------
 * Rank 0 allocates the job's result buffer (pv_peer_alloc: device memory of
 * the current device + a PV_PEER_HANDLE_BYTES IPC handle it sends to the other
 * ranks); every other rank maps it (pv_peer_open: a device pointer into rank
 * 0's memory, peer access over NVLink / NVSwitch enabled on first use) and
 * passes a slice of it as the OUTPUT of its walk (pv_translate_words
 * out_word), so each lane word is stored into rank 0's memory by the kernel
 * that computes it: the result return is fused into the walk, no gather step
 * and no collective.  pv_peer_close unmaps, pv_peer_free (rank 0) frees. */
#define PV_PEER_HANDLE_BYTES 64
int pv_peer_alloc(uint64_t bytes, void** dev_ptr, uint8_t* handle);
int pv_peer_open(const uint8_t* handle, void** dev_ptr);
int pv_peer_close(void* dev_ptr);
int pv_peer_free(void* dev_ptr);
/* Stream-ordered copy between any two device / pinned host pointers (peer
 * mappings included). */
int pv_memcpy(void* dst, const void* src, uint64_t bytes, void* stream);

/* ---- measurement hook ------------------------------------------------------ */
/* pv_timing(1) resets and starts recording a CUDA event pair around every
 * launch of the library's dominant kernels (on the stream they are launched
 * on); pv_timing(0) stops.  pv_timing_ms(kernel, &launches) synchronises the
 * recorded events and returns the summed milliseconds of the named kernel
 * ("ordered_apply") since the last reset.  Not a reference interface: bench.py
 * uses it for the roofline's per-launch duration. */
int pv_timing(int enable);
double pv_timing_ms(const char* kernel, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* PV_H_ */
