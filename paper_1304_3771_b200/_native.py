"""ctypes binding of ``libpv.so`` (the C ABI declared in ``include/pv.h``).

The library is built in-tree (``paper_1304_3771_b200/libpv.so``) by
``__graft_entry__.build()`` / ``make -C paper_1304_3771_b200/csrc``.  Loading
it does not need a GPU; calling a compute entry point does, and every such
call goes through :func:`lib` which raises :class:`NativeUnavailable` when
the library or a CUDA device is missing -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeUnavailable

# PV_LIB: another build of the same library (A/B experiments of compile-time variants)
LIB_PATH = os.environ.get("PV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpv.so")

# ---- constants mirrored from include/pv.h --------------------------------
ABI_VERSION = 5
SUCCESS = 0
EINVAL = -22
ENOMEM = -12
ECUDA = -1000

ST_OK = 0x000
ST_FAULT = 0x010
ST_FAULT2 = 0x020
ST_TRAP = 0x040
ST_TRAP2 = 0x060
ST_NODE_OOR = 0x080
ST_NODE_OOR2 = 0x0A0
ST_DATA_OOR = 0x100
ST_CONFLICT = 0x400

ONE_STAGE = 1
TWO_STAGE = 2
ONE_STAGE_4L = 3  # extension geometry (BASELINE config 3)
FLAG_PS = 0x80

VA32 = 0x1
OUT_PFN = 0x2
CONCURRENT = 0x4  # pv.h PV_CONCURRENT: one walker CTA per SM
OUT_PACKED = 0x8  # pv.h PV_OUT_PACKED: one u64 per lane
SERVER_IDLE = 0x100  # pv.h PV_SERVER_IDLE: the caller's stream has nothing pending
SM_SPLIT_FINE = 0x1  # pv.h PV_SM_SPLIT_FINE
SM_SPLIT_INTERLEAVE = 0x2  # pv.h PV_SM_SPLIT_INTERLEAVE
PACKED_ERR = 1 << 63
PACKED_VALUE_BITS = 42
PACKED_SPILL_VALUE = (1 << 42) - 1
W32_ERR = 0x80000000  # pv.h pv_translate_words lane words
W32_VA = 0x40000000
W32_COMPACT_MASK = 0x1FFFFF
EXC_WORDS = 4         # sizeof(pv_exc) / 8
EXC_STRIPES = 32      # pv.h PV_EXC_STRIPES
HAS_TWO_STAGE = 0x80000000
HAS_4L = 0x40000000

TO_GUEST = 0
FROM_GUEST = 1
COPY_ALIGNED16 = 0x100
CONFLICT_OVERLAP = 0x1  # pv.h PV_CONFLICT_OVERLAP: ordered apply
CONFLICT_TABLE = 0x2    # pv.h PV_CONFLICT_TABLE: page by page

FOP_WORDS = 17     # FileOp words (kind + 16 fields), pv.h PV_FOP_WORDS
FRAME_BYTES = 40   # sizeof(pv_frame)
FRAME_OK, FRAME_PENDING, FRAME_CONSUMED, FRAME_UNPACKABLE, FRAME_BAD_KIND = 0, 1, 2, 3, 4
FRAME_ORPHAN, FRAME_DUP_FIRST, FRAME_UNKNOWN_VCPU, FRAME_UNKNOWN_PROCESS = 5, 6, 7, 8

FIFO_MAX = 32
# struct sizes in 8-byte words (all structs are u64-aligned)
SPACE_WORDS = 4    # pv_space
SEG_WORDS = 4      # pv_seg
SHIM_WORDS = 4     # pv_shim
OP_WORDS = 4       # pv_op
RESULT_WORDS = 4   # pv_op_result
FIFO_WORDS = 2 * FIFO_MAX + 4  # pv_fifo

# every symbol include/pv.h declares
EXPORTS = (
    "pv_abi_version", "pv_translate_chunk", "pv_status_name", "pv_translate", "pv_translate_words",
    "pv_fifo_replay", "pv_copy_plan", "pv_copy_plan_nodes", "pv_copy_stamp", "pv_copy_exec",
    "pv_copy_fifo_replay", "pv_scatter_pages", "pv_gather_pages", "pv_stream_sync", "pv_stream_idle", "pv_upload", "pv_sm_split", "pv_set_sm_budget", "pv_peer_alloc", "pv_peer_open", "pv_peer_close",
    "pv_peer_free", "pv_memcpy", "pv_index_encode",
    "pv_fifo_scratch_bytes", "pv_copy_ordered_scratch_bytes", "pv_copy_ordered", "pv_result_encode",
    "pv_result_decode", "pv_timing", "pv_timing_ms", "pv_copy_shim_scratch_bytes", "pv_copy_shim",
    "pv_map_scratch_bytes", "pv_map_plan", "pv_map_commit",
    "pv_frame_pack", "pv_frame_identify", "pv_frame_assemble_scratch_bytes", "pv_frame_assemble",
    "pv_walk_one", "pv_copy_small", "pv_server_walk", "pv_server_copy_small", "pv_server_stop",
    "pv_server_resident", "pv_host_alloc", "pv_host_free", "pv_image_create", "pv_image_destroy",
)

_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_p = ctypes.c_void_p

_SIGNATURES = {
    "pv_abi_version": (ctypes.c_int, []),
    "pv_translate_chunk": (_u64, []),
    "pv_status_name": (ctypes.c_char_p, [_u32]),
    "pv_translate": (ctypes.c_int, [_p, _u64, _p, _p, _u32, _u64, _p, _u32, _p, _p, _p, _p, _p]),
    "pv_translate_words": (ctypes.c_int, [_p, _u64, _p, _p, _u32, _u64, _p, _u32, _p, _p, _p, _u64, _p, _u64, _p]),
    "pv_index_encode": (ctypes.c_int, [_p, _u64, _p, _p, _u64, _u64, _p, _p, _p]),
    "pv_fifo_replay": (ctypes.c_int, [_p, _u32, _p, _p, _p, _u32, _u64, _u64, _u32, _p, _p, _p, _p, _u64, _p]),
    "pv_fifo_scratch_bytes": (_u64, [_u64, _u64, _u32]),
    "pv_copy_ordered_scratch_bytes": (_u64, [_u64, _u64]),
    "pv_copy_shim_scratch_bytes": (_u64, [_u64]),
    "pv_map_scratch_bytes": (_u64, []),
    "pv_frame_pack": (ctypes.c_int, [_p, _u64, _p, _p, _p, _p, _p, _p, _p]),
    "pv_frame_identify": (ctypes.c_int, [_p, _u64, _p, _u32, _p, _p, _u32, _p, _p, _p]),
    "pv_frame_assemble_scratch_bytes": (_u64, [_u64]),
    "pv_frame_assemble": (ctypes.c_int, [_p, _u64, _p, _p, _p, _p, _u64, _p]),
    "pv_map_plan": (ctypes.c_int, [_p, _u64, _u64, _u64, _p, _u64, _p, _p, _p, _p]),
    "pv_map_commit": (ctypes.c_int, [_p, _u64, _u64, _u64, _p, _u64, _p, _p, _u64, _p, _p, _u32, _p, _u64, _u64, _p,
                                     _p, _p]),
    "pv_copy_shim": (ctypes.c_int, [_p, _u64, _p, _p, _p, _u64, _p, _u64, _p, _p, _p, _p, _p, _p, _u64, _p]),
    "pv_result_encode": (ctypes.c_int, [_p, _u64, _p, _p, _p, _p, _u64, _p, _p, _p]),
    "pv_result_decode": (ctypes.c_int, [_p, _u64, _p, _u64, _p, _p, _p]),
    "pv_copy_ordered": (ctypes.c_int, [_p, _u64, _p, _u64, _p, _u64, _p, _p, _p, _p, _p, _u64, _p, _p, _p, _u64, _p]),
    "pv_copy_plan": (ctypes.c_int, [_p, _u64, _p, _p, _u64, _p, _u64, _u32, _p, _p, _p, _p, _p, _u32, _p, _p]),
    "pv_copy_plan_nodes": (ctypes.c_int, [_p, _u64, _p, _p, _u64, _p, _u64, _p, _p, _p, _p, _p, _u64, _u32, _p]),
    "pv_copy_stamp": (ctypes.c_int, [_p, _u64, _u64, _p, _p, _p, _u64, _u32, _p, _p, _p]),
    "pv_copy_exec": (ctypes.c_int, [_p, _u64, _p, _u64, _p, _u64, _u32, _p, _p, _p, _p, _p, _u64, _p, _p, _p, _p]),
    "pv_copy_fifo_replay": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, _u32, _u64, _u64, _u32, _p, _u64, _p, _p, _p,
                                            _p, _u64, _p]),
    "pv_scatter_pages": (ctypes.c_int, [_p, _u64, _p, _u64, _p, _p]),
    "pv_gather_pages": (ctypes.c_int, [_p, _u64, _p, _u64, _p, _p]),
    "pv_stream_sync": (ctypes.c_int, [_p]),
    "pv_stream_idle": (ctypes.c_int, [_p]),
    "pv_upload": (ctypes.c_int, [_p, _p, _u64, _p]),
    "pv_sm_split": (ctypes.c_int, [_u32, _u32, _p, _p, _p, _p]),
    "pv_set_sm_budget": (_u32, [_u32]),
    "pv_peer_alloc": (ctypes.c_int, [_u64, _p, _p]),
    "pv_peer_open": (ctypes.c_int, [_p, _p]),
    "pv_peer_close": (ctypes.c_int, [_p]),
    "pv_peer_free": (ctypes.c_int, [_p]),
    "pv_memcpy": (ctypes.c_int, [_p, _p, _u64, _p]),
    "pv_timing": (ctypes.c_int, [ctypes.c_int]),
    "pv_timing_ms": (ctypes.c_double, [ctypes.c_char_p, _p]),
    "pv_walk_one": (ctypes.c_int, [_p, _u64, _p, _u64, _u32, _p, _u64, _p]),
    "pv_copy_small": (ctypes.c_int, [_p, _u64, _p, _p, _u64, _p, _p, _u64, _p]),
    "pv_server_walk": (ctypes.c_int, [_p, _u64, _p, _u64, _u32, _p, _p]),
    "pv_server_copy_small": (ctypes.c_int, [_p, _u64, _p, _p, _u64, _p, _p, _u32, _p]),
    "pv_server_stop": (ctypes.c_int, []),
    "pv_server_resident": (ctypes.c_int, []),
    "pv_image_create": (ctypes.c_int, [_u64, _p, _u32, _u64, _p, _p, _p]),
    "pv_image_destroy": (ctypes.c_int, [_p]),
    "pv_host_alloc": (_p, [_u64]),
    "pv_host_free": (None, [_p]),
}

SMALL_PAGES = 64  # pv.h PV_SMALL_PAGES


class PvSpace(ctypes.Structure):
    _fields_ = [("s1_base", _u64), ("s1_root_pfn", _u64), ("s2_root_pfn", _u64), ("mode", _u64)]


class PvOpResult(ctypes.Structure):
    _fields_ = [("copied", _u64), ("value", _u64), ("aux", _u64), ("status", _u32), ("fail_page", _u32)]


class PvOneResult(ctypes.Structure):
    _fields_ = [("value", _u64), ("aux", _u64), ("status", _u64), ("seq", _u64)]


class PvSmallOp(ctypes.Structure):
    _fields_ = [("space", PvSpace), ("gva", _u64), ("len", _u64), ("direction", _u32), ("reserved", _u32),
                ("pre_hpa", _u64 * SMALL_PAGES)]


class PvSmallResult(ctypes.Structure):
    _fields_ = [("op", PvOpResult), ("page_hpa", _u64 * SMALL_PAGES), ("page_status", _u32 * SMALL_PAGES),
                ("seq", _u64)]

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpv.so and bind its signatures (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with __graft_entry__.build() "
                "or `make -C paper_1304_3771_b200/csrc`")
        cdll = ctypes.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(cdll, name)
            fn.restype = res
            fn.argtypes = args
        if cdll.pv_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libpv.so ABI version mismatch; rebuild it")
        _lib = cdll
        return _lib


# cudaStream_t handles that may have library work queued since a per-call
# operation last found them idle (percall.py skips the stream query otherwise)
busy_streams: set = set()
_cuda_ok = False
_raw_stream = None


def lib() -> ctypes.CDLL:
    """The library, for a compute call: requires a CUDA device.  The calling
    thread's current stream is noted as possibly busy (the caller is about to
    queue work on it)."""
    global _cuda_ok, _raw_stream
    if not _cuda_ok:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("the HAS data plane runs on a CUDA device and none is visible")
        _raw_stream = torch._C._cuda_getCurrentRawStream
        _cuda_ok = True
    import torch

    busy_streams.add(_raw_stream(torch.cuda.current_device()))
    return load()


def stream_idle(stream: int) -> bool:
    """True when everything queued on the cudaStream_t ``stream`` has completed."""
    r = load().pv_stream_idle(stream)
    if r < 0:
        check(r, "pv_stream_idle")
    return r == 1


def check(rc: int, what: str) -> None:
    if rc == SUCCESS:
        return
    if rc <= ECUDA:
        raise RuntimeError(f"{what}: CUDA error {ECUDA - rc}")
    raise ValueError(f"{what}: libpv returned {rc}")
