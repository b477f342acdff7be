"""The C-ABI library loads without a GPU and exports every declared symbol."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200.errors import NativeUnavailable

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions() -> list[str]:
    with open(os.path.join(ROOT, "include", "pv.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pv_[a-z0-9_]+)\s*\(", src)) - {"pv_op", "pv_space"})


def test_header_and_binding_agree():
    assert declared_functions() == sorted(N.EXPORTS)


def test_library_exports_every_symbol():
    lib = N.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.pv_abi_version() == N.ABI_VERSION
    assert lib.pv_translate_chunk() > 0
    assert lib.pv_status_name(0x013) == b"page_fault"
    assert lib.pv_status_name(0x100) == b"out_of_range"


def test_argument_validation_needs_no_gpu():
    lib = N.load()
    # NULL buffers are rejected before any CUDA call
    assert lib.pv_translate(None, 4096, None, None, 1, 1, None, 0, None, None, None, None, None) == N.EINVAL
    assert lib.pv_copy_plan(None, 4096, None, None, 1, None, 1, 0, None, None, None, None, None, 0, None,
                            None) == N.EINVAL
    # bad image size / flags
    assert lib.pv_translate(ctypes.c_void_p(8), 4095, ctypes.c_void_p(8), ctypes.c_void_p(8), 1, 1,
                            ctypes.c_void_p(8), 0, None, ctypes.c_void_p(8), ctypes.c_void_p(8), None,
                            None) == N.EINVAL
    assert lib.pv_index_encode(None, 4096, None, None, 0, 1, None, None, None) == N.EINVAL
    # 4-byte lane words: frames must fit 28 bits (images below 2^40 bytes); PV_OUT_PACKED is not a words flag
    p8 = ctypes.c_void_p(8)
    cnt = ctypes.c_void_p(8)
    assert lib.pv_translate_words(None, 4096, p8, p8, 1, 1, p8, 0, None, p8, None, 0, cnt, 0, None) == N.EINVAL
    assert lib.pv_translate_words(p8, 1 << 40, p8, p8, 1, 1, p8, 0, None, p8, None, 0, cnt, 0, None) == N.EINVAL
    assert lib.pv_translate_words(p8, 4096, p8, p8, 1, 1, p8, N.OUT_PACKED, None, p8, None, 0, cnt, 0,
                                  None) == N.EINVAL
    assert lib.pv_translate_words(p8, 4096, p8, p8, 1, 1, p8, 0, None, p8, None, 5, cnt, 0, None) == N.EINVAL
    # per-call server / uploads / peer buffers: argument errors come back before any CUDA call
    assert lib.pv_server_walk(None, 4096, p8, 0, 0, p8, None) == N.EINVAL
    assert lib.pv_server_walk(p8, 4096, p8, 0, 0x4, p8, None) == N.EINVAL  # unknown flag
    assert lib.pv_server_copy_small(p8, 4096, None, p8, 0, p8, None, 0, None) == N.EINVAL
    assert lib.pv_upload(ctypes.c_void_p(16), ctypes.c_void_p(17), 64, None) == N.EINVAL  # misaligned source
    assert lib.pv_upload(None, None, 0, None) == N.SUCCESS  # nothing to move
    assert lib.pv_peer_open(None, None) == N.EINVAL
    assert lib.pv_peer_alloc(0, None, None) == N.EINVAL
    assert lib.pv_sm_split(0, 0, None, None, None, None) == N.EINVAL
    assert lib.pv_memcpy(None, None, 0, None) == N.SUCCESS


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1304_3771_b200 import memvirt as mv

    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, "shadow")
    sp = memv.create_process(g)
    memv.map_region(sp, 0x2000_0000, 1)
    with pytest.raises(NativeUnavailable):
        memv.translator(sp).translate(0x2000_0000)
    with pytest.raises(NativeUnavailable):
        mv.walk(memv.host_mem, sp.shadow_root.root_pfn, 0x2000_0000)
