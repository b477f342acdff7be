"""Host/device coherence is lazy and range-limited (image.py): after a device
copy writes many pages, a host read gathers only the pages it reads, and
every byte the host reads is current."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import has as be
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu


class _G:
    def __init__(self):
        self.id, self.mem_mode = 0, "shadow"


def test_host_read_after_big_copy_gathers_only_what_it_reads(cuda):
    memv, guest, space = W.build_c1("shadow", device=True)
    img = memv.host_mem.backing
    rec = be.GuestProcessRecord(_G(), space, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    n = 32 << 20
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    out = acc.copy_to_user_batch([W.C1_GVA], [n], src)
    assert out == [n]
    # one table word: the shadow root's first entry -- one page gathered, not 8192
    root = space.shadow_root.root_pfn
    word = memv.host_mem.read_word(root, 0)
    assert word & 1
    pending = int(img._pending.sum())
    assert pending >= n // 4096 - 1, pending
    # a 10-byte guest read via the reference-style per-call path sees the device's bytes
    tr = memv.translator(space, use_cache=False)
    hpa = tr.translate(W.C1_GVA + 12345)
    got = memv.host_mem.read(hpa, 10)
    assert got == src[12345:12355].cpu().numpy().tobytes()
    assert int(img._pending.sum()) == pending - 1
    # the whole image on demand: every page current
    raw = np.frombuffer(memv.host_mem.read(0, memv.host_mem.size_bytes), dtype=np.uint8)
    assert int(img._pending.sum()) == 0
    back = bytearray(n)
    from paper_1304_3771_b200 import memvirt as mv
    assert mv.copy_user_buffer("from_guest", W.C1_GVA, n, back, translator=tr, host_mem=memv.host_mem) == n
    assert bytes(back) == src.cpu().numpy().tobytes()
    # the host mirror and HBM agree byte for byte
    assert np.array_equal(raw, img.device().cpu().numpy())
