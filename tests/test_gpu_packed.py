"""PV_OUT_PACKED on the device: one u64 per lane carries the same result as
the (value, status) pair (include/pv.h), for every status kind the walks
produce -- faults at every level, traps, TDP-stage faults with gpas past the
slot, node reads past the image, wide values that spill into aux -- and the
host pipeline (memvirt.translate_many) returns the same lanes either way."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import memvirt as mv
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _c4(mode):
    memv, guest, space = W.build_c1(mode)
    W.corrupt_c4(memv, space, mode)
    if mode == "tdp":  # guest PTEs past the slot, wide ones too: TDP-stage faults with big gpas
        gm = space.guest.mem
        root = space.guest_root.root_pfn
        mid = gm.read_word(root, (W.C1_GVA >> 30) & 3) >> 12
        leaf = gm.read_word(mid, (W.C1_GVA >> 21) & 0x1FF) >> 12
        gm.write_word(leaf, 3, ((gm.size_bytes >> 12) + 9) << 12 | 0x3)
        gm.write_word(leaf, 4, (0x3FFFF_FFFF_FF) << 12 | 0x3)  # gpa far beyond 2^42
    return memv, space


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
@pytest.mark.parametrize("va64", [False, True])
def test_packed_lanes_equal_unpacked(cuda, mode, va64):
    memv, space = _c4(mode)
    tr = memv.translator(space, use_cache=False)
    img = memv.host_mem.backing
    rng = np.random.default_rng(3)
    vas = np.concatenate([W.C1_GVA + rng.integers(0, 64 << 20, 150_000), rng.integers(0, 1 << 32, 50_000),
                          W.C1_GVA + np.arange(8) * 4096]).astype(np.uint64)
    if va64:
        vas[::7] |= np.uint64(1) << np.uint64(50)  # aliasing VAs: one-stage faults report them (spill)
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas), 0)], image=img)
    d = torch.from_numpy(vas.view(np.int64) if va64 else vas.astype(np.uint32).view(np.int32)).cuda()
    v, s, a = dp.translate_lanes(img, plan, d)
    pw, ps, pa = dp.translate_lanes(img, plan, d, packed=True)
    assert ps is None
    v, s, a = v.cpu().numpy().view(np.uint64), s.cpu().numpy().view(np.uint32), a.cpu().numpy()
    uv, us = dp.unpack_lanes(pw.cpu().numpy(), pa.cpu().numpy())
    assert (s != 0).any()
    assert np.array_equal(us, s) and np.array_equal(uv, v)
    # TDP-stage traps keep their gpa in aux either way
    trap2 = (s & 0xFF0) == 0x060
    assert np.array_equal(pa.cpu().numpy()[trap2], a[trap2])


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_translate_many_packed_equals_unpacked(cuda, mode):
    memv, space = _c4(mode)
    tr = memv.translator(space, use_cache=False)
    rng = np.random.default_rng(9)
    vas = (W.C1_GVA + rng.integers(0, 64 << 20, 3_000_000)).astype(np.uint32)
    host = torch.from_numpy(vas.view(np.int32)).pin_memory()
    (v, s, a), = mv.translate_many([(tr, host)], chunk=1 << 20)
    (w, none, pa), = mv.translate_many([(tr, host)], chunk=1 << 20, packed=True)
    assert none is None
    uv, us = dp.unpack_lanes(w.numpy(), pa.numpy())
    assert np.array_equal(us, s.numpy().view(np.uint32)) and np.array_equal(uv, v.numpy().view(np.uint64))
