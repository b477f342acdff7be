"""SM partitions (include/pv.h pv_sm_split / pv_set_sm_budget): a walk on one
green-context partition beside a copy batch on the other gives the results
of the same calls back to back, and grid budgets reset after the block."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import has as be
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu


class _G:
    def __init__(self):
        self.id, self.mem_mode = 0, "shadow"


@pytest.mark.parametrize("fine", [False, True])
@pytest.mark.parametrize("interleave", [False, True])
def test_split_partitions_are_disjoint_and_cover_the_device(cuda, fine, interleave):
    sp = dp.SmSplit(48, fine=fine, interleave=interleave)
    total = torch.cuda.get_device_properties(0).multi_processor_count
    assert sp.sms[0] >= 48 and sp.sms[0] + sp.sms[1] == total
    if fine:
        assert sp.sms[0] == 48  # single-SM granularity: exactly the count asked for
    lib = N.lib()
    with sp.on(1):
        assert lib.pv_set_sm_budget(sp.sms[1]) == sp.sms[1]  # set inside the block
    assert lib.pv_set_sm_budget(0) == 0  # and reset after it


def test_walk_beside_copy_on_partitions_equals_serial(cuda):
    memv, guest, space = W.build_c1("shadow", device=True)
    img = memv.host_mem.backing
    tr = memv.translator(space, use_cache=False)
    vas = W.c1_vas(1_000_000)
    d = torch.from_numpy(vas.astype(np.uint32).view(np.int32)).cuda()
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas), 0)], image=img)
    rec = be.GuestProcessRecord(_G(), space, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    n = 16 << 20
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda",
                        generator=torch.Generator("cuda").manual_seed(3))

    def walk(words, exc):
        dp.translate_words(img, plan, d, words, exc)

    serial_w = torch.empty(len(vas), dtype=torch.int32, device="cuda")
    walk(serial_w, dp.ExcList(4096))
    torch.cuda.synchronize()
    split = dp.SmSplit(64)
    w = torch.empty_like(serial_w)
    cnt = dp.ExcList(4096)
    ev = torch.cuda.Event()
    ev.record()
    for k in (0, 1):
        split.streams[k].wait_event(ev)
    with split.on(0):
        walk(w, cnt)
    with split.on(1):
        out = acc.copy_to_user_batch([W.C1_GVA + 4096], [n], src)
    torch.cuda.synchronize()
    assert out == [n]
    assert torch.equal(w, serial_w)
    assert cnt.read()[1] == 0
    # the copy landed: read it back through the reference-style API
    got = np.frombuffer(bytes(acc.copy_from_user(W.C1_GVA + 4096 + 12345, 4096)), dtype=np.uint8)
    assert np.array_equal(got, src[12345:12345 + 4096].cpu().numpy())
