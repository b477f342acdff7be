"""GPU: extension geometry (BASELINE config 3, 16 GiB mixed 4 KiB / 2 MiB
mmap, 4-level tables) -- device walker and copier vs the C restatement
(parity unpinned by the reference, see tests/test_ext4l.py)."""

from __future__ import annotations

import random

import numpy as np
import pytest
import torch

from conftest import status_outcome
from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import errors as er
from paper_1304_3771_b200 import ext4l as X

pytestmark = pytest.mark.gpu


def _check(mem, t, vas, *, out_pfn=False):
    raw = mem.backing.host_for_read()
    sp = t.space
    plan = dp.TranslatePlan([sp], [(0, len(vas), 0)])
    v, s, a = dp.translate_lanes(mem.backing, plan, torch.tensor(vas.view(np.int64), device="cuda"),
                                 out_pfn=out_pfn)
    ov, os_, oa = O.translate(raw, O.space(sp.s1_base, sp.s1_root_pfn, 0, N.ONE_STAGE_4L), vas, want_pfn=out_pfn,
                              threads=0)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), os_)
    assert np.array_equal(v.cpu().numpy().view(np.uint64), ov)
    return os_


def test_c3_16gib_sequential_and_strided(cuda):
    mem, t = X.build_c3()
    seq = X.c3_sequential()
    st = _check(mem, t, seq)
    assert (st == 0).all() and len(seq) == 4_194_304
    st = _check(mem, t, X.c3_strided(), out_pfn=True)
    assert (st == 0).all()


def test_4l_faults_traps_and_aliasing(cuda):
    region = 256 << 20
    mem, t = X.build_c3(region)
    rng = random.Random(44)
    # corrupt entries at every level
    t.set_entry(X.C3_VA + 3 * X.LARGE, 3, 0)                               # PD entry not present
    t.set_entry(X.C3_VA + 5 * X.LARGE + 7 * 4096, 4, (1234 << 12) | 0x4)   # PT entry trapping
    t.set_entry(X.C3_VA + 9 * X.LARGE + 9 * 4096, 4, 0)                    # PT hole
    t.set_entry(X.C3_VA + 12 * X.LARGE, 3, (0xFFFFFF << 12) | 0x1)          # PT node past the image
    t.set_entry(X.C3_VA + (1 << 30) + 5, 2, 0x4)                          # PDPT entry trapping
    t.map_2m(X.C3_VA + region + (4 << 20), 0x200)                           # a lone 2 MiB page
    vas = [X.C3_VA + rng.randrange(region + (8 << 20)) for _ in range(200_000)]
    vas += [X.C3_VA + (1 << 30) + rng.randrange(1 << 20) for _ in range(100)]
    vas += [(rng.randrange(1, 1 << 16) << 48) | (X.C3_VA + rng.randrange(region)) for _ in range(1000)]  # alias
    vas += [rng.randrange(1 << 48) for _ in range(1000)]
    vas = np.array(vas, dtype=np.uint64)
    st = _check(mem, t, vas)
    kinds = {int(x) & 0xFF0 for x in st}
    assert {0x000, 0x010, 0x040, 0x080} <= kinds
    # the generic kernel's 4-byte lane words (+ exception records for the traps) decode to the same lanes
    plan = dp.TranslatePlan([t.space], [(0, len(vas), 0)])
    d = torch.tensor(vas.view(np.int64), device="cuda")
    v, s, _ = dp.translate_lanes(mem.backing, plan, d)
    w = torch.empty(len(vas), dtype=torch.int32, device="cuda")
    xl = dp.ExcList(len(vas))
    dp.translate_words(mem.backing, plan, d, w, xl)
    exc, n, overflow = xl.read()
    assert not overflow
    assert n == int(((st & 0xFF0) == 0x040).sum())  # traps carry their node: one record each
    wv, ws, _ = dp.unpack_words(w.cpu().numpy(), vas, exc)
    assert np.array_equal(ws, st) and np.array_equal(wv, v.cpu().numpy().view(np.uint64))
    levels = {int(x) & 0xF for x in st if int(x) & 0xFF0 == 0x010}
    assert {1, 3, 4} <= levels


def test_4l_copy_roundtrip_across_page_sizes(cuda):
    region = 64 << 20
    mem, t = X.build_c3(region)
    raw = mem.backing.host_for_read().copy()
    gva = X.C3_VA + X.LARGE - 1000          # spans a 2 MiB leaf into a 4 KiB region
    n = 3 * X.LARGE + 777
    data = np.frombuffer(random.Random(1).randbytes(n), dtype=np.uint8)
    ops = np.array([[gva, n, 0, 0]], np.uint64)
    out = dp.copy_ops(mem.backing, [t.space], ops, N.TO_GUEST, torch.from_numpy(data.copy()).cuda())[0]
    assert out.status == 0 and out.copied == n
    sp = t.space
    O.copy(raw, O.space(sp.s1_base, sp.s1_root_pfn, 0, N.ONE_STAGE_4L).reshape(1, 4), ops, data.copy(), 0)
    assert np.array_equal(mem.backing.host_for_read(), raw)
    assert X.walk4(mem, t.root, gva) == X.walk4(mem, t.root, gva - 5)
    with pytest.raises(er.PageFault):
        X.walk4(mem, t.root, X.C3_VA + region + 4096)


def test_c1_in_4level_geometry(cuda):
    """BASELINE configs[0] as written (4-level 4 KiB table, 16,384 shuffled
    pages, 1 M random VAs + a 64 MiB copy_to_user, aligned and +0x800) vs
    the C restatement."""
    mem, t = X.build_c1_4l()
    vas = X.c1_4l_vas()
    st = _check(mem, t, vas)
    assert (st == 0).all()
    # faults past the mapped region and above it at every level
    rng = np.random.default_rng(7)
    wild = np.concatenate([X.C1_4L_VA + rng.integers(64 << 20, 1 << 32, 50_000, dtype=np.int64).astype(np.uint64),
                           rng.integers(0, 1 << 48, 50_000, dtype=np.int64).astype(np.uint64)])
    st = _check(mem, t, wild)
    assert (st != 0).any()
    sp = t.space
    for off, n in ((0, 64 << 20), (0x800, (64 << 20) - 4096)):
        src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        raw = mem.backing.host_for_read().copy()
        outs = dp.copy_ops(mem.backing, [sp], np.array([[X.C1_4L_VA + off, n, 0, 0]], np.uint64), N.TO_GUEST, src)
        assert outs[0].status == 0 and outs[0].copied == n
        O.copy(raw, O.space(sp.s1_base, sp.s1_root_pfn, 0, N.ONE_STAGE_4L).reshape(1, 4),
               np.array([[X.C1_4L_VA + off, n, 0, 0]], np.uint64), src.cpu().numpy(), 0, threads=0)
        assert np.array_equal(mem.backing.host_for_read(), raw)
