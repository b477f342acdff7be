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


# ---- pv_translate_words: 4-byte lane words + exception records ----------------------------

def _split(img, plan, d):
    v, s, a = dp.translate_lanes(img, plan, d)
    return v.cpu().numpy().view(np.uint64), s.cpu().numpy().view(np.uint32), a.cpu().numpy().view(np.uint64)


def _words(img, plan, d, cap, lane_base=0, out_pfn=False):
    """(words, records counted, LaneExceptions written, overflow)."""
    w = torch.empty(d.numel(), dtype=torch.int32, device="cuda")
    exc = dp.ExcList(cap)
    dp.translate_words(img, plan, d, w, exc, lane_base, out_pfn=out_pfn)
    got, n, overflow = exc.read()
    _words.last = exc
    return w.cpu().numpy(), n, got, overflow


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
@pytest.mark.parametrize("va64", [False, True])
def test_word_lanes_equal_split(cuda, mode, va64):
    """Every status kind (faults at every level, traps, TDP-stage faults with
    wide gpas, aliasing u64 VAs) decodes to the (value, status, aux) of the
    split form; only lanes whose value is not their own va take a record."""
    memv, space = _c4(mode)
    tr = memv.translator(space, use_cache=False)
    img = memv.host_mem.backing
    rng = np.random.default_rng(11)
    vas = np.concatenate([W.C1_GVA + rng.integers(0, 64 << 20, 150_000), rng.integers(0, 1 << 32, 50_000),
                          W.C1_GVA + np.arange(8) * 4096]).astype(np.uint64)
    if va64:
        vas[::7] |= np.uint64(1) << np.uint64(50)
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas), 0)], image=img)
    d = torch.from_numpy(vas.view(np.int64) if va64 else vas.astype(np.uint32).view(np.int32)).cuda()
    v, s, a = _split(img, plan, d)
    w, n, exc, overflow = _words(img, plan, d, cap=len(vas), lane_base=1000)
    assert not overflow and n == len(exc) and len(set(exc.lane.tolist())) == n
    exc.lane -= 1000
    assert np.array_equal(exc.status, s[exc.lane])
    uv, us, ua = dp.unpack_words(w, d.cpu().numpy(), exc)
    assert (s != 0).any() and n > 0
    assert np.array_equal(us, s) and np.array_equal(uv, v)
    trap2 = (s & 0xFF0) == 0x060
    assert np.array_equal(ua[trap2], a[trap2])
    # the records are exactly the failing lanes whose value is not their va (or that carry a gpa)
    vv = d.cpu().numpy().view(np.uint32 if not va64 else np.uint64).astype(np.uint64)
    need = (s != 0) & ((v != vv) | trap2)
    assert np.array_equal(np.sort(exc.lane), np.flatnonzero(need))
    # PV_OUT_PFN: the same words' frames are the walk's pfns
    vp, sp_, _ = dp.translate_lanes(img, plan, d, out_pfn=True)
    wp, _, exc_p, _ = _words(img, plan, d, cap=len(vas), out_pfn=True)
    pv_, ps_, _ = dp.unpack_words(wp, d.cpu().numpy(), exc_p, out_pfn=True)
    assert np.array_equal(pv_, vp.cpu().numpy().view(np.uint64)) and np.array_equal(ps_, sp_.cpu().numpy().view(np.uint32))


def test_word_lanes_overflowing_list(cuda):
    """Records past exc_cap are counted, not written; the words stay exact."""
    memv, space = _c4("shadow")  # traps: one record per trapping lane
    tr = memv.translator(space, use_cache=False)
    img = memv.host_mem.backing
    rng = np.random.default_rng(12)
    vas = (W.C1_GVA + rng.integers(0, 64 << 20, 200_000)).astype(np.uint32)
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas), 0)], image=img)
    d = torch.from_numpy(vas.view(np.int32)).cuda()
    w_full, n, exc_full, overflow = _words(img, plan, d, cap=len(vas))
    assert n > 64 and not overflow
    # 64 records of room: 2 per stripe; every record is counted, each stripe writes what fits
    w_small, n_small, exc_small, overflow = _words(img, plan, d, cap=64)
    counts = _words.last._last
    assert overflow and n_small == n == int(counts.sum())
    assert len(exc_small) == int(np.minimum(counts, 2).sum())
    assert set(exc_small.lane.tolist()) <= set(exc_full.lane.tolist())
    assert np.array_equal(w_small, w_full)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_translate_many_words_equal_split(cuda, mode):
    """The host pipeline in 4-byte words (two jobs, several chunks, a list
    too small for the batch's exceptions: it re-runs) returns the lanes of
    the split form."""
    memv, space = _c4(mode)
    tr = memv.translator(space, use_cache=False)
    rng = np.random.default_rng(13)
    jobs = []
    for n in (3_000_000, 1_234_567):
        vas = (W.C1_GVA + rng.integers(0, 64 << 20, n)).astype(np.uint32)
        jobs.append((tr, torch.from_numpy(vas.view(np.int32)).pin_memory()))
    split = mv.translate_many(jobs, chunk=1 << 20)
    from paper_1304_3771_b200 import dataplane as dpl
    got = dpl.translate_host_many(tr.image, [(tr.device_space, h) for _, h in jobs], chunk=1 << 20, words=True,
                                  exc_cap=64)
    via_api = mv.translate_many(jobs, chunk=1 << 20, words=True)
    for (v, s, a), (w, none, exc), (w2, _, exc2), (_, host) in zip(split, got, via_api, jobs):
        assert none is None and w.dtype == torch.int32
        assert np.array_equal(w.numpy(), w2.numpy())
        uv, us, ua = dp.unpack_words(w.numpy(), host.numpy(), exc)
        assert np.array_equal(us, s.numpy().view(np.uint32)) and np.array_equal(uv, v.numpy().view(np.uint64))
        assert np.array_equal(ua, a.numpy().view(np.uint64))
    assert dp.last_host_io["d2h"] >= 4 * sum(h.numel() for _, h in jobs)


def test_translate_many_words_empty_inputs(cuda):
    memv, space = _c4("shadow")
    tr = memv.translator(space, use_cache=False)
    assert mv.translate_many([], words=True) == []
    (w, none, exc), = mv.translate_many([(tr, torch.zeros(0, dtype=torch.int32).pin_memory())], words=True)
    assert w.numel() == 0 and none is None and len(exc) == 0
    v, s, a = dp.unpack_words(w.numpy(), np.zeros(0, np.uint32), exc)
    assert len(v) == len(s) == len(a) == 0
