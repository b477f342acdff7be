"""The hybrid resolver's trap shim on the device (pv_copy_shim) vs the reference.

* the "shim" scenario (every kind of trapping shadow entry: simple leaf traps,
  one slot reached through two shadow paths, a shadow-only leaf whose guest
  walk faults, a trapping mid entry, a guest page past the slot) replayed per
  op and as batches must give the reference's recorded outcomes, hardware
  translation count and final image digest;
* at BASELINE config 4 size (C1 tables, 20 % of shadow leaves not present,
  10 % trapping) hybrid copy batches -- disjoint and overlapping, both
  directions -- must equal the oracle's sequential restatement byte for byte.
"""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest
import scenarios as S
from conftest import load_json
from oracle import oracle as O
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import errors as er
from paper_1304_3771_b200 import has as be
from paper_1304_3771_b200 import memvirt as mv
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _as_outcome(res, er_mod):
    def fn():
        if isinstance(res, BaseException):
            raise res
        return res

    return S.outcome(fn, er_mod)


def _digest(b: bytes) -> int:
    return int.from_bytes(hashlib.sha256(b).digest()[:8], "little")


def test_shim_scenario_per_op(cuda):
    w = S.shim_build(mv, be, er)
    got = S.shim_query(w, mv, be, er)
    exp = load_json("shim.json")
    assert got["rows"] == exp["rows"]
    assert got["hw_translations"] == exp["hw_translations"]
    assert got["image_sha"] == exp["image_sha"]


def test_shim_scenario_batched(cuda):
    """Consecutive same-direction ops as one batch each."""
    w = S.shim_build(mv, be, er)
    exp = load_json("shim.json")
    acc = be.HardwareHasAccess(w["rec"], w["memv"])
    rows = []
    i = 0
    ops = S.SHIM_OPS
    while i < len(ops):
        j = i
        while j < len(ops) and ops[j][0] == ops[i][0]:
            j += 1
        gvas = [g for _, g, _ in ops[i:j]]
        lens = [n for _, _, n in ops[i:j]]
        if ops[i][0] == "to":
            src = b"".join(S.shim_payload(k, ops[k][2]) for k in range(i, j))
            rows += [_as_outcome(o, er) for o in acc.copy_to_user_batch(gvas, lens, src)]
        else:
            payload, outs = acc.copy_from_user_batch(gvas, lens)
            host = payload.cpu().numpy().tobytes()
            off = 0
            for o, n in zip(outs, lens):
                rows.append(["ok", _digest(host[off:off + n])] if not isinstance(o, BaseException)
                            else _as_outcome(o, er))
                off += n
        i = j
    assert rows == exp["rows"]
    assert w["rec"].hw_translations == exp["hw_translations"]
    assert S.sha(S.image_bytes(w["memv"].host_mem)) == exp["image_sha"]


@pytest.fixture(scope="module")
def c4hw(cuda):
    memv, guest, space = W.build_c1("shadow")
    W.corrupt_c4(memv, space, "shadow")
    rec = be.GuestProcessRecord(S._Guest(0, "shadow"), space, memv)
    acc = be.HardwareHasAccess(rec, memv)
    return memv, guest, space, rec, acc


def _oracle_args(memv, guest, space, rec):
    img = np.frombuffer(memv.host_mem.read(0, memv.host_mem.size_bytes), dtype=np.uint8).copy()
    sp = O.space(0, rec.active_hybrid.root_pfn)
    shim = np.array([guest.base_hpa, guest.mem.size_bytes, space.guest_root.root_pfn, space.shadow_root.root_pfn],
                    np.uint64)
    return img, sp, shim


def _ops(seed: int, n: int, max_len: int, overlap: bool):
    rng = random.Random(seed)
    gvas, lens = [], []
    for i in range(n):
        if overlap:
            gva = W.C1_GVA + rng.randrange(256 * 1024)
        else:
            gva = W.C1_GVA + i * (64 * 1024 * 1024 // n) + rng.randrange(64)
        gvas.append(gva)
        lens.append(rng.randint(1, max_len))
    return gvas, lens


@pytest.mark.parametrize("overlap", [False, True])
def test_c4_hybrid_copy_batch_vs_oracle(c4hw, overlap):
    memv, guest, space, rec, acc = c4hw
    n = 3000
    gvas, lens = _ops(77 + overlap, n, 16 * 1024 if not overlap else 6000, overlap)
    if not overlap:
        lens = [min(l, 64 * 1024 * 1024 // n - 64) for l in lens]
    src = np.random.default_rng(5).integers(0, 256, sum(lens), dtype=np.uint8)
    img, sp, shim = _oracle_args(memv, guest, space, rec)
    offs = np.zeros(n, np.uint64)
    offs[1:] = np.cumsum(np.array(lens[:-1], np.uint64))
    ops = np.stack([np.array(gvas, np.uint64), np.array(lens, np.uint64), offs, np.zeros(n, np.uint64)], 1)
    exp, cut, cnt = O.copy_hybrid(img, sp, shim, ops, src.copy(), 0)
    assert cut == n, "every trap of this world is a simple leaf trap"
    before = rec.hw_translations
    outs = acc.copy_to_user_batch(gvas, lens, src)
    assert rec.hw_translations - before == cnt
    n_fault = 0
    for i, o in enumerate(outs):
        st = int(exp[i, 3]) & 0xFFFFFFFF
        if st == 0:
            assert o == lens[i], i
        else:
            n_fault += 1
            assert isinstance(o, er.PageFault), (i, o)
            assert (o.va, o.level, o.bytes_copied) == (int(exp[i, 1]), st & 0xF, int(exp[i, 0])), i
    assert n_fault > 0
    got = np.frombuffer(memv.host_mem.read(0, memv.host_mem.size_bytes), dtype=np.uint8)
    assert np.array_equal(got, img)
    # read everything back through the (now partly fixed) hybrid table
    payload, outs2 = acc.copy_from_user_batch(gvas, lens)
    buf = np.zeros(sum(lens), np.uint8)
    exp2, cut2, _ = O.copy_hybrid(img, sp, shim, ops, buf, 1)
    assert cut2 == n
    host = payload.cpu().numpy()
    for i, o in enumerate(outs2):
        st = int(exp2[i, 3]) & 0xFFFFFFFF
        a, b = int(offs[i]), int(offs[i]) + (lens[i] if st == 0 else int(exp2[i, 0]))
        assert np.array_equal(host[a:b], buf[a:b]), i
        assert (o == lens[i]) if st == 0 else isinstance(o, er.PageFault), i


def test_shim_trap_free_batch_unchanged(c4hw):
    """A batch whose pages never trap leaves the scratch clean and writes no
    table word (the empty-shim fast path)."""
    memv, guest, space, rec, acc = c4hw
    img = memv.host_mem.backing
    gva = W.C1_GVA
    # find a run of 4 present, non-trapping pages
    tr = memv.translator(space, use_cache=False)
    hp, st, _ = tr.translate_batch(np.arange(W.C1_PAGES, dtype=np.uint64) * 4096 + W.C1_GVA)
    ok = np.flatnonzero(st == 0)
    gva = W.C1_GVA + int(ok[0]) * 4096
    out = acc.copy_to_user_batch([gva], [100], b"x" * 100)
    assert out == [100]
    scratch = dp._per_stream(img, "shim", dp._Grow).t  # the current stream's scratch
    assert scratch is not None and int(scratch[:24].sum()) == 0
