"""Data-plane parity on the GPU: this package's CUDA path vs the reference.

Two anchors:
* the golden fixtures recorded from the reference itself (every outcome of
  the scripted scenarios, including exceptions, cache counters and the
  final image digest);
* the C oracle (pinned to the same fixtures by tests/test_oracle.py) at the
  BASELINE config sizes, compared lane by lane and byte by byte.
All results must be bit-exact.
"""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest
import torch

import scenarios as S
from conftest import load_json, status_outcome
from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import errors as er
from paper_1304_3771_b200 import has as be
from paper_1304_3771_b200 import memvirt as mv

pytestmark = pytest.mark.gpu


def test_spec_known_answers(cuda):
    w = S.spec_build(mv, be, er)
    assert S.spec_query(w, mv, be, er) == load_json("spec.json")["expected"]


def test_walks_scenario(cuda):
    w = S.walks_build(mv, be, er)
    got = S.walks_query(w, mv, be, er)
    exp = load_json("walks.json")["expected"]
    for key in exp:
        assert got[key] == exp[key], key


def test_copies_scenario(cuda):
    w = S.copies_build(mv, be, er)
    got = S.copies_query(w, mv, be, er)
    exp = load_json("copies.json")["expected"]
    for key in exp:
        assert got[key] == exp[key], key


def test_c01_single_and_batch(cuda):
    w = S.c01_build(mv, be, er)
    g = load_json("c01.json")
    assert S.c01_query(w, mv, be, er) == g["expected"]
    # the same 10,000 addresses as one device batch
    space = dp.Space(w["guest"].mem.base, w["space"].guest_root.root_pfn)
    plan = dp.TranslatePlan([space], [(0, len(w["samples"]), 0)])
    vas = torch.tensor(np.array(w["samples"], dtype=np.uint64).view(np.int64), device="cuda")
    v, s, a = dp.translate_lanes(w["memv"].host_mem.backing, plan, vas)
    v = v.cpu().numpy().view(np.uint64)
    s = s.cpu().numpy().view(np.uint32)
    a = a.cpu().numpy().view(np.uint64)
    got = [status_outcome(int(s[i]), int(v[i]), int(a[i]), w["samples"][i]) for i in range(len(s))]
    assert got == g["expected"]


def test_c03_hybrid(cuda):
    worlds = S.c03_build(mv, be, er)
    exp = [load_json(f"c03_{i}.json")["expected"] for i in range(len(worlds))]
    assert S.c03_query(worlds, mv, be, er) == exp


@pytest.fixture(scope="module", params=["shadow", "tdp"])
def c1(request, cuda):
    w = S.c1_build(mv, be, er, request.param)
    g = load_json(f"c1_{request.param}.json")
    host = w["memv"].host_mem
    raw = np.frombuffer(S.image_bytes(host), dtype=np.uint8).copy()
    assert hashlib.sha256(raw.tobytes()).hexdigest() == g["image_sha"]
    tr = w["memv"].translator(w["space"], use_cache=False)
    sp = tr.device_space
    osp = O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode)
    return dict(w=w, g=g, raw=raw, tr=tr, osp=osp, mode=request.param)


def test_c1_translate_1m_vs_oracle_and_reference(c1):
    vas = S.c1_vas()
    hpa, st, aux = c1["tr"].translate_batch(vas)
    v, s, a = O.translate(c1["raw"], c1["osp"], vas, threads=0)
    assert np.array_equal(st, s)
    assert np.array_equal(hpa, v)
    assert np.array_equal(aux, a)
    n = c1["g"]["n_vas"]
    got = [status_outcome(int(st[i]), int(hpa[i]), int(aux[i]), int(vas[i])) for i in range(n)]
    assert got == c1["g"]["expected"]


def test_c1_translate_6m_stage_table_prepass(c1):
    """Batches of >= 8 chunks per CTA take the walker's other arm: per-segment
    stage tables built by the pre-pass (both stages for TDP spaces) and
    grid-stride chunks -- 6 M lanes (10 % outside the region: faults at
    every level) over two segments of the same space, against the oracle."""
    rng = np.random.default_rng(6)
    n = 6 << 20
    vas = np.where(rng.random(n) < 0.9, S.C1_GVA + rng.integers(0, 64 << 20, n),
                   rng.integers(0, 1 << 32, n)).astype(np.uint64)
    tr = c1["tr"]
    img = c1["w"]["memv"].host_mem.backing
    plan = dp.TranslatePlan([tr.device_space], [(0, n // 3, 0), (n // 3, n, 0)], image=img)
    v, s, a = dp.translate_lanes(img, plan, torch.from_numpy(vas.astype(np.uint32).view(np.int32)).cuda())
    ov, os_, oa = O.translate(c1["raw"], c1["osp"], vas, threads=0)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), os_)
    assert np.array_equal(v.cpu().numpy().view(np.uint64), ov)
    assert np.array_equal(a.cpu().numpy().view(np.uint64), oa)
    assert (os_ != 0).any() and (os_ == 0).any()


def test_c1_translate_cached_fifo_replay(c1):
    w = c1["w"]
    vas = S.c1_vas(200_000)
    # mix in a looped 8-page phase so hits and evictions both happen
    loop = np.array([S.C1_GVA + (i % 8) * 4096 + i % 4096 for i in range(20_000)], dtype=np.uint64)
    vas = np.concatenate([vas[:100_000], loop, vas[100_000:]])
    cache = mv.TranslationCache()
    tr = w["memv"].translator(w["space"], cache)
    hpa, st, aux = tr.translate_batch(vas)
    ocache = O.new_cache()
    v, s, a = O.translate_cached(c1["raw"], c1["osp"], vas, ocache)
    assert np.array_equal(st, s) and np.array_equal(hpa, v)
    entries, hits, misses = O.cache_state(ocache)
    assert (cache.hits, cache.misses) == (hits, misses)
    assert cache.entries() == entries


def _c1_copy(c1, gva, length, *, cached: bool, direction: str):
    w = c1["w"]
    data = np.frombuffer(random.Random(3771).randbytes(length), dtype=np.uint8)
    img_ref = c1["raw"].copy()
    cache = mv.TranslationCache()
    tr = w["memv"].translator(w["space"], cache, use_cache=cached)
    host = w["memv"].host_mem
    before = np.frombuffer(S.image_bytes(host), dtype=np.uint8).copy()
    if direction == "to_guest":
        n = mv.copy_user_buffer("to_guest", gva, length, data.tobytes(), translator=tr, host_mem=host)
        oc = O.new_cache() if cached else None
        res = O.copy(before, O.space(*[int(x) for x in c1["osp"]]).reshape(1, 4),
                     np.array([[gva, length, 0, 0]], np.uint64), data.copy(), 0,
                     caches=oc, op_cache=[0] if cached else None)
        assert n == length and int(res[0, 0]) == length
        after = np.frombuffer(S.image_bytes(host), dtype=np.uint8)
        assert np.array_equal(after, before)
        if cached:
            entries, hits, misses = O.cache_state(oc)
            assert (cache.hits, cache.misses, cache.entries()) == (hits, misses, entries)
    else:
        back = bytearray(length)
        n = mv.copy_user_buffer("from_guest", gva, length, back, translator=tr, host_mem=host)
        out = np.zeros(length, np.uint8)
        O.copy(before, O.space(*[int(x) for x in c1["osp"]]).reshape(1, 4),
               np.array([[gva, length, 0, 0]], np.uint64), out, 1)
        assert n == length and bytes(back) == out.tobytes()
    del img_ref


@pytest.mark.parametrize("cached", [False, True])
def test_c1_copy_to_user_64mib(c1, cached):
    _c1_copy(c1, S.C1_GVA, 64 << 20, cached=cached, direction="to_guest")
    _c1_copy(c1, S.C1_GVA + 0x800, (64 << 20) - 4096, cached=cached, direction="to_guest")


def test_c1_copy_from_user_64mib(c1):
    _c1_copy(c1, S.C1_GVA + 0x123, (64 << 20) - 8192, cached=False, direction="from_guest")


def _corrupt(memv, space, mode, seed=1304):
    """C4: 20% of leaf PTEs NOT_PRESENT, 10% TRAPPING (shadow only)."""
    rng = random.Random(seed)
    if mode == "shadow":
        ed = mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
    else:
        g = space.guest
        ed = mv.TableEditor(g.mem, space.guest_root, g.os_alloc.alloc)
    for p in range(S.C1_PAGES):
        r = rng.random()
        va = S.C1_GVA + p * 4096
        if r < 0.2:
            ed.set_leaf_state(va, mv.EntryState.NOT_PRESENT)
        elif r < 0.3 and mode == "shadow":
            ed.set_leaf_state(va, mv.EntryState.TRAPPING)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_c4_fault_heavy_translate_and_copy(cuda, mode):
    w = S.c1_build(mv, be, er, mode)
    memv, space = w["memv"], w["space"]
    _corrupt(memv, space, mode)
    if mode == "tdp":
        # guest PTEs pointing past the slot: TDP-stage faults
        ed = mv.TableEditor(space.guest.mem, space.guest_root, space.guest.os_alloc.alloc)
        for p in range(0, S.C1_PAGES, 97):
            ed.map(S.C1_GVA + p * 4096, (200 << 20) >> 12, replace=True)
    tr = memv.translator(space, use_cache=False)
    sp = tr.device_space
    osp = O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode)
    rng = random.Random(4)
    vas = np.array([S.C1_GVA + rng.randrange(64 << 20) if rng.random() < 0.9 else rng.randrange(1 << 32)
                    for _ in range(300_000)], dtype=np.uint64)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    hpa, st, aux = tr.translate_batch(vas)
    v, s, a = O.translate(raw, osp, vas, threads=0)
    assert np.array_equal(st, s) and np.array_equal(hpa, v) and np.array_equal(aux, a)
    kinds = set((s & 0xFF0).tolist())
    assert 0x010 in kinds and (0x040 in kinds if mode == "shadow" else 0x020 in kinds)
    # a batch of copies that stop at the first bad page, with bytes_copied
    rec = be.GuestProcessRecord(S._Guest(0, mode), space, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    gvas = [S.C1_GVA + rng.randrange(60 << 20) for _ in range(64)]
    lens = [rng.randrange(1, 5 * 4096) for _ in gvas]
    # disjoint destinations: sort and space them
    gvas = [S.C1_GVA + i * (1 << 20) + rng.randrange(4096) for i in range(64)]
    src = np.frombuffer(random.Random(5).randbytes(sum(lens)), dtype=np.uint8)
    outs = acc.copy_to_user_batch(gvas, lens, src.tobytes())
    ops = dp.page_spans  # noqa: F841 (keep import used)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    orows = np.stack([np.array(gvas, np.uint64), np.array(lens, np.uint64), offs, np.zeros(64, np.uint64)], 1)
    oc = O.new_cache()
    res = O.copy(raw, osp.reshape(1, 4), orows, src.copy(), 0, caches=oc, op_cache=[0] * 64)
    after = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8)
    assert np.array_equal(after, raw)
    for o, r in zip(outs, res):
        st_o = int(r[3]) & 0xFFFFFFFF
        if st_o == 0:
            assert o == int(r[1 - 1])
        else:
            assert isinstance(o, Exception)
            if (st_o & 0xFF0) in (0x010, 0x020):
                assert isinstance(o, er.PageFault) and o.bytes_copied == int(r[0])
            elif (st_o & 0xFF0) == 0x040:
                assert isinstance(o, er.TrapExit)
    entries, hits, misses = O.cache_state(oc)
    assert (rec.translation_cache.hits, rec.translation_cache.misses) == (hits, misses)


def test_overlapping_batch_is_last_writer_wins(cuda):
    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, "shadow")
    sp = memv.create_process(g)
    memv.map_region(sp, S.BUF, 16)
    rec = be.GuestProcessRecord(S._Guest(0, "shadow"), sp, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    rng = random.Random(9)
    gvas = [S.BUF + rng.randrange(8 * 4096) for _ in range(40)]
    lens = [rng.randrange(64, 4096) for _ in gvas]
    src = np.frombuffer(random.Random(10).randbytes(sum(lens)), dtype=np.uint8)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    outs = acc.copy_to_user_batch(gvas, lens, src.tobytes())
    assert outs == lens
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    orows = np.stack([np.array(gvas, np.uint64), np.array(lens, np.uint64), offs, np.zeros(40, np.uint64)], 1)
    tr = rec.translator
    s = tr.device_space
    O.copy(raw, O.space(s.s1_base, s.s1_root_pfn).reshape(1, 4), orows, src.copy(), 0)
    assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)


def test_lanes_api_rejects_missing_gpu_never_falls_back(cuda):
    # the data plane is the CUDA library: it must be the thing loaded
    lib = N.lib()
    assert lib.pv_abi_version() == N.ABI_VERSION


def _oracle_of(memv, tr, vas):
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    sp = tr.device_space
    return O.translate(raw, O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode), vas, threads=0)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_leaf_index_coherent_with_host_and_device_writes(cuda, mode):
    """The leaf index is a cache: host edits of indexed leaf nodes, device
    copies that land inside a leaf node, and index on/off all agree with the
    oracle on the current tables."""
    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, mode)
    sp = memv.create_process(g)
    memv.map_region(sp, S.BUF, 600)  # two leaf nodes
    tr = memv.translator(sp, use_cache=False)
    rng = random.Random(12)
    vas = np.array([S.BUF + rng.randrange(700 * 4096) for _ in range(50_000)], dtype=np.uint64)

    def check():
        hpa, st, aux = tr.translate_batch(vas)
        v, s, a = _oracle_of(memv, tr, vas)
        assert np.array_equal(st, s) and np.array_equal(hpa, v)
        space = tr.device_space
        plan = dp.TranslatePlan([space], [(0, len(vas), 0)], use_index=False)
        d = torch.tensor(vas.view(np.int64), device="cuda")
        v2, s2, _ = dp.translate_lanes(memv.host_mem.backing, plan, d)
        assert np.array_equal(s2.cpu().numpy().view(np.uint32), s)
        assert np.array_equal(v2.cpu().numpy().view(np.uint64), v)

    check()
    # host edit of an indexed leaf node
    if mode == "shadow":
        ed = mv.TableEditor(memv.host_mem, sp.shadow_root, memv.host_alloc.alloc)
        ed.set_leaf_state(S.BUF + 7 * 4096, mv.EntryState.TRAPPING)
    else:
        ed = mv.TableEditor(g.mem, sp.guest_root, g.os_alloc.alloc)
    ed.set_leaf_state(S.BUF + 9 * 4096, mv.EntryState.NOT_PRESENT)
    ed.map(S.BUF + 11 * 4096, 0x7FFF_FFFF, replace=True)  # pfn beyond 2^30 -> escape code
    check()
    # a device copy that writes into a leaf node page (shadow: the shadow leaf;
    # tdp: the guest's own leaf node, reached through a driver mapping)
    if mode == "shadow":
        leaf_page = memv.host_mem.read_word(memv.host_mem.read_word(sp.shadow_root.root_pfn, 0) >> 12,
                                            (S.BUF >> 21) & 0x1FF) >> 12
        hpa = leaf_page << 12
    else:
        top = g.mem.read_word(sp.guest_root.root_pfn, 0) >> 12
        leaf_page = g.mem.read_word(top, (S.BUF >> 21) & 0x1FF) >> 12
        hpa = g.base_hpa + (leaf_page << 12)
    memv.map_page_into_guest(sp, 0x5000_0000, hpa, mode)
    words = np.array([(0x1234 + i) << 12 | (1 if i % 3 else 4 if mode == "shadow" else 0) for i in range(64)],
                     dtype=np.uint64)
    n = mv.copy_user_buffer("to_guest", 0x5000_0000 + 8 * 32, 64 * 8, words.tobytes(), translator=tr,
                            host_mem=memv.host_mem)
    assert n == 512
    check()


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_host_pipelined_translate_equals_device_path(cuda, mode):
    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, mode)
    sp = memv.create_process(g)
    memv.map_region(sp, S.BUF, 300)
    tr = memv.translator(sp, use_cache=False)
    rng = np.random.default_rng(3)
    vas = (S.BUF + rng.integers(0, 400 * 4096, 25_000)).astype(np.uint32)
    v, s, a = dp.translate_host_pipelined(memv.host_mem.backing, tr.device_space,
                                          torch.from_numpy(vas.view(np.int32)), chunk=4096)
    hv, hs, ha = tr.translate_batch(vas.astype(np.uint64))
    assert np.array_equal(v.numpy().view(np.uint64), hv)
    assert np.array_equal(s.numpy().view(np.uint32), hs)
    assert np.array_equal(a.numpy().view(np.uint64), ha)
    assert (hs != 0).any() and (hs == 0).any()



def _fifo_world(mode="shadow", pages=40):
    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, mode)
    sp = memv.create_process(g)
    memv.map_region(sp, S.BUF, pages)
    # a page whose PTE points past the image: walk ok, data access OutOfRange
    if mode == "shadow":
        mv.TableEditor(memv.host_mem, sp.shadow_root, memv.host_alloc.alloc).map(S.BUF + pages * 4096, 0xF_FFFF)
    return memv, g, sp


@pytest.mark.parametrize("cap", [1, 3, 10, 32])
@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_parallel_fifo_replay_lanes_vs_sequential_oracle(cuda, cap, mode):
    """K4 over long translate streams: small key sets (hits, evictions,
    re-insertions), faulting keys, and stale initial entries that must win
    over the tables."""
    memv, g, sp = _fifo_world(mode)
    rng = random.Random(cap * 7 + len(mode))
    pages = list(range(0, 50))  # 40 mapped + holes
    vas = np.array([S.BUF + rng.choice(pages[: rng.choice([4, 9, 12, 50])]) * 4096 + rng.randrange(4096)
                    for _ in range(120_000)], dtype=np.uint64)
    stale = [((S.BUF >> 12) + 2, 0x77777), ((S.BUF >> 12) + 45, 0x12345), ((S.BUF >> 12) + 7, 0x55)][:cap]
    cache = mv.TranslationCache(cap)
    for k, v in stale:
        cache.insert(k, v)
    cache.hits, cache.misses = 5, 6
    tr = memv.translator(sp, cache)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    spc = tr.device_space
    ocache = O.new_cache(cap, stale, 5, 6)
    v, s, a = O.translate_cached(raw, O.space(spc.s1_base, spc.s1_root_pfn, spc.s2_root_pfn, spc.mode), vas, ocache)
    hv, hs, ha = tr.translate_batch(vas)
    assert np.array_equal(hs, s) and np.array_equal(hv, v)
    entries, hits, misses = O.cache_state(ocache)
    assert (cache.hits, cache.misses, cache.entries()) == (hits, misses, entries)
    assert 0 < hits < len(vas)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_parallel_fifo_replay_copy_plans_vs_sequential_oracle(cuda, mode):
    """K4 over copy plans: thousands of small ops (1-3 pages) with faults,
    out-of-range data pages and stale entries; ops stop at their first bad
    page, overlapping destinations are last-writer-wins."""
    memv, g, sp = _fifo_world(mode)
    rng = random.Random(99)
    rec = be.GuestProcessRecord(S._Guest(0, mode), sp, memv)
    for k, v in [((S.BUF >> 12) + 3, (S.BUF >> 12) + 999), ((S.BUF >> 12) + 44, 0x1234)]:
        rec.translation_cache.insert(k, v if mode == "tdp" else memv.host_mem.read_word(0, 0) * 0 + 0x1200 + k % 7)
    acc = be.SoftwareHasAccess(rec, memv)
    n_ops = 3000
    gvas = [S.BUF + rng.randrange(46 * 4096) for _ in range(n_ops)]
    lens = [rng.randrange(1, 3 * 4096) for _ in range(n_ops)]
    src = np.frombuffer(random.Random(7).randbytes(sum(lens)), dtype=np.uint8)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    c0 = rec.translation_cache
    ocache = O.new_cache(c0.capacity, c0.entries(), c0.hits, c0.misses)
    outs = acc.copy_to_user_batch(gvas, lens, src.tobytes())
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    rows = np.stack([np.array(gvas, np.uint64), np.array(lens, np.uint64), offs, np.zeros(n_ops, np.uint64)], 1)
    spc = rec.translator.device_space
    res = O.copy(raw, O.space(spc.s1_base, spc.s1_root_pfn, spc.s2_root_pfn, spc.mode).reshape(1, 4), rows,
                 src.copy(), 0, caches=ocache, op_cache=[0] * n_ops)
    assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)
    kinds = set()
    for o, r in zip(outs, res):
        st = int(r[3]) & 0xFFFFFFFF
        kinds.add(st & 0xFF0)
        if st == 0:
            assert o == int(r[0])
        elif (st & 0xFF0) in (0x010, 0x020):
            assert isinstance(o, er.PageFault) and o.bytes_copied == int(r[0])
        elif st == 0x100:
            assert isinstance(o, er.OutOfRange)
    entries, hits, misses = O.cache_state(ocache)
    assert (rec.translation_cache.hits, rec.translation_cache.misses) == (hits, misses)
    assert rec.translation_cache.entries() == entries
    assert 0 in kinds and (0x010 in kinds or 0x020 in kinds)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_parallel_fifo_replay_copy_from_user_batch(cuda, mode):
    """copy_from_user batches never conflict, so the whole batch runs through
    one plan + parallel FIFO replay + exec; compare with the sequential oracle."""
    memv, g, sp = _fifo_world(mode)
    rng = random.Random(5)
    rec = be.GuestProcessRecord(S._Guest(0, mode), sp, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    data = np.frombuffer(random.Random(1).randbytes(40 * 4096), dtype=np.uint8)
    assert acc.copy_to_user(S.BUF, data.tobytes()) == len(data)
    # a stale entry: page 5 -> the frame of page 2 (valid memory, wrong page)
    stale = memv.translator(sp, use_cache=False).translate(S.BUF + 2 * 4096) >> 12
    rec.translation_cache.flush_page((S.BUF >> 12) + 5)
    rec.translation_cache.insert((S.BUF >> 12) + 5, stale)
    n_ops = 5000
    gvas = [S.BUF + rng.randrange(46 * 4096) for _ in range(n_ops)]
    lens = [rng.randrange(1, 3 * 4096) for _ in range(n_ops)]
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    c0 = rec.translation_cache
    ocache = O.new_cache(c0.capacity, c0.entries(), c0.hits, c0.misses)
    payload, outs = acc.copy_from_user_batch(gvas, lens)
    payload = payload.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    rows = np.stack([np.array(gvas, np.uint64), np.array(lens, np.uint64), offs, np.zeros(n_ops, np.uint64)], 1)
    spc = rec.translator.device_space
    obuf = np.zeros(sum(lens), np.uint8)
    res = O.copy(raw, O.space(spc.s1_base, spc.s1_root_pfn, spc.s2_root_pfn, spc.mode).reshape(1, 4), rows,
                 obuf, 1, caches=ocache, op_cache=[0] * n_ops)
    for i, (o, r) in enumerate(zip(outs, res)):
        st = int(r[3]) & 0xFFFFFFFF
        done = int(r[0])
        a = int(offs[i])
        assert np.array_equal(payload[a:a + done], obuf[a:a + done]), i
        if st == 0:
            assert o == lens[i]
        else:
            assert isinstance(o, Exception)
    entries, hits, misses = O.cache_state(ocache)
    assert (rec.translation_cache.hits, rec.translation_cache.misses) == (hits, misses)
    assert rec.translation_cache.entries() == entries


def test_c2_ioctl_trace_ordered_fifo_batch(cuda):
    """BASELINE config 2 (scaled to 80k ops): IOCTL_SNAPSHOT blobs staged
    with copy_to_user into 8 processes' 1 MiB arenas of a TDP guest through
    the software HAS (FIFO-cached translators), heavily overlapping ->
    last-writer-wins.  One device batch (plan + parallel FIFO replay + ordered
    apply) must leave the bytes and cache counters of the sequential oracle."""
    from paper_1304_3771_b200 import workloads as W

    memv, guest, spaces = W.build_c2()
    procs, gvas, lens = W.c2_trace(80_000)
    buf, offs = W.c2_payload(lens)
    trs = [memv.translator(sp, mv.TranslationCache()) for sp in spaces]
    dspaces = [t.device_space for t in trs]
    rows = np.stack([gvas, lens, offs, procs], 1).astype(np.uint64)
    groups = [np.flatnonzero(procs == p) for p in range(len(spaces))]
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    outs = dp.copy_ops(memv.host_mem.backing, dspaces, rows, N.TO_GUEST, torch.from_numpy(buf).cuda(),
                       caches=[t.cache for t in trs], fifo_groups=groups)
    assert all(o.status == 0 and o.copied == int(n) for o, n in zip(outs, lens))
    ocaches = np.stack([O.new_cache() for _ in spaces])
    ospaces = np.stack([O.space(s.s1_base, s.s1_root_pfn, s.s2_root_pfn, s.mode) for s in dspaces])
    O.copy(raw, ospaces, rows, buf.copy(), 0, caches=ocaches, op_cache=procs.astype(np.int32))
    assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)
    for t, oc in zip(trs, ocaches):
        entries, hits, misses = O.cache_state(oc)
        assert (t.cache.hits, t.cache.misses, t.cache.entries()) == (hits, misses, entries)


@pytest.mark.parametrize("seed", [0, 1])
def test_ordered_apply_stress_faults_hot_pages_unaligned(cuda, seed):
    """The ordered (last-writer-wins) path on its corner cases: thousands of
    chunks on a few hot pages (deep per-page streams), every source/destination
    byte alignment, multi-page ops, ops that fault part-way (prefix written,
    later pages dead), zero-length ops and overlapping source ranges -- bytes
    and per-op results equal the sequential oracle."""
    from paper_1304_3771_b200 import workloads as W

    memv, guest, spaces = W.build_c2(3)
    trs = [memv.translator(sp, use_cache=False) for sp in spaces]
    dspaces = [t.device_space for t in trs]
    rng = np.random.default_rng(seed)
    arena = W.C2_ARENA_GVA
    arena_bytes = W.C2_ARENA_PAGES * 4096
    n = 12_000
    kind = rng.integers(0, 10, n)
    gva = np.where(kind < 5, arena + rng.integers(0, 4 * 4096, n),                 # 4 hot pages
                   arena + rng.integers(0, arena_bytes, n))
    ln = np.where(kind < 5, rng.integers(1, 4097, n), rng.integers(0, 3 * 4096 + 77, n))
    tail = kind == 9                                                                   # run off the arena
    gva[tail] = arena + arena_bytes - rng.integers(1, 6000, int(tail.sum()))
    ln[tail] = rng.integers(1, 9000, int(tail.sum()))
    gva[kind == 8] = 0x4000_0000 + rng.integers(0, 1 << 20, int((kind == 8).sum()))  # unmapped: faults at once
    ln[rng.random(n) < 0.01] = 0
    buf_bytes = 1 << 22
    boff = rng.integers(0, buf_bytes - 3 * 4096 - 100, n)
    buf = rng.integers(0, 256, buf_bytes, dtype=np.uint8)
    proc = rng.integers(0, len(spaces), n)
    rows = np.stack([gva, ln, boff, proc], 1).astype(np.uint64)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    outs = dp.copy_ops(memv.host_mem.backing, dspaces, rows, N.TO_GUEST, torch.from_numpy(buf).cuda())
    ospaces = np.stack([O.space(s.s1_base, s.s1_root_pfn, s.s2_root_pfn, s.mode) for s in dspaces])
    ores = O.copy(raw, ospaces, rows, buf.copy(), 0)
    assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)
    got = np.array([[o.copied, o.value, o.aux, o.status | (o.fail_page << 32)] for o in outs], np.uint64)
    assert np.array_equal(got, ores)
    assert {o.status for o in outs} != {0}


def test_resultpage_encode_decode_deliver_batch(cuda):
    """a batch of result records encoded into result pages
    on the device is byte-identical to the reference codec, decodes back, and
    the inline blobs delivered with guest_write semantics (uncached, prefix
    then fault with bytes_copied 0, last writer wins) match the oracle."""
    from paper_1304_3771_b200 import resultpage as rp
    from paper_1304_3771_b200 import workloads as W

    memv, guest, spaces = W.build_c2(4)
    recs = S.resultpage_records()
    rng = random.Random(8)
    # one result page per record: reserved-looking frames high in the slot
    gpas = [(guest.mem.n_pages - 200 + i) << 12 for i in range(len(recs))]
    hpas = [memv.gpa_to_hpa(g, 0) for g in gpas]
    errs = rp.encode_batch(memv.host_mem, hpas, recs)
    assert all(e is None for e in errs)
    for hpa, r in zip(hpas, recs):
        enc = rp.encode(*r)
        assert memv.host_mem.read(hpa, len(enc)) == enc
    dec = rp.decode_batch(memv.host_mem, hpas)
    assert dec == [rp.decode(rp.encode(*r)) for r in recs]
    # delivery into the processes' arenas (overlapping), some unmapped targets
    procs = [rng.randrange(4) for _ in recs]
    gvas = [0 if rng.random() < 0.1 else (W.C2_ARENA_GVA + rng.randrange(W.C2_ARENA_PAGES * 4096 + 8192))
            for _ in recs]
    arena_end = W.C2_ARENA_GVA + W.C2_ARENA_PAGES * 4096
    for i, r in enumerate(recs):  # blobs that run off the arena: fault after a written prefix
        if r[2] and len(r[2]) > 64 and not r[3] and i % 3 == 0:
            gvas[i] = arena_end - 40
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    out = rp.deliver_batch(memv, [spaces[p] for p in procs], hpas, gvas)
    # oracle: guest_write one record after another
    for i, (status, values, blob, staged) in enumerate(recs):
        if not blob or staged or gvas[i] == 0:
            assert out[i] is None
            continue
        tr = memv.translator(spaces[procs[i]], use_cache=False).device_space
        osp = O.space(tr.s1_base, tr.s1_root_pfn, tr.s2_root_pfn, tr.mode).reshape(1, 4)
        res = O.copy(raw, osp, np.array([[gvas[i], len(blob), 0, 0]], np.uint64),
                     np.frombuffer(blob, dtype=np.uint8).copy(), 0)
        st = int(res[0, 3]) & 0xFFFFFFFF
        if st == 0:
            assert out[i] is None
        else:
            assert isinstance(out[i], er.PageFault) and out[i].bytes_copied == 0
    assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)
    assert any(isinstance(o, er.PageFault) for o in out)
    # codec errors
    errs = rp.encode_batch(memv.host_mem, [hpas[0]], [(0, (), b"z" * 4061, False)])
    assert isinstance(errs[0], ValueError)


@pytest.mark.parametrize("va32", [False, True])
@pytest.mark.parametrize("out_pfn", [False, True])
def test_mixed_space_batch_segments_and_lane_formats(cuda, va32, out_pfn):
    """One pv_translate launch over shadow, TDP, hybrid and guest-window
    spaces in ragged segments (including empty ones and segments that end
    mid-chunk), u32 or u64 VAs (u64 with bits >= 32 set: aliasing), address
    or pfn output -- lane by lane against the oracle, with and without the
    leaf index."""
    w = S.walks_build(mv, be, er)
    memv, p0, p1, g1 = w["memv"], w["p0"], w["p1"], w["g1"]
    spaces = [memv.translator(p0, use_cache=False).device_space,
              memv.translator(p1, use_cache=False).device_space,
              dp.Space(0, w["hroot"].root_pfn),
              dp.Space(g1.mem.base, p1.guest_root.root_pfn)]
    rng = random.Random(va32 * 2 + out_pfn)
    sizes = [5000, 0, 2048, 1, 7777, 2047, 4096, 300]
    bounds, lane = [], 0
    vas = []
    for i, n in enumerate(sizes):
        bounds.append((lane, lane + n, i % len(spaces)))
        for _ in range(n):
            va = rng.choice(S.walk_vas()) if rng.random() < 0.5 else S.BUF + rng.randrange(80 * 4096)
            if not va32 and rng.random() < 0.2:
                va |= rng.randrange(1, 1 << 20) << 32
            vas.append(va & 0xFFFFFFFF if va32 else va)
        lane += n
    vas = np.array(vas, dtype=np.uint64)
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    exp_v = np.zeros(len(vas), np.uint64)
    exp_s = np.zeros(len(vas), np.uint32)
    exp_a = np.zeros(len(vas), np.uint64)
    for b, e, si in bounds:
        if e > b:
            s = spaces[si]
            v, st, a = O.translate(raw, O.space(s.s1_base, s.s1_root_pfn, s.s2_root_pfn, s.mode), vas[b:e],
                                   want_pfn=out_pfn, threads=0)
            exp_v[b:e], exp_s[b:e], exp_a[b:e] = v, st, a
    d = torch.tensor(vas.astype(np.uint32).view(np.int32) if va32 else vas.view(np.int64), device="cuda")
    for use_index in (True, False):
        plan = dp.TranslatePlan(spaces, bounds, use_index=use_index)
        v, s, a = dp.translate_lanes(memv.host_mem.backing, plan, d, out_pfn=out_pfn)
        assert np.array_equal(s.cpu().numpy().view(np.uint32), exp_s)
        assert np.array_equal(v.cpu().numpy().view(np.uint64), exp_v)
        assert np.array_equal(a.cpu().numpy().view(np.uint64), exp_a)
    assert len(set((exp_s & 0xFF0).tolist())) >= 4


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_tma_bulk_exec_coaligned_batches_vs_oracle(cuda, mode):
    """The TMA bulk exec (pv_copy.cu exec_bulk_kernel) runs when the host
    proves every op's buffer and guest address co-aligned mod 16: random
    heads (< 16 B through the LSU), 16-byte middles through TMA, random
    tails, ops over 1-6 pages, faulting pages mid-op, both directions,
    against the sequential oracle byte for byte."""
    w = S.c1_build(mv, be, er, mode)
    memv, space = w["memv"], w["space"]
    _corrupt(memv, space, mode)
    tr = memv.translator(space, use_cache=False)
    sp = tr.device_space
    osp = O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode).reshape(1, 4)
    img = memv.host_mem.backing
    rng = random.Random(31 + len(mode))
    n_ops = 700
    res_mod = [rng.randrange(16) for _ in range(n_ops)]
    gv = [S.C1_GVA + i * (96 << 10) + 16 * rng.randrange(256) + res_mod[i] for i in range(n_ops)]
    ln = [rng.choice([rng.randrange(1, 64), rng.randrange(1, 6 * 4096), 4096, 3 * 4096]) for _ in range(n_ops)]
    boff, off = [], 0
    for i in range(n_ops):
        off = (off + 15) // 16 * 16 + res_mod[i]  # buffer offset congruent to the gva mod 16
        boff.append(off)
        off += ln[i]
    rows = np.stack([np.array(gv, np.uint64), np.array(ln, np.uint64), np.array(boff, np.uint64),
                     np.zeros(n_ops, np.uint64)], 1)
    plan = dp.CopyPlan([sp], rows)
    for direction in (N.TO_GUEST, N.FROM_GUEST):
        raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
        src_h = np.frombuffer(random.Random(direction).randbytes(off + 64), dtype=np.uint8).copy()
        buf = torch.from_numpy(src_h.copy()).cuda()
        assert dp.exec_hint(plan, buf.data_ptr()) == N.COPY_ALIGNED16  # the bulk path is the one under test
        dp.copy_launch(img, plan, direction, buf)
        got = plan.results.cpu().numpy().view(np.uint64)
        want = O.copy(raw, osp, rows, src_h, direction)
        assert np.array_equal(got[:, 0], want[:, 0]) and np.array_equal(got[:, 3], want[:, 3])
        if direction == N.TO_GUEST:
            assert int(plan.conflict.item()) == 0
            assert np.array_equal(np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8), raw)
        else:
            assert np.array_equal(buf.cpu().numpy(), src_h)
        kinds = set((want[:, 3] & 0xFF0).tolist())
        assert 0 in kinds and len(kinds) > 1  # complete ops and faulting ops both present


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_c4_device_translate_matches_reference_digest(cuda, mode):
    """The device's outcomes for 100 k VAs over BASELINE config 4 tables fold
    into the digest of the REFERENCE's own translator (tests/golden/
    c4_digest.json, generated from devfsim by tests/golden/gen_golden.py)."""
    g = load_json("c4_digest.json")[mode]
    w = S.c1_build(mv, be, er, mode)
    S.c4_corrupt(mv, w, mode)
    assert S.sha(S.image_bytes(w["memv"].host_mem)) == g["image_sha"]
    tr = w["memv"].translator(w["space"], use_cache=False)
    vas = S.c4_vas(g["n_vas"])
    hpa, st, aux = tr.translate_batch(vas)
    got = [status_outcome(int(st[i]), int(hpa[i]), int(aux[i]), int(vas[i])) for i in range(len(vas))]
    assert got[:50] == g["head"]
    assert S.digest(got) == g["digest"]


def test_c2_staging_device_matches_reference_digest(cuda):
    """The device copy batch (plan, exact parallel FIFO-10 replay, conflict
    stamp, ordered last-writer-wins apply) over the c2_digest trace leaves the
    reference's final memory, outcomes and cache states."""
    g = load_json("c2_digest.json")
    w = S.c2_build(mv, be, er)
    ops = S.c2_ops(g["n_ops"])
    rows, blobs, off = [], [], 0
    for p, gva, ln in ops:
        rows.append((gva, ln, off, p))
        blobs.append(S.snapshot_blob(ln))
        off += ln
    rows = np.array(rows, dtype=np.uint64)
    buf = torch.from_numpy(np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()).cuda()
    memv = w["memv"]
    sps = [memv.translator(sp, use_cache=False).device_space for sp in w["spaces"]]
    caches = [mv.TranslationCache(10) for _ in sps]
    groups = [list(range(p, len(ops), S.C2_PROCS)) for p in range(S.C2_PROCS)]
    outs = dp.copy_ops(memv.host_mem.backing, sps, rows, N.TO_GUEST, buf, caches=caches, fifo_groups=groups)
    got = [["ok", int(o.copied)] if o.status == 0 else ["status", int(o.status)] for o in outs]
    assert got[:50] == g["head"] and S.digest(got) == g["digest"]
    assert S.sha(S.image_bytes(memv.host_mem)) == g["image_sha"]
    for c, (hits, misses, entries) in zip(caches, g["caches"]):
        assert (c.hits, c.misses, [list(x) for x in c.entries()]) == (hits, misses, entries)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_c1_copy_matches_reference_digest(cuda, mode):
    """BASELINE config 1's 64 MiB copy_to_user (aligned, then unaligned at
    +0x800) through the FIFO-cached software HAS on the device leaves the
    memory, outcomes and cache state the reference leaves
    (tests/golden/c1_copy_digest.json)."""
    g = load_json("c1_copy_digest.json")[mode]
    w = S.c1_build(mv, be, er, mode)
    memv = w["memv"]
    rec = be.GuestProcessRecord(S._Guest(0, mode), w["space"], memv)
    acc = be.SoftwareHasAccess(rec, memv)
    data = S.c1_copy_payload()
    out = [S.outcome(lambda: acc.copy_to_user(S.C1_GVA, data), er),
           S.outcome(lambda: acc.copy_to_user(S.C1_GVA + 0x800, data[:(64 << 20) - 4096]), er)]
    assert out == g["outcomes"]
    c = rec.translation_cache
    assert [c.hits, c.misses, [list(e) for e in c.entries()]] == g["cache"]
    assert S.sha(S.image_bytes(memv.host_mem)) == g["image_sha"]
