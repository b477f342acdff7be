"""Randomised parity sweep of the data plane against the CPU oracle.

Each seed builds a small world (shadow or TDP guest, two processes, leaf
PTEs randomly not-present / trapping), then checks against the oracle, lane
by lane and byte by byte:
  * translate batches over both processes in several segments, u32 or u64
    lanes, sized to land on either walker arm (in-kernel staging for small
    batches, the stage-table pre-pass + grid-stride chunks for >= 8 chunks per
    CTA), 15 % of the VAs outside the mapped region;
  * copy batches in both directions whose buffers are 16-byte co-aligned with
    their guest addresses (TMA bulk exec) or not (LSU exec), disjoint or
    overlapping destinations (ordered last-writer-wins path), with faulting
    pages mid-op;
  * a FIFO-cached (software HAS) copy batch over both processes.
"""

from __future__ import annotations

import random

import numpy as np
import pytest
import torch

import scenarios as S
from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import memvirt as mv

SEEDS = list(range(8))


def _world(seed: int):
    rng = random.Random(seed)
    mode = "shadow" if seed % 2 == 0 else "tdp"
    memv = mv.MemoryVirtualizer()
    g = memv.add_guest(0, mode)
    procs = [memv.create_process(g) for _ in range(2)]
    pages = [rng.randrange(24, 64) for _ in procs]
    for sp, n in zip(procs, pages):
        memv.map_region(sp, S.BUF, n)
        if mode == "shadow":
            ed = mv.TableEditor(memv.host_mem, sp.shadow_root, memv.host_alloc.alloc)
        else:
            ed = mv.TableEditor(g.mem, sp.guest_root, g.os_alloc.alloc)
        for p in range(n):
            r = rng.random()
            if r < 0.12:
                ed.set_leaf_state(S.BUF + p * 4096, mv.EntryState.NOT_PRESENT)
            elif r < 0.18 and mode == "shadow":
                ed.set_leaf_state(S.BUF + p * 4096, mv.EntryState.TRAPPING)
    trs = [memv.translator(sp, use_cache=False) for sp in procs]
    return rng, mode, memv, procs, pages, trs


def _raw(memv) -> np.ndarray:
    return np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()


def _ospace(sp: dp.Space) -> np.ndarray:
    return O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_translate_fuzz(cuda, seed):
    rng, mode, memv, procs, pages, trs = _world(seed)
    img = memv.host_mem.backing
    big = seed in (3, 6)  # >= 8 chunks per CTA: the pre-pass arm
    n = (5 << 20) + rng.randrange(1 << 18) if big else rng.randrange(1, 300_000)
    nprng = np.random.default_rng(seed)
    span = max(pages) * 4096 + 8 * 4096
    vas = np.where(nprng.random(n) < 0.85, S.BUF + nprng.integers(0, span, n),
                   nprng.integers(0, 1 << 32, n)).astype(np.uint64)
    # segments: alternate the two processes over random cut points
    cuts = sorted({0, n, *[rng.randrange(n) for _ in range(rng.randrange(1, 5))]})
    bounds = [(a, b, i % 2) for i, (a, b) in enumerate(zip(cuts, cuts[1:])) if b > a]
    spaces = [t.device_space for t in trs]
    plan = dp.TranslatePlan(spaces, bounds, image=img, use_index=rng.random() < 0.8)
    u32 = rng.random() < 0.5
    dv = torch.from_numpy(vas.astype(np.uint32).view(np.int32) if u32 else vas.view(np.int64)).cuda()
    v, s, a = dp.translate_lanes(img, plan, dv)
    v, s, a = (v.cpu().numpy().view(np.uint64), s.cpu().numpy().view(np.uint32), a.cpu().numpy().view(np.uint64))
    raw = _raw(memv)
    for lo, hi, si in bounds:
        ov, os_, oa = O.translate(raw, _ospace(spaces[si]), vas[lo:hi], threads=0)
        assert np.array_equal(s[lo:hi], os_), (seed, lo, hi)
        assert np.array_equal(v[lo:hi], ov), (seed, lo, hi)
        assert np.array_equal(a[lo:hi], oa), (seed, lo, hi)
    assert (s == 0).any() and (s != 0).any()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_copy_fuzz(cuda, seed):
    rng, mode, memv, procs, pages, trs = _world(seed)
    img = memv.host_mem.backing
    spaces = [t.device_space for t in trs]
    coaligned = seed % 4 < 2
    overlap = seed % 3 == 0
    n_ops = rng.randrange(50, 400)
    rows, off = [], 0
    for i in range(n_ops):
        p = rng.randrange(2)
        length = rng.choice([rng.randrange(1, 64), rng.randrange(1, 3 * 4096), 4096])
        limit = (pages[p] + 2) * 4096  # some ops run past the mapped pages: faults mid-op
        if overlap:
            gva = S.BUF + rng.randrange(min(limit, 6 * 4096))
        else:
            gva = S.BUF + (i * (limit // n_ops) // 16) * 16 + rng.randrange(16)
            length = max(1, min(length, limit // n_ops - 32))
        if coaligned:
            off = (off + 15) // 16 * 16 + (gva % 16)
        rows.append((gva, length, off, p))
        off += length + (0 if coaligned else rng.randrange(3))
    rows = np.array(rows, dtype=np.uint64)
    ospaces = np.stack([_ospace(sp) for sp in spaces])
    for direction in (N.TO_GUEST, N.FROM_GUEST):
        raw = _raw(memv)
        buf_h = np.frombuffer(random.Random(seed * 7 + direction).randbytes(off + 64), dtype=np.uint8).copy()
        buf = torch.from_numpy(buf_h.copy()).cuda()
        if coaligned:
            plan = dp.CopyPlan(spaces, rows)
            assert dp.exec_hint(plan, buf.data_ptr()) == N.COPY_ALIGNED16
        outs = dp.copy_ops(img, spaces, rows, direction, buf)
        want = O.copy(raw, ospaces, rows, buf_h, direction, threads=1)  # in order: destinations may overlap
        for o, r in zip(outs, want):
            assert (o.copied, o.status) == (int(r[0]), int(r[3]) & 0xFFFFFFFF), (seed, direction)
            if o.status != 0:
                assert o.fail_page == int(r[3]) >> 32
        if direction == N.TO_GUEST:
            assert np.array_equal(_raw(memv), raw), seed
        else:
            assert np.array_equal(buf.cpu().numpy(), buf_h), seed


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:4])
def test_fifo_cached_copy_fuzz(cuda, seed):
    """Software HAS: per-process FIFO-10 caches replayed exactly over an
    interleaved two-process copy batch (counters and entries too)."""
    rng, mode, memv, procs, pages, trs = _world(seed)
    img = memv.host_mem.backing
    spaces = [t.device_space for t in trs]
    n_ops = rng.randrange(200, 1500)
    rows, off = [], 0
    for i in range(n_ops):
        p = rng.randrange(2)
        gva = S.BUF + rng.randrange((pages[p] + 1) * 4096)
        length = rng.randrange(1, 2 * 4096)
        rows.append((gva, length, off, p))
        off += length
    rows = np.array(rows, dtype=np.uint64)
    caches = [mv.TranslationCache(10) for _ in procs]
    groups = [list(np.flatnonzero(rows[:, 3] == p)) for p in range(2)]
    raw = _raw(memv)
    buf_h = np.frombuffer(random.Random(seed).randbytes(off + 16), dtype=np.uint8).copy()
    outs = dp.copy_ops(img, spaces, rows, N.TO_GUEST, torch.from_numpy(buf_h.copy()).cuda(), caches=caches,
                       fifo_groups=groups)
    oc = np.ascontiguousarray(np.stack([O.new_cache(10) for _ in procs]))
    want = O.copy(raw, np.stack([_ospace(sp) for sp in spaces]), rows, buf_h, N.TO_GUEST, caches=oc,
                  op_cache=rows[:, 3].astype(np.int32))
    for o, r in zip(outs, want):
        assert (o.copied, o.status) == (int(r[0]), int(r[3]) & 0xFFFFFFFF), seed
    assert np.array_equal(_raw(memv), raw), seed
    for p, c in enumerate(caches):
        entries, hits, misses = O.cache_state(oc[p])
        assert (c.entries(), c.hits, c.misses) == (entries, hits, misses), (seed, p)
