"""The per-call server (include/pv.h pv_server_walk / pv_server_copy_small):
the resident kernel answers the reference's one-call-per-op entry points
exactly like the launch-per-call kernels and the oracle, stays ordered behind
work queued on the caller's stream, exits by itself when idle, and is parked
before batch launches."""

from __future__ import annotations

import threading
import time

import numpy as np
import pytest
import torch

import scenarios as S
from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import has as be
from paper_1304_3771_b200 import memvirt as mv
from paper_1304_3771_b200 import percall
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu


class _G:
    def __init__(self, mode="shadow"):
        self.id, self.mem_mode = 0, mode


def _walks(pc, img, sp, vas):
    return [pc.walk(img, sp, int(v), False) for v in vas]


def _resident_after(call) -> bool:
    """Whether the server is resident right after ``call`` (it leaves on its
    own after 200 us idle: a GC pause between the two may outlast that, so
    a few tries)."""
    lib = N.lib()
    for _ in range(5):
        call()
        if lib.pv_server_resident() == 1:
            return True
    return False


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_server_walks_equal_launches_and_oracle(cuda, mode):
    memv, space = W.build_c1(mode)[0::2]
    W.corrupt_c4(memv, space, mode)
    tr = memv.translator(space, use_cache=False)
    img = memv.host_mem.backing
    sp = tr.device_space
    rng = np.random.default_rng(21)
    vas = np.concatenate([W.C1_GVA + rng.integers(0, 64 << 20, 3000),
                          rng.integers(0, 1 << 32, 500)]).astype(np.uint64)
    pc = percall.get()
    got = _walks(pc, img, sp, vas)
    assert _resident_after(lambda: pc.walk(img, sp, int(vas[0]), False))
    percall.park()
    assert N.lib().pv_server_resident() == 0
    percall._SERVER = False
    try:
        launched = _walks(pc, img, sp, vas)
    finally:
        percall._SERVER = True
    assert got == launched
    raw = np.frombuffer(S.image_bytes(memv.host_mem), dtype=np.uint8).copy()
    v, s, a = O.translate(raw, O.space(sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode), vas, threads=0)
    assert [g[0] for g in got] == s.tolist()
    assert any(g[0] != 0 for g in got)
    ok = s == 0
    assert np.array_equal(np.array([g[1] for g in got], dtype=np.uint64)[ok], v[ok])
    # the public entry point goes through the same server
    for i in range(200):
        if s[i] == 0:
            assert tr.translate(int(vas[i])) == int(v[i])
        else:
            with pytest.raises(Exception):
                tr.translate(int(vas[i]))


def test_server_exits_when_idle_and_device_sync_returns(cuda):
    memv, guest, space = W.build_c1("shadow")
    tr = memv.translator(space, use_cache=False)
    lib = N.lib()
    assert _resident_after(lambda: tr.translate(W.C1_GVA + 5))
    t0 = time.perf_counter()
    torch.cuda.synchronize()  # waits for the server's idle exit, not forever
    assert time.perf_counter() - t0 < 0.5
    assert lib.pv_server_resident() == 0
    # and it comes back on the next call
    assert tr.translate(W.C1_GVA + 5) == tr.translate(W.C1_GVA + 5)
    assert _resident_after(lambda: tr.translate(W.C1_GVA + 5))


def test_server_call_is_ordered_behind_the_callers_stream(cuda):
    """A leaf PTE rewritten on the device by work still queued on the
    caller's stream is what the per-call walk sees (the call takes the
    stream-ordered launch), and the call does not return before that work."""
    memv, guest, space = W.build_c1("shadow", device=True)
    tr = memv.translator(space, use_cache=False)
    hm = memv.host_mem
    va = W.C1_GVA + 7 * 4096 + 0x10
    before = tr.translate(va)
    root = space.shadow_root.root_pfn
    mid = hm.read_word(root, (va >> 30) & 3) >> 12
    leaf = hm.read_word(mid, (va >> 21) & 0x1FF) >> 12
    at = leaf * 4096 + ((va >> 12) & 0x1FF) * 8
    dev = memv.host_mem.backing.device()
    old = dev[at:at + 8].clone()
    new_pfn = (before >> 12) + 3
    word = torch.tensor([new_pfn << 12 | 1], dtype=torch.int64).view(torch.uint8).cuda()
    torch.cuda._sleep(200_000_000)  # ~0.1 s of queued work ahead of the write
    dev[at:at + 8].copy_(word)
    memv.host_mem.backing.note_device_write()  # the image contract for device writes
    t0 = time.perf_counter()
    after = int(percall.get().walk(memv.host_mem.backing, tr.device_space, va, False)[1])
    waited = time.perf_counter() - t0
    assert after == (new_pfn << 12) | (va & 0xFFF)
    assert waited > 0.02
    dev[at:at + 8].copy_(old)
    torch.cuda.synchronize()
    assert tr.translate(va) == before


def test_server_copies_equal_reference_semantics(cuda):
    """copy_to_user / copy_from_user of 64 B .. 16 KiB through the server
    (unaligned, page-crossing, faulting mid-op) match the launch form."""
    results = {}
    for use_server in (True, False):
        percall.park()
        percall._SERVER = use_server
        try:
            memv = mv.MemoryVirtualizer(64 << 20)
            g = memv.add_guest(0, "shadow", 16 << 20)
            sp = memv.create_process(g)
            memv.map_region(sp, S.BUF, 8)  # pages 8.. are unmapped: ops past them fault
            rec = be.GuestProcessRecord(_G(), sp, memv)
            acc = be.SoftwareHasAccess(rec, memv)
            rng = np.random.default_rng(5)
            log = []
            for i in range(300):
                off = int(rng.integers(0, 10 * 4096))
                n = int(rng.choice([64, 4096, 5000, 16384]))
                data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
                try:
                    log.append(("w", acc.copy_to_user(S.BUF + off, data)))
                except Exception as exc:  # noqa: BLE001
                    log.append(("w", type(exc).__name__, getattr(exc, "bytes_copied", None)))
                try:
                    log.append(("r", bytes(acc.copy_from_user(S.BUF + int(rng.integers(0, 9 * 4096)), 3000))))
                except Exception as exc:  # noqa: BLE001
                    log.append(("r", type(exc).__name__, getattr(exc, "bytes_copied", None)))
            results[use_server] = log
        finally:
            percall._SERVER = True
    assert results[True] == results[False]
    assert any(e[1] == "PageFault" for e in results[True] if len(e) == 3)


def test_server_threads(cuda):
    """Per-call walks from four host threads at once (the reference's dual
    threads call ctx.mem concurrently): every answer is its own."""
    memv, guest, space = W.build_c1("shadow")
    tr = memv.translator(space, use_cache=False)
    rng = np.random.default_rng(8)
    vas = (W.C1_GVA + rng.integers(0, 64 << 20, 4 * 500)).astype(np.uint64)
    want = [tr.translate(int(v)) for v in vas]
    got = [None] * len(vas)

    def work(k):
        for i in range(k, len(vas), 4):
            got[i] = tr.translate(int(vas[i]))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got == want


def test_batch_launch_parks_the_server(cuda):
    memv, guest, space = W.build_c1("shadow")
    tr = memv.translator(space, use_cache=False)
    vas = W.c1_vas(100_000)
    assert _resident_after(lambda: tr.translate(W.C1_GVA))
    hpa, st, aux = tr.translate_batch(vas)
    assert N.lib().pv_server_resident() == 0
    assert (st == 0).all()
    assert int(hpa[0]) == tr.translate(int(vas[0]))
