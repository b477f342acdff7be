"""Batched table construction on the device (pv_map_plan / pv_map_commit) vs
the reference's per-page map loop.

The device builder runs whenever the image already lives in HBM and a batch
has at least ``memvirt.DEVICE_MAP_MIN`` pages.  Every world below is built
twice -- device builder and host path -- and must be byte-identical; the C1
worlds must also match the image digest recorded from the reference itself.
"""

from __future__ import annotations

import random

import numpy as np
import pytest

import scenarios as S
from conftest import load_json
from paper_1304_3771_b200 import errors as er
from paper_1304_3771_b200 import memvirt as mv

pytestmark = pytest.mark.gpu


def _c1(mode: str, device: bool):
    memv = mv.MemoryVirtualizer(host_bytes=S.C1_HOST)
    if device:
        memv.host_mem.backing.device()
    guest = memv.add_guest(0, mode, S.C1_GUEST)
    space = memv.create_process(guest)
    order = list(range(S.C1_PAGES))
    random.Random(1304).shuffle(order)
    memv.map_pages(space, [S.C1_GVA + p * 4096 for p in order])
    return memv, guest, space


def _raw(memv) -> bytes:
    return S.image_bytes(memv.host_mem)


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_c1_device_build_matches_reference(cuda, mode):
    memv, guest, space = _c1(mode, device=True)
    assert memv.host_mem.backing._dev_dirty_any, "the device builder did not run"
    assert S.sha(_raw(memv)) == load_json(f"c1_{mode}.json")["image_sha"]
    # and the data plane walks the device-built tables
    tr = memv.translator(space, use_cache=False)
    vas = S.c1_vas(20000)
    hpa, st, _ = tr.translate_batch(vas)
    exp = load_json(f"c1_{mode}.json")["expected"]
    got = [["ok", int(h)] if s == 0 else None for h, s in zip(hpa.tolist(), st.tolist())]
    assert got == [e if e[0] == "ok" else None for e in exp]


def test_incremental_maps_reuse_dirty_frames(cuda, monkeypatch):
    """Maps into existing tables (new and existing nodes mixed), with freed
    frames that hold host-written and device-written bytes handed out again
    (they must be zeroed), region after region."""
    worlds = []
    for device in (True, False):
        monkeypatch.setenv("PV_DEVICE_MAP", "1" if device else "0")
        memv = mv.MemoryVirtualizer(host_bytes=160 << 20)
        memv.host_mem.backing.device()
        g = memv.add_guest(0, "shadow", 128 << 20)
        sp = memv.create_process(g)
        memv.map_region(sp, 0x1000_0000, 5000)
        # dirty some frames on both sides, then free them to both allocators
        tr = memv.translator(sp, use_cache=False)
        data = bytes(range(256)) * 64
        for k in range(0, 40, 3):
            mv.copy_user_buffer("to_guest", 0x1000_0000 + k * 4096, len(data), data, translator=tr,
                                host_mem=memv.host_mem)
        for k in range(1, 40, 3):
            g.mem.write(k * 4096 + 100, b"\xAA" * 300)
        for k in range(60):
            g.os_alloc.free(6 + k)
            memv.host_alloc.free(200 + k)
        memv.map_region(sp, 0x1000_0000 + 5000 * 4096, 6000)      # extends into existing + new nodes
        memv.map_region(sp, 0x5000_0000, 4500)                    # a new top entry
        order = list(range(4200))
        random.Random(7).shuffle(order)
        memv.map_pages(sp, [0x8000_0000 + p * 4096 for p in order])
        worlds.append(_raw(memv))
    assert worlds[0] == worlds[1]


def test_device_build_rejects_like_the_loop(cuda, monkeypatch):
    """A batch that repeats a page or hits an already-mapped slot is built by
    the per-page loop: same pages mapped before the error, same exception."""
    outs = []
    for device in (True, False):
        monkeypatch.setenv("PV_DEVICE_MAP", "1" if device else "0")
        memv = mv.MemoryVirtualizer(host_bytes=160 << 20)
        memv.host_mem.backing.device()
        g = memv.add_guest(0, "shadow", 128 << 20)
        sp = memv.create_process(g)
        memv.map_region(sp, 0x1000_0000, 4096)
        res = []
        for gvas in ([0x2000_0000 + p * 4096 for p in range(5000)] + [0x2000_0000 + 17 * 4096],
                     [0x3000_0000 + p * 4096 for p in range(4100)] + [0x1000_0000 + 5 * 4096]):
            try:
                memv.map_pages(sp, gvas)
                res.append("ok")
            except er.AlreadyMapped as e:
                res.append(str(e))
        outs.append((res, _raw(memv)))
    assert outs[0][0] == outs[1][0] and "already mapped" in outs[0][0][0]
    assert outs[0][1] == outs[1][1]


def _digest(memv) -> str:
    import hashlib

    h = hashlib.sha256()
    host = memv.host_mem.backing.host_for_read()
    for s in range(0, len(host), 1 << 28):
        h.update(host[s:s + (1 << 28)])
    return h.hexdigest()


def test_c5_scaled_world_device_equals_host(cuda, monkeypatch):
    """The bench's C5 world (1/32 size: 8 shadow guests, 3 processes each)
    built in HBM is byte-identical to the host-built one."""
    from paper_1304_3771_b200 import workloads as W

    cfg = W.C5Config().scaled(32)
    monkeypatch.setenv("PV_DEVICE_MAP", "1")
    a = W.build_c5(cfg, device=True)
    img = a.memv.host_mem.backing
    assert img._dev_dirty_any or img._pending_any or img.host_epoch > 0
    da = _digest(a.memv)
    del a
    monkeypatch.setenv("PV_DEVICE_MAP", "0")
    b = W.build_c5(cfg, device=False)
    assert da == _digest(b.memv)
