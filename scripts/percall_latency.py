"""Per-call latency of the drop-in entry points vs the reference.

The reference's drivers call ``ctx.mem.copy_to_user`` once per op and
``ProcessTranslator.translate`` once per page (devices.py:148, 254, 316;
backend.py:92-104; memvirt.py:585-628), so the per-call cost of each entry
point matters next to the batch throughput.  This times, on one box, each
call through this package (B200 data plane) and through the unmodified
reference (pure Python, ``baseline/_ref``), in the same process:

    walk, walk_guest, ProcessTranslator.translate (shadow / TDP, uncached and
    cached), resolve_hybrid, SoftwareHasAccess / HardwareHasAccess
    copy_to_user and copy_from_user of 64 B and 4 KiB.

Prints one JSON object {call: {"ours_us": .., "ref_us": .., "speedup": ..}}
(median of 5 repetitions of N calls each, perf_counter wall time per call).
"""

from __future__ import annotations

import json
import os
import random
import statistics
import sys
import time
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))

BUF = 0x2000_0000


def build(mv, be, mode):
    memv = mv.MemoryVirtualizer(64 << 20)
    guest = memv.add_guest(0, mode, 16 << 20)
    space = memv.create_process(guest)
    memv.map_region(space, BUF, 64)
    rec = be.GuestProcessRecord(types.SimpleNamespace(id=0, mem_mode=mode), space, memv)
    return memv, space, rec


def per_call_us(fn, n, reps=5):
    for _ in range(min(n, 200)):
        fn()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        out.append((time.perf_counter() - t0) / n * 1e6)
    return statistics.median(out)


def calls(mv, be, n):
    rng = random.Random(1)
    vas = [BUF + rng.randrange(63 * 4096) for _ in range(4096)]
    it = iter(range(1 << 60))
    va = lambda: vas[next(it) & 4095]  # noqa: E731
    res = {}
    memv, space, rec = build(mv, be, "shadow")
    tmem, tspace, trec = build(mv, be, "tdp")
    res["walk (shadow table)"] = per_call_us(lambda: mv.walk(memv.host_mem, space.shadow_root.root_pfn, va()), n)
    res["walk_guest"] = per_call_us(lambda: mv.walk_guest(va(), space.guest_root, space.guest.mem), n)
    tr = memv.translator(space, use_cache=False)
    res["translate shadow uncached"] = per_call_us(lambda: tr.translate(va()), n)
    ttr = tmem.translator(tspace, use_cache=False)
    res["translate tdp uncached"] = per_call_us(lambda: ttr.translate(va()), n)
    res["translate shadow cached (FIFO-10, random VAs)"] = per_call_us(lambda: rec.translator.translate(va()), n)
    rec.activate_hybrid(memv)
    res["resolve_hybrid"] = per_call_us(lambda: mv.resolve_hybrid(va(), rec.active_hybrid, memv.host_mem), n)
    sw = be.SoftwareHasAccess(rec, memv)
    hw = be.HardwareHasAccess(rec, memv)
    d64, d4k = bytes(range(64)), bytes(4096)
    res["SoftwareHasAccess.copy_to_user 64 B"] = per_call_us(lambda: sw.copy_to_user(va(), d64), n)
    res["SoftwareHasAccess.copy_to_user 4 KiB"] = per_call_us(lambda: sw.copy_to_user(BUF + 4096 * (next(it) % 60), d4k), n)
    res["SoftwareHasAccess.copy_from_user 4 KiB"] = per_call_us(lambda: sw.copy_from_user(BUF + 4096 * (next(it) % 60), 4096), n)
    res["HardwareHasAccess.copy_to_user 4 KiB"] = per_call_us(lambda: hw.copy_to_user(BUF + 4096 * (next(it) % 60), d4k), n)
    res["HardwareHasAccess.copy_from_user 4 KiB"] = per_call_us(lambda: hw.copy_from_user(BUF + 4096 * (next(it) % 60), 4096), n)
    tsw = be.SoftwareHasAccess(trec, tmem)
    res["SoftwareHasAccess.copy_to_user 4 KiB (tdp)"] = per_call_us(lambda: tsw.copy_to_user(BUF + 4096 * (next(it) % 60) + 0x80, d4k), n)
    return res


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    import devfsim.backend as rb
    import devfsim.memvirt as rm
    import torch

    from paper_1304_3771_b200 import has, memvirt

    from paper_1304_3771_b200 import percall

    ours = calls(memvirt, has, n)  # the resident per-call server (default)
    percall.park()
    percall._SERVER = False
    launch = calls(memvirt, has, n)  # one kernel launch per call (PV_PERCALL_SERVER=0)
    percall._SERVER = True
    torch.cuda.synchronize()
    ref = calls(rm, rb, n)
    out = {k: {"ours_us": round(ours[k], 2), "ours_launch_per_call_us": round(launch[k], 2),
               "ref_us": round(ref[k], 2), "speedup": round(ref[k] / ours[k], 2)}
           for k in ours}
    # where a per-call walk's time goes: the device round trip alone (one launch + result in pinned
    # memory, no translator layers) and a generic GPU round trip (one tiny torch kernel + sync)
    memv, space, _ = build(memvirt, has, "shadow")
    img = memv.host_mem.backing
    sp = memv.translator(space, use_cache=False).device_space
    pc = percall.get()
    floor = {"percall.walk (server: one mailbox round trip)": per_call_us(lambda: pc.walk(img, sp, BUF + 0x123, False), n)}
    percall.park()
    percall._SERVER = False
    floor["percall.walk (one pv_walk_one launch + spin on pinned result)"] = \
        per_call_us(lambda: pc.walk(img, sp, BUF + 0x123, False), n)
    percall._SERVER = True
    x = torch.zeros(1, device="cuda")
    s = torch.cuda.current_stream()
    floor["torch: one tiny kernel + stream synchronize"] = per_call_us(lambda: (x.add_(1), s.synchronize()), n)
    floor = {k: round(v, 2) for k, v in floor.items()}
    print(json.dumps({"calls": out, "device_round_trip_us": floor, "n": n, "gpu": torch.cuda.get_device_name(0),
                      "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t")},
                     indent=1))


if __name__ == "__main__":
    main()
