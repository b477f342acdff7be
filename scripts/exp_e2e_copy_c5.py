"""The C5 end-to-end copy leg call by call (not part of the product): per
HardwareHasAccess.copy_to_user_batch wall time vs the raw H2D of its payload,
and a cProfile of the leg."""
import cProfile
import io
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench as B
    from paper_1304_3771_b200 import has

    wl = B.Workload("c5", 0, 1, 1)
    memv = wl.memv
    recs = {}
    for g, p, ops, offs in wl.proc_ops:
        rec = has.GuestProcessRecord(B._FakeGuest(g), wl.world.spaces[g][p], memv)
        rec.hybrid = B._Prebuilt(wl.world.hybrid_roots[g][p])
        recs[(g, p)] = has.HardwareHasAccess(rec, memv)
    payload = [(torch.empty(int(ops[:, 1].sum()), dtype=torch.uint8).pin_memory(), g, p, ops)
               for g, p, ops, offs in wl.proc_ops]
    for t, *_ in payload:
        t.random_(0, 256)

    def leg():
        ts = []
        for t, g, p, ops in payload:
            t0 = time.perf_counter()
            recs[(g, p)].copy_to_user_batch(ops[:, 0], ops[:, 1], t)
            ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        return ts

    leg()
    t0 = time.perf_counter()
    ts = leg()
    total = time.perf_counter() - t0
    nbytes = sum(t.numel() for t, *_ in payload)
    print(f"leg: {total * 1e3:.1f} ms for {nbytes / 1e9:.2f} GB = {nbytes / total / 1e9:.1f} GB/s; calls: "
          f"{len(ts)} x median {np.median(ts) * 1e3:.2f} ms (min {min(ts) * 1e3:.2f}, max {max(ts) * 1e3:.2f})")
    dev = torch.empty(payload[0][0].numel(), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t, *_ in payload:
        dev[:t.numel()].copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    raw = time.perf_counter() - t0
    print(f"raw H2D of the same payloads: {raw * 1e3:.1f} ms = {nbytes / raw / 1e9:.1f} GB/s; "
          f"per payload {raw / len(payload) * 1e3:.2f} ms; ops per call {len(payload[0][3])}")
    pr = cProfile.Profile()
    pr.enable()
    leg()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
    print(s.getvalue()[:5000])


if __name__ == "__main__":
    main()
