"""Where the end-to-end copy leg's time goes (not part of the product): one
HardwareHasAccess/SoftwareHasAccess.copy_to_user_batch of a pinned host
payload vs the raw H2D of the same bytes, on the C1 world, and a cProfile of
the call."""
import cProfile
import io
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _G:
    def __init__(self):
        self.id, self.mem_mode = 0, "shadow"


def main():
    import torch

    from paper_1304_3771_b200 import has as be
    from paper_1304_3771_b200 import workloads as W

    memv, guest, space = W.build_c1("shadow", device=True)
    rec = be.GuestProcessRecord(_G(), space, memv)
    acc = be.SoftwareHasAccess(rec, memv)
    n_ops, op = 16, 4 << 20
    src = torch.empty(n_ops * op, dtype=torch.uint8).pin_memory()
    src.random_(0, 256)
    gvas = [W.C1_GVA + i * op for i in range(n_ops)]
    lens = [op] * n_ops
    dev = torch.empty_like(src, device="cuda")

    def call():
        out = acc.copy_to_user_batch(gvas, lens, src)
        assert out == lens

    def h2d():
        dev.copy_(src, non_blocking=True)
        torch.cuda.synchronize()

    for f in (call, h2d):
        for _ in range(3):
            f()
    for name, f in (("copy_to_user_batch (64 MiB pinned)", call), ("raw H2D 64 MiB + sync", h2d)):
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        print(f"{name}: median {np.median(ts) * 1e3:.3f} ms  best {min(ts) * 1e3:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        call()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25)
    print(s.getvalue()[:6000])


if __name__ == "__main__":
    main()
