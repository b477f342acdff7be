"""Walker design options of the north star, A/B (not part of the product): the library under PV_LIB
(product / -DPV_TR_WARP_BALLOT=1 / -DPV_TR_DEDUP=1) timed on (a) C4's fault-heavy walk, (b) a hot-page
walk (16 M lanes over 256 pages, every page repeated within a warp), graph-replayed."""
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=30):
    import torch

    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    import torch

    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import workloads as W

    tag = os.path.basename(os.environ.get("PV_LIB", "product"))
    # (a) C4 fault-heavy
    memv, guest, space = W.build_c1("shadow", device=True)
    W.corrupt_c4(memv, space, "shadow")
    img = memv.host_mem.backing
    rng = random.Random(4)
    vas_h = np.array([W.C1_GVA + rng.randrange(64 << 20) if rng.random() < 0.9 else rng.randrange(1 << 32)
                      for _ in range(1 << 20)], dtype=np.uint32)
    tr = memv.translator(space, use_cache=False)
    vas = torch.from_numpy(vas_h.view(np.int32)).cuda()
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas_h), 0)], image=img)
    out = (torch.empty(len(vas_h), dtype=torch.int64, device="cuda"), torch.empty(len(vas_h), dtype=torch.int32, device="cuda"),
           torch.zeros(len(vas_h), dtype=torch.int64, device="cuda"))
    c4 = timed(lambda: dp.translate_lanes(img, plan, vas, out=out))
    ref = out[1].clone()
    # (b) hot pages: 16 M lanes over 256 pages of a clean C1 world
    memv2, guest2, space2 = W.build_c1("shadow", device=True)
    img2 = memv2.host_mem.backing
    tr2 = memv2.translator(space2, use_cache=False)
    r = np.random.default_rng(5)
    hot = (W.C1_GVA + r.integers(0, 256, 16 << 20) * 4096 + r.integers(0, 4096, 16 << 20)).astype(np.uint32)
    vas2 = torch.from_numpy(hot.view(np.int32)).cuda()
    plan2 = dp.TranslatePlan([tr2.device_space], [(0, len(hot), 0)], image=img2)
    w = torch.empty(len(hot), dtype=torch.int32, device="cuda")
    xl = dp.ExcList(4096)
    hotms = timed(lambda: dp.translate_words(img2, plan2, vas2, w, xl))
    print(f"{tag:>22}: C4 fault-heavy walk {c4 * 1e3:.1f} us ({len(vas_h) / c4 / 1e6:.1f} G/s) | hot pages "
          f"{hotms * 1e3:.1f} us ({len(hot) / hotms / 1e6:.1f} G/s)", flush=True)


if __name__ == "__main__":
    main()
