"""C4 walk: (value, status, aux) form vs 4-byte words + exception records, event-timed (not part of the product)."""
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1304_3771_b200 import dataplane as dp
    from paper_1304_3771_b200 import workloads as W

    memv, guest, space = W.build_c1("shadow", device=True)
    W.corrupt_c4(memv, space, "shadow")
    img = memv.host_mem.backing
    rng = random.Random(4)
    vas_h = np.array([W.C1_GVA + rng.randrange(64 << 20) if rng.random() < 0.9 else rng.randrange(1 << 32)
                      for _ in range(1 << 20)], dtype=np.uint32)
    vas = torch.from_numpy(vas_h.view(np.int32)).cuda()
    tr = memv.translator(space, use_cache=False)
    plan = dp.TranslatePlan([tr.device_space], [(0, len(vas_h), 0)], image=img)
    out = (torch.empty(len(vas_h), dtype=torch.int64, device="cuda"), torch.empty(len(vas_h), dtype=torch.int32, device="cuda"),
           torch.zeros(len(vas_h), dtype=torch.int64, device="cuda"))
    w = torch.empty(len(vas_h), dtype=torch.int32, device="cuda")
    xl = dp.ExcList(len(vas_h))
    forms = {"split": lambda: dp.translate_lanes(img, plan, vas, out=out),
             "packed": lambda: dp.translate_lanes(img, plan, vas, out=(out[0], None, out[2]), packed=True),
             "words": lambda: (xl.reset(), dp.translate_words(img, plan, vas, w, xl)),
             "words (no reset)": lambda: dp.translate_words(img, plan, vas, w, xl)}
    for name, fn in forms.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        torch.cuda.synchronize()
        import time
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{name:>18}: {a.elapsed_time(b) / 50 * 1e3:.1f} us per launch (GPU timeline), host enqueue "
              f"{(t1 - t0) / 200 * 1e6:.1f} us per call", flush=True)
    # the same forms replayed from CUDA graphs (no host in the loop)
    for name in ("split", "words"):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            forms[name]()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"{name:>18} graph: {a.elapsed_time(b) / 50 * 1e3:.1f} us per replay", flush=True)


if __name__ == "__main__":
    main()
