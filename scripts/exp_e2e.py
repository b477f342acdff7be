"""e2e translate experiments on the C5 world (host tensors in/out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1304_3771_b200 import workloads as W, memvirt as mv, dataplane as dp

cfg = W.C5Config()
wd = W.build_c5(cfg)
wd.memv.host_mem.backing.device()
jobs = []
for g in range(cfg.guests):
    for p, v in enumerate(W.c5_vas(cfg, g)):
        jobs.append((wd.memv.translator(wd.spaces[g][p], use_cache=False), torch.from_numpy(v.view(np.int32)).pin_memory()))
n = sum(t.numel() for _, t in jobs)

def timed(name, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name}: {dt*1e3:.1f} ms  {n/dt/1e9:.2f} G translations/s", flush=True)

timed("translate_batch per process", lambda: [tr.translate_batch(t) for tr, t in jobs])
timed("translate_many", lambda: mv.translate_many(jobs))
for ch in (1 << 20, 1 << 21, 1 << 23):
    timed(f"translate_many chunk={ch}", lambda: mv.translate_many(jobs, chunk=ch))
# raw PCIe reference: pinned H2D of VAs + D2H of 12 B/lane
src = torch.cat([t for _, t in jobs]).pin_memory()
dst = torch.empty(n * 3, dtype=torch.int32, pin_memory=True)
d_src = torch.empty_like(src, device="cuda"); d_dst = torch.empty(n * 3, dtype=torch.int32, device="cuda")
timed("pure PCIe copies (4 B in, 12 B out)", lambda: (d_src.copy_(src, non_blocking=True), dst.copy_(d_dst, non_blocking=True)))
