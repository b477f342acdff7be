"""Time the C5 translate launch alone (full size), for kernel variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1304_3771_b200 import dataplane as dp, workloads as W

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = W.C5Config() if scale == 1 else W.C5Config().scaled(scale)
wd = W.build_c5(cfg)
img = wd.memv.host_mem.backing
img.device()
spaces, bounds, parts = [], [], []
lane = 0
for g in range(cfg.guests):
    for p, v in enumerate(W.c5_vas(cfg, g)):
        spaces.append(W.c5_shadow_space(wd, g, p)); bounds.append((lane, lane + len(v), len(spaces) - 1)); parts.append(v); lane += len(v)
vas = torch.from_numpy(np.concatenate(parts).view(np.int32)).cuda()
out = (torch.empty(lane, dtype=torch.int64, device="cuda"), torch.empty(lane, dtype=torch.int32, device="cuda"), torch.zeros(lane, dtype=torch.int64, device="cuda"))
for use_index in (True, False):
    plan = dp.TranslatePlan(spaces, bounds, use_index=use_index)
    for _ in range(3): dp.translate_lanes(img, plan, vas, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): dp.translate_lanes(img, plan, vas, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"index={use_index} ms/launch {ms:.3f}  G translations/s {lane/ms/1e6:.1f}", flush=True)
