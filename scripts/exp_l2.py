"""Experiment: walker time at full C5 vs L2 persisting carve-out size."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1304_3771_b200 import dataplane as dp, workloads as W

cfg = W.C5Config()
wd = W.build_c5(cfg)
img = wd.memv.host_mem.backing
img.device()
spaces, bounds, parts = [], [], []
lane = 0
for g in range(cfg.guests):
    for p, v in enumerate(W.c5_vas(cfg, g)):
        spaces.append(W.c5_shadow_space(wd, g, p)); bounds.append((lane, lane + len(v), len(spaces) - 1)); parts.append(v); lane += len(v)
vas = torch.from_numpy(np.concatenate(parts).view(np.int32)).cuda()
plan = dp.TranslatePlan(spaces, bounds)
out = (torch.empty(lane, dtype=torch.int64, device="cuda"), torch.empty(lane, dtype=torch.int32, device="cuda"), torch.zeros(lane, dtype=torch.int64, device="cuda"))
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
prop = torch.cuda.get_device_properties(0)
print("L2", prop.L2_cache_size)
def run(tag):
    for _ in range(3): dp.translate_lanes(img, plan, vas, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): dp.translate_lanes(img, plan, vas, out=out)
    e1.record(); torch.cuda.synchronize()
    print(tag, "ms/launch", e0.elapsed_time(e1) / 10, flush=True)
run("default")
if rt is not None:
    for mb in (32, 64, 96, 120):
        r = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(mb << 20))
        val = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(val), ctypes.c_int(0x06))
        run(f"persist {mb} MiB (rc={r}, limit={val.value>>20} MiB)")
