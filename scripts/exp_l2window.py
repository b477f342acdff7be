"""Experiment: C5 walker with an L2 access-policy window over the leaf index."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1304_3771_b200 import dataplane as dp, workloads as W

class Window(ctypes.Structure):
    _fields_ = [("base_ptr", ctypes.c_void_p), ("num_bytes", ctypes.c_size_t), ("hitRatio", ctypes.c_float),
                ("hitProp", ctypes.c_int), ("missProp", ctypes.c_int)]

class AttrValue(ctypes.Union):
    _fields_ = [("accessPolicyWindow", Window), ("pad", ctypes.c_char * 64)]

rt = ctypes.CDLL("libcudart.so.12")
cfg = W.C5Config()
wd = W.build_c5(cfg)
img = wd.memv.host_mem.backing
img.device()
spaces, bounds, parts, lane = [], [], [], 0
for g in range(cfg.guests):
    for p, v in enumerate(W.c5_vas(cfg, g)):
        spaces.append(W.c5_shadow_space(wd, g, p)); bounds.append((lane, lane + len(v), len(spaces) - 1)); parts.append(v); lane += len(v)
vas = torch.from_numpy(np.concatenate(parts).view(np.int32)).cuda()
out = (torch.empty(lane, dtype=torch.int64, device="cuda"), torch.empty(lane, dtype=torch.int32, device="cuda"), torch.zeros(lane, dtype=torch.int64, device="cuda"))
plan = dp.TranslatePlan(spaces, bounds)
dp.translate_lanes(img, plan, vas, out=out)
codes = img.leaf_index.codes
print("leaf index bytes", codes.numel() * 4, flush=True)
stream = torch.cuda.current_stream()

def run(tag):
    for _ in range(3): dp.translate_lanes(img, plan, vas, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): dp.translate_lanes(img, plan, vas, out=out)
    e1.record(); torch.cuda.synchronize()
    print(tag, f"{e0.elapsed_time(e1)/10:.3f} ms", flush=True)

run("no window")
for mb in (48, 64, 80):
    rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(mb << 20))
    lim = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(lim), ctypes.c_int(0x06))
    v = AttrValue()
    v.accessPolicyWindow.base_ptr = codes.data_ptr()
    v.accessPolicyWindow.num_bytes = min(codes.numel() * 4, lim.value)
    v.accessPolicyWindow.hitRatio = 1.0
    v.accessPolicyWindow.hitProp = 2   # cudaAccessPropertyPersisting
    v.accessPolicyWindow.missProp = 1  # cudaAccessPropertyStreaming
    rc = rt.cudaStreamSetAttribute(ctypes.c_void_p(stream.cuda_stream), ctypes.c_int(1), ctypes.byref(v))
    run(f"window {v.accessPolicyWindow.num_bytes >> 20} MiB (limit {lim.value >> 20} MiB, rc {rc})")
