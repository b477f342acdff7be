"""A/B the copy exec kernel variants on the full C5 copy batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1304_3771_b200 import workloads as W, dataplane as dp, _native as N

cfg = W.C5Config()
wd = W.build_c5(cfg)
img = wd.memv.host_mem.backing
dev = img.device()
spaces, rows, off = [], [], 0
for g in range(cfg.guests):
    for p, ops in enumerate(W.c5_ops(cfg, g)):
        spaces.append(W.c5_hybrid_space(wd, g, p))
        offs = off + np.arange(len(ops), dtype=np.uint64) * np.uint64(cfg.op_bytes)
        rows.append(np.stack([ops[:, 0], ops[:, 1], offs, np.full(len(ops), len(spaces) - 1, np.uint64)], 1))
        off += int(ops[:, 1].sum())
plan = dp.CopyPlan(spaces, np.concatenate(rows))
src = torch.randint(0, 256, (off,), dtype=torch.uint8, device="cuda")
dp.copy_launch(img, plan, N.TO_GUEST, src)
torch.cuda.synchronize()
lib = N.lib()
s = torch.cuda.current_stream()
def run(flags):
    N.check(lib.pv_copy_exec(dev.data_ptr(), img.nbytes, plan.ops.data_ptr(), plan.n_ops, plan.page_off.data_ptr(),
                             plan.n_pages, flags, plan.page_hpa.data_ptr(), plan.page_status.data_ptr(),
                             plan.page_aux.data_ptr(), plan.first_bad.data_ptr(), src.data_ptr(), src.numel(),
                             plan.results.data_ptr(), None, None, s.cuda_stream), "exec")
for name, flags in (("generic", N.TO_GUEST), ("aligned16", N.TO_GUEST | N.COPY_ALIGNED16),
                    ("generic", N.TO_GUEST), ("aligned16", N.TO_GUEST | N.COPY_ALIGNED16)):
    for _ in range(3): run(flags)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): run(flags)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {2 * off / ms / 1e6:.0f} GB/s", flush=True)
