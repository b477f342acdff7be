"""Chunk size of the host translate pipeline (memvirt.translate_many) on the
C5 world, 1 GPU: H2D of VAs / translate / D2H of results overlap per chunk."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1304_3771_b200 import dataplane as dp, memvirt as mv

wl = bench.Workload("c5", 0, 1, 1)
memv = wl.memv
host_vas = [(torch.from_numpy(v.view(np.int32)).pin_memory(), g, p) for g, p, v in wl.proc_vas]
trs = {(g, p): memv.translator(wl.world.spaces[g][p], use_cache=False) for g, p, _ in wl.proc_vas}
pairs = [(trs[(g, p)], t) for t, g, p in host_vas]
n = sum(t.numel() for t, *_ in host_vas)
for chunk in (1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 25):
    mv.translate_many(pairs, chunk=chunk)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        mv.translate_many(pairs, chunk=chunk)
        ts.append(time.perf_counter() - t0)
    b = min(ts)
    print(f"chunk {chunk >> 20} M lanes: best {b*1e3:.1f} ms  {n/b/1e9:.2f} G/s  D2H {dp.last_host_io['d2h']/b/1e9:.1f} GB/s", flush=True)
