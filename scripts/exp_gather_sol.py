"""Speed-of-light check: 128 M random 4-byte gathers from a 65 MB array
(the leaf index footprint) with torch's own gather kernel."""
import torch
n, m = 128 << 20, 65323008 // 4
tab = torch.randint(0, 1 << 30, (m,), dtype=torch.int32, device="cuda")
idx = torch.randint(0, m, (n,), dtype=torch.int64, device="cuda")
idx32 = idx.to(torch.int32)
out = torch.empty(n, dtype=torch.int32, device="cuda")
for name, fn in (("index_select int64 idx", lambda: torch.index_select(tab, 0, idx, out=out)),
                 ("take (gather)", lambda: torch.take(tab, idx))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {n/ms/1e6:.1f} G gathers/s", flush=True)
