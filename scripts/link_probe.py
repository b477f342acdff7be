"""Host-link speed of light for the end-to-end translate leg (not part of the
product): pinned H2D alone, D2H alone and both at once (the translate_many
pipeline moves the VAs in and the lane words out concurrently), for the
byte counts of a C5 step (512 MiB each way in 4-byte words).

    python scripts/link_probe.py [MiB]
"""
import json
import sys

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    n = mib << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    gb = n / 1e9
    print(json.dumps({"bytes_each_way": n, "h2d_ms": t_h2d, "h2d_gbs": gb / t_h2d * 1e3, "d2h_ms": t_d2h,
                      "d2h_gbs": gb / t_d2h * 1e3, "duplex_ms": t_both, "duplex_gbs_each_way": gb / t_both * 1e3,
                      "gpu": torch.cuda.get_device_name()}, indent=1))


if __name__ == "__main__":
    main()
