"""Do small descriptor uploads queue behind a large H2D on another stream (not
part of the product)?  Times 8 x 4 KiB pinned H2D copies on stream B issued
right after a 64 MiB pinned H2D on stream A, and the same small copies done by
a kernel reading mapped pinned memory."""
import time

import torch


def main():
    big_h = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
    big_d = torch.empty_like(big_h, device="cuda")
    small_h = [torch.empty(4096, dtype=torch.uint8).pin_memory() for _ in range(8)]
    small_d = [torch.empty(4096, dtype=torch.uint8, device="cuda") for _ in range(8)]
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    for trial in range(3):
        torch.cuda.synchronize()
        e0, e_big, e_small = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(a)
        b.wait_event(e0)
        with torch.cuda.stream(a):
            big_d.copy_(big_h, non_blocking=True)
            e_big.record(a)
        with torch.cuda.stream(b):
            for h, d in zip(small_h, small_d):
                d.copy_(h, non_blocking=True)
            e_small.record(b)
        torch.cuda.synchronize()
        print(f"trial {trial}: big H2D done at {e0.elapsed_time(e_big):.3f} ms, small copies done at "
              f"{e0.elapsed_time(e_small):.3f} ms")
    # small copies alone
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(b)
    with torch.cuda.stream(b):
        for h, d in zip(small_h, small_d):
            d.copy_(h, non_blocking=True)
    e1.record(b)
    torch.cuda.synchronize()
    print(f"small copies alone: {e0.elapsed_time(e1):.3f} ms")


if __name__ == "__main__":
    main()
