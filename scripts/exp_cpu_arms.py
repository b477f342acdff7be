"""Why the two CPU figures differ (not part of the product): the oracle port's
translation rate over the C5 lanes on the reference arm's host-built world,
on a fresh copy of the same table bytes, and across repeated passes."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench as B
    from oracle import oracle as O

    wl = B._HostOnlyWorkload("c5", 1)
    proc_vas, _ = B._oracle_inputs(wl)
    backing = wl.memv.host_mem.backing
    full = backing.host_for_read()
    span = wl.memv.HOST_PRIVATE_BYTES
    copy_priv = full[:span].copy()
    threads = B.cpu_threads()
    print("threads", threads, "cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))

    def rate(img):
        n = 0
        t0 = time.perf_counter()
        for sp, v in proc_vas:
            O.translate(img, sp, v.astype(np.uint64), threads=threads)
            n += len(v)
        return n / (time.perf_counter() - t0) / 1e9

    for k in range(4):
        print(f"pass {k}: host mirror {rate(full):.3f} G/s | fresh copy of the host-private region {rate(copy_priv):.3f} G/s",
              flush=True)
    for t in (8, 32, 64):
        if t <= len(os.sched_getaffinity(0)):
            threads = t
            print(f"threads {t}: {rate(full):.3f} G/s", flush=True)


if __name__ == "__main__":
    main()
