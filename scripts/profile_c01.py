"""cProfile of the reference's acceptance check c01 (test_acceptance.py:90-127) through the drop-in
(not part of the product): where its 10,000 per-call walk_guest calls and the table edits spend time."""
import cProfile
import io
import os
import pstats
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))


def main():
    from paper_1304_3771_b200.install import install

    install("devfsim")
    from devfsim.errors import PageFault
    from devfsim.memvirt import KERNEL_BASE, PAGE_SIZE, MemoryVirtualizer, TableEditor, walk_guest

    def body():
        t0 = time.perf_counter()
        rng = random.Random(101)
        memv = MemoryVirtualizer()
        guest = memv.add_guest(0, "shadow")
        space = memv.create_process(guest)
        editor = TableEditor(guest.mem, space.guest_root, guest.os_alloc.alloc)
        pages = rng.sample(range(KERNEL_BASE // PAGE_SIZE), 1500)
        for page in pages:
            editor.map(page * PAGE_SIZE, rng.randrange(guest.mem.n_pages))
        t1 = time.perf_counter()
        raw = guest.mem.read(0, guest.mem.size_bytes)
        t2 = time.perf_counter()
        samples = [p * PAGE_SIZE + rng.randrange(PAGE_SIZE) for p in rng.choices(pages, k=5000)]
        samples += [rng.randrange(2**32) for _ in range(5000)]
        for va in samples:
            try:
                walk_guest(va, space.guest_root, guest.mem)
            except PageFault:
                pass
        t3 = time.perf_counter()
        print(f"maps {t1 - t0:.3f} s, read {t2 - t1:.3f} s, 10k walks {t3 - t2:.3f} s", flush=True)

    body()
    pr = cProfile.Profile()
    pr.enable()
    body()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(20)
    print(s.getvalue()[:5000])


if __name__ == "__main__":
    main()
