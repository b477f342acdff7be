"""cProfile of per-call copy_to_user / copy_from_user (not part of the product)."""
import cProfile
import io
import os
import pstats
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1304_3771_b200 import has, memvirt

    memv = memvirt.MemoryVirtualizer(64 << 20)
    guest = memv.add_guest(0, "shadow", 16 << 20)
    space = memv.create_process(guest)
    memv.map_region(space, 0x2000_0000, 64)
    rec = has.GuestProcessRecord(types.SimpleNamespace(id=0, mem_mode="shadow"), space, memv)
    sw = has.SoftwareHasAccess(rec, memv)
    d4k = bytes(4096)
    for i in range(200):
        sw.copy_to_user(0x2000_0000 + 4096 * (i % 60), d4k)
    pr = cProfile.Profile()
    pr.enable()
    for i in range(2000):
        sw.copy_to_user(0x2000_0000 + 4096 * (i % 60), d4k)
    for i in range(2000):
        sw.copy_from_user(0x2000_0000 + 4096 * (i % 60), 4096)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
    print(s.getvalue()[:7000])


if __name__ == "__main__":
    main()
