"""Checks of the drop-in inside the reference's own stack (test infrastructure).

Run as a script in its own process (``install`` rebinds module globals
process-wide): ``python tests/dropin_checks.py <check> [--no-install]``;
prints one JSON object.  The reference package (``devfsim``) comes from the
git-ignored ``baseline/_ref`` (staged by ``__graft_entry__.build()``), which
travels to the GPU box; ``/root/reference`` is never read here.

checks:
* ``identity``  -- the seams the install swaps (no data-plane call; CPU ok)
* ``digests``   -- harness._run_equivalence_script(seed, mode, has) for seeds
                   5/42/77 under the three valid combos (harness.py:650-762)
* ``badaddr``   -- a driver copy that faults partway through the stack:
                   Frontend.vfs_dispatch -> Backend.execute_fileop ->
                   ClassDriver.handle_op -> ctx.mem (devices.py:410-424)
* ``staging``   -- oversized ioctl blobs staged through ctx.mem.copy_to_user
                   (backend.py:526-534) and read back by Frontend.guest_read
                   (frontend.py:212-221), blocking and non-blocking
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

# SURVEY.md §4, recorded from the reference (identical for all 3 combos)
GOLDEN_DIGESTS = {
    5: "f8151df0e2fc8e9d5de628697a0fa86b1dffad18698324265edd8ebf79379744",
    42: "6af506ec98d0fb73822a0aa0e24dc07efcfcfdf1a686268a939c36d7407f581a",
    77: "84daafa72820494802aff5d5e12e3de7e928c7bc81fbd376fe511d1284fbe770",
}
COMBOS = [("blocking", "software"), ("nonblocking", "software"), ("blocking", "hardware")]
BUF = 0x2000_0000


def check_identity() -> dict:
    import devfsim.backend as rb
    import devfsim.errors as re
    import devfsim.memvirt as rm
    import devfsim.world as rw

    from paper_1304_3771_b200 import errors as pe
    from paper_1304_3771_b200 import has, memvirt

    out = {
        "memvirt_swapped": all(getattr(rm, n) is getattr(memvirt, n) for n in (
            "PhysMem", "MemoryVirtualizer", "TableEditor", "TranslationCache", "ProcessTranslator", "walk",
            "walk_guest", "copy_user_buffer", "HybridTopLevel", "resolve_hybrid", "resolve_hybrid_with_fixup")),
        "backend_swapped": all(getattr(rb, n) is getattr(has, n) for n in (
            "SoftwareHasAccess", "HardwareHasAccess", "HostNativeAccess", "_HybridResolver", "GuestProcessRecord")),
        "backend_copy_user_buffer": rb.copy_user_buffer is memvirt.copy_user_buffer,
        "errors_identical": all(getattr(pe, n) is getattr(re, n) for n in (
            "SimError", "PageFault", "TrapExit", "TrapFixupFailed", "OutOfRange", "PoolExhausted", "AlreadyMapped",
            "TdpUnsupported")),
        "memvirt_raises_ref_classes": memvirt.PageFault is re.PageFault and memvirt.PoolExhausted is re.PoolExhausted,
    }
    world = rw.World()
    try:
        out["world_memv"] = type(world.memv) is memvirt.MemoryVirtualizer
        guest = world.add_guest(vcpus=1, mem_mode="shadow")
        process = world.new_process(guest)
        out["space_type"] = type(process.space) is memvirt.ProcessSpace
        process.space.va_next = process.space.va_limit
        try:
            process.space.alloc_va_range(4096)
            out["pool_exhausted_caught"] = False
        except re.PoolExhausted:
            out["pool_exhausted_caught"] = True
        rec = world.backend.record_process_root(guest.id, process.pid)
        out["record_type"] = type(rec) is has.GuestProcessRecord
        out["host_access_type"] = type(world.backend.host_access) is has.HostNativeAccess
    finally:
        world.close()
    return out


def check_digests(seeds=(5, 42, 77)) -> dict:
    from devfsim.harness import _run_equivalence_script

    got = {}
    for seed in seeds:
        for mode, has_mode in COMBOS:
            digest, n = _run_equivalence_script(seed, mode, has_mode)
            got[f"{seed}/{mode}/{has_mode}"] = digest
    ok = all(d == GOLDEN_DIGESTS[int(k.split("/")[0])] for k, d in got.items())
    return {"digests": got, "all_match_golden": ok}


def _fb_world(has_mode: str, mode: str = "blocking", mem_mode: str = "shadow", pages: int = 1):
    from devfsim.devices import FbDevice
    from devfsim.world import World

    world = World(has_mode=has_mode)
    guest = world.add_guest(vcpus=1, mem_mode=mem_mode)
    fb = world.add_device(FbDevice(3, "fb", world.clock))
    world.set_mode(guest, fb, mode)
    process = world.new_process(guest)
    world.map_buffer(process, BUF, pages)
    return world, guest, process


def _run(world, process, fn):
    sys.path.insert(0, os.path.join(REF, "devfsim_tests"))
    box = {}
    thread = world.new_thread(process)

    def body(t):
        try:
            box["result"] = fn(t)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            box["error"] = exc

    thread.start(body)
    thread.join(60.0)
    if "error" in box:
        raise box["error"]
    return box["result"]


def check_badaddr() -> dict:
    from devfsim.hypercall import FileOp, FileOpKind
    from devfsim.workloads import open_device

    out = {}
    for has_mode, mem_mode in (("software", "shadow"), ("software", "tdp"), ("hardware", "shadow")):
        for direction in ("read", "write"):
            world, guest, process = _fb_world(has_mode, mem_mode=mem_mode, pages=1)
            try:
                frontend = world.frontends[guest.id]

                def fn(t):
                    file = frontend.files["/dev/fb"]
                    handle = open_device(frontend, t, file)
                    kind = FileOpKind.READ if direction == "read" else FileOpKind.WRITE
                    # 8 KiB from BUF + 0x800: 2 KiB land in the mapped page, the
                    # next page is not mapped -> PageFault(bytes_copied=2048)
                    res = frontend.vfs_dispatch(t, file, FileOp(kind=kind, handle=handle, gva=BUF + 0x800,
                                                                 length=2 * 4096, offset=0))
                    return int(res.status), list(res.values), frontend.guest_read(t, BUF, 4096).hex()[:64]

                status, values, head = _run(world, process, fn)
                out[f"{has_mode}/{mem_mode}/{direction}"] = {"status": status, "values": values, "head": head}
            finally:
                world.close()
    return out


def check_staging() -> dict:
    import hashlib

    from devfsim import resultpage
    from devfsim.devices import IOCTL_SNAPSHOT, EventDevice
    from devfsim.hypercall import FileOp, FileOpKind
    from devfsim.world import World
    from devfsim.workloads import open_device

    out = {}
    for mode in ("blocking", "nonblocking"):
        for mem_mode in ("shadow", "tdp"):
            world = World()
            try:
                guest = world.add_guest(vcpus=1, mem_mode=mem_mode)
                evt = world.add_device(EventDevice(1, "evt", world.clock))
                world.set_mode(guest, evt, mode)
                process = world.new_process(guest)
                world.map_buffer(process, BUF, 3)
                frontend = world.frontends[guest.id]

                def fn(t):
                    file = frontend.files["/dev/evt"]
                    handle = open_device(frontend, t, file)
                    h = hashlib.sha256()
                    rows = []
                    lens = [64, 600, 4096, resultpage.BLOB_CAPACITY + 1, 3 * 4096 - 0x80]
                    if mode == "blocking":
                        # a blob past the mapped buffer: the staging copy faults
                        # outside handle_op, so the PageFault reaches the caller
                        # (backend.py:526-534); non-blocking it would kill the
                        # dual thread, as in the reference
                        lens.append(3 * 4096)
                    for arg_len in lens:
                        try:
                            res = frontend.vfs_dispatch(t, file, FileOp(kind=FileOpKind.IOCTL, handle=handle,
                                                                         cmd=IOCTL_SNAPSHOT, arg_gva=BUF + 0x80,
                                                                         arg_len=arg_len))
                            rows.append((arg_len, int(res.status), list(res.values)))
                        except Exception as exc:  # noqa: BLE001 - the reference raises here too
                            rows.append((arg_len, type(exc).__name__, str(exc), getattr(exc, "bytes_copied", None)))
                        h.update(frontend.guest_read(t, BUF, 3 * 4096))
                    return rows, h.hexdigest()

                rows, digest = _run(world, process, fn)
                out[f"{mode}/{mem_mode}"] = {"rows": rows, "memory_sha256": digest}
            except BaseException as exc:  # noqa: BLE001 - reported as the outcome
                out[f"{mode}/{mem_mode}"] = {"error": f"{type(exc).__module__}.{type(exc).__name__}: {exc}"}
            finally:
                world.close()
    return out


CHECKS = {"identity": check_identity, "digests": check_digests, "badaddr": check_badaddr,
          "staging": check_staging}


def main(argv) -> None:
    name = argv[1]
    if "--no-install" not in argv:
        from paper_1304_3771_b200.install import install

        install("devfsim")
    print(json.dumps(CHECKS[name](), sort_keys=True))


if __name__ == "__main__":
    main(sys.argv)
