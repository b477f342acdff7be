"""Scripted scenarios run identically against the reference and this package.

Every function takes the module handles ``(mv, be, er)`` -- memvirt-like,
backend-like (HAS access classes, GuestProcessRecord) and errors-like -- so
``tests/golden/gen_golden.py`` can run them on the reference
(``devfsim.memvirt`` / ``devfsim.backend`` / ``devfsim.errors``, imported
from /root/reference in the build container only) to produce the committed
fixtures, and the tests can run them on ``paper_1304_3771_b200`` and compare.

Each scenario has a *build* phase (control plane only: table construction,
allocators, raw word edits -- runs without a GPU) and a *query* phase (data
plane: walks, translations, copies -- needs the GPU for this package).
Outcomes are JSON-able lists.
"""

from __future__ import annotations

import hashlib
import json
import random
import struct

import numpy as np

BUF = 0x2000_0000
PAGE = 4096


class _Guest:
    """Stand-in for devfsim.guest.Guest: GuestProcessRecord reads .id and
    .mem_mode only (backend.py:267-286)."""

    def __init__(self, gid: int, mem_mode: str):
        self.id = gid
        self.mem_mode = mem_mode


def outcome(fn, er):
    try:
        return ["ok", int(fn())]
    except er.PageFault as f:
        return ["fault", int(f.va), int(f.level), int(f.bytes_copied)]
    except er.TrapFixupFailed:
        return ["fixup_failed"]
    except er.TrapExit as t:
        return ["trap", int(t.va), int(t.level), int(t.node_pfn), int(t.index)]
    except er.OutOfRange:
        return ["oor"]
    except struct.error:
        return ["struct"]


def image_bytes(mem) -> bytes:
    """Whole host image as bytes (works for both implementations)."""
    return mem.read(0, mem.size_bytes)


def sparse_pages(raw: bytes):
    arr = np.frombuffer(raw, dtype=np.uint8).reshape(-1, PAGE)
    nz = np.flatnonzero(arr.any(axis=1))
    return nz.astype(np.uint32), arr[nz].copy()


def sha(raw: bytes) -> str:
    return hashlib.sha256(raw).hexdigest()


# ---- scenario "spec": the spec's known answers (test_memvirt.py:111-128)

def spec_build(mv, be, er):
    mem = mv.PhysMem(64 * PAGE)
    alloc = mv.FrameAllocator(mem, 16, 32)
    root = mv.PageTableRoot(mv.TableKind.GUEST, alloc.alloc())
    ed = mv.TableEditor(mem, root, alloc.alloc)
    for page in range(8):
        ed.map(page * PAGE, page)
    mem2 = mv.PhysMem(64 * PAGE)
    # hand-built chain: gva page 5 -> gpa page 9 (root 1, mid 2, leaf 3)
    mem2.write_word(1, 0, (2 << 12) | 0x3)
    mem2.write_word(2, 0, (3 << 12) | 0x3)
    mem2.write_word(3, 5, (9 << 12) | 0x3)
    return dict(mem=mem, root=root, mem2=mem2, root2=mv.PageTableRoot(mv.TableKind.GUEST, 1))


def spec_query(w, mv, be, er):
    out = []
    out.append(outcome(lambda: mv.walk_guest(0x0000_3004, w["root"], w["mem"]), er))
    out.append(outcome(lambda: mv.walk_guest(0x0000_5010, w["root2"], w["mem2"]), er))
    out.append(outcome(lambda: mv.walk_guest(0x0020_0000, w["root2"], w["mem2"]), er))
    out.append(outcome(lambda: mv.walk_guest(0x0000_6000, w["root2"], w["mem2"]), er))
    out.append(outcome(lambda: mv.walk_guest(0xDEAD_B000, mv.PageTableRoot(mv.TableKind.GUEST, 9),
                                             w["mem2"]), er))
    return out


# ---- scenario "walks": shadow + TDP guests, driver maps, corrupted entries

def walks_build(mv, be, er):
    memv = mv.MemoryVirtualizer()
    g0 = memv.add_guest(0, "shadow")
    g1 = memv.add_guest(1, "tdp")
    p0 = memv.create_process(g0)
    p1 = memv.create_process(g1)
    rng = random.Random(1304)
    for sp in (p0, p1):
        memv.map_region(sp, BUF, 40)
        memv.map_region(sp, BUF + 40 * PAGE, 30)        # extends existing nodes
        order = list(range(64))
        rng.shuffle(order)
        for pg in order:
            memv.map_process_page(sp, 0x3000_0000 + pg * PAGE)
        memv.map_region(sp, 0x4020_0000 - 3 * PAGE, 9)  # crosses a mid boundary
    dev = memv.host_alloc.alloc()
    memv.host_mem.write(dev * PAGE, b"\xD5" * 64)
    memv.map_page_into_guest(p0, 0x5000_0000, dev << 12, "shadow")
    memv.map_page_into_guest(p1, 0x5000_0000, dev << 12, "tdp")
    sh = mv.TableEditor(memv.host_mem, p0.shadow_root, memv.host_alloc.alloc)
    sh.set_leaf_state(BUF + 3 * PAGE, mv.EntryState.TRAPPING)
    sh.set_leaf_state(BUF + 5 * PAGE, mv.EntryState.NOT_PRESENT)
    gp1 = mv.TableEditor(g1.mem, p1.guest_root, g1.os_alloc.alloc)
    gp1.set_leaf_state(BUF + 7 * PAGE, mv.EntryState.NOT_PRESENT)
    # guest PTE whose gpa lies beyond the 16 MiB slot: TDP-stage fault
    gp1.map(0x6000_0000, (32 << 20) >> 12)
    # guest PTE whose gpa is inside the slot but beyond... page 0x800 of the slot
    gp1.map(0x6000_1000, 0x800)
    # shadow top entry 2 pointing at a node far past the image: struct.error
    memv.host_mem.write_word(p0.shadow_root.root_pfn, 2, (0xF_FFFF << 12) | 0x3)
    # a trapping top-level entry in a second shadow process
    p2 = memv.create_process(g0)
    memv.map_region(p2, BUF, 4)
    memv.host_mem.write_word(p2.shadow_root.root_pfn, 0,
                             memv.host_mem.read_word(p2.shadow_root.root_pfn, 0) | 0x4)
    hybrid = mv.HybridTopLevel(memv.host_mem, memv.host_alloc)
    hroot = hybrid.build(p0.shadow_root, memv.host_kernel_root)
    return dict(memv=memv, g0=g0, g1=g1, p0=p0, p1=p1, p2=p2, hroot=hroot, dev=dev)


def walk_vas(seed: int = 77, n_random: int = 120) -> list[int]:
    rng = random.Random(seed)
    vas = [BUF + i * PAGE + rng.randrange(PAGE) for i in range(80)]
    vas += [0x3000_0000 + i * PAGE + rng.randrange(PAGE) for i in range(0, 70, 3)]
    vas += [0x4020_0000 + i * PAGE - 3 * PAGE + 5 for i in range(10)]
    vas += [0x5000_0000, 0x5000_0FFF, 0x6000_0010, 0x6000_1234, 0x7000_0000, 0x8000_0000, 0x8123_4567,
            0xC000_0000, 0xC000_0000 + 63 * PAGE + 7, 0xC004_0000, 0xFFFF_FFFF, 0]
    vas += [(1 << 32) | (BUF + 9 * PAGE + 1), (7 << 40) | (BUF + 11 * PAGE)]
    vas += [rng.randrange(1 << 32) for _ in range(n_random)]
    return vas


def walks_query(w, mv, be, er):
    memv, p0, p1, p2 = w["memv"], w["p0"], w["p1"], w["p2"]
    g0, g1 = w["g0"], w["g1"]
    host = memv.host_mem
    vas = walk_vas()
    res = {}
    res["walk_shadow"] = [outcome(lambda: mv.walk(host, p0.shadow_root.root_pfn, va), er) for va in vas]
    res["walk_shadow_p2"] = [outcome(lambda: mv.walk(host, p2.shadow_root.root_pfn, va), er) for va in vas[:40]]
    res["walk_guest0"] = [outcome(lambda: mv.walk_guest(va, p0.guest_root, g0.mem), er) for va in vas]
    res["walk_guest1"] = [outcome(lambda: mv.walk_guest(va, p1.guest_root, g1.mem), er) for va in vas]
    gpas = [v & 0x3FF_FFFF for v in vas] + [16 << 20, (16 << 20) - 1, 1 << 33]
    res["walk_tdp"] = [outcome(lambda: mv.walk(host, g1.tdp_root.root_pfn, gpa), er) for gpa in gpas]
    res["hybrid"] = [outcome(lambda: mv.resolve_hybrid(va, w["hroot"], host), er) for va in vas]
    for name, sp in (("p0", p0), ("p1", p1)):
        unc = memv.translator(sp, use_cache=False)
        res[f"translate_{name}"] = [outcome(lambda: unc.translate(va), er) for va in vas]
        cache = mv.TranslationCache()
        tr = memv.translator(sp, cache)
        seq = vas[:60] + vas[:60] + [BUF + (i % 12) * PAGE + i for i in range(200)]
        res[f"cached_{name}"] = [outcome(lambda: tr.translate(va), er) for va in seq]
        res[f"cached_{name}_state"] = [cache.hits, cache.misses, [list(e) for e in cache.entries()]]
    res["gpa_to_hpa"] = [outcome(lambda: memv.gpa_to_hpa(g, 1), er) for g in gpas[:40]]
    return res


# ---- scenario "copies": user-buffer copies through every translator kind

def copies_build(mv, be, er):
    memv = mv.MemoryVirtualizer()
    g0 = memv.add_guest(0, "shadow")
    g1 = memv.add_guest(1, "tdp")
    p0 = memv.create_process(g0)
    p1 = memv.create_process(g1)
    for sp in (p0, p1):
        memv.map_region(sp, BUF, 24)
        memv.map_region(sp, 0x3000_0000, 3)   # 4th page unmapped
    sh = mv.TableEditor(memv.host_mem, p0.shadow_root, memv.host_alloc.alloc)
    sh.set_leaf_state(BUF + 10 * PAGE, mv.EntryState.TRAPPING)
    r0 = be.GuestProcessRecord(_Guest(0, "shadow"), p0, memv)
    r1 = be.GuestProcessRecord(_Guest(1, "tdp"), p1, memv)
    return dict(memv=memv, p0=p0, p1=p1, r0=r0, r1=r1)


COPY_CASES = [  # (gva, length)
    (BUF, 3 * PAGE), (BUF + 0x800, 12 * 1024), (BUF + 0x123, 5000), (BUF + 4095, 2), (BUF, 0),
    (BUF + 20 * PAGE + 100, 6 * PAGE), (0x3000_0000 + 17, 4 * PAGE), (BUF + 9 * PAGE, 3 * PAGE),
    (BUF + 2 * PAGE + 1, 1), (0x7000_0000, 100), (BUF + 12 * PAGE + 3, 4 * PAGE + 9),
]


def _payload(n: int, seed: int) -> bytes:
    return random.Random(seed).randbytes(n)


def copies_query(w, mv, be, er):
    memv, p0, p1 = w["memv"], w["p0"], w["p1"]
    res = {}
    for name, sp in (("p0", p0), ("p1", p1)):
        for cached in (False, True):
            cache = mv.TranslationCache()
            tr = memv.translator(sp, cache, use_cache=cached)
            rows = []
            for i, (gva, n) in enumerate(COPY_CASES):
                data = _payload(n, 1000 + i)
                rows.append(outcome(lambda: mv.copy_user_buffer("to_guest", gva, n, data, translator=tr,
                                                                host_mem=memv.host_mem), er))
                back = bytearray(n)
                o = outcome(lambda: mv.copy_user_buffer("from_guest", gva, n, back, translator=tr,
                                                        host_mem=memv.host_mem), er)
                rows.append(o + [sha(bytes(back))])
            rows.append([cache.hits, cache.misses, [list(e) for e in cache.entries()]])
            res[f"{name}_{'cached' if cached else 'uncached'}"] = rows
    # access classes: software (cached) and hardware (hybrid + shim) HAS
    for name, rec in (("sw0", w["r0"]), ("sw1", w["r1"])):
        acc = be.SoftwareHasAccess(rec, memv)
        rows = []
        for i, (gva, n) in enumerate(COPY_CASES[:8]):
            data = _payload(n, 2000 + i)
            rows.append(outcome(lambda: acc.copy_to_user(gva, data), er))
            rows.append(outcome(lambda: int.from_bytes(hashlib.sha256(acc.copy_from_user(gva, n)).digest()[:8],
                                                       "little"), er))
        rows.append([rec.translation_cache.hits, rec.translation_cache.misses])
        res[name] = rows
    acc = be.HardwareHasAccess(w["r0"], memv)
    rows = []
    for i, (gva, n) in enumerate(COPY_CASES):
        data = _payload(n, 3000 + i)
        rows.append(outcome(lambda: acc.copy_to_user(gva, data), er))
        rows.append(outcome(lambda: int.from_bytes(hashlib.sha256(acc.copy_from_user(gva, n)).digest()[:8],
                                                   "little"), er))
    rows.append([w["r0"].hw_translations])
    res["hw0"] = rows
    res["image_sha"] = sha(image_bytes(memv.host_mem))
    return res


# ---- scenario "c01": acceptance criterion 1 (test_acceptance.py:90-127)

def c01_build(mv, be, er):
    rng = random.Random(101)
    memv = mv.MemoryVirtualizer()
    guest = memv.add_guest(0, "shadow")
    space = memv.create_process(guest)
    ed = mv.TableEditor(guest.mem, space.guest_root, guest.os_alloc.alloc)
    pages = rng.sample(range(mv.KERNEL_BASE // PAGE), 1500)
    for page in pages:
        ed.map(page * PAGE, rng.randrange(guest.mem.n_pages))
    samples = [page * PAGE + rng.randrange(PAGE) for page in rng.choices(pages, k=5000)]
    samples += [rng.randrange(2 ** 32) for _ in range(5000)]
    return dict(memv=memv, guest=guest, space=space, samples=samples)


def c01_query(w, mv, be, er):
    return [outcome(lambda: mv.walk_guest(va, w["space"].guest_root, w["guest"].mem), er) for va in w["samples"]]


# ---- scenario "c03": hybrid merge (test_acceptance.py:184-224), first trials

def c03_build(mv, be, er, trials: int = 4):
    rng = random.Random(303)
    worlds = []
    for _ in range(trials):
        memv = mv.MemoryVirtualizer()
        memv.add_guest(0, "shadow")
        space = memv.create_process(memv.guest_memory(0))
        se = mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
        user = rng.sample(range(mv.KERNEL_BASE // PAGE), 30)
        trapping = set(rng.sample(user, 5))
        for page in user:
            st = mv.EntryState.TRAPPING if page in trapping else mv.EntryState.PRESENT
            se.map(page * PAGE, memv.host_alloc.alloc(), state=st)
        host_root = mv.PageTableRoot(mv.TableKind.HOST, memv.host_alloc.alloc())
        he = mv.TableEditor(memv.host_mem, host_root, memv.host_alloc.alloc)
        kernel = rng.sample(range(mv.KERNEL_BASE // PAGE, 2 ** 20), 30)
        for page in kernel:
            he.map(page * PAGE, memv.host_alloc.alloc())
        hybrid = mv.HybridTopLevel(memv.host_mem, memv.host_alloc).build(space.shadow_root, host_root)
        vas = [p * PAGE + rng.randrange(PAGE) for p in rng.choices(user + kernel, k=600)]
        vas += [rng.randrange(2 ** 32) for _ in range(450)]
        worlds.append(dict(memv=memv, space=space, host_root=host_root, hybrid=hybrid, vas=vas))
    return worlds


def c03_query(worlds, mv, be, er):
    out = []
    for w in worlds:
        out.append([outcome(lambda: mv.resolve_hybrid(va, w["hybrid"], w["memv"].host_mem), er) for va in w["vas"]])
    return out


# ---- scenario "fifo": cache law traces (test_memvirt.py:509-521; c02)

def fifo_traces():
    rng = random.Random(42)
    traces = []
    for _ in range(200):
        traces.append([rng.randrange(16) for _ in range(rng.randrange(5, 60))])
    rng = random.Random(202)
    for _ in range(300):
        traces.append([rng.randrange(18) for _ in range(rng.randrange(3, 50))])
    return traces


def fifo_query(mv):
    out = []
    for tr in fifo_traces():
        c = mv.TranslationCache()
        for key in tr:
            if c.lookup(key) is None:
                c.insert(key, key * 3 + 1)
        out.append([c.hits, c.misses, [list(e) for e in c.entries()]])
    return out


# ---- C1 (BASELINE config 1, reference geometry): full-size table build

C1_HOST = 128 << 20
C1_GUEST = 96 << 20
C1_GVA = 0x1000_0000
C1_PAGES = 16384


def c1_build(mv, be, er, mode: str):
    memv = mv.MemoryVirtualizer(host_bytes=C1_HOST)
    guest = memv.add_guest(0, mode, C1_GUEST)
    space = memv.create_process(guest)
    order = list(range(C1_PAGES))
    random.Random(1304).shuffle(order)
    if hasattr(memv, "map_pages"):
        memv.map_pages(space, [C1_GVA + p * PAGE for p in order])
    else:
        for p in order:
            memv.map_process_page(space, C1_GVA + p * PAGE)
    return dict(memv=memv, guest=guest, space=space)


def c1_vas(n: int = 1_000_000) -> np.ndarray:
    rng = random.Random(3771)
    return np.array([C1_GVA + rng.randrange(64 << 20) for _ in range(n)], dtype=np.uint64)


# ---- scenario "c4_digest": BASELINE config 4 tables, 100 k VAs, pinned by digest

def c4_corrupt(mv, w, mode: str, seed: int = 1304) -> None:
    """20 % of the C1 leaf PTEs NOT_PRESENT, 10 % TRAPPING (shadow only; the
    reference's TDP tables cannot trap), on the shadow table or the guest
    table (TDP); TDP worlds also get guest PTEs past the slot on every 97th
    page (TDP-stage faults)."""
    memv, space = w["memv"], w["space"]
    rng = random.Random(seed)
    if mode == "shadow":
        ed = mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
    else:
        g = space.guest
        ed = mv.TableEditor(g.mem, space.guest_root, g.os_alloc.alloc)
    for p in range(C1_PAGES):
        r = rng.random()
        va = C1_GVA + p * PAGE
        if r < 0.2:
            ed.set_leaf_state(va, mv.EntryState.NOT_PRESENT)
        elif r < 0.3 and mode == "shadow":
            ed.set_leaf_state(va, mv.EntryState.TRAPPING)
    if mode == "tdp":
        for p in range(0, C1_PAGES, 97):
            ed.map(C1_GVA + p * PAGE, (200 << 20) >> 12, replace=True)


def c4_vas(n: int = 100_000) -> np.ndarray:
    """90 % in the C1 region, 10 % uniform over 2^32 (faults at every level)."""
    rng = random.Random(4404)
    return np.array([C1_GVA + rng.randrange(64 << 20) if rng.random() < 0.9 else rng.randrange(1 << 32)
                     for _ in range(n)], dtype=np.uint64)


def digest(outcomes) -> str:
    return hashlib.sha256(json.dumps(outcomes, separators=(",", ":")).encode()).hexdigest()


# ---- scenario "resultpage": record codec (resultpage.py:44-61)

def resultpage_records():
    rng = random.Random(4060)
    recs = [(0, (), None, False), (14, (4096,), None, False), (0, (1, 2, 3, 4, 5, 6, 7), b"", False),
            (0, (9,), b"\x01\x02\x03", False), (3, (0xFFFFFFFF, 1), bytes(range(256)) * 15, True),
            (0, (len(b"x" * 4060),), b"x" * 4060, False)]
    for _ in range(20):
        n = rng.randrange(0, 4061)
        recs.append((rng.randrange(16), tuple(rng.randrange(1 << 32) for _ in range(rng.randrange(0, 7))),
                     rng.randbytes(n) if rng.random() < 0.8 else None, rng.random() < 0.3))
    return recs


def resultpage_query(rp):
    out = []
    for status, values, blob, staged in resultpage_records():
        enc = rp.encode(status, values, blob, staged)
        d = rp.decode(enc + bytes(64))
        out.append([enc.hex(), d.status, list(d.values), d.blob.hex() if d.blob is not None else None, d.staged])
    try:
        rp.encode(0, (), b"z" * 4061)
        out.append("no error")
    except ValueError:
        out.append("ValueError")
    return out


# ---- scenario "shim": the hybrid resolver's default trap shim (backend.py:117-128,
# 288-296; memvirt.py:685-696) over every kind of trapping shadow entry

ALIAS = 0x2C00_0000   # its shadow mid entry is made to share BUF's leaf node
NOGUEST = 0x3000_0000  # shadow-only trapping leaf: the shim's guest walk faults
MIDTRAP = 0x2800_0000  # trapping shadow mid entry: the retry traps again


def shim_build(mv, be, er):
    memv = mv.MemoryVirtualizer()
    g0 = memv.add_guest(0, "shadow")
    p0 = memv.create_process(g0)
    memv.map_region(p0, BUF, 64)
    memv.map_region(p0, ALIAS, 64)
    memv.map_region(p0, MIDTRAP, 4)
    host = memv.host_mem
    sh = mv.TableEditor(host, p0.shadow_root, memv.host_alloc.alloc)
    for k in (3, 4, 5, 17, 30, 31, 32, 40, 50, 60):
        sh.set_leaf_state(BUF + k * PAGE, mv.EntryState.TRAPPING)
    # ALIAS's shadow mid entry -> BUF's leaf node (two paths to one slot)
    top = host.read_word(p0.shadow_root.root_pfn, 0)
    mid_node = top >> 12
    host.write_word(mid_node, (ALIAS >> 21) & 0x1FF, host.read_word(mid_node, (BUF >> 21) & 0x1FF))
    # a shadow-only trapping leaf (no guest mapping behind it)
    sh.map(NOGUEST, 0x1234, state=mv.EntryState.TRAPPING)
    # a trapping mid entry
    host.write_word(mid_node, (MIDTRAP >> 21) & 0x1FF, host.read_word(mid_node, (MIDTRAP >> 21) & 0x1FF) | 0x4)
    # BUF page 40: the guest maps it past the slot (gpa_to_hpa: OutOfRange)
    gm = g0.mem
    groot = p0.guest_root.root_pfn
    gmid = gm.read_word(groot, 0) >> 12
    gleaf = gm.read_word(gmid, (BUF >> 21) & 0x1FF) >> 12
    gm.write_word(gleaf, 40, ((g0.mem.size_bytes >> 12) + 7) << 12 | 0x3)
    rec = be.GuestProcessRecord(_Guest(0, "shadow"), p0, memv)
    return dict(memv=memv, p0=p0, g0=g0, rec=rec)


SHIM_OPS = [  # (direction, gva, length)
    ("to", ALIAS + 5 * PAGE + 7, 100),      # first reach of the shared slot: fixed from ALIAS's guest page
    ("to", BUF + 2 * PAGE + 100, 4 * PAGE),  # 3, 4 simple traps; 5 reads ALIAS's fix
    ("from", BUF + 3 * PAGE, 2 * PAGE + 9),
    ("to", BUF + 16 * PAGE, 3 * PAGE),
    ("to", NOGUEST + 8, 64),                # shim: walk_guest faults -> PageFault(page va)
    ("to", BUF + 29 * PAGE + 5, 5 * PAGE),
    ("to", MIDTRAP + PAGE, 100),            # retry traps at level 2 -> TrapFixupFailed
    ("to", BUF + 39 * PAGE, 2 * PAGE),      # shim: gpa past the slot -> OutOfRange
    ("to", BUF + 50 * PAGE - 10, 20),
    ("from", BUF + 49 * PAGE, 3 * PAGE),
    ("to", BUF + 70 * PAGE, 10),            # not present
    ("to", BUF + 5 * PAGE, 10),
    ("to", BUF + 59 * PAGE + 1, 2 * PAGE),  # 60 trap, 61 ok
    ("from", ALIAS + 4 * PAGE, 3 * PAGE),
]


def shim_payload(i: int, n: int) -> bytes:
    return _payload(n, 5000 + i)


def shim_query(w, mv, be, er):
    memv, rec = w["memv"], w["rec"]
    acc = be.HardwareHasAccess(rec, memv)
    rows = []
    for i, (d, gva, n) in enumerate(SHIM_OPS):
        if d == "to":
            data = shim_payload(i, n)
            rows.append(outcome(lambda: acc.copy_to_user(gva, data), er))
        else:
            rows.append(outcome(lambda: int.from_bytes(hashlib.sha256(acc.copy_from_user(gva, n)).digest()[:8],
                                                       "little"), er))
    return dict(rows=rows, hw_translations=rec.hw_translations, image_sha=sha(image_bytes(memv.host_mem)))


# ---- scenario "frames": hypercall framing (hypercall.py:110-211)

def frames_ops(hc, n: int = 600, seed: int = 808):
    """Random ops of every kind with random 32-bit words, plus ops whose
    layout words do not fit (unpackable) and page faults with large tags."""
    rng = random.Random(seed)
    kinds = list(hc.FileOpKind)
    ops = []
    for i in range(n):
        kind = rng.choice(kinds)
        vals = {f: rng.randrange(2 ** 32) for f in hc.ARG_LAYOUT[kind]}
        if i % 37 == 5:
            vals[rng.choice(hc.ARG_LAYOUT[kind])] = 2 ** 32 + rng.randrange(1000)
        ops.append(hc.FileOp(kind=kind, **vals))
    return ops


def op_outcome(op):
    if op is None:
        return None
    return [int(op.kind)] + [int(getattr(op, f)) for f in ("device_id", "handle", "gva", "length", "offset", "flags",
                                                               "cmd", "arg_gva", "arg_len", "prot", "event_mask",
                                                               "timeout_ms", "pid", "access", "vma_start",
                                                               "vma_length")]


def frame_outcome(f):
    return [int(f.opcode), [int(a) for a in f.args], int(f.vcpu), int(f.virtual_cr3)]


def exc_name(e) -> str:
    return type(e).__name__


def frames_pack_query(hc):
    out = []
    for i, op in enumerate(frames_ops(hc)):
        try:
            out.append([frame_outcome(f) for f in hc.pack(op, vcpu=i % 4, virtual_cr3=0x40 + (i % 3),
                                                          tag=(i * 2654435761) & 0x1_FFFF_FFFF)])
        except Exception as e:  # noqa: BLE001
            out.append(["err", exc_name(e)])
    return out


def frames_stream(hc, seed: int = 909, n_ops: int = 400):
    """An interleaved frame stream of several (guest, process) sources with
    page faults split across other traffic, reused tags, orphan
    continuations, duplicate first frames and bad opcodes."""
    rng = random.Random(seed)
    srcs = [(0, 1), (0, 2), (1, 1), (1, 7)]
    queue = {s: [] for s in srcs}
    stream = []
    for i, op in enumerate(frames_ops(hc, n_ops, seed)):
        s = srcs[i % len(srcs)]
        try:
            fr = hc.pack(op, vcpu=s[0], virtual_cr3=0x100 * (s[1] + 1), tag=rng.randrange(6))
        except Exception:  # noqa: BLE001
            continue
        queue[s].extend(fr)
        while any(queue.values()) and rng.random() < 0.6:
            q = rng.choice([x for x in srcs if queue[x]])
            stream.append((queue[q].pop(0), q))
        r = rng.random()
        if r < 0.03:
            stream.append((hc.HypercallFrame(hc.OPCODE_CONTINUATION, (rng.randrange(6), 1, 2, 0, 0, 0), 0, 0),
                           rng.choice(srcs)))
        elif r < 0.05:
            stream.append((hc.HypercallFrame(int(hc.FileOpKind.PAGE_FAULT), (rng.randrange(6), 9, 9, 9, 9, 9), 0, 0),
                           rng.choice(srcs)))
        elif r < 0.06:
            stream.append((hc.HypercallFrame(rng.choice([0, 10, 0x7E]), (0,) * 6, 0, 0), rng.choice(srcs)))
    for q in srcs:
        stream.extend((f, q) for f in queue[q])
    return stream


def frames_feed_query(hc):
    asm = hc.FrameAssembler()
    out = []
    for f, (g, p) in frames_stream(hc):
        try:
            out.append(op_outcome(asm.feed(f, g, p)))
        except Exception as e:  # noqa: BLE001
            out.append(["err", exc_name(e)])
    return out


def frames_registry(hc):
    reg = hc.VcpuRegistry()
    for v, g in ((0, 0), (1, 0), (2, 1), (5, 1)):
        reg.register_vcpu(v, g)
    for g, cr3, pid in ((0, 0x100, 11), (0, 0x200, 12), (1, 0x100, 21), (1, 0x800, 22)):
        reg.register_process(g, cr3, pid)
    return reg


def frames_identify_query(hc):
    reg = frames_registry(hc)
    out = []
    for vcpu in range(7):
        for cr3 in (0x100, 0x200, 0x800, 0x999):
            f = hc.HypercallFrame(int(hc.FileOpKind.POLL), (0,) * 6, vcpu, cr3)
            try:
                out.append(list(reg.identify(f)))
            except Exception as e:  # noqa: BLE001
                out.append(["err", exc_name(e)])
    return out


# ---- scenario "c2_digest": BASELINE config 2 staging, pinned by digest

C2_ARENA = 0x2000_0000
C2_PAGES = 256
C2_PROCS = 8


def c2_build(mv, be, er):
    """One TDP guest, 8 processes with a 256-page arena each."""
    memv = mv.MemoryVirtualizer()
    guest = memv.add_guest(0, "tdp")
    spaces = []
    for _ in range(C2_PROCS):
        sp = memv.create_process(guest)
        memv.map_region(sp, C2_ARENA, C2_PAGES)
        spaces.append(sp)
    return dict(memv=memv, guest=guest, spaces=spaces)


def c2_ops(n: int, seed: int = 2022):
    """(proc, gva, len) of an IOCTL_SNAPSHOT trace: op i in process i % 8,
    len randint(64, 4096) at a random arena offset (overlapping writes)."""
    rng = random.Random(seed)
    return [(i % C2_PROCS, C2_ARENA + rng.randrange((1 << 20) - 4096), rng.randint(64, 4096)) for i in range(n)]


def snapshot_blob(n: int) -> bytes:
    """EventDevice IOCTL_SNAPSHOT blob (devices.py:162-166)."""
    return bytes(((j * 7 + 3) & 0xFF) for j in range(n))


def c2_reference_run(w, mv, be, er, ops):
    """copy_to_user of every op's blob in program order through each process's
    FIFO-cached software HAS (backend.py:75-114).  Returns (per-op outcome,
    per-process (hits, misses, entries))."""
    memv = w["memv"]
    recs = [be.GuestProcessRecord(_Guest(0, "tdp"), sp, memv) for sp in w["spaces"]]
    accs = [be.SoftwareHasAccess(r, memv) for r in recs]
    out = [outcome(lambda: accs[p].copy_to_user(gva, snapshot_blob(ln)), er) for p, gva, ln in ops]
    caches = [[r.translation_cache.hits, r.translation_cache.misses, [list(e) for e in r.translation_cache.entries()]]
              for r in recs]
    return out, caches


# ---- scenario "c1_copy_digest": BASELINE config 1's 64 MiB copy_to_user

def c1_copy_payload() -> bytes:
    return random.Random(3771).randbytes(64 << 20)


def c1_copy_reference_run(w, mv, be, er, mode: str):
    """copy_to_user of the 64 MiB payload at the region start, then of its
    first 64 MiB - 4 KiB at +0x800 (unaligned), through the process's
    FIFO-cached software HAS; returns the two outcomes and the cache state."""
    memv = w["memv"]
    rec = be.GuestProcessRecord(_Guest(0, mode), w["space"], memv)
    acc = be.SoftwareHasAccess(rec, memv)
    data = c1_copy_payload()
    out = [outcome(lambda: acc.copy_to_user(C1_GVA, data), er),
           outcome(lambda: acc.copy_to_user(C1_GVA + 0x800, data[:(64 << 20) - 4096]), er)]
    c = rec.translation_cache
    return out, [c.hits, c.misses, [list(e) for e in c.entries()]]
