"""Synthetic worlds and op traces of the BASELINE configurations.

Built with this package's own control plane (whose table bytes are pinned to
the reference by tests/test_control_plane.py), for bench.py and the
large-scale tests.  Config numbering follows BASELINE.json ``configs``:

* C1 -- one guest, 96 MiB slot, 16,384 pages mapped in shuffled order at
  0x1000_0000, 1 M random VAs + a 64 MiB copy_to_user;
* C4 -- C1 tables with 20 % of leaf PTEs not-present and 10 % trapping;
* C5 -- 8 shadow guests x 8 GiB, host-private region raised to 256 MiB,
  3 processes per guest, per guest 16 M random VAs + 1 GiB of copy ops;
  guest g is owned by rank g mod N.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

import numpy as np

from . import dataplane as dp
from . import memvirt as mv

PAGE = 4096
GIB = 1 << 30
MIB = 1 << 20


# ---- C1 / C4 ---------------------------------------------------------------------

C1_HOST = 128 * MIB
C1_GUEST = 96 * MIB
C1_GVA = 0x1000_0000
C1_PAGES = 16384


def build_c1(mode: str = "shadow", device: bool = False):
    memv = mv.MemoryVirtualizer(host_bytes=C1_HOST)
    if device:
        memv.host_mem.backing.device()  # tables built in HBM
    guest = memv.add_guest(0, mode, C1_GUEST)
    space = memv.create_process(guest)
    order = list(range(C1_PAGES))
    random.Random(1304).shuffle(order)
    memv.map_pages(space, np.array([C1_GVA + p * PAGE for p in order], dtype=np.int64))
    return memv, guest, space


def c1_vas(n: int = 1_000_000) -> np.ndarray:
    """Random(3771).randrange(64 MiB) offsets, as in SURVEY.md 8(d)."""
    rng = random.Random(3771)
    return np.array([C1_GVA + rng.randrange(64 * MIB) for _ in range(n)], dtype=np.uint64)


def corrupt_c4(memv, space, mode: str, seed: int = 1304) -> None:
    """20 % of leaf PTEs -> NOT_PRESENT, 10 % -> TRAPPING (shadow only)."""
    rng = random.Random(seed)
    if mode == "shadow":
        ed = mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
    else:
        ed = mv.TableEditor(space.guest.mem, space.guest_root, space.guest.os_alloc.alloc)
    for p in range(C1_PAGES):
        r = rng.random()
        if r < 0.2:
            ed.set_leaf_state(C1_GVA + p * PAGE, mv.EntryState.NOT_PRESENT)
        elif r < 0.3 and mode == "shadow":
            ed.set_leaf_state(C1_GVA + p * PAGE, mv.EntryState.TRAPPING)


# ---- C5 ----------------------------------------------------------------------------

@dataclass
class C5Config:
    guests: int = 8
    guest_bytes: int = 8 * GIB
    host_private: int = 256 * MIB
    procs: int = 3
    pages_per_proc: int = 680_000          # 2.59 GiB mapped per process
    region_gva: int = 0x1000_0000
    vas_per_guest: int = 16 * MIB          # 16,777,216 translations
    copy_bytes_per_guest: int = 1 * GIB
    op_bytes: int = 4 * MIB
    op_offset: int = 0x80                  # ops start 128 B into a page
    seed: int = 5

    def scaled(self, factor: int) -> "C5Config":
        """A proportionally smaller copy (tests only)."""
        return C5Config(self.guests, self.guest_bytes // factor, self.host_private, self.procs,
                        self.pages_per_proc // factor, self.region_gva, self.vas_per_guest // factor,
                        self.copy_bytes_per_guest // factor, self.op_bytes, self.op_offset, self.seed)


@dataclass
class C5World:
    cfg: C5Config
    memv: mv.MemoryVirtualizer
    spaces: list = field(default_factory=list)        # [guest][proc] ProcessSpace
    hybrid_roots: list = field(default_factory=list)  # [guest][proc] PageTableRoot


def c5_slot(cfg: C5Config, g: int) -> tuple[int, int]:
    """Byte range of guest g's slot: the host-private region comes first,
    then the slots in guest order (memvirt.py:433-480 carving)."""
    base = cfg.host_private + g * cfg.guest_bytes
    return base, base + cfg.guest_bytes


def c5_residency(cfg: C5Config, guests) -> list[tuple[int, int]]:
    """What a rank owning ``guests`` holds in HBM: the
    host-private region (every table node of the walks) + its guests' slots."""
    return [(0, cfg.host_private)] + [c5_slot(cfg, g) for g in guests]


def build_c5(cfg: C5Config, device: bool = False, resident_guests=None) -> C5World:
    """The whole 8-guest world (every rank builds the same control plane, so
    hpas are identical across ranks; a rank only touches its own guests'
    pages).  ``device``: allocate the HBM image first so the tables are built
    there (pv_map_plan / pv_map_commit) instead of on the host mirror.
    ``resident_guests``: hold only the host-private region and these guests'
    slots in HBM (a guest-sharded rank); the other guests' tables are built
    on the host mirror and never reach the device."""
    cls = type("C5Virtualizer", (mv.MemoryVirtualizer,), {"HOST_PRIVATE_BYTES": cfg.host_private})
    memv = cls(host_bytes=cfg.host_private + cfg.guests * cfg.guest_bytes)
    if resident_guests is not None:
        memv.host_mem.backing.set_residency(c5_residency(cfg, resident_guests))
    if device:
        memv.host_mem.backing.device()
    world = C5World(cfg, memv)
    for g in range(cfg.guests):
        guest = memv.add_guest(g, "shadow", cfg.guest_bytes)
        row, hrow = [], []
        for _ in range(cfg.procs):
            sp = memv.create_process(guest)
            memv.map_region(sp, cfg.region_gva, cfg.pages_per_proc)
            row.append(sp)
        world.spaces.append(row)
    for g in range(cfg.guests):
        hrow = []
        for sp in world.spaces[g]:
            hrow.append(mv.HybridTopLevel(memv.host_mem, memv.host_alloc).build(sp.shadow_root,
                                                                                 memv.host_kernel_root))
        world.hybrid_roots.append(hrow)
    return world


def c5_shadow_space(world: C5World, g: int, p: int) -> dp.Space:
    return dp.Space(0, world.spaces[g][p].shadow_root.root_pfn)


def c5_hybrid_space(world: C5World, g: int, p: int) -> dp.Space:
    return dp.Space(0, world.hybrid_roots[g][p].root_pfn)


def c5_shim(world: C5World, g: int, p: int) -> dp.Shim:
    """The default trap shim of process p of guest g (backend.py:288-296)."""
    sp = world.spaces[g][p]
    return dp.Shim(sp.guest.base_hpa, sp.guest.mem.size_bytes, sp.guest_root.root_pfn, sp.shadow_root.root_pfn)


def c5_vas(cfg: C5Config, guest: int) -> list[np.ndarray]:
    """Per process of ``guest``: uniform random u32 VAs over its mapped region."""
    rng = np.random.default_rng(cfg.seed * 1000 + guest)
    n = cfg.vas_per_guest
    counts = [n // cfg.procs + (1 if p < n % cfg.procs else 0) for p in range(cfg.procs)]
    span = cfg.pages_per_proc * PAGE
    return [(cfg.region_gva + rng.integers(0, span, size=c, dtype=np.int64)).astype(np.uint32) for c in counts]


def c5_ops(cfg: C5Config, guest: int) -> list[np.ndarray]:
    """Per process of ``guest``: copy ops (gva, len) at distinct slots of the
    mapped region, ``op_offset`` bytes into a page; slots are one op plus two
    pages apart so no two ops touch the same page."""
    rng = random.Random(cfg.seed * 7919 + guest)
    n_ops = cfg.copy_bytes_per_guest // cfg.op_bytes
    stride = cfg.op_bytes + 2 * PAGE
    slots = (cfg.pages_per_proc * PAGE - cfg.op_offset) // stride - 1
    out = []
    per = [n_ops // cfg.procs + (1 if p < n_ops % cfg.procs else 0) for p in range(cfg.procs)]
    for p in range(cfg.procs):
        chosen = rng.sample(range(slots), per[p])
        gvas = np.array([cfg.region_gva + s * stride + cfg.op_offset for s in chosen], dtype=np.uint64)
        lens = np.full(per[p], cfg.op_bytes, dtype=np.uint64)
        out.append(np.stack([gvas, lens], axis=1))
    return out


# ---- C2 ----------------------------------------------------------------------------

C2_ARENA_GVA = 0x2000_0000
C2_ARENA_PAGES = 256
C2_PROCS = 8


def build_c2(n_procs: int = C2_PROCS):
    """One TDP guest, ``n_procs`` processes each with a 256-page arena at
    0x2000_0000."""
    memv = mv.MemoryVirtualizer()
    guest = memv.add_guest(0, "tdp")
    spaces = []
    for _ in range(n_procs):
        sp = memv.create_process(guest)
        memv.map_region(sp, C2_ARENA_GVA, C2_ARENA_PAGES)
        spaces.append(sp)
    return memv, guest, spaces


def c2_trace(n_ops: int, n_procs: int = C2_PROCS, seed: int = 3771):
    """IOCTL_SNAPSHOT trace: op i runs in process i % n_procs with
    arg_len = randint(64, 4096) at arg_gva = arena + randrange(1 MiB - 4096).
    Returns (proc, gva, len) arrays in program order."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(64, 4097, size=n_ops, dtype=np.int64)
    gvas = C2_ARENA_GVA + rng.integers(0, (1 << 20) - 4096, size=n_ops, dtype=np.int64)
    procs = np.arange(n_ops, dtype=np.int64) % n_procs
    return procs, gvas, lens


IOCTL_SNAPSHOT = 0x5A4E  # devices.py:35


def snapshot_blob(n: int) -> np.ndarray:
    """The EventDevice IOCTL_SNAPSHOT result blob (devices.py:162-166)."""
    return ((np.arange(n, dtype=np.int64) * 7 + 3) & 0xFF).astype(np.uint8)


def c2_payload(lens: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Per-op blobs laid out back to back: (buffer, offsets)."""
    offs = np.zeros(len(lens), dtype=np.int64)
    if len(lens) > 1:
        np.cumsum(lens[:-1], out=offs[1:])
    total = int(lens.sum())
    pos = np.arange(total, dtype=np.int64) - np.repeat(offs, lens)
    return ((pos * 7 + 3) & 0xFF).astype(np.uint8), offs
