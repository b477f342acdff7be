"""Extension geometry: 4-level tables with 2 MiB pages (BASELINE config 3).

The reference only has 32-bit VAs, three levels and 4 KiB pages (SURVEY.md
0.1: "64-bit 4-level paging" and "large pages" are explicit non-goals,
README.md:159-162), so this geometry has no reference semantics: it reuses
the reference's entry codec (``target_pfn << 12 | flags``, trapping before
present, writable ignored) over 48-bit VAs split 9/9/9/9/12, and lets a
level-3 entry with ``PS`` (0x80) map a 2 MiB page.  Parity is pinned only by
the C restatement in ``oracle/pvoracle.c`` (``orc_walk4``) -- "parity
unpinned" by the reference.

:class:`Table4` builds such tables on the host mirror (vectorised for large
regions); walks and copies go through the same device entry points as the
reference geometry with ``mode = PV_ONE_STAGE_4L``.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from . import dataplane as dp
from .errors import AlreadyMapped
from .memvirt import FLAG_PRESENT, FLAG_TRAPPING, FLAG_WRITABLE, FrameAllocator, PhysMem

FLAG_PS = N.FLAG_PS
LEVEL_SHIFT = (39, 30, 21, 12)
PAGE = 4096
LARGE = 1 << 21


def indices(va: int) -> tuple[int, int, int, int]:
    return tuple((va >> s) & 0x1FF for s in LEVEL_SHIFT)


class Table4:
    """A 4-level table whose nodes come from ``alloc`` in ``mem``."""

    def __init__(self, mem: PhysMem, alloc: FrameAllocator):
        self.mem = mem
        self.alloc = alloc
        self.root = alloc.alloc()

    @property
    def space(self) -> dp.Space:
        return dp.Space(self.mem.base, self.root, 0, N.ONE_STAGE_4L)

    def _node(self, va: int, depth: int) -> int:
        """Node at ``depth`` (0 = root .. 3 = PT) on va's path, created."""
        node = self.root
        for level in range(depth):
            i = indices(va)[level]
            w = self.mem.read_word(node, i)
            if w & (FLAG_PRESENT | FLAG_TRAPPING):
                node = w >> 12
                continue
            child = self.alloc.alloc()
            self.mem.write_word(node, i, (child << 12) | FLAG_PRESENT | FLAG_WRITABLE)
            node = child
        return node

    def map_4k(self, va: int, pfn: int, *, flags: int = FLAG_PRESENT | FLAG_WRITABLE, replace: bool = False):
        node = self._node(va, 3)
        i = indices(va)[3]
        if not replace and self.mem.read_word(node, i) & (FLAG_PRESENT | FLAG_TRAPPING):
            raise AlreadyMapped(f"{va:#x} already mapped")
        self.mem.write_word(node, i, (pfn << 12) | flags)

    def map_2m(self, va: int, pfn: int, *, flags: int = FLAG_PRESENT | FLAG_WRITABLE, replace: bool = False):
        if va % LARGE or pfn % 512:
            raise ValueError("2 MiB mappings need 2 MiB-aligned va and frame")
        node = self._node(va, 2)
        i = indices(va)[2]
        if not replace and self.mem.read_word(node, i) & (FLAG_PRESENT | FLAG_TRAPPING):
            raise AlreadyMapped(f"{va:#x} already mapped")
        self.mem.write_word(node, i, (pfn << 12) | flags | FLAG_PS)

    def set_entry(self, va: int, level: int, word: int) -> None:
        """Raw write of va's entry at ``level`` (1..4) -- fault injection."""
        node = self._node(va, level - 1)
        self.mem.write_word(node, indices(va)[level - 1], word)

    def map_mixed(self, va0: int, pfn0: int, n_large: int) -> None:
        """``n_large`` 2 MiB regions from va0 -> frames from pfn0: even
        regions as one 2 MiB leaf, odd regions as 512 4 KiB leaves in reversed
        frame order.  Vectorised: node frames are taken up front in VA order."""
        if va0 % LARGE or pfn0 % 512:
            raise ValueError("mixed mappings need 2 MiB alignment")
        mem = self.mem
        img = mem.backing
        words = img.host_for_write(0, 0).view(np.uint64)
        base_w = mem.base // 8
        r = np.arange(n_large, dtype=np.int64)
        vas = va0 + r * LARGE
        l1 = (vas >> 39) & 0x1FF
        l2 = (vas >> 30) & 0x1FF
        l3 = (vas >> 21) & 0x1FF
        # level-2 / level-3 nodes (created in VA order, existing ones reused)
        pd_of = {}
        for a, b in sorted(set(zip(l1.tolist(), l2.tolist()))):
            pd_of[(a, b)] = self._node((a << 39) | (b << 30), 2)
        pd = np.array([pd_of[(a, b)] for a, b in zip(l1.tolist(), l2.tolist())], dtype=np.int64)
        large = (r % 2) == 0
        existing = words[base_w + pd * 512 + l3]
        if ((existing & np.uint64(FLAG_PRESENT | FLAG_TRAPPING)) != 0).any():
            raise AlreadyMapped("mixed region overlaps existing mappings")
        frames = pfn0 + r * 512
        lw = (frames[large].astype(np.uint64) << np.uint64(12)) | np.uint64(FLAG_PRESENT | FLAG_WRITABLE | FLAG_PS)
        words[base_w + pd[large] * 512 + l3[large]] = lw
        # 4 KiB regions: one PT node each
        small = np.flatnonzero(~large)
        pts = self.alloc.alloc_many(len(small))
        words[base_w + pd[small] * 512 + l3[small]] = (pts.astype(np.uint64) << np.uint64(12)) | \
            np.uint64(FLAG_PRESENT | FLAG_WRITABLE)
        j = np.arange(512, dtype=np.int64)
        pt_idx = (base_w + pts[:, None] * 512 + j[None, :]).ravel()
        tgt = (frames[small][:, None] + (511 - j)[None, :]).ravel()
        words[pt_idx] = (tgt.astype(np.uint64) << np.uint64(12)) | np.uint64(FLAG_PRESENT | FLAG_WRITABLE)
        pages = np.unique(np.concatenate([((base_w + pd * 512) * 8) // PAGE, (pt_idx * 8) // PAGE]))
        img.mark_host_pages(pages)


def walk4(mem: PhysMem, root: int, va: int) -> int:
    """Device walk of a 4-level table: the 4 KiB frame of ``va``."""
    status, value, aux = dp.translate_one(mem.backing, dp.Space(mem.base, root, 0, N.ONE_STAGE_4L), va,
                                          out_pfn=True)
    if status:
        dp.raise_for(status, value, aux, va, mem.backing.nbytes)
    return value


# ---- C3 world -----------------------------------------------------------------------

C3_VA = 0x7F00_0000_0000
C3_NODE_BYTES = 64 << 20


def build_c3(region_bytes: int = 16 << 30):
    """BASELINE config 3: ``region_bytes`` of device memory mmapped at C3_VA,
    alternating 2 MiB leaves and 4 KiB leaves.  Image = node pool + region."""
    mem = PhysMem(C3_NODE_BYTES + region_bytes)
    alloc = FrameAllocator(mem, 1, C3_NODE_BYTES // PAGE - 1)
    t = Table4(mem, alloc)
    t.map_mixed(C3_VA, C3_NODE_BYTES // PAGE, region_bytes // LARGE)
    return mem, t


def c3_sequential(region_bytes: int = 16 << 30) -> np.ndarray:
    return (C3_VA + np.arange(0, region_bytes, PAGE, dtype=np.uint64) + np.uint64(0x5A)).astype(np.uint64)


def c3_strided(region_bytes: int = 16 << 30) -> np.ndarray:
    return (C3_VA + np.arange(0, region_bytes, LARGE + PAGE, dtype=np.uint64) + np.uint64(0x18)).astype(np.uint64)


# ---- C1 in 4-level geometry (BASELINE configs[0] as written) ----------------------

C1_4L_VA = 0x7F00_1000_0000
C1_4L_NODE_BYTES = 16 << 20


def build_c1_4l(n_pages: int = 16384, host_bytes: int = 128 << 20, seed: int = 1304):
    """BASELINE configs[0] literally: one address space under a 4-level
    4 KiB page table, 16,384 data pages mapped at C1_4L_VA in
    ``random.Random(1304).shuffle`` order (scattered frames, like the
    reference-geometry C1 of SURVEY.md 8(d)).  Image = node pool + data
    frames; nodes come from the pool's FIFO allocator in VA-walk order."""
    import random

    mem = PhysMem(host_bytes)
    alloc = FrameAllocator(mem, 1, C1_4L_NODE_BYTES // PAGE - 1)
    t = Table4(mem, alloc)
    order = list(range(n_pages))
    random.Random(seed).shuffle(order)
    data0 = C1_4L_NODE_BYTES // PAGE
    for k, p in enumerate(order):
        t.map_4k(C1_4L_VA + p * PAGE, data0 + k)
    return mem, t


def c1_4l_vas(n: int = 1_000_000, seed: int = 3771) -> np.ndarray:
    """Random(3771).randrange(64 MiB) offsets from C1_4L_VA."""
    import random

    rng = random.Random(seed)
    return np.array([C1_4L_VA + rng.randrange(64 << 20) for _ in range(n)], dtype=np.uint64)
