"""Drop-in ``memvirt``: page tables, translators and user copies over HBM.

Same public names, signatures, return values and exceptions as the
reference's ``devfsim/memvirt.py``; the design underneath differs:

* physical memory is a :class:`~.image.MemoryImage` (numpy host mirror +
  flat HBM image with page-granular lazy coherence) instead of a bytearray;
* the control plane -- frame allocators, :class:`TableEditor`,
  :class:`MemoryVirtualizer` table construction, the hybrid top-level merge
  -- runs on the host mirror (it is bookkeeping, not the hot path), with a
  vectorised bulk mapper for large regions that reproduces the reference's
  allocation order exactly;
* the data plane -- :func:`walk`, :func:`walk_guest`,
  :meth:`ProcessTranslator.translate` / ``translate_batch``,
  :func:`copy_user_buffer`, :func:`resolve_hybrid` -- runs as sm_100a
  kernels through the C ABI (``include/pv.h``); there is no CPU fallback.

Address geometry (memvirt.py:3-9): 32-bit VAs, 4 KiB pages, three levels
with a 4-entry top table (2/9/9/12); entries are little-endian u64 words
``target_pfn << 12 | flags`` with P=0x1, W=0x2, T=0x4.
"""

from __future__ import annotations

import enum
import struct
import threading
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, NewType

import numpy as np

from . import _native as N
from . import dataplane as dp
from . import percall
from .errors import (
    AlreadyMapped,
    OutOfRange,
    PageFault,
    PoolExhausted,
    TdpUnsupported,
    TrapExit,
    TrapFixupFailed,
)
from .image import MemoryImage

Gva = NewType("Gva", int)
Gpa = NewType("Gpa", int)
Hva = NewType("Hva", int)
Hpa = NewType("Hpa", int)

PAGE_SIZE = 4096
PAGE_SHIFT = 12
PAGE_MASK = PAGE_SIZE - 1
ENTRY_SIZE = 8
TOP_ENTRIES = 4
TABLE_ENTRIES = 512
ADDRESS_BITS = 32
KERNEL_BASE = 0xC000_0000

LEVEL_TOP = 1
LEVEL_MID = 2
LEVEL_LEAF = 3

FLAG_PRESENT = 0x1
FLAG_WRITABLE = 0x2
FLAG_TRAPPING = 0x4

_LE64 = struct.Struct("<Q")


class TableKind(enum.Enum):
    GUEST = "guest"
    SHADOW = "shadow"
    TDP = "tdp"
    HOST = "host"
    HYBRID = "hybrid"


class EntryState(enum.Enum):
    NOT_PRESENT = "not_present"
    PRESENT = "present"
    TRAPPING = "trapping"


@dataclass(frozen=True)
class PageTableEntry:
    state: EntryState
    target_pfn: int
    writable: bool


@dataclass(frozen=True)
class PageTableRoot:
    kind: TableKind
    root_pfn: int
    owner_process: int | None = None


_STATE_BITS = {EntryState.PRESENT: FLAG_PRESENT, EntryState.TRAPPING: FLAG_TRAPPING,
               EntryState.NOT_PRESENT: 0}


def encode_entry(entry: PageTableEntry) -> int:
    """PTE word of ``entry`` (memvirt.py:99-107)."""
    return ((entry.target_pfn << PAGE_SHIFT) | _STATE_BITS[entry.state]
            | (FLAG_WRITABLE if entry.writable else 0))


def entry_state(word: int) -> EntryState:
    """Trapping wins over present (memvirt.py:110-116)."""
    if word & FLAG_TRAPPING:
        return EntryState.TRAPPING
    return EntryState.PRESENT if word & FLAG_PRESENT else EntryState.NOT_PRESENT


def decode_entry(word: int) -> PageTableEntry:
    return PageTableEntry(entry_state(word), word >> PAGE_SHIFT, bool(word & FLAG_WRITABLE))


def split_va(va: int) -> tuple[int, int, int, int]:
    """(top, mid, leaf, offset); top keeps 2 bits so VA bits >= 32 alias."""
    return (va >> 30) & 0x3, (va >> 21) & 0x1FF, (va >> 12) & 0x1FF, va & PAGE_MASK


# ---- physical memory ------------------------------------------------------------

class PhysMem:
    """A window of ``size_bytes`` at byte ``base`` of a :class:`MemoryImage`.

    ``PhysMem(n)`` owns a fresh image; ``PhysMem(n, backing=other.backing,
    base=b)`` aliases another memory, exactly like the reference's guest
    slots (memvirt.py:124-146).  Reads and writes go to the host mirror and
    are bounds-checked against the window; ``read_word`` / ``write_word`` are
    bounded only by the image (the reference leaves them unchecked).
    """

    def __init__(self, size_bytes: int, *, backing=None, base: int = 0):
        if size_bytes % PAGE_SIZE:
            raise ValueError("memory size must be a multiple of the page size")
        if backing is None:
            backing, base = MemoryImage(size_bytes), 0
        elif not isinstance(backing, MemoryImage):
            backing = MemoryImage.adopt(backing)
        if base + size_bytes > backing.nbytes:
            raise OutOfRange("window exceeds backing buffer")
        self._img = backing
        self._base = base
        self.size_bytes = size_bytes

    @property
    def n_pages(self) -> int:
        return self.size_bytes // PAGE_SIZE

    @property
    def backing(self) -> MemoryImage:
        return self._img

    @property
    def base(self) -> int:
        return self._base

    def _check(self, addr: int, length: int) -> None:
        if addr < 0 or addr + length > self.size_bytes:
            raise OutOfRange(f"access [{addr:#x}, +{length}) beyond {self.size_bytes:#x}")

    def read(self, addr: int, length: int) -> bytes:
        self._check(addr, length)
        off = self._base + addr
        return self._img.host_for_read(off, off + length)[off:off + length].tobytes()

    def write(self, addr: int, data) -> None:
        data = bytes(data)
        self._check(addr, len(data))
        off = self._base + addr
        host = self._img.host_for_write(off, off + len(data))
        host[off:off + len(data)] = np.frombuffer(data, dtype=np.uint8)

    def read_word(self, pfn: int, index: int) -> int:
        off = self._base + pfn * PAGE_SIZE + index * ENTRY_SIZE
        return _LE64.unpack_from(self._img.host_for_read(off, off + ENTRY_SIZE), off)[0]

    def write_word(self, pfn: int, index: int, word: int) -> None:
        off = self._base + pfn * PAGE_SIZE + index * ENTRY_SIZE
        if off < 0 or off + ENTRY_SIZE > self._img.nbytes:
            raise struct.error(f"pack_into requires a buffer of at least {off + ENTRY_SIZE} bytes")
        _LE64.pack_into(self._img.host_for_write(off, off + ENTRY_SIZE), off, word)

    def zero_page(self, pfn: int) -> None:
        self._check(pfn * PAGE_SIZE, PAGE_SIZE)
        self._img.zero_pages(np.array([(self._base >> PAGE_SHIFT) + pfn], dtype=np.int64))

    def dump_hex(self, pfn: int) -> str:
        """32 bytes per line, address-prefixed (memvirt.py:181-188)."""
        raw = self.read(pfn * PAGE_SIZE, PAGE_SIZE)
        start = pfn * PAGE_SIZE
        return "\n".join(f"{start + i:08x}  {raw[i:i + 32].hex()}" for i in range(0, PAGE_SIZE, 32))


# ---- allocators -------------------------------------------------------------------

class FrameAllocator:
    """FIFO frame allocator over ``[first_pfn, first_pfn + n_pages)``.

    Equivalent to the reference's deque of every pfn (memvirt.py:191-213)
    but O(1) in space: untouched frames are handed out from a cursor over the
    initial range, freed frames queue behind it in free order.  Frames are
    zeroed on allocation.
    """

    def __init__(self, mem: PhysMem, first_pfn: int, n_pages: int):
        self._mem = mem
        self._first = first_pfn
        self._cursor = first_pfn
        self._end = first_pfn + max(n_pages, 0)
        self._freed: deque[int] = deque()
        self._lock = threading.Lock()

    @property
    def free_count(self) -> int:
        return (self._end - self._cursor) + len(self._freed)

    def _take(self, count: int) -> np.ndarray:
        with self._lock:
            if count > self.free_count:
                raise PoolExhausted("frame allocator empty")
            fresh = min(count, self._end - self._cursor)
            out = np.arange(self._cursor, self._cursor + fresh, dtype=np.int64)
            self._cursor += fresh
            if fresh < count:
                tail = [self._freed.popleft() for _ in range(count - fresh)]
                out = np.concatenate([out, np.array(tail, dtype=np.int64)])
            return out

    def alloc(self) -> int:
        pfn = int(self._take(1)[0])
        self._mem.zero_page(pfn)
        return pfn

    def alloc_many(self, count: int) -> np.ndarray:
        """``count`` frames in allocation order, zeroed (batch of alloc())."""
        pfns = self._take(count)
        if count:
            self._mem._img.zero_pages((self._mem.base >> PAGE_SHIFT) + pfns)
        return pfns

    def free(self, pfn: int) -> None:
        with self._lock:
            self._freed.append(pfn)


class ReservedPagePool:
    """Hypervisor-reserved gpa pages + guest-donated table pages
    (memvirt.py:216-241)."""

    def __init__(self, free_gpa_pages: list[int], free_guest_pt_pages: list[int]):
        self.free_gpa_pages: deque[int] = deque(free_gpa_pages)
        self.free_guest_pt_pages: deque[int] = deque(free_guest_pt_pages)
        self._lock = threading.Lock()

    def _pop(self, queue: deque, what: str) -> int:
        with self._lock:
            if not queue:
                raise PoolExhausted(f"no {what} left")
            return queue.popleft()

    def take_gpa_page(self) -> int:
        return self._pop(self.free_gpa_pages, "reserved guest physical pages")

    def take_pt_page(self) -> int:
        return self._pop(self.free_guest_pt_pages, "donated guest page-table pages")


# ---- data-plane walks ---------------------------------------------------------------

def _space_of(mem: PhysMem, root_pfn: int) -> dp.Space:
    return dp.Space(mem.base, root_pfn, 0, N.ONE_STAGE)


def _raise_lane(status: int, value: int, aux: int, va: int, mem: PhysMem) -> None:
    dp.raise_for(status, value, aux, va, mem.backing.nbytes)


def walk(mem: PhysMem, root_pfn: int, va: int) -> int:
    """Three-level walk on the device; returns the leaf target pfn
    (memvirt.py:244-259).  PageFault / TrapExit name the stopping level."""
    status, value, aux = dp.translate_one(mem.backing, _space_of(mem, root_pfn), va, out_pfn=True)
    if status:
        _raise_lane(status, value, aux, va, mem)
    return value


def walk_guest(gva: Gva, root: PageTableRoot, guest_mem: PhysMem) -> Gpa:
    """gva -> gpa through the guest's own table (memvirt.py:262-267)."""
    if root.kind is not TableKind.GUEST:
        raise ValueError(f"walk_guest needs a guest root, got {root.kind}")
    status, value, aux = dp.translate_one(guest_mem.backing, _space_of(guest_mem, root.root_pfn), gva)
    if status:
        _raise_lane(status, value, aux, gva, guest_mem)
    return Gpa(value)


# ---- table construction (control plane, host mirror) ---------------------------------

class TableEditor:
    """Creates and edits the entries of one table (memvirt.py:270-333).

    Intermediate nodes come from ``node_alloc`` and are installed present +
    writable; trapping entries are accepted only in shadow tables.
    """

    def __init__(self, mem: PhysMem, root: PageTableRoot, node_alloc: Callable[[], int]):
        self._mem = mem
        self._root = root
        self._alloc = node_alloc

    def _leaf_slot(self, va: int, create: bool) -> tuple[int, int]:
        top, mid, leaf, _ = split_va(va)
        node = self._root.root_pfn
        for index in (top, mid):
            word = self._mem.read_word(node, index)
            if entry_state(word) is not EntryState.NOT_PRESENT:
                node = word >> PAGE_SHIFT
                continue
            if not create:
                # the reference names the level with an identity test,
                # ``LEVEL_TOP if index is top else LEVEL_MID``
                # (memvirt.py:290): CPython's small ints make a missing mid
                # node whose mid index equals the top index (0..3) a level-1
                # fault; value equality reproduces that in this range
                raise PageFault(va, LEVEL_TOP if index == top else LEVEL_MID)
            child = self._alloc()
            self._mem.write_word(node, index, (child << PAGE_SHIFT) | FLAG_PRESENT | FLAG_WRITABLE)
            node = child
        return node, leaf

    def _require_trap_legal(self, state: EntryState) -> None:
        if state is EntryState.TRAPPING and self._root.kind is not TableKind.SHADOW:
            raise ValueError("trapping entries are legal only in shadow tables")

    def map(self, va: int, target_pfn: int, *, writable: bool = True,
            state: EntryState = EntryState.PRESENT, replace: bool = False) -> None:
        if va & PAGE_MASK:
            raise ValueError("mapping address must be page aligned")
        self._require_trap_legal(state)
        node, leaf = self._leaf_slot(va, create=True)
        if not replace and entry_state(self._mem.read_word(node, leaf)) is not EntryState.NOT_PRESENT:
            raise AlreadyMapped(f"{va:#010x} already mapped in {self._root.kind.value} table")
        self._mem.write_word(node, leaf, encode_entry(PageTableEntry(state, target_pfn, writable)))

    def entry_at(self, va: int) -> PageTableEntry:
        node, leaf = self._leaf_slot(va, create=False)
        return decode_entry(self._mem.read_word(node, leaf))

    def set_leaf_state(self, va: int, state: EntryState) -> None:
        """Flip a leaf's state, keeping its target and W bit."""
        self._require_trap_legal(state)
        node, leaf = self._leaf_slot(va, create=False)
        old = decode_entry(self._mem.read_word(node, leaf))
        self._mem.write_word(node, leaf, encode_entry(PageTableEntry(state, old.target_pfn, old.writable)))

    def is_mapped(self, va: int) -> bool:
        try:
            return self.entry_at(va).state is not EntryState.NOT_PRESENT
        except PageFault:
            return False


class _BulkMapper:
    """Vectorised form of many ``TableEditor.map`` calls in order.

    Reproduces the sequential result bit for bit -- the same node frames, in
    the same allocation order, interleaved with data-frame allocations the
    caller describes -- provided every target leaf is currently not present,
    no page repeats and every existing node is inside the memory.  Callers
    check :meth:`applicable` and fall back to the per-page loop otherwise.
    """

    def __init__(self, mem: PhysMem, root_pfn: int, vas: np.ndarray):
        self.mem = mem
        self.root = root_pfn
        self.vas = vas.astype(np.int64)
        self.top = (self.vas >> 30) & 0x3
        self.mid = (self.vas >> 21) & 0x1FF
        self.leaf = (self.vas >> 12) & 0x1FF
        self.words = mem.backing.host_for_read()
        base = mem.base
        self._limit_pfn = (mem.backing.nbytes - base) // PAGE_SIZE

        def word(pfn, idx):
            return self.words[base + pfn * PAGE_SIZE + idx * 8: base + pfn * PAGE_SIZE + idx * 8 + 8] \
                .view(np.uint64)[0]

        self._word = word
        # Existing top entries.
        self.top_word = np.array([int(word(root_pfn, t)) for t in range(4)], dtype=np.uint64)

    def _words_at(self, nodes: np.ndarray, idx: np.ndarray) -> np.ndarray:
        off = self.mem.base + nodes.astype(np.int64) * PAGE_SIZE + idx.astype(np.int64) * 8
        return self.words.view(np.uint64)[off // 8] if self.mem.base % 8 == 0 else None

    def plan(self):
        """Compute which pages need a new mid / leaf node."""
        top_present = (self.top_word & np.uint64(FLAG_PRESENT | FLAG_TRAPPING)) != 0
        tp = top_present[self.top]
        # first page (in order) per top index / per (top, mid)
        _, first_top = np.unique(self.top, return_index=True)
        new_mid = np.zeros(len(self.vas), dtype=bool)
        new_mid[first_top] = True
        new_mid &= ~tp
        tm = (self.top << 9) | self.mid
        _, first_tm = np.unique(tm, return_index=True)
        first_tm_mask = np.zeros(len(self.vas), dtype=bool)
        first_tm_mask[first_tm] = True
        # existing mid node for present tops
        mid_node_of_top = (self.top_word >> np.uint64(PAGE_SHIFT)).astype(np.int64)
        mid_exists = np.zeros(len(self.vas), dtype=bool)
        self.leaf_node = np.full(len(self.vas), -1, dtype=np.int64)
        if tp.any():
            sel = np.flatnonzero(tp)
            nodes = mid_node_of_top[self.top[sel]]
            if (nodes >= self._limit_pfn).any():
                return False
            w = self._words_at(nodes, self.mid[sel])
            if w is None:
                return False
            present = (w & np.uint64(FLAG_PRESENT | FLAG_TRAPPING)) != 0
            mid_exists[sel] = present
            self.leaf_node[sel[present]] = (w[present] >> np.uint64(PAGE_SHIFT)).astype(np.int64)
        new_leaf = first_tm_mask & ~mid_exists
        self.new_mid = new_mid
        self.new_leaf = new_leaf
        self.mid_exists = mid_exists
        # leaves of existing leaf nodes must be free
        if mid_exists.any():
            sel = np.flatnonzero(mid_exists)
            if (self.leaf_node[sel] >= self._limit_pfn).any():
                return False
            w = self._words_at(self.leaf_node[sel], self.leaf[sel])
            if ((w & np.uint64(FLAG_PRESENT | FLAG_TRAPPING)) != 0).any():
                return False
        return True

    def commit(self, mid_pfns: np.ndarray, leaf_pfns: np.ndarray, targets: np.ndarray, leaf_flags: int) -> None:
        """Write the table given the frames allocated for new nodes (in page
        order) and the leaf targets."""
        mem = self.mem
        n = len(self.vas)
        mid_node_of_top = (self.top_word >> np.uint64(PAGE_SHIFT)).astype(np.int64)
        # new mid nodes
        new_mid_idx = np.flatnonzero(self.new_mid)
        for pfn, i in zip(mid_pfns.tolist(), new_mid_idx.tolist()):
            t = int(self.top[i])
            mem.write_word(self.root, t, (pfn << PAGE_SHIFT) | FLAG_PRESENT | FLAG_WRITABLE)
            mid_node_of_top[t] = pfn
        mid_node = mid_node_of_top[self.top]
        # new leaf nodes, then every page's leaf node
        tm = (self.top << 9) | self.mid
        leaf_of_tm = {}
        new_leaf_idx = np.flatnonzero(self.new_leaf)
        img = mem.backing
        u64 = img.host.view(np.uint64)
        base_w = mem.base // 8
        if len(new_leaf_idx):
            offs = base_w + mid_node[new_leaf_idx] * 512 + self.mid[new_leaf_idx]
            words = (leaf_pfns.astype(np.uint64) << np.uint64(PAGE_SHIFT)) | np.uint64(FLAG_PRESENT | FLAG_WRITABLE)
            img.host_for_write_pages(np.unique(offs * 8 // PAGE_SIZE))
            u64[offs] = words
            for pfn, i in zip(leaf_pfns.tolist(), new_leaf_idx.tolist()):
                leaf_of_tm[int(tm[i])] = pfn
        leaf_node = self.leaf_node.copy()
        need = leaf_node < 0
        if need.any():
            keys = tm[need]
            leaf_node[need] = np.array([leaf_of_tm[int(k)] for k in np.unique(keys)], dtype=np.int64)[
                np.searchsorted(np.unique(keys), keys)]
        offs = base_w + leaf_node * 512 + self.leaf
        words = (targets.astype(np.uint64) << np.uint64(PAGE_SHIFT)) | np.uint64(leaf_flags)
        img.host_for_write_pages(np.unique(offs * 8 // PAGE_SIZE))
        u64[offs] = words
        assert n == len(offs)


class TranslationCache:
    """Per-process FIFO of (gva page, hpa page), capacity 10
    (memvirt.py:336-374): linear lookup, insert on miss only, strictly
    oldest-first eviction regardless of hits."""

    CAPACITY = 10

    def __init__(self, capacity: int = CAPACITY):
        self.capacity = capacity
        self._entries: deque[tuple[int, int]] = deque()
        self.hits = 0
        self.misses = 0

    def __len__(self) -> int:
        return len(self._entries)

    @property
    def lookups(self) -> int:
        return self.hits + self.misses

    def lookup(self, gva_page: int) -> int | None:
        for page, hpa_page in self._entries:
            if page == gva_page:
                self.hits += 1
                return hpa_page
        self.misses += 1
        return None

    def insert(self, gva_page: int, hpa_page: int) -> None:
        if len(self._entries) >= self.capacity:
            self._entries.popleft()
        self._entries.append((gva_page, hpa_page))

    def flush_page(self, gva_page: int) -> None:
        self._entries = deque(e for e in self._entries if e[0] != gva_page)

    def entries(self) -> list[tuple[int, int]]:
        return list(self._entries)

    def _load_state(self, entries, hits: int, misses: int) -> None:
        """Adopt the state the device replay produced."""
        self._entries = deque(entries)
        self.hits = hits
        self.misses = misses


@dataclass
class GuestMemory:
    guest_id: int
    mem: PhysMem
    base_hpa: int
    mem_mode: str
    os_alloc: FrameAllocator
    pool: ReservedPagePool
    tdp_root: PageTableRoot | None = None


@dataclass
class ProcessSpace:
    pid: int
    guest: GuestMemory
    guest_root: PageTableRoot
    shadow_root: PageTableRoot | None
    va_next: int = 0x4000_0000
    va_limit: int = 0xC000_0000
    driver_mappings: dict[int, int] = field(default_factory=dict)
    _va_lock: threading.Lock = field(default_factory=threading.Lock, repr=False)

    @property
    def cr3(self) -> int:
        return self.guest_root.root_pfn

    def alloc_va_range(self, length: int) -> int:
        span = -(-length // PAGE_SIZE) * PAGE_SIZE
        with self._va_lock:
            start = self.va_next
            if start + span > self.va_limit:
                raise PoolExhausted("guest virtual address space exhausted")
            self.va_next = start + span
            return start


class MemoryVirtualizer:
    """Host memory, guest slots and all table construction
    (memvirt.py:419-565).  Guest slots follow the host-private region
    linearly, so gpa -> hpa is one base offset per guest."""

    DEFAULT_HOST_BYTES = 64 * 1024 * 1024
    DEFAULT_GUEST_BYTES = 16 * 1024 * 1024
    HOST_PRIVATE_BYTES = 16 * 1024 * 1024
    KERNEL_PAGES = 64
    POOL_GPA_PAGES = 64
    POOL_PT_PAGES = 64

    def __init__(self, host_bytes: int = DEFAULT_HOST_BYTES):
        self.host_mem = PhysMem(host_bytes)
        private_pages = self.HOST_PRIVATE_BYTES // PAGE_SIZE
        self.host_alloc = FrameAllocator(self.host_mem, 1, private_pages - 1)
        self._slots: dict[int, tuple[int, int]] = {}
        self._next_slot = self.HOST_PRIVATE_BYTES
        self._guests: dict[int, GuestMemory] = {}
        self._next_pid = 1
        self.host_kernel_root = self._build_host_table()

    def _build_host_table(self) -> PageTableRoot:
        root = PageTableRoot(TableKind.HOST, self.host_alloc.alloc())
        editor = TableEditor(self.host_mem, root, self.host_alloc.alloc)
        for i in range(self.KERNEL_PAGES):
            frame = self.host_alloc.alloc()
            self.host_mem.write(frame * PAGE_SIZE, bytes([i & 0xFF]) * 16)
            editor.map(KERNEL_BASE + i * PAGE_SIZE, frame)
        return root

    def guest_base_offset(self, guest_id: int) -> int:
        return self._slots[guest_id][0]

    def guest_memory(self, guest_id: int) -> GuestMemory:
        return self._guests[guest_id]

    def add_guest(self, guest_id: int, mem_mode: str, size_bytes: int = DEFAULT_GUEST_BYTES) -> GuestMemory:
        if mem_mode not in ("shadow", "tdp"):
            raise ValueError(f"unknown memory mode {mem_mode!r}")
        base = self._next_slot
        if base + size_bytes > self.host_mem.size_bytes:
            raise OutOfRange("host memory cannot fit another guest slot")
        self._next_slot = base + size_bytes
        self._slots[guest_id] = (base, size_bytes)
        mem = PhysMem(size_bytes, backing=self.host_mem.backing, base=base)
        pages = size_bytes // PAGE_SIZE
        # the top POOL_GPA_PAGES frames are hypervisor-reserved (never seen by
        # the guest OS allocator); the pt pool is donated from ordinary frames
        os_alloc = FrameAllocator(mem, 1, pages - 1 - self.POOL_GPA_PAGES)
        reserved = list(range(pages - self.POOL_GPA_PAGES, pages))
        donated = [int(p) for p in os_alloc.alloc_many(self.POOL_PT_PAGES)]
        guest = GuestMemory(guest_id=guest_id, mem=mem, base_hpa=base, mem_mode=mem_mode,
                            os_alloc=os_alloc, pool=ReservedPagePool(reserved, donated))
        if mem_mode == "tdp":
            guest.tdp_root = self._build_tdp(guest)
        self._guests[guest_id] = guest
        return guest

    def _build_tdp(self, guest: GuestMemory) -> PageTableRoot:
        """TDP table covering the whole slot at its linear offset
        (memvirt.py:482-489), built with the bulk mapper."""
        root = PageTableRoot(TableKind.TDP, self.host_alloc.alloc())
        n = guest.mem.n_pages
        gpas = np.arange(n, dtype=np.int64) << PAGE_SHIFT
        targets = (guest.base_hpa >> PAGE_SHIFT) + np.arange(n, dtype=np.int64)
        _bulk_map(self.host_mem, root, self.host_alloc, gpas, targets, FLAG_PRESENT | FLAG_WRITABLE)
        return root

    def gpa_to_hpa(self, gpa: Gpa, guest_id: int) -> Hpa:
        """Linear memory-slot translation (memvirt.py:491-497)."""
        base, size = self._slots[guest_id]
        if not 0 <= gpa < size:
            raise OutOfRange(f"gpa {gpa:#x} beyond guest slot of {size:#x}")
        return Hpa(base + gpa)

    def create_process(self, guest: GuestMemory) -> ProcessSpace:
        pid = self._next_pid
        self._next_pid += 1
        guest_root = PageTableRoot(TableKind.GUEST, guest.os_alloc.alloc(), pid)
        shadow_root = None
        if guest.mem_mode == "shadow":
            shadow_root = PageTableRoot(TableKind.SHADOW, self.host_alloc.alloc(), pid)
        return ProcessSpace(pid=pid, guest=guest, guest_root=guest_root, shadow_root=shadow_root)

    def map_process_page(self, space: ProcessSpace, gva: Gva, *, writable: bool = True) -> Gpa:
        """Guest-OS mapping of one fresh data frame at ``gva``, mirrored
        into the shadow table under shadow paging (memvirt.py:508-522)."""
        guest = space.guest
        frame = guest.os_alloc.alloc()
        TableEditor(guest.mem, space.guest_root, guest.os_alloc.alloc).map(gva, frame, writable=writable)
        if space.shadow_root is not None:
            hpa = self.gpa_to_hpa(Gpa(frame << PAGE_SHIFT), guest.guest_id)
            TableEditor(self.host_mem, space.shadow_root, self.host_alloc.alloc).map(
                gva, hpa >> PAGE_SHIFT, writable=writable)
        return Gpa(frame << PAGE_SHIFT)

    def map_region(self, space: ProcessSpace, gva: Gva, n_pages: int) -> None:
        """``n_pages`` consecutive map_process_page calls."""
        self.map_pages(space, np.arange(n_pages, dtype=np.int64) * PAGE_SIZE + gva)

    def map_pages(self, space: ProcessSpace, gvas) -> None:
        """map_process_page for every gva of ``gvas`` in order -- vectorised.

        Bit-identical to the per-page loop (same frames, same order of data
        and node allocations, same words); falls back to that loop whenever
        the fast path's preconditions do not hold.
        """
        gvas = np.asarray(gvas, dtype=np.int64)
        if len(gvas) == 0:
            return
        if not _bulk_process_map(self, space, gvas):
            for g in gvas.tolist():
                self.map_process_page(space, Gva(g))

    def map_page_into_guest(self, space: ProcessSpace, gva: Gva, hpa: Hpa, mode: str,
                            cache: TranslationCache | None = None) -> None:
        """Backend-created mapping of a device/system page
        (memvirt.py:528-559): guest table -> fresh reserved gpa (nodes from
        the donated pool); shadow: shadow table -> hpa; TDP: TDP -> hpa."""
        if gva & PAGE_MASK:
            raise ValueError("gva must be page aligned")
        guest = space.guest
        guest_editor = TableEditor(guest.mem, space.guest_root, guest.pool.take_pt_page)
        if guest_editor.is_mapped(gva):
            raise AlreadyMapped(f"driver bug: {gva:#010x} is already mapped")
        reserved = guest.pool.take_gpa_page()
        if mode == "shadow":
            if space.shadow_root is None:
                raise ValueError("shadow-mode map for a guest without shadow tables")
            TableEditor(self.host_mem, space.shadow_root, self.host_alloc.alloc).map(
                gva, hpa >> PAGE_SHIFT, replace=True)
        elif mode == "tdp":
            if guest.tdp_root is None:
                raise ValueError("tdp-mode map for a guest without a TDP table")
            TableEditor(self.host_mem, guest.tdp_root, self.host_alloc.alloc).map(
                reserved << PAGE_SHIFT, hpa >> PAGE_SHIFT, replace=True)
        else:
            raise ValueError(f"unknown map mode {mode!r}")
        guest_editor.map(gva, reserved)
        space.driver_mappings[gva >> PAGE_SHIFT] = hpa >> PAGE_SHIFT
        if cache is not None:
            cache.flush_page(gva >> PAGE_SHIFT)

    def translator(self, space: ProcessSpace, cache: TranslationCache | None = None,
                   use_cache: bool = True) -> "ProcessTranslator":
        return ProcessTranslator(self, space, TranslationCache() if cache is None else cache,
                                 use_cache=use_cache)


# Batches of at least this many pages are built on the device when the image
# already lives there (pv_map_plan / pv_map_commit); smaller ones stay on the
# host mirror.  PV_DEVICE_MAP=0 disables the device builder.
DEVICE_MAP_MIN = 4096


def _device_map_ok(mem: PhysMem, n: int, alloc: "FrameAllocator | None" = None) -> bool:
    """Build on the device?  On a partially resident image (a guest-sharded
    rank) only when every node the builder reads or writes is in HBM: the
    allocator's frames (``alloc``), else the whole window."""
    import os

    img = mem.backing
    if not (img.on_device and n >= DEVICE_MAP_MIN and os.environ.get("PV_DEVICE_MAP", "1") != "0"):
        return False
    if not img.partial:
        return True
    if alloc is not None:
        return img.resident(mem.base + alloc._first * PAGE_SIZE, mem.base + alloc._end * PAGE_SIZE)
    return img.resident(mem.base, mem.base + mem.size_bytes)


def _device_map(mem: PhysMem, root: PageTableRoot, alloc: FrameAllocator, vas: np.ndarray,
                targets: np.ndarray, leaf_flags: int) -> bool:
    """_bulk_map on the device; False (nothing changed) when the batch is not
    exactly buildable there."""
    tb = dp.TableBuild(mem.backing, mem.base, root.root_pfn, dp._to_dev(vas.astype(np.int64)))
    bad, cnt = (int(x) for x in tb.summary().cpu().tolist())
    if bad != -1 or cnt > alloc.free_count:
        return False
    tb.commit(alloc._take(cnt), data_first=False, targets=dp._to_dev(np.asarray(targets, dtype=np.int64)),
              leaf_flags=leaf_flags)
    return True


def _device_process_map(memv: "MemoryVirtualizer", space: "ProcessSpace", gvas: np.ndarray) -> bool:
    """map_process_page over ``gvas`` on the device (guest table with
    data-first frames, then the shadow table); False when not applicable."""
    import torch

    guest = space.guest
    vas = dp._to_dev(gvas.astype(np.int64))
    gt = dp.TableBuild(guest.mem.backing, guest.mem.base, space.guest_root.root_pfn, vas)
    parts = [gt.summary()]
    st = None
    if space.shadow_root is not None:
        st = dp.TableBuild(memv.host_mem.backing, memv.host_mem.base, space.shadow_root.root_pfn, vas)
        parts.append(st.summary())
    stats = torch.cat(parts).cpu().tolist()
    if any(int(b) != -1 for b in stats[0::2]):
        return False
    n = len(gvas)
    if n + int(stats[1]) > guest.os_alloc.free_count:
        return False
    if st is not None and int(stats[3]) > memv.host_alloc.free_count:
        return False
    data = torch.empty(n, dtype=torch.int64, device="cuda")
    gt.commit(guest.os_alloc._take(n + int(stats[1])), data_first=True, leaf_flags=FLAG_PRESENT | FLAG_WRITABLE,
              out_data=data)
    if st is not None:
        st.commit(memv.host_alloc._take(int(stats[3])), data_first=False, targets=data,
                  target_add=guest.base_hpa >> PAGE_SHIFT, leaf_flags=FLAG_PRESENT | FLAG_WRITABLE)
    return True


def _bulk_map(mem: PhysMem, root: PageTableRoot, alloc: FrameAllocator, vas: np.ndarray,
              targets: np.ndarray, leaf_flags: int) -> None:
    """TableEditor(mem, root, alloc.alloc).map(va, target) for each pair in
    order, vectorised (node frames are the only allocations)."""
    if _device_map_ok(mem, len(vas), alloc) and mem.backing.resident(
            mem.base + root.root_pfn * PAGE_SIZE, mem.base + (root.root_pfn + 1) * PAGE_SIZE) and \
            not (vas & PAGE_MASK).any() and _device_map(mem, root, alloc, vas, targets, leaf_flags):
        return
    bm = _BulkMapper(mem, root.root_pfn, vas)
    if not _distinct_pages(vas) or not bm.plan():
        editor = TableEditor(mem, root, alloc.alloc)
        for va, t in zip(vas.tolist(), targets.tolist()):
            editor.map(va, t, writable=bool(leaf_flags & FLAG_WRITABLE))
        return
    # per page: [new mid node][new leaf node] in that order
    need = bm.new_mid.astype(np.int64) + bm.new_leaf.astype(np.int64)
    frames = alloc.alloc_many(int(need.sum()))
    mid_pfns, leaf_pfns = _split_node_frames(bm.new_mid, bm.new_leaf, frames, data_first=False)
    bm.commit(mid_pfns, leaf_pfns, targets, leaf_flags)


def _distinct_pages(vas: np.ndarray) -> bool:
    """No two addresses share a (top, mid, leaf) slot (VA bits >= 32 alias)."""
    keys = (vas >> PAGE_SHIFT) & 0xFFFFF
    return len(np.unique(keys)) == len(keys)


def _split_node_frames(new_mid: np.ndarray, new_leaf: np.ndarray, frames: np.ndarray, *, data_first: bool):
    """Assign a frame sequence to (data?, mid, leaf) requests page by page."""
    per = new_mid.astype(np.int64) + new_leaf.astype(np.int64) + (1 if data_first else 0)
    start = np.zeros(len(per), dtype=np.int64)
    np.cumsum(per[:-1], out=start[1:])
    off = start + (1 if data_first else 0)
    mid_pfns = frames[off[new_mid]]
    leaf_pfns = frames[(off + new_mid.astype(np.int64))[new_leaf]]
    data_pfns = frames[start] if data_first else None
    if data_first:
        return data_pfns, mid_pfns, leaf_pfns
    return mid_pfns, leaf_pfns


def _bulk_process_map(memv: MemoryVirtualizer, space: ProcessSpace, gvas: np.ndarray) -> bool:
    """Vectorised map_process_page over ``gvas``; False if not applicable."""
    if (gvas & PAGE_MASK).any() or (gvas < 0).any():
        return False
    if _device_map_ok(space.guest.mem, len(gvas)) and (
            space.shadow_root is None or _device_map_ok(memv.host_mem, len(gvas), memv.host_alloc)):
        return _device_process_map(memv, space, gvas)
    if not _distinct_pages(gvas):
        return False
    guest = space.guest
    gm = _BulkMapper(guest.mem, space.guest_root.root_pfn, gvas)
    if not gm.plan():
        return False
    sm = None
    if space.shadow_root is not None:
        sm = _BulkMapper(memv.host_mem, space.shadow_root.root_pfn, gvas)
        if not sm.plan():
            return False
    # guest OS allocator: per page [data][mid?][leaf?]
    per = 1 + gm.new_mid.astype(np.int64) + gm.new_leaf.astype(np.int64)
    if int(per.sum()) > guest.os_alloc.free_count:
        return False
    if sm is not None:
        if int(sm.new_mid.sum() + sm.new_leaf.sum()) > memv.host_alloc.free_count:
            return False
    frames = guest.os_alloc.alloc_many(int(per.sum()))
    data, g_mid, g_leaf = _split_node_frames(gm.new_mid, gm.new_leaf, frames, data_first=True)
    gm.commit(g_mid, g_leaf, data, FLAG_PRESENT | FLAG_WRITABLE)
    if sm is not None:
        hframes = memv.host_alloc.alloc_many(int(sm.new_mid.sum() + sm.new_leaf.sum()))
        s_mid, s_leaf = _split_node_frames(sm.new_mid, sm.new_leaf, hframes, data_first=False)
        targets = (guest.base_hpa >> PAGE_SHIFT) + data
        sm.commit(s_mid, s_leaf, targets, FLAG_PRESENT | FLAG_WRITABLE)
    return True


# ---- translators ---------------------------------------------------------------------

class ProcessTranslator:
    """gva -> hpa for one guest process (memvirt.py:568-601).

    Shadow paging walks the shadow table; TDP walks the guest table to the
    gpa and the TDP table to the hpa.  ``translate`` is the reference's
    per-address call (FIFO cache consulted first); ``translate_batch`` is the
    batched data-plane form over a whole array of addresses.
    """

    def __init__(self, memv: MemoryVirtualizer, space: ProcessSpace, cache: TranslationCache,
                 use_cache: bool = True):
        self._memv = memv
        self.space = space
        self.cache = cache
        self.use_cache = use_cache
        self._ds = None  # (shadow root, guest root, tdp root, mode, dp.Space) of the last device_space

    @property
    def device_space(self) -> dp.Space:
        space = self.space
        guest = space.guest
        c = self._ds
        # roots are frozen objects: the cached descriptor stands while the same ones are in place
        if c is not None and c[0] is space.shadow_root and c[1] is space.guest_root and c[2] is guest.tdp_root \
                and c[3] == guest.mem_mode:
            return c[4]
        if guest.mem_mode == "shadow":
            ds = dp.Space(self._memv.host_mem.base, space.shadow_root.root_pfn, 0, N.ONE_STAGE)
        else:
            ds = dp.Space(guest.mem.base, space.guest_root.root_pfn, guest.tdp_root.root_pfn, N.TWO_STAGE)
        self._ds = (space.shadow_root, space.guest_root, guest.tdp_root, guest.mem_mode, ds)
        return ds

    @property
    def image(self) -> MemoryImage:
        return self._memv.host_mem.backing

    def translate(self, gva: Gva) -> Hpa:
        page, off = gva >> PAGE_SHIFT, gva & PAGE_MASK
        if self.use_cache:
            cached = self.cache.lookup(page)
            if cached is not None:
                return Hpa((cached << PAGE_SHIFT) | off)
        status, value, aux = dp.translate_one(self.image, self.device_space, gva)
        if status:
            dp.raise_for(status, value, aux, gva, self.image.nbytes)
        if self.use_cache:
            self.cache.insert(page, value >> PAGE_SHIFT)
        return Hpa(value)

    def _resolve_page(self, gva: Gva) -> int:
        status, value, aux = dp.translate_one(self.image, self.device_space, gva, out_pfn=True)
        if status:
            dp.raise_for(status, value, aux, gva, self.image.nbytes)
        return value

    def translate_batch(self, gvas, *, use_cache: bool | None = None):
        """Translate every address of ``gvas`` as consecutive ``translate``
        calls would, without raising: returns ``(hpa, status, aux)``.

        ``gvas``: a CUDA tensor (int64/int32, results stay on the device) or
        anything numpy accepts (results come back as numpy uint64/uint32).
        Lanes with ``status != 0`` hold the fault record (see
        :func:`lane_error`).  With the cache in use the process's FIFO state
        and counters advance exactly as the per-address loop would.
        """
        return translate_batch(self, gvas, use_cache=use_cache)


def translate_batch(translator: ProcessTranslator, gvas, *, use_cache: bool | None = None):
    import torch

    on_device = isinstance(gvas, torch.Tensor) and gvas.is_cuda
    host_tensor = isinstance(gvas, torch.Tensor) and not gvas.is_cuda
    cache_on = translator.use_cache if use_cache is None else use_cache
    if host_tensor and not cache_on:
        # host in / host out: chunked H2D | translate | D2H pipeline
        return dp.translate_host_pipelined(translator.image, translator.device_space, gvas)
    if on_device:
        vas = gvas if gvas.dtype in (torch.int64, torch.int32) else gvas.to(torch.int64)
    elif host_tensor:
        # (pinned) host tensor in, pinned host tensors out: async copies on
        # the current stream, one synchronisation at the end
        src = gvas if gvas.dtype in (torch.int64, torch.int32) else gvas.to(torch.int64)
        vas = src.to("cuda", non_blocking=True)
    else:
        host = np.ascontiguousarray(np.asarray(gvas, dtype=np.uint64)).view(np.int64)
        vas = dp._to_dev(host)
    n = vas.numel()
    plan = dp.TranslatePlan([translator.device_space], [(0, n, 0)])
    value, status, aux = dp.translate_lanes(translator.image, plan, vas)
    if cache_on and n:
        cap = dp.fifo_capacity([translator.cache])
        fifo = dp._to_dev(dp.pack_fifo([translator.cache]))
        lane_idx = torch.arange(n, dtype=torch.int64, device="cuda")
        dp.fifo_replay_lanes(vas, lane_idx, np.array([0, n], dtype=np.int64), fifo, value, status, cap)
        dp.unpack_fifo(fifo.cpu().numpy(), [translator.cache])
    if on_device:
        return value, status, aux
    if host_tensor:
        outs = []
        for t in (value, status, aux):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            outs.append(h)
        torch.cuda.current_stream().synchronize()
        return tuple(outs)
    return (value.cpu().numpy().view(np.uint64), status.cpu().numpy().view(np.uint32),
            aux.cpu().numpy().view(np.uint64))


def translate_many(pairs, *, chunk: int = 1 << 23, packed: bool = False, words: bool = False, out=None):
    """``translate_batch`` for several uncached translators at once, host
    tensors in and out: ``pairs = [(translator, host_vas), ...]`` -> one
    pipelined H2D / translate / D2H stream over every pair (they must share
    one physical memory).  Returns ``[(hpa, status, aux), ...]`` as pinned
    host tensors; ``packed=True`` returns ``[(words, None, aux), ...]`` with
    one lane word per VA (hpa, or the status and value of the exception the
    lane raises; ``dataplane.unpack_lanes``), 8 bytes per lane instead of 12;
    ``words=True`` returns ``[(words, None, exceptions), ...]`` with one
    4-byte word per VA (the frame number, or the status of the exception the
    lane raises) and the exception records of the lanes whose value the word
    cannot carry (``dataplane.unpack_words``) -- as many bytes back as VAs
    in.  ``out``: per pair pinned host tensors to fill (see
    ``dataplane.translate_host_many``)."""
    import torch

    if not pairs:
        return []
    image = pairs[0][0].image
    jobs = []
    for tr, vas in pairs:
        if tr.use_cache:
            raise ValueError("translate_many runs uncached translators (the FIFO cache needs translate_batch)")
        if tr.image is not image:
            raise ValueError("translate_many needs translators of one physical memory")
        if not isinstance(vas, torch.Tensor):
            vas = torch.from_numpy(np.ascontiguousarray(np.asarray(vas, dtype=np.uint64)).view(np.int64))
        jobs.append((tr.device_space, vas))
    return dp.translate_host_many(image, jobs, chunk=chunk, packed=packed, words=words, out=out)


def lane_error(status: int, value: int, aux: int, va: int, image_bytes: int) -> Exception | None:
    """The exception a translate_batch lane stands for (None if OK)."""
    try:
        dp.raise_for(int(status), int(value), int(aux), int(va), image_bytes)
    except Exception as exc:  # noqa: BLE001 - returned, not raised
        return exc
    return None


# ---- user-buffer copies --------------------------------------------------------------

def copy_user_buffer(direction: str, gva: Gva, length: int, host_buf, *, translator,
                     host_mem: PhysMem) -> int:
    """Copy ``length`` bytes between ``host_buf`` and guest process memory
    (memvirt.py:604-628), on the device.

    One translation per page touched; on a fault the pages before it are
    copied and the raised PageFault carries ``bytes_copied``.
    """
    if direction not in ("to_guest", "from_guest"):
        raise ValueError(f"unknown direction {direction!r}")
    if length <= 0:
        return 0
    if ((gva + length - 1) >> PAGE_SHIFT) - (gva >> PAGE_SHIFT) < percall.SMALL_PAGES:
        # one op of <= 64 pages (every driver copy of the reference): one
        # launch through the per-call path
        copied, err = _copy_small(direction, gva, length, host_buf, translator, host_mem)
        if err is not None:
            raise err
        return copied
    import torch

    to_guest = direction == "to_guest"
    if to_guest:
        # a host_buf shorter than ``length`` behaves like the reference's
        # slices of it (memvirt.py:624): every page is still translated, only
        # the bytes the buffer holds are written (the kernels clamp at
        # buf_bytes).  The reference bounds-checks the shorter write; here the
        # page's full chunk is checked.
        src = np.frombuffer(bytes(host_buf[0:length]), dtype=np.uint8)
        avail = len(src)
        buf = dp._to_dev(src) if avail else torch.zeros(1, dtype=torch.uint8, device="cuda")
    else:
        avail = length
        buf = torch.empty(length, dtype=torch.uint8, device="cuda")
    space = getattr(translator, "device_space", None)
    if space is None:
        copied, err = _copy_foreign_translator(direction, gva, length, buf, translator, host_mem, avail)
    else:
        copied, err = _copy_device(direction, gva, length, buf, translator, host_mem, space, buf_bytes=avail)
    if not to_guest and copied:
        host_buf[0:copied] = buf[:copied].cpu().numpy().tobytes()
    if err is not None:
        raise err
    return copied


def _fifo_presim(cache: TranslationCache, pages: list[int]) -> list:
    """Which pages of an op the FIFO cache will answer (their cached hpa
    page) if the op runs to its end: lookup + insert-on-miss on a copy of the
    cache (memvirt.py:357-368).  Pages of one op are distinct, so a miss's
    insert only matters through the evictions it causes."""
    entries = deque(cache._entries)
    out = []
    for p in pages:
        hit = None
        for key, val in entries:
            if key == p:
                hit = val
                break
        out.append(hit)
        if hit is None:
            if len(entries) >= cache.capacity:
                entries.popleft()
            entries.append((p, None))
    return out


def _fifo_replay(cache: TranslationCache, pages: list[int], res, n_looked: int, bad: int, status: int) -> None:
    """Advance the real cache exactly as translate() would have over the
    first ``n_looked`` pages: hits count, misses count and insert the
    device's translation -- except a failing walk (no insert); a page whose
    data access was out of range did translate, so it is inserted."""
    for k in range(n_looked):
        hit = cache.lookup(pages[k])
        if hit is None and (k < bad or dp.kind(status) == N.ST_DATA_OOR):
            cache.insert(pages[k], int(res.page_hpa[k]) >> PAGE_SHIFT)


def _copy_small(direction, gva, length, host_buf, translator, host_mem):
    """copy_user_buffer of an op of at most percall.SMALL_PAGES pages, one
    pv_copy_small launch per run (the hybrid resolver's shim restarts a run
    at the trapped page, resolve_hybrid_with_fixup, memvirt.py:685-696).
    Same outcomes, cache state and counters as the batch path."""
    pc = percall.get()
    image = host_mem.backing
    to_guest = direction == "to_guest"
    d = N.TO_GUEST if to_guest else N.FROM_GUEST
    stage = pc.stage
    if to_guest:
        data = host_buf[0:length]
        avail = len(data)
        if avail:
            stage[:avail] = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    else:
        avail = length
    space = getattr(translator, "device_space", None)
    if space is None:
        return _copy_small_foreign(direction, gva, length, host_buf, translator, host_mem, pc, avail)
    cache = translator.cache if getattr(translator, "use_cache", False) else None
    retry = getattr(translator, "_on_trap", None)
    count = getattr(translator, "_count", None)
    done = 0
    shimmed = False
    while True:
        cur0 = gva + done
        rest = length - done
        n = ((cur0 + rest - 1) >> PAGE_SHIFT) - (cur0 >> PAGE_SHIFT) + 1
        pages = pre = None
        if cache is not None:
            pages = [((cur0 >> PAGE_SHIFT) + k) for k in range(n)]
            hits = _fifo_presim(cache, pages)
            pre = [None if h is None else (h << PAGE_SHIFT) | (cur0 & PAGE_MASK if k == 0 else 0)
                   for k, h in enumerate(hits)]
        res = pc.copy(image, space, cur0, rest, d, done, avail, pre)
        op = res.op
        status = int(op.status)
        bad = n if status == N.ST_OK else int(op.fail_page)
        if to_guest:
            percall.write_through(image, res, cur0, rest, bad, stage, done, avail)
        if cache is not None:
            _fifo_replay(cache, pages, res, n if status == N.ST_OK else bad + 1, bad, status)
        if status == N.ST_OK:
            if count is not None:
                count(n)
            copied = length
            break
        copied = done + int(op.copied)
        k = dp.kind(status)
        cur = gva + copied
        if k in (N.ST_TRAP, N.ST_TRAP2) and retry is not None:
            if shimmed and bad == 0:
                if count is not None:
                    count(1)
                _finish_from_guest(to_guest, host_buf, stage, copied)
                return copied, TrapFixupFailed(f"still trapping at {cur:#010x} after shim fixup")
            if count is not None:
                count(bad)
            trap = TrapExit(cur if k == N.ST_TRAP else int(op.aux), status & 0xF, int(op.value),
                            (status >> 16) & 0x1FF)
            err = retry(trap)
            if err is not None:
                if count is not None:
                    count(1)
                if isinstance(err, PageFault):
                    err.bytes_copied = copied
                _finish_from_guest(to_guest, host_buf, stage, copied)
                return copied, err
            done = copied
            shimmed = True
            continue
        if count is not None:
            count(bad + 1)
        chunk = min(length - copied, PAGE_SIZE - (cur & PAGE_MASK))
        _finish_from_guest(to_guest, host_buf, stage, copied)
        try:
            dp.raise_for(status, int(op.value), int(op.aux), cur, image.nbytes, chunk=chunk, bytes_copied=copied)
        except Exception as exc:  # noqa: BLE001
            return copied, exc
        return copied, None
    _finish_from_guest(to_guest, host_buf, stage, copied)
    return copied, None


def _finish_from_guest(to_guest, host_buf, stage, copied):
    if not to_guest and copied:
        host_buf[0:copied] = stage[:copied].tobytes()


def _copy_small_foreign(direction, gva, length, host_buf, translator, host_mem, pc, avail):
    """Small copy through a duck-typed translator: its translate() runs per
    page on the host (it is the caller's object), stopping at the first
    exception; the bytes of the pages before it move in one launch."""
    image = host_mem.backing
    to_guest = direction == "to_guest"
    pre = []
    err = None
    copied = 0
    while copied < length:
        cur = gva + copied
        chunk = min(length - copied, PAGE_SIZE - (cur & PAGE_MASK))
        try:
            hpa = translator.translate(Gva(cur))
        except PageFault as fault:
            fault.bytes_copied = copied
            err = fault
            break
        except Exception as exc:  # noqa: BLE001
            err = exc
            break
        n = max(0, min(chunk, avail - copied)) if to_guest else chunk
        if hpa < 0 or hpa + n > host_mem.size_bytes:
            err = OutOfRange(f"access [{hpa:#x}, +{n}) beyond {host_mem.size_bytes:#x}")
            break
        pre.append(host_mem.base + hpa)
        copied += chunk
    if pre:
        span = copied  # bytes of the pages that translated
        space = dp.Space(0, 0, 0, N.ONE_STAGE)
        res = pc.copy(image, space, gva, span, N.TO_GUEST if to_guest else N.FROM_GUEST, 0, avail, pre)
        if int(res.op.status) != N.ST_OK:
            raise RuntimeError(f"pv_copy_small failed on pre-translated pages: status {int(res.op.status):#x}")
        if to_guest:
            percall.write_through(image, res, gva, span, len(pre), pc.stage, 0, avail)
    _finish_from_guest(to_guest, host_buf, pc.stage, copied)
    return copied, err


def _copy_device(direction, gva, length, buf, translator, host_mem, space, first_shimmed=False, buf_bytes=None):
    """Device plan/exec for our own translators (cached, uncached, hybrid)."""
    op = np.array([[gva & dp.U64, length, 0, 0]], dtype=np.uint64)
    d = N.TO_GUEST if direction == "to_guest" else N.FROM_GUEST
    image = host_mem.backing
    caches = [translator.cache] if getattr(translator, "use_cache", False) else None
    groups = [[0]] if caches is not None else None
    retry = getattr(translator, "_on_trap", None)
    done = 0
    shimmed = first_shimmed  # the first page of this run was just fixed by the shim
    while True:
        cur_op = op.copy()
        cur_op[0, 0] = (gva + done) & dp.U64
        cur_op[0, 1] = length - done
        cur_op[0, 2] = done
        out = dp.copy_ops(image, [space], cur_op, d, buf, caches=caches, fifo_groups=groups,
                          shims=[getattr(translator, "device_shim", None)], buf_bytes=buf_bytes)[0]
        count = getattr(translator, "_count", None)
        if out.status == N.ST_OK:
            if count is not None:
                count(int(dp.page_spans(cur_op[:, 0], cur_op[:, 1])[0]))
            return length, None
        copied = done + out.copied
        k = dp.kind(out.status)
        cur = (gva + copied) if out.fail_page == 0 else (((gva + done) >> PAGE_SHIFT) + out.fail_page) << PAGE_SHIFT
        if k in (N.ST_TRAP, N.ST_TRAP2) and retry is not None:
            # hardware HAS: one shim call, then one retry of the trapping
            # page (resolve_hybrid_with_fixup, memvirt.py:685-696).  The
            # retry is page 0 of the next run; trapping there again is fatal.
            if shimmed and out.fail_page == 0:
                if count is not None:
                    count(1)
                return copied, TrapFixupFailed(f"still trapping at {cur:#010x} after shim fixup")
            if count is not None:
                count(out.fail_page)  # the trapping page is counted by its retry
            trap = TrapExit(cur if k == N.ST_TRAP else out.aux, out.status & 0xF, out.value,
                            (out.status >> 16) & 0x1FF)
            err = retry(trap)
            if err is not None:
                if count is not None:
                    count(1)
                if isinstance(err, PageFault):
                    err.bytes_copied = copied
                return copied, err
            done = copied
            shimmed = True
            continue
        if count is not None:
            count(out.fail_page + 1)
        chunk = min(length - copied, PAGE_SIZE - (cur & PAGE_MASK))
        try:
            dp.raise_for(out.status, out.value, out.aux, cur, image.nbytes, chunk=chunk, bytes_copied=copied)
        except Exception as exc:  # noqa: BLE001
            return copied, exc
        return copied, None


def _copy_foreign_translator(direction, gva, length, buf, translator, host_mem, avail=None):
    """A duck-typed translator object: translate per page through it, move
    the bytes with device copies on the HBM image (``avail``: bytes ``buf``
    holds; chunks past it move only those, like the reference's slices)."""
    avail = length if avail is None else avail
    image = host_mem.backing
    dev = image.device()
    copied = 0
    while copied < length:
        cur = gva + copied
        chunk = min(length - copied, PAGE_SIZE - (cur & PAGE_MASK))
        try:
            hpa = translator.translate(Gva(cur))
        except PageFault as fault:
            fault.bytes_copied = copied
            return copied, fault
        except Exception as exc:  # noqa: BLE001
            return copied, exc
        start = host_mem.base + hpa
        n = max(0, min(chunk, avail - copied)) if direction == "to_guest" else chunk
        if hpa < 0 or hpa + n > host_mem.size_bytes:
            return copied, OutOfRange(f"access [{hpa:#x}, +{n}) beyond {host_mem.size_bytes:#x}")
        if direction == "to_guest":
            if n:
                with image.writing():
                    dev[start:start + n].copy_(buf[copied:copied + n])
                    image._dev_dirty[start >> PAGE_SHIFT:((start + n - 1) >> PAGE_SHIFT) + 1] = 1
        else:
            buf[copied:copied + chunk].copy_(dev[start:start + chunk])
        copied += chunk
    return copied, None


# ---- hybrid address space ------------------------------------------------------------

class HybridTopLevel:
    """Per-process merged top level: shadow entries 0-2 + host entry 3
    (memvirt.py:631-668).  Rebuilt only when a source word changed; the same
    root frame is reused."""

    def __init__(self, host_mem: PhysMem, host_alloc: FrameAllocator):
        self._host_mem = host_mem
        self._host_alloc = host_alloc
        self._root: PageTableRoot | None = None
        self._snapshot: tuple[int, ...] | None = None

    def build(self, shadow_root: PageTableRoot, host_root: PageTableRoot) -> PageTableRoot:
        if shadow_root.kind is not TableKind.SHADOW:
            raise TdpUnsupported("hybrid top level needs a shadow table; TDP guests have none")
        if host_root.kind is not TableKind.HOST:
            raise ValueError("kernel entries must come from a host table")
        mem = self._host_mem
        words = tuple(mem.read_word(shadow_root.root_pfn, i) for i in range(3)) + \
            (mem.read_word(host_root.root_pfn, 3),)
        if self._root is not None and words == self._snapshot:
            return self._root
        if self._root is None:
            self._root = PageTableRoot(TableKind.HYBRID, self._host_alloc.alloc(), shadow_root.owner_process)
        for i, w in enumerate(words):
            mem.write_word(self._root.root_pfn, i, w)
        self._snapshot = words
        return self._root


def build_hybrid_top_level(shadow_root: PageTableRoot, host_root: PageTableRoot,
                           host_mem: PhysMem, host_alloc: FrameAllocator) -> PageTableRoot:
    return HybridTopLevel(host_mem, host_alloc).build(shadow_root, host_root)


def resolve_hybrid(va: int, root: PageTableRoot, host_mem: PhysMem) -> Hpa:
    """MMU-style walk of a merged table on the device (memvirt.py:677-682)."""
    if root.kind is not TableKind.HYBRID:
        raise ValueError(f"resolve_hybrid needs a hybrid root, got {root.kind}")
    status, value, aux = dp.translate_one(host_mem.backing, _space_of(host_mem, root.root_pfn), va)
    if status:
        _raise_lane(status, value, aux, va, host_mem)
    return Hpa(value)


def resolve_hybrid_with_fixup(va: int, root: PageTableRoot, host_mem: PhysMem,
                              shim: Callable[[TrapExit], None]) -> Hpa:
    """One shim call on a trap, then one retry; a second trap is fatal
    (memvirt.py:685-696)."""
    try:
        return resolve_hybrid(va, root, host_mem)
    except TrapExit as trap:
        shim(trap)
    try:
        return resolve_hybrid(va, root, host_mem)
    except TrapExit as trap:
        raise TrapFixupFailed(f"still trapping at {va:#010x} after shim fixup") from trap
