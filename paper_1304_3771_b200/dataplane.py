"""Host runtime of the HBM data plane: batching, launch, status decoding.

Everything here drives libpv kernels (``include/pv.h``) on the current CUDA
stream; nothing computes a translation or moves a payload byte on the CPU.
The functions are the batched forms of the reference's hot path:

* :func:`translate_lanes` -- K1, a batch of walks / translations
  (memvirt.py:244-267, 596-601, 677-682);
* :func:`fifo_replay_lanes` -- K4, the FIFO-10 cache applied to a batch
  (memvirt.py:336-374, 585-594);
* :func:`copy_ops` -- K2/K3, a batch of copy_user_buffer operations with the
  reference's prefix-on-fault semantics (memvirt.py:604-628);
* :func:`translate_one` -- a batch of one, used by the per-address drop-in
  entry points (walk, translate, resolve_hybrid).

Status words are decoded back into the reference's exceptions by
:func:`raise_for`.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import struct
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import percall
from .errors import OutOfRange, PageFault, TrapExit

PAGE_SIZE = 4096
PAGE_SHIFT = 12
PAGE_MASK = PAGE_SIZE - 1
U64 = (1 << 64) - 1


@dataclass(frozen=True)
class Space:
    """A translator as the kernels see it (pv_space)."""

    s1_base: int
    s1_root_pfn: int
    s2_root_pfn: int = 0
    mode: int = N.ONE_STAGE

    def words(self) -> list[int]:
        return [self.s1_base, self.s1_root_pfn, self.s2_root_pfn, self.mode]


@dataclass(frozen=True)
class Shim:
    """The default trap shim of one hybrid space (pv_shim): the guest
    process whose shadow leaves it re-syncs (backend.py:288-296)."""

    guest_base: int
    guest_bytes: int
    guest_root_pfn: int
    shadow_root_pfn: int

    def words(self) -> list[int]:
        return [self.guest_base, self.guest_bytes, self.guest_root_pfn, self.shadow_root_pfn]


NO_SHIM = Shim(0, 0, 0, 0)


def _i64(values) -> np.ndarray:
    """uint64 bit patterns as an int64 array (torch has no uint64 math)."""
    return np.asarray(values, dtype=np.uint64).view(np.int64)


def _to_dev(arr: np.ndarray, stream=None):
    import torch

    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(arr)
    if t.numel() * t.element_size() >= 1 << 16:
        t = t.pin_memory()
    return t.to("cuda", non_blocking=True)


_UPLOAD_MAX = 1 << 20  # arrays up to this size go through pv_upload (SM loads), larger ones through DMA
_uploads_in_flight: list = []  # (event, pinned block) until the stream has passed the upload


def _to_dev_many(arrays):
    """Device copies of several host arrays, the small ones (< 1 MiB together
    per array) packed into one pinned block and moved by one pv_upload
    kernel: SM loads over the host link, which do not queue behind a large
    H2D already in flight on another stream (a copy batch's payload), so the
    batch's plan runs while its payload is still arriving."""
    import torch

    arrs = [np.ascontiguousarray(a) for a in arrays]
    if torch.cuda.is_current_stream_capturing():
        return [_to_dev(a) for a in arrs]
    small = [i for i, a in enumerate(arrs) if a.nbytes <= _UPLOAD_MAX]
    out = [None] * len(arrs)
    for i, a in enumerate(arrs):
        if i not in small:
            out[i] = _to_dev(a)
    if small:
        offs, total = [], 0
        for i in small:
            offs.append(total)
            total += (arrs[i].nbytes + 15) & ~15
        total = max(total, 16)
        host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for i, o in zip(small, offs):
            hv[o:o + arrs[i].nbytes] = arrs[i].reshape(-1).view(np.uint8)
        dev = torch.empty(total, dtype=torch.uint8, device="cuda")
        stream = _stream()
        N.check(N.lib().pv_upload(dev.data_ptr(), host.data_ptr(), total, stream.cuda_stream), "pv_upload")
        ev = torch.cuda.Event()
        ev.record(stream)
        while _uploads_in_flight and _uploads_in_flight[0][0].query():
            _uploads_in_flight.pop(0)
        _uploads_in_flight.append((ev, host))
        for i, o in zip(small, offs):
            a = arrs[i]
            dt = torch.from_numpy(a.reshape(-1)[:0]).dtype
            out[i] = dev[o:o + a.nbytes].view(dt).view(a.shape)
    return out


def _stream():
    import torch

    return torch.cuda.current_stream()


# ---- status decoding ---------------------------------------------------------

def kind(status: int) -> int:
    return status & 0xFF0


def raise_for(status: int, value: int, aux: int, va: int, image_bytes: int, chunk: int = 0,
              bytes_copied: int | None = None) -> None:
    """Raise the reference exception a lane / op status stands for."""
    k = kind(status)
    level = status & 0xF
    if k == N.ST_OK:
        return
    if k in (N.ST_FAULT, N.ST_FAULT2):
        fault = PageFault(value, level)
        if bytes_copied is not None:
            fault.bytes_copied = bytes_copied
        raise fault
    if k == N.ST_TRAP:
        raise TrapExit(va, level, value, (status >> 16) & 0x1FF)
    if k == N.ST_TRAP2:
        raise TrapExit(aux, level, value, (status >> 16) & 0x1FF)
    if k in (N.ST_NODE_OOR, N.ST_NODE_OOR2):
        # The reference's unchecked read_word (memvirt.py:170-172) fails inside
        # struct.unpack_from for a node past the buffer.
        raise struct.error(f"page-table node read past the end of a {image_bytes}-byte memory "
                           f"(walk of {value:#x}, level {level})")
    if k == N.ST_DATA_OOR:
        raise OutOfRange(f"access [{value:#x}, +{chunk}) beyond {image_bytes:#x}")
    raise RuntimeError(f"unknown data-plane status {status:#x}")


# ---- single-lane fast path ---------------------------------------------------

def translate_one(image, space: Space, va: int, *, out_pfn: bool = False) -> tuple[int, int, int]:
    """One walk/translation on the device: returns (status, value, aux).
    One request to the per-call server (or one pv_walk_one launch), result
    in pinned memory (percall.py)."""
    return percall.get().walk(image, space, va, out_pfn)


# ---- K1: batched translation -------------------------------------------------

def build_segments(bounds: list[tuple[int, int, int]]) -> np.ndarray:
    """(begin, end, space) runs -> pv_seg rows with chunk0 prefix sums."""
    lib = N.load()
    chunk = int(lib.pv_translate_chunk())
    rows = []
    c0 = 0
    for begin, end, sp in bounds:
        if end <= begin:
            continue
        rows.append((begin, end, c0, sp))
        c0 += (end - begin + chunk - 1) // chunk
    return np.array(rows, dtype=np.uint64).reshape(-1, 4), c0


class PvIndex(ctypes.Structure):
    """pv_index (include/pv.h)."""

    _fields_ = [("slot_of", ctypes.c_void_p), ("leaf_codes", ctypes.c_void_p), ("slot_page", ctypes.c_void_p),
                ("n_slots", ctypes.c_uint64)]


NO_SLOT = 0xFFFFFFFF


class LeafIndex:
    """The leaf index of one MemoryImage (pv.h ``pv_index``): 4-byte codes of
    the leaf-level table nodes that translate batches walk, L2-resident where
    the reference's 8-byte PTEs are not.  A cache keyed by page contents:

    * :meth:`ensure` indexes the leaf nodes reachable from some spaces (host
      scan of their top and mid levels, then one encode launch);
    * host writes to an indexed page re-encode its slot when the image pushes
      them (:meth:`on_push`);
    * device writes are caught through the image's device dirty map before
      the map is cleared or the next translate launch (:meth:`sync_device_writes`).
    Leaf nodes that are not indexed are walked through the raw PTEs, so the
    index can only change speed, never results.

    Threads: every change runs under the image lock and records ``_ready``
    on its stream; a translate on another stream waits for that event
    (:meth:`wait_ready`) before it reads the codes, and replaced tensors stay
    alive (``_retired``) until the next device-wide synchronisation.
    """

    def __init__(self, image):
        import torch

        self.image = image
        self.slot_of_host = np.full(image.npages, NO_SLOT, dtype=np.uint32)
        self.pages = np.zeros(0, dtype=np.int64)
        self.slot_of = torch.full((image.npages,), -1, dtype=torch.int32, device="cuda")
        self.slot_page = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.codes = torch.zeros(512, dtype=torch.int32, device="cuda")
        self.seen_dev_epoch = image.dev_write_epoch
        self._scanned: dict = {}  # space -> image.host_epoch of its last scan
        self._ready = None        # (stream handle, event) after the last change
        self._retired: list = []  # replaced tensors other streams may still read

    @property
    def n_slots(self) -> int:
        return len(self.pages)

    def _device_pages(self, pages: list[int]) -> np.ndarray:
        """Whole pages read from HBM (always current: host writes are pushed
        first), so scanning tables never pulls the device's data writes back."""
        import torch

        if not pages:
            return np.zeros((0, PAGE_SIZE // 8), dtype=np.uint64)
        dev = self.image.device()
        pfns = torch.tensor(np.asarray(pages, dtype=np.int64), device="cuda")
        dst = torch.empty(len(pages) * PAGE_SIZE, dtype=torch.uint8, device="cuda")
        N.check(N.lib().pv_gather_pages(dev.data_ptr(), self.image.nbytes, pfns.data_ptr(), len(pages),
                                        dst.data_ptr(), _stream().cuda_stream), "pv_gather_pages")
        return dst.cpu().numpy().view(np.uint64).reshape(len(pages), PAGE_SIZE // 8)

    def leaf_pages(self, spaces: list["Space"]) -> np.ndarray:
        """Absolute image pages of every leaf node the spaces can reach."""
        nbytes = self.image.nbytes
        stages = []
        for sp in spaces:
            stages.append((sp.s1_base, sp.s1_root_pfn))
            if sp.mode == N.TWO_STAGE:
                stages.append((0, sp.s2_root_pfn))
        stages = [(b, r) for b, r in dict.fromkeys(stages)
                  if b % PAGE_SIZE == 0 and b < nbytes and r < (nbytes - b) // PAGE_SIZE]
        roots = self._device_pages([b // PAGE_SIZE + r for b, r in stages])
        mids = []  # (absolute mid page, window base)
        for (base, _), words in zip(stages, roots):
            lim = (nbytes - base) // PAGE_SIZE
            for w in words[:4].tolist():
                if not (w & 4 or not w & 1 or (w >> PAGE_SHIFT) >= lim):
                    mids.append((base // PAGE_SIZE + (w >> PAGE_SHIFT), base))
        mids = list(dict.fromkeys(mids))
        out = []
        for (_, base), words in zip(mids, self._device_pages([m for m, _ in mids])):
            lim = np.uint64((nbytes - base) // PAGE_SIZE)
            ok = (words & np.uint64(5)) == np.uint64(1)
            leaf = words[ok] >> np.uint64(PAGE_SHIFT)
            out.append(leaf[leaf < lim].astype(np.int64) + base // PAGE_SIZE)
        return np.unique(np.concatenate(out)) if out else np.zeros(0, dtype=np.int64)

    def _changed(self) -> None:
        import torch

        stream = torch.cuda.current_stream()
        if torch.cuda.is_current_stream_capturing():
            return
        ev = torch.cuda.Event()
        ev.record(stream)
        self._ready = (stream.cuda_stream, ev)

    def wait_ready(self) -> None:
        """Order the current stream after the index's last change."""
        import torch

        ready = self._ready
        # a capture starts from a synchronised device (torch.cuda.graph), and
        # a capturing stream may not wait on uncaptured work
        if ready is not None and ready[0] != torch.cuda.current_stream().cuda_stream and \
                not torch.cuda.is_current_stream_capturing():
            torch.cuda.current_stream().wait_event(ready[1])

    def release_retired(self) -> None:
        """Drop replaced tensors (call after a device-wide synchronisation)."""
        self._retired.clear()

    def ensure(self, spaces: list["Space"]) -> None:
        """Index the leaf nodes ``spaces`` reach.  A space is rescanned only
        after host writes changed the image (tables are edited host-side;
        a structural change the scan misses only costs speed: unindexed leaf
        nodes are walked raw)."""
        with self.image._lock:
            self._ensure(spaces)

    def _ensure(self, spaces: list["Space"]) -> None:
        import torch

        dev = self.image.device()
        epoch = self.image.host_epoch
        todo = [sp for sp in spaces if self._scanned.get(sp) != epoch]
        if not todo:
            return
        for sp in todo:
            self._scanned[sp] = epoch
        pages = self.leaf_pages(todo)
        new = pages[self.slot_of_host[pages] == NO_SLOT]
        if len(new) == 0:
            return
        first = self.n_slots
        slots = np.arange(first, first + len(new), dtype=np.int64)
        self.slot_of_host[new] = slots.astype(np.uint32)
        self.pages = np.concatenate([self.pages, new])
        self.wait_ready()
        slot_page = torch.from_numpy(self.pages.copy()).to("cuda")
        codes = torch.empty(self.n_slots * 512, dtype=torch.int32, device="cuda")
        if first:
            codes[: first * 512].copy_(self.codes[: first * 512])
        self._retired += [self.slot_page, self.codes]
        self.slot_page, self.codes = slot_page, codes
        self.slot_of[torch.from_numpy(new).to("cuda")] = torch.from_numpy(slots.astype(np.int32)).to("cuda")
        self._encode(dev, None, first, len(new), None)
        self._changed()

    def _encode(self, dev, slots, first, n, dirty) -> None:
        lib = N.lib()
        N.check(lib.pv_index_encode(dev.data_ptr(), self.image.nbytes, self.slot_page.data_ptr(),
                                    None if slots is None else slots.data_ptr(), first, n, self.codes.data_ptr(),
                                    None if dirty is None else dirty.data_ptr(), _stream().cuda_stream),
                "pv_index_encode")

    def on_push(self, pages: np.ndarray, dev) -> None:
        """Host wrote these pages (now in HBM): re-encode indexed ones."""
        s = self.slot_of_host[pages]
        s = s[s != NO_SLOT].astype(np.int64)
        if len(s):
            import torch

            with self.image._lock:
                self.wait_ready()
                self._encode(dev, torch.from_numpy(s).to("cuda"), 0, len(s), None)
                self._changed()

    def sync_device_writes(self) -> None:
        """Re-encode indexed pages the device wrote since the last sync (after
        the writes of every stream, see MemoryImage.wait_writers)."""
        img = self.image
        with img._lock:
            epoch = img.dev_write_epoch
            if self.seen_dev_epoch != epoch and self.n_slots and img.on_device:
                img.wait_writers()
                self.wait_ready()
                self._encode(img._dev, None, 0, self.n_slots, img.dirty_map())
                self._changed()
            self.seen_dev_epoch = epoch

    def abi(self) -> PvIndex:
        """pv_index of the current tensors (a fresh struct per call: threads
        never share one), after ordering the stream behind the last change."""
        with self.image._lock:
            self.wait_ready()
            return PvIndex(self.slot_of.data_ptr(), self.codes.data_ptr(), self.slot_page.data_ptr(), self.n_slots)


def leaf_index(image) -> LeafIndex:
    if image.leaf_index is None:
        with image._lock:
            if image.leaf_index is None:
                image.device()
                image.leaf_index = LeafIndex(image)
    return image.leaf_index


class TranslatePlan:
    """Device-resident descriptors of a translate batch (reusable).

    ``image`` (optional) indexes the leaf nodes the spaces reach (pv.h leaf
    index) so the walks gather 4-byte L2-resident codes; ``use_index=False``
    walks the raw 8-byte PTEs only."""

    def __init__(self, spaces: list[Space], bounds: list[tuple[int, int, int]], *, image=None,
                 use_index: bool = True):
        segs, n_chunks = build_segments(bounds)
        self.host_spaces = list(spaces)
        self.spaces = _to_dev(_i64([sp.words() for sp in spaces]).reshape(-1, 4))
        self.segs = _to_dev(segs.view(np.int64))
        self.n_segs = len(segs)
        self.n_chunks = n_chunks
        self.two = any(sp.mode == N.TWO_STAGE for sp in spaces)
        self.four = any(sp.mode == N.ONE_STAGE_4L for sp in spaces)
        self.use_index = use_index and not self.four and os.environ.get("PV_LEAF_INDEX", "1") != "0"
        self._indexed = False
        if image is not None and self.use_index:
            leaf_index(image).ensure(self.host_spaces)
            self._indexed = True


def unpack_lanes(packed, aux=None) -> tuple[np.ndarray, np.ndarray]:
    """(value uint64, status uint32) of PV_OUT_PACKED lane words (pv.h):
    a word without PV_PACKED_ERR is the value of a lane that translated;
    otherwise bits 42-62 hold the compact status and bits 0-41 the value, or
    PV_PACKED_SPILL_VALUE when the value was wider and lives in ``aux``."""
    w = np.asarray(packed).view(np.uint64)
    err = (w >> np.uint64(63)).astype(bool)
    compact = ((w >> np.uint64(N.PACKED_VALUE_BITS)) & np.uint64(0x1FFFFF)).astype(np.uint32)
    status = np.where(err, (compact & np.uint32(0xFFF)) | ((compact >> np.uint32(12)) << np.uint32(16)),
                      np.uint32(0)).astype(np.uint32)
    low = w & np.uint64(N.PACKED_SPILL_VALUE)
    value = np.where(err, low, w)
    spill = err & (low == np.uint64(N.PACKED_SPILL_VALUE))
    if spill.any():
        if aux is None:
            raise ValueError("spilled lanes need the aux array")
        value = value.copy()
        value[spill] = np.asarray(aux).view(np.uint64)[spill]
    return value, status


class SmSplit:
    """Two disjoint SM partitions of the current device (pv_sm_split, green
    contexts): ``streams[0]`` runs on a group of at least ``first_sms`` SMs,
    ``streams[1]`` on the rest.  ``with split.on(k):`` makes partition k's
    stream current and sizes the library's grids for its SMs, so a walk (SM->L2
    request bound) on one partition and a page copy (HBM bound) on the other
    run side by side without sharing SMs."""

    def __init__(self, first_sms: int, fine: bool = False, interleave: bool = False):
        import torch

        lib = N.lib()
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        na, nb = ctypes.c_uint32(), ctypes.c_uint32()
        flags = (N.SM_SPLIT_FINE if fine else 0) | (N.SM_SPLIT_INTERLEAVE if interleave else 0)
        N.check(lib.pv_sm_split(first_sms, flags, ctypes.byref(a), ctypes.byref(b), ctypes.byref(na),
                                ctypes.byref(nb)), "pv_sm_split")
        self.fine, self.interleave = fine, interleave
        self.placement = ("interleaved " if interleave else "") + ("single SMs" if fine else "8-SM groups")
        self.streams = (torch.cuda.ExternalStream(a.value), torch.cuda.ExternalStream(b.value))
        self.sms = (int(na.value), int(nb.value))

    @contextlib.contextmanager
    def on(self, k: int):
        import torch

        lib = N.lib()
        with torch.cuda.stream(self.streams[k]):
            old = lib.pv_set_sm_budget(self.sms[k])
            try:
                yield self.streams[k]
            finally:
                lib.pv_set_sm_budget(old)


class LaneExceptions:
    """Exception records of a pv_translate_words batch (pv.h pv_exc): the
    lanes whose 4-byte word cannot carry the exception's value (traps, TDP
    stage faults), job-local lane index order unspecified."""

    __slots__ = ("lane", "value", "aux", "status")

    def __init__(self, lane=None, value=None, aux=None, status=None):
        self.lane = np.zeros(0, np.int64) if lane is None else lane
        self.value = np.zeros(0, np.uint64) if value is None else value
        self.aux = np.zeros(0, np.uint64) if aux is None else aux
        self.status = np.zeros(0, np.uint32) if status is None else status

    def __len__(self) -> int:
        return len(self.lane)

    @classmethod
    def from_records(cls, recs: np.ndarray) -> "LaneExceptions":
        r = np.asarray(recs).view(np.uint64).reshape(-1, N.EXC_WORDS)
        return cls(r[:, 0].astype(np.int64), r[:, 1].copy(), r[:, 2].copy(), (r[:, 3] & np.uint64(0xFFFFFFFF)).astype(np.uint32))


class ExcList:
    """The device exception list of pv_translate_words (pv.h): PV_EXC_STRIPES
    counters and room for ``cap`` records (``cap / PV_EXC_STRIPES`` per
    stripe).  ``reset()`` zeroes the counters on the current stream;
    ``read()`` returns ``(LaneExceptions, total, overflow)`` -- overflow: some
    stripe counted more records than it holds (re-run with ``needed()``)."""

    def __init__(self, cap: int):
        import torch

        self.per = -(-int(cap) // N.EXC_STRIPES) if cap > 0 else 0
        self.rec = torch.empty(max(self.per * N.EXC_STRIPES, 1) * N.EXC_WORDS, dtype=torch.int64, device="cuda")
        self.cnt = torch.zeros(N.EXC_STRIPES, dtype=torch.int64, device="cuda")
        self._last = np.zeros(N.EXC_STRIPES, np.int64)

    @property
    def cap(self) -> int:
        return self.per * N.EXC_STRIPES

    def reset(self) -> None:
        """Zero the counters (stream-ordered; graph-capturable)."""
        self.cnt.zero_()

    def needed(self) -> int:
        """A capacity that holds every stripe's records of the last :meth:`read`."""
        return int(self._last.max()) * N.EXC_STRIPES

    def read(self):
        counts = self._last = self.cnt.cpu().numpy()
        total = int(counts.sum())
        overflow = bool((counts > self.per).any())
        take = np.minimum(counts, self.per)
        if total == 0:
            return LaneExceptions(), 0, overflow
        recs = self.rec[: self.per * N.EXC_STRIPES * N.EXC_WORDS].view(N.EXC_STRIPES, self.per, N.EXC_WORDS)
        parts = [recs[st, : int(t)].cpu().numpy() for st, t in enumerate(take) if t]
        return LaneExceptions.from_records(np.concatenate(parts)), total, overflow


def unpack_words(words, vas, exc: LaneExceptions | None = None, *, out_pfn: bool = False):
    """(value uint64, status uint32, aux uint64) of pv_translate_words lane
    words (pv.h): a word without PV_W32_ERR is the lane's frame number (value
    = frame << 12 | va & 0xFFF, or the frame under ``out_pfn``); otherwise bits
    0-20 are the compact status and the value is the lane's va (PV_W32_VA) or
    comes from its exception record in ``exc``."""
    w = np.asarray(words).view(np.uint32)
    v = np.asarray(vas)
    va = v.view(np.uint32).astype(np.uint64) if v.dtype.itemsize == 4 else v.view(np.uint64)
    err = (w & np.uint32(N.W32_ERR)) != 0
    compact = w & np.uint32(N.W32_COMPACT_MASK)
    status = np.where(err, (compact & np.uint32(0xFFF)) | ((compact >> np.uint32(12)) << np.uint32(16)),
                      np.uint32(0)).astype(np.uint32)
    frame = w.astype(np.uint64)
    value = frame if out_pfn else (frame << np.uint64(PAGE_SHIFT)) | (va & np.uint64(0xFFF))
    value = np.where(err, va, value)
    aux = np.zeros(len(w), np.uint64)
    need = err & ((w & np.uint32(N.W32_VA)) == 0)
    if need.any():
        if exc is None:
            raise ValueError("lanes with exception records need the LaneExceptions of the batch")
        have = np.zeros(len(w), bool)
        have[exc.lane] = True
        if not np.array_equal(have, need):
            raise ValueError("exception records do not match the lanes that need them")
        value[exc.lane] = exc.value
        aux[exc.lane] = exc.aux
    return value, status, aux


def translate_words(image, plan: TranslatePlan, vas, words, exc: ExcList, lane_base: int = 0, *,
                    out_pfn: bool = False, concurrent: bool = False) -> None:
    """pv_translate_words over every lane of ``vas`` (int64 or int32 cuda
    tensor) into ``words`` (int32 cuda tensor, one per lane, or a raw device
    address -- e.g. a slice of rank 0's shard.PeerResultBuffer); exception
    records go to ``exc`` (an :class:`ExcList`, not reset here),
    asynchronously on the current stream."""
    percall.park()  # the per-call server must not hold a CTA slot this grid counts on
    import torch

    lib = N.lib()
    dev_img = image.device()
    flags = (N.VA32 if vas.dtype == torch.int32 else 0) | (N.OUT_PFN if out_pfn else 0) | \
        (N.CONCURRENT if concurrent else 0)
    if plan.two:
        flags |= N.HAS_TWO_STAGE
    if plan.four:
        flags |= N.HAS_4L
    idx = _plan_index(image, plan)
    cap = exc.cap
    N.check(lib.pv_translate_words(dev_img.data_ptr(), image.nbytes, plan.spaces.data_ptr(), plan.segs.data_ptr(),
                                   plan.n_segs, plan.n_chunks, vas.data_ptr(), flags, idx,
                                   words if isinstance(words, int) else words.data_ptr(),
                                   exc.rec.data_ptr() if cap else None, cap, exc.cnt.data_ptr(), lane_base,
                                   _stream().cuda_stream), "pv_translate_words")


def _plan_index(image, plan: TranslatePlan):
    """byref(pv_index) for a plan that walks through the leaf index, else None."""
    if not plan.use_index:
        return None
    li = leaf_index(image)
    if not plan._indexed:
        li.ensure(plan.host_spaces)
        plan._indexed = True
    li.sync_device_writes()
    idx_abi = li.abi()
    return ctypes.byref(idx_abi)


def translate_lanes(image, plan: TranslatePlan, vas, *, out_pfn: bool = False, out=None, concurrent: bool = False,
                    packed: bool = False):
    """Translate every lane of ``vas`` (int64 or int32 cuda tensor).

    Returns ``(value int64, status int32, aux int64)`` device tensors, written
    asynchronously on the current stream.  ``out`` may pass preallocated
    tensors of the same shapes.  ``concurrent``: the walk shares the GPU with
    a kernel on another stream (pv.h PV_CONCURRENT, one CTA per SM).
    ``packed``: value holds PV_OUT_PACKED lane words (:func:`unpack_lanes`)
    and status is None.
    """
    percall.park()  # the per-call server must not hold a CTA slot this grid counts on
    import torch

    lib = N.lib()
    dev_img = image.device()
    n = vas.numel()
    if out is None:
        value = torch.empty(n, dtype=torch.int64, device="cuda")
        status = None if packed else torch.empty(n, dtype=torch.int32, device="cuda")
        aux = torch.zeros(n, dtype=torch.int64, device="cuda")
    else:
        value, status, aux = out
    flags = (N.VA32 if vas.dtype == torch.int32 else 0) | (N.OUT_PFN if out_pfn else 0) | \
        (N.CONCURRENT if concurrent else 0) | (N.OUT_PACKED if packed else 0)
    if plan.two:
        flags |= N.HAS_TWO_STAGE
    if plan.four:
        flags |= N.HAS_4L
    idx = _plan_index(image, plan)
    N.check(lib.pv_translate(dev_img.data_ptr(), image.nbytes, plan.spaces.data_ptr(), plan.segs.data_ptr(),
                             plan.n_segs, plan.n_chunks, vas.data_ptr(), flags, idx, value.data_ptr(),
                             None if status is None else status.data_ptr(),
                             None if aux is None else aux.data_ptr(), _stream().cuda_stream), "pv_translate")
    return value, status, aux


def translate_host_pipelined(image, space: Space, host_vas, chunk: int = 1 << 23):
    """Translate a (pinned) host tensor of VAs; results come back as pinned
    host tensors (see :func:`translate_host_many`)."""
    return translate_host_many(image, [(space, host_vas)], chunk=chunk)[0]


# bytes the last translate_host_many call moved each way (bench accounting)
last_host_io = {"h2d": 0, "d2h": 0}


def translate_host_many(image, jobs, chunk: int = 1 << 23, *, packed: bool = False, words: bool = False, out=None,
                        exc_cap: int = 1 << 20):
    """Translate several host VA tensors (``jobs = [(space, vas), ...]``) in
    one pipeline: chunks of every job stream through two device buffer sets,
    H2D of chunk i+1 and D2H of chunk i-1 run on side streams while chunk i
    translates, one synchronisation at the end.  Returns per job pinned
    ``(value int64, status int32, aux int64)``; ``aux`` only travels for
    two-stage spaces (one-stage walks never produce a TDP-stage trap).

    ``packed``: per job ``(words int64, None, aux)`` with one PV_OUT_PACKED
    word per lane (8 bytes back instead of 12; :func:`unpack_lanes`); aux
    travels for two-stage spaces and u64 VAs (spilled values).  ``out``: per
    job the pinned host tensors to fill (e.g. views of a buffer shared with
    another process); ``None`` entries are allocated.

    ``words``: per job ``(words int32, None, LaneExceptions)`` -- one
    pv_translate_words lane word per VA (4 bytes back, as many as the VAs
    going in; :func:`unpack_words`) plus the exception records of the lanes
    whose value the word cannot carry, fetched after the pipeline drains (a
    batch with more than ``exc_cap`` such lanes runs again with room for all
    of them)."""
    import torch

    if words:
        return _translate_host_words(image, jobs, chunk, out, exc_cap)

    outs, work = [], []
    dtype = torch.int32
    srcs = []
    for space, host_vas in jobs:
        if host_vas.dtype not in (torch.int32, torch.int64):
            host_vas = host_vas.to(torch.int64)
        if host_vas.dtype == torch.int64:
            dtype = torch.int64
        srcs.append((space, host_vas))
    for k, (space, host_vas) in enumerate(srcs):
        src = host_vas if host_vas.dtype == dtype else host_vas.to(dtype)
        if not src.is_pinned():
            src = src.pin_memory()
        n = src.numel()
        two = space.mode == N.TWO_STAGE
        need_aux = two or (packed and dtype == torch.int64)
        given = out[k] if out is not None and out[k] is not None else (None, None, None)
        value = given[0] if given[0] is not None else torch.empty(n, dtype=torch.int64, pin_memory=True)
        status = None if packed else (given[1] if given[1] is not None else
                                      torch.empty(n, dtype=torch.int32, pin_memory=True))
        # one-stage walks never produce a TDP-stage trap: aux is identically 0
        if need_aux:
            aux = given[2] if given[2] is not None else torch.empty(n, dtype=torch.int64, pin_memory=True)
        else:
            aux = torch.zeros(1, dtype=torch.int64).expand(n)
        outs.append((value, status, aux))
        for start in range(0, n, chunk):
            work.append((space, need_aux, src, value, status, aux, start, min(chunk, n - start)))
    per_lane_out = 8 if packed else 12
    last_host_io["h2d"] = sum(w[2].element_size() * w[7] for w in work)
    last_host_io["d2h"] = sum(w[7] * (per_lane_out + (8 if w[1] else 0)) for w in work)  # value (+ status) (+ aux)
    if not work:
        return outs
    compute = torch.cuda.current_stream()
    h2d, d2h, bufs = _pipe(dtype, chunk, False)
    h2d.wait_stream(compute)  # the caller's earlier work first
    for i, (space, need_aux, src, value, status, aux, start, m) in enumerate(work):
        d_vas, d_val, d_st, d_aux, ev_in, ev_done, ev_out = bufs[i % 2]
        if i >= 2:
            h2d.wait_event(ev_out)  # buffers of chunk i-2 fully drained
        with torch.cuda.stream(h2d):
            d_vas[:m].copy_(src[start:start + m], non_blocking=True)
            ev_in.record(h2d)
        compute.wait_event(ev_in)
        if need_aux:
            d_aux[:m].zero_()
        translate_lanes(image, _host_plan(image, space, m), d_vas[:m],
                        out=(d_val[:m], None if packed else d_st[:m], d_aux[:m]), packed=packed)
        ev_done.record(compute)
        d2h.wait_event(ev_done)
        with torch.cuda.stream(d2h):
            value[start:start + m].copy_(d_val[:m], non_blocking=True)
            if not packed:
                status[start:start + m].copy_(d_st[:m], non_blocking=True)
            if need_aux:
                aux[start:start + m].copy_(d_aux[:m], non_blocking=True)
            ev_out.record(d2h)
    d2h.synchronize()
    compute.synchronize()
    return outs


_pipe_tls = threading.local()


def _pipe(dtype, chunk: int, words: bool, nbuf: int = 2):
    """The calling thread's side streams, ``nbuf`` device chunk buffer sets
    and events of the host pipeline, reused across calls (every call drains
    them before it returns)."""
    import torch

    cache = getattr(_pipe_tls, "cache", None)
    if cache is None:
        cache = _pipe_tls.cache = {}
    key = (torch.cuda.current_device(), dtype, chunk, words, nbuf)
    st = cache.get(key)
    if st is None:
        if words:
            bufs = [(torch.empty(chunk, dtype=dtype, device="cuda"), torch.empty(chunk, dtype=torch.int32, device="cuda"),
                     torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()) for _ in range(nbuf)]
        else:
            bufs = [(torch.empty(chunk, dtype=dtype, device="cuda"), torch.empty(chunk, dtype=torch.int64, device="cuda"),
                     torch.empty(chunk, dtype=torch.int32, device="cuda"), torch.zeros(chunk, dtype=torch.int64, device="cuda"),
                     torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()) for _ in range(2)]
        st = cache[key] = (torch.cuda.Stream(), torch.cuda.Stream(), bufs)
    return st


def _host_plan(image, space: Space, m: int) -> "TranslatePlan":
    """The one-segment TranslatePlan of ``m`` lanes through ``space``, kept on
    the image across calls (descriptors are uploaded once)."""
    cache = getattr(image, "_host_plans", None)
    if cache is None:
        cache = image._host_plans = {}
    plan = cache.get((space, m))
    if plan is None:
        if len(cache) > 512:
            cache.clear()
        plan = cache[(space, m)] = TranslatePlan([space], [(0, m, 0)], image=image)
    return plan


_WORD_BUFS = 2


def _translate_host_words(image, jobs, chunk: int, out, exc_cap: int):
    """translate_host_many(words=True): the same two-buffer-set pipeline with
    4-byte lane words each way; the exception records of every chunk append
    to one device list read once at the end."""
    import torch

    # pipeline shape (A/B knobs): lanes per chunk and chunk buffer sets in flight
    chunk = int(os.environ.get("PV_HOST_WORD_CHUNK", chunk))
    nbuf = int(os.environ.get("PV_HOST_WORD_BUFS", _WORD_BUFS))
    srcs, dtype = [], torch.int32
    for space, host_vas in jobs:
        if host_vas.dtype not in (torch.int32, torch.int64):
            host_vas = host_vas.to(torch.int64)
        if host_vas.dtype == torch.int64:
            dtype = torch.int64
        srcs.append((space, host_vas))
    outs, work, base = [], [], []
    lane0 = 0
    for k, (space, host_vas) in enumerate(srcs):
        src = host_vas if host_vas.dtype == dtype else host_vas.to(dtype)
        if not src.is_pinned():
            src = src.pin_memory()
        n = src.numel()
        given = out[k] if out is not None and out[k] is not None else (None, None, None)
        w = given[0] if given[0] is not None else torch.empty(n, dtype=torch.int32, pin_memory=True)
        if w.dtype != torch.int32 or w.numel() != n:
            raise ValueError("words=True fills int32 tensors of one word per VA")
        outs.append(w)
        base.append(lane0)
        for start in range(0, n, chunk):
            work.append((space, src, w, lane0, start, min(chunk, n - start)))
        lane0 += n
    total = lane0
    cap = min(total, exc_cap)
    compute = torch.cuda.current_stream()
    exc_list = ExcList(cap)
    if work:
        h2d, d2h, bufs = _pipe(dtype, chunk, True, nbuf)
        h2d.wait_stream(compute)  # the caller's earlier work (and the counter reset above) first
        for i, (space, src, w, l0, start, m) in enumerate(work):
            d_vas, d_w, ev_in, ev_done, ev_out = bufs[i % nbuf]
            if i >= nbuf:
                h2d.wait_event(ev_out)  # buffers of chunk i-nbuf fully drained
            with torch.cuda.stream(h2d):
                d_vas[:m].copy_(src[start:start + m], non_blocking=True)
                ev_in.record(h2d)
            compute.wait_event(ev_in)
            translate_words(image, _host_plan(image, space, m), d_vas[:m], d_w[:m], exc_list, l0 + start)
            ev_done.record(compute)
            d2h.wait_event(ev_done)
            with torch.cuda.stream(d2h):
                w[start:start + m].copy_(d_w[:m], non_blocking=True)
                ev_out.record(d2h)
        d2h.synchronize()
    allx, n_exc, overflow = exc_list.read()
    if overflow:  # a stripe ran out of room: once more with room for every stripe's records
        return _translate_host_words(image, jobs, chunk, out, exc_list.needed())
    last_host_io["h2d"] = sum(w[1].element_size() * w[5] for w in work)
    last_host_io["d2h"] = 4 * total + 8 * N.EXC_STRIPES + n_exc * 8 * N.EXC_WORDS
    excs = [LaneExceptions() for _ in outs]
    if n_exc:
        job = np.searchsorted(np.asarray(base, np.int64), allx.lane, side="right") - 1
        for k in np.unique(job):
            sel = job == k
            excs[k] = LaneExceptions(allx.lane[sel] - base[k], allx.value[sel], allx.aux[sel], allx.status[sel])
    return [(w, None, x) for w, x in zip(outs, excs)]


# ---- K4: FIFO cache state packing -------------------------------------------

def pack_fifo(caches) -> np.ndarray:
    """TranslationCache objects -> pv_fifo rows (int64 view)."""
    rows = np.zeros((len(caches), N.FIFO_WORDS), dtype=np.uint64)
    for i, c in enumerate(caches):
        if not 1 <= c.capacity <= N.FIFO_MAX:
            raise ValueError(f"device FIFO replay supports capacities 1..{N.FIFO_MAX}, got {c.capacity}")
        entries = c.entries()
        for j, (k, v) in enumerate(entries):
            rows[i, j] = k & U64
            rows[i, N.FIFO_MAX + j] = v & U64
        rows[i, 2 * N.FIFO_MAX] = c.hits
        rows[i, 2 * N.FIFO_MAX + 1] = c.misses
        rows[i, 2 * N.FIFO_MAX + 2] = c.capacity | (len(entries) << 32)
        rows[i, 2 * N.FIFO_MAX + 3] = 0  # head = 0
    return rows.view(np.int64)


def unpack_fifo(rows: np.ndarray, caches) -> None:
    rows = rows.view(np.uint64)
    for i, c in enumerate(caches):
        cap = int(rows[i, 2 * N.FIFO_MAX + 2]) & 0xFFFFFFFF
        length = int(rows[i, 2 * N.FIFO_MAX + 2]) >> 32
        head = int(rows[i, 2 * N.FIFO_MAX + 3]) & 0xFFFFFFFF
        entries = []
        for j in range(length):
            slot = (head + j) % cap
            entries.append((int(rows[i, slot]), int(rows[i, N.FIFO_MAX + slot])))
        c._load_state(entries, int(rows[i, 2 * N.FIFO_MAX]), int(rows[i, 2 * N.FIFO_MAX + 1]))


def _windows(proc_off: np.ndarray) -> np.ndarray:
    """Per-process window offsets (32 lookups per window) from lookup offsets."""
    counts = np.diff(proc_off.astype(np.int64))
    win = np.zeros(len(proc_off), dtype=np.int64)
    np.cumsum((counts + 31) // 32, out=win[1:])
    return win


def fifo_capacity(caches) -> int:
    caps = {c.capacity for c in caches}
    if len(caps) != 1:
        raise ValueError("a FIFO replay batch needs one cache capacity for every process")
    cap = caps.pop()
    if not 1 <= cap <= N.FIFO_MAX:
        raise ValueError(f"device FIFO replay supports capacities 1..{N.FIFO_MAX}, got {cap}")
    return cap


def _fifo_scratch(n_lookups: int, n_windows: int, cap: int):
    import torch

    nbytes = int(N.load().pv_fifo_scratch_bytes(n_lookups, n_windows, cap))
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda"), nbytes


def fifo_replay_lanes(vas, lane_idx, proc_off: np.ndarray, fifo_dev, value, status, capacity: int) -> None:
    """K4 over translate lanes: lookups of process p are lanes
    lane_idx[proc_off[p]:proc_off[p+1]] in order (proc_off host array)."""
    import torch

    lib = N.lib()
    flags = N.VA32 if vas.dtype == torch.int32 else 0
    win = _windows(proc_off)
    scratch, nbytes = _fifo_scratch(int(proc_off[-1]), int(win[-1]), capacity)
    off_d = _to_dev(np.asarray(proc_off, dtype=np.int64))
    win_d = _to_dev(win)
    N.check(lib.pv_fifo_replay(vas.data_ptr(), flags, lane_idx.data_ptr(), off_d.data_ptr(), win_d.data_ptr(),
                               len(proc_off) - 1, int(proc_off[-1]), int(win[-1]), capacity, fifo_dev.data_ptr(),
                               value.data_ptr(),
                               status.data_ptr(), scratch.data_ptr(), nbytes, _stream().cuda_stream),
            "pv_fifo_replay")


# ---- K2/K3: batched copy -----------------------------------------------------

def page_spans(gva: np.ndarray, length: np.ndarray) -> np.ndarray:
    gva = gva.astype(np.uint64)
    length = length.astype(np.uint64)
    span = np.zeros(len(gva), dtype=np.uint64)
    nz = length > 0
    span[nz] = ((gva[nz] + length[nz] - np.uint64(1)) >> np.uint64(PAGE_SHIFT)) - (gva[nz] >> np.uint64(PAGE_SHIFT)) \
        + np.uint64(1)
    return span


class CopyPlan:
    """Device-resident descriptors of a copy batch (reusable across runs)."""

    def __init__(self, spaces: list[Space], ops: np.ndarray, *, fifo_groups=None, shims=None):
        """``ops``: uint64 rows (gva, len, buf_off, space).  ``fifo_groups``:
        optional list of lists of op indices, one per process whose
        TranslationCache applies (program order).  ``shims``: optional
        :class:`Shim` (or None) per space -- the hybrid resolver's trap shim
        runs on the device for those spaces (pv_copy_shim)."""
        import torch

        ops = np.ascontiguousarray(ops, dtype=np.uint64).reshape(-1, 4)
        self.n_ops = len(ops)
        spans = page_spans(ops[:, 0], ops[:, 1])
        page_off = np.zeros(self.n_ops + 1, dtype=np.uint64)
        np.cumsum(spans, out=page_off[1:])
        self.n_pages = int(page_off[-1])
        self.host_ops = ops
        self.host_page_off = page_off
        up = [_i64([sp.words() for sp in spaces]).reshape(-1, 4), ops.view(np.int64), page_off.view(np.int64)]
        if shims is not None and any(sh is not None for sh in shims):
            up.append(_i64([(sh or NO_SHIM).words() for sh in shims]).reshape(-1, 4))
        up = _to_dev_many(up)
        self.spaces, self.ops, self.page_off = up[0], up[1], up[2]
        np_ = max(self.n_pages, 1)
        self.page_hpa = torch.empty(np_, dtype=torch.int64, device="cuda")
        self.page_status = torch.empty(np_, dtype=torch.int32, device="cuda")
        self.page_aux = torch.empty(np_, dtype=torch.int64, device="cuda")
        self.first_bad = torch.empty(max(self.n_ops, 1), dtype=torch.int64, device="cuda")
        self.results = torch.empty((max(self.n_ops, 1), 4), dtype=torch.int64, device="cuda")
        self.conflict = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.shims = None
        if len(up) > 3:
            self.shims = up[3]
            self.shim_written = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.fifo_groups = fifo_groups
        if fifo_groups is not None:
            # lookup stream: the pages of each process's ops, op order, page order
            po = page_off.astype(np.int64)
            sp = spans.astype(np.int64)
            look_op, look_page, lk_off = [], [], [0]
            for g in fifo_groups:
                g = np.asarray(g, dtype=np.int64)
                cnt = sp[g]
                total = int(cnt.sum())
                excl = np.zeros(len(g), dtype=np.int64)
                if len(g) > 1:
                    np.cumsum(cnt[:-1], out=excl[1:])
                look_op.append(np.repeat(g, cnt))
                look_page.append(np.repeat(po[g] - excl, cnt) + np.arange(total, dtype=np.int64))
                lk_off.append(lk_off[-1] + total)
            lk_off = np.asarray(lk_off, dtype=np.int64)
            lop = np.concatenate(look_op) if look_op else np.zeros(0, np.int64)
            lpg = np.concatenate(look_page) if look_page else np.zeros(0, np.int64)
            self.fifo_lookups = int(lk_off[-1])
            self.fifo_win = _windows(lk_off)
            lop = lop.astype(np.uint32).view(np.int32) if len(lop) else np.zeros(1, np.int32)
            lpg = lpg if len(lpg) else np.zeros(1, np.int64)
            self.fifo_look_op, self.fifo_look_page, self.fifo_off, self.fifo_win_d = _to_dev_many(
                [lop, lpg, lk_off, self.fifo_win])
            self.fifo_scratch = None


def _aligned16(plan: "CopyPlan", buf_ptr: int) -> bool:
    """(gva - (buf + buf_off)) % 16 == 0 for every op (host check, cached)."""
    key = buf_ptr % 16
    cache = plan.__dict__.setdefault("_aligned_cache", {})
    if key not in cache:
        o = plan.host_ops
        cache[key] = bool(len(o) == 0 or (((o[:, 0] - o[:, 2] - np.uint64(key)) % np.uint64(16)) == 0).all())
    return cache[key]


CopyPlan.aligned16 = lambda self, buf_ptr: _aligned16(self, buf_ptr)


def exec_hint(plan: "CopyPlan", buf_ptr: int) -> int:
    """pv_copy_exec flag selecting the TMA bulk path (host-proven alignment)."""
    if os.environ.get("PV_EXEC_LSU") == "1":
        return 0
    return N.COPY_ALIGNED16 if plan.aligned16(buf_ptr) else 0


def _stream_key() -> int:
    return _stream().cuda_stream


def _per_stream(obj, name: str, make):
    """State of ``obj`` private to the current CUDA stream (created by
    ``make()`` on first use).  Calls on one stream run in order and may reuse
    it; calls on another stream (another host thread, SURVEY.md 8(b)
    threading) never share it."""
    table = obj.__dict__.setdefault("_per_stream_state", {})
    key = (name, _stream_key())
    st = table.get(key)
    if st is None:
        st = table[key] = make()
    return st


class OwnerMap:
    """Conflict maps of one (image, stream): ``map`` holds one u64 per page,
    the stamps (epoch << 40 | chunk + 1) of pv_copy_stamp; ``nodes`` one u32
    per page, the table-node marks of pv_copy_plan_nodes.  Each to_guest
    batch takes a new epoch, so neither map is cleared between batches."""

    def __init__(self, npages: int):
        import torch

        self.map = torch.zeros(npages, dtype=torch.int64, device="cuda")
        self.nodes = torch.zeros(npages, dtype=torch.int32, device="cuda")
        self.npages = npages
        self.epoch = 0

    def next_epoch(self) -> int:
        self.epoch += 1
        if self.epoch >= 1 << 24:
            self.map.zero_()
            self.nodes.zero_()
            self.epoch = 1
        return self.epoch


def _owner_map(image) -> OwnerMap:
    """The current stream's conflict stamp map of ``image``."""
    return _per_stream(image, "owner", lambda: OwnerMap(image.npages))


class _Grow:
    """A zero-filled device byte buffer that grows on demand."""

    def __init__(self):
        self.t = None

    def get(self, need: int):
        import torch

        if self.t is None or self.t.numel() < need:
            self.t = torch.zeros(max(need, 1), dtype=torch.uint8, device="cuda")
        return self.t


def _shim_scratch(image, n_pages: int):
    """The current stream's zero-filled scratch of pv_copy_shim for
    ``image`` (grown on demand; every call leaves it zero-filled)."""
    need = int(N.lib().pv_copy_shim_scratch_bytes(n_pages))
    return _per_stream(image, "shim", _Grow).get(need)


def copy_launch(image, plan: CopyPlan, direction: int, buf, *, fifo_dev=None, fifo_cap: int = 10,
                detect_conflicts: bool = True, track_dirty: bool = True, buf_ready=None,
                buf_bytes: int | None = None) -> None:
    """Enqueue plan (+ FIFO replay) (+ conflict stamp) + exec on the current
    stream.  Results land in ``plan.results`` / ``plan.conflict``.
    ``buf_ready`` (a CUDA event, optional): the buffer is still arriving on
    another stream; only the exec waits for it, the plan passes overlap it.
    ``buf_bytes`` (default ``buf.numel()``): bytes of ``buf`` the ops may
    touch; chunks reaching past it move only what the buffer holds."""
    with image._lock:  # enqueue atomically w.r.t. MemoryImage.pull (threads)
        _copy_launch(image, plan, direction, buf, fifo_dev, fifo_cap, detect_conflicts, track_dirty, buf_ready,
                     buf_bytes)


def _copy_launch(image, plan, direction, buf, fifo_dev, fifo_cap, detect_conflicts, track_dirty, buf_ready,
                 buf_bytes) -> None:
    percall.park()  # the per-call server must not hold a CTA slot this grid counts on
    lib = N.lib()
    dev_img = image.device()
    s = _stream().cuda_stream
    if plan.n_ops == 0:
        return
    plan.first_bad.fill_(-1)
    plan.results.zero_()
    plan.conflict.zero_()
    if plan.n_pages:
        stamp = direction == N.TO_GUEST and detect_conflicts
        if stamp:
            # a to_guest batch marks the table nodes its walks read: a chunk
            # landing on one is a table hazard (pv_copy_plan_nodes)
            owner = _owner_map(image)
            epoch = owner.next_epoch()
            N.check(lib.pv_copy_plan_nodes(dev_img.data_ptr(), image.nbytes, plan.spaces.data_ptr(),
                                           plan.ops.data_ptr(), plan.n_ops, plan.page_off.data_ptr(), plan.n_pages,
                                           plan.page_hpa.data_ptr(), plan.page_status.data_ptr(),
                                           plan.page_aux.data_ptr(), plan.first_bad.data_ptr(),
                                           owner.nodes.data_ptr(), owner.npages, epoch, s), "pv_copy_plan_nodes")
        else:
            N.check(lib.pv_copy_plan(dev_img.data_ptr(), image.nbytes, plan.spaces.data_ptr(), plan.ops.data_ptr(),
                                     plan.n_ops, plan.page_off.data_ptr(), plan.n_pages, direction,
                                     plan.page_hpa.data_ptr(), plan.page_status.data_ptr(), plan.page_aux.data_ptr(),
                                     plan.first_bad.data_ptr(), None, 0, None, s), "pv_copy_plan")
        if plan.shims is not None:
            scratch = _shim_scratch(image, plan.n_pages)
            N.check(lib.pv_copy_shim(dev_img.data_ptr(), image.nbytes, plan.spaces.data_ptr(), plan.shims.data_ptr(),
                                     plan.ops.data_ptr(), plan.n_ops, plan.page_off.data_ptr(), plan.n_pages,
                                     plan.page_hpa.data_ptr(), plan.page_status.data_ptr(), plan.first_bad.data_ptr(),
                                     image.dirty_map().data_ptr(), plan.shim_written.data_ptr(), scratch.data_ptr(),
                                     scratch.numel(), s), "pv_copy_shim")
        if fifo_dev is not None and plan.fifo_lookups:
            cap = fifo_cap
            if plan.fifo_scratch is None or plan.fifo_cap != cap:
                plan.fifo_cap = cap
                plan.fifo_scratch = _fifo_scratch(plan.fifo_lookups, int(plan.fifo_win[-1]), cap)
            scratch, nbytes = plan.fifo_scratch
            N.check(lib.pv_copy_fifo_replay(plan.ops.data_ptr(), plan.page_off.data_ptr(),
                                            plan.fifo_look_page.data_ptr(), plan.fifo_look_op.data_ptr(),
                                            plan.fifo_off.data_ptr(), plan.fifo_win_d.data_ptr(),
                                            plan.fifo_off.numel() - 1, plan.fifo_lookups, int(plan.fifo_win[-1]), cap,
                                            fifo_dev.data_ptr(), image.nbytes,
                                            plan.page_hpa.data_ptr(), plan.page_status.data_ptr(),
                                            plan.first_bad.data_ptr(), scratch.data_ptr(), nbytes, s),
                    "pv_copy_fifo_replay")
        abort = None
        if stamp:
            N.check(lib.pv_copy_stamp(plan.page_off.data_ptr(), plan.n_ops, plan.n_pages, plan.page_hpa.data_ptr(),
                                      plan.first_bad.data_ptr(), owner.map.data_ptr(), image.npages, epoch,
                                      plan.conflict.data_ptr(), owner.nodes.data_ptr(), s), "pv_copy_stamp")
            abort = plan.conflict.data_ptr()
        dirty = image.dirty_map().data_ptr() if (direction == N.TO_GUEST and track_dirty) else None
        # batches whose buffer and guest pages are 16-byte co-aligned move
        # through the TMA bulk exec (pv_copy.cu exec_bulk_kernel); the LSU exec
        # takes the rest (PV_EXEC_LSU=1 forces it, for A/B runs)
        hint = exec_hint(plan, buf.data_ptr())
        if buf_ready is not None:
            _stream().wait_event(buf_ready)
        N.check(lib.pv_copy_exec(dev_img.data_ptr(), image.nbytes, plan.ops.data_ptr(), plan.n_ops,
                                 plan.page_off.data_ptr(), plan.n_pages, direction | hint, plan.page_hpa.data_ptr(),
                                 plan.page_status.data_ptr(), plan.page_aux.data_ptr(), plan.first_bad.data_ptr(),
                                 buf.data_ptr(), buf.numel() if buf_bytes is None else buf_bytes,
                                 plan.results.data_ptr(), dirty, abort, s),
                "pv_copy_exec")
        if direction == N.TO_GUEST:
            image.note_device_write()


@dataclass
class OpOutcome:
    """Per-op outcome of a copy batch (decoded pv_op_result)."""

    status: int
    copied: int
    value: int
    aux: int
    fail_page: int


def decode_results(res: np.ndarray) -> list[OpOutcome]:
    r = res.view(np.uint64)
    out = []
    for row in r:
        out.append(OpOutcome(status=int(row[3]) & 0xFFFFFFFF, copied=int(row[0]), value=int(row[1]),
                             aux=int(row[2]), fail_page=int(row[3]) >> 32))
    return out


def copy_ordered(image, plan: CopyPlan, buf, buf_bytes: int | None = None) -> None:
    """Ordered execution of a planned to_guest batch whose chunks share
    destination pages (pv_copy_ordered): exact last-writer-wins."""
    percall.park()  # the per-call server must not hold a CTA slot this grid counts on
    import torch

    lib = N.lib()
    dev_img = image.device()
    nbytes = int(lib.pv_copy_ordered_scratch_bytes(plan.n_pages, image.nbytes))
    scratch = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    with image.writing():
        N.check(lib.pv_copy_ordered(dev_img.data_ptr(), image.nbytes, plan.ops.data_ptr(), plan.n_ops,
                                    plan.page_off.data_ptr(), plan.n_pages, plan.page_hpa.data_ptr(),
                                    plan.page_status.data_ptr(), plan.page_aux.data_ptr(), plan.first_bad.data_ptr(),
                                    buf.data_ptr(), buf.numel() if buf_bytes is None else buf_bytes,
                                    plan.results.data_ptr(), image.dirty_map().data_ptr(),
                                    scratch.data_ptr(), nbytes, _stream().cuda_stream), "pv_copy_ordered")


def copy_ops(image, spaces: list[Space], ops: np.ndarray, direction: int, buf, *, caches=None, fifo_groups=None,
             detect_conflicts: bool = True, shims=None, buf_ready=None, buf_bytes: int | None = None) -> list[OpOutcome]:
    """Run a batch of copies with the reference's sequential semantics.

    ``caches`` (with ``fifo_groups``) are host TranslationCache objects whose
    state is replayed on the device and written back.  When the stamp pass
    finds two chunks of a to_guest batch writing one hpa page, the exec kernel
    stands down and the batch runs through the ordered path
    (:func:`copy_ordered`), which reproduces last-writer-wins exactly.  When a
    chunk would land on a page-table node the batch walks (a table hazard,
    pv_copy_plan_nodes), nothing moves and the batch runs page by page in
    program order instead (:func:`_copy_pagewise`).
    """
    cap = fifo_capacity(caches) if caches is not None else 10
    plan = CopyPlan(spaces, ops, fifo_groups=fifo_groups if caches is not None else None, shims=shims)
    fifo_dev = _to_dev_many([pack_fifo(caches).view(np.int64)])[0] if caches is not None else None
    copy_launch(image, plan, direction, buf, fifo_dev=fifo_dev, fifo_cap=cap, detect_conflicts=detect_conflicts,
                buf_ready=buf_ready, buf_bytes=buf_bytes)
    conflict = int(plan.conflict.item()) if direction == N.TO_GUEST and detect_conflicts else 0
    if conflict & N.CONFLICT_TABLE:
        if plan.shims is not None and int(plan.shim_written.item()):
            image.note_device_write()
        return _copy_pagewise(image, spaces, plan.host_ops, direction, buf, caches, fifo_groups, shims, buf_bytes)
    if conflict:
        copy_ordered(image, plan, buf, buf_bytes)
    results = decode_results(plan.results.cpu().numpy())
    if plan.shims is not None and int(plan.shim_written.item()):
        image.note_device_write()  # the shim rewrote shadow leaves
    if caches is not None:
        unpack_fifo(fifo_dev.cpu().numpy(), caches)
    return results


def _copy_pagewise(image, spaces, ops, direction, buf, caches, fifo_groups, shims, buf_bytes) -> list[OpOutcome]:
    """A to_guest batch with a table hazard, one page at a time in program
    order: each page is a one-chunk batch (translated -- through its
    process's FIFO cache when there is one -- then written), so later pages
    walk the tables earlier chunks wrote, exactly like copy_user_buffer
    (memvirt.py:615-627).  With hybrid spaces (``shims``), the batch stops
    at the first op whose page still traps after the device shim: the caller
    finishes that op through the per-op shim and re-plans the rest."""
    group_of = {}
    if caches is not None:
        for g, members in enumerate(fifo_groups):
            for i in members:
                group_of[int(i)] = g
    out = []
    stopped = False
    for i, row in enumerate(np.asarray(ops, dtype=np.uint64).reshape(-1, 4)):
        gva, length, off, sp = (int(x) for x in row)
        if stopped:
            out.append(OpOutcome(status=N.ST_OK, copied=0, value=0, aux=0, fail_page=0))
            continue
        g = group_of.get(i)
        sub_caches = None if g is None else [caches[g]]
        res = OpOutcome(status=N.ST_OK, copied=length, value=0, aux=0, fail_page=0)
        done, k = 0, 0
        while done < length:
            cur = (gva + done) & U64
            chunk = min(length - done, PAGE_SIZE - (cur & PAGE_MASK))
            sub = np.array([[cur, chunk, off + done, 0]], dtype=np.uint64)
            r = copy_ops(image, [spaces[sp]], sub, direction, buf, caches=sub_caches,
                         fifo_groups=[[0]] if sub_caches is not None else None, detect_conflicts=False,
                         shims=None if shims is None else [shims[sp]], buf_bytes=buf_bytes)[0]
            if r.status != N.ST_OK:
                res = OpOutcome(status=r.status, copied=done, value=r.value, aux=r.aux, fail_page=k)
                stopped = shims is not None and kind(r.status) in (N.ST_TRAP, N.ST_TRAP2)
                break
            done += chunk
            k += 1
        out.append(res)
    return out




# ---- batched table construction (pv_map_plan / pv_map_commit) ------------------

def _map_scratch(image):
    """The current stream's pv_map_plan scratch for ``image``."""
    return _per_stream(image, "map", _Grow).get(int(N.lib().pv_map_scratch_bytes()))


class TableBuild:
    """One table of a batched map on the device: the plan of ``vas`` (device
    int64 tensor, page aligned) over the window at byte ``base`` with root
    ``root_pfn`` (pv_map_plan).  ``need`` / ``bad`` / ``count`` stay on the
    device until :meth:`stats` reads them."""

    def __init__(self, image, base: int, root_pfn: int, vas):
        import torch

        lib = N.lib()
        self.image, self.base, self.root, self.vas = image, base, root_pfn, vas
        n = vas.numel()
        dev = image.device()
        self.need = torch.empty(n, dtype=torch.uint8, device="cuda")
        self.bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        N.check(lib.pv_map_plan(dev.data_ptr(), image.nbytes, base, root_pfn, vas.data_ptr(), n,
                                self.need.data_ptr(), self.bad.data_ptr(), _map_scratch(image).data_ptr(),
                                _stream().cuda_stream), "pv_map_plan")
        self.nodes = (self.need & 1).to(torch.int64) + (self.need >> 1).to(torch.int64)

    def summary(self):
        """Device scalars (bad page or -1, node frames needed) for one sync."""
        import torch

        return torch.stack([self.bad[0], self.nodes.sum()])

    def commit(self, frames: np.ndarray, *, data_first: bool, targets=None, target_add: int = 0,
               leaf_flags: int = 0x3, out_data=None) -> None:
        """Write the table given the frames drawn from the allocator (in
        allocation order)."""
        import torch

        lib = N.lib()
        image = self.image
        dev = image.device()
        per = self.nodes + (1 if data_first else 0)
        frame_off = torch.cumsum(per, 0) - per
        fr = _to_dev(frames.astype(np.int64)) if len(frames) else None
        pages = (self.base >> PAGE_SHIFT) + frames
        hot = image._maybe_nonzero[pages] if len(frames) else np.zeros(0, bool)
        hot_d = _to_dev(hot.astype(np.uint8)) if hot.any() else None
        with image.writing():
            N.check(lib.pv_map_commit(dev.data_ptr(), image.nbytes, self.base, self.root, self.vas.data_ptr(),
                                      self.vas.numel(), self.need.data_ptr(), None if fr is None else fr.data_ptr(),
                                      len(frames), frame_off.data_ptr(), None if hot_d is None else hot_d.data_ptr(),
                                      1 if data_first else 0, None if targets is None else targets.data_ptr(), target_add,
                                      leaf_flags, None if out_data is None else out_data.data_ptr(),
                                      image.dirty_map().data_ptr(), _stream().cuda_stream), "pv_map_commit")
        image.host_epoch += 1  # table structure changed: leaf-index scans must look again
