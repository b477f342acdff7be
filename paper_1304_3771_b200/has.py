"""Drop-in HAS access classes: the operator API device drivers call.

Drivers only ever see ``ctx.mem`` with ``copy_to_user(gva, data) -> int``,
``copy_from_user(gva, length) -> bytes`` and ``map_page(gva, hpa)``
(devices.py:8-11).  This module provides the reference's implementations of
that interface (backend.py:75-216) with the copies running on the HBM data
plane, plus batch forms that move many operations per launch:

* ``copy_to_user_batch(gvas, lengths, src, offsets=None)``
* ``copy_from_user_batch(gvas, lengths) -> (payload, outcomes)``

A batch behaves exactly like the same calls issued one after another
(translation per page, FIFO cache state, prefix-on-fault, last-writer-wins on
overlapping destinations); per-op outcomes are the bytes copied (int) or the
exception instance the single call would have raised.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _native as N
from . import dataplane as dp
from .errors import PageFault, SimError, TdpUnsupported
from .memvirt import (
    PAGE_MASK,
    PAGE_SHIFT,
    PAGE_SIZE,
    Gva,
    HybridTopLevel,
    MemoryVirtualizer,
    ProcessSpace,
    TableEditor,
    TranslationCache,
    copy_user_buffer,
    resolve_hybrid_with_fixup,
    walk_guest,
)


class GuestProcessRecord:
    """Backend state of one guest process (backend.py:259-296): the stored
    root, one FIFO cache + translator shared by the process's threads, the
    per-process hybrid top level and the default trap shim."""

    def __init__(self, guest, space: ProcessSpace, memv: MemoryVirtualizer):
        self.guest_id = guest.id
        self.pid = space.pid
        self.guest = guest
        self.space = space
        self.stored_pt_root = space.guest_root
        self.translation_cache = TranslationCache()
        self.translator = memv.translator(space, self.translation_cache)
        self.result_pages: dict[int, tuple[int, int]] = {}
        self.hybrid = HybridTopLevel(memv.host_mem, memv.host_alloc)
        self.active_hybrid = None
        self.hw_translations = 0
        self.dispatch_lock = threading.RLock()
        self._memv = memv

    def activate_hybrid(self, memv: MemoryVirtualizer) -> None:
        if self.guest.mem_mode == "tdp":
            raise TdpUnsupported("hybrid table activation for a TDP guest")
        self.active_hybrid = self.hybrid.build(self.space.shadow_root, memv.host_kernel_root)

    def trap_shim(self, trap) -> None:
        """Re-sync the trapping shadow leaf from the guest's own tables."""
        space, memv = self.space, self._memv
        page_va = trap.va & ~PAGE_MASK
        gpa = walk_guest(Gva(page_va), space.guest_root, space.guest.mem)
        hpa = memv.gpa_to_hpa(gpa, self.guest_id)
        TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc).map(
            page_va, hpa >> PAGE_SHIFT, replace=True)


def _as_src_tensor(src):
    import torch

    if isinstance(src, torch.Tensor):
        return src if src.is_cuda else src.to("cuda")
    return dp._to_dev(np.frombuffer(bytes(src), dtype=np.uint8) if not isinstance(src, np.ndarray)
                      else np.ascontiguousarray(src, dtype=np.uint8))


_h2d_stream = None


def _src_async(src):
    """(device tensor, ready event or None).  A pinned host tensor starts its
    H2D copy on a side stream, so the batch's plan / shim / stamp passes (and
    the host work building them) overlap the transfer; only the exec waits."""
    import torch

    global _h2d_stream
    if isinstance(src, torch.Tensor) and not src.is_cuda and src.is_pinned():
        if _h2d_stream is None:
            _h2d_stream = torch.cuda.Stream()
        side = _h2d_stream
        side.wait_stream(torch.cuda.current_stream())  # the destination allocation is ordered on the main stream
        with torch.cuda.stream(side):
            dev = torch.empty(src.shape, dtype=src.dtype, device="cuda")
            dev.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        dev.record_stream(torch.cuda.current_stream())
        return dev, ev
    return _as_src_tensor(src), None


def _ops_rows(gvas, lengths, offsets, src_bytes=None):
    """pv_op rows (gva, len, buf_off, space 0).  With ``src_bytes`` (a
    to_guest source of that many bytes) each op has the slice semantics of
    ``copy_to_user(gva, src[off:off + len])``: a slice running past the
    source is shorter, so the op copies (and translates) fewer bytes."""
    gvas = np.asarray(gvas, dtype=np.uint64)
    lengths = np.asarray(lengths, dtype=np.uint64)
    if offsets is None:
        offsets = np.zeros(len(lengths), dtype=np.uint64)
        if len(lengths) > 1:
            np.cumsum(lengths[:-1], out=offsets[1:])
    offsets = np.asarray(offsets, dtype=np.uint64)
    if len(gvas) != len(lengths) or len(offsets) != len(lengths):
        raise ValueError("gvas, lengths and offsets must have one entry per op")
    if src_bytes is not None:
        room = np.where(offsets < np.uint64(src_bytes), np.uint64(src_bytes) - offsets, np.uint64(0))
        lengths = np.minimum(lengths, room)
    return np.stack([gvas, lengths, offsets, np.zeros(len(gvas), np.uint64)], axis=1)


def _nbytes(src) -> int:
    import torch

    if isinstance(src, torch.Tensor):
        return src.numel() * src.element_size()
    if isinstance(src, np.ndarray):
        return src.nbytes
    return len(memoryview(src).cast("B"))


def _decode_outcome(out: dp.OpOutcome, row, image_bytes: int):
    if out.status == N.ST_OK:
        return int(row[1])
    gva, length = int(row[0]), int(row[1])
    cur = gva + out.copied
    chunk = min(length - out.copied, PAGE_SIZE - (cur & PAGE_MASK))
    try:
        dp.raise_for(out.status, out.value, out.aux, cur, image_bytes, chunk=chunk, bytes_copied=out.copied)
    except (SimError, Exception) as exc:  # noqa: BLE001 - returned per op
        return exc
    return out.copied


class _BatchMixin:
    """Batch copies through one translator (``self._batch_translator``)."""

    def _batch(self, direction: int, rows: np.ndarray, buf, buf_ready=None):
        tr = self._batch_translator()
        image = self._memv.host_mem.backing
        space = tr.device_space
        caches = [tr.cache] if getattr(tr, "use_cache", False) else None
        groups = [list(range(len(rows)))] if caches is not None else None
        if not hasattr(tr, "_on_trap"):
            outs = dp.copy_ops(image, [space], rows, direction, buf, caches=caches, fifo_groups=groups,
                               buf_ready=buf_ready)
            return [_decode_outcome(o, r, image.nbytes) for o, r in zip(outs, rows)]
        # Hybrid resolver: the device runs the default shim for every trap it
        # can resolve exactly (pv_copy_shim).  Any other trap changes the
        # shadow table for every later page on the host, so the batch is cut
        # at that op, which finishes through the per-op shim loop, and the
        # rest is re-planned.  The device stops every op after the cut (no
        # byte moves through the pre-shim tables); with a replaced trap_shim
        # (device_shim None) nothing is fixed on the device and the first
        # trapping op is the cut.
        results = []
        start = 0
        shim = tr.device_shim or dp.NO_SHIM
        while start < len(rows):
            part = rows[start:]
            outs = dp.copy_ops(image, [space], part, direction, buf, shims=[shim], buf_ready=buf_ready)
            cut = next((i for i, o in enumerate(outs) if dp.kind(o.status) in (N.ST_TRAP, N.ST_TRAP2)), None)
            upto = len(outs) if cut is None else cut
            spans = dp.page_spans(part[:upto, 0], part[:upto, 1])  # _HybridResolver: one translation per page
            n = 0
            for o, r, sp in zip(outs[:upto], part[:upto], spans.tolist()):
                n += sp if o.status == N.ST_OK else o.fail_page + 1
                results.append(_decode_outcome(o, r, image.nbytes))
            tr._count(n)
            if cut is None:
                break
            r = part[cut]
            # pages before the trap were already copied by this batch
            o = outs[cut]
            results.append(self._finish_trapped(direction, r, buf, o))
            start += cut + 1
        return results

    def _finish_trapped(self, direction, row, buf, out):
        from .memvirt import _copy_device

        tr = self._batch_translator()
        gva, length, off = int(row[0]), int(row[1]), int(row[2])
        tr._count(out.fail_page)
        done = out.copied
        err = tr._on_trap(_trap_of(out, gva, done))
        if err is not None:
            tr._count(1)
            if isinstance(err, PageFault):
                err.bytes_copied = done
            return err
        view = buf[off:off + length]
        copied, err = _copy_device("to_guest" if direction == N.TO_GUEST else "from_guest", gva + done,
                                   length - done, view[done:], tr, self._memv.host_mem, tr.device_space,
                                   first_shimmed=True)
        if err is not None:
            if isinstance(err, PageFault):
                err.bytes_copied = done + copied
            return err
        return length

    def copy_to_user_batch(self, gvas, lengths, src, offsets=None):
        """copy_to_user(gvas[i], src[offsets[i]:offsets[i]+lengths[i]]) for
        every i, in order, on the device.  Returns per-op outcomes."""
        self._bump(len(gvas))
        rows = _ops_rows(gvas, lengths, offsets, src_bytes=_nbytes(src))
        buf, ready = _src_async(src)
        return self._batch(N.TO_GUEST, rows, buf, ready)

    def copy_from_user_batch(self, gvas, lengths):
        """copy_from_user for every op, in order.  Returns ``(payload,
        outcomes)``: payload is a device uint8 tensor with op i's bytes at
        its exclusive-prefix-sum offset."""
        import torch

        self._bump(len(gvas))
        rows = _ops_rows(gvas, lengths, None)
        total = int(np.asarray(lengths, dtype=np.uint64).sum())
        buf = torch.zeros(max(total, 1), dtype=torch.uint8, device="cuda")
        return buf[:total], self._batch(N.FROM_GUEST, rows, buf)


def _trap_of(out: dp.OpOutcome, gva: int, done: int):
    from .errors import TrapExit

    cur = gva + done
    k = dp.kind(out.status)
    return TrapExit(cur if k == N.ST_TRAP else out.aux, out.status & 0xF, out.value, (out.status >> 16) & 0x1FF)


class SoftwareHasAccess(_BatchMixin):
    """User-memory routines over software page walks through the process's
    FIFO-cached translator (backend.py:75-114)."""

    copies = 0
    maps = 0

    def __init__(self, record: GuestProcessRecord, memv: MemoryVirtualizer, log=None):
        self._record = record
        self._memv = memv
        self._log = log

    def _bump(self, n: int = 1) -> None:
        SoftwareHasAccess.copies += n

    def _batch_translator(self):
        return self._record.translator

    def copy_to_user(self, gva: int, data: bytes) -> int:
        self._bump()
        return copy_user_buffer("to_guest", Gva(gva), len(data), data, translator=self._record.translator,
                                host_mem=self._memv.host_mem)

    def copy_from_user(self, gva: int, length: int) -> bytes:
        self._bump()
        buf = bytearray(length)
        copy_user_buffer("from_guest", Gva(gva), length, buf, translator=self._record.translator,
                         host_mem=self._memv.host_mem)
        return bytes(buf)

    def map_page(self, gva: int, hpa: int) -> None:
        SoftwareHasAccess.maps += 1
        rec = self._record
        self._memv.map_page_into_guest(rec.space, Gva(gva), hpa, rec.space.guest.mem_mode,
                                       cache=rec.translation_cache)
        if self._log is not None:
            self._log.append("map", guest=rec.guest_id, process=rec.pid, gva=hex(gva), hpa=hex(hpa),
                             route="software")


class _HybridResolver:
    """Per-page resolution through the merged table with one shim fixup
    (backend.py:117-128).  ``device_space`` / ``_count`` / ``_on_trap`` let
    copy_user_buffer run whole copies on the device."""

    use_cache = False

    def __init__(self, record: GuestProcessRecord, memv: MemoryVirtualizer):
        self._record = record
        self._memv = memv

    @property
    def device_space(self) -> dp.Space:
        return dp.Space(self._memv.host_mem.base, self._record.active_hybrid.root_pfn, 0, N.ONE_STAGE)

    @property
    def device_shim(self):
        """The default shim as the device runs it (pv_copy_shim), or None when
        the record's shim was replaced (then traps go to the host per op)."""
        rec = self._record
        if "trap_shim" in rec.__dict__ or type(rec).trap_shim is not GuestProcessRecord.trap_shim:
            return None
        space, memv = rec.space, self._memv
        base = memv.guest_base_offset(rec.guest_id)
        return dp.Shim(base, space.guest.mem.size_bytes, space.guest_root.root_pfn, space.shadow_root.root_pfn)

    def _count(self, n: int) -> None:
        self._record.hw_translations += n

    def _on_trap(self, trap):
        try:
            self._record.trap_shim(trap)
        except Exception as exc:  # noqa: BLE001 - surfaced as the copy's error
            return exc
        return None

    def translate(self, gva: int) -> int:
        self._record.hw_translations += 1
        return resolve_hybrid_with_fixup(gva, self._record.active_hybrid, self._memv.host_mem,
                                         self._record.trap_shim)


class HardwareHasAccess(_BatchMixin):
    """User-memory routines over the activated hybrid address space
    (backend.py:131-174): copies are plain walks of the merged table; maps
    edit the shadow table only."""

    copies = 0
    maps = 0

    def __init__(self, record: GuestProcessRecord, memv: MemoryVirtualizer, log=None):
        self._record = record
        self._memv = memv
        self._log = log
        record.activate_hybrid(memv)
        self._resolver = _HybridResolver(record, memv)

    def _bump(self, n: int = 1) -> None:
        HardwareHasAccess.copies += n

    def _batch_translator(self):
        return self._resolver

    def copy_to_user(self, gva: int, data: bytes) -> int:
        self._bump()
        return copy_user_buffer("to_guest", Gva(gva), len(data), data, translator=self._resolver,
                                host_mem=self._memv.host_mem)

    def copy_from_user(self, gva: int, length: int) -> bytes:
        self._bump()
        buf = bytearray(length)
        copy_user_buffer("from_guest", Gva(gva), length, buf, translator=self._resolver,
                         host_mem=self._memv.host_mem)
        return bytes(buf)

    def map_page(self, gva: int, hpa: int) -> None:
        HardwareHasAccess.maps += 1
        rec = self._record
        space = rec.space
        TableEditor(self._memv.host_mem, space.shadow_root, self._memv.host_alloc.alloc).map(
            gva, hpa >> PAGE_SHIFT, replace=True)
        space.driver_mappings[gva >> PAGE_SHIFT] = hpa >> PAGE_SHIFT
        if self._log is not None:
            self._log.append("map", guest=rec.guest_id, process=rec.pid, gva=hex(gva), hpa=hex(hpa),
                             route="hardware")


class HostNativeAccess:
    """Unmarked context: a native host process whose pages materialise on
    first touch (backend.py:177-216).  Chunks move on the device image."""

    def __init__(self, memv: MemoryVirtualizer):
        self._memv = memv
        self._pages: dict[int, int] = {}

    def _page(self, va: int) -> int:
        page = va >> PAGE_SHIFT
        if page not in self._pages:
            self._pages[page] = self._memv.host_alloc.alloc()
        return self._pages[page]

    def translate(self, va: int) -> int:
        return (self._page(va) << PAGE_SHIFT) | (va & PAGE_MASK)

    def copy_to_user(self, va: int, data: bytes) -> int:
        return copy_user_buffer("to_guest", Gva(va), len(data), data, translator=self,
                                host_mem=self._memv.host_mem)

    def copy_from_user(self, va: int, length: int) -> bytes:
        buf = bytearray(length)
        copy_user_buffer("from_guest", Gva(va), length, buf, translator=self, host_mem=self._memv.host_mem)
        return bytes(buf)

    def map_page(self, va: int, hpa: int) -> None:
        self._pages[va >> PAGE_SHIFT] = hpa >> PAGE_SHIFT
