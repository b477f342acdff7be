"""Physical-memory image: host mirror + HBM copy with page-granular coherence.

The reference keeps host physical memory as one Python ``bytearray`` with
guest memories as windows into it (memvirt.py:124-188, 433-480).  Here the
bytes live twice:

* ``host`` -- a numpy ``uint8`` array (lazily committed by the OS, so a
  64 GiB image costs only the pages actually touched).  The control plane
  (table editors, allocators zeroing frames, result pages, tests) reads and
  writes it byte-exactly like the reference's bytearray.
* ``device`` -- a flat ``torch.uint8`` tensor in HBM that every data-plane
  kernel (translate / copy) reads and writes.

Coherence is page-granular and lazy:

* host writes mark pages in ``_host_dirty``; the next device operation
  scatters exactly those pages into HBM (one H2D copy + ``pv_scatter_pages``);
* kernels that write the image (``to_guest`` copies) set one byte per written
  page in the device-side ``_dev_dirty`` map; the next host access downloads
  the map and gathers exactly those pages back (``pv_gather_pages`` + one D2H).

A timed data-plane loop therefore never synchronises with the host.

Threads (calls on distinct streams are safe): every kernel
launch that writes the image is enqueued under the image lock
(:meth:`MemoryImage.writing`), which also records the writing stream's
last event; :meth:`pull` holds the same lock, waits for every stream and
then gathers, so no device write can slip between reading the dirty map
and clearing it; the leaf index makes its stream wait for other streams'
writes before re-encoding (:meth:`wait_writers`).
"""

from __future__ import annotations

import contextlib
import threading

import numpy as np

from . import _native

PAGE_SIZE = 4096
PAGE_SHIFT = 12

# Move at most this many pages per staging round trip (256 MiB).
_STAGE_PAGES = 65536


def _zeroed_host(nbytes: int) -> np.ndarray:
    """Zero-filled host mirror.  Large images are anonymous MAP_NORESERVE
    mappings: untouched pages cost neither RAM nor commit charge."""
    if nbytes < (1 << 30):
        return np.zeros(nbytes, dtype=np.uint8)
    import mmap

    flags = mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | getattr(mmap, "MAP_NORESERVE", 0x4000)
    mm = mmap.mmap(-1, nbytes, flags=flags, prot=mmap.PROT_READ | mmap.PROT_WRITE)
    return np.frombuffer(mm, dtype=np.uint8)


class MemoryImage:
    """One physical memory (the reference's host ``bytearray``)."""

    def __init__(self, nbytes: int, host: np.ndarray | None = None):
        if nbytes % PAGE_SIZE:
            raise ValueError("memory size must be a multiple of the page size")
        self.nbytes = nbytes
        self.npages = nbytes // PAGE_SIZE
        self.host = _zeroed_host(nbytes) if host is None else host
        self._host_dirty = np.zeros(self.npages, dtype=np.bool_)
        self._host_dirty_any = False
        # pages that may hold non-zero bytes (host or device side); frames
        # that were never written need no work to be zeroed
        self._maybe_nonzero = np.zeros(self.npages, dtype=np.bool_) if host is None else \
            np.ones(self.npages, dtype=np.bool_)
        self._dev = None          # torch.uint8 [nbytes]
        self._dev_key = None      # (_dev, data_ptr, device index) (device_ptr)
        self._dev_dirty = None    # torch.uint8 [npages]
        self._dev_dirty_any = False
        self._pending = np.zeros(self.npages, dtype=np.bool_)  # device-written, not yet gathered
        self._pending_any = False
        self.dev_write_epoch = 0  # bumped by every device write (leaf-index coherence)
        self.host_epoch = 0       # bumped by every push of host writes into HBM
        self.leaf_index = None    # dataplane.LeafIndex, created on first indexed translate
        self._resident = None     # per-page bool mask of the pages held in HBM (None: all)
        self._res_ranges = None   # the resident byte ranges
        self._vmm = None          # pv_image_create handle of a partially resident image
        self.device_bytes = 0     # HBM held by the device image
        self._lock = threading.RLock()
        self._writers: dict = {}  # cuda stream handle -> event after its last image write

    @classmethod
    def adopt(cls, buf) -> "MemoryImage":
        """Wrap an existing bytes-like buffer (its contents are copied)."""
        data = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
        img = cls(len(data), host=data)
        img._host_dirty[:] = True
        img._host_dirty_any = True
        return img

    def __len__(self) -> int:
        return self.nbytes

    # ---- residency (guest-sharded ranks) --------------------
    def set_residency(self, ranges) -> None:
        """Hold only the byte ranges ``[(first, end), ...]`` in HBM (call
        before the first :meth:`device`).  Offsets stay the reference's hpas;
        the rest of the image lives on the host mirror only -- the control
        plane builds it there, and it is never pushed to or pulled from the
        device (pv_image_create backs it with a shared junk hole)."""
        if self._dev is not None:
            raise RuntimeError("residency must be set before the device image exists")
        mask = np.zeros(self.npages, dtype=np.bool_)
        rr = []
        for first, end in ranges:
            first, end = int(first), int(end)
            if not 0 <= first <= end <= self.nbytes or first % PAGE_SIZE or end % PAGE_SIZE:
                raise ValueError(f"bad resident range [{first:#x}, {end:#x})")
            mask[first >> PAGE_SHIFT:end >> PAGE_SHIFT] = True
            rr.append((first, end))
        self._resident = mask
        self._res_ranges = rr

    @property
    def partial(self) -> bool:
        return self._resident is not None

    def resident(self, first: int, end: int) -> bool:
        """Every page of bytes [first, end) is held in HBM."""
        if self._resident is None:
            return True
        if end <= first:
            return True
        return bool(self._resident[first >> PAGE_SHIFT:((end - 1) >> PAGE_SHIFT) + 1].all())

    def _alloc_device(self):
        import ctypes

        import torch

        if self._resident is None:
            self.device_bytes = self.nbytes
            return torch.zeros(self.nbytes, dtype=torch.uint8, device="cuda")
        lib = _native.lib()
        flat = np.asarray([x for r in self._res_ranges for x in r], dtype=np.uint64)
        ptr, handle, held = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        _native.check(lib.pv_image_create(self.nbytes, flat.ctypes.data if len(flat) else None, len(self._res_ranges),
                                          0, ctypes.byref(ptr), ctypes.byref(handle), ctypes.byref(held)),
                      "pv_image_create")
        self._vmm = handle.value
        self.device_bytes = int(held.value)
        dev = torch.cuda.current_device()

        class _Cai:  # zero-copy torch view of the reserved range
            __cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (ptr.value, False),
                                        "version": 3, "strides": None}

        t = torch.as_tensor(_Cai(), device=f"cuda:{dev}")
        assert t.data_ptr() == ptr.value
        return t

    def __del__(self):
        vmm = getattr(self, "_vmm", None)
        if vmm:
            try:
                self._dev = None
                _native.lib().pv_image_destroy(vmm)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass

    # ---- host side --------------------------------------------------------
    # Device writes are pulled back lazily and only where the host looks:
    # a host read / write of bytes [first, end) gathers the device-written
    # pages of that range (``_pending``), so one read_word after a C5 step
    # moves one page, not the 8 GiB the step wrote.
    def host_for_read(self, first: int = 0, end: int | None = None) -> np.ndarray:
        """Host array, current with device writes in bytes [first, end)
        (default: the whole image)."""
        if self._dev_dirty_any or self._pending_any:
            self.pull(first, self.nbytes if end is None else end)
        return self.host

    def host_for_write(self, first: int, end: int) -> np.ndarray:
        """Host array, current in bytes [first, end), after marking them
        dirty (``end <= first``: current everywhere, nothing marked)."""
        if self._dev_dirty_any or self._pending_any:
            if end > first:
                self.pull(first, end)
            else:
                self.pull()
        if end > first:
            span = slice(first >> PAGE_SHIFT, ((end - 1) >> PAGE_SHIFT) + 1)
            self._host_dirty[span] = True
            self._maybe_nonzero[span] = True
            self._host_dirty_any = True
        return self.host

    def host_for_write_pages(self, pages) -> np.ndarray:
        """Host array, current in ``pages``, after marking them dirty."""
        pages = np.asarray(pages, dtype=np.int64)
        if self._dev_dirty_any or self._pending_any:
            self.pull_pages(pages)
        self.mark_host_pages(pages)
        return self.host

    def mark_host_pages(self, pages) -> None:
        self._host_dirty[pages] = True
        self._maybe_nonzero[pages] = True
        self._host_dirty_any = True

    def zero_pages(self, pages: np.ndarray) -> None:
        """Zero whole pages (frame allocation); free for never-written ones.
        A page the device wrote is simply overwritten (never pulled)."""
        pages = np.asarray(pages, dtype=np.int64)
        if self._dev_dirty_any:
            self._collect_pending()
        if self._pending_any:
            dev_written = pages[self._pending[pages]]
            self._pending[dev_written] = False
            self._maybe_nonzero[dev_written] = True
        hot = pages[self._maybe_nonzero[pages]]
        if len(hot):
            self.host.reshape(self.npages, PAGE_SIZE)[hot] = 0
            self._host_dirty[hot] = True
            self._host_dirty_any = True

    # ---- device side ------------------------------------------------------
    @property
    def on_device(self) -> bool:
        return self._dev is not None

    def device(self):
        """The HBM image, current with every host write (allocates lazily)."""
        import torch

        with self._lock:
            if self._dev is None:
                _native.lib()  # fail loudly without a GPU / the library
                self._dev = self._alloc_device()
                self._dev_dirty = torch.zeros(self.npages, dtype=torch.uint8, device="cuda")
            if self._host_dirty_any:
                self.push()
            return self._dev

    def device_ptr(self) -> tuple[int, int]:
        """(data pointer, device index) of the HBM image, current with every
        host write -- the per-call fast path of :meth:`device` (no lock when
        the image is resident and no host write is pending)."""
        d = self._dev
        if d is None or self._host_dirty_any:
            d = self.device()
        k = self._dev_key
        if k is None or k[0] is not d:
            k = self._dev_key = (d, d.data_ptr(), d.device.index)
        return k[1], k[2]

    def dirty_map(self):
        """Device page map that writing kernels set (call after device())."""
        return self._dev_dirty

    def note_device_write(self) -> None:
        import torch

        with self._lock:
            stream = torch.cuda.current_stream()
            if not torch.cuda.is_current_stream_capturing():
                ev = self._writers.get(stream.cuda_stream)
                if ev is None:
                    ev = self._writers[stream.cuda_stream] = torch.cuda.Event()
                ev.record(stream)
            self._dev_dirty_any = True
            self.dev_write_epoch += 1
            _native.busy_streams.add(stream.cuda_stream)  # per-call ops query it before skipping ahead

    @contextlib.contextmanager
    def writing(self):
        """Enqueue image-writing kernels inside this block: it holds the image
        lock (so :meth:`pull` never interleaves with the enqueue) and notes
        the device write after it."""
        with self._lock:
            yield
            self.note_device_write()

    def wait_writers(self) -> None:
        """Make the current stream wait for every other stream's last image
        write (no host synchronisation)."""
        import torch

        if torch.cuda.is_current_stream_capturing():
            return  # a capture starts from a synchronised device (torch.cuda.graph)
        with self._lock:
            stream = torch.cuda.current_stream()
            for handle, ev in self._writers.items():
                if handle != stream.cuda_stream:
                    stream.wait_event(ev)

    def push(self) -> None:
        """Scatter host-dirty pages into HBM."""
        import torch

        with self._lock:
            dirty = self._host_dirty if self._resident is None else (self._host_dirty & self._resident)
            pages = np.flatnonzero(dirty)
            if len(pages) == 0 or self._dev is None:
                self._host_dirty_any = False
                return
            lib = _native.lib()
            stream = torch.cuda.current_stream()
            host2d = self.host.reshape(self.npages, PAGE_SIZE)
            for s in range(0, len(pages), _STAGE_PAGES):
                idx = pages[s:s + _STAGE_PAGES]
                staging = torch.from_numpy(host2d[idx]).pin_memory()
                src = staging.to("cuda", non_blocking=True)
                pfns = torch.from_numpy(idx.astype(np.uint64).view(np.int64)).to("cuda", non_blocking=True)
                _native.check(lib.pv_scatter_pages(self._dev.data_ptr(), self.nbytes, pfns.data_ptr(),
                                                   len(idx), src.data_ptr(), stream.cuda_stream),
                              "pv_scatter_pages")
                if self.leaf_index is not None:
                    self.leaf_index.on_push(idx, self._dev)
                stream.synchronize()  # staging buffers are freed at scope exit
            self._host_dirty[:] = False
            self._host_dirty_any = False
            self.host_epoch += 1

    def _collect_pending(self) -> None:
        """Move the device dirty map into ``_pending`` (host bitmap of pages
        the device wrote and the host has not gathered yet)."""
        import torch

        with self._lock:
            if not self._dev_dirty_any or self._dev is None:
                self._dev_dirty_any = False
                return
            stream = torch.cuda.current_stream()
            # device writes of every stream (other host threads) land first;
            # new ones cannot be enqueued while the lock is held
            torch.cuda.synchronize()
            if self.leaf_index is not None:
                self.leaf_index.sync_device_writes()  # before the dirty map is cleared
            dmap = self._dev_dirty.cpu().numpy().astype(np.bool_)
            if self._resident is not None:
                dmap &= self._resident  # writes that landed in the hole are junk
            self._pending |= dmap
            self._maybe_nonzero |= dmap  # frame zeroing must not skip them (TableBuild.commit)
            self._pending_any = bool(self._pending.any())
            self._dev_dirty.zero_()
            stream.synchronize()
            self._dev_dirty_any = False
            if self.leaf_index is not None:
                self.leaf_index.release_retired()  # every stream drained above

    def pull(self, first: int = 0, end: int | None = None) -> None:
        """Gather the device-written pages of bytes [first, end) (default:
        all) back into the host mirror."""
        end = self.nbytes if end is None else end
        if end <= first:
            return
        with self._lock:
            self._collect_pending()
            if not self._pending_any:
                return
            lo, hi = first >> PAGE_SHIFT, ((end - 1) >> PAGE_SHIFT) + 1
            self._gather(np.flatnonzero(self._pending[lo:hi]) + lo)

    def pull_pages(self, pages) -> None:
        """Gather the device-written pages among ``pages``."""
        with self._lock:
            self._collect_pending()
            if not self._pending_any:
                return
            pages = np.unique(np.asarray(pages, dtype=np.int64))
            self._gather(pages[self._pending[pages]])

    def _gather(self, pages: np.ndarray) -> None:
        import torch

        if len(pages) == 0:
            return
        lib = _native.lib()
        stream = torch.cuda.current_stream()
        host2d = self.host.reshape(self.npages, PAGE_SIZE)
        for s in range(0, len(pages), _STAGE_PAGES):
            idx = pages[s:s + _STAGE_PAGES]
            pfns = torch.from_numpy(idx.astype(np.uint64).view(np.int64)).to("cuda", non_blocking=True)
            dst = torch.empty(len(idx) * PAGE_SIZE, dtype=torch.uint8, device="cuda")
            _native.check(lib.pv_gather_pages(self._dev.data_ptr(), self.nbytes, pfns.data_ptr(), len(idx),
                                              dst.data_ptr(), stream.cuda_stream), "pv_gather_pages")
            host2d[idx] = dst.cpu().numpy().reshape(len(idx), PAGE_SIZE)
            self._maybe_nonzero[idx] = True
        self._pending[pages] = False
        self._pending_any = bool(self._pending.any())

    def sync(self) -> None:
        """Make host and device agree (pull device writes, push host writes)."""
        self.pull()
        if self._dev is not None:
            self.push()
