"""Per-call data plane: one walk or one small copy per launch.

The reference's drivers make one ``ctx.mem.copy_to_user`` call per op and
one ``ProcessTranslator.translate`` call per page (devices.py:148, 254, 316;
backend.py:92-104; memvirt.py:585-628).  A batch pipeline (descriptor
tensors, plan / stamp / exec launches, result copies) costs hundreds of
microseconds per such call; this path costs one kernel launch:

* the request goes to a resident server kernel through a mailbox in
  host-mapped pinned memory (``pv_server_walk`` / ``pv_server_copy_small``,
  include/pv.h): no launch, no H2D copy, no device allocation per call --
  one link round trip there and back (``profiles/r02_percall_latency.json``);
  when the calling thread's stream still has work queued, the same request
  is launched on that stream instead (``pv_walk_one`` / ``pv_copy_small``)
  so the call stays ordered behind it;
* results are published last with a sequence number the library spins on
  (one ctypes call per operation);
* payloads move between the op's pinned staging buffer and HBM inside the
  same kernel (zero-copy over the PCIe/C2C link), so a 4 KiB copy_to_user is
  one request end to end.

``PV_PERCALL_SERVER=0`` launches a kernel per call instead (the A/B form).
Batch launches park the server first (:func:`park`): while resident it holds
a CTA slot of one SM that grids sized to fill every SM count on.

One :class:`PerCall` per host thread (thread-local), so calls from different
threads never share a result block; each call runs on the thread's current
torch stream and is therefore ordered after everything the thread queued on
it before.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native as N

PAGE_SIZE = 4096
PAGE_SHIFT = 12
PAGE_MASK = PAGE_SIZE - 1
SMALL_PAGES = N.SMALL_PAGES
STAGE_BYTES = SMALL_PAGES * PAGE_SIZE

_tls = threading.local()
_SPIN = 20000  # result polls before falling back to a stream synchronisation
_SERVER = os.environ.get("PV_PERCALL_SERVER", "1") != "0"
_server_used = False


def _idle_flag(stream: int) -> int:
    """PV_SERVER_IDLE unless the library queued work on ``stream`` since a
    per-call operation last found it idle; a busy stream is queried once and
    forgotten when it has drained (the query then runs in the library)."""
    if stream not in N.busy_streams:
        return N.SERVER_IDLE
    if N.stream_idle(stream):
        N.busy_streams.discard(stream)
        return N.SERVER_IDLE
    return 0


def park() -> None:
    """Stop the per-call server if it may be resident (before a batch launch).
    Not while the current stream is being captured into a CUDA graph (the stop
    synchronises the server's stream); the server then leaves on its own
    after its idle time."""
    global _server_used
    if _server_used:
        import torch

        if torch.cuda.is_current_stream_capturing():
            return
        _server_used = False
        N.check(N.lib().pv_server_stop(), "pv_server_stop")


class PerCall:
    """Pinned request / result blocks and staging of one host thread."""

    def __init__(self):
        global _raw
        lib = N.lib()
        if _raw is None:
            import torch

            _raw = torch._C._cuda_getCurrentRawStream
        self.lib = lib
        self._blocks = []

        def pinned(nbytes):
            ptr = lib.pv_host_alloc(nbytes)
            if not ptr:
                raise MemoryError("pv_host_alloc failed")
            self._blocks.append(ptr)
            return ptr

        self.one_ptr = pinned(ctypes.sizeof(N.PvOneResult))
        self.one = N.PvOneResult.from_address(self.one_ptr)
        self.small_ptr = pinned(ctypes.sizeof(N.PvSmallResult))
        self.small = N.PvSmallResult.from_address(self.small_ptr)
        self.stage_ptr = pinned(STAGE_BYTES)
        self.stage = np.ctypeslib.as_array((ctypes.c_uint8 * STAGE_BYTES).from_address(self.stage_ptr))
        self.space = N.PvSpace()
        self.space_ref = ctypes.byref(self.space)
        self.op = N.PvSmallOp()
        self.op_ref = ctypes.byref(self.op)
        self.seq = 0
        self._spaces = {}
        self._op_space = None

    def __del__(self):
        lib = getattr(self, "lib", None)
        for ptr in getattr(self, "_blocks", ()):
            try:
                lib.pv_host_free(ptr)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass

    def _wait(self, block, seq, stream) -> None:
        for _ in range(_SPIN):
            if block.seq == seq:
                return
        N.check(self.lib.pv_stream_sync(stream), "pv_stream_sync")
        if block.seq != seq:
            raise RuntimeError("per-call kernel did not publish its result")

    def _space_ref(self, space):
        """byref of a pv_space holding ``space`` (one struct per distinct space, reused)."""
        ref = self._spaces.get(space)
        if ref is None:
            if len(self._spaces) > 4096:
                self._spaces.clear()
            st = N.PvSpace(space.s1_base, space.s1_root_pfn, space.s2_root_pfn, space.mode)
            ref = self._spaces[space] = ctypes.byref(st)
        return ref

    def walk(self, image, space, va: int, out_pfn: bool) -> tuple[int, int, int]:
        """(status, value, aux) of one walk / translation (pv_server_walk, or
        pv_walk_one with PV_PERCALL_SERVER=0)."""
        if _SERVER:
            global _server_used
            _server_used = True
            dev_ptr, dev_index = image.device_ptr()
            stream = _raw(dev_index)
            rc = self.lib.pv_server_walk(dev_ptr, image.nbytes, self._space_ref(space), va & 0xFFFFFFFFFFFFFFFF,
                                         (N.OUT_PFN if out_pfn else 0) | _idle_flag(stream), self.one_ptr, stream)
            if rc:
                N.check(rc, "pv_server_walk")
            one = self.one
            return one.status & 0xFFFFFFFF, one.value, one.aux
        dev = image.device()
        stream = _raw_stream(dev)
        self.seq += 1
        N.check(self.lib.pv_walk_one(dev.data_ptr(), image.nbytes, self._space_ref(space), va & 0xFFFFFFFFFFFFFFFF,
                                     N.OUT_PFN if out_pfn else 0, self.one_ptr, self.seq, stream), "pv_walk_one")
        self._wait(self.one, self.seq, stream)
        one = self.one
        return int(one.status) & 0xFFFFFFFF, int(one.value), int(one.aux)

    def copy(self, image, space, gva: int, length: int, direction: int, buf_off: int, avail: int,
             pre=None) -> N.PvSmallResult:
        """One copy of at most SMALL_PAGES pages between the staging buffer
        (bytes [buf_off, avail)) and the image (pv_copy_small).  ``pre``:
        per-page byte hpas the caller resolved (None = walk on the device).
        Returns the pinned result block (valid until the next call)."""
        dev_ptr, dev_index = image.device_ptr()
        op = self.op
        if self._op_space is not space:  # the pv_space inside the op, refilled when the space changes
            sp = op.space
            sp.s1_base, sp.s1_root_pfn, sp.s2_root_pfn, sp.mode = space.s1_base, space.s1_root_pfn, \
                space.s2_root_pfn, space.mode
            self._op_space = space
        op.gva = gva & 0xFFFFFFFFFFFFFFFF
        op.len = length
        op.direction = direction
        n = 0 if length == 0 else ((gva + length - 1) >> PAGE_SHIFT) - (gva >> PAGE_SHIFT) + 1
        ctypes.memset(ctypes.addressof(op.pre_hpa), 0, 8 * n)
        if pre is not None:
            for k, h in enumerate(pre):
                if h is not None:
                    op.pre_hpa[k] = h + 1
        stream = _raw(dev_index)
        # no device dirty marks: the caller writes the same bytes through to
        # the host mirror (write_through), so no page goes device-stale
        if _SERVER:
            global _server_used
            _server_used = True
            rc = self.lib.pv_server_copy_small(dev_ptr, image.nbytes, self.op_ref, self.stage_ptr + buf_off,
                                               max(avail - buf_off, 0), self.small_ptr, None, _idle_flag(stream),
                                               stream)
            if rc:
                N.check(rc, "pv_server_copy_small")
        else:
            self.seq += 1
            N.check(self.lib.pv_copy_small(dev_ptr, image.nbytes, self.op_ref, self.stage_ptr + buf_off,
                                           max(avail - buf_off, 0), self.small_ptr, None, self.seq,
                                           stream), "pv_copy_small")
            self._wait(self.small, self.seq, stream)
        return self.small


_raw = None


def _raw_stream(dev) -> int:
    """cudaStream_t of the calling thread's current torch stream on the
    image's device (without building a torch Stream object)."""
    global _raw
    if _raw is None:
        import torch

        _raw = torch._C._cuda_getCurrentRawStream
    return _raw(dev.device.index)


def write_through(image, res, gva: int, length: int, n_ok: int, stage: np.ndarray, buf_off: int,
                  avail: int) -> None:
    """Mirror a to_guest small copy's bytes into the host image (the device
    wrote the same bytes into HBM): pages 0 .. n_ok-1 of the op, each chunk
    clamped at the staging bytes available.  Indexed leaf-table pages among
    them are re-encoded (dataplane.LeafIndex)."""
    host = image.host
    pages = []
    for k in range(n_ok):
        cur = gva if k == 0 else ((gva >> PAGE_SHIFT) + k) << PAGE_SHIFT
        done = cur - gva
        chunk = min(length - done, PAGE_SIZE - (cur & PAGE_MASK))
        at = buf_off + done
        m = max(0, min(chunk, avail - at))
        if m == 0:
            continue
        hpa = int(res.page_hpa[k])
        host[hpa:hpa + m] = stage[at:at + m]
        pages.append(hpa >> PAGE_SHIFT)
    if pages:
        idx = np.asarray(pages, dtype=np.int64)
        image._maybe_nonzero[idx] = True
        if image.leaf_index is not None:
            image.leaf_index.on_push(idx, image._dev)


def get() -> PerCall:
    pc = getattr(_tls, "pc", None)
    if pc is None:
        pc = _tls.pc = PerCall()
    return pc
