"""Drop-in forwarding wire format: hypercall frames (hypercall.py of the reference).

A file operation travels from the guest's CVD frontend to the host backend as
frames of one opcode plus exactly six 32-bit argument slots (hypercall.py:
23-137); page_fault takes two frames paired by a tag; the backend identifies
the issuer from the vCPU and the virtual CR3 and reassembles operations
(hypercall.py:145-211).  Same names, fields, errors and results as the
reference for the per-frame calls (``pack``, ``FrameAssembler.feed``,
``VcpuRegistry.identify``), plus batch forms that run on the device
(``pv_frame_pack`` / ``pv_frame_identify`` / ``pv_frame_assemble``,
SURVEY.md 8(f) row 4):

* :func:`pack_batch` -- many operations to one frame array;
* :meth:`FrameAssembler.feed_batch` -- many frames in order, pending first
  frames carried across batches exactly like the per-frame calls;
* :meth:`VcpuRegistry.identify_batch` / :func:`dispatch_batch` -- identify +
  reassemble a frame array, the backend's ``dispatch`` loop (backend.py:
  436-446) without the per-op execution.

Per-frame outcomes of a batch equal the per-frame calls with each error
caught: errors never change the assembler's state in the reference.
"""

from __future__ import annotations

import enum
import threading
from dataclasses import dataclass, fields, replace

import numpy as np

from . import _native as N
from .errors import UnknownProcess, UnknownVcpu, Unpackable

WORD_MASK = 0xFFFF_FFFF
FRAME_SLOTS = 6
MAX_OP_WORDS = 2 * FRAME_SLOTS


class FileOpKind(enum.IntEnum):
    OPEN = 1
    RELEASE = 2
    READ = 3
    WRITE = 4
    IOCTL = 5
    MMAP = 6
    PAGE_FAULT = 7
    POLL = 8
    NOTIFY_SUBSCRIBE = 9


OPCODE_CONTINUATION = 0x7F

ARG_LAYOUT: dict[FileOpKind, tuple[str, ...]] = {  # hypercall.py:46-58
    FileOpKind.OPEN: ("device_id", "flags"),
    FileOpKind.RELEASE: ("handle",),
    FileOpKind.READ: ("handle", "gva", "length", "offset"),
    FileOpKind.WRITE: ("handle", "gva", "length", "offset"),
    FileOpKind.IOCTL: ("handle", "cmd", "arg_gva", "arg_len", "gva", "flags"),
    FileOpKind.MMAP: ("handle", "gva", "length", "prot", "offset", "flags"),
    FileOpKind.POLL: ("handle", "event_mask", "timeout_ms"),
    FileOpKind.NOTIFY_SUBSCRIBE: ("handle", "pid"),
    FileOpKind.PAGE_FAULT: ("handle", "gva", "access", "vma_start", "vma_length", "offset", "flags"),
}

TWO_FRAME_KINDS = frozenset({FileOpKind.PAGE_FAULT})


@dataclass(frozen=True)
class FileOp:
    """One device-file operation; unused fields stay zero (hypercall.py:62-82)."""

    kind: FileOpKind
    device_id: int = 0
    handle: int = 0
    gva: int = 0
    length: int = 0
    offset: int = 0
    flags: int = 0
    cmd: int = 0
    arg_gva: int = 0
    arg_len: int = 0
    prot: int = 0
    event_mask: int = 0
    timeout_ms: int = 0
    pid: int = 0
    access: int = 0
    vma_start: int = 0
    vma_length: int = 0

    def with_fields(self, **kwargs) -> "FileOp":
        return replace(self, **kwargs)


FILEOP_FIELDS = tuple(f.name for f in fields(FileOp) if f.name != "kind")
_FIELD_INDEX = {name: i for i, name in enumerate(FILEOP_FIELDS)}


@dataclass(frozen=True)
class HypercallFrame:
    opcode: int
    args: tuple[int, ...]  # always exactly FRAME_SLOTS wide
    vcpu: int
    virtual_cr3: int

    def __post_init__(self):
        if len(self.args) != FRAME_SLOTS:
            raise Unpackable(f"frame must carry {FRAME_SLOTS} slots, got {len(self.args)}")


@dataclass(frozen=True)
class HypercallResult:
    status: int
    values: tuple[int, ...] = ()


def _op_words(op: FileOp) -> list[int]:
    words = []
    for name in ARG_LAYOUT[op.kind]:
        value = getattr(op, name)
        if not 0 <= value <= WORD_MASK:
            raise Unpackable(f"{name}={value:#x} does not fit a 32-bit slot")
        words.append(value)
    return words


def _pad(words: list[int]) -> tuple[int, ...]:
    return tuple(words + [0] * (FRAME_SLOTS - len(words)))


def pack(op: FileOp, *, vcpu: int, virtual_cr3: int, tag: int = 0) -> list[HypercallFrame]:
    """Frame a file operation: one frame, or two for page_fault
    (hypercall.py:125-137)."""
    words = _op_words(op)
    if op.kind in TWO_FRAME_KINDS:
        head, tail = words[:FRAME_SLOTS - 1], words[FRAME_SLOTS - 1:]
        return [
            HypercallFrame(int(op.kind), _pad([tag & WORD_MASK] + head), vcpu, virtual_cr3),
            HypercallFrame(OPCODE_CONTINUATION, _pad([tag & WORD_MASK] + tail), vcpu, virtual_cr3),
        ]
    if len(words) > FRAME_SLOTS:
        raise Unpackable(f"{op.kind.name} needs {len(words)} slots in one frame")
    return [HypercallFrame(int(op.kind), _pad(words), vcpu, virtual_cr3)]


def unpack_args(kind: FileOpKind, words: list[int]) -> FileOp:
    return FileOp(kind=kind, **dict(zip(ARG_LAYOUT[kind], words)))


# ---- array forms -------------------------------------------------------------------

FRAME_DTYPE = np.dtype([("opcode", "<u4"), ("args", "<u4", (FRAME_SLOTS,)), ("vcpu", "<u4"),
                        ("virtual_cr3", "<u8")])
assert FRAME_DTYPE.itemsize == N.FRAME_BYTES


def ops_to_array(ops) -> np.ndarray:
    """FileOps -> uint64 rows {kind, fields...} (pv.h PV_FOP_WORDS).  A field
    that no uint64 can hold is clamped to 2^64-1 (still unpackable)."""
    out = np.zeros((len(ops), N.FOP_WORDS), dtype=np.uint64)
    for i, op in enumerate(ops):
        out[i, 0] = int(op.kind)
        for j, name in enumerate(FILEOP_FIELDS):
            v = getattr(op, name)
            out[i, 1 + j] = v if 0 <= v < 1 << 64 else (1 << 64) - 1
    return out


def op_from_row(row) -> FileOp:
    kind = FileOpKind(int(row[0]))
    return FileOp(kind=kind, **{name: int(row[1 + _FIELD_INDEX[name]]) for name in ARG_LAYOUT[kind]})


def frames_to_array(frames) -> np.ndarray:
    out = np.zeros(len(frames), dtype=FRAME_DTYPE)
    for i, f in enumerate(frames):
        out[i] = (f.opcode, f.args, f.vcpu, f.virtual_cr3)
    return out


def frame_from_row(r) -> HypercallFrame:
    return HypercallFrame(int(r["opcode"]), tuple(int(a) for a in r["args"]), int(r["vcpu"]), int(r["virtual_cr3"]))


def _dev(arr: np.ndarray):
    from . import dataplane as dp

    return dp._to_dev(np.ascontiguousarray(arr).view(np.uint8))


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _frame_error(status: int, ops_row=None):
    kind = status & 0xFF
    if kind == N.FRAME_UNPACKABLE:
        name = FILEOP_FIELDS[status >> 8]
        value = int(ops_row[1 + (status >> 8)]) if ops_row is not None else 0
        return Unpackable(f"{name}={value:#x} does not fit a 32-bit slot")
    if kind == N.FRAME_ORPHAN:
        return Unpackable("continuation frame without a matching first frame")
    if kind == N.FRAME_DUP_FIRST:
        return Unpackable("second first-frame before continuation")
    if kind == N.FRAME_BAD_KIND:
        return ValueError("not a valid FileOpKind")
    return RuntimeError(f"frame status {status:#x}")


_SCRATCH: dict = {}
_SCRATCH_LOCK = threading.Lock()


def _cached(name: str, nbytes: int):
    """Device scratch reused across calls on the current stream; every
    stream (every host thread issuing on its own stream) has its own."""
    import torch

    key = (name, _stream())
    with _SCRATCH_LOCK:
        t = _SCRATCH.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
            _SCRATCH[key] = t
    return t


def pack_device(ops, vcpu, cr3, tags, *, n_frames: int | None = None):
    """pv_frame_pack over device arrays (ops: int64 [n, PV_FOP_WORDS];
    vcpu / cr3 / tags: int64 [n]).  Returns (frames uint8 [m*40],
    frame_off int64 [n], status int32 [n]) on the device.  ``n_frames``
    (n + the number of page faults) saves a device sync when the caller
    knows it.  Frame slots of ops whose status is not OK are undefined."""
    import torch

    n = ops.shape[0]
    if n_frames is not None and n_frames == n:
        # the caller vouches for one frame per op (no PAGE_FAULT op): frame i is op i's
        frame_off = torch.arange(n, dtype=torch.int64, device="cuda")
    else:
        per = 1 + (ops[:, 0] == int(FileOpKind.PAGE_FAULT)).to(torch.int64)
        frame_off = torch.cumsum(per, 0) - per
    m = n_frames if n_frames is not None else (int(frame_off[-1].item() + per[-1].item()) if n else 0)
    frames = torch.empty(max(m, 1) * N.FRAME_BYTES, dtype=torch.uint8, device="cuda")
    status = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    if n:
        N.check(N.lib().pv_frame_pack(ops.data_ptr(), n, vcpu.data_ptr(), cr3.data_ptr(), tags.data_ptr(),
                                      frame_off.data_ptr(), frames.data_ptr(), status.data_ptr(), _stream()),
                "pv_frame_pack")
    return frames[:m * N.FRAME_BYTES], frame_off, status[:n]


def pack_batch(ops, *, vcpu, virtual_cr3, tags=None):
    """``pack`` for every op on the device.  ``vcpu`` / ``virtual_cr3`` /
    ``tags``: scalars or per-op sequences.  Returns a list whose entry i is
    op i's list of HypercallFrames, or the Unpackable it raises."""
    import torch

    n = len(ops)
    if n == 0:
        return []
    rows = ops_to_array(ops)

    def col(v):
        a = np.broadcast_to(np.asarray(v if v is not None else 0, dtype=np.uint64), (n,)).copy()
        return torch.from_numpy(a.view(np.int64)).cuda()

    frames, off, status = pack_device(torch.from_numpy(rows.view(np.int64)).cuda(), col(vcpu), col(virtual_cr3),
                                      col(None if tags is None else np.asarray(tags, dtype=np.uint64) & WORD_MASK))
    fr = frames.cpu().numpy().view(FRAME_DTYPE)
    off, status = off.cpu().numpy(), status.cpu().numpy().view(np.uint32)
    out = []
    for i in range(n):
        if status[i] != N.FRAME_OK:
            out.append(_frame_error(int(status[i]), rows[i]))
            continue
        k = 2 if rows[i, 0] == int(FileOpKind.PAGE_FAULT) else 1
        out.append([frame_from_row(fr[off[i] + j]) for j in range(k)])
    return out


def assemble_device(frames, record, status):
    """pv_frame_assemble over device arrays (frames uint8 [m*40], record /
    status int32 [m]; status holds the identify outcome).  Returns ops
    int64 [m, PV_FOP_WORDS] (rows of frames whose status is not OK are
    undefined); status is updated in place."""
    import torch

    m = frames.numel() // N.FRAME_BYTES
    ops = torch.empty((max(m, 1), N.FOP_WORDS), dtype=torch.int64, device="cuda")
    if m:
        lib = N.lib()
        nbytes = int(lib.pv_frame_assemble_scratch_bytes(m))
        scratch = _cached("assemble", nbytes)
        N.check(lib.pv_frame_assemble(frames.data_ptr(), m, record.data_ptr(), ops.data_ptr(), status.data_ptr(),
                                      scratch.data_ptr(), nbytes, _stream()), "pv_frame_assemble")
    return ops[:m]


class FrameAssembler:
    """Reassembles operations from frames, pairing continuations
    (hypercall.py:145-175).  ``feed`` is the reference's per-frame call;
    ``feed_batch`` runs many frames on the device with the same state."""

    def __init__(self):
        self._pending: dict[tuple[int, int, int], HypercallFrame] = {}
        self._lock = threading.Lock()

    def feed(self, frame: HypercallFrame, guest: int, process: int) -> FileOp | None:
        with self._lock:
            if frame.opcode == OPCODE_CONTINUATION:
                key = (guest, process, frame.args[0])
                head = self._pending.pop(key, None)
                if head is None:
                    raise Unpackable("continuation frame without a matching first frame")
                kind = FileOpKind(head.opcode)
                n_tail = len(ARG_LAYOUT[kind]) - (FRAME_SLOTS - 1)
                return unpack_args(kind, list(head.args[1:]) + list(frame.args[1:1 + n_tail]))
            kind = FileOpKind(frame.opcode)
            if kind in TWO_FRAME_KINDS:
                key = (guest, process, frame.args[0])
                if key in self._pending:
                    raise Unpackable("second first-frame before continuation")
                self._pending[key] = frame
                return None
            return unpack_args(kind, list(frame.args[:len(ARG_LAYOUT[kind])]))

    def feed_batch(self, frames, guests, processes) -> list:
        """``feed(frames[i], guests[i], processes[i])`` for every i in order,
        on the device.  Entry i of the result is the FileOp, None (a first
        frame now pending) or the exception the call raises."""
        import torch

        frames = list(frames)
        n = len(frames)
        if n == 0:
            return []
        guests = np.broadcast_to(np.asarray(guests, dtype=np.int64), (n,))
        processes = np.broadcast_to(np.asarray(processes, dtype=np.int64), (n,))
        with self._lock:
            carried = list(self._pending.items())
            self._pending = {}
            keys = [(g, p) for (g, p, _), _ in carried] + list(zip(guests.tolist(), processes.tolist()))
            allf = [f for _, f in carried] + frames
            uniq = {k: i for i, k in enumerate(dict.fromkeys(keys))}
            record = np.array([uniq[k] for k in keys], dtype=np.uint32)
            fr = _dev(frames_to_array(allf))
            rec_d = torch.from_numpy(record.view(np.int32)).cuda()
            status = torch.zeros(len(allf), dtype=torch.int32, device="cuda")
            ops = assemble_device(fr, rec_d, status).cpu().numpy().view(np.uint64)
            st = status.cpu().numpy().view(np.uint32)
            out = []
            for i, f in enumerate(allf):
                s = int(st[i])
                if s == N.FRAME_PENDING:
                    g, p = keys[i]
                    self._pending[(g, p, f.args[0])] = f
                if i < len(carried):
                    continue
                if s == N.FRAME_OK:
                    out.append(op_from_row(ops[i]))
                elif s in (N.FRAME_PENDING, N.FRAME_CONSUMED):
                    out.append(None)
                else:
                    out.append(_frame_error(s))
            return out


class VcpuRegistry:
    """The hypervisor's view of vCPUs and process page-table roots
    (hypercall.py:178-211), with a batch form on the device."""

    def __init__(self):
        self._vcpu_guest: dict[int, int] = {}
        self._process_by_cr3: dict[tuple[int, int], int] = {}
        self._lock = threading.Lock()

    def register_vcpu(self, vcpu: int, guest: int) -> None:
        with self._lock:
            self._vcpu_guest[vcpu] = guest

    def register_process(self, guest: int, cr3: int, pid: int) -> None:
        with self._lock:
            self._process_by_cr3[(guest, cr3)] = pid

    def guest_of(self, vcpu: int) -> int:
        with self._lock:
            try:
                return self._vcpu_guest[vcpu]
            except KeyError:
                raise UnknownVcpu(f"vcpu {vcpu} is not registered") from None

    def identify(self, frame: HypercallFrame) -> tuple[int, int]:
        guest = self.guest_of(frame.vcpu)
        with self._lock:
            pid = self._process_by_cr3.get((guest, frame.virtual_cr3))
        if pid is None:
            raise UnknownProcess(f"cr3 {frame.virtual_cr3:#x} matches no process of guest {guest}")
        return guest, pid

    def device_tables(self):
        """(vcpu_guest i32, reg_guest u64, reg_cr3 u64, reg_pid list) for
        pv_frame_identify; the registry sorted by (guest, cr3)."""
        import torch

        with self._lock:
            nv = max(self._vcpu_guest, default=-1) + 1
            vg = np.full(max(nv, 1), -1, dtype=np.int32)
            for v, g in self._vcpu_guest.items():
                vg[v] = g
            reg = sorted(self._process_by_cr3.items())
        rg = np.array([g for (g, _), _ in reg] or [0], dtype=np.uint64)
        rc = np.array([c for (_, c), _ in reg] or [0], dtype=np.uint64)
        return (torch.from_numpy(vg).cuda(), nv, torch.from_numpy(rg.view(np.int64)).cuda(),
                torch.from_numpy(rc.view(np.int64)).cuda(), len(reg), [(g, p) for (g, _), p in reg])

    def identify_device(self, frames, tables=None):
        """pv_frame_identify over a device frame array; returns (record,
        status) int32 device tensors and the record -> (guest, pid) list."""
        import torch

        vg, nv, rg, rc, nreg, recs = tables or self.device_tables()
        m = frames.numel() // N.FRAME_BYTES
        record = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        status = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        if m:
            N.check(N.lib().pv_frame_identify(frames.data_ptr(), m, vg.data_ptr(), nv, rg.data_ptr(), rc.data_ptr(),
                                              nreg, record.data_ptr(), status.data_ptr(), _stream()),
                    "pv_frame_identify")
        return record[:m], status[:m], recs

    def identify_batch(self, frames) -> list:
        """identify() for every frame on the device: (guest, pid) or the
        exception it raises."""
        frames = list(frames)
        if not frames:
            return []
        arr = frames_to_array(frames)
        record, status, recs = self.identify_device(_dev(arr))
        record, status = record.cpu().numpy(), status.cpu().numpy()
        out = []
        for i, f in enumerate(frames):
            if status[i] == N.FRAME_UNKNOWN_VCPU:
                out.append(UnknownVcpu(f"vcpu {f.vcpu} is not registered"))
            elif status[i] == N.FRAME_UNKNOWN_PROCESS:
                g = self._vcpu_guest.get(f.vcpu)
                out.append(UnknownProcess(f"cr3 {f.virtual_cr3:#x} matches no process of guest {g}"))
            else:
                out.append(recs[int(record[i])])
        return out


def identify(frame: HypercallFrame, registry: VcpuRegistry) -> tuple[int, int]:
    return registry.identify(frame)


def dispatch_device(frames, registry: VcpuRegistry, tables=None):
    """The backend's receive loop (backend.py:436-446: identify, then feed)
    for a device frame array with a fresh assembler: returns (ops int64
    [m, PV_FOP_WORDS], status int32 [m], record int32 [m], record list)."""
    record, status, recs = registry.identify_device(frames, tables)
    ops = assemble_device(frames, record, status)
    return ops, status, record, recs
