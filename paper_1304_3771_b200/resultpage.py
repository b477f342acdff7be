"""Drop-in ``resultpage`` plus batched device forms.

The record layout is the reference's (resultpage.py:1-16): little endian
``status u32, flags u32 (bit 0: staged), values 6 x u32, blob_len u32``
(36 bytes) then up to 4060 bytes of inline blob.  :func:`encode` /
:func:`decode` are the per-record host codecs with the reference's
signatures; :func:`encode_batch` / :func:`decode_batch` write / read a batch
of records in the HBM image in one launch each (``pv_result_encode`` /
``pv_result_decode``), and :func:`deliver_batch` is the guest side's
``guest_write`` of inline blobs (frontend.py:166-169, 203-210) as one copy
batch through uncached translators.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import dataplane as dp
from .errors import OutOfRange, PageFault
from .memvirt import PAGE_SIZE

_LAYOUT = struct.Struct("<II6II")
HEADER_BYTES = _LAYOUT.size  # 36
BLOB_CAPACITY = PAGE_SIZE - HEADER_BYTES
FLAG_STAGED = 0x1


@dataclass(frozen=True)
class ResultRecord:
    status: int
    values: tuple[int, ...]
    blob: bytes | None
    staged: bool

    @property
    def total_bytes(self) -> int:
        return HEADER_BYTES + (len(self.blob) if self.blob else 0)


def _six(values) -> tuple[int, ...]:
    v = tuple(values)[:6]
    return v + (0,) * (6 - len(v))


def encode(status: int, values: tuple[int, ...], blob: bytes | None = None, staged: bool = False) -> bytes:
    """One record (resultpage.py:44-51)."""
    if blob is not None and len(blob) > BLOB_CAPACITY:
        raise ValueError("inline blob exceeds the result page")
    return _LAYOUT.pack(status, FLAG_STAGED if staged else 0, *_six(values), len(blob) if blob else 0) + (blob or b"")


def decode(page: bytes) -> ResultRecord:
    """One record (resultpage.py:54-61): a staged record carries no blob."""
    status, flags, *rest = _LAYOUT.unpack_from(page, 0)
    values, n = tuple(rest[:6]), rest[6]
    staged = bool(flags & FLAG_STAGED)
    blob = bytes(page[HEADER_BYTES:HEADER_BYTES + n]) if n and not staged else None
    return ResultRecord(status, values, blob, staged)


def _headers(records) -> np.ndarray:
    h = np.zeros((len(records), 9), dtype=np.uint32)
    for i, (status, values, blob, staged) in enumerate(records):
        h[i, 0] = status & 0xFFFFFFFF
        h[i, 1] = FLAG_STAGED if staged else 0
        h[i, 2:8] = _six(values)
        h[i, 8] = len(blob) if blob else 0
    return h


def encode_batch(host_mem, page_hpas, records) -> list[Exception | None]:
    """Write ``records[i] = (status, values, blob, staged)`` at
    ``page_hpas[i]`` of ``host_mem`` on the device (one launch).  Returns
    per-record errors (OutOfRange / ValueError) or None."""
    import torch

    hpas = np.asarray(page_hpas, dtype=np.uint64)
    if len(np.unique(hpas >> np.uint64(12))) != len(hpas):
        raise ValueError("one record per result page per batch")
    n = len(records)
    if n == 0:
        return []
    image = host_mem.backing
    lib = N.lib()
    dev = image.device()
    blobs = [r[2] or b"" for r in records]
    offs = np.zeros(n, dtype=np.uint64)
    if n > 1:
        np.cumsum([len(b) for b in blobs[:-1]], out=offs[1:])
    payload = np.frombuffer(b"".join(blobs) or b"\0", dtype=np.uint8)
    buf = dp._to_dev(payload)
    hdr = dp._to_dev(_headers(records).view(np.int32))
    hp = dp._to_dev((hpas + np.uint64(host_mem.base)).view(np.int64))
    of = dp._to_dev(offs.view(np.int64))
    status = torch.empty(n, dtype=torch.int32, device="cuda")
    with image.writing():
        N.check(lib.pv_result_encode(dev.data_ptr(), image.nbytes, hp.data_ptr(), hdr.data_ptr(), buf.data_ptr(),
                                     of.data_ptr(), n, status.data_ptr(), image.dirty_map().data_ptr(),
                                     dp._stream().cuda_stream), "pv_result_encode")
    out = []
    for i, st in enumerate(status.cpu().numpy().view(np.uint32).tolist()):
        if st == N.ST_OK:
            out.append(None)
        elif st == N.ST_CONFLICT:
            out.append(ValueError("inline blob exceeds the result page"))
        else:
            out.append(OutOfRange(f"access [{int(hpas[i]):#x}, +{HEADER_BYTES + len(blobs[i])}) beyond "
                                  f"{host_mem.size_bytes:#x}"))
    return out


def decode_headers(host_mem, page_hpas):
    """Device decode of the record headers: (header[n, 9] uint32, ok[n])."""
    import torch

    hpas = np.asarray(page_hpas, dtype=np.uint64)
    n = len(hpas)
    image = host_mem.backing
    lib = N.lib()
    dev = image.device()
    hp = dp._to_dev((hpas + np.uint64(host_mem.base)).view(np.int64))
    hdr = torch.zeros((max(n, 1), 9), dtype=torch.int32, device="cuda")
    status = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    N.check(lib.pv_result_decode(dev.data_ptr(), image.nbytes, hp.data_ptr(), n, hdr.data_ptr(), status.data_ptr(),
                                 dp._stream().cuda_stream), "pv_result_decode")
    return hdr.cpu().numpy().view(np.uint32)[:n], status.cpu().numpy()[:n] == 0


def decode_batch(host_mem, page_hpas) -> list[ResultRecord]:
    """Records at ``page_hpas`` (headers decoded on the device; inline blobs
    read back for the records that carry one)."""
    hdr, ok = decode_headers(host_mem, page_hpas)
    out = []
    for i, hpa in enumerate(np.asarray(page_hpas, dtype=np.uint64).tolist()):
        if not ok[i]:
            raise OutOfRange(f"result page {hpa:#x} beyond {host_mem.size_bytes:#x}")
        status, flags, n = int(hdr[i, 0]), int(hdr[i, 1]), int(hdr[i, 8])
        staged = bool(flags & FLAG_STAGED)
        blob = host_mem.read(hpa + HEADER_BYTES, n) if n and not staged else None
        out.append(ResultRecord(status, tuple(int(v) for v in hdr[i, 2:8]), blob, staged))
    return out


def deliver_batch(memv, spaces, page_hpas, arg_gvas) -> list[Exception | None]:
    """Guest-side delivery of inline blobs (frontend.py:166-169): for each
    record with an inline blob and a non-zero ``arg_gvas[i]``, the
    ``guest_write`` of the blob through an uncached translator of
    ``spaces[i]`` -- one device copy batch sourced from the result pages in
    the image.  guest_write does not annotate bytes_copied, so a PageFault
    keeps bytes_copied = 0 (pages before it are written, as in the
    reference)."""
    hdr, ok = decode_headers(memv.host_mem, page_hpas)
    hpas = np.asarray(page_hpas, dtype=np.uint64)
    rows, idx, uniq = [], [], {}
    tr_spaces = []
    for i, (sp, gva) in enumerate(zip(spaces, arg_gvas)):
        n = int(hdr[i, 8])
        if not ok[i] or gva == 0 or n == 0 or (int(hdr[i, 1]) & FLAG_STAGED):
            continue
        space = memv.translator(sp, use_cache=False).device_space
        if space not in uniq:
            uniq[space] = len(tr_spaces)
            tr_spaces.append(space)
        rows.append((gva, n, int(hpas[i]) + memv.host_mem.base + HEADER_BYTES, uniq[space]))
        idx.append(i)
    result: list[Exception | None] = [None] * len(hpas)
    if not rows:
        return result
    image = memv.host_mem.backing
    outs = dp.copy_ops(image, tr_spaces, np.array(rows, dtype=np.uint64), N.TO_GUEST, image.device())
    for i, row, o in zip(idx, rows, outs):
        if o.status == N.ST_OK:
            continue
        try:
            dp.raise_for(o.status, o.value, o.aux, row[0] + o.copied, image.nbytes)
        except PageFault as f:
            f.bytes_copied = 0
            result[i] = f
        except Exception as e:  # noqa: BLE001
            result[i] = e
    return result
