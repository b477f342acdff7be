"""PV_OUT_PACKED lane words (include/pv.h): the host decoder on CPU."""

from __future__ import annotations

import numpy as np

from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp


def _pack(status: int, value: int) -> tuple[int, int | None]:
    """The device's pack_lane restated (pv_common.cuh)."""
    if status == 0:
        return value, None
    compact = (status & 0xFFF) | (((status >> 16) & 0x1FF) << 12)
    if value >> 42:
        return N.PACKED_ERR | (compact << 42) | N.PACKED_SPILL_VALUE, value
    return N.PACKED_ERR | (compact << 42) | value, None


def test_unpack_lanes_round_trip():
    rng = np.random.default_rng(5)
    statuses = [0, 0x011, 0x012, 0x013, 0x021, 0x023, 0x041 | (3 << 16), 0x043 | (511 << 16),
                0x062 | (17 << 16), 0x081, 0x0A2]
    vals, sts, words, aux = [], [], [], []
    for _ in range(4000):
        st = int(rng.choice(statuses))
        v = int(rng.integers(0, 1 << 40)) if rng.random() < 0.9 else int(rng.integers(0, 1 << 62)) | (1 << 50)
        if st == 0:
            v &= (1 << 40) - 1
        w, spilled = _pack(st, v)
        vals.append(v)
        sts.append(st)
        words.append(w)
        aux.append(0 if spilled is None else spilled)
    words = np.array(words, dtype=np.uint64)
    aux = np.array(aux, dtype=np.uint64)
    v, s = dp.unpack_lanes(words.view(np.int64), aux.view(np.int64))
    assert np.array_equal(v, np.array(vals, dtype=np.uint64))
    assert np.array_equal(s, np.array(sts, dtype=np.uint32))


def test_unpack_words_decodes_every_form():
    """pv_translate_words lane words (include/pv.h) on CPU: frames, faults
    whose value is the lane's va, and lanes resolved from exception records."""
    rng = np.random.default_rng(6)
    n = 5000
    vas = rng.integers(0, 1 << 32, n).astype(np.uint32)
    frames = rng.integers(0, 1 << 28, n).astype(np.uint64)
    kind = rng.integers(0, 3, n)  # 0 ok, 1 va-valued fault, 2 record
    st = np.where(kind == 0, 0, np.where(kind == 1, 0x013, 0x062 | (17 << 16))).astype(np.uint32)
    compact = (st & 0xFFF) | (((st >> 16) & 0x1FF) << 12)
    words = np.where(kind == 0, frames, np.where(kind == 1, N.W32_ERR | N.W32_VA | compact,
                                                  N.W32_ERR | compact)).astype(np.uint32)
    rec_lanes = np.flatnonzero(kind == 2)
    rec_vals = rng.integers(0, 1 << 62, len(rec_lanes)).astype(np.uint64)
    rec_aux = rng.integers(0, 1 << 40, len(rec_lanes)).astype(np.uint64)
    order = rng.permutation(len(rec_lanes))
    recs = np.zeros((len(rec_lanes), N.EXC_WORDS), np.uint64)
    recs[:, 0] = rec_lanes[order]
    recs[:, 1] = rec_vals[order]
    recs[:, 2] = rec_aux[order]
    recs[:, 3] = st[rec_lanes[order]]
    exc = dp.LaneExceptions.from_records(recs.view(np.int64))
    v, s, a = dp.unpack_words(words.view(np.int32), vas.view(np.int32), exc)
    want = np.where(kind == 0, (frames << np.uint64(12)) | (vas.astype(np.uint64) & np.uint64(0xFFF)),
                    vas.astype(np.uint64))
    want[rec_lanes] = rec_vals
    assert np.array_equal(v, want) and np.array_equal(s, st)
    assert np.array_equal(a[rec_lanes], rec_aux) and not a[kind != 2].any()
    try:
        dp.unpack_words(words, vas, None)
    except ValueError:
        pass
    else:
        raise AssertionError("record lanes without records must not decode")
