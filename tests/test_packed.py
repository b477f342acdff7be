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
