"""Extension geometry (BASELINE config 3): 4-level tables with 2 MiB pages.

No reference semantics exist for it, so parity is "unpinned"
by the reference: the CPU test checks the host table builder and the C
restatement against the closed-form mapping the builder promises; the GPU
tests check the device walker / copier against that restatement.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import status_outcome
from oracle import oracle as O
from paper_1304_3771_b200 import ext4l as X

REGION = 64 << 20


def _expected_frames(vas: np.ndarray, pfn0: int) -> np.ndarray:
    off = (vas - np.uint64(X.C3_VA)).astype(np.int64)
    r = off // X.LARGE
    j = (off % X.LARGE) // 4096
    return np.where(r % 2 == 0, pfn0 + r * 512 + j, pfn0 + r * 512 + 511 - j).astype(np.uint64)


def test_builder_and_oracle_closed_form():
    mem, t = X.build_c3(REGION)
    img = mem.backing.host_for_read()
    vas = np.concatenate([X.c3_sequential(REGION), X.c3_strided(REGION)])
    sp = O.space(0, t.root, 0, 3)
    v, s, _ = O.translate(img, sp, vas, want_pfn=True, threads=0)
    assert (s == 0).all()
    assert np.array_equal(v, _expected_frames(vas, X.C3_NODE_BYTES // 4096))
    # outside the region: faults at the level where the path stops
    v, s, _ = O.translate(img, sp, np.array([X.C3_VA - 4096, X.C3_VA + REGION, 0x1234], np.uint64), threads=0)
    assert [int(x) & 0xFF0 for x in s] == [0x010] * 3


def test_c1_4level_builder_and_oracle_closed_form():
    """BASELINE configs[0] in 4-level geometry: page p of the region (mapped
    k-th in the shuffled order) translates to data frame data0 + k."""
    import random

    mem, t = X.build_c1_4l()
    img = mem.backing.host_for_read()
    order = list(range(16384))
    random.Random(1304).shuffle(order)
    frame_of = np.empty(16384, dtype=np.uint64)
    frame_of[np.array(order)] = X.C1_4L_NODE_BYTES // 4096 + np.arange(16384, dtype=np.uint64)
    vas = X.c1_4l_vas(20_000)
    v, s, _ = O.translate(img, O.space(0, t.root, 0, 3), vas, want_pfn=True, threads=0)
    assert (s == 0).all()
    assert np.array_equal(v, frame_of[((vas - np.uint64(X.C1_4L_VA)) >> np.uint64(12)).astype(np.int64)])
