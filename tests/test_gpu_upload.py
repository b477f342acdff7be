"""pv_upload (include/pv.h): SM-driven host -> device copies of descriptor
arrays, exact for every size and dtype mix, and not queued behind a large
DMA transfer in flight on another stream."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1304_3771_b200 import dataplane as dp

pytestmark = pytest.mark.gpu


def test_to_dev_many_is_exact(cuda):
    rng = np.random.default_rng(4)
    arrays = [rng.integers(-2**62, 2**62, n, dtype=np.int64) for n in (0, 1, 3, 17, 4096, 70_000)]
    arrays += [rng.integers(-2**31, 2**31, n, dtype=np.int32) for n in (1, 5, 1000)]
    arrays.append(rng.integers(0, 2**62, (33, 4), dtype=np.int64))
    arrays.append(rng.integers(0, 2**62, 200_000, dtype=np.int64))  # > 1 MiB: DMA path
    devs = dp._to_dev_many(arrays)
    torch.cuda.synchronize()
    for a, d in zip(arrays, devs):
        assert d.is_cuda and tuple(d.shape) == a.shape
        assert np.array_equal(d.cpu().numpy(), a)


def test_upload_does_not_wait_for_a_big_h2d(cuda):
    big_h = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
    big_d = torch.empty_like(big_h, device="cuda")
    side = torch.cuda.Stream()
    small = np.arange(1024, dtype=np.int64)
    dp._to_dev_many([small])  # warm the pinned-block cache: only the GPU timeline is under test
    torch.cuda.synchronize()
    e0, e_big, e_small = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record()
    side.wait_event(e0)
    with torch.cuda.stream(side):
        big_d.copy_(big_h, non_blocking=True)
        e_big.record(side)
    d, = dp._to_dev_many([small])
    e_small.record()
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), small)
    # ~9 ms of DMA on the link; the upload finishes long before it
    assert e0.elapsed_time(e_small) < 0.5 * e0.elapsed_time(e_big)
