"""GPU parity at the remaining BASELINE configurations (oracle-checked).

* C3, reference-geometry slice: BASELINE config 3 (16 GiB device mmap with
  mixed 4 KiB / 2 MiB pages, 4-level tables) is not expressible in the
  reference (3-level 32-bit VAs, no large pages); its pinned
  part is a 2.5 GiB slice of 4 KiB pages in reference geometry, walked with
  sequential (4 KiB stride) and strided (2 MiB + 4 KiB) batches.
* C5, scaled: all 8 shadow guests x 3 processes of the bench world at 1/16
  size, every rank-sharded guest batch translated and copied exactly as
  bench.py does, compared with the oracle.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import dataplane as dp
from paper_1304_3771_b200 import memvirt as mv
from paper_1304_3771_b200 import shard
from paper_1304_3771_b200 import workloads as W

pytestmark = pytest.mark.gpu

GIB = 1 << 30


def _raw(memv) -> np.ndarray:
    return np.frombuffer(memv.host_mem.read(0, memv.host_mem.size_bytes), dtype=np.uint8).copy()


@pytest.mark.parametrize("mode", ["shadow", "tdp"])
def test_c3_reference_geometry_slice(cuda, mode):
    size = (5 * GIB) // 2
    memv = mv.MemoryVirtualizer(host_bytes=size + (64 << 20))
    guest = memv.add_guest(0, mode, size + (16 << 20))
    sp = memv.create_process(guest)
    base = 0x1000_0000
    pages = size // 4096
    memv.map_region(sp, base, pages)
    tr = memv.translator(sp, use_cache=False)
    seq = (base + np.arange(pages, dtype=np.uint64) * 4096 + 0x123).astype(np.uint64)
    strided = (base + np.arange(0, size, (2 << 20) + 4096, dtype=np.uint64) + 7).astype(np.uint64)
    raw = _raw(memv)
    s = tr.device_space
    osp = O.space(s.s1_base, s.s1_root_pfn, s.s2_root_pfn, s.mode)
    for vas in (seq, strided, np.concatenate([strided, seq[::97] + np.uint64(size)])):
        hv, hs, ha = tr.translate_batch(vas)
        v, st, a = O.translate(raw, osp, vas, threads=0)
        assert np.array_equal(hs, st) and np.array_equal(hv, v) and np.array_equal(ha, a)
    # a 256 MiB sequential copy_from_user across the slice
    n = 256 << 20
    back = bytearray(n)
    assert mv.copy_user_buffer("from_guest", base + 0x80, n, back, translator=tr, host_mem=memv.host_mem) == n
    out = np.zeros(n, np.uint8)
    O.copy(raw, osp.reshape(1, 4), np.array([[base + 0x80, n, 0, 0]], np.uint64), out, 1)
    assert bytes(back) == out.tobytes()


def test_c5_scaled_bench_world_sharded(cuda):
    """The bench's C5 step (translate + hybrid-HAS copy batch) at 1/16 size,
    for the shard of every rank of a 2-rank run, against the oracle."""
    cfg = W.C5Config().scaled(16)
    wd = W.build_c5(cfg)
    memv = wd.memv
    img = memv.host_mem.backing
    for world in (1, 2):
        for rank in range(world):
            owned = shard.owned_guests(cfg.guests, rank, world)
            spaces, bounds, parts, lane = [], [], [], 0
            for g in owned:
                for p, v in enumerate(W.c5_vas(cfg, g)):
                    spaces.append(W.c5_shadow_space(wd, g, p))
                    bounds.append((lane, lane + len(v), len(spaces) - 1))
                    parts.append(v)
                    lane += len(v)
            vas = np.concatenate(parts)
            plan = dp.TranslatePlan(spaces, bounds)
            v, s, _ = dp.translate_lanes(img, plan, torch.from_numpy(vas.view(np.int32)).cuda())
            v = v.cpu().numpy().view(np.uint64)
            s = s.cpu().numpy().view(np.uint32)
            raw = _raw(memv)
            for b, e, si in bounds:
                sp = spaces[si]
                ov, os_, _ = O.translate(raw, O.space(sp.s1_base, sp.s1_root_pfn), vas[b:e].astype(np.uint64),
                                         threads=0)
                assert np.array_equal(v[b:e], ov) and np.array_equal(s[b:e], os_)
            assert (s == 0).all()
    # one copy batch over all guests (hybrid spaces), like the bench step
    c_spaces, rows, off = [], [], 0
    for g in range(cfg.guests):
        for p, ops in enumerate(W.c5_ops(cfg, g)):
            c_spaces.append(W.c5_hybrid_space(wd, g, p))
            offs = off + np.arange(len(ops), dtype=np.uint64) * np.uint64(cfg.op_bytes)
            rows.append(np.stack([ops[:, 0], ops[:, 1], offs, np.full(len(ops), len(c_spaces) - 1, np.uint64)], 1))
            off += int(ops[:, 1].sum())
    rows = np.concatenate(rows)
    src = torch.randint(0, 256, (off,), dtype=torch.uint8, device="cuda")
    raw = _raw(memv)
    outs = dp.copy_ops(img, c_spaces, rows, N.TO_GUEST, src)
    assert all(o.status == 0 for o in outs)
    ospaces = np.stack([O.space(s.s1_base, s.s1_root_pfn) for s in c_spaces])
    O.copy(raw, ospaces, rows, src.cpu().numpy(), 0, threads=0)
    assert np.array_equal(_raw(memv), raw)


@pytest.mark.gpu
def test_bench_two_ranks_one_device(cuda, tmp_path):
    """bench.py's N>1 path (torchrun, guest sharding, barrier, max over
    ranks, per-guest results returned to rank 0) on a one-GPU box: both ranks
    share cuda:0 and talk over gloo (PV_BENCH_SHARED_DEVICE=1)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PV_BENCH_SHARED_DEVICE="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--scale", "8", "--gather", "--no-e2e",
           "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 prints exactly one line
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["faulting_lanes"] == 0
    assert line["gather_to_rank0"]["complete"] is True
    assert line["config"]["sharding"] == "guest g -> rank g mod 2"
