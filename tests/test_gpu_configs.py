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

import scenarios as S
from oracle import oracle as O
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import has as be
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
    common = ["--steps", "2", "--warmup", "3", "--scale", "8", "--gather", "--no-e2e", "--no-cpu-baseline"]
    one = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "1"] + common, cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    single = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][-1])
    env = dict(os.environ, PV_BENCH_SHARED_DEVICE="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(root, "bench.py"),
           "--gpus", "2"] + [c for c in common if c != "--no-e2e"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 prints exactly one line
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["faulting_lanes"] == 0
    assert line["gather_to_rank0"]["complete"] is True
    # the walk of rank 1 stored its lane words straight into rank 0's buffer (peer mapping), in the timed step
    r0 = line["results_to_rank0"]
    assert isinstance(r0, dict) and r0["verified"] is True and r0["in_timed_region"] is True, r0
    assert line["config"]["sharding"] == "guest g -> rank g mod 2"
    assert line["parity"]["ok"] is True and single["parity"]["ok"] is True
    # every guest's results, returned to rank 0, bit-identical to the one-rank run
    assert line["gather_to_rank0"]["digest"] == single["gather_to_rank0"]["digest"] is not None
    # each rank holds the host-private region + its 4 guests' slots (+ the hole), not the whole world
    cfg = W.C5Config().scaled(8)
    img = line["hbm_image"]
    assert single["hbm_image"]["device_bytes"] == img["image_bytes"]
    owned = cfg.host_private + 4 * cfg.guest_bytes
    assert owned <= img["device_bytes"] <= owned + (256 << 20), img
    assert img["device_bytes"] < 0.6 * img["image_bytes"]
    # end to end at N = 2: both ranks' lane words land in the host buffer rank 0 reads
    e2e = line["e2e"]
    assert e2e["lanes_equal_device_results"] is True and e2e["gather_to_rank0"]["verified"] is True


@pytest.mark.gpu
def test_graph_replayed_step_equals_eager(cuda):
    """bench.py replays its step phases as CUDA graphs: a captured translate
    (large enough for the stage-table pre-pass and its stream-ordered
    scratch) + hybrid copy batch (device trap shim: cooperative kernel, 10 %
    trapping leaves) replayed once must leave exactly what the eager launches
    leave -- lane results, op results and every byte of memory."""

    def world():
        memv, guest, space = W.build_c1("shadow", device=True)
        W.corrupt_c4(memv, space, "shadow")
        rec = be.GuestProcessRecord(S._Guest(0, "shadow"), space, memv)
        acc = be.HardwareHasAccess(rec, memv)
        tr = memv.translator(space, use_cache=False)
        return memv, space, acc, tr

    rng = np.random.default_rng(11)
    vas_h = (W.C1_GVA + rng.integers(0, 64 << 20, 5 << 20)).astype(np.uint32)
    n_ops, op_len = 1024, 16 << 10
    gv = np.uint64(W.C1_GVA) + np.arange(n_ops, dtype=np.uint64) * np.uint64(op_len) + np.uint64(0x40)
    rows = np.stack([gv, np.full(n_ops, op_len - 0x80, np.uint64), np.arange(n_ops, dtype=np.uint64) * np.uint64(op_len),
                     np.zeros(n_ops, np.uint64)], 1)
    src = torch.randint(0, 256, (n_ops * op_len,), dtype=torch.uint8, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(5))
    outs = []
    for graphed in (False, True):
        memv, space, acc, tr = world()
        img = memv.host_mem.backing
        vas = torch.from_numpy(vas_h.view(np.int32)).cuda()
        tplan = dp.TranslatePlan([tr.device_space], [(0, len(vas_h), 0)], image=img)
        cplan = dp.CopyPlan([acc._resolver.device_space], rows, shims=[acc._resolver.device_shim])
        out = (torch.empty(len(vas_h), dtype=torch.int64, device="cuda"),
               torch.empty(len(vas_h), dtype=torch.int32, device="cuda"),
               torch.zeros(len(vas_h), dtype=torch.int64, device="cuda"))
        dp.translate_lanes(img, tplan, vas, out=out)  # leaf index built outside any capture
        dp._shim_scratch(img, cplan.n_pages)
        dp._owner_map(img)
        torch.cuda.synchronize()

        def phase_translate():
            dp.translate_lanes(img, tplan, vas, out=out)

        def phase_copy():
            cplan.shim_written.zero_()
            dp.copy_launch(img, cplan, N.TO_GUEST, src)

        if graphed:
            gs = [torch.cuda.CUDAGraph() for _ in range(2)]
            for g, fn in zip(gs, (phase_translate, phase_copy)):
                with torch.cuda.graph(g):
                    fn()
            out[0].fill_(-1)
            for g in gs:
                g.replay()
        else:
            phase_translate()
            phase_copy()
        img.note_device_write()
        torch.cuda.synchronize()
        outs.append((out[0].cpu().numpy(), out[1].cpu().numpy(), cplan.results.cpu().numpy(),
                     int(cplan.shim_written.item()), _raw(memv)))
    (v0, s0, r0, w0, m0), (v1, s1, r1, w1, m1) = outs
    assert w0 > 0 and w0 == w1  # the shim fixed trapping slots in both
    assert (s0 != 0).any() and np.array_equal(s0, s1) and np.array_equal(v0, v1)
    assert np.array_equal(r0, r1) and np.array_equal(m0, m1)
