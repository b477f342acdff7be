"""The hypercall frame codec on the device (pv_frame_pack / identify /
assemble) against the reference's recorded outcomes and, at scale, the
CPU oracle (oracle/frames.py)."""

from __future__ import annotations

import random

import numpy as np
import pytest
import torch

import scenarios as S
from conftest import load_json
from oracle import frames as OF
from paper_1304_3771_b200 import _native as N
from paper_1304_3771_b200 import hypercall as hc

pytestmark = pytest.mark.gpu


def _outcome(x):
    if isinstance(x, BaseException):
        return ["err", type(x).__name__]
    return S.op_outcome(x)


def test_pack_batch_matches_reference(cuda):
    ops = S.frames_ops(hc)
    got = hc.pack_batch(ops, vcpu=[i % 4 for i in range(len(ops))],
                        virtual_cr3=[0x40 + (i % 3) for i in range(len(ops))],
                        tags=[(i * 2654435761) & 0x1_FFFF_FFFF for i in range(len(ops))])
    out = [["err", type(r).__name__] if isinstance(r, BaseException) else [S.frame_outcome(f) for f in r]
           for r in got]
    assert out == load_json("frames.json")["pack"]


@pytest.mark.parametrize("n_batches", [1, 3, 17])
def test_feed_batch_matches_reference(cuda, n_batches):
    """The stream fed in batches: first frames pending at a batch end are
    carried into the next batch exactly like per-frame feeding."""
    stream = S.frames_stream(hc)
    asm = hc.FrameAssembler()
    bounds = np.linspace(0, len(stream), n_batches + 1).astype(int)
    out = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        part = stream[a:b]
        out += [_outcome(x) for x in asm.feed_batch([f for f, _ in part], [k[0] for _, k in part],
                                                    [k[1] for _, k in part])]
    assert out == load_json("frames.json")["feed"]
    # the carried state equals the per-frame assembler's
    ref = hc.FrameAssembler()
    for f, (g, p) in stream:
        try:
            ref.feed(f, g, p)
        except Exception:  # noqa: BLE001
            pass
    assert asm._pending == ref._pending


def test_identify_batch_matches_reference(cuda):
    reg = S.frames_registry(hc)
    frames = [hc.HypercallFrame(int(hc.FileOpKind.POLL), (0,) * 6, v, c)
              for v in range(7) for c in (0x100, 0x200, 0x800, 0x999)]
    out = [["err", type(x).__name__] if isinstance(x, BaseException) else list(x) for x in reg.identify_batch(frames)]
    assert out == load_json("frames.json")["identify"]


def test_dispatch_one_million_frames_vs_oracle(cuda):
    """1 M frames from 64 processes of 4 guests (half ioctls, page faults
    split across other traffic, some unknown vCPUs / CR3s): device identify +
    assemble equal the oracle's sequential automaton frame by frame."""
    rng = np.random.default_rng(3)
    n_ops = 700_000
    reg = hc.VcpuRegistry()
    for v in range(8):
        reg.register_vcpu(v, v % 4)
    procs = [(g, 0x1000 * (p + 1), 100 * g + p) for g in range(4) for p in range(16)]
    for g, cr3, pid in procs:
        reg.register_process(g, cr3, pid)
    kinds = rng.choice([5, 5, 5, 3, 4, 7, 8], n_ops)
    src = rng.integers(0, len(procs), n_ops)
    rows = np.zeros((n_ops, N.FOP_WORDS), dtype=np.uint64)
    rows[:, 0] = kinds
    rows[:, 1:] = rng.integers(0, 1 << 32, (n_ops, N.FOP_WORDS - 1), dtype=np.uint64)
    vcpu = np.array([procs[s][0] for s in src], dtype=np.uint64) + 4 * rng.integers(0, 2, n_ops).astype(np.uint64)
    cr3 = np.array([procs[s][1] for s in src], dtype=np.uint64)
    bad = rng.random(n_ops) < 0.001
    cr3[bad] = 0x999
    vcpu[rng.random(n_ops) < 0.001] = 31
    tags = rng.integers(0, 8, n_ops).astype(np.uint64)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()  # noqa: E731
    frames, off, st = hc.pack_device(t(rows), t(vcpu), t(cr3), t(tags))
    assert int((st != 0).sum()) == 0
    # interleave: move every continuation frame a random distance later
    fr = frames.cpu().numpy().view(hc.FRAME_DTYPE).copy()
    order = np.arange(len(fr), dtype=np.float64)
    cont = fr["opcode"] == hc.OPCODE_CONTINUATION
    order[cont] += rng.integers(1, 50, int(cont.sum()))
    fr = fr[np.argsort(order, kind="stable")]
    ops, status, record, recs = hc.dispatch_device(hc._dev(fr), reg)
    ops = ops.cpu().numpy().view(np.uint64)
    status = status.cpu().numpy().view(np.uint32)
    record = record.cpu().numpy()
    # oracle: identify, then feed in order
    vg = {v: v % 4 for v in range(8)}
    pmap = {(g, c): pid for g, c, pid in procs}
    keys, tuples, idmask = [], [], []
    for r in fr:
        idn = OF.identify(vg, pmap, int(r["vcpu"]), int(r["virtual_cr3"]))
        idmask.append(isinstance(idn, tuple))
        keys.append(idn if isinstance(idn, tuple) else None)
    sel = [i for i in range(len(fr)) if idmask[i]]
    got_ok = 0
    exp, _ = OF.assemble([(int(fr[i]["opcode"]), tuple(int(a) for a in fr[i]["args"]), 0, 0) for i in sel],
                         [keys[i] for i in sel])
    exp_at = dict(zip(sel, exp))
    for i in range(len(fr)):
        if not idmask[i]:
            assert status[i] in (N.FRAME_UNKNOWN_VCPU, N.FRAME_UNKNOWN_PROCESS), i
            continue
        assert recs[record[i]] == keys[i], i
        e = exp_at[i]
        if e is None:
            assert status[i] in (N.FRAME_PENDING, N.FRAME_CONSUMED), i
        elif e == "unpackable":
            assert status[i] in (N.FRAME_ORPHAN, N.FRAME_DUP_FIRST), i
        else:
            assert status[i] == N.FRAME_OK, i
            kind, vals = e
            row = ops[i]
            assert int(row[0]) == kind
            assert all(int(row[1 + hc._FIELD_INDEX[k]]) == v for k, v in vals.items()), i
            got_ok += 1
    assert got_ok > n_ops * 0.9
