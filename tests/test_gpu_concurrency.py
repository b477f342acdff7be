"""Threads on distinct streams (SURVEY.md 8(b) threading).

The reference's dual threads call ``ctx.mem`` concurrently, one per guest
thread (backend.py:316-363), each process with its own record, cache and
translator.  Here two host threads, each on its own CUDA stream, drive two
processes of one world at once -- overlapping to_guest batches (conflict
stamps + ordered last-writer-wins), from_guest batches, translate batches,
hybrid batches through the device trap shim -- and every outcome, cache
state and the final memory must equal the same scripts run one after
another: through the unmodified reference (``baseline/_ref``) where it is
cheap, and through this package on one thread for the large batches.
"""

from __future__ import annotations

import hashlib
import os
import random
import sys
import threading
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu

BUF = 0x2000_0000
PAGE = 4096
ARENA = 48  # mapped pages per process


def _impl(kind):
    if kind == "ref":
        if not os.path.isdir(os.path.join(REF, "devfsim")):
            pytest.skip("baseline/_ref not staged (run __graft_entry__.build())")
        if REF not in sys.path:
            sys.path.append(REF)
        import devfsim.backend as be
        import devfsim.memvirt as mv
    else:
        from paper_1304_3771_b200 import has as be
        from paper_1304_3771_b200 import memvirt as mv
    return types.SimpleNamespace(mv=mv, be=be)


def _world(impl, n_proc: int, traps=()):
    memv = impl.mv.MemoryVirtualizer(64 << 20)
    guest = memv.add_guest(0, "shadow", 24 << 20)
    recs = []
    for _ in range(n_proc):
        space = memv.create_process(guest)
        memv.map_region(space, BUF, ARENA)
        ed = impl.mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
        for k in traps:
            ed.set_leaf_state(BUF + k * PAGE, impl.mv.EntryState.TRAPPING)
        recs.append(impl.be.GuestProcessRecord(types.SimpleNamespace(id=0, mem_mode="shadow"), space, memv))
    return memv, recs


def _script(seed: int, rounds: int, n_ops: int):
    """Per round: a to_guest batch with overlapping destinations (and a few
    ops past the arena: faults), a from_guest batch, a translate batch."""
    rng = random.Random(seed)
    out = []
    for _ in range(rounds):
        gv = [BUF + rng.randrange(0, (ARENA + 2) * PAGE) for _ in range(n_ops)]
        ln = [rng.randrange(1, 2 * PAGE) for _ in range(n_ops)]
        data = rng.randbytes(sum(ln))
        rg = [BUF + rng.randrange(0, (ARENA + 1) * PAGE) for _ in range(n_ops)]
        rl = [rng.randrange(0, PAGE + 100) for _ in range(n_ops)]
        tv = [BUF + rng.randrange(0, (ARENA + 4) * PAGE) for _ in range(4 * n_ops)]
        out.append((gv, ln, data, rg, rl, tv))
    return out


def _exc(e):
    return (type(e).__name__, {k: getattr(e, k) for k in ("va", "level", "bytes_copied", "node_pfn", "index")
                               if hasattr(e, k)})


def _run_ref(impl, memv, rec, acc, script):
    """The script as the reference runs it: one call per op, in order."""
    log = []
    tr = memv.translator(rec.space, use_cache=False)
    for gv, ln, data, rg, rl, tv in script:
        off = 0
        for g, n in zip(gv, ln):
            try:
                log.append(("w", acc.copy_to_user(g, data[off:off + n])))
            except Exception as e:  # noqa: BLE001
                log.append(("w", _exc(e)))
            off += n
        for g, n in zip(rg, rl):
            try:
                log.append(("r", acc.copy_from_user(g, n)))
            except Exception as e:  # noqa: BLE001
                log.append(("r", _exc(e)))
        for v in tv:
            try:
                log.append(("t", tr.translate(v)))
            except Exception as e:  # noqa: BLE001
                log.append(("t", _exc(e)))
    return log


def _run_mine(memv, rec, acc, script, stream=None):
    """The same script through the batch API, on ``stream``."""
    import torch

    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import dataplane as dp

    log = []
    tr = memv.translator(rec.space, use_cache=False)
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        for gv, ln, data, rg, rl, tv in script:
            for r in acc.copy_to_user_batch(gv, ln, np.frombuffer(data, dtype=np.uint8)):
                log.append(("w", _exc(r) if isinstance(r, Exception) else r))
            payload, res = acc.copy_from_user_batch(rg, rl)
            payload = payload.cpu().numpy().tobytes()
            off = 0
            for r, n in zip(res, rl):
                log.append(("r", _exc(r) if isinstance(r, Exception) else payload[off:off + n]))
                off += n
            hpa, st, aux = tr.translate_batch(np.asarray(tv, dtype=np.uint64))
            for v, h, s, a in zip(tv, hpa.tolist(), st.tolist(), aux.tolist()):
                if s == N.ST_OK:
                    log.append(("t", h))
                else:
                    try:
                        dp.raise_for(s, h, a, v, memv.host_mem.size_bytes)
                    except Exception as e:  # noqa: BLE001
                        log.append(("t", _exc(e)))
        torch.cuda.current_stream().synchronize()
    return log


def _state(memv, recs):
    return (hashlib.sha256(memv.host_mem.read(0, memv.host_mem.size_bytes)).hexdigest(),
            [(r.translation_cache.entries(), r.translation_cache.hits, r.translation_cache.misses,
              r.hw_translations) for r in recs])


def _threads(fns):
    errs = []
    outs = [None] * len(fns)
    start = threading.Barrier(len(fns))

    def run(i):
        try:
            start.wait()
            outs[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return outs


@pytest.mark.parametrize("has_mode", ["software", "hardware"])
def test_two_threads_two_streams_match_sequential_reference(cuda, has_mode):
    """Two processes' scripts on two threads / two streams at once == the
    reference running them one after the other (per-process order is all
    the reference guarantees; the processes' destinations are disjoint)."""
    import torch

    traps = (5, 9, 30) if has_mode == "hardware" else ()
    scripts = [_script(100 + p, rounds=6, n_ops=40) for p in range(2)]
    ref, mine = _impl("ref"), _impl("mine")

    memv, recs = _world(ref, 2, traps)
    cls = ref.be.SoftwareHasAccess if has_mode == "software" else ref.be.HardwareHasAccess
    expect = [_run_ref(ref, memv, r, cls(r, memv), sc) for r, sc in zip(recs, scripts)]
    expect_state = _state(memv, recs)

    for attempt in range(3):  # a few interleavings
        memv, recs = _world(mine, 2, traps)
        cls = mine.be.SoftwareHasAccess if has_mode == "software" else mine.be.HardwareHasAccess
        accs = [cls(r, memv) for r in recs]
        streams = [torch.cuda.Stream() for _ in recs]
        got = _threads([lambda i=i: _run_mine(memv, recs[i], accs[i], scripts[i], streams[i]) for i in range(2)])
        torch.cuda.synchronize()
        for p in range(2):
            for j, (a, b) in enumerate(zip(expect[p], got[p])):
                assert a == b, (attempt, p, j, str(a)[:200], str(b)[:200])
            assert len(expect[p]) == len(got[p])
        assert _state(memv, recs) == expect_state, attempt


def test_four_threads_large_overlapping_batches_match_one_thread(cuda):
    """Four processes, 2048-op overlapping to_guest batches (ordered apply,
    per-stream conflict stamps) + from_guest batches, four threads / four
    streams at once == the same four scripts on one thread in sequence."""
    import torch

    mine = _impl("mine")
    scripts = [_script(900 + p, rounds=3, n_ops=2048) for p in range(4)]
    memv, recs = _world(mine, 4)
    accs = [mine.be.SoftwareHasAccess(r, memv) for r in recs]
    seq = [_run_mine(memv, r, a, sc) for r, a, sc in zip(recs, accs, scripts)]
    seq_state = _state(memv, recs)

    memv, recs = _world(mine, 4)
    accs = [mine.be.SoftwareHasAccess(r, memv) for r in recs]
    streams = [torch.cuda.Stream() for _ in recs]
    got = _threads([lambda i=i: _run_mine(memv, recs[i], accs[i], scripts[i], streams[i]) for i in range(4)])
    torch.cuda.synchronize()
    for p in range(4):
        assert got[p] == seq[p], p
    assert _state(memv, recs) == seq_state


@pytest.mark.parametrize("has_mode", ["software", "hardware"])
def test_per_call_threads_match_sequential_reference(cuda, has_mode):
    """Three threads making the reference's one-call-per-op calls at once
    (each through the per-call server, each on its own stream), while a
    fourth runs batches on another process: every per-call outcome, the
    caches and the final memory equal the reference run one after another."""
    import torch

    traps = (5, 9, 30) if has_mode == "hardware" else ()
    scripts = [_script(300 + p, rounds=2, n_ops=24) for p in range(4)]
    ref, mine = _impl("ref"), _impl("mine")

    memv, recs = _world(ref, 4, traps)
    cls = ref.be.SoftwareHasAccess if has_mode == "software" else ref.be.HardwareHasAccess
    expect = [_run_ref(ref, memv, r, cls(r, memv), sc) for r, sc in zip(recs, scripts)]
    expect_state = _state(memv, recs)

    memv, recs = _world(mine, 4, traps)
    cls = mine.be.SoftwareHasAccess if has_mode == "software" else mine.be.HardwareHasAccess
    accs = [cls(r, memv) for r in recs]
    streams = [torch.cuda.Stream() for _ in recs]

    def per_call(i):
        with torch.cuda.stream(streams[i]):
            return _run_ref(mine, memv, recs[i], accs[i], scripts[i])

    fns = [lambda i=i: per_call(i) for i in range(3)]
    fns.append(lambda: _run_mine(memv, recs[3], accs[3], scripts[3], streams[3]))
    got = _threads(fns)
    torch.cuda.synchronize()
    for p in range(4):
        assert len(expect[p]) == len(got[p])
        for j, (a, b) in enumerate(zip(expect[p], got[p])):
            assert a == b, (p, j, str(a)[:200], str(b)[:200])
    assert _state(memv, recs) == expect_state
