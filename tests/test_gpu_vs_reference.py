"""Differential tests against the live reference (``devfsim`` from baseline/_ref).

The reference is pure Python, so it runs on the GPU box's host beside the
device path: the same worlds are built with ``devfsim.memvirt`` and with this
package, the same randomised op scripts run through both (per-call
``copy_user_buffer`` and the batch API), and every outcome (bytes copied or
the exception with its fields), every cache state and the final host-memory
SHA-256 must agree.  No ``install`` here: the two implementations live side
by side in one process.
"""

from __future__ import annotations

import hashlib
import os
import random
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "devfsim")),
                                 reason="baseline/_ref not staged (run __graft_entry__.build())")]

BUF = 0x2000_0000
PAGE = 4096


@pytest.fixture(scope="module")
def ref():
    if REF not in sys.path:
        sys.path.append(REF)
    import devfsim.backend as rb
    import devfsim.memvirt as rm

    return types.SimpleNamespace(mv=rm, be=rb)


@pytest.fixture(scope="module")
def mine(cuda):
    from paper_1304_3771_b200 import has, memvirt

    return types.SimpleNamespace(mv=memvirt, be=has)


def _world(impl, mode, mapped_pages, holes, host_bytes=64 << 20, guest_bytes=16 << 20):
    memv = impl.mv.MemoryVirtualizer(host_bytes)
    guest = memv.add_guest(0, mode, guest_bytes)
    space = memv.create_process(guest)
    for i in range(mapped_pages):
        if i not in holes:
            memv.map_process_page(space, BUF + i * PAGE)
    rec = impl.be.GuestProcessRecord(types.SimpleNamespace(id=0, mem_mode=mode), space, memv)
    return memv, space, rec


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as exc:  # noqa: BLE001 - compared field by field
        fields = {k: getattr(exc, k) for k in ("va", "level", "bytes_copied", "node_pfn", "index") if hasattr(exc, k)}
        return (type(exc).__name__, fields)


def _sha(memv) -> str:
    return hashlib.sha256(memv.host_mem.read(0, memv.host_mem.size_bytes)).hexdigest()


def _script(seed: int, n_ops: int, span_pages: int):
    rng = random.Random(seed)
    ops = []
    for i in range(n_ops):
        direction = rng.choice(["to_guest", "from_guest"])
        gva = BUF + rng.randrange(0, span_pages * PAGE)
        length = rng.choice([0, 1, 15, 16, 17, rng.randrange(1, 3 * PAGE), PAGE, 2 * PAGE + 3])
        short = rng.random() < 0.3  # host_buf shorter than length
        blen = rng.randrange(0, length + 1) if short else length
        ops.append((direction, gva, length, blen, rng.randbytes(blen)))
    return ops


def _run_script(impl, memv, translator, ops):
    outs = []
    for direction, gva, length, blen, data in ops:
        if direction == "to_guest":
            outs.append(_outcome(lambda: impl.mv.copy_user_buffer(
                "to_guest", gva, length, data, translator=translator, host_mem=memv.host_mem)))
        else:
            buf = bytearray(blen)
            res = _outcome(lambda: impl.mv.copy_user_buffer(
                "from_guest", gva, length, buf, translator=translator, host_mem=memv.host_mem))
            outs.append((res, bytes(buf).hex()))
    return outs


@pytest.mark.parametrize("kind", ["shadow-cached", "tdp-cached", "shadow-uncached", "hybrid"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_copy_user_buffer_scripts_match_reference(ref, mine, kind, seed):
    """Per-call copy_user_buffer over random scripts: short host buffers
    (slice semantics, memvirt.py:624-626), unaligned starts, zero lengths,
    faults on holes and past the mapped region, both directions."""
    mode = "tdp" if kind.startswith("tdp") else "shadow"
    holes = {3, 7}
    ops = _script(seed, 60, 12)
    results = []
    for impl in (ref, mine):
        memv, space, rec = _world(impl, mode, 10, holes)
        if kind == "hybrid":
            rec.activate_hybrid(memv)
            translator = impl.be._HybridResolver(rec, memv)
        elif kind.endswith("uncached"):
            translator = memv.translator(space, use_cache=False)
        else:
            translator = rec.translator
        outs = _run_script(impl, memv, translator, ops)
        results.append((outs, _sha(memv), rec.translation_cache.entries(), rec.translation_cache.hits,
                        rec.translation_cache.misses, rec.hw_translations))
    r, m = results
    for i, (a, b) in enumerate(zip(r[0], m[0])):
        assert a == b, (i, ops[i][:4], a, b)
    assert r[1:] == m[1:]


@pytest.mark.parametrize("has_mode", ["software", "hardware"])
def test_batch_with_short_source_matches_sequential_reference(ref, mine, has_mode):
    """copy_to_user_batch(gvas, lengths, src, offsets) == copy_to_user(gva,
    src[off:off + len]) in order: slices running past src are shorter."""
    rng = random.Random(7)
    src = rng.randbytes(3 * PAGE)
    n = 40
    gvas = [BUF + rng.randrange(0, 9 * PAGE) for _ in range(n)]
    lengths = [rng.randrange(0, 2 * PAGE) for _ in range(n)]
    offsets = [rng.randrange(0, 4 * PAGE) for _ in range(n)]  # some start past the end of src
    results = []
    for impl in (ref, mine):
        memv, space, rec = _world(impl, "shadow", 10, {5})
        cls = impl.be.SoftwareHasAccess if has_mode == "software" else impl.be.HardwareHasAccess
        acc = cls(rec, memv)
        if impl is ref:
            outs = [_outcome(lambda g=g, o=o, ln=ln: acc.copy_to_user(g, src[o:o + ln]))
                    for g, ln, o in zip(gvas, lengths, offsets)]
        else:
            outs = []
            for res in acc.copy_to_user_batch(gvas, lengths, np.frombuffer(src, dtype=np.uint8), offsets):
                if isinstance(res, Exception):
                    fields = {k: getattr(res, k) for k in ("va", "level", "bytes_copied", "node_pfn", "index")
                              if hasattr(res, k)}
                    outs.append((type(res).__name__, fields))
                else:
                    outs.append(("ok", res))
        results.append((outs, _sha(memv), rec.translation_cache.entries(), rec.translation_cache.lookups,
                        rec.hw_translations))
    assert results[0] == results[1]
