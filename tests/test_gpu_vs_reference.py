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


@pytest.mark.parametrize("direction", ["to_guest", "from_guest"])
def test_hybrid_batch_with_replaced_shim_matches_sequential_reference(ref, mine, direction):
    """HardwareHasAccess batch whose record's trap_shim is replaced: every trap
    cuts the batch, and no op after the cut may move a byte through the
    pre-shim tables -- here the shim remaps the trapping page onto another
    page's frame and unmaps a page a later op of the same batch uses
    (backend.py:117-128, 288-296; memvirt.py:685-696, 604-628)."""
    rng = random.Random(11)
    n = 24
    gvas = [BUF + rng.randrange(0, 40 * PAGE) for _ in range(n)]
    lengths = [rng.randrange(1, 3 * PAGE) for _ in range(n)]
    gvas[0], lengths[0] = BUF + 3 * PAGE + 40, 2 * PAGE          # traps at page 3
    gvas[1], lengths[1] = BUF + 12 * PAGE + 5, 300               # unmapped by the shim
    gvas[5], lengths[5] = BUF + 10 * PAGE - 8, 64                # traps at page 10
    src = rng.randbytes(sum(lengths))
    results = []
    for impl in (ref, mine):
        memv, space, rec = _world(impl, "shadow", 48, set())
        host = memv.host_mem
        ed = impl.mv.TableEditor(host, space.shadow_root, memv.host_alloc.alloc)
        for k in (3, 10, 20, 33):
            ed.set_leaf_state(BUF + k * PAGE, impl.mv.EntryState.TRAPPING)
        # distinct bytes in every guest page (the from_guest reads see them)
        acc0 = impl.be.SoftwareHasAccess(rec, memv)
        calls = []

        def shim(trap, impl=impl, memv=memv, space=space, calls=calls):
            page_va = trap.va & ~(PAGE - 1)
            calls.append(page_va)
            e = impl.mv.TableEditor(memv.host_mem, space.shadow_root, memv.host_alloc.alloc)
            other = memv.translator(space, use_cache=False).translate(BUF + (40 + len(calls)) * PAGE)
            e.map(page_va, other >> 12, replace=True)
            e.set_leaf_state(BUF + 12 * PAGE, impl.mv.EntryState.NOT_PRESENT)

        for k in range(48):
            if k not in (3, 10, 20, 33):
                acc0.copy_to_user(BUF + k * PAGE, bytes([k + 1]) * PAGE)
        rec.trap_shim = shim
        acc = impl.be.HardwareHasAccess(rec, memv)
        if impl is ref:
            if direction == "to_guest":
                outs, off = [], 0
                for g, ln in zip(gvas, lengths):
                    outs.append(_outcome(lambda g=g, o=off, ln=ln: acc.copy_to_user(g, src[o:o + ln])))
                    off += ln
            else:
                outs = [_outcome(lambda g=g, ln=ln: acc.copy_from_user(g, ln)) for g, ln in zip(gvas, lengths)]
        else:
            if direction == "to_guest":
                res = acc.copy_to_user_batch(gvas, lengths, np.frombuffer(src, dtype=np.uint8))
            else:
                payload, res = acc.copy_from_user_batch(gvas, lengths)
                payload = payload.cpu().numpy().tobytes()
            outs, off = [], 0
            for r, ln in zip(res, lengths):
                if isinstance(r, Exception):
                    fields = {k: getattr(r, k) for k in ("va", "level", "bytes_copied", "node_pfn", "index")
                              if hasattr(r, k)}
                    outs.append((type(r).__name__, fields))
                elif direction == "to_guest":
                    outs.append(("ok", r))
                else:
                    outs.append(("ok", payload[off:off + ln]))
                off += ln
        results.append((outs, calls, _sha(memv), rec.hw_translations))
    r, m = results
    for i, (a, b) in enumerate(zip(r[0], m[0])):
        assert a == b, (i, gvas[i] - BUF, lengths[i], a if len(str(a)) < 200 else str(a)[:200])
    assert r[1:] == m[1:]


# ---- table hazards: copies that write a page-table node the same copy / batch walks --------

def _hazard_world(impl, mode):
    """A process whose gva W (page 20 of the region) maps the guest's own
    leaf table node (TDP: guest tables live in guest memory; shadow: a
    driver map of the shadow leaf node's hpa, HardwareHasAccess.map_page
    style), so a copy into W rewrites the PTEs of the region's pages."""
    memv, space, rec = _world(impl, mode, 40, set())
    W = BUF + 20 * PAGE
    if mode == "tdp":
        gm = space.guest.mem
        root = space.guest_root.root_pfn
        mid = gm.read_word(root, (BUF >> 30) & 3) >> 12
        leaf = gm.read_word(mid, (BUF >> 21) & 0x1FF) >> 12
        words = [gm.read_word(leaf, i) for i in range(512)]
        gm.write_word(leaf, 20, (leaf << 12) | 0x3)
        words[20] = (leaf << 12) | 0x3
    else:
        hm = memv.host_mem
        root = space.shadow_root.root_pfn
        mid = hm.read_word(root, (BUF >> 30) & 3) >> 12
        leaf = hm.read_word(mid, (BUF >> 21) & 0x1FF) >> 12
        words = [hm.read_word(leaf, i) for i in range(512)]
        hm.write_word(leaf, 20, (leaf << 12) | 0x3)
        words[20] = (leaf << 12) | 0x3
    return memv, space, rec, W, words


def _pte_bytes(words, first, last, redirect):
    """Bytes of PTE entries [first, last) with some entries replaced."""
    out = bytearray()
    for i in range(first, last):
        out += int(redirect.get(i, words[i])).to_bytes(8, "little")
    return bytes(out)


@pytest.mark.parametrize("mode,has_mode", [("tdp", "software"), ("shadow", "software"), ("shadow", "hardware")])
@pytest.mark.parametrize("path", ["batch", "small_op", "large_op"])
def test_copy_writing_walked_table_nodes_matches_reference(ref, mine, mode, has_mode, path):
    """A to_guest copy whose chunk lands on a table node that a later page of
    the same op / batch walks: the reference translates page k, writes chunk
    k, then walks page k + 1 through the rewritten table (memvirt.py:604-628).
    Redirects, unmaps and FIFO-cached stale hits are all in play; the device
    detects the hazard (pv_copy_plan_nodes / copy_small) and goes page by page."""
    seed = {"tdp": 1, "shadow": 2}[mode] * 10 + {"software": 1, "hardware": 2}[has_mode] + 100 * len(path)
    results = []
    for impl in (ref, mine):
        rng = random.Random(seed)  # the same script for both implementations
        memv, space, rec, W, words = _hazard_world(impl, mode)
        cls = impl.be.SoftwareHasAccess if has_mode == "software" else impl.be.HardwareHasAccess
        acc = cls(rec, memv)
        redirect = {5: words[9], 7: 0, 21: words[11], 22: words[12], 30: words[3]}
        if path == "batch":
            ops = [(BUF + 5 * PAGE + 10, 64, rng.randbytes(64)),           # cached before the redirect
                   (W + 8 * 5, 8, _pte_bytes(words, 5, 6, redirect)),      # page 5 -> page 9's frame
                   (W + 8 * 7, 8, _pte_bytes(words, 7, 8, redirect)),      # page 7 -> not present
                   (BUF + 5 * PAGE + 100, 200, rng.randbytes(200)),        # hits the FIFO entry (software)
                   (BUF + 7 * PAGE, 300, rng.randbytes(300)),              # faults
                   (BUF + 9 * PAGE + 4000, PAGE, rng.randbytes(PAGE))]
            ops += [(BUF + rng.randrange(0, 19 * PAGE), rng.randrange(1, 2 * PAGE), None) for _ in range(30)]
            ops = [(g, n, d if d is not None else rng.randbytes(n)) for g, n, d in ops]
        elif path == "small_op":   # chunk 0 rewrites entries 21.., chunk 1 is page 21
            data = _pte_bytes(words, 21, 512, redirect) + rng.randbytes(50)
            ops = [(W + 8 * 21, len(data), data)]
        else:                      # > 64 pages: the single-op batch path
            data = _pte_bytes(words, 21, 512, redirect) + rng.randbytes(70 * PAGE)
            ops = [(W + 8 * 21, len(data), data)]
        if impl is ref:
            outs = [_outcome(lambda g=g, d=d: acc.copy_to_user(g, d)) for g, n, d in ops]
        elif path == "batch":
            src = b"".join(d for _, _, d in ops)
            outs = []
            for r in acc.copy_to_user_batch([g for g, _, _ in ops], [n for _, n, _ in ops],
                                            np.frombuffer(src, dtype=np.uint8)):
                if isinstance(r, Exception):
                    outs.append((type(r).__name__, {k: getattr(r, k) for k in
                                                    ("va", "level", "bytes_copied", "node_pfn", "index")
                                                    if hasattr(r, k)}))
                else:
                    outs.append(("ok", r))
        else:
            outs = [_outcome(lambda g=g, d=d: acc.copy_to_user(g, d)) for g, n, d in ops]
        results.append((outs, _sha(memv), rec.translation_cache.entries(), rec.translation_cache.hits,
                        rec.translation_cache.misses, rec.hw_translations))
    r, m = results
    for i, (a, b) in enumerate(zip(r[0], m[0])):
        assert a == b, (i, a, b)
    assert r[1:] == m[1:]
