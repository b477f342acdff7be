"""Pin the CPU oracle (oracle/pvoracle.c) against the reference's own outputs.

The golden fixtures were produced by running the reference (devfsim) on the
scripted scenarios (tests/golden/gen_golden.py); here the C restatement runs
on the same memory images and must give the same outcome for every address.
CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_image, load_json, status_outcome
from oracle import oracle as O


def _walk_outcomes(img, base, root, vas, *, want_pfn, s2=None):
    sp = O.space(base, root, s2 or 0, 2 if s2 is not None else 1)
    v, s, a = O.translate(img, sp, vas, want_pfn=want_pfn, threads=1)
    return [status_outcome(int(s[i]), int(v[i]), int(a[i]), int(vas[i])) for i in range(len(vas))]


@pytest.fixture(scope="module")
def walks():
    meta = load_json("walks.json")
    return load_image("walks"), meta


def test_walks_image_matches_sha(walks):
    import hashlib

    img, meta = walks
    assert hashlib.sha256(img.tobytes()).hexdigest() == meta["image_sha"]


def test_walk_shadow_and_hybrid(walks):
    img, m = walks
    vas = m["vas"]
    e = m["expected"]
    assert _walk_outcomes(img, 0, m["p0_shadow"], vas, want_pfn=True) == e["walk_shadow"]
    assert _walk_outcomes(img, 0, m["p2_shadow"], vas[:40], want_pfn=True) == e["walk_shadow_p2"]
    assert _walk_outcomes(img, 0, m["hroot"], vas, want_pfn=False) == e["hybrid"]


def test_walk_guest_windows(walks):
    img, m = walks
    vas = m["vas"]
    e = m["expected"]
    assert _walk_outcomes(img, m["g0_base"], m["p0_guest"], vas, want_pfn=False) == e["walk_guest0"]
    assert _walk_outcomes(img, m["g1_base"], m["p1_guest"], vas, want_pfn=False) == e["walk_guest1"]


def test_walk_tdp_table(walks):
    img, m = walks
    gpas = [v & 0x3FF_FFFF for v in m["vas"]] + [16 << 20, (16 << 20) - 1, 1 << 33]
    assert _walk_outcomes(img, 0, m["g1_tdp"], gpas, want_pfn=True) == m["expected"]["walk_tdp"]


def test_translate_uncached_shadow_and_tdp(walks):
    img, m = walks
    vas = m["vas"]
    e = m["expected"]
    assert _walk_outcomes(img, 0, m["p0_shadow"], vas, want_pfn=False) == e["translate_p0"]
    assert _walk_outcomes(img, m["g1_base"], m["p1_guest"], vas, want_pfn=False, s2=m["g1_tdp"]) == \
        e["translate_p1"]


def test_translate_cached_fifo(walks):
    img, m = walks
    vas = m["vas"]
    seq = vas[:60] + vas[:60] + [0x2000_0000 + (i % 12) * 4096 + i for i in range(200)]
    for name, sp in (("p0", O.space(0, m["p0_shadow"])), ("p1", O.space(m["g1_base"], m["p1_guest"], m["g1_tdp"], 2))):
        cache = O.new_cache()
        v, s, a = O.translate_cached(img, sp, seq, cache)
        got = [status_outcome(int(s[i]), int(v[i]), int(a[i]), seq[i]) for i in range(len(seq))]
        assert got == m["expected"][f"cached_{name}"]
        entries, hits, misses = O.cache_state(cache)
        hits_e, misses_e, entries_e = m["expected"][f"cached_{name}_state"]
        assert (hits, misses) == (hits_e, misses_e)
        assert [list(e) for e in entries] == entries_e


def test_c01_translation_oracle():
    img = load_image("c01")
    m = load_json("c01.json")
    got = _walk_outcomes(img, m["guest_base"], m["guest_root"], m["samples"], want_pfn=False)
    assert got == m["expected"]


@pytest.mark.parametrize("trial", range(4))
def test_c03_hybrid(trial):
    img = load_image(f"c03_{trial}")
    m = load_json(f"c03_{trial}.json")
    assert _walk_outcomes(img, 0, m["hybrid"], m["vas"], want_pfn=False) == m["expected"]


def test_multithreaded_equals_single():
    img = load_image("c01")
    m = load_json("c01.json")
    sp = O.space(m["guest_base"], m["guest_root"])
    vas = np.array(m["samples"] * 20, dtype=np.uint64)
    one = O.translate(img, sp, vas, threads=1)
    many = O.translate(img, sp, vas, threads=0)
    for a, b in zip(one, many):
        assert np.array_equal(a, b)
