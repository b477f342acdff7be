"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/gen_golden.py [/root/reference/pkg/src]

It imports the reference's devfsim package read-only, runs the scripted
scenarios of tests/scenarios.py against it and records every outcome plus
sparse snapshots of the memory images.  The committed outputs are what the
CPU tests (oracle + control plane) and the GPU tests (data plane) compare
against.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/
import scenarios as S  # noqa: E402


def load_reference(src: str):
    sys.dont_write_bytecode = True
    sys.path.insert(0, src)
    from devfsim import backend, errors, memvirt  # noqa: E402

    return memvirt, backend, errors


def load_resultpage():
    from devfsim import resultpage  # noqa: E402

    return resultpage


def save_image(name: str, mem, extra: dict, meta: dict) -> None:
    raw = S.image_bytes(mem)
    pages, data = S.sparse_pages(raw)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), pages=pages, data=data,
                        nbytes=np.array([len(raw)], dtype=np.uint64), **extra)
    meta = dict(meta, image_sha=S.sha(raw))
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(meta, f)


def main(src: str) -> None:
    mv, be, er = load_reference(src)

    w = S.spec_build(mv, be, er)
    with open(os.path.join(HERE, "spec.json"), "w") as f:
        json.dump({"expected": S.spec_query(w, mv, be, er),
                   "mem_sha": S.sha(S.image_bytes(w["mem"])), "mem2_sha": S.sha(S.image_bytes(w["mem2"]))}, f)

    w = S.walks_build(mv, be, er)
    memv = w["memv"]
    meta = dict(
        p0_shadow=w["p0"].shadow_root.root_pfn, p0_guest=w["p0"].guest_root.root_pfn,
        p1_guest=w["p1"].guest_root.root_pfn, p2_shadow=w["p2"].shadow_root.root_pfn,
        g0_base=w["g0"].base_hpa, g1_base=w["g1"].base_hpa, g1_tdp=w["g1"].tdp_root.root_pfn,
        hroot=w["hroot"].root_pfn, vas=S.walk_vas(),
    )
    build_raw_sha = S.sha(S.image_bytes(memv.host_mem))
    meta["expected"] = S.walks_query(w, mv, be, er)
    save_image("walks", memv.host_mem, {}, dict(meta, build_sha=build_raw_sha))

    w = S.copies_build(mv, be, er)
    build_sha = S.sha(S.image_bytes(w["memv"].host_mem))
    res = S.copies_query(w, mv, be, er)
    with open(os.path.join(HERE, "copies.json"), "w") as f:
        json.dump({"build_sha": build_sha, "expected": res}, f)

    w = S.c01_build(mv, be, er)
    meta = dict(guest_root=w["space"].guest_root.root_pfn, guest_base=w["guest"].base_hpa,
                samples=w["samples"], expected=S.c01_query(w, mv, be, er))
    save_image("c01", w["memv"].host_mem, {}, meta)

    worlds = S.c03_build(mv, be, er)
    expected = S.c03_query(worlds, mv, be, er)
    for i, (wd, exp) in enumerate(zip(worlds, expected)):
        meta = dict(hybrid=wd["hybrid"].root_pfn, shadow=wd["space"].shadow_root.root_pfn,
                    host_root=wd["host_root"].root_pfn, vas=wd["vas"], expected=exp)
        save_image(f"c03_{i}", wd["memv"].host_mem, {}, meta)

    with open(os.path.join(HERE, "fifo.json"), "w") as f:
        json.dump({"expected": S.fifo_query(mv)}, f)

    for mode in ("shadow", "tdp"):
        w = S.c1_build(mv, be, er, mode)
        memv, space, guest = w["memv"], w["space"], w["guest"]
        vas = S.c1_vas(20000)
        tr = memv.translator(space, use_cache=False)
        expected = [S.outcome(lambda: tr.translate(int(va)), er) for va in vas]
        meta = dict(
            image_sha=S.sha(S.image_bytes(memv.host_mem)),
            shadow_root=space.shadow_root.root_pfn if space.shadow_root else None,
            guest_root=space.guest_root.root_pfn, guest_base=guest.base_hpa,
            tdp_root=guest.tdp_root.root_pfn if guest.tdp_root else None,
            n_vas=len(vas), expected=expected,
        )
        with open(os.path.join(HERE, f"c1_{mode}.json"), "w") as f:
            json.dump(meta, f)
    # BASELINE config 4 tables (corrupted leaves, traps, TDP-stage faults): 100 k VAs per mode,
    # every outcome folded into one digest (the fixture stays small)
    c4 = {}
    for mode in ("shadow", "tdp"):
        w = S.c1_build(mv, be, er, mode)
        S.c4_corrupt(mv, w, mode)
        vas = S.c4_vas()
        tr = w["memv"].translator(w["space"], use_cache=False)
        out = [S.outcome(lambda: tr.translate(int(va)), er) for va in vas]
        kinds = {}
        for o in out:
            kinds[o[0]] = kinds.get(o[0], 0) + 1
        c4[mode] = dict(image_sha=S.sha(S.image_bytes(w["memv"].host_mem)), n_vas=len(vas),
                        digest=S.digest(out), kinds=kinds, head=out[:50])
    with open(os.path.join(HERE, "c4_digest.json"), "w") as f:
        json.dump(c4, f)
    # BASELINE config 2 staging: 20 k overlapping IOCTL_SNAPSHOT blobs through 8 FIFO-cached
    # software-HAS processes of one TDP guest, in program order
    w = S.c2_build(mv, be, er)
    ops = S.c2_ops(20000)
    out, caches = S.c2_reference_run(w, mv, be, er, ops)
    with open(os.path.join(HERE, "c2_digest.json"), "w") as f:
        json.dump(dict(n_ops=len(ops), image_sha=S.sha(S.image_bytes(w["memv"].host_mem)), digest=S.digest(out),
                       head=out[:50], caches=caches), f)
    c1c = {}
    for mode in ("shadow", "tdp"):
        w = S.c1_build(mv, be, er, mode)
        out, cache = S.c1_copy_reference_run(w, mv, be, er, mode)
        c1c[mode] = dict(outcomes=out, cache=cache, image_sha=S.sha(S.image_bytes(w["memv"].host_mem)))
    with open(os.path.join(HERE, "c1_copy_digest.json"), "w") as f:
        json.dump(c1c, f)
    w = S.shim_build(mv, be, er)
    build_sha = S.sha(S.image_bytes(w["memv"].host_mem))
    res = S.shim_query(w, mv, be, er)
    with open(os.path.join(HERE, "shim.json"), "w") as f:
        json.dump(dict(res, build_sha=build_sha, shadow_root=w["p0"].shadow_root.root_pfn,
                       guest_root=w["p0"].guest_root.root_pfn, guest_base=w["g0"].base_hpa,
                       guest_bytes=w["g0"].mem.size_bytes, hybrid_root=w["rec"].active_hybrid.root_pfn), f)
    from devfsim import hypercall as hc  # noqa: E402

    with open(os.path.join(HERE, "frames.json"), "w") as f:
        json.dump({"pack": S.frames_pack_query(hc), "feed": S.frames_feed_query(hc),
                   "identify": S.frames_identify_query(hc)}, f)
    with open(os.path.join(HERE, "resultpage.json"), "w") as f:
        json.dump({"expected": S.resultpage_query(load_resultpage())}, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
