"""Hypercall framing: the CPU oracle (oracle/frames.py) and this package's
per-frame host API against the reference's recorded outcomes
(tests/golden/frames.json, from tests/golden/gen_golden.py).  CPU only."""

from __future__ import annotations

import scenarios as S
from conftest import load_json
from oracle import frames as OF
from paper_1304_3771_b200 import hypercall as hc


def _oracle_pack_outcomes():
    out = []
    for i, op in enumerate(S.frames_ops(hc)):
        vals = {f: getattr(op, f) for f in hc.ARG_LAYOUT[op.kind]}
        r = OF.pack(int(op.kind), vals, i % 4, 0x40 + (i % 3), (i * 2654435761) & 0x1_FFFF_FFFF)
        out.append(["err", "Unpackable"] if r == "unpackable" else [[o, list(a), v, c] for o, a, v, c in r])
    return out


def _oracle_op(o):
    if o is None:
        return None
    if o == "unpackable":
        return ["err", "Unpackable"]
    if o == "valueerror":
        return ["err", "ValueError"]
    kind, vals = o
    return S.op_outcome(hc.FileOp(kind=hc.FileOpKind(kind), **vals))


def test_oracle_pack_matches_reference():
    assert _oracle_pack_outcomes() == load_json("frames.json")["pack"]


def test_oracle_assemble_matches_reference():
    stream = S.frames_stream(hc)
    got, _ = OF.assemble([(f.opcode, f.args, f.vcpu, f.virtual_cr3) for f, _ in stream], [k for _, k in stream])
    assert [_oracle_op(o) for o in got] == load_json("frames.json")["feed"]


def test_oracle_identify_matches_reference():
    vg = {0: 0, 1: 0, 2: 1, 5: 1}
    procs = {(0, 0x100): 11, (0, 0x200): 12, (1, 0x100): 21, (1, 0x800): 22}
    out = []
    for vcpu in range(7):
        for cr3 in (0x100, 0x200, 0x800, 0x999):
            r = OF.identify(vg, procs, vcpu, cr3)
            out.append(list(r) if isinstance(r, tuple) else
                       ["err", {"unknownvcpu": "UnknownVcpu", "unknownprocess": "UnknownProcess"}[r]])
    assert out == load_json("frames.json")["identify"]


def test_host_api_matches_reference():
    g = load_json("frames.json")
    assert S.frames_pack_query(hc) == g["pack"]
    assert S.frames_feed_query(hc) == g["feed"]
    assert S.frames_identify_query(hc) == g["identify"]
