"""CPU restatement of the reference's hypercall framing -- TEST
INFRASTRUCTURE ONLY (tests and nothing else import it).

Restated from /root/reference/pkg/src/devfsim/hypercall.py:
  pack            hypercall.py:110-137 (_op_words, _pad, pack)
  assemble        hypercall.py:145-175 (FrameAssembler.feed, in order, each
                  error caught; errors leave the pending map unchanged)
  identify        hypercall.py:178-211 (VcpuRegistry.identify)
on plain tuples: an op is (kind, {field: value}), a frame is
(opcode, (6 args), vcpu, cr3).  Pinned to the reference by
tests/test_frames.py over tests/golden/frames.json.
"""

from __future__ import annotations

WORD_MASK = 0xFFFF_FFFF
SLOTS = 6
CONT = 0x7F
PAGE_FAULT = 7
LAYOUT = {
    1: ("device_id", "flags"),
    2: ("handle",),
    3: ("handle", "gva", "length", "offset"),
    4: ("handle", "gva", "length", "offset"),
    5: ("handle", "cmd", "arg_gva", "arg_len", "gva", "flags"),
    6: ("handle", "gva", "length", "prot", "offset", "flags"),
    7: ("handle", "gva", "access", "vma_start", "vma_length", "offset", "flags"),
    8: ("handle", "event_mask", "timeout_ms"),
    9: ("handle", "pid"),
}


def pack(kind: int, values: dict, vcpu: int, cr3: int, tag: int = 0):
    """Frames of one op, or "unpackable"."""
    words = []
    for name in LAYOUT[kind]:
        v = values.get(name, 0)
        if not 0 <= v <= WORD_MASK:
            return "unpackable"
        words.append(v)
    pad = lambda w: tuple(w + [0] * (SLOTS - len(w)))  # noqa: E731
    if kind == PAGE_FAULT:
        t = tag & WORD_MASK
        return [(kind, pad([t] + words[:5]), vcpu, cr3), (CONT, pad([t] + words[5:]), vcpu, cr3)]
    return [(kind, pad(words), vcpu, cr3)]


def assemble(frames, keys, pending=None):
    """Feed frames in order; keys[i] = (guest, process).  Returns the
    per-frame outcomes ((kind, values) | None | "unpackable" | "valueerror")
    and the pending map afterwards."""
    pending = dict(pending or {})
    out = []
    for (opcode, args, _vcpu, _cr3), (g, p) in zip(frames, keys):
        if opcode == CONT:
            head = pending.pop((g, p, args[0]), None)
            if head is None:
                out.append("unpackable")
                continue
            words = list(head[1][1:]) + list(args[1:3])
            out.append((PAGE_FAULT, dict(zip(LAYOUT[PAGE_FAULT], words))))
            continue
        if opcode not in LAYOUT:
            out.append("valueerror")
            continue
        if opcode == PAGE_FAULT:
            key = (g, p, args[0])
            if key in pending:
                out.append("unpackable")
                continue
            pending[key] = (opcode, args)
            out.append(None)
            continue
        out.append((opcode, dict(zip(LAYOUT[opcode], args[:len(LAYOUT[opcode])]))))
    return out, pending


def identify(vcpu_guest: dict, procs: dict, vcpu: int, cr3: int):
    if vcpu not in vcpu_guest:
        return "unknownvcpu"
    g = vcpu_guest[vcpu]
    pid = procs.get((g, cr3))
    return "unknownprocess" if pid is None else (g, pid)
