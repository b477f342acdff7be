"""Exception vocabulary of the HAS data plane.

Same class names, base class and fields as the reference's ``errors.py``
(``errors.py:11-133``) so callers can catch either interchangeably by name;
the device path rebuilds these from the per-lane / per-op status words of the
C ABI (``include/pv.h``, PV_ST_*).
"""

from __future__ import annotations


class SimError(Exception):
    """Root of every error raised by this package (errors.py:11-12)."""


class PageFault(SimError):
    """A walk reached a not-present entry (errors.py:15-26).

    ``level``: 1 top, 2 mid, 3 leaf.  ``bytes_copied``: completed prefix of
    a user-buffer copy that stopped at this fault.
    """

    def __init__(self, va: int, level: int, bytes_copied: int = 0):
        self.va = va
        self.level = level
        self.bytes_copied = bytes_copied
        super().__init__(f"page fault at {va:#010x} (level {level})")


class TrapExit(SimError):
    """A walk reached a trapping entry (errors.py:29-37)."""

    def __init__(self, va: int, level: int, node_pfn: int, index: int):
        self.va = va
        self.level = level
        self.node_pfn = node_pfn
        self.index = index
        super().__init__(f"trap exit at {va:#010x} (level {level})")


class TrapFixupFailed(SimError):
    """The shim ran once and the address still traps (errors.py:40-41)."""


class OutOfRange(SimError):
    """An access beyond its memory or memory slot (errors.py:44-45)."""


class PoolExhausted(SimError):
    """A frame allocator or reserved pool ran dry (errors.py:48-49)."""


class AlreadyMapped(SimError):
    """A map request hit a page that is already mapped (errors.py:52-53)."""


class TdpUnsupported(SimError):
    """Hybrid (hardware) HAS requested for a TDP guest (errors.py:56-57)."""


class NativeUnavailable(RuntimeError):
    """The CUDA data plane (libpv.so on a CUDA device) is not available.

    Raised by every data-plane entry point instead of falling back to a CPU
    path: the product has no CPU fallback.
    """


class UnknownVcpu(SimError):
    """Hypercall frame carries a vCPU id not registered to any guest (errors.py:64-65)."""


class Unpackable(SimError):
    """A file operation cannot be framed or a frame sequence is malformed (errors.py:68-69)."""


class UnknownProcess(SimError):
    """A frame's virtual CR3 matches no process of its guest (errors.py:80-81)."""
