"""Install seam: run a stock ``devfsim`` on the B200 data plane.

``install(devfsim)`` swaps this package in at the seams the reference itself
uses:

* ``devfsim.memvirt`` -- every class / function the module defines
  (``PhysMem``, ``MemoryVirtualizer``, ``TableEditor``, ``TranslationCache``,
  ``ProcessTranslator``, ``walk``, ``walk_guest``, ``copy_user_buffer``,
  ``HybridTopLevel``, ``resolve_hybrid(_with_fixup)``, the entry codec ...)
  is replaced by :mod:`.memvirt`'s, in ``devfsim.memvirt`` itself and in
  every ``devfsim`` module that imported it by name (``backend.py:52-65``
  imports ``copy_user_buffer`` / ``HybridTopLevel`` / ``TableEditor`` ...,
  ``world.py:15`` ``MemoryVirtualizer``, so ``World.memv`` becomes ours);
* ``devfsim.backend`` -- the ``ctx.mem`` implementations and the process
  record (``SoftwareHasAccess`` / ``HardwareHasAccess`` / ``HostNativeAccess``
  / ``_HybridResolver`` / ``GuestProcessRecord``, backend.py:75-296) are
  replaced by :mod:`.has`'s, so ``Backend.execute_fileop``
  (backend.py:503-539) hands drivers the device-backed access objects;
* exceptions -- this package raises the reference's own classes from then
  on: every ``paper_1304_3771_b200`` module's binding of an exception name
  that ``devfsim.errors`` defines is rebound to the reference class, so the
  reference's handlers catch device faults (``ClassDriver.handle_op``,
  devices.py:423-424: ``PageFault -> ERR_BAD_ADDRESS, (bytes_copied,)``;
  ``Frontend._mmap_retry``, frontend.py:190-193: ``PoolExhausted``).

The swap is by object identity: a ``devfsim`` module attribute is replaced
only when it *is* the reference object being swapped, so unrelated names are
never touched.  Call it before building any ``World``; it is idempotent.
Installing is process-wide (it rebinds module globals) -- run the reference
suite through it in its own process.
"""

from __future__ import annotations

import importlib
import sys
import types

_installed: dict[str, object] = {}

# devfsim.backend names this package provides (backend.py:75-296)
_BACKEND_NAMES = ("SoftwareHasAccess", "_HybridResolver", "HardwareHasAccess", "HostNativeAccess",
                  "GuestProcessRecord")


def _package_modules(prefix: str) -> list[types.ModuleType]:
    return [m for name, m in list(sys.modules.items())
            if m is not None and (name == prefix or name.startswith(prefix + "."))]


def _rebind(modules, mapping: dict[int, object]) -> int:
    """Replace module globals that are (by identity) keys of ``mapping``."""
    n = 0
    for mod in modules:
        d = vars(mod)
        for name, obj in list(d.items()):
            new = mapping.get(id(obj))
            if new is not None and new is not obj:
                d[name] = new
                n += 1
    return n


def _swappable(obj) -> bool:
    return isinstance(obj, type) or isinstance(obj, types.FunctionType)


def warm() -> None:
    """Bring the device path up before its first use: the CUDA context, the
    library's kernels (lazily loaded on first launch), the per-call server
    and the pinned per-call blocks -- about a second of one-time cost that
    would otherwise land inside the first translate / copy_to_user a caller
    times.  A no-op without a CUDA device."""
    import numpy as np
    import torch

    if not torch.cuda.is_available():
        return
    from . import memvirt as mv

    for mode in ("shadow", "tdp"):
        memv = mv.MemoryVirtualizer()
        guest = memv.add_guest(0, mode)
        space = memv.create_process(guest)
        memv.map_region(space, 0x2000_0000, 4)
        for cached in (False, True):
            tr = memv.translator(space, mv.TranslationCache()) if cached else memv.translator(space, use_cache=False)
            tr.translate(0x2000_0010)  # per-call server
            tr.translate_batch(np.arange(0x2000_0000, 0x2000_5000, 0x800, dtype=np.uint64))
            data = bytes(3 * 4096)
            mv.copy_user_buffer("to_guest", 0x2000_0800, len(data), data, translator=tr, host_mem=memv.host_mem)
            back = bytearray(len(data))
            mv.copy_user_buffer("from_guest", 0x2000_0800, len(back), back, translator=tr, host_mem=memv.host_mem)
    torch.cuda.synchronize()


def install(devfsim=None, *, warm_device: bool = True):
    """Swap this package into ``devfsim`` (a module or its import name;
    default ``"devfsim"``).  Returns the ``devfsim`` package.
    ``warm_device``: bring the device path up now (:func:`warm`), so the
    reference's callers never pay the one-time CUDA start-up inside an
    operation they time."""
    if devfsim is None or isinstance(devfsim, str):
        devfsim = importlib.import_module(devfsim or "devfsim")
    root = devfsim.__name__
    if _installed.get(root) is devfsim:
        return devfsim
    ref_errors = importlib.import_module(root + ".errors")
    ref_memvirt = importlib.import_module(root + ".memvirt")
    ref_backend = importlib.import_module(root + ".backend")
    # the rest of the reference package, so every by-name import is rebound now
    for sub in ("world", "frontend", "devices", "guest", "interrupts", "resultpage", "harness", "workloads"):
        try:
            importlib.import_module(f"{root}.{sub}")
        except ImportError:
            pass

    from . import errors as ours_errors
    from . import has as ours_has
    from . import memvirt as ours_memvirt
    # import every module of this package that binds exception names
    from . import dataplane, hypercall, resultpage  # noqa: F401

    pkg = __name__.rsplit(".", 1)[0]

    # 1. exception identity: ours -> the reference's classes
    exc_map = {}
    for name, obj in vars(ours_errors).items():
        ref = getattr(ref_errors, name, None)
        if isinstance(obj, type) and issubclass(obj, BaseException) and isinstance(ref, type):
            exc_map[id(obj)] = ref
    _rebind(_package_modules(pkg), exc_map)

    # 2. memvirt + backend access classes: the reference's objects -> ours
    swap = {}
    for name, ref_obj in vars(ref_memvirt).items():
        if name.startswith("__") or not _swappable(ref_obj):
            continue
        if getattr(ref_obj, "__module__", None) != ref_memvirt.__name__:
            continue  # re-exported names (errors, typing helpers) are not memvirt's own
        mine = getattr(ours_memvirt, name, None)
        if mine is None:
            raise RuntimeError(f"{pkg}.memvirt has no drop-in for {root}.memvirt.{name}")
        swap[id(ref_obj)] = mine
    for name in _BACKEND_NAMES:
        swap[id(getattr(ref_backend, name))] = getattr(ours_has, name)
    _rebind(_package_modules(root), swap)

    _installed[root] = devfsim
    if warm_device:
        warm()
    return devfsim


def installed(devfsim=None) -> bool:
    root = "devfsim" if devfsim is None else getattr(devfsim, "__name__", devfsim)
    return root in _installed
