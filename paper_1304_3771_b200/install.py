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


def install(devfsim=None):
    """Swap this package into ``devfsim`` (a module or its import name;
    default ``"devfsim"``).  Returns the ``devfsim`` package."""
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
    return devfsim


def installed(devfsim=None) -> bool:
    root = "devfsim" if devfsim is None else getattr(devfsim, "__name__", devfsim)
    return root in _installed
