"""ctypes wrapper of oracle/_build/liboracle.so (TEST INFRASTRUCTURE ONLY).

The C file restates the reference's walk / translate / FIFO cache /
copy_user_buffer (see the citations in pvoracle.c); this module adapts numpy
arrays to it.  Built by ``make -C oracle`` (also done by
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

_p = ctypes.c_void_p
_u64 = ctypes.c_uint64
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(os.path.join(HERE, "pvoracle.c")):
            build()
        l = ctypes.CDLL(LIB)
        l.orc_walk.restype = ctypes.c_uint32
        l.orc_walk.argtypes = [_p, _u64, _u64, _u64, _u64, ctypes.c_int, _p]
        l.orc_translate1.restype = ctypes.c_uint32
        l.orc_translate1.argtypes = [_p, _u64, _p, _u64, ctypes.c_int, _p, _p]
        l.orc_translate.restype = None
        l.orc_translate.argtypes = [_p, _u64, _p, _p, _u64, ctypes.c_int, _p, _p, _p, ctypes.c_int]
        l.orc_translate_cached.restype = None
        l.orc_translate_cached.argtypes = [_p, _u64, _p, _p, _u64, _p, _p, _p, _p]
        l.orc_copy.restype = None
        l.orc_copy.argtypes = [_p, _u64, _p, _p, _u64, _p, ctypes.c_int, _p, _p, _p, ctypes.c_int]
        l.orc_copy_hybrid.restype = _u64
        l.orc_copy_hybrid.argtypes = [_p, _u64, _p, _p, _p, _u64, _p, ctypes.c_int, _p, _p]
        _lib = l
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def space(s1_base: int, s1_root: int, s2_root: int = 0, mode: int = 1) -> np.ndarray:
    return np.array([s1_base, s1_root, s2_root, mode], dtype=np.uint64)


def translate(img: np.ndarray, sp: np.ndarray, vas, *, want_pfn: bool = False, threads: int = 0):
    """Uncached batch translation: (value u64, status u32, aux u64)."""
    vas = np.ascontiguousarray(vas, dtype=np.uint64)
    n = len(vas)
    value = np.zeros(n, np.uint64)
    status = np.zeros(n, np.uint32)
    aux = np.zeros(n, np.uint64)
    lib().orc_translate(_ptr(img), img.nbytes, _ptr(sp), _ptr(vas), n, int(want_pfn), _ptr(value), _ptr(status),
                        _ptr(aux), threads)
    return value, status, aux


def new_cache(capacity: int = 10, entries=(), hits: int = 0, misses: int = 0) -> np.ndarray:
    c = np.zeros(68, np.uint64)
    for j, (k, v) in enumerate(entries):
        c[j] = k
        c[32 + j] = v
    c[64] = hits
    c[65] = misses
    c[66] = capacity | (len(entries) << 32)
    return c


def cache_state(c: np.ndarray):
    cap = int(c[66]) & 0xFFFFFFFF
    n = int(c[66]) >> 32
    head = int(c[67]) & 0xFFFFFFFF
    entries = [(int(c[(head + j) % cap]), int(c[32 + (head + j) % cap])) for j in range(n)]
    return entries, int(c[64]), int(c[65])


def translate_cached(img: np.ndarray, sp: np.ndarray, vas, cache: np.ndarray):
    vas = np.ascontiguousarray(vas, dtype=np.uint64)
    n = len(vas)
    value = np.zeros(n, np.uint64)
    status = np.zeros(n, np.uint32)
    aux = np.zeros(n, np.uint64)
    lib().orc_translate_cached(_ptr(img), img.nbytes, _ptr(sp), _ptr(vas), n, _ptr(cache), _ptr(value),
                               _ptr(status), _ptr(aux))
    return value, status, aux


def copy(img: np.ndarray, spaces: np.ndarray, ops: np.ndarray, buf: np.ndarray, direction: int, *, caches=None,
         op_cache=None, threads: int = 1) -> np.ndarray:
    """Run copy ops in order on ``img`` (modified in place for to_guest);
    returns result rows (copied, value, aux, status | fail_page << 32)."""
    spaces = np.ascontiguousarray(spaces, dtype=np.uint64).reshape(-1, 4)
    ops = np.ascontiguousarray(ops, dtype=np.uint64).reshape(-1, 4)
    res = np.zeros((len(ops), 4), np.uint64)
    cptr = _ptr(caches) if caches is not None else None
    optr = _ptr(np.ascontiguousarray(op_cache, dtype=np.int32)) if op_cache is not None else None
    if op_cache is not None:
        op_cache = np.ascontiguousarray(op_cache, dtype=np.int32)
        optr = _ptr(op_cache)
    lib().orc_copy(_ptr(img), img.nbytes, _ptr(spaces), _ptr(ops), len(ops), _ptr(buf), direction, cptr, optr,
                   _ptr(res), threads)
    return res


ST_SHIM_HOST = 0x800


def copy_hybrid(img: np.ndarray, spaces: np.ndarray, shims: np.ndarray, ops: np.ndarray, buf: np.ndarray,
                direction: int):
    """Hybrid-resolver copies with the default trap shim, in order (rows as
    :func:`copy`).  Returns (results, cut op index or len(ops), translations)."""
    spaces = np.ascontiguousarray(spaces, dtype=np.uint64).reshape(-1, 4)
    shims = np.ascontiguousarray(shims, dtype=np.uint64).reshape(-1, 4)
    ops = np.ascontiguousarray(ops, dtype=np.uint64).reshape(-1, 4)
    res = np.zeros((len(ops), 4), np.uint64)
    count = np.zeros(1, np.uint64)
    cut = lib().orc_copy_hybrid(_ptr(img), img.nbytes, _ptr(spaces), _ptr(shims), _ptr(ops), len(ops), _ptr(buf),
                                direction, _ptr(res), _ptr(count))
    return res, int(cut), int(count[0])
