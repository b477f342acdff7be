"""Stage the unmodified reference into the git-ignored ``baseline/_ref``.

* ``devfsim`` itself: ``pip install --no-index --no-build-isolation --no-deps
  --target baseline/_ref`` from a scratch copy of ``/root/reference/pkg``
  (the mount is read-only and the build writes into its source tree);
* the reference's own test suite, copied to ``baseline/_ref/devfsim_tests``,
  so ``tests/test_gpu_dropin.py`` can run it through the drop-in on the GPU
  box (where ``/root/reference`` does not exist).

``baseline/_ref`` is git-ignored (never committed) and not gpurun-ignored
(it travels with the snapshot).  Idempotent: a stamp of the source tree's
file sizes and mtimes skips the work when nothing changed.  Called by
``__graft_entry__.build()``; a no-op where ``/root/reference`` is absent.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")
STAMP = os.path.join(DEST, ".staged")


def _stamp() -> str:
    h = hashlib.sha256()
    for base, dirs, files in sorted(os.walk(SRC)):
        dirs.sort()
        for f in sorted(files):
            p = os.path.join(base, f)
            st = os.stat(p)
            h.update(f"{os.path.relpath(p, SRC)}:{st.st_size}:{int(st.st_mtime)}\n".encode())
    return h.hexdigest()


def stage(force: bool = False) -> bool:
    if not os.path.isdir(SRC):
        return False
    want = _stamp()
    if not force and os.path.exists(STAMP) and open(STAMP).read() == want:
        return True
    with tempfile.TemporaryDirectory() as tmp:
        copy = os.path.join(tmp, "pkg")
        shutil.copytree(SRC, copy)
        shutil.rmtree(DEST, ignore_errors=True)
        subprocess.run([sys.executable, "-m", "pip", "install", "-q", "--no-index", "--no-build-isolation",
                        "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DEST, copy], check=True)
    tests = os.path.join(DEST, "devfsim_tests")
    os.makedirs(tests, exist_ok=True)
    for f in os.listdir(os.path.join(SRC, "tests")):
        if f.endswith(".py"):
            shutil.copy(os.path.join(SRC, "tests", f), tests)
    with open(STAMP, "w") as f:
        f.write(want)
    return True


if __name__ == "__main__":
    print("staged" if stage(force="--force" in sys.argv) else "no reference here")
