"""The drop-in inside the reference's own stack.

Every check runs in its own process (``install`` rebinds module globals
process-wide) over the unmodified reference staged in ``baseline/_ref``:

* the install seam swaps ``devfsim.memvirt``, the ``devfsim.backend`` access
  classes and the exception identity (CPU: no data-plane call);
* the mode-equivalence digests of seeds 5/42/77 (from
  harness.py:650-762: every caller-visible result + guest memory through
  Frontend -> Backend -> ClassDriver -> ctx.mem) equal the golden values;
* a driver copy faulting partway returns ERR_BAD_ADDRESS with
  ``(bytes_copied,)`` (devices.py:423-424) and ioctl blob staging
  (backend.py:526-534) behaves like the reference, run side by side with the
  uninstalled reference in another process;
* the reference's own test files pass with the drop-in installed.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "devfsim_tests")
CHECKS = os.path.join(ROOT, "tests", "dropin_checks.py")

needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "devfsim")),
                               reason="baseline/_ref not staged (run __graft_entry__.build())")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests"), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


def _check(name: str, install: bool = True, timeout: int = 600) -> dict:
    args = [sys.executable, CHECKS, name] + ([] if install else ["--no-install"])
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout, env=_env(), cwd=ROOT)
    assert p.returncode == 0, p.stderr[-4000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@needs_ref
def test_install_swaps_the_seams():
    out = _check("identity")
    assert all(out.values()), out


@needs_ref
@pytest.mark.gpu
def test_mode_equivalence_digests_through_dropin():
    out = _check("digests")
    assert out["all_match_golden"], out["digests"]
    assert len(out["digests"]) == 9


@needs_ref
@pytest.mark.gpu
def test_faulting_driver_copy_returns_bad_address():
    mine = _check("badaddr")
    ref = _check("badaddr", install=False)
    assert mine == ref
    for key, row in mine.items():
        assert row["status"] == 14 and row["values"][0] == 2048, (key, row)


@needs_ref
@pytest.mark.gpu
def test_ioctl_blob_staging_matches_reference():
    mine = _check("staging")
    ref = _check("staging", install=False)
    assert mine == ref
    assert mine["blocking/shadow"]["rows"][-1][1] == "PageFault"


# reference tests that assert on wall-clock rates (test_acceptance.py:280-324 and the harness scenarios
# they run): the only ones rerun once on failure
TIMED = ("test_c06_concurrency_ordering", "test_c07_poll_semantics")

REF_FILES = ["test_memvirt.py", "test_acceptance.py", "test_backend.py", "test_frontend.py", "test_devices.py",
             "test_interrupts.py", "test_guest.py", "test_hypercall.py", "test_harness.py"]


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("name", REF_FILES)
def test_reference_suite_through_dropin(name, tmp_path):
    """The reference's own test file, run by pytest in a fresh process with
    the drop-in installed before any test module imports devfsim."""
    report = tmp_path / "outcomes.json"
    env = _env()
    env["PV_REFSUITE_JSON"] = str(report)
    p = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REF_TESTS, name), "-q", "-p", "refsuite_plugin",
                        "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir", REF_TESTS],
                       capture_output=True, text=True, timeout=1500, env=env, cwd=str(tmp_path))
    out = json.loads(report.read_text()) if report.exists() else {"outcomes": {}}
    failed = {k: v for k, v in out["outcomes"].items() if v != "passed"}
    timing = [k for k in failed if any(t in k for t in TIMED)]
    if failed and len(timing) == len(failed):
        # wall-clock acceptance checks of the reference (real-time threads racing a
        # compute loop) fail under box noise now and then: rerun those once
        report.unlink(missing_ok=True)
        ids = [os.path.join(REF_TESTS, k) for k in timing]
        p = subprocess.run([sys.executable, "-m", "pytest", *ids, "-q", "-p", "refsuite_plugin", "-p",
                            "no:cacheprovider", "-o", "addopts=", "--rootdir", REF_TESTS],
                           capture_output=True, text=True, timeout=1500, env=env, cwd=str(tmp_path))
        again = json.loads(report.read_text()) if report.exists() else {"outcomes": {}}
        out["rerun_once"] = again["outcomes"]
        for k, v in again["outcomes"].items():
            out["outcomes"][k] = v
        failed = {k: v for k, v in out["outcomes"].items() if v != "passed"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"refsuite_{name[:-3]}.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    assert p.returncode == 0 and not failed and out["outcomes"], (failed, p.stdout[-6000:])
