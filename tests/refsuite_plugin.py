"""pytest plugin: run the reference's own test suite through the drop-in.

Loaded with ``-p refsuite_plugin`` (tests/ on sys.path) in a separate pytest
process over the reference's tests (staged by ``__graft_entry__.build()``
under the git-ignored ``baseline/_ref/devfsim_tests``).  It installs this
package into ``devfsim`` before any test module imports it, so every
``devfsim.memvirt`` / ``devfsim.backend`` name the tests and the reference's
own modules use resolves to the B200 data plane (install.py).
"""

from __future__ import annotations

import json
import os

from paper_1304_3771_b200.install import install

install("devfsim")

_outcomes: dict[str, str] = {}


def pytest_runtest_logreport(report):
    if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
        _outcomes[report.nodeid] = report.outcome


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PV_REFSUITE_JSON")
    if path:
        with open(path, "w") as f:
            json.dump({"exitstatus": int(exitstatus), "outcomes": _outcomes}, f, indent=0, sort_keys=True)
