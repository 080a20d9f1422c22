"""Drop-in proof: the REFERENCE package runs its own test suite on the B200
kernels.

oracle/build_ref.sh builds oracle/_ref/dropin/pkg: the reference pkg as
shipped plus the two things a maintainer would add — integration/b200.py as
``fedsim/backends/b200.py`` (a ctypes binding of the C ABI in
include/fedsim_b200.h) and integration/backends_init.patch (FEDSIM_BACKEND
accepts "b200"; reference backends/__init__.py:23-43). With
FEDSIM_BACKEND=b200 every ``get_backend()`` call of the reference's model,
client, selection, server and experiment modules lands on the sm_100a
kernels, and the reference's own tests (pkg/tests, 179 tests) must pass.

The reference's backend-parity test (tests/test_backends.py:30-58) compares
``fedsim.backends._core`` with numpy; it is also run a second time with the
compared module pointed at ``fedsim.backends.b200`` (the one-line import
swap is the only change), so b200 vs numpy is checked at the reference's
own 1e-12 tolerance and exact sign counts.

The tree is a build product (git-ignored, shipped with the snapshot): the
test skips when it was not built (no /root/reference where build() ran).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

from tests.conftest import ROOT, cuda_ok

DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin", "pkg")
LIB = os.path.join(ROOT, "paper_2503_15448_b200", "_fedsim_b200.so")

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device"),
    pytest.mark.skipif(not os.path.isdir(DROPIN), reason="oracle/_ref/dropin not built (oracle/build_ref.sh)"),
]


def _env() -> dict:
    env = dict(os.environ, FEDSIM_BACKEND="b200", FEDSIM_B200_LIB=LIB, PYTHONPATH=os.path.join(DROPIN, "src"))
    env.pop("PYTEST_ADDOPTS", None)
    return env


def _pytest(args, cwd) -> tuple[int, str, dict]:
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *args], cwd=cwd,
                       env=_env(), capture_output=True, text=True, timeout=1500)
    out = p.stdout + p.stderr
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|skipped|errors?)", out)}
    return p.returncode, out, counts


def test_reference_suite_on_b200_backend():
    # the active backend really is b200 inside the reference package
    probe = subprocess.run([sys.executable, "-c", "from fedsim.backends import backend_name, get_backend;"
                            "print(backend_name(), get_backend().__file__)"], env=_env(), capture_output=True,
                           text=True, timeout=300)
    assert probe.returncode == 0, probe.stderr
    assert probe.stdout.split()[0] == "b200", probe.stdout
    rc, out, counts = _pytest(["tests"], DROPIN)
    print(out[-3000:])
    assert rc == 0, out[-6000:]
    assert counts.get("passed", 0) >= 170 and counts.get("failed", 0) == 0, counts


def test_reference_backend_parity_against_b200(tmp_path):
    src = open(os.path.join(DROPIN, "tests", "test_backends.py")).read()
    swapped = src.replace('"fedsim.backends._core"', '"fedsim.backends.b200"')
    assert swapped != src
    (tmp_path / "test_backends_b200.py").write_text(swapped)
    rc, out, counts = _pytest([str(tmp_path / "test_backends_b200.py")], str(tmp_path))
    print(out[-2000:])
    assert rc == 0, out[-4000:]
    assert counts.get("passed", 0) >= 6 and counts.get("skipped", 0) == 0, counts
