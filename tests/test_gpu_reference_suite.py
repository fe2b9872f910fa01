"""The reference's own C++ test programs (proj/tests/acceptance.cpp and the
doctest unit suites test_{stencil,layout,memsim,planner,engine}.cpp), compiled
UNMODIFIED against include/so2dr + libso2dr_b200.so by tests/cxx/Makefile --
the drop-in proof. The binaries are built in the build container (where
/root/reference exists) and travel to the GPU box in build/ref_tests/."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_tests")


def _run(name, timeout):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    return subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=BIN)


def test_reference_acceptance_suite_passes():
    p = _run("acceptance", 900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("PASS  criterion") == 11, p.stdout


def test_reference_unit_suites_pass():
    p = _run("unit_tests", 900)
    print(p.stdout[-2000:])
    assert p.returncode == 0, (p.stdout + p.stderr)[-5000:]
