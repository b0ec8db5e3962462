"""The reference's OWN unit suites (tests/test_engine.cpp, test_metrics.cpp,
test_rng.cpp, test_graph.cpp) and acceptance binary, compiled unchanged
against the B200 drop-in (integration/pglayout_b200_engine.cpp replacing
src/engine.cpp, libpgl_b200.so underneath) by integration/Makefile. The
binaries are built in the build container (the reference sources only exist
there) and travel in oracle/_ref/conformance/."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "conformance")


def run(name, timeout=900):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (make -C integration; needs /root/reference)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=timeout)
    print(p.stdout[-4000:])
    print(p.stderr[-4000:])
    return p


@pytest.mark.parametrize("suite", ["test_engine", "test_metrics", "test_rng", "test_graph", "test_gfa_io"])
def test_reference_unit_suite_passes_on_b200_facade(gpu, suite):
    p = run(suite)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "failed: 0" in p.stdout


@pytest.mark.slow
def test_reference_acceptance_on_b200_facade(gpu):
    p = run("acceptance", timeout=1500)
    assert "[FAIL]" not in p.stdout, p.stdout
    assert p.returncode == 0
