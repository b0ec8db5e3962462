"""The reference's own host-side unit suites, compiled unchanged against the
drop-in facades (integration/pglayout_b200_io.cpp replaces src/gfa.cpp and
src/layout_io.cpp; integration/pglayout_b200_engine.cpp replaces
src/engine.cpp) by integration/Makefile. These two suites need no GPU:
test_gfa_io.cpp exercises parse_gfa / write_gfa / write_layout_tsv /
read_layout_tsv (all served by libpgl_b200's multithreaded IO), and
test_graph.cpp the graph model the facades build."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "conformance")


@pytest.mark.parametrize("suite", ["test_gfa_io", "test_graph"])
def test_reference_host_suite_passes_on_facade(suite):
    path = os.path.join(BIN, suite)
    if not os.path.exists(path):
        pytest.skip(f"{suite} not built (make -C integration; needs /root/reference)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "failed: 0" in p.stdout
