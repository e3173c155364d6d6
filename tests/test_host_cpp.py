"""Runs the C++ port of the reference's unit / acceptance checks (tests/cpp/test_host.cpp)
against the host setup library and the CPU oracle.  CPU only."""
import subprocess

import oracle_binding as ob


def test_reference_unit_port():
    ob.ensure_built()
    proc = subprocess.run([ob.TEST_BIN], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout[-4000:] + proc.stderr[-2000:]
    assert "0 failures" in proc.stdout
