"""The opt-in stage kernels kept as measured alternatives stay
parity-green: the warp-specialised N >= 4 kernel (wedge_ws.cu, PDG_WEDGE_WS=1), the
thread-per-DOF-column low-order kernel (wedge_lo.cu, PDG_WEDGE_LO=1) and the
thread-per-(wedge, slice) N = 1 kernel (wedge_sl.cu, PDG_WEDGE_SL=1).  The selection is
read once per process, so each case runs tests/optin_check.py in a subprocess:
one RHS (<= 1e-12 per field) and 2 LSERK steps (<= 1e-10) against the oracle on a
mesh where every team / CTA loops over several tickets."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env,degree", [("PDG_WEDGE_SL", 1), ("PDG_WEDGE_LO", 1), ("PDG_WEDGE_LO", 2),
                                        ("PDG_WEDGE_LO", 3), ("PDG_WEDGE_WS", 4), ("PDG_WEDGE_WS", 5)])
def test_optin_kernel_matches_oracle(env, degree):
    r = subprocess.run([sys.executable, os.path.join(HERE, "optin_check.py"), str(degree)],
                       env={**os.environ, env: "1"}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
