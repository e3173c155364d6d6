"""The AB3 step fused into the exact DMMA wedge stage kernel (M_AB3: rhs into
the history slot and u_{n+1} = u_n + dt/12 (23 f_n - 16 f_{n-1} + 5 f_{n-2}) in
the epilogue, one launch per step; wedge-only meshes, N = 4..7): against the
oracle's AB3 (solver.cpp:559-581) and bitwise against the unfused path (rhs
launch + update kernel, PDG_AB3_FUSED=0) run in a separate process."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from parity_util import config2_mesh, rel_l2

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("degree", [4, 5, 6, 7])
def test_fused_ab3_matches_oracle(degree):
    d = pdg.build_discretization(config2_mesh(6, (2, 2, 2)), degree)
    u0 = np.random.default_rng(degree).uniform(-1, 1, d.total_dofs)
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx = pdg.DeviceContext(d, flags=pdg.capi.CTX_TIMING)
    ctx.set_state(u0)
    ctx.step(dt, 8, integrator="ab3")
    kt = ctx.kernel_times(reset=True)
    # 2 LSERK bootstrap steps (2 x (1 rhs + 5 stages)) + 6 fused AB3 launches
    assert kt["wedge_launches"] == 2 * 6 + 6 and kt["tet_launches"] == 0, kt
    assert rel_l2(ctx.get_state(), ob.ab3(d, u0, dt, 8)) <= 1e-10
    ctx.close()


def _run_ab3(fused):
    code = (
        "import sys, json, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_1607_03399_b200 as pdg\n"
        "from parity_util import config2_mesh\n"
        "d = pdg.build_discretization(config2_mesh(6, (2, 2, 2)), 5)\n"
        "u0 = np.random.default_rng(3).uniform(-1, 1, d.total_dofs)\n"
        "ctx = pdg.DeviceContext(d); ctx.set_state(u0); ctx.step(1e-3, 7, integrator='ab3')\n"
        "np.save(sys.argv[1], ctx.get_state())\n") % (os.path.dirname(HERE), HERE)
    return code


def test_fused_ab3_bitwise_equals_unfused(tmp_path):
    outs = []
    for fused in ("1", "0"):
        path = str(tmp_path / f"ab3_{fused}.npy")
        env = dict(os.environ, PDG_AB3_FUSED=fused)
        r = subprocess.run([sys.executable, "-c", _run_ab3(fused), path], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
