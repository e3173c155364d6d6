"""Subprocess body of tests/test_gpu_optin_kernels.py: one RHS and 2 LSERK steps of the
kernel selected by the environment (PDG_WEDGE_SL / PDG_WEDGE_LO / PDG_WEDGE_WS, read once
per process) on a mesh where every CTA / team runs several tickets, against the oracle.
usage: optin_check.py N"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle_binding as ob  # noqa: E402
import paper_1607_03399_b200 as pdg  # noqa: E402
from parity_util import config2_mesh, field_errors, rel_l2  # noqa: E402

N = int(sys.argv[1])
threads = os.cpu_count() or 4
m = config2_mesh(10, (15, 15, 20)) if N >= 4 else config2_mesh(100, (2, 2, 2))
d = pdg.build_discretization(m, N, threads=threads)
u = np.random.default_rng(11 + N).uniform(-1.0, 1.0, d.total_dofs)
ctx = d.device()
errs = field_errors(d, ctx.rhs(u), ob.rhs(d, u, threads=threads))
li = ctx.launch_info()["wedge"]
assert li["launched"] == 1 and li["tickets"] >= 2 * li["teams"], li
dt = pdg.estimate_dt(d, 0.5)
ctx.set_state(u)
ctx.step(dt, 2)
rel = rel_l2(ctx.get_state(), ob.lserk(d, u, dt, 2, threads=threads))
print(f"N={N} rhs {max(errs):.2e} step {rel:.2e}")
assert max(errs) <= 1e-12 and rel <= 1e-10, (errs, rel)
