"""One fused LSERK step on a hybrid box large enough that every tet team runs several
batches (so the cross-batch synchronisation -- slot parity, end-of-batch exchange --
is exercised), checked against the CPU oracle.  Run under compute-sanitizer racecheck."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_binding as ob  # noqa: E402
import paper_1607_03399_b200 as pdg  # noqa: E402

N, nx, nzw, nzt = (int(x) for x in sys.argv[1:5])
mesh = pdg.structured_hybrid_box(nx, nx, nzw, nzt, (1.0, 1.0), (1.0, 4.0))
d = pdg.build_discretization(mesh, N)
u = np.random.default_rng(1607).uniform(-1.0, 1.0, d.total_dofs)
dt = pdg.estimate_dt(d, 0.5)
ctx = d.device()
ctx.set_state(u)
ctx.step(dt, 1)
got = ctx.get_state()
want = ob.lserk(d, u, dt, 1)
rel = np.linalg.norm(got - want) / np.linalg.norm(want)
print(f"N={N} hybrid wedges={mesh.num_wedges()} step rel L2 {rel:.2e}")
assert rel <= 1e-10
