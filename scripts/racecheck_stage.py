"""One fused LSERK step of the stage kernels on a layered mesh large enough that every
team / CTA runs several elements / chunks (so the cross-iteration synchronisation --
parity buffers, dropped end barriers -- is exercised), checked against the CPU oracle.
Run under `compute-sanitizer --tool racecheck` (scripts/gpu_racecheck.sh)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_binding as ob  # noqa: E402
import paper_1607_03399_b200 as pdg  # noqa: E402

N, mass, n, subl = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), [int(x) for x in sys.argv[4].split(",")]
mesh = pdg.layered_mesh(n, [-1.0, -0.4, 0.2, 1.0], subl, [(1.0, 1.0), (1.0, 4.0), (1.0, 2.25)])
d = pdg.build_discretization(mesh, N, mass=mass)
u = np.random.default_rng(1607).uniform(-1.0, 1.0, d.total_dofs)
dt = pdg.estimate_dt(d, 0.5)
ctx = d.device()
ctx.set_state(u)
ctx.step(dt, 1)
got = ctx.get_state()
want = ob.lserk(d, u, dt, 1)
rel = np.linalg.norm(got - want) / np.linalg.norm(want)
print(f"N={N} {mass} wedges={mesh.num_wedges()} step rel L2 {rel:.2e}")
assert rel <= 1e-10
