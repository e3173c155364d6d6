#!/usr/bin/env python3
"""Simulated-time throughput of the three device integrators on the configs[1]
mesh (1e6 layered wedges, exact mass): LSERK45 at the estimated dt, AB3 at a
quarter of it (dt_scale, solver.hpp:114) and multi-rate AB3 (2 rate levels on
this mesh: the kappa = 1 layer steps twice as long).  Reports the device time
to advance the same simulated span (after each integrator's bootstrap) and
DOF x simulated-time per second."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1607_03399_b200 as pdg  # noqa: E402
from parity_util import config2_mesh  # noqa: E402


def timed(ctx, fn):
    stream = torch.cuda.ExternalStream(ctx.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def main(degree=int(os.environ.get("DEGREE", "5")), span_steps=int(os.environ.get("SPAN", "12"))):
    d = pdg.build_discretization(config2_mesh(100, (15, 15, 20)), degree, threads=os.cpu_count() or 1)
    u0 = pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0]).u
    dt = pdg.estimate_dt(d, 0.5)
    span = span_steps * dt
    out = {"degree": degree, "wedges": d.num_elements(), "dofs": d.total_dofs, "span": span}
    # LSERK45
    ctx = pdg.DeviceContext(d)
    ctx.set_state(u0)
    ctx.step(dt, 2)
    ms = timed(ctx, lambda: ctx.step(dt, span_steps))
    out["lserk4"] = {"ms": ms, "rhs_evals_per_elem": 5 * span_steps}
    # AB3 at dt/4 after its 2-step bootstrap
    ctx.set_state(u0)
    ctx.step(dt / 4, 4, integrator="ab3")
    ms = timed(ctx, lambda: ctx.step(dt / 4, 4 * span_steps, integrator="ab3"))
    out["ab3"] = {"ms": ms, "rhs_evals_per_elem": 4 * span_steps}
    ctx.close()
    # multi-rate AB3, fine step dt/4, macro step 2 fine steps
    mctx = pdg.DeviceContext(d, flags=pdg.capi.CTX_MRAB_LEVELS(3))
    lev, nlev = mctx.mrab_levels()
    mctx.set_state(u0)
    macro = (1 << (nlev - 1))
    mctx.step(dt / 4, 4, integrator="mrab")
    nm = int(round(4 * span_steps / macro))
    ms = timed(mctx, lambda: mctx.step(dt / 4, nm, integrator="mrab"))
    share = [float((lev == g).mean()) for g in range(nlev)]
    out["mrab"] = {"ms": ms, "levels": nlev, "level_share": share,
                   "rhs_evals_per_elem": 4 * span_steps * sum(s / (1 << g) for g, s in enumerate(share))}
    mctx.close()
    for k in ("lserk4", "ab3", "mrab"):
        out[k]["dof_time_per_s"] = d.total_dofs * span / (out[k]["ms"] / 1e3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
