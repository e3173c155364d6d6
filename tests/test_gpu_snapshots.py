"""Snapshot streaming of the device run driver (
run_simulation snapshot semantics, solver.cpp:625-644): a snapshot at the
start and whenever the time passes the next multiple of the interval, each
the state at that step (streamed device -> pinned host while stepping goes on)."""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg

pytestmark = pytest.mark.gpu


def expected_snapshot_steps(t0, dt, steps, interval):
    """(step index, time) of every snapshot under the reference's rule"""
    out = [(0, t0)]
    nxt = t0 + interval
    t = t0
    for n in range(steps):
        t += dt
        if t + 1e-12 >= nxt:
            out.append((n + 1, t))
            while nxt <= t + 1e-12:
                nxt += interval
    return out


@pytest.mark.parametrize("integrator", ["lserk4", "ab3"])
def test_snapshots_match_reference_schedule_and_states(integrator):
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1, (1.0, 1.0), (1.0, 4.0)), 3)
    s = pdg.make_initial_state(d)
    u0 = s.u.copy()
    got = []
    opts = pdg.RunOptions(final_time=0.3, integrator=integrator, snapshot_interval=0.07,
                          snapshot_cb=lambda u, t, k: got.append((k, t, u)))
    res = pdg.run_simulation(d, s, opts)
    want = expected_snapshot_steps(0.0, res.dt, res.steps, 0.07)
    assert [k for k, _, _ in got] == list(range(len(want)))
    for (k, t, u), (nstep, tw) in zip(got, want):
        assert abs(t - tw) <= 1e-12
        ref = ob.lserk(d, u0, res.dt, nstep) if integrator == "lserk4" else ob.ab3(d, u0, res.dt, nstep)
        assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref), (k, nstep)
    assert np.array_equal(got[-1][2], s.u) or res.steps != want[-1][0]


def test_no_snapshots_without_callback():
    d = pdg.build_discretization(pdg.structured_wedge_box(2), 2)
    s = pdg.make_initial_state(d)
    res = pdg.run_simulation(d, s, pdg.RunOptions(final_time=0.1, snapshot_interval=0.01))
    assert res.steps > 0
