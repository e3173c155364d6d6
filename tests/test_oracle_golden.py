"""Pins the CPU oracle against the reference's published numbers
(tests/golden/paper_convergence.json, transcribed from PAPER.md): L2 errors of the
standing-wave problem on structured / unstructured / Arnold wedge meshes, N=1..3."""
import json
import os

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_convergence.json")))


def oracle_error(family, h, N):
    d = pdg.build_discretization(pdg.make_family_mesh(family, h), N)
    s = pdg.make_initial_state(d)
    u, t, info = ob.run(d, s.u, 0.0, 1.0, 0.5, 0.0, 1.0, 8)
    assert info["stable"] == 1.0
    return pdg.l2_error(d, u, t)


@pytest.mark.parametrize("N", [1, 2, 3])
def test_structured_errors_match_paper(N):
    ref = GOLD["structured_errors"][str(N)]
    hs = GOLD["h"]
    errs = []
    for k, h in enumerate(hs[:3] if N == 3 else hs[:4]):
        e = oracle_error("structured", h, N)
        tol = 0.1 if h == 2.0 else 1e-2
        assert abs(e - ref[k]) <= tol * ref[k], (N, h, e, ref[k])
        errs.append(e)
    rate = pdg.fit_rate(hs[: len(errs)], errs)
    # pre-asymptotic levels; the paper's rate uses h down to 0.125
    assert abs(rate - GOLD["rates"]["structured"][N - 1]) <= 0.35


@pytest.mark.parametrize("family", ["unstructured", "arnold"])
def test_family_errors_within_acceptance_band(family):
    ref = GOLD[f"{family}_errors"]["2"]
    for k, h in enumerate([2.0, 1.0, 0.5]):
        e = oracle_error(family, h, 2)
        f = GOLD["acceptance"]["error_band_factor"]
        assert ref[k] / f <= e <= ref[k] * f, (family, h, e, ref[k])


def test_oracle_serial_and_parallel_update_identical():
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1), 3)
    u = np.random.default_rng(3).uniform(-1, 1, d.total_dofs)
    dt = pdg.estimate_dt(d, 0.5)
    a = ob.lserk(d, u, dt, 2, threads=1, parallel_update=False)
    b = ob.lserk(d, u, dt, 2, threads=4, parallel_update=True)
    assert np.array_equal(a, b)
