"""pdg_disc_from_arrays (include/prismdg_b200.h): a Discretization assembled from
a caller's flattened arrays -- the reference's own Discretization members
(solver.hpp:29-59: mesh, geom, wedge_ops, tet_ops, face_data) -- so the device
path can run on operators the reference's Eigen setup built.  CPU checks: the
round trip rebuilds the same discretization bit for bit (connectivity recovered
from nbr_nodes, the oracle's RHS identical), the caller's operators are the ones
used (not rebuilt), and malformed input is rejected with the reference's
exception types."""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg

MESHES = {
    "hybrid": lambda: pdg.structured_hybrid_box(2, 2, 1, 1, (1.0, 1.0), (1.0, 4.0)),
    "unstructured": lambda: pdg.make_family_mesh("unstructured", 0.5),
    "spectra": lambda: pdg.spectra_mesh(),
}


@pytest.mark.parametrize("name", sorted(MESHES))
@pytest.mark.parametrize("degree", [1, 3])
def test_round_trip_is_bitwise(name, degree):
    d = pdg.build_discretization(MESHES[name](), degree)
    a = pdg.export_arrays(d)
    d2 = pdg.discretization_from_arrays(a)
    assert d2.total_dofs == d.total_dofs
    assert np.array_equal(d2.elem_offset(), d.elem_offset())
    nb, nf, pid = d.face_table()
    nb2, nf2, _ = d2.face_table()
    assert np.array_equal(nb, nb2) and np.array_equal(nf, nf2)
    u = np.random.default_rng(degree).uniform(-1, 1, d.total_dofs)
    assert np.array_equal(ob.rhs(d2, u, threads=2), ob.rhs(d, u, threads=2))
    assert ob.energy(d2, u) == ob.energy(d, u)
    assert pdg.estimate_dt(d2, 0.5) == pdg.estimate_dt(d, 0.5)


def test_callers_operators_are_used():
    """A caller operator that differs (here: one wedge's lifts scaled) changes the
    rhs of exactly that wedge -- the ingest copies, it does not rebuild."""
    d = pdg.build_discretization(MESHES["hybrid"](), 2)
    a = pdg.export_arrays(d)
    a["tri_lift"][0] *= 1.5
    a["quad_lift"][0] *= 1.5
    d2 = pdg.discretization_from_arrays(a)
    u = np.random.default_rng(0).uniform(-1, 1, d.total_dofs)
    r1, r2 = ob.rhs(d, u, threads=1), ob.rhs(d2, u, threads=1)
    off = d.elem_offset()
    assert not np.array_equal(r1[off[0]:off[1]], r2[off[0]:off[1]])
    assert np.array_equal(r1[off[1]:], r2[off[1]:])


def test_rejects_malformed_arrays():
    d = pdg.build_discretization(MESHES["hybrid"](), 2)
    a = pdg.export_arrays(d)
    bad = dict(a)
    bad["face_nbr_nodes"] = a["face_nbr_nodes"].copy()
    q = int(np.nonzero(a["face_nbr"] >= 0)[0][0])
    bad["face_nbr_nodes"][q, 0] = 10_000  # not a node of any neighbour face
    with pytest.raises(pdg.MeshError):
        pdg.discretization_from_arrays(bad)
    bad = dict(a)
    bad["face_nbr"] = a["face_nbr"].copy()
    bad["face_nbr"][q] = -1  # one-sided pairing
    with pytest.raises(pdg.MeshError):
        pdg.discretization_from_arrays(bad)
    bad = dict(a)
    bad["face_my_nodes"] = np.zeros_like(a["face_nbr_nodes"])  # not the reference face-node lists
    with pytest.raises(pdg.ConfigError):
        pdg.discretization_from_arrays(bad)
    bad = dict(a)
    del bad["tri_lift"]
    with pytest.raises(pdg.ConfigError):
        pdg.discretization_from_arrays(bad)
