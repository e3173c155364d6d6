"""assemble_global on the GPU (analysis.cpp:12-40): the
distance-2 coloured probe batches give exactly the column-by-column operator,
the reference's 20000-DOF cap is kept, and the config-4 spectrum criteria
(acceptance.cpp:103-131) hold on the assembled device operator."""
import numpy as np
import pytest

import paper_1607_03399_b200 as pdg

pytestmark = pytest.mark.gpu


def columns(ctx, n, cols):
    out = np.empty((n, len(cols)))
    e = np.zeros(n)
    for k, j in enumerate(cols):
        e[j] = 1.0
        out[:, k] = ctx.rhs(e)
        e[j] = 0.0
    return out


@pytest.mark.parametrize("mesh_fn,degree,mass", [
    (lambda: pdg.spectra_mesh(), 2, "exact"),
    (lambda: pdg.structured_hybrid_box(3, 3, 2, 1, (1.0, 1.0), (1.0, 4.0)), 2, "exact"),
    (lambda: pdg.perturb_vertically(pdg.structured_wedge_box(3), 0.3, 5), 2, "wadg"),
])
def test_colored_assembly_equals_column_probes(mesh_fn, degree, mass):
    d = pdg.build_discretization(mesh_fn(), degree, mass=mass)
    n = d.total_dofs
    A = pdg.assemble_global(d)
    rng = np.random.default_rng(0)
    cols = np.unique(np.concatenate([rng.integers(0, n, 60), [0, n - 1]]))
    want = columns(d.device(), n, cols)
    assert np.array_equal(A[:, cols], want)


def test_assembly_cap():
    d = pdg.build_discretization(pdg.structured_wedge_box(3), 3)  # 54 wedges x 160 = 8640 DOF: fine
    assert pdg.assemble_global(d).shape == (d.total_dofs, d.total_dofs)
    big = pdg.build_discretization(pdg.structured_wedge_box(4), 3)  # 128 x 160 = 20480 DOF
    with pytest.raises(pdg.capi.AnalysisError):
        pdg.assemble_global(big)


def test_config4_spectra_on_device_operator():
    mesh = pdg.spectra_mesh()
    out = {}
    for mass in ("exact", "wadg", "lumped"):
        for flux in ("upwind", "central"):
            d = pdg.build_discretization(mesh, 2, flux=flux, mass=mass)
            ev = pdg.spectrum(pdg.assemble_global(d))
            out[(mass, flux)] = (ev.real.max(), np.abs(ev.real).max(), np.abs(ev).max())
    for mass in ("exact", "wadg"):
        assert out[(mass, "upwind")][0] <= 1e-10 * out[(mass, "upwind")][2]
        assert out[(mass, "central")][1] <= 1e-8 * out[(mass, "central")][2]
    assert out[("lumped", "upwind")][0] > 0.0 and out[("lumped", "central")][0] > 0.0
