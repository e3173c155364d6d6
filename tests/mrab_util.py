"""Rate levels of the multi-rate AB3 integrator, restated in numpy (test side):
level(e) = the largest g <= L with h_e / c_e >= 2^g min_k h_k / c_k, where
h = volume / surface area (estimate_dt's per-element term, solver.cpp:437-447)."""
import numpy as np


def element_rates(d):
    ne = d.num_elements()
    nw = int(d.info.num_wedges)
    arr = d.mesh.arrays() if d.mesh is not None else None
    rho_kappa = arr["media"]
    rate = np.zeros(ne)
    import paper_1607_03399_b200 as pdg
    from paper_1607_03399_b200.capi import check, lib
    a = pdg.export_arrays(d)
    for e in range(ne):
        if e < nw:
            vol, area = a["wedge_geom"][e, 3], a["wedge_geom"][e, 4]
        else:
            vol, area = a["tet_geom"][e - nw, 1], a["tet_geom"][e - nw, 2]
        rho, kappa = rho_kappa[e]
        rate[e] = (vol / area) / np.sqrt(kappa / rho)
    return rate


def levels(d, L):
    rate = element_rates(d)
    rmin = rate.min()
    lev = np.zeros(len(rate), dtype=np.int32)
    for g in range(1, L + 1):
        lev[rate >= np.ldexp(rmin, g) * (1 - 1e-12)] = g
    return lev


def two_level_mesh(surface_n=2):
    """two layers of equal thickness, kappa 1 | 4 (c = 1 | 2): the slow layer
    steps twice as long as the fast one"""
    import paper_1607_03399_b200 as pdg
    return pdg.layered_mesh(surface_n, [-1.0, 0.0, 1.0], [1, 1], [(1.0, 1.0), (1.0, 4.0)])
