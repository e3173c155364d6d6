"""Shared helpers of the GPU parity tests (vectorised, so they stay cheap at 1e6 elements)."""
import numpy as np

import paper_1607_03399_b200 as pdg

CONFIG2_MEDIA = [(1.0, 1.0), (1.0, 4.0), (1.0, 2.25)]
CONFIG2_INTERFACES = [-1.0, -0.4, 0.2, 1.0]


def config2_mesh(surface_n=100, sublayers=(15, 15, 20)):
    """BASELINE configs[1] / SURVEY 8(d) row 2: stack_layers on the structured
    n-surface, flat layers z = -1 -> -0.4 -> 0.2 -> 1, kappa = 1, 4, 2.25.
    n=100 x (15,15,20) is the 1e6-wedge benchmark mesh; n=10 x (15,15,20) its
    1/100-size copy (same layering, 10,000 wedges)."""
    return pdg.layered_mesh(surface_n, CONFIG2_INTERFACES, list(sublayers), CONFIG2_MEDIA)


def field_blocks(d, v):
    """[(K, 4, Np) view of the wedge blocks, (K, 4, Np) view of the tet blocks]"""
    nw, nt = int(d.info.num_wedges), int(d.info.num_tets)
    npw, npt = int(d.info.np_wedge), int(d.info.np_tet)
    v = np.asarray(v)
    out = []
    if nw:
        out.append(v[: nw * 4 * npw].reshape(nw, 4, npw))
    if nt:
        out.append(v[nw * 4 * npw:].reshape(nt, 4, npt))
    return out


def field_errors(d, got, want):
    """max-abs error / max-abs value of each of the 4 fields (p, ux, uy, uz)."""
    errs = []
    for f in range(4):
        num = max(np.abs(g[:, f, :] - w[:, f, :]).max() for g, w in zip(field_blocks(d, got), field_blocks(d, want)))
        den = max(np.abs(w[:, f, :]).max() for w in field_blocks(d, want))
        errs.append(num / max(den, 1e-300))
    return errs


def rel_l2(got, want):
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))
