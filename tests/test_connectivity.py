"""Connectivity and face maps are bit-exact with the reference's greedy matcher
(mesh.cpp:398-481), restated here independently in numpy on small meshes."""
import numpy as np
import pytest

import paper_1607_03399_b200 as pdg

WEDGE_FACES = [[0, 1, 2], [3, 4, 5], [0, 1, 4, 3], [1, 2, 5, 4], [2, 0, 3, 5]]
TET_FACES = [[0, 1, 2], [0, 1, 3], [1, 2, 3], [0, 2, 3]]


def greedy_reference(d, mesh):
    """owners map keyed by sorted vertex ids, first (e,f) owns; greedy nearest unused node."""
    arr = mesh.arrays()
    V, W, T = arr["vertices"], arr["wedges"], arr["tets"]
    nw = W.shape[0]
    xyz = d.node_coords()
    off = d.elem_offset()
    node_off = np.concatenate([[0], np.cumsum(np.diff(off) // 4)])
    owners = {}
    for e in range(nw + T.shape[0]):
        faces = WEDGE_FACES if e < nw else TET_FACES
        verts = W[e] if e < nw else T[e - nw]
        for f, fv in enumerate(faces):
            owners.setdefault(tuple(sorted(verts[fv])), []).append((e, f))
    out = {}
    for key, lst in owners.items():
        if len(lst) != 2:
            continue
        (ea, fa), (eb, fb) = lst
        ma, _ = d.face_nodes(ea, fa)
        mb, _ = d.face_nodes(eb, fb)
        ca, cb = xyz[node_off[ea] + ma], xyz[node_off[eb] + mb]
        va = W[ea] if ea < nw else T[ea - nw]
        vb = W[eb] if eb < nw else T[eb - nw]
        diam = max(np.ptp(V[va], axis=0).max(), 0)  # only used for the tolerance scale
        da = max(np.linalg.norm(V[va][i] - V[va][j]) for i in range(len(va)) for j in range(len(va)))
        db = max(np.linalg.norm(V[vb][i] - V[vb][j]) for i in range(len(vb)) for j in range(len(vb)))
        tol = 1e-10 * max(da, db)
        used = np.zeros(len(ca), bool)
        perm = np.zeros(len(ca), int)
        for i in range(len(ca)):
            dist = np.linalg.norm(cb - ca[i], axis=1)
            dist[used] = np.inf
            j = int(np.argmin(dist))
            assert dist[j] <= tol
            perm[i] = j
            used[j] = True
        inv = np.zeros_like(perm)
        inv[perm] = np.arange(len(perm))
        out[(ea, fa)] = (eb, fb, perm)
        out[(eb, fb)] = (ea, fa, inv)
    return out


@pytest.mark.parametrize("maker,degree", [
    (lambda: pdg.structured_hybrid_box(2, 2, 1, 1), 3),
    (lambda: pdg.make_family_mesh("unstructured", 0.5), 4),
    (lambda: pdg.spectra_mesh(), 5),
    (lambda: pdg.structured_hybrid_box(1, 2, 1, 2), 2),
])
def test_face_maps_bit_exact(maker, degree):
    mesh = maker()
    d = pdg.build_discretization(mesh, degree)
    ref = greedy_reference(d, mesh)
    nbr, nbr_face, pid = d.face_table()
    counts = [5] * int(d.info.num_wedges) + [4] * int(d.info.num_tets)
    fo = np.concatenate([[0], np.cumsum(counts)])
    n_int = 0
    for e in range(len(counts)):
        for f in range(counts[e]):
            q = fo[e] + f
            if (e, f) not in ref:
                assert nbr[q] == -1
                continue
            eb, fb, perm = ref[(e, f)]
            assert (nbr[q], nbr_face[q]) == (eb, fb)
            assert np.array_equal(d.perm(int(pid[q])), perm)
            n_int += 1
    assert n_int == 2 * d.info.num_interior_pairs


def test_large_layered_mesh_connectivity_counts():
    m = pdg.layered_mesh(20, [-1.0, 0.0, 1.0], [3, 4], [(1.0, 1.0), (1.0, 4.0)])
    d = pdg.build_discretization(m, 2)
    ntri = 2 * 20 * 20
    layers = 7
    assert d.info.num_wedges == ntri * layers
    # interior tri faces between layers + interior quad faces within layers
    interior_quads = (3 * ntri - 4 * 20) // 2
    assert d.info.num_interior_pairs == ntri * (layers - 1) + interior_quads * layers
    assert d.info.num_boundary_faces == 2 * ntri + 4 * 20 * layers
