"""VTK snapshot writer (snapshot.cpp:68-139 format): counts and data round trip on CPU."""
import numpy as np

import paper_1607_03399_b200 as pdg


def read_vtk(path):
    lines = open(path).read().split("\n")
    out, i = {}, 0
    while i < len(lines):
        tok = lines[i].split()
        if tok and tok[0] == "POINTS":
            n = int(tok[1])
            out["points"] = np.array([list(map(float, l.split())) for l in lines[i + 1:i + 1 + n]])
            i += n
        elif tok and tok[0] == "CELLS":
            out["ncells"], out["csize"] = int(tok[1]), int(tok[2])
        elif tok and tok[0] == "CELL_TYPES":
            n = int(tok[1])
            out["types"] = np.array(list(map(int, lines[i + 1:i + 1 + n])))
            i += n
        elif tok and tok[0] == "SCALARS":
            name = tok[1]
            n = out["points"].shape[0]
            out[name] = np.array(list(map(float, lines[i + 2:i + 2 + n])))
            i += n + 1
        i += 1
    return out


def test_vtk_counts_and_fields(tmp_path):
    N = 3
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1), N)
    u = np.random.default_rng(3).uniform(-1, 1, d.total_dofs)
    path = str(tmp_path / "snap.vtk")
    pdg.write_vtk_snapshot(d, u, path)
    v = read_vtk(path)
    nw, nt = int(d.info.num_wedges), int(d.info.num_tets)
    assert v["points"].shape == (int(d.info.total_nodes), 3)
    tri_cells, tet_cells = N * N, N ** 3  # sub-triangles of the lattice; sub-tets
    assert v["ncells"] == nw * tri_cells * N + nt * tet_cells
    assert v["csize"] == nw * tri_cells * N * 7 + nt * tet_cells * 5
    assert np.count_nonzero(v["types"] == 13) == nw * tri_cells * N
    assert np.count_nonzero(v["types"] == 10) == nt * tet_cells
    off = d.elem_offset()
    p = np.concatenate([u[off[e]:off[e] + (off[e + 1] - off[e]) // 4] for e in range(d.num_elements())])
    assert np.array_equal(v["p"], p)  # %.17g round trips exactly
    assert np.allclose(v["points"], d.node_coords(), rtol=0, atol=0)
