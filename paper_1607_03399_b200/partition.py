"""Mesh partitioning for multi-GPU runs: owned elements + one ghost layer.

The reference is single-process (SPEC.md:218 lists distributed runs as a
non-goal); this module implements the north star's sharding:

* every element is owned by exactly one rank;
* a rank's local mesh holds its owned elements plus the ghost layer, i.e.
  every non-owned element that shares a face with an owned one;
* before each LSERK stage a rank receives, from their owners, the current
  face traces (4 fields x face nodes) of its ghosts on the faces they share
  with its owned elements -- the only ghost data the RHS reads (`trace_plan`).
  Owned elements then see exactly the neighbour data of the single-domain
  run, so their RHS (and therefore the time-stepping) is the same as the
  global one (tests/test_partition.py checks this bit for bit with gloo).

Two partitioners are provided:
* `partition_mesh` -- generic: contiguous ranges of a Morton order of element
  centroids (the device order of one GPU), any wedge/tet mesh;
* `layered_slab` -- the weak-scaling benchmark mesh (config 5): rank r owns a
  slab of sublayers of a layered wedge mesh; ghosts are the one sublayer below
  and above, and only triangular faces are cut;
* `layered_strong` -- the strong-scaling one: one fixed layered mesh whose
  sublayers are split into nranks contiguous z ranges.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import solver as S

WEDGE_FACES = [[0, 1, 2], [3, 4, 5], [0, 1, 4, 3], [1, 2, 5, 4], [2, 0, 3, 5]]
TET_FACES = [[0, 1, 2], [0, 1, 3], [1, 2, 3], [0, 2, 3]]


@dataclass
class LocalPartition:
    rank: int
    nranks: int
    mesh: "S.HybridMesh"
    owned: np.ndarray                    # uint8 per local element
    local_to_global: np.ndarray          # global element id of each local element (-1 if n/a)
    # exchange plan: peer -> local element ids, identically ordered on both sides
    send: dict = field(default_factory=dict)
    recv: dict = field(default_factory=dict)

    @property
    def n_owned(self):
        return int(self.owned.sum())


def _morton_keys(c):
    lo, hi = c.min(0), c.max(0)
    span = np.where(hi > lo, hi - lo, 1.0)
    t = np.clip((c - lo) / span, 0.0, 1.0)
    q = (t * 2097151.0).astype(np.uint64)

    def spread(x):
        x = x & np.uint64(0x1FFFFF)
        x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
        x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
        x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
        x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
        x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
        return x

    return spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))


def element_adjacency(wedges, tets):
    """Face-neighbour lists from shared sorted vertex keys (mesh.cpp:398-437 semantics)."""
    nw, nt = len(wedges), len(tets)
    keys, elem = [], []
    for e_arr, faces, base in ((wedges, WEDGE_FACES, 0), (tets, TET_FACES, nw)):
        if len(e_arr) == 0:
            continue
        for fv in faces:
            k = np.sort(e_arr[:, fv], axis=1)
            if k.shape[1] == 3:
                k = np.concatenate([np.full((k.shape[0], 1), -1, k.dtype), k], axis=1)
            keys.append(k)
            elem.append(np.arange(len(e_arr)) + base)
    keys = np.concatenate(keys)
    elem = np.concatenate(elem)
    order = np.lexsort(keys.T[::-1])
    ks, es = keys[order], elem[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    a, b = es[:-1][same], es[1:][same]
    ne = nw + nt
    nbrs = [[] for _ in range(ne)]
    for x, y in zip(a.tolist(), b.tolist()):
        nbrs[x].append(y)
        nbrs[y].append(x)
    return nbrs


def partition_mesh(mesh: "S.HybridMesh", nranks: int, rank: int) -> LocalPartition:
    """Generic partition: contiguous ranges of the Morton order of element centroids."""
    arr = mesh.arrays()
    V, W, T, M = arr["vertices"], arr["wedges"], arr["tets"], arr["media"]
    nw, nt = len(W), len(T)
    cent = np.concatenate([V[W].mean(axis=1) if nw else np.zeros((0, 3)), V[T].mean(axis=1) if nt else np.zeros((0, 3))])
    order = np.argsort(_morton_keys(cent), kind="stable")
    owner = np.empty(nw + nt, dtype=np.int64)
    owner[order] = np.minimum(np.arange(nw + nt) * nranks // (nw + nt), nranks - 1)
    nbrs = element_adjacency(W, T)

    def ghosts_of(r):
        own = np.nonzero(owner == r)[0]
        g = set()
        for e in own.tolist():
            for q in nbrs[e]:
                if owner[q] != r:
                    g.add(q)
        return own, np.array(sorted(g), dtype=np.int64)

    own, ghost = ghosts_of(rank)
    local = np.concatenate([own, ghost])
    # local mesh keeps the global wedge-then-tet order (element kind blocks)
    local = np.sort(local)
    lw = local[local < nw]
    lt = local[local >= nw] - nw
    used = np.unique(np.concatenate([W[lw].ravel(), T[lt].ravel()]))
    remap = np.full(len(V), -1, dtype=np.int64)
    remap[used] = np.arange(len(used))
    lmesh = S.mesh_from_arrays(V[used], remap[W[lw]], remap[T[lt]], M[local])
    g2l = {int(g): i for i, g in enumerate(local.tolist())}
    owned = (owner[local] == rank).astype(np.uint8)
    part = LocalPartition(rank, nranks, lmesh, owned, local.copy())
    for peer in range(nranks):
        if peer == rank:
            continue
        peer_own, peer_ghost = ghosts_of(peer)
        # what the peer needs from me: its ghosts that I own; what I need: my ghosts it owns
        snd = peer_ghost[owner[peer_ghost] == rank]
        rcv = ghost[owner[ghost] == peer]
        if len(snd):
            part.send[peer] = np.array([g2l[int(g)] for g in snd], dtype=np.int64)
        if len(rcv):
            part.recv[peer] = np.array([g2l[int(g)] for g in rcv], dtype=np.int64)
    return part


def _slab_layers(slab_interfaces, slab_sublayers, slab_media, nranks, slab_height):
    """(z_bottom, z_top, media, owner) of every sublayer of the stacked slabs."""
    layers = []
    for r in range(nranks):
        z0 = r * slab_height
        for k in range(len(slab_sublayers)):
            zb, zt = slab_interfaces[k] + z0, slab_interfaces[k + 1] + z0
            for m in range(slab_sublayers[k]):
                f0, f1 = m / slab_sublayers[k], (m + 1) / slab_sublayers[k]
                layers.append((zb + f0 * (zt - zb), zb + f1 * (zt - zb), tuple(slab_media[k]), r))
    return layers


def layered_global(surface_n: int, slab_interfaces, slab_sublayers, slab_media, nranks: int,
                   slab_height: float = 2.0):
    """The single-domain mesh that `layered_slab` partitions (same vertex sheets)."""
    xy, tris = S.structured_surface(surface_n)
    nv = xy.shape[0]
    layers = _slab_layers(slab_interfaces, slab_sublayers, slab_media, nranks, slab_height)
    return S.stack_layers(xy, tris, [S.LayerSpec(np.full(nv, zb), np.full(nv, zt), 1, med)
                                     for (zb, zt, med, _) in layers])


def _sublayer_partition(surface_n, layers, nranks, rank) -> LocalPartition:
    """Partition of a stack of single sublayers (z_bottom, z_top, media, owner),
    owners contiguous and ascending in z: rank r keeps its owned sublayers plus
    one ghost sublayer below and above; only triangular faces are cut."""
    xy, tris = S.structured_surface(surface_n)
    nv, ntri = xy.shape[0], tris.shape[0]
    owner_of = np.array([lay[3] for lay in layers])
    mine = np.nonzero(owner_of == rank)[0]
    if len(mine) == 0:
        raise ValueError(f"rank {rank} owns no sublayer ({len(layers)} sublayers over {nranks} ranks)")
    first = int(mine[0]) - (1 if rank > 0 else 0)
    last = int(mine[-1]) + 1 + (1 if rank < nranks - 1 else 0)  # exclusive
    specs = [S.LayerSpec(np.full(nv, zb), np.full(nv, zt), 1, med) for (zb, zt, med, _) in layers[first:last]]
    lmesh = S.stack_layers(xy, tris, specs)
    owners = np.repeat(owner_of[first:last], ntri)
    owned = (owners == rank).astype(np.uint8)
    glob = np.arange(first * ntri, last * ntri, dtype=np.int64)
    part = LocalPartition(rank, nranks, lmesh, owned, glob)
    tri_ids = np.arange(ntri, dtype=np.int64)
    nlocal = last - first
    if rank > 0:  # below: my first owned sublayer goes down, the ghost sublayer 0 comes up
        part.send[rank - 1] = 1 * ntri + tri_ids
        part.recv[rank - 1] = 0 * ntri + tri_ids
    if rank < nranks - 1:
        top_owned = nlocal - 2
        part.send[rank + 1] = top_owned * ntri + tri_ids
        part.recv[rank + 1] = (nlocal - 1) * ntri + tri_ids
    return part


def layered_slab(surface_n: int, slab_interfaces, slab_sublayers, slab_media, nranks: int, rank: int,
                 slab_height: float = 2.0) -> LocalPartition:
    """Weak-scaling layered mesh (config 5): rank r owns the r-th copy of the slab
    (stacked in z), plus one ghost sublayer below and above."""
    layers = _slab_layers(slab_interfaces, slab_sublayers, slab_media, nranks, slab_height)
    return _sublayer_partition(surface_n, layers, nranks, rank)


def layered_strong_layers(slab_interfaces, slab_sublayers, slab_media, nranks: int):
    """Sublayers of ONE slab (the single-GPU mesh) with contiguous owners: the
    total work is fixed and the sublayers are split as evenly as possible."""
    layers = _slab_layers(slab_interfaces, slab_sublayers, slab_media, 1, 0.0)
    n = len(layers)
    return [(zb, zt, med, min(q * nranks // n, nranks - 1)) for q, (zb, zt, med, _) in enumerate(layers)]


def layered_strong(surface_n: int, slab_interfaces, slab_sublayers, slab_media, nranks: int,
                   rank: int) -> LocalPartition:
    """Strong-scaling layered mesh (config 5 strong): the single-domain mesh of
    `layered_mesh(surface_n, slab_interfaces, slab_sublayers, slab_media)` with
    its sublayers split into nranks contiguous z ranges."""
    layers = layered_strong_layers(slab_interfaces, slab_sublayers, slab_media, nranks)
    return _sublayer_partition(surface_n, layers, nranks, rank)


def face_offsets(disc) -> np.ndarray:
    """start of each element's faces in the (element, face) tables (wedges 5, tets 4)."""
    nw, nt = int(disc.info.num_wedges), int(disc.info.num_tets)
    return np.concatenate([5 * np.arange(nw + 1), 5 * nw + 4 * np.arange(1, nt + 1)]).astype(np.int64)


def trace_plan(part: LocalPartition, disc):
    """Face-trace exchange plan: peer -> (local elements, faces) to send / receive.

    Send to q: faces of my owned elements in part.send[q] whose neighbour is a
    ghost I receive from q.  Receive from q: faces of my ghosts in part.recv[q]
    whose neighbour I own.  Both ranks enumerate the same physical faces in the
    same order (element lists are identically ordered, element-local face
    numbering is the global one), so the per-face trace lists align."""
    nbr, _, _ = disc.face_table()
    off = face_offsets(disc)
    out = {"send": {}, "recv": {}}
    for q in sorted(set(part.send) | set(part.recv)):
        ghost_from_q = np.zeros(len(part.owned), dtype=bool)
        if q in part.recv:
            ghost_from_q[part.recv[q]] = True
        for kind, ids, want in (("send", part.send.get(q), lambda nb: ghost_from_q[nb]),
                                ("recv", part.recv.get(q), lambda nb: part.owned[nb] != 0)):
            if ids is None:
                continue
            elems, faces = [], []
            for e in ids.tolist():
                for f in range(off[e + 1] - off[e]):
                    nb = nbr[off[e] + f]
                    if nb >= 0 and want(nb):
                        elems.append(e)
                        faces.append(f)
            out[kind][q] = (np.array(elems, dtype=np.int64), np.array(faces, dtype=np.int32))
    return out
