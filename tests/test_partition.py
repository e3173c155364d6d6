"""Multi-rank decomposition on CPU: world_size-2 gloo runs of the
partition + ghost-exchange logic, stepped with the CPU oracle, must reproduce the
single-domain oracle bit for bit on every owned element.  The GPU path
(`paper_1607_03399_b200.distributed`) uses the same partitions and exchange plans
with NCCL in place of gloo."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from paper_1607_03399_b200 import partition as P

LSERK_A = [0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
           -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0]
LSERK_B = [1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
           1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
           2277821191437.0 / 14882151754819.0]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def element_blocks(off, ids):
    return [np.arange(off[e], off[e + 1]) for e in ids]


def exchange(u, off, part):
    """ghost refresh over gloo: send owned boundary elements, receive ghosts"""
    import torch
    reqs, bufs = [], {}
    for q in sorted(set(part.send) | set(part.recv)):
        if q in part.send:
            data = np.concatenate([u[b] for b in element_blocks(off, part.send[q])])
            reqs.append(dist.isend(torch.from_numpy(data.copy()), q))
        if q in part.recv:
            n = sum(off[e + 1] - off[e] for e in part.recv[q])
            bufs[q] = torch.zeros(int(n), dtype=torch.float64)
            reqs.append(dist.irecv(bufs[q], q))
    for r in reqs:
        r.wait()
    for q, buf in bufs.items():
        blocks = element_blocks(off, part.recv[q])
        u[np.concatenate(blocks)] = buf.numpy()


def trace_index(d, plan_side):
    """reference-layout state offsets of the face traces of (element, face) pairs"""
    off = d.elem_offset()
    out = []
    for e, f in zip(*plan_side):
        my, _ = d.face_nodes(int(e), int(f))
        npe = (off[e + 1] - off[e]) // 4
        for fld in range(4):
            out.append(off[e] + fld * npe + np.asarray(my, dtype=np.int64))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def exchange_traces(u, plan):
    """face-trace refresh over gloo (what the GPU path ships): only the shared faces"""
    import torch
    reqs, bufs = [], {}
    for q in sorted(set(plan["send_idx"]) | set(plan["recv_idx"])):
        if q in plan["send_idx"]:
            reqs.append(dist.isend(torch.from_numpy(u[plan["send_idx"][q]].copy()), q))
        if q in plan["recv_idx"]:
            bufs[q] = torch.zeros(len(plan["recv_idx"][q]), dtype=torch.float64)
            reqs.append(dist.irecv(bufs[q], q))
    for r in reqs:
        r.wait()
    for q, buf in bufs.items():
        u[plan["recv_idx"][q]] = buf.numpy()


def run_rank(rank, world, port, case, degree, nsteps, out_dir, mode="elements"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = make_partition(case, world, rank)
        d = pdg.build_discretization(part.mesh, degree)
        off = d.elem_offset()
        if mode == "traces":
            tp = P.trace_plan(part, d)
            plan = {"send_idx": {q: trace_index(d, v) for q, v in tp["send"].items()},
                    "recv_idx": {q: trace_index(d, v) for q, v in tp["recv"].items()}}
        u = pdg.make_initial_state(d, "gaussian", [0.35, 0.1, -0.05, 0.2]).u
        dt = 0.01
        res = np.zeros_like(u)
        owned_idx = np.concatenate(element_blocks(off, np.nonzero(part.owned)[0]))
        for _ in range(nsteps):
            for s in range(5):
                if mode == "traces":
                    exchange_traces(u, plan)
                else:
                    exchange(u, off, part)
                r = ob.rhs(d, u, threads=1)
                res[owned_idx] = LSERK_A[s] * res[owned_idx] + dt * r[owned_idx]
                u[owned_idx] += LSERK_B[s] * res[owned_idx]
        own = np.nonzero(part.owned)[0]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 gids=part.local_to_global[own],
                 states=np.concatenate([u[b] for b in element_blocks(off, own)]),
                 sizes=np.array([off[e + 1] - off[e] for e in own]))
    finally:
        dist.destroy_process_group()


def make_partition(case, world, rank):
    if case == "hybrid":
        return P.partition_mesh(pdg.structured_hybrid_box(3, 3, 2, 2, (1.0, 1.0), (1.0, 4.0)), world, rank)
    if case == "unstructured":
        return P.partition_mesh(pdg.make_family_mesh("unstructured", 0.5), world, rank)
    if case == "strong":
        return P.layered_strong(4, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world, rank)
    return P.layered_slab(4, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world, rank)


def global_mesh(case, world):
    if case == "hybrid":
        return pdg.structured_hybrid_box(3, 3, 2, 2, (1.0, 1.0), (1.0, 4.0))
    if case == "unstructured":
        return pdg.make_family_mesh("unstructured", 0.5)
    if case == "strong":
        return P.layered_global(4, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], 1)
    return P.layered_global(4, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world)


@pytest.mark.parametrize("case,mode", [("hybrid", "elements"), ("unstructured", "elements"), ("layered", "elements"),
                                       ("hybrid", "traces"), ("unstructured", "traces"), ("layered", "traces"),
                                       ("strong", "traces")])
def test_two_rank_lserk_matches_single_domain(case, mode, tmp_path):
    """Whole-element ghost refresh and face-trace-only refresh (the GPU path's) both
    reproduce the single-domain run bit for bit: the RHS reads nothing else of a ghost."""
    world, degree, nsteps = 2, 2, 3
    mp.spawn(run_rank, args=(world, free_port(), case, degree, nsteps, str(tmp_path), mode), nprocs=world, join=True)
    d = pdg.build_discretization(global_mesh(case, world), degree)
    ug = pdg.make_initial_state(d, "gaussian", [0.35, 0.1, -0.05, 0.2]).u
    res = np.zeros_like(ug)
    for _ in range(nsteps):  # same update arithmetic as the ranks (numpy, no FMA contraction)
        for s in range(5):
            r = ob.rhs(d, ug, threads=1)
            res = LSERK_A[s] * res + 0.01 * r
            ug += LSERK_B[s] * res
    off = d.elem_offset()
    seen = 0
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        pos = 0
        for g, n in zip(z["gids"], z["sizes"]):
            got = z["states"][pos:pos + n]
            want = ug[off[g]:off[g + 1]]
            assert np.array_equal(got, want), (case, r, int(g), np.abs(got - want).max())
            pos += n
            seen += 1
    assert seen == d.num_elements()


def test_partition_plans_are_consistent():
    mesh = pdg.structured_hybrid_box(3, 3, 2, 2)
    world = 3
    parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    owned_total = sum(p.n_owned for p in parts)
    assert owned_total == mesh.num_elements()
    for p in parts:
        for q, ids in p.send.items():
            # what p sends to q is exactly what q receives from p, in the same global order
            assert np.array_equal(p.local_to_global[ids], parts[q].local_to_global[parts[q].recv[p.rank]])
            assert np.all(p.owned[ids] == 1)
            assert np.all(parts[q].owned[parts[q].recv[p.rank]] == 0)


def test_trace_plans_align_and_are_smaller():
    mesh = pdg.structured_hybrid_box(3, 3, 2, 2)
    world = 3
    parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    discs = [pdg.build_discretization(p.mesh, 3) for p in parts]
    plans = [P.trace_plan(p, d) for p, d in zip(parts, discs)]
    for p, d, pl in zip(parts, discs, plans):
        for q, (elems, faces) in pl["send"].items():
            re, rf = plans[q]["recv"][p.rank]
            # same global elements and faces, in the same order, on both sides
            assert np.array_equal(p.local_to_global[elems], parts[q].local_to_global[re])
            assert np.array_equal(faces, rf)
            assert len(trace_index(d, (elems, faces))) == len(trace_index(discs[q], (re, rf)))
            whole = sum((d.elem_offset()[e + 1] - d.elem_offset()[e]) for e in p.send[q])
            assert len(trace_index(d, (elems, faces))) < whole
