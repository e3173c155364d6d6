"""Device side of the decomposition on one GPU: two partitioned contexts
(`pdg_create_partitioned`) exchange ghost states with `pdg_pack_states` /
`pdg_unpack_states` before every stage (`pdg_step_stage`).  Per-element device
arithmetic does not depend on the partition, so owned elements must match the
single-domain GPU run bit for bit.  NCCL replaces the local copy in
`paper_1607_03399_b200.distributed` (one GPU per rank)."""
import ctypes as C

import numpy as np
import pytest

import paper_1607_03399_b200 as pdg
from paper_1607_03399_b200 import capi, partition as P
from paper_1607_03399_b200.capi import check, lib

pytestmark = pytest.mark.gpu


class Rank:
    def __init__(self, part, degree):
        import torch
        self.part = part
        self.disc = pdg.build_discretization(part.mesh, degree)
        owned = np.ascontiguousarray(part.owned, dtype=np.uint8)
        h = C.c_void_p()
        check(lib().pdg_create_partitioned(self.disc.handle, 0, 0, owned.ctypes.data_as(C.POINTER(C.c_ubyte)),
                                           C.byref(h)))
        self.ctx = h
        ne = self.disc.num_elements()
        d2l = np.zeros(ne, dtype=np.int64)
        check(lib().pdg_device_order(self.ctx, d2l.ctypes.data_as(capi.I64P)))
        self.l2d = np.empty(ne, dtype=np.int64)
        self.l2d[d2l] = np.arange(ne)
        self.per = 4 * max(self.disc.info.np_wedge, self.disc.info.np_tet)
        self.torch = torch

    def dev_ids(self, local_ids):
        return self.torch.tensor(self.l2d[local_ids], dtype=self.torch.int64, device="cuda")

    def close(self):
        lib().pdg_destroy(self.ctx)


def exchange(ranks):
    torch = ranks[0].torch
    for r in ranks:
        for q, ids in r.part.send.items():
            src = r.dev_ids(ids)
            buf = torch.zeros((len(ids), r.per), dtype=torch.float64, device="cuda")
            check(lib().pdg_pack_states(r.ctx, C.c_void_p(src.data_ptr()), len(ids), C.c_void_p(buf.data_ptr())))
            check(lib().pdg_synchronize(r.ctx))
            dst_rank = ranks[q]
            dst = dst_rank.dev_ids(dst_rank.part.recv[r.part.rank])
            check(lib().pdg_unpack_states(dst_rank.ctx, C.c_void_p(dst.data_ptr()), len(ids),
                                          C.c_void_p(buf.data_ptr())))
            check(lib().pdg_synchronize(dst_rank.ctx))


@pytest.mark.parametrize("case,degree", [("hybrid", 3), ("layered", 4), ("unstructured", 5)])
def test_partitioned_contexts_match_single_domain(case, degree):
    world = 3 if case == "hybrid" else 2
    if case == "hybrid":
        mesh = pdg.structured_hybrid_box(4, 4, 2, 2, (1.0, 1.0), (1.0, 4.0))
        parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    elif case == "unstructured":
        mesh = pdg.make_family_mesh("unstructured", 0.5)
        parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    else:
        mesh = P.layered_global(5, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world)
        parts = [P.layered_slab(5, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world, r)
                 for r in range(world)]
    ranks = [Rank(p, degree) for p in parts]
    dt, nsteps = 0.004, 3
    for r in ranks:
        u = pdg.make_initial_state(r.disc, "gaussian", [0.35, 0.1, -0.05, 0.2]).u
        check(lib().pdg_set_state(r.ctx, C.c_void_p(u.ctypes.data), 0))
    for _ in range(nsteps):
        for s in range(5):
            exchange(ranks)
            for r in ranks:
                check(lib().pdg_step_stage(r.ctx, dt, s))
    # single domain on the same GPU
    d = pdg.build_discretization(mesh, degree)
    ctx = d.device()
    ctx.set_state(pdg.make_initial_state(d, "gaussian", [0.35, 0.1, -0.05, 0.2]).u)
    ctx.step(dt, nsteps)
    ug = ctx.get_state()
    off = d.elem_offset()
    seen = 0
    for r in ranks:
        ul = np.zeros(r.disc.total_dofs)
        check(lib().pdg_get_state(r.ctx, C.c_void_p(ul.ctypes.data), 0))
        loff = r.disc.elem_offset()
        for le in np.nonzero(r.part.owned)[0]:
            g = r.part.local_to_global[le]
            assert np.array_equal(ul[loff[le]:loff[le + 1]], ug[off[g]:off[g + 1]]), (case, r.part.rank, le)
            seen += 1
        r.close()
    assert seen == d.num_elements()


def exchange_traces(ranks, plans, offs):
    """face-trace refresh between contexts on one GPU (pdg_gather_values / pdg_scatter_values)"""
    torch = ranks[0].torch
    for r in ranks:
        for q in plans[r.part.rank]["send"]:
            src = torch.tensor(offs[r.part.rank]["send"][q], dtype=torch.int64, device="cuda")
            dst = torch.tensor(offs[q]["recv"][r.part.rank], dtype=torch.int64, device="cuda")
            assert src.numel() == dst.numel()
            buf = torch.zeros(src.numel(), dtype=torch.float64, device="cuda")
            check(lib().pdg_gather_values(r.ctx, C.c_void_p(src.data_ptr()), src.numel(), C.c_void_p(buf.data_ptr()),
                                          None))
            check(lib().pdg_synchronize(r.ctx))
            check(lib().pdg_scatter_values(ranks[q].ctx, C.c_void_p(dst.data_ptr()), dst.numel(),
                                           C.c_void_p(buf.data_ptr()), None))
            check(lib().pdg_synchronize(ranks[q].ctx))


@pytest.mark.parametrize("case,degree", [("hybrid", 2), ("layered", 5), ("unstructured", 3)])
def test_trace_exchange_with_interior_boundary_split(case, degree):
    """The overlapped multi-GPU schedule: interior launch (no ghost data), face-trace
    refresh, boundary launch -- bitwise equal to the single-domain run."""
    from paper_1607_03399_b200.distributed import trace_offsets
    world = 3 if case == "hybrid" else 2
    if case == "hybrid":
        mesh = pdg.structured_hybrid_box(4, 4, 2, 2, (1.0, 1.0), (1.0, 4.0))
        parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    elif case == "unstructured":
        mesh = pdg.make_family_mesh("unstructured", 0.5)
        parts = [P.partition_mesh(mesh, world, r) for r in range(world)]
    else:
        mesh = P.layered_global(5, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world)
        parts = [P.layered_slab(5, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], world, r)
                 for r in range(world)]
    ranks = [Rank(p, degree) for p in parts]
    plans = [P.trace_plan(r.part, r.disc) for r in ranks]
    offs = [{k: {q: trace_offsets(r.ctx, *v, r.per) for q, v in pl[k].items()} for k in ("send", "recv")}
            for r, pl in zip(ranks, plans)]
    for r in ranks:
        counts = (C.c_int64 * 6)()
        check(lib().pdg_partition_counts(r.ctx, counts))
        assert 0 < counts[4] + counts[5] < counts[0] + counts[1]  # some interior, some boundary
    dt, nsteps = 0.004, 2
    for r in ranks:
        u = pdg.make_initial_state(r.disc, "gaussian", [0.35, 0.1, -0.05, 0.2]).u
        check(lib().pdg_set_state(r.ctx, C.c_void_p(u.ctypes.data), 0))
    for _ in range(nsteps):
        for s in range(5):
            for r in ranks:
                check(lib().pdg_step_stage_part(r.ctx, dt, s, 1))
            exchange_traces(ranks, plans, offs)  # reads owned boundary values, writes ghost traces
            for r in ranks:
                check(lib().pdg_step_stage_part(r.ctx, dt, s, 2))
    d = pdg.build_discretization(mesh, degree)
    ctx = d.device()
    ctx.set_state(pdg.make_initial_state(d, "gaussian", [0.35, 0.1, -0.05, 0.2]).u)
    ctx.step(dt, nsteps)
    ug = ctx.get_state()
    off = d.elem_offset()
    seen = 0
    for r in ranks:
        ul = np.zeros(r.disc.total_dofs)
        check(lib().pdg_get_state(r.ctx, C.c_void_p(ul.ctypes.data), 0))
        loff = r.disc.elem_offset()
        for le in np.nonzero(r.part.owned)[0]:
            g = r.part.local_to_global[le]
            assert np.array_equal(ul[loff[le]:loff[le + 1]], ug[off[g]:off[g + 1]]), (case, r.part.rank, le)
            seen += 1
        r.close()
    assert seen == d.num_elements()


def test_partitioned_context_refuses_whole_domain_calls():
    """A partitioned context's ghosts are only current right after the caller's
    exchange: whole-step / rhs / phase / assembly entries refuse it; the watchdog
    scans owned elements only (a NaN planted in a ghost is not reported)."""
    part = P.layered_slab(4, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)], 2, 0)
    r = Rank(part, 2)
    try:
        n = r.disc.total_dofs
        u = np.zeros(n)
        ghost = int(np.nonzero(part.owned == 0)[0][0])
        off = r.disc.elem_offset()
        u[off[ghost]] = np.nan
        check(lib().pdg_set_state(r.ctx, u.ctypes.data_as(capi.DP), 0))
        bad = C.c_int64()
        check(lib().pdg_check_finite(r.ctx, C.byref(bad)))
        assert bad.value == -1
        assert lib().pdg_step_lserk(r.ctx, 1e-3, 1, None) == capi.PDG_ERR_CONFIG
        out = np.zeros(n)
        assert lib().pdg_rhs(r.ctx, u.ctypes.data_as(capi.DP), out.ctypes.data_as(capi.DP), 0) == capi.PDG_ERR_CONFIG
        assert lib().pdg_wedge_volume(r.ctx) == capi.PDG_ERR_CONFIG
        # the per-stage entry the distributed driver uses still works
        u[off[ghost]] = 0.0
        check(lib().pdg_set_state(r.ctx, u.ctypes.data_as(capi.DP), 0))
        check(lib().pdg_step_stage(r.ctx, 1e-3, 0))
    finally:
        r.close()
