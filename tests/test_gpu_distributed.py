"""The multi-GPU driver itself (`distributed.DistributedLSERK`, the code `bench.py --gpus N`
runs) on one GPU: one Python thread per rank, each with its own partitioned device
context, library stream and exchange stream, so the interior launch, the face-trace
gather / transfer / scatter on the exchange stream and the boundary launch run
concurrently exactly as on N GPUs.  Only NCCL is replaced: `ThreadComm` hands the
send buffers between the rank threads (NCCL refuses two ranks on one device).  Owned
elements must equal the single-domain GPU run bit for bit."""
import threading

import numpy as np
import pytest

import paper_1607_03399_b200 as pdg
from paper_1607_03399_b200 import partition as P

pytestmark = pytest.mark.gpu


class ThreadComm:
    """torch.distributed's point-to-point surface (P2POp, batch_isend_irecv) between
    threads of one process; one `view(rank)` per rank thread"""

    isend, irecv = "isend", "irecv"

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=120)
        self.box = {}
        self.calls = [0] * world

    def view(self, rank):
        hub = self

        class View:
            isend, irecv = hub.isend, hub.irecv

            @staticmethod
            def P2POp(op, tensor, peer):
                return (op, tensor, peer)

            @staticmethod
            def batch_isend_irecv(ops):
                import torch
                hub.calls[rank] += 1
                torch.cuda.current_stream().synchronize()  # the gathered traces are complete
                for op, t, q in ops:
                    if op == hub.isend:
                        hub.box[(rank, q)] = t
                hub.barrier.wait()
                for op, t, q in ops:
                    if op == hub.irecv:
                        src = hub.box[(q, rank)]
                        assert src.numel() == t.numel(), "send / recv plans disagree"
                        t.copy_(src)
                torch.cuda.current_stream().synchronize()
                hub.barrier.wait()  # peers may overwrite their send buffers again
                return []

        return View()


def _partitions(case, world):
    if case == "layered":
        shape = (6, [-1.0, 0.0, 1.0], [2, 3], [(1.0, 1.0), (1.0, 4.0)])
        return P.layered_global(*shape, world), [P.layered_slab(*shape, world, r) for r in range(world)]
    if case == "hybrid":
        mesh = pdg.structured_hybrid_box(4, 4, 2, 2, (1.0, 1.0), (1.0, 4.0))
    else:
        mesh = pdg.make_family_mesh("unstructured", 0.5)
    return mesh, [P.partition_mesh(mesh, world, r) for r in range(world)]


@pytest.mark.parametrize("case,world,degree", [("layered", 2, 3), ("layered", 3, 5), ("hybrid", 3, 4),
                                               ("unstructured", 2, 2)])
def test_distributed_lserk_threads_match_single_domain(case, world, degree):
    from paper_1607_03399_b200.distributed import DistributedLSERK
    mesh, parts = _partitions(case, world)
    comm = ThreadComm(world)
    dt, nsteps, init = 0.004, 3, [0.35, 0.1, -0.05, 0.2]
    solvers = [DistributedLSERK(p, degree, device=0, comm=comm.view(p.rank)) for p in parts]
    for sv in solvers:
        sv.set_state(pdg.make_initial_state(sv.disc, "gaussian", init).u)
    errors = []

    def run(sv):
        try:
            sv.step(dt, nsteps)
            sv.synchronize()
        except BaseException as exc:  # surfaced below
            errors.append(exc)
            comm.barrier.abort()

    threads = [threading.Thread(target=run, args=(sv,)) for sv in solvers]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    assert all(c == 5 * nsteps for c in comm.calls)  # one exchange per LSERK stage on every rank

    d = pdg.build_discretization(mesh, degree)
    ctx = d.device()
    ctx.set_state(pdg.make_initial_state(d, "gaussian", init).u)
    ctx.step(dt, nsteps)
    ug = ctx.get_state()
    off = d.elem_offset()
    seen = 0
    for sv in solvers:
        ul = sv.get_state()
        loff = sv.disc.elem_offset()
        for le in np.nonzero(sv.part.owned)[0]:
            g = sv.part.local_to_global[le]
            assert np.array_equal(ul[loff[le]:loff[le + 1]], ug[off[g]:off[g + 1]]), (case, sv.part.rank, le)
            seen += 1
        sv.close()
    assert seen == d.num_elements()
