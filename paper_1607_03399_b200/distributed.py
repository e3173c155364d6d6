"""Multi-GPU time stepping: one rank per GPU, ghost exchange before every stage.

Each rank owns a `partition.LocalPartition`; the device context computes only
owned elements (ghosts are ordered after them, `pdg_create_partitioned`).
Before each of the 5 LSERK stages the boundary elements' states are packed on
the device (`pdg_pack_states`), exchanged with the neighbour ranks through
`torch.distributed` point-to-point ops (NCCL over NVLink / NVSwitch on B200;
no collective is involved), and unpacked into the ghost slots
(`pdg_unpack_states`).  All device work is issued on the library's stream, so
the exchange is stream-ordered with the stage kernels.  The only collective is
the optional energy all-reduce (two doubles; watchdog semantics).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from . import solver as S
from .capi import check, lib


class DistributedLSERK:
    def __init__(self, part, degree: int, device: int = 0, flux="upwind", mass="exact", threads=0):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.part = part
        self.disc = S.build_discretization(part.mesh, degree, flux=flux, mass=mass, threads=threads)
        owned = np.ascontiguousarray(part.owned, dtype=np.uint8)
        h = C.c_void_p()
        check(lib().pdg_create_partitioned(self.disc.handle, device, 0,
                                           owned.ctypes.data_as(C.POINTER(C.c_ubyte)), C.byref(h)))
        self.ctx = h
        counts = (C.c_int64 * 4)()
        check(lib().pdg_active_counts(self.ctx, counts))
        self.n_owned_wedges, self.n_owned_tets = int(counts[0]), int(counts[1])
        ne = self.disc.num_elements()
        d2l = np.zeros(ne, dtype=np.int64)
        check(lib().pdg_device_order(self.ctx, d2l.ctypes.data_as(capi.I64P)))
        l2d = np.empty(ne, dtype=np.int64)
        l2d[d2l] = np.arange(ne)
        dev = torch.device("cuda", device)
        self.device = dev
        self.stream = torch.cuda.ExternalStream(lib().pdg_stream(self.ctx), device=dev)
        per = 4 * max(self.disc.info.np_wedge, self.disc.info.np_tet)
        self.peers = sorted(set(part.send) | set(part.recv))
        self.send_idx, self.recv_idx, self.send_buf, self.recv_buf = {}, {}, {}, {}
        for q in self.peers:
            s_ids = l2d[part.send[q]] if q in part.send else np.zeros(0, np.int64)
            r_ids = l2d[part.recv[q]] if q in part.recv else np.zeros(0, np.int64)
            self.send_idx[q] = torch.tensor(s_ids, dtype=torch.int64, device=dev)
            self.recv_idx[q] = torch.tensor(r_ids, dtype=torch.int64, device=dev)
            self.send_buf[q] = torch.zeros((len(s_ids), per), dtype=torch.float64, device=dev)
            self.recv_buf[q] = torch.zeros((len(r_ids), per), dtype=torch.float64, device=dev)
        self.exchange_bytes = sum(b.numel() * 8 for b in self.send_buf.values())

    def close(self):
        if self.ctx is not None and self.ctx.value:
            lib().pdg_destroy(self.ctx)
            self.ctx = None

    def set_state(self, u_local):
        u = np.ascontiguousarray(u_local, dtype=np.float64)
        check(lib().pdg_set_state(self.ctx, C.c_void_p(u.ctypes.data), 0))

    def get_state(self):
        out = np.zeros(self.disc.total_dofs)
        check(lib().pdg_get_state(self.ctx, C.c_void_p(out.ctypes.data), 0))
        return out

    def exchange(self):
        torch, dist = self.torch, self.dist
        if not self.peers:
            return
        with torch.cuda.stream(self.stream):
            for q in self.peers:
                n = self.send_idx[q].numel()
                if n:
                    check(lib().pdg_pack_states(self.ctx, C.c_void_p(self.send_idx[q].data_ptr()), n,
                                                C.c_void_p(self.send_buf[q].data_ptr())))
            ops = []
            for q in self.peers:
                if self.send_buf[q].numel():
                    ops.append(dist.P2POp(dist.isend, self.send_buf[q], q))
                if self.recv_buf[q].numel():
                    ops.append(dist.P2POp(dist.irecv, self.recv_buf[q], q))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            for q in self.peers:
                n = self.recv_idx[q].numel()
                if n:
                    check(lib().pdg_unpack_states(self.ctx, C.c_void_p(self.recv_idx[q].data_ptr()), n,
                                                  C.c_void_p(self.recv_buf[q].data_ptr())))

    def step(self, dt: float, nsteps: int = 1):
        for _ in range(nsteps):
            for s in range(5):
                self.exchange()
                check(lib().pdg_step_stage(self.ctx, dt, s))

    def energy(self):
        e = C.c_double()
        check(lib().pdg_energy(self.ctx, C.byref(e)))
        t = self.torch.tensor([e.value], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return float(t.item())

    def synchronize(self):
        check(lib().pdg_synchronize(self.ctx))
