"""Multi-GPU time stepping: one rank per GPU, face-trace exchange every stage,
overlapped with the interior elements.

Each rank owns a `partition.LocalPartition`; the device context computes only
owned elements, ordered interior (no ghost neighbour) first, then boundary,
then ghosts (`pdg_create_partitioned`).  Per LSERK stage:
  exchange stream:  wait for the previous stage; gather the face traces the
                    peers need (`pdg_gather_values`, 4 fields x face nodes of
                    the shared faces only, `partition.trace_plan`); NCCL
                    point-to-point send/recv (`batch_isend_irecv`, NVLink /
                    NVSwitch on B200; no collective); scatter the received
                    traces into the ghost slots (`pdg_scatter_values`).
  compute stream:   interior stage launch (`pdg_step_stage_part(.., 1)`),
                    concurrently with the exchange; then wait for it and run
                    the boundary launch (`pdg_step_stage_part(.., 2)`).
The only collective is the energy all-reduce (one double; watchdog/logging).
`exchange="elements"` keeps the round-1 whole-element exchange without overlap.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from . import partition as P
from . import solver as S
from .capi import check, lib


def trace_offsets(ctx, elems, faces, per):
    """device-layout state offsets of the face traces of (local element, face) pairs"""
    n = len(elems)
    out = np.zeros(max(1, n * per), dtype=np.int64)
    cnt = C.c_int64()
    e = np.ascontiguousarray(elems, dtype=np.int64)
    f = np.ascontiguousarray(faces, dtype=np.int32)
    check(lib().pdg_trace_offsets(ctx, n, e.ctypes.data_as(capi.I64P), f.ctypes.data_as(capi.IP),
                                  out.ctypes.data_as(capi.I64P), C.byref(cnt)))
    return out[: cnt.value]


class DistributedLSERK:
    def __init__(self, part, degree: int, device: int = 0, flux="upwind", mass="exact", threads=0,
                 exchange="traces", flags=0, comm=None):
        """flags: pdg_create flags (capi.CTX_TIMING for per-launch event timing); comm: the
        point-to-point / all-reduce module, torch.distributed unless a test passes a stand-in"""
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, (comm if comm is not None else dist)
        self.part = part
        self.disc = S.build_discretization(part.mesh, degree, flux=flux, mass=mass, threads=threads)
        owned = np.ascontiguousarray(part.owned, dtype=np.uint8)
        h = C.c_void_p()
        check(lib().pdg_create_partitioned(self.disc.handle, device, flags,
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
        self.mode = exchange
        self.peers = sorted(set(part.send) | set(part.recv))
        self.send_idx, self.recv_idx, self.send_buf, self.recv_buf = {}, {}, {}, {}
        if exchange == "traces":
            plan = P.trace_plan(part, self.disc)
            for q in self.peers:
                for kind, store, bufs in (("send", self.send_idx, self.send_buf),
                                          ("recv", self.recv_idx, self.recv_buf)):
                    elems, faces = plan[kind].get(q, (np.zeros(0, np.int64), np.zeros(0, np.int32)))
                    offs = trace_offsets(self.ctx, elems, faces, per)
                    store[q] = torch.tensor(offs, dtype=torch.int64, device=dev)
                    bufs[q] = torch.zeros(len(offs), dtype=torch.float64, device=dev)
        else:
            for q in self.peers:
                s_ids = l2d[part.send[q]] if q in part.send else np.zeros(0, np.int64)
                r_ids = l2d[part.recv[q]] if q in part.recv else np.zeros(0, np.int64)
                self.send_idx[q] = torch.tensor(s_ids, dtype=torch.int64, device=dev)
                self.recv_idx[q] = torch.tensor(r_ids, dtype=torch.int64, device=dev)
                self.send_buf[q] = torch.zeros((len(s_ids), per), dtype=torch.float64, device=dev)
                self.recv_buf[q] = torch.zeros((len(r_ids), per), dtype=torch.float64, device=dev)
        self.exchange_bytes = sum(b.numel() * 8 for b in self.send_buf.values())
        self.xstream = torch.cuda.Stream(device=dev)  # exchange stream (overlaps the interior launch)

    def close(self):
        if self.ctx is not None and self.ctx.value:
            lib().pdg_destroy(self.ctx)
            self.ctx = None

    def set_state(self, u_local):
        u = np.ascontiguousarray(u_local, dtype=np.float64)
        check(lib().pdg_set_state(self.ctx, C.c_void_p(u.ctypes.data), 0))

    def get_state(self, out=None):
        """local state in the reference layout; `out` may be a (pinned) float64 host array"""
        if out is None:
            out = np.zeros(self.disc.total_dofs)
        check(lib().pdg_get_state(self.ctx, C.c_void_p(out.ctypes.data), 0))
        return out

    def kernel_times(self, reset=False):
        wms, tms = C.c_double(), C.c_double()
        wl, tl = C.c_int64(), C.c_int64()
        check(lib().pdg_kernel_times(self.ctx, C.byref(wms), C.byref(wl), C.byref(tms), C.byref(tl), int(reset)))
        return {"wedge_ms": wms.value, "wedge_launches": wl.value, "tet_ms": tms.value, "tet_launches": tl.value}

    def stage_bytes(self):
        """algorithmic bytes of one whole stage over the owned elements (5-stage average)"""
        wb, tb = C.c_double(), C.c_double()
        check(lib().pdg_stage_bytes(self.ctx, C.byref(wb), C.byref(tb)))
        return wb.value, tb.value

    def _p2p(self):
        dist = self.dist
        ops = []
        for q in self.peers:
            if self.send_buf[q].numel():
                ops.append(dist.P2POp(dist.isend, self.send_buf[q], q))
            if self.recv_buf[q].numel():
                ops.append(dist.P2POp(dist.irecv, self.recv_buf[q], q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def exchange(self):
        """whole-element ghost refresh on the library stream (exchange="elements")"""
        torch = self.torch
        if not self.peers:
            return
        with torch.cuda.stream(self.stream):
            for q in self.peers:
                n = self.send_idx[q].numel()
                if n:
                    check(lib().pdg_pack_states(self.ctx, C.c_void_p(self.send_idx[q].data_ptr()), n,
                                                C.c_void_p(self.send_buf[q].data_ptr())))
            self._p2p()
            for q in self.peers:
                n = self.recv_idx[q].numel()
                if n:
                    check(lib().pdg_unpack_states(self.ctx, C.c_void_p(self.recv_idx[q].data_ptr()), n,
                                                  C.c_void_p(self.recv_buf[q].data_ptr())))

    def _stage_overlapped(self, dt, s):
        """face traces on the exchange stream while the interior elements run"""
        torch = self.torch
        self.xstream.wait_stream(self.stream)  # traces of the previous stage's result
        with torch.cuda.stream(self.xstream):
            for q in self.peers:
                n = self.send_idx[q].numel()
                if n:
                    check(lib().pdg_gather_values(self.ctx, C.c_void_p(self.send_idx[q].data_ptr()), n,
                                                     C.c_void_p(self.send_buf[q].data_ptr()),
                                                     C.c_void_p(self.xstream.cuda_stream)))
            self._p2p()
            for q in self.peers:
                n = self.recv_idx[q].numel()
                if n:
                    check(lib().pdg_scatter_values(self.ctx, C.c_void_p(self.recv_idx[q].data_ptr()), n,
                                                      C.c_void_p(self.recv_buf[q].data_ptr()),
                                                      C.c_void_p(self.xstream.cuda_stream)))
        check(lib().pdg_step_stage_part(self.ctx, dt, s, 1))  # interior: no ghost data
        self.stream.wait_stream(self.xstream)
        check(lib().pdg_step_stage_part(self.ctx, dt, s, 2))  # boundary: after the exchange

    def step(self, dt: float, nsteps: int = 1):
        for _ in range(nsteps):
            for s in range(5):
                if self.mode == "traces":
                    self._stage_overlapped(dt, s)
                else:
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
