"""Python mirror of the reference's mesh / discretization / solver API over the C ABI.

Names follow proj/include/prismdg/{mesh,solver,analysis}.hpp so tests read like
the reference's own: ``build_discretization(structured_wedge_box(2), 3)``,
``compute_rhs(d, u)``, ``run_simulation(d, state, opts)``.  Everything that
evaluates the semi-discrete operator runs on the GPU; host-side helpers
(``estimate_dt``, initial states, ``l2_error``) call the C++ setup library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import check, lib

_dp = lambda a: a.ctypes.data_as(capi.DP)  # noqa: E731
_ip = lambda a: a.ctypes.data_as(capi.IP)  # noqa: E731


def _media(m):
    if m is None:
        return None
    arr = (C.c_double * 2)(float(m[0]), float(m[1]))
    return C.cast(arr, capi.DP)


class HybridMesh:
    """Owning handle of a prismdg::HybridMesh (mesh.hpp:22-41)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().pdg_mesh_free(self._h)
            self._h = C.c_void_p(None)

    @property
    def handle(self):
        return self._h

    def counts(self):
        c = (C.c_int64 * 3)()
        check(lib().pdg_mesh_counts(self._h, c))
        return int(c[0]), int(c[1]), int(c[2])

    def num_wedges(self):
        return self.counts()[1]

    def num_tets(self):
        return self.counts()[2]

    def num_elements(self):
        _, w, t = self.counts()
        return w + t

    def arrays(self):
        nv, nw, nt = self.counts()
        v = np.zeros((nv, 3))
        w = np.zeros((nw, 6), dtype=np.int32)
        t = np.zeros((nt, 4), dtype=np.int32)
        m = np.zeros((nw + nt, 2))
        check(lib().pdg_mesh_export(self._h, _dp(v), _ip(w), _ip(t), _dp(m)))
        return {"vertices": v, "wedges": w, "tets": t, "media": m}

    def volume(self):
        out = C.c_double()
        check(lib().pdg_mesh_volume(self._h, C.byref(out)))
        return out.value

    def save(self, path: str):
        check(lib().pdg_mesh_save(self._h, path.encode()))


def _mesh_from(fn, *args) -> HybridMesh:
    out = C.c_void_p()
    check(fn(*args, C.byref(out)))
    return HybridMesh(out.value)


def structured_hybrid_box(nx, ny, nz_wedge, nz_tet, wedge_media=(1.0, 1.0), tet_media=(1.0, 1.0)):
    return _mesh_from(lib().pdg_mesh_structured_hybrid_box, nx, ny, nz_wedge, nz_tet,
                      _media(wedge_media), _media(tet_media))


def structured_wedge_box(n, media=(1.0, 1.0)):
    return structured_hybrid_box(n, n, n, 0, media, media)


def unstructured_wedge_box(n, xy_jitter, z_amplitude, seed, media=(1.0, 1.0)):
    return _mesh_from(lib().pdg_mesh_unstructured_wedge_box, n, xy_jitter, z_amplitude, seed, _media(media))


def arnold_wedge_box(n, delta, media=(1.0, 1.0)):
    return _mesh_from(lib().pdg_mesh_arnold_wedge_box, n, delta, _media(media))


def perturb_vertically(mesh: HybridMesh, amplitude, seed):
    return _mesh_from(lib().pdg_mesh_perturb_vertically, mesh.handle, amplitude, seed)


FAMILIES = {"structured": 0, "unstructured": 1, "arnold": 2}


def make_family_mesh(family, h, seed=20160311, xy_jitter=0.15, z_amplitude=0.3, arnold_delta=0.25):
    fam = FAMILIES[family] if isinstance(family, str) else int(family)
    return _mesh_from(lib().pdg_mesh_family, fam, h, seed, xy_jitter, z_amplitude, arnold_delta)


def spectra_mesh(seed=42, amplitude=0.3):
    return _mesh_from(lib().pdg_mesh_spectra, seed, amplitude)


def mesh_from_arrays(vertices, wedges, tets, media):
    v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    w = np.ascontiguousarray(wedges, dtype=np.int32).reshape(-1, 6)
    t = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
    m = np.ascontiguousarray(media, dtype=np.float64).reshape(-1, 2)
    return _mesh_from(lib().pdg_mesh_from_arrays, v.shape[0], _dp(v), w.shape[0], _ip(w), t.shape[0], _ip(t), _dp(m))


def load_mesh(path: str):
    return _mesh_from(lib().pdg_mesh_load, path.encode())


@dataclass
class LayerSpec:
    """mesh.hpp:50-55"""

    z_bottom: np.ndarray
    z_top: np.ndarray
    sublayers: int = 1
    media: tuple = (1.0, 1.0)


def stack_layers(xy, triangles, layers: list[LayerSpec]):
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    tris = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
    nv, nl = xy.shape[0], len(layers)
    zb = np.ascontiguousarray(np.stack([np.asarray(l.z_bottom, dtype=np.float64) for l in layers]))
    zt = np.ascontiguousarray(np.stack([np.asarray(l.z_top, dtype=np.float64) for l in layers]))
    sub = np.array([l.sublayers for l in layers], dtype=np.int32)
    med = np.ascontiguousarray(np.array([l.media for l in layers], dtype=np.float64))
    return _mesh_from(lib().pdg_mesh_stack_layers, nv, _dp(xy), tris.shape[0], _ip(tris), nl,
                      _dp(zb), _dp(zt), _ip(sub), _dp(med))


def structured_surface(n):
    """The 'layers' mesh-kind surface of config.cpp:232-243."""
    i, j = np.meshgrid(np.arange(n + 1), np.arange(n + 1))
    xy = np.stack([-1.0 + 2.0 * i.ravel() / n, -1.0 + 2.0 * j.ravel() / n], axis=1)
    tris = []
    for jj in range(n):
        for ii in range(n):
            a = jj * (n + 1) + ii
            tris.append((a, a + 1, a + n + 2))
            tris.append((a, a + n + 2, a + n + 1))
    return xy, np.array(tris, dtype=np.int32)


def layered_mesh(surface_n, interfaces, sublayers, media):
    """Flat layers: `interfaces` z values (len L+1), per-layer sublayers and (rho, kappa)."""
    xy, tris = structured_surface(surface_n)
    nv = xy.shape[0]
    layers = [LayerSpec(np.full(nv, interfaces[k]), np.full(nv, interfaces[k + 1]), sublayers[k], media[k])
              for k in range(len(sublayers))]
    return stack_layers(xy, tris, layers)


class Discretization:
    """Owning handle of a prismdg::Discretization (solver.hpp:29-59)."""

    def __init__(self, handle: int, mesh: HybridMesh):
        self._h = C.c_void_p(handle)
        self.mesh = mesh
        info = capi.DiscInfo()
        check(lib().pdg_disc_get_info(self._h, C.byref(info)))
        self.info = info
        self.degree = info.degree
        self.total_dofs = int(info.total_dofs)
        self._ctx = None

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None:
            ctx.close()
        if getattr(self, "_h", None) and self._h.value:
            lib().pdg_disc_free(self._h)
            self._h = C.c_void_p(None)

    @property
    def handle(self):
        return self._h

    def num_elements(self):
        return int(self.info.num_wedges + self.info.num_tets)

    def elem_offset(self):
        out = np.zeros(self.num_elements() + 1, dtype=np.int64)
        check(lib().pdg_disc_elem_offset(self._h, out.ctypes.data_as(capi.I64P)))
        return out

    def face_table(self):
        n = int(self.info.num_faces)
        nbr = np.zeros(n, dtype=np.int32)
        nf = np.zeros(n, dtype=np.int32)
        pid = np.zeros(n, dtype=np.int32)
        check(lib().pdg_disc_face_table(self._h, _ip(nbr), _ip(nf), _ip(pid)))
        return nbr, nf, pid

    def perm(self, perm_id):
        n = C.c_int()
        check(lib().pdg_disc_perm(self._h, perm_id, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        check(lib().pdg_disc_perm(self._h, perm_id, _ip(out), C.byref(n)))
        return out

    def face_nodes(self, e, f):
        n = C.c_int()
        check(lib().pdg_disc_face_nodes(self._h, e, f, None, None, C.byref(n)))
        my = np.zeros(n.value, dtype=np.int32)
        nb = np.zeros(n.value, dtype=np.int32)
        check(lib().pdg_disc_face_nodes(self._h, e, f, _ip(my), _ip(nb), C.byref(n)))
        return my, nb

    def node_coords(self):
        xyz = np.zeros((int(self.info.total_nodes), 3))
        check(lib().pdg_disc_node_coords(self._h, _dp(xyz)))
        return xyz

    def wedge_ops(self, w):
        nt, nq = self.info.nt, self.info.nq
        L = np.zeros(nt * nt)
        Q = np.zeros(3 * nq * nt)
        s = np.zeros(18)
        check(lib().pdg_disc_wedge_ops(self._h, w, _dp(L), _dp(Q), _dp(s)))
        return L.reshape(nt, nt).T.copy(), Q.reshape(3, nq, nt).transpose(0, 2, 1).copy(), s

    def device(self, flags=0, device=0):
        """The device context (created once, like the host shim's DeviceHandle)."""
        if self._ctx is None or self._ctx.flags != flags:
            if self._ctx is not None:
                self._ctx.close()
            self._ctx = DeviceContext(self, device=device, flags=flags)
        return self._ctx


DISC_ARRAY_FIELDS = ("vertices", "wedges", "tets", "media", "wedge_geom", "tet_geom", "tri_lift", "quad_lift", "txJ",
                     "tyJ", "wedge_scalars", "tet_scalars", "face_nbr", "face_tau", "face_normal", "face_my_nodes",
                     "face_nbr_nodes")


def export_arrays(disc: "Discretization") -> dict:
    """The flattened per-element arrays of pdg_disc_arrays (the reference's
    Discretization members, solver.hpp:29-59) of an existing discretization."""
    info = disc.info
    N, nq, nt = info.degree, info.nq, info.nt
    nw, ntet, nf = int(info.num_wedges), int(info.num_tets), int(info.num_faces)
    max_nfp = max(nq * nq, nt)
    cnt = np.zeros(3, dtype=np.int64)
    check(lib().pdg_disc_mesh_export(disc.handle, cnt.ctypes.data_as(capi.I64P), None, None, None, None))
    a = {"degree": N, "qmode": {0: 0, 1: 1, 2: 2}[info.mass_mode], "flux_mode": info.flux_mode,
         "vertices": np.zeros((int(cnt[0]), 3)), "wedges": np.zeros((nw, 6), np.int32),
         "tets": np.zeros((ntet, 4), np.int32), "media": np.zeros((nw + ntet, 2)),
         "wedge_geom": np.zeros((nw, 11)), "tet_geom": np.zeros((ntet, 3)), "txJ": np.zeros((nw, nq)),
         "tyJ": np.zeros((nw, nq)), "wedge_scalars": np.zeros((nw, 7)), "tet_scalars": np.zeros((ntet, 13)),
         "face_nbr": np.zeros(nf, np.int32), "face_tau": np.zeros((nf, 2)), "face_normal": np.zeros((nf, 3)),
         "face_nbr_nodes": np.zeros((nf, max_nfp), np.int32)}
    check(lib().pdg_disc_mesh_export(disc.handle, None, _dp(a["vertices"]), _ip(a["wedges"]), _ip(a["tets"]),
                                     _dp(a["media"])))
    check(lib().pdg_disc_export_arrays(disc.handle, _dp(a["wedge_geom"]), _dp(a["tet_geom"]), _dp(a["txJ"]),
                                       _dp(a["tyJ"]), _dp(a["wedge_scalars"]), _dp(a["tet_scalars"]),
                                       _ip(a["face_nbr"]), _dp(a["face_tau"]), _dp(a["face_normal"]),
                                       _ip(a["face_nbr_nodes"])))
    if nw and info.mass_mode != 2:
        a["tri_lift"] = np.zeros((nw, nt * nt))
        a["quad_lift"] = np.zeros((nw, 3 * nq * nt))
        for w in range(nw):
            check(lib().pdg_disc_wedge_ops(disc.handle, w, _dp(a["tri_lift"][w]), _dp(a["quad_lift"][w]), None))
    return a


def discretization_from_arrays(arrays: dict, mesh=None) -> "Discretization":
    """pdg_disc_from_arrays: a Discretization from a caller's flattened arrays
    (e.g. the reference's own Eigen-built operators)."""
    s = capi.DiscArrays()
    s.degree = int(arrays["degree"])
    s.qmode = int(arrays.get("qmode", 0))
    s.flux_mode = int(arrays.get("flux_mode", 0))
    s.tau_p = float(arrays.get("tau_p", 0.0))
    s.tau_u = float(arrays.get("tau_u", 0.0))
    keep = {}
    for name in DISC_ARRAY_FIELDS:
        v = arrays.get(name)
        if v is None:
            continue
        is_int = name in ("wedges", "tets", "face_nbr", "face_my_nodes", "face_nbr_nodes")
        arr = np.ascontiguousarray(v, dtype=np.int32 if is_int else np.float64)
        keep[name] = arr
        setattr(s, name, arr.ctypes.data_as(capi.IP if is_int else capi.DP))
    s.num_vertices = len(keep["vertices"])
    s.num_wedges = len(keep["wedges"]) if "wedges" in keep else 0
    s.num_tets = len(keep["tets"]) if "tets" in keep else 0
    out = C.c_void_p()
    check(lib().pdg_disc_from_arrays(C.byref(s), C.byref(out)))
    return Discretization(out.value, mesh)


def build_discretization(mesh: HybridMesh, degree: int, flux="upwind", tau_p=0.0, tau_u=0.0,
                         mass="exact", threads=0, host_lifts=True) -> Discretization:
    """build_discretization (solver.hpp:61-63).  mass: "exact" | "lumped" | "wadg".
    host_lifts=False (wadg only) skips the per-wedge exact lifts on the host too."""
    out = C.c_void_p()
    flags = 0 if host_lifts else 1  # PDG_DISC_NO_HOST_LIFTS
    check(lib().pdg_disc_build_ex(mesh.handle, degree, capi.FLUX[flux], tau_p, tau_u, capi.MASS[mass],
                                  threads, flags, C.byref(out)))
    return Discretization(out.value, mesh)


class DeviceContext:
    """pdg_ctx: the discretization resident on one GPU (include/prismdg_b200.h)."""

    def __init__(self, disc: Discretization, device=0, flags=0):
        self.disc = disc
        self.flags = flags
        out = C.c_void_p()
        check(lib().pdg_create(disc.handle, device, flags, C.byref(out)))
        self._h = out

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().pdg_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    @staticmethod
    def _ptr(a):
        """(pointer, on_device) for numpy arrays or CUDA torch tensors."""
        if hasattr(a, "data_ptr"):
            return C.c_void_p(a.data_ptr()), int(bool(a.is_cuda))
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data), 0

    def set_state(self, u):
        p, dev = self._ptr(u)
        check(lib().pdg_set_state(self._h, p, dev))

    def get_state(self, out=None):
        if out is None:
            out = np.zeros(self.disc.total_dofs)
        p, dev = self._ptr(out)
        check(lib().pdg_get_state(self._h, p, dev))
        return out

    def rhs(self, u, out=None):
        if out is None:
            out = np.zeros(self.disc.total_dofs)
        pu, du = self._ptr(u)
        po, do = self._ptr(out)
        assert du == do
        check(lib().pdg_rhs(self._h, pu, po, du))
        return out

    def phase(self, which: str):
        check(getattr(lib(), f"pdg_{which}")(self._h))

    def set_rhs(self, r):
        p, dev = self._ptr(r)
        check(lib().pdg_set_rhs(self._h, p, dev))

    def get_rhs(self, out=None):
        if out is None:
            out = np.zeros(self.disc.total_dofs)
        p, dev = self._ptr(out)
        check(lib().pdg_get_rhs(self._h, p, dev))
        return out

    def step(self, dt, nsteps=1, t=0.0, integrator="lserk4"):
        """TimeStepper::step x nsteps on the resident state (lserk4 or ab3, solver.cpp:536-581);
        integrator="mrab": nsteps multi-rate AB3 macro steps of fine step dt."""
        tt = C.c_double(t)
        fn = {"ab3": lib().pdg_step_ab3, "mrab": lib().pdg_step_mrab}.get(integrator, lib().pdg_step_lserk)
        check(fn(self._h, dt, nsteps, C.byref(tt)))
        return tt.value

    def energy(self):
        e = C.c_double()
        check(lib().pdg_energy(self._h, C.byref(e)))
        return e.value

    def check_finite(self):
        e = C.c_int64()
        check(lib().pdg_check_finite(self._h, C.byref(e)))
        return int(e.value)

    def synchronize(self):
        check(lib().pdg_synchronize(self._h))

    def stream(self):
        return lib().pdg_stream(self._h)

    def kernel_times(self, reset=False):
        wms, tms = C.c_double(), C.c_double()
        wl, tl = C.c_int64(), C.c_int64()
        check(lib().pdg_kernel_times(self._h, C.byref(wms), C.byref(wl), C.byref(tms), C.byref(tl), int(reset)))
        return {"wedge_ms": wms.value, "wedge_launches": wl.value, "tet_ms": tms.value, "tet_launches": tl.value}

    def stage_bytes(self):
        wb, tb = C.c_double(), C.c_double()
        check(lib().pdg_stage_bytes(self._h, C.byref(wb), C.byref(tb)))
        return wb.value, tb.value

    def mrab_levels(self):
        """(rate level of every reference element, number of levels)"""
        lev = np.zeros(self.disc.num_elements(), dtype=np.int32)
        n = C.c_int()
        check(lib().pdg_mrab_levels(self._h, _ip(lev), C.byref(n)))
        return lev, n.value

    def launch_info(self):
        """last wedge / tet stage launch: {launched, teams, tickets, per_ticket} each"""
        out = np.zeros(8, dtype=np.int64)
        check(lib().pdg_launch_info(self._h, out.ctypes.data_as(capi.I64P)))
        keys = ("launched", "teams", "tickets", "per_ticket")
        return {"wedge": dict(zip(keys, out[:4].tolist())), "tet": dict(zip(keys, out[4:].tolist()))}

    def device_order(self):
        out = np.zeros(self.disc.num_elements(), dtype=np.int64)
        check(lib().pdg_device_order(self._h, out.ctypes.data_as(capi.I64P)))
        return out


# ---------------------------------------------------------------- solver API
def compute_rhs(disc: Discretization, u: np.ndarray) -> np.ndarray:
    """compute_rhs (solver.hpp:67) on the GPU."""
    return disc.device().rhs(np.ascontiguousarray(u, dtype=np.float64))


def compute_energy(disc: Discretization, u: np.ndarray) -> float:
    ctx = disc.device()
    ctx.set_state(np.ascontiguousarray(u, dtype=np.float64))
    return ctx.energy()


def estimate_dt(disc: Discretization, cfl: float) -> float:
    out = C.c_double()
    check(lib().pdg_disc_estimate_dt(disc.handle, cfl, C.byref(out)))
    return out.value


@dataclass
class SolutionState:
    u: np.ndarray
    time: float = 0.0


def make_initial_state(disc: Discretization, kind="standing_wave", params=None, t0=0.0) -> SolutionState:
    k = {"standing_wave": 0, "gaussian": 1}[kind]
    if params is None:
        params = [1.0, 1.0] if k == 0 else [0.25, 0.0, 0.0, 0.0]
    par = np.ascontiguousarray(params, dtype=np.float64)
    u = np.zeros(disc.total_dofs)
    check(lib().pdg_disc_initial_state(disc.handle, k, _dp(par), t0, _dp(u)))
    return SolutionState(u=u, time=t0)


def l2_error(disc: Discretization, u: np.ndarray, time: float) -> float:
    """l2_error against the standing-wave pressure (analysis.cpp:53-91)."""
    out = C.c_double()
    uu = np.ascontiguousarray(u, dtype=np.float64)
    check(lib().pdg_disc_l2_error(disc.handle, _dp(uu), time, C.byref(out)))
    return out.value


@dataclass
class RunOptions:
    """solver.hpp:126-137"""

    final_time: float = 1.0
    cfl: float = 0.5
    fixed_dt: float = 0.0
    energy_interval: float = 0.0
    watchdog_every: int = 50
    blowup_factor: float = 10.0
    integrator: str = "lserk4"  # IntegratorKind: "lserk4" | "ab3" | "mrab" (context with multi-rate levels)
    snapshot_interval: float = 0.0  # 0: no snapshots
    snapshot_cb: object = None  # callable(u: np.ndarray (copy), time: float, index: int)
    mrab_levels: int = 3  # integrator="mrab": up to this many extra rate levels (PDG_CTX_MRAB_LEVELS)


@dataclass
class RunResult:
    steps: int
    dt: float
    final_time: float
    initial_energy: float
    final_energy: float
    max_energy_increase: float
    energy_log: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))


def run_simulation(disc: Discretization, state: SolutionState, opts: RunOptions, max_log=100000) -> RunResult:
    """run_simulation (solver.hpp:148-149), state resident on the GPU for the run."""
    n = int(disc.total_dofs)
    if opts.snapshot_cb is not None and opts.snapshot_interval > 0.0:
        user_cb = opts.snapshot_cb

        def _cb(u_ptr, t, index, _user):
            user_cb(np.ctypeslib.as_array(u_ptr, shape=(n,)).copy(), float(t), int(index))

        cb = capi.SNAPSHOT_CB(_cb)
    else:
        cb = capi.SNAPSHOT_CB()
    o = capi.RunOptions(opts.final_time, opts.cfl, opts.fixed_dt, opts.energy_interval,
                        opts.watchdog_every, opts.blowup_factor, {"ab3": 1, "mrab": 2}.get(opts.integrator, 0),
                        opts.snapshot_interval, cb, None)
    r = capi.RunResult()
    log = np.zeros(2 * max_log)
    t = C.c_double(state.time)
    state.u = np.ascontiguousarray(state.u, dtype=np.float64)
    try:
        flags = capi.CTX_MRAB_LEVELS(opts.mrab_levels) if opts.integrator == "mrab" else 0
        check(lib().pdg_run_simulation(disc.device(flags=flags).handle, _dp(state.u), C.byref(t), C.byref(o), C.byref(r),
                                       _dp(log), max_log))
    finally:
        state.time = t.value  # on a watchdog failure: the failure time, like the reference
    n = min(r.num_logged, max_log)
    return RunResult(r.steps, r.dt, r.final_time, r.initial_energy, r.final_energy, r.max_energy_increase,
                     log[: 2 * n].reshape(n, 2))


def fit_rate(h, err):
    h = np.asarray(h, dtype=float)[-3:]
    e = np.asarray(err, dtype=float)[-3:]
    return float(np.polyfit(np.log(h), np.log(e), 1)[0])


def assemble_global(disc: Discretization) -> np.ndarray:
    """assemble_global (analysis.cpp:12-40): dense RHS operator, n x n (numpy,
    A[i, j] = d rhs_i / d u_j), built on the GPU from colored unit probes."""
    n = int(disc.total_dofs)
    a = np.zeros((n, n), order="F")
    check(lib().pdg_assemble_operator(disc.device().handle, a.ctypes.data_as(capi.DP)))
    return a


def spectrum(A: np.ndarray) -> np.ndarray:
    """spectrum (analysis.cpp:42-52): eigenvalues sorted by real then imaginary part."""
    ev = np.linalg.eigvals(A)
    return ev[np.lexsort((ev.imag, ev.real))]


def write_vtk_snapshot(disc: Discretization, u, path: str) -> None:
    """write_vtk_snapshot (snapshot.cpp:68-139): legacy ASCII VTK of the nodal state."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    check(lib().pdg_write_vtk(disc.handle, _dp(u), path.encode()))
