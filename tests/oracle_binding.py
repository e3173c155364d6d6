"""ctypes binding of the CPU oracle (oracle/, TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this.
This module never imports the product package: liboracle.so carries its own
copy of the host setup code, so bench.py's CPU arm (``layered_disc`` below)
runs without libprismdg_b200.so.  ``PDG_ORACLE_LIB`` selects another build of
the same sources (bench.py builds one with -march=native on the host it runs on).
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.environ.get("PDG_ORACLE_LIB") or os.path.join(ORACLE_DIR, "build", "liboracle.so")
TEST_BIN = os.path.join(ORACLE_DIR, "build", "test_host")

_lib = None


def ensure_built():
    if not os.path.exists(LIB) or (LIB.startswith(os.path.join(ORACLE_DIR, "build", "")) and
                                   not os.path.exists(TEST_BIN)):
        subprocess.run(["make", "-C", ORACLE_DIR, "-j8"], check=True, capture_output=True)


def lib():
    global _lib
    if _lib is None:
        ensure_built()
        h = C.CDLL(LIB)
        dp, vp = C.POINTER(C.c_double), C.c_void_p
        h.orc_last_error.restype = C.c_char_p
        h.orc_rhs.argtypes = [vp, dp, dp, C.c_int]
        h.orc_phase.argtypes = [vp, C.c_int, dp, dp]
        h.orc_lserk.argtypes = [vp, dp, C.c_double, C.c_int, C.c_int, C.c_int]
        h.orc_energy.argtypes = [vp, dp, C.c_int, dp]
        h.orc_ab3.argtypes = [vp, dp, C.c_double, C.c_int, C.c_int]
        h.orc_mrab.argtypes = [vp, dp, C.POINTER(C.c_int), C.c_int, C.c_double, C.c_int, C.c_int]
        h.orc_run.argtypes = [vp, dp, dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, dp]
        h.orc_gll_newton.argtypes = [C.c_int, dp, dp]
        ip = C.POINTER(C.c_int)
        h.orc_disc_stack_layers.argtypes = [C.c_int, dp, C.c_int, ip, C.c_int, dp, dp, ip, dp, C.c_int, C.c_int,
                                            C.POINTER(vp)]
        h.orc_disc_counts.argtypes = [vp, C.POINTER(C.c_longlong)]
        h.orc_disc_gaussian.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_double, dp]
        h.orc_disc_estimate_dt.argtypes = [vp, C.c_double, dp]
        h.orc_disc_free.argtypes = [vp]
        h.orc_disc_free.restype = None
        _lib = h
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ok(st):
    if st != 0:
        raise RuntimeError(lib().orc_last_error().decode())


def rhs(disc, u, threads=4):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    _ok(lib().orc_rhs(disc.handle, _dp(u), _dp(out), threads))
    return out


def phase(disc, which, u, rhs_inout):
    u = np.ascontiguousarray(u, dtype=np.float64)
    _ok(lib().orc_phase(disc.handle, which, _dp(u), _dp(rhs_inout)))
    return rhs_inout


def lserk(disc, u, dt, nsteps, threads=4, parallel_update=True):
    u = np.array(u, dtype=np.float64, copy=True)
    _ok(lib().orc_lserk(disc.handle, _dp(u), dt, nsteps, threads, int(parallel_update)))
    return u


def ab3(disc, u, dt, nsteps, threads=4):
    u = np.array(u, dtype=np.float64, copy=True)
    _ok(lib().orc_ab3(disc.handle, _dp(u), dt, nsteps, threads))
    return u


def mrab(disc, u, level, nlev, dt, nmacro, threads=4):
    """multi-rate AB3 (pdg_step_mrab's algorithm): level[e] = rate level of element e"""
    u = np.array(u, dtype=np.float64, copy=True)
    lev = np.ascontiguousarray(level, dtype=np.int32)
    _ok(lib().orc_mrab(disc.handle, _dp(u), lev.ctypes.data_as(C.POINTER(C.c_int)), nlev, dt, nmacro, threads))
    return u


def energy(disc, u, threads=4):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = C.c_double()
    _ok(lib().orc_energy(disc.handle, _dp(u), threads, C.byref(out)))
    return out.value


def run(disc, u, time, final_time, cfl=0.5, fixed_dt=0.0, energy_interval=0.0, threads=4):
    u = np.array(u, dtype=np.float64, copy=True)
    t = C.c_double(time)
    out = np.zeros(7)
    _ok(lib().orc_run(disc.handle, _dp(u), C.byref(t), final_time, cfl, fixed_dt, energy_interval, threads,
                      _dp(out)))
    keys = ["steps", "dt", "final_time", "initial_energy", "final_energy", "max_energy_increase", "stable"]
    return u, t.value, dict(zip(keys, out.tolist()))


# ---- the oracle's own discretizations (no product library) ------------------
def structured_surface(n):
    """The 'layers' mesh-kind surface of config.cpp:232-243 (as solver.structured_surface)."""
    i, j = np.meshgrid(np.arange(n + 1), np.arange(n + 1))
    xy = np.stack([-1.0 + 2.0 * i.ravel() / n, -1.0 + 2.0 * j.ravel() / n], axis=1)
    a = (np.arange(n)[:, None] * (n + 1) + np.arange(n)[None, :]).ravel()
    tris = np.stack([np.stack([a, a + 1, a + n + 2], 1), np.stack([a, a + n + 2, a + n + 1], 1)], 1).reshape(-1, 3)
    return np.ascontiguousarray(xy), np.ascontiguousarray(tris, dtype=np.int32)


class OracleDisc:
    """A prismdg::Discretization built inside liboracle.so (exact mass, upwind)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        c = (C.c_longlong * 3)()
        _ok(lib().orc_disc_counts(self._h, c))
        self.total_dofs, self.num_wedges, self.num_tets = int(c[0]), int(c[1]), int(c[2])

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().orc_disc_free(self._h)
            self._h = C.c_void_p(None)

    def gaussian(self, width=0.25, center=(0.0, 0.0, 0.0)):
        u = np.zeros(self.total_dofs)
        _ok(lib().orc_disc_gaussian(self._h, width, center[0], center[1], center[2], _dp(u)))
        return u

    def estimate_dt(self, cfl=0.5):
        out = C.c_double()
        _ok(lib().orc_disc_estimate_dt(self._h, cfl, C.byref(out)))
        return out.value


def layered_disc(surface_n, interfaces, sublayers, media, degree, threads=4):
    """stack_layers on the structured surface with flat interfaces (the bench mesh)."""
    xy, tris = structured_surface(surface_n)
    nv, nl = xy.shape[0], len(sublayers)
    zb = np.ascontiguousarray(np.stack([np.full(nv, float(interfaces[k])) for k in range(nl)]))
    zt = np.ascontiguousarray(np.stack([np.full(nv, float(interfaces[k + 1])) for k in range(nl)]))
    sub = np.ascontiguousarray(sublayers, dtype=np.int32)
    med = np.ascontiguousarray(np.array(media, dtype=np.float64).reshape(nl, 2))
    ip = C.POINTER(C.c_int)
    out = C.c_void_p()
    _ok(lib().orc_disc_stack_layers(nv, _dp(xy), tris.shape[0], tris.ctypes.data_as(ip), nl, _dp(zb), _dp(zt),
                                    sub.ctypes.data_as(ip), _dp(med), degree, threads, C.byref(out)))
    return OracleDisc(out.value)
