"""ctypes binding of the CPU oracle (oracle/, TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "build", "liboracle.so")
TEST_BIN = os.path.join(ORACLE_DIR, "build", "test_host")

_lib = None


def ensure_built():
    if not (os.path.exists(LIB) and os.path.exists(TEST_BIN)):
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
        h.orc_run.argtypes = [vp, dp, dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, dp]
        h.orc_gll_newton.argtypes = [C.c_int, dp, dp]
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
