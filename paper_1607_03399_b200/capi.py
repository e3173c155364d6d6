"""ctypes binding of the C ABI in include/prismdg_b200.h.

The shared library is built in-tree (paper_1607_03399_b200/_lib) by
``__graft_entry__.build()``.  Loading fails loudly if it is missing: there is
no Python or CPU fallback for the device path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libprismdg_b200.so")
# development only: load an alternative in-tree build (kernel configuration sweeps)
LIB_PATH = os.environ.get("PDG_LIB_PATH", LIB_PATH)
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "prismdg_b200.h")

PDG_OK = 0
PDG_ERR_CONFIG = 2
PDG_ERR_NUMERICAL = 3
PDG_ERR_MESH = 4
PDG_ERR_CUDA = 5
PDG_ERR_ANALYSIS = 6

FLUX = {"upwind": 0, "central": 1, "custom": 2}
MASS = {"exact": 0, "lumped": 1, "wadg": 2}
CTX_NATIVE_ORDER = 1
CTX_TIMING = 2


def CTX_MRAB_LEVELS(levels: int) -> int:
    """PDG_CTX_MRAB_LEVELS(L): up to L+1 multi-rate levels"""
    return (levels & 15) << 8


class PdgError(RuntimeError):
    """Base class; subclasses mirror the reference exception taxonomy (types.hpp:14-34)."""

    status = -1


class ConfigError(PdgError):
    status = PDG_ERR_CONFIG


class NumericalError(PdgError):
    status = PDG_ERR_NUMERICAL


class MeshError(PdgError):
    status = PDG_ERR_MESH


class DeviceError(PdgError):
    status = PDG_ERR_CUDA


class AnalysisError(PdgError):
    status = PDG_ERR_ANALYSIS


_ERRORS = {c.status: c for c in (ConfigError, NumericalError, MeshError, DeviceError, AnalysisError)}


class DiscInfo(C.Structure):
    _fields_ = [
        ("degree", C.c_int), ("nq", C.c_int), ("nt", C.c_int), ("np_wedge", C.c_int), ("np_tet", C.c_int),
        ("num_wedges", C.c_int64), ("num_tets", C.c_int64), ("total_dofs", C.c_int64),
        ("total_nodes", C.c_int64), ("num_faces", C.c_int64),
        ("num_perms", C.c_int), ("num_interior_pairs", C.c_int), ("num_boundary_faces", C.c_int),
        ("flux_mode", C.c_int), ("mass_mode", C.c_int),
    ]


class DiscArrays(C.Structure):
    """pdg_disc_arrays: the reference's Discretization flattened (solver.hpp:29-59)."""
    _fields_ = [
        ("degree", C.c_int), ("qmode", C.c_int), ("flux_mode", C.c_int), ("tau_p", C.c_double),
        ("tau_u", C.c_double), ("num_vertices", C.c_int64), ("num_wedges", C.c_int64), ("num_tets", C.c_int64),
        ("vertices", C.POINTER(C.c_double)), ("wedges", C.POINTER(C.c_int)), ("tets", C.POINTER(C.c_int)),
        ("media", C.POINTER(C.c_double)), ("wedge_geom", C.POINTER(C.c_double)),
        ("tet_geom", C.POINTER(C.c_double)), ("tri_lift", C.POINTER(C.c_double)),
        ("quad_lift", C.POINTER(C.c_double)), ("txJ", C.POINTER(C.c_double)), ("tyJ", C.POINTER(C.c_double)),
        ("wedge_scalars", C.POINTER(C.c_double)), ("tet_scalars", C.POINTER(C.c_double)),
        ("face_nbr", C.POINTER(C.c_int)), ("face_tau", C.POINTER(C.c_double)),
        ("face_normal", C.POINTER(C.c_double)), ("face_my_nodes", C.POINTER(C.c_int)),
        ("face_nbr_nodes", C.POINTER(C.c_int)),
    ]


SNAPSHOT_CB = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_double, C.c_int, C.c_void_p)


class RunOptions(C.Structure):
    _fields_ = [
        ("final_time", C.c_double), ("cfl", C.c_double), ("fixed_dt", C.c_double),
        ("energy_interval", C.c_double), ("watchdog_every", C.c_int), ("blowup_factor", C.c_double),
        ("integrator", C.c_int), ("snapshot_interval", C.c_double), ("snapshot_cb", SNAPSHOT_CB),
        ("snapshot_user", C.c_void_p),
    ]


class RunResult(C.Structure):
    _fields_ = [
        ("steps", C.c_int), ("dt", C.c_double), ("final_time", C.c_double),
        ("initial_energy", C.c_double), ("final_energy", C.c_double),
        ("max_energy_increase", C.c_double), ("num_logged", C.c_int),
    ]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)
I64P = C.POINTER(C.c_int64)

# name -> (restype, argtypes)
SIGNATURES = {
    "pdg_last_error": (C.c_char_p, []),
    "pdg_abi_version": (C.c_int, []),
    "pdg_mesh_structured_hybrid_box": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, DP, DP, PP]),
    "pdg_mesh_unstructured_wedge_box": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_uint64, DP, PP]),
    "pdg_mesh_arnold_wedge_box": (C.c_int, [C.c_int, C.c_double, DP, PP]),
    "pdg_mesh_stack_layers": (C.c_int, [C.c_int, DP, C.c_int, IP, C.c_int, DP, DP, IP, DP, PP]),
    "pdg_mesh_perturb_vertically": (C.c_int, [P, C.c_double, C.c_uint64, PP]),
    "pdg_mesh_family": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double, C.c_double, PP]),
    "pdg_mesh_spectra": (C.c_int, [C.c_uint64, C.c_double, PP]),
    "pdg_mesh_from_arrays": (C.c_int, [C.c_int64, DP, C.c_int64, IP, C.c_int64, IP, DP, PP]),
    "pdg_mesh_load": (C.c_int, [C.c_char_p, PP]),
    "pdg_mesh_save": (C.c_int, [P, C.c_char_p]),
    "pdg_mesh_counts": (C.c_int, [P, I64P]),
    "pdg_mesh_export": (C.c_int, [P, DP, IP, IP, DP]),
    "pdg_mesh_volume": (C.c_int, [P, DP]),
    "pdg_mesh_free": (None, [P]),
    "pdg_disc_build": (C.c_int, [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, PP]),
    "pdg_disc_build_ex": (C.c_int, [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                    PP]),
    "pdg_disc_get_info": (C.c_int, [P, C.POINTER(DiscInfo)]),
    "pdg_disc_elem_offset": (C.c_int, [P, I64P]),
    "pdg_disc_face_table": (C.c_int, [P, IP, IP, IP]),
    "pdg_disc_perm": (C.c_int, [P, C.c_int, IP, IP]),
    "pdg_disc_face_nodes": (C.c_int, [P, C.c_int64, C.c_int, IP, IP, IP]),
    "pdg_disc_face_phys": (C.c_int, [P, DP, DP, DP]),
    "pdg_disc_node_coords": (C.c_int, [P, DP]),
    "pdg_disc_initial_state": (C.c_int, [P, C.c_int, DP, C.c_double, DP]),
    "pdg_disc_estimate_dt": (C.c_int, [P, C.c_double, DP]),
    "pdg_disc_l2_error": (C.c_int, [P, DP, C.c_double, DP]),
    "pdg_disc_wedge_ops": (C.c_int, [P, C.c_int64, DP, DP, DP]),
    "pdg_disc_free": (None, [P]),
    "pdg_disc_from_arrays": (C.c_int, [C.POINTER(DiscArrays), PP]),
    "pdg_disc_export_arrays": (C.c_int, [P, DP, DP, DP, DP, DP, DP, IP, DP, DP, IP]),
    "pdg_disc_mesh_export": (C.c_int, [P, I64P, DP, IP, IP, DP]),
    "pdg_create": (C.c_int, [P, C.c_int, C.c_int, PP]),
    "pdg_destroy": (None, [P]),
    "pdg_set_state": (C.c_int, [P, P, C.c_int]),
    "pdg_get_state": (C.c_int, [P, P, C.c_int]),
    "pdg_rhs": (C.c_int, [P, P, P, C.c_int]),
    "pdg_wedge_volume": (C.c_int, [P]),
    "pdg_wedge_surface": (C.c_int, [P]),
    "pdg_tet_volume": (C.c_int, [P]),
    "pdg_tet_surface": (C.c_int, [P]),
    "pdg_get_rhs": (C.c_int, [P, P, C.c_int]),
    "pdg_set_rhs": (C.c_int, [P, P, C.c_int]),
    "pdg_step_lserk": (C.c_int, [P, C.c_double, C.c_int, DP]),
    "pdg_step_ab3": (C.c_int, [P, C.c_double, C.c_int, DP]),
    "pdg_step_mrab": (C.c_int, [P, C.c_double, C.c_int, DP]),
    "pdg_mrab_levels": (C.c_int, [P, IP, IP]),
    "pdg_energy": (C.c_int, [P, DP]),
    "pdg_check_finite": (C.c_int, [P, I64P]),
    "pdg_synchronize": (C.c_int, [P]),
    "pdg_stream": (C.c_void_p, [P]),
    "pdg_kernel_times": (C.c_int, [P, DP, I64P, DP, I64P, C.c_int]),
    "pdg_stage_bytes": (C.c_int, [P, DP, DP]),
    "pdg_device_order": (C.c_int, [P, I64P]),
    "pdg_launch_info": (C.c_int, [P, I64P]),
    "pdg_run_simulation": (C.c_int, [P, DP, DP, C.POINTER(RunOptions), C.POINTER(RunResult), DP, C.c_int]),
    "pdg_create_partitioned": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(C.c_ubyte), PP]),
    "pdg_active_counts": (C.c_int, [P, I64P]),
    "pdg_step_stage": (C.c_int, [P, C.c_double, C.c_int]),
    "pdg_pack_states": (C.c_int, [P, P, C.c_int64, P]),
    "pdg_unpack_states": (C.c_int, [P, P, C.c_int64, P]),
    "pdg_partition_counts": (C.c_int, [P, I64P]),
    "pdg_assemble_operator": (C.c_int, [P, DP]),
    "pdg_write_vtk": (C.c_int, [P, DP, C.c_char_p]),
    "pdg_step_stage_part": (C.c_int, [P, C.c_double, C.c_int, C.c_int]),
    "pdg_trace_offsets": (C.c_int, [P, C.c_int64, I64P, IP, I64P, I64P]),
    "pdg_gather_values": (C.c_int, [P, P, C.c_int64, P, P]),
    "pdg_scatter_values": (C.c_int, [P, P, C.c_int64, P, P]),
}


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Every function the public header declares (used by the ABI tests)."""
    with open(path) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(pdg_[a-z0-9_]+)\s*\(", text)))


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != PDG_OK:
        msg = lib().pdg_last_error().decode()
        raise _ERRORS.get(status, PdgError)(msg)
