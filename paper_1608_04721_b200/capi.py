"""ctypes mirror of include/apbf_gpu.h and the loader of the CUDA library.

The product path is ``libapbf_gpu.so`` (built in-tree by ``_build.py`` from
``csrc/*.cu`` for sm_100a).  There is no fallback: if the library is missing
or cannot be loaded, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# APBF_LIB names an alternative in-tree build (A/B of compile-time variants)
LIB_PATH = os.path.join(HERE, os.environ.get("APBF_LIB", "libapbf_gpu.so"))

APBF_OK = 0
APBF_ERR_INVALID_ARGUMENT = 1
APBF_ERR_RUNTIME = 2
APBF_ERR_NUMERICAL = 3
APBF_ERR_CUDA = 4
APBF_ERR_OUT_OF_RANGE = 5

MODE_PBF, MODE_APBF = 0, 1
LOD_DTC, LOD_DTVS = 0, 1
SDF_HALF_SPACE, SDF_SPHERE, SDF_BOX, SDF_CONE = 0, 1, 2, 3


class apbf_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("particle", C.c_int32), ("pass_", C.c_char * 32),
                ("message", C.c_char * 224)]


class apbf_solver_config(C.Structure):
    _fields_ = [("dt_frame", C.c_float), ("substeps", C.c_int32), ("n_min", C.c_int32),
                ("n_max", C.c_int32), ("rest_density", C.c_float), ("h", C.c_float),
                ("epsilon", C.c_float), ("gravity", C.c_float * 3),
                ("stab_iterations", C.c_int32), ("stab_threshold", C.c_int32),
                ("particle_radius", C.c_float), ("mode", C.c_int32),
                ("velocity_cap", C.c_float), ("inactive_lambda_zero", C.c_int32),
                ("deterministic", C.c_int32), ("record_residuals", C.c_int32),
                ("xsph_viscosity", C.c_float), ("vorticity_epsilon", C.c_float)]


class apbf_sdf_primitive(C.Structure):
    _fields_ = [("kind", C.c_int32), ("interior", C.c_int32), ("p", C.c_float * 3),
                ("q", C.c_float * 3), ("a", C.c_float), ("b", C.c_float)]


class apbf_camera(C.Structure):
    _fields_ = [("eye", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("vertical_fov", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("near_clip", C.c_float)]


class apbf_lod_config(C.Structure):
    _fields_ = [("model", C.c_int32), ("d_min", C.c_float), ("d_max", C.c_float),
                ("n_min", C.c_int32), ("n_max", C.c_int32), ("auto_range", C.c_int32)]


class apbf_frame_stats(C.Structure):
    _fields_ = [("frame", C.c_int32), ("n_residuals", C.c_int32), ("wall_ms", C.c_double),
                ("avg_density_pct", C.c_double), ("min_density_pct", C.c_double),
                ("max_density_pct", C.c_double), ("total_iterations", C.c_int64),
                ("contacts", C.c_int64), ("residuals", C.POINTER(C.c_double)),
                ("residuals_capacity", C.c_int32), ("reserved", C.c_int32)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32)

_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_ep = C.POINTER(apbf_error)

# name -> (restype, argtypes); every symbol declared in include/apbf_gpu.h.
SIGNATURES = {
    "apbf_gpu_abi_version": (C.c_int32, []),
    "apbf_gpu_device_count": (C.c_int32, []),
    "apbf_gpu_solver_create": (C.c_int32, [C.POINTER(apbf_solver_config),
                                           C.POINTER(apbf_sdf_primitive), C.c_int32, C.c_float,
                                           C.c_int32, C.POINTER(C.c_void_p), _ep]),
    "apbf_gpu_solver_destroy": (None, [C.c_void_p]),
    "apbf_gpu_set_state": (C.c_int32, [C.c_void_p, C.c_int32, _fp, _fp, _fp, _fp, _fp, _fp, _ip,
                                       _ep]),
    "apbf_gpu_get_state": (C.c_int32, [C.c_void_p, _fp, _fp, _fp, _fp, _fp, _fp, _ip, _ep]),
    "apbf_gpu_particle_count": (C.c_int32, [C.c_void_p]),
    "apbf_gpu_stream": (C.c_void_p, [C.c_void_p]),
    "apbf_gpu_step_frame": (C.c_int32, [C.c_void_p, C.POINTER(apbf_camera),
                                        C.POINTER(apbf_lod_config), C.c_int32,
                                        C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_step_frame_with_levels": (C.c_int32, [C.c_void_p, C.c_int32,
                                                    C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_set_iteration_observer": (C.c_int32, [C.c_void_p, OBSERVER, C.c_void_p]),
    "apbf_gpu_set_frame_metrics": (C.c_int32, [C.c_void_p, C.c_int32]),
    "apbf_gpu_set_phase_timing": (C.c_int32, [C.c_void_p, C.c_int32]),
    "apbf_gpu_last_phase_ms": (C.c_int32, [C.c_void_p, _fp]),
    "apbf_gpu_last_neighbor_stats": (C.c_int32, [C.c_void_p, _lp, _lp]),
    "apbf_gpu_set_kernel_timing": (C.c_int32, [C.c_void_p, C.c_int32, _ep]),
    "apbf_gpu_kernel_times": (C.c_int32, [C.c_void_p, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), _lp, _lp]),
    "apbf_gpu_launch_count": (C.c_uint64, []),
    "apbf_gpu_group_create": (C.c_int32, [C.POINTER(apbf_solver_config),
                                          C.POINTER(apbf_sdf_primitive), C.c_int32, C.c_float,
                                          C.c_int32, _ip, C.POINTER(C.c_void_p), _ep]),
    "apbf_gpu_group_destroy": (None, [C.c_void_p]),
    "apbf_gpu_group_size": (C.c_int32, [C.c_void_p]),
    "apbf_gpu_group_set_state": (C.c_int32, [C.c_void_p, C.c_int32, _fp, _fp, _fp, _fp, _fp, _fp,
                                             _ip, _ep]),
    "apbf_gpu_group_get_state": (C.c_int32, [C.c_void_p, _fp, _fp, _fp, _fp, _fp, _fp, _ip, _ep]),
    "apbf_gpu_group_particle_counts": (C.c_int32, [C.c_void_p, _ip]),
    "apbf_gpu_group_step_frame": (C.c_int32, [C.c_void_p, C.POINTER(apbf_camera),
                                              C.POINTER(apbf_lod_config), C.c_int32,
                                              C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_group_step_frame_with_levels": (C.c_int32, [C.c_void_p, C.c_int32,
                                                          C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_nccl_unique_id": (C.c_int32, [C.POINTER(C.c_uint8), _ep]),
    "apbf_gpu_solver_attach_nccl": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32,
                                                C.POINTER(C.c_uint8), _ep]),
    "apbf_gpu_slab_set_state": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int64, _fp, _fp, _fp, _fp,
                                            _fp, _fp, _ip, _ep]),
    "apbf_slab_partition": (C.c_int32, [_lp, C.c_int32, C.c_int32, C.c_int32, _ip, _ip]),
    "apbf_gpu_grid_build": (C.c_int32, [C.c_int32, _fp, C.c_float, C.c_float, _ip, _fp, _ip, _ip,
                                        C.c_int64, _lp, _ep]),
    "apbf_gpu_neighbor_lists": (C.c_int32, [C.c_int32, _fp, C.c_float, C.c_float, _ip, _ip,
                                            C.c_int64, _lp, _ep]),
    "apbf_gpu_all_densities": (C.c_int32, [C.c_int32, _fp, _fp, C.c_float, _fp, _ep]),
    "apbf_gpu_vorticity": (C.c_int32, [C.c_int32, _fp, _fp, C.c_float, _fp, _ep]),
    "apbf_gpu_host_alloc": (C.c_void_p, [C.c_size_t]),
    "apbf_gpu_set_fast_math": (C.c_int32, [C.c_void_p, C.c_int32]),
    "apbf_gpu_host_free": (None, [C.c_void_p]),
    "apbf_gpu_lod_dtc": (C.c_int32, [C.c_int32, _fp, C.POINTER(apbf_camera),
                                     C.POINTER(apbf_lod_config), _ip, _ep]),
    "apbf_gpu_lod_dtvs": (C.c_int32, [C.c_int32, _fp, C.POINTER(apbf_camera),
                                      C.POINTER(apbf_lod_config), C.c_float, _ip, _ep]),
    "apbf_gpu_splat": (C.c_int32, [C.c_int32, _fp, C.c_float, C.POINTER(apbf_camera), _fp, _ep]),
    "apbf_gpu_count_contacts": (C.c_int32, [C.c_int32, _fp, C.POINTER(apbf_sdf_primitive),
                                            C.c_int32, C.c_float, C.c_float, _lp, _ep]),
    "apbf_gpu_step_frame_host": (C.c_int32, [C.c_void_p, C.c_int32, _fp, _fp, _fp, _fp, _fp, _fp, _ip,
                                             C.POINTER(apbf_camera), C.POINTER(apbf_lod_config), C.c_int32,
                                             C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_blend_lod": (C.c_int32, [C.c_int32, C.c_int32, C.POINTER(_ip), _ip, _ep]),
    "apbf_gpu_step_frame_multi": (C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(apbf_camera),
                                              C.POINTER(apbf_lod_config), C.c_int32,
                                              C.POINTER(apbf_frame_stats), _ep]),
    "apbf_gpu_render_level_image": (C.c_int32, [C.c_int32, _fp, _ip, C.c_float, C.POINTER(apbf_camera),
                                                C.c_int32, C.c_int32, C.POINTER(C.c_uint8), _ep]),
    "apbf_gpu_render_levels": (C.c_int32, [C.c_void_p, C.POINTER(apbf_camera), C.c_float, C.c_int32,
                                           C.c_int32, C.POINTER(C.c_uint8), _ep]),
}

_LIB = None


def header_symbols() -> list[str]:
    """Function names declared in include/apbf_gpu.h (parsed, for tests)."""
    import re
    path = os.path.join(os.path.dirname(HERE), "include", "apbf_gpu.h")
    text = open(path).read()
    return sorted(set(re.findall(r"\b(apbf_gpu_[a-z_0-9]+)\s*\(", text)))


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA library (no GPU needed to load) and bind the signatures."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"APBF CUDA library not built: {path} is missing (run __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def lib() -> C.CDLL:
    return load()
