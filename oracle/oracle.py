"""TEST INFRASTRUCTURE ONLY -- Python bindings of the CPU checkers.

* ``Oracle*``  -> oracle/liboracle.so: the plain-C float32 restatement of the
  reference path (apbf_oracle.c), file:line cited per function.
* ``Ref*``     -> oracle/_ref/libapbf_ref.so: the UNMODIFIED reference sources
  compiled against the Eigen-subset shim (oracle/Makefile); Solver<float>
  (prec=4) or Solver<double> (prec=8, as the reference ships).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product (paper_1608_04721_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1608_04721_b200 import capi
from paper_1608_04721_b200.api import (Camera, FrameStats, LodModelConfig, ParticleSet, SdfScene,
                                       SolverConfig, raise_for)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libapbf_ref.so")

F32 = np.float32
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)


def fp(a):
    return a.ctypes.data_as(_fp)


def ip(a):
    return a.ctypes.data_as(_ip)


def dp(a):
    return a.ctypes.data_as(_dp)


# ===================================================== C restatement

_O = None


def olib():
    global _O
    if _O is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError("oracle/liboracle.so not built (make -C oracle)")
        L = C.CDLL(ORACLE_LIB)
        E = C.POINTER(capi.apbf_error)
        sig = {
            "orc_solver_create": (C.c_void_p, [C.POINTER(capi.apbf_solver_config),
                                               C.POINTER(capi.apbf_sdf_primitive), C.c_int32,
                                               C.c_float, E]),
            "orc_solver_destroy": (None, [C.c_void_p]),
            "orc_set_state": (C.c_int32, [C.c_void_p, C.c_int32, _fp, _fp, _fp, _fp, _fp, _fp, _ip, E]),
            "orc_get_state": (C.c_int32, [C.c_void_p, _fp, _fp, _fp, _fp, _fp, _fp, _ip]),
            "orc_step_frame": (C.c_int32, [C.c_void_p, C.POINTER(capi.apbf_camera),
                                           C.POINTER(capi.apbf_lod_config), C.c_int32,
                                           C.POINTER(capi.apbf_frame_stats), E]),
            "orc_step_frame_with_levels": (C.c_int32, [C.c_void_p, C.c_int32,
                                                       C.POINTER(capi.apbf_frame_stats), E]),
            "orc_set_iteration_observer": (None, [C.c_void_p, capi.OBSERVER, C.c_void_p]),
            "orc_set_frame_metrics": (None, [C.c_void_p, C.c_int32]),
            "orc_last_permutation": (C.c_int32, [C.c_void_p, _ip]),
            "orc_density_kernel_r2": (C.c_float, [C.c_float, C.c_float]),
            "orc_gradient_kernel": (None, [_fp, C.c_float, _fp]),
            "orc_grid_build": (C.c_int32, [C.c_int32, _fp, C.c_float, C.c_float, _ip, _fp, _ip, _ip,
                                           C.c_int64, _lp, E]),
            "orc_neighbor_lists": (C.c_int32, [C.c_int32, _fp, C.c_float, C.c_float, _ip, _ip,
                                               C.c_int64, _lp, E]),
            "orc_compute_density": (C.c_float, [C.c_int32, _ip, _ip, _fp, _fp, C.c_float]),
            "orc_compute_lambda": (C.c_float, [C.c_int32, _ip, _ip, _fp, _fp, _fp,
                                               C.POINTER(capi.apbf_solver_config)]),
            "orc_compute_deltap": (None, [C.c_int32, _ip, _ip, _fp, _fp, _fp, _ip,
                                          C.POINTER(capi.apbf_solver_config), C.c_int32, _fp]),
            "orc_all_densities": (C.c_int32, [C.c_int32, _fp, _fp, C.c_float, _fp, E]),
            "orc_lod_dtc": (C.c_int32, [C.c_int32, _fp, C.POINTER(capi.apbf_camera),
                                        C.POINTER(capi.apbf_lod_config), _ip, E]),
            "orc_lod_dtvs": (C.c_int32, [C.c_int32, _fp, C.POINTER(capi.apbf_camera),
                                         C.POINTER(capi.apbf_lod_config), C.c_float, _ip, E]),
            "orc_splat": (C.c_int32, [C.c_int32, _fp, C.c_float, C.POINTER(capi.apbf_camera), _fp, E]),
            "orc_count_contacts": (C.c_int32, [C.c_int32, _fp, C.POINTER(capi.apbf_sdf_primitive),
                                               C.c_int32, C.c_float, C.c_float, _lp, E]),
            "orc_scene_distance": (C.c_int32, [C.POINTER(capi.apbf_sdf_primitive), C.c_int32,
                                               C.c_float, _fp, _fp, _fp, E]),
            "orc_map_distance_to_level": (C.c_int32, [C.c_float, C.c_float, C.c_float, C.c_int32,
                                                      C.c_int32]),
            "orc_percentile": (C.c_float, [_fp, C.c_int32, C.c_float]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _O = L
    return _O


def _pos(p):
    return np.ascontiguousarray(np.asarray(p, dtype=F32).reshape(-1, 3))


class OracleSolver:
    """Same interface as paper_1608_04721_b200.Solver, on the C restatement."""

    def __init__(self, cfg: SolverConfig, scene: SdfScene | None = None):
        self.L = olib()
        self.cfg = cfg
        scene = scene if scene is not None else SdfScene()
        prims, n = scene.to_c()
        err = capi.apbf_error()
        self.h = self.L.orc_solver_create(C.byref(cfg.to_c()), prims, n, scene.gradient_step,
                                          C.byref(err))
        if not self.h:
            raise_for(err.code, err)
        self._res = (C.c_double * max(1, cfg.substeps * cfg.range.n_max))()
        self._obs = None
        self._obs_c = None
        self._state = None

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_solver_destroy(self.h)
            self.h = None

    @property
    def iteration_observer(self):
        return self._obs

    @iteration_observer.setter
    def iteration_observer(self, fn):
        self._obs = fn

        def tramp(user, s, it):
            st = self._state
            self._get(st)
            fn(int(s), int(it), st)

        self._obs_c = capi.OBSERVER(tramp) if fn else capi.OBSERVER()
        self.L.orc_set_iteration_observer(self.h, self._obs_c, None)

    def set_frame_metrics(self, on: bool):
        self.L.orc_set_frame_metrics(self.h, int(on))

    def _set(self, s: ParticleSet):
        s._normalise()
        err = capi.apbf_error()
        rc = self.L.orc_set_state(self.h, s.count(), fp(s.x), fp(s.x_star), fp(s.v), fp(s.mass),
                                  fp(s.inv_mass), fp(s.lambda_), ip(s.level), C.byref(err))
        raise_for(rc, err)

    def _get(self, s: ParticleSet):
        self.L.orc_get_state(self.h, fp(s.x), fp(s.x_star), fp(s.v), fp(s.mass), fp(s.inv_mass),
                             fp(s.lambda_), ip(s.level))

    def _stats(self):
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        return st

    def step_frame(self, state, cam: Camera, lod: LodModelConfig, frame: int) -> FrameStats:
        self._set(state)
        self._state = state
        st, err = self._stats(), capi.apbf_error()
        rc = self.L.orc_step_frame(self.h, C.byref(cam.to_c()), C.byref(lod.to_c()), frame,
                                   C.byref(st), C.byref(err))
        self._get(state)
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame_with_levels(self, state, frame: int) -> FrameStats:
        self._set(state)
        self._state = state
        st, err = self._stats(), capi.apbf_error()
        rc = self.L.orc_step_frame_with_levels(self.h, frame, C.byref(st), C.byref(err))
        self._get(state)
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def last_permutation(self, n: int) -> np.ndarray:
        p = np.zeros(max(1, n), np.int32)
        self.L.orc_last_permutation(self.h, ip(p))
        return p[:n]


def oracle_grid_build(positions, h, padding):
    L = olib()
    p = _pos(positions)
    n = p.shape[0]
    perm = np.zeros(max(1, n), np.int32)
    origin = np.zeros(3, F32)
    dims = np.zeros(3, np.int32)
    cells = C.c_int64()
    err = capi.apbf_error()
    rc = L.orc_grid_build(n, fp(p), h, padding, ip(perm), fp(origin), ip(dims), None, 0,
                          C.byref(cells), C.byref(err))
    raise_for(rc, err)
    cs = np.zeros(cells.value + 1, np.int32)
    rc = L.orc_grid_build(n, fp(p), h, padding, ip(perm), fp(origin), ip(dims), ip(cs), cs.shape[0],
                          C.byref(cells), C.byref(err))
    raise_for(rc, err)
    return perm[:n], origin, dims, cs


def oracle_neighbor_lists(positions, h, padding):
    L = olib()
    p = _pos(positions)
    n = p.shape[0]
    off = np.zeros(n + 1, np.int32)
    tot = C.c_int64()
    err = capi.apbf_error()
    rc = L.orc_neighbor_lists(n, fp(p), h, padding, ip(off), None, 0, C.byref(tot), C.byref(err))
    raise_for(rc, err)
    idx = np.zeros(max(1, tot.value), np.int32)
    rc = L.orc_neighbor_lists(n, fp(p), h, padding, ip(off), ip(idx), idx.shape[0], C.byref(tot),
                              C.byref(err))
    raise_for(rc, err)
    return off, idx[:tot.value]


def oracle_all_densities(positions, masses, h):
    L = olib()
    p = _pos(positions)
    m = np.ascontiguousarray(masses, dtype=F32)
    rho = np.zeros(max(1, p.shape[0]), F32)
    err = capi.apbf_error()
    rc = L.orc_all_densities(p.shape[0], fp(p), fp(m), h, fp(rho), C.byref(err))
    raise_for(rc, err)
    return rho[:p.shape[0]]


def oracle_lod(positions, cam: Camera, cfg: LodModelConfig, r: float | None = None):
    L = olib()
    p = _pos(positions)
    out = np.zeros(max(1, p.shape[0]), np.int32)
    err = capi.apbf_error()
    if r is None:
        rc = L.orc_lod_dtc(p.shape[0], fp(p), C.byref(cam.to_c()), C.byref(cfg.to_c()), ip(out),
                           C.byref(err))
    else:
        rc = L.orc_lod_dtvs(p.shape[0], fp(p), C.byref(cam.to_c()), C.byref(cfg.to_c()), r, ip(out),
                            C.byref(err))
    raise_for(rc, err)
    return out[:p.shape[0]]


def oracle_splat(positions, r, cam: Camera):
    L = olib()
    p = _pos(positions)
    out = np.zeros(cam.width * cam.height, F32)
    err = capi.apbf_error()
    rc = L.orc_splat(p.shape[0], fp(p), r, C.byref(cam.to_c()), fp(out), C.byref(err))
    raise_for(rc, err)
    return out.reshape(cam.height, cam.width)


def oracle_count_contacts(scene: SdfScene, positions, r):
    L = olib()
    p = _pos(positions)
    prims, n = scene.to_c()
    out = C.c_int64()
    err = capi.apbf_error()
    rc = L.orc_count_contacts(p.shape[0], fp(p), prims, n, scene.gradient_step, r, C.byref(out),
                              C.byref(err))
    raise_for(rc, err)
    return int(out.value)


def oracle_scene_distance(scene: SdfScene, point):
    L = olib()
    prims, n = scene.to_c()
    q = np.asarray(point, F32)
    phi = np.zeros(1, F32)
    g = np.zeros(3, F32)
    err = capi.apbf_error()
    rc = L.orc_scene_distance(prims, n, scene.gradient_step, fp(q), fp(phi), fp(g), C.byref(err))
    raise_for(rc, err)
    return float(phi[0]), g


# ========================================== reference through the shim

class ref_config(C.Structure):
    _fields_ = [("dt_frame", C.c_double), ("substeps", C.c_int32), ("n_min", C.c_int32),
                ("n_max", C.c_int32), ("rest_density", C.c_double), ("h", C.c_double),
                ("epsilon", C.c_double), ("gravity", C.c_double * 3),
                ("stab_iterations", C.c_int32), ("stab_threshold", C.c_int32),
                ("particle_radius", C.c_double), ("mode", C.c_int32),
                ("velocity_cap", C.c_double), ("inactive_lambda_zero", C.c_int32),
                ("deterministic", C.c_int32), ("record_residuals", C.c_int32)]


class ref_prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("interior", C.c_int32), ("p", C.c_double * 3),
                ("q", C.c_double * 3), ("a", C.c_double), ("b", C.c_double)]


class ref_camera(C.Structure):
    _fields_ = [("eye", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("vertical_fov", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("near_clip", C.c_double)]


class ref_lod(C.Structure):
    _fields_ = [("model", C.c_int32), ("d_min", C.c_double), ("d_max", C.c_double),
                ("n_min", C.c_int32), ("n_max", C.c_int32), ("auto_range", C.c_int32)]


class ref_stats(C.Structure):
    _fields_ = [("frame", C.c_int32), ("n_residuals", C.c_int32), ("wall_ms", C.c_double),
                ("avg_density_pct", C.c_double), ("min_density_pct", C.c_double),
                ("max_density_pct", C.c_double), ("total_iterations", C.c_int64),
                ("contacts", C.c_int64), ("residuals", C.c_double * 256)]


class ref_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("particle", C.c_int32), ("pass_", C.c_char * 32),
                ("message", C.c_char * 224)]


class ref_scenario(C.Structure):
    _fields_ = [("n_particles", C.c_int32), ("n_prims", C.c_int32), ("mass", C.c_double),
                ("cfg", ref_config), ("prims", ref_prim * 8), ("grad_step", C.c_double),
                ("cam", ref_camera), ("lod", ref_lod), ("frames", C.c_int32),
                ("hash", C.c_uint64)]


_R = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def rlib():
    global _R
    if _R is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libapbf_ref.so not built (needs /root/reference)")
        L = C.CDLL(REF_LIB)
        E = C.POINTER(ref_error)
        sig = {
            "ref_omp_threads": (C.c_int32, []),
            "ref_solver_create": (C.c_void_p, [C.c_int32, C.POINTER(ref_config), C.POINTER(ref_prim),
                                               C.c_int32, C.c_double, E]),
            "ref_solver_destroy": (None, [C.c_void_p]),
            "ref_set_state": (C.c_int32, [C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _ip]),
            "ref_get_state": (C.c_int32, [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _ip]),
            "ref_step_frame": (C.c_int32, [C.c_void_p, C.POINTER(ref_camera), C.POINTER(ref_lod),
                                           C.c_int32, C.POINTER(ref_stats), E]),
            "ref_step_frame_with_levels": (C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(ref_stats), E]),
            "ref_grid_build": (C.c_int32, [C.c_int32, C.c_int32, _dp, C.c_double, C.c_double, _ip, _dp,
                                           _ip, _ip, C.c_int64, _lp, E]),
            "ref_neighbor_lists": (C.c_int32, [C.c_int32, C.c_int32, _dp, C.c_double, C.c_double, _ip,
                                               _ip, C.c_int64, _lp, E]),
            "ref_all_densities": (C.c_int32, [C.c_int32, C.c_int32, _dp, _dp, C.c_double, _dp, E]),
            "ref_lod_levels": (C.c_int32, [C.c_int32, C.c_int32, _dp, C.POINTER(ref_camera),
                                           C.POINTER(ref_lod), C.c_double, _ip, E]),
            "ref_splat": (C.c_int32, [C.c_int32, C.c_int32, _dp, C.c_double, C.POINTER(ref_camera),
                                      _dp, E]),
            "ref_scene_distance": (C.c_int32, [C.c_int32, C.POINTER(ref_prim), C.c_int32, C.c_double,
                                               _dp, _dp, _dp, E]),
            "ref_density_kernel_r2": (C.c_double, [C.c_int32, C.c_double, C.c_double]),
            "ref_gradient_kernel": (None, [C.c_int32, _dp, C.c_double, _dp]),
            "ref_build_scenario": (C.c_int32, [C.c_char_p, C.c_double, C.c_uint64,
                                               C.POINTER(ref_scenario), _dp, E]),
            "ref_splitmix64_first": (C.c_uint64, [C.c_uint64]),
            "ref_render_level_image": (C.c_int32, [C.c_int32, C.c_int32, _dp, _ip, C.c_double,
                                                   C.POINTER(ref_camera), C.c_int32, C.c_int32,
                                                   C.POINTER(C.c_uint8), E]),
            "ref_write_particle_snapshot": (C.c_int32, [C.c_int32, C.c_int32, _dp, _ip, C.c_char_p, E]),
            "ref_run_scenario": (C.c_int32, [C.c_char_p, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                                             C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_char_p,
                                             C.c_int32, C.c_int32, E]),
            "ref_format_bench_report": (C.c_int32, [C.c_int32, C.POINTER(C.c_char_p), _dp,
                                                    C.POINTER(C.c_int64), _ip, _ip, C.c_char_p, C.c_int32,
                                                    E]),
            "ref_parse_bench_mode": (C.c_int32, [C.c_char_p, _ip, _ip, _ip, E]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _R = L
    return _R


def _rraise(rc, err):
    if rc:
        e = capi.apbf_error()
        e.code = err.code
        e.particle = err.particle
        e.pass_ = err.pass_
        e.message = err.message
        raise_for(rc, e)


def ref_cfg(cfg: SolverConfig) -> ref_config:
    c = ref_config()
    c.dt_frame = cfg.dt_frame
    c.substeps = cfg.substeps
    c.n_min, c.n_max = cfg.range.n_min, cfg.range.n_max
    c.rest_density = cfg.rest_density
    c.h = cfg.h
    c.epsilon = cfg.epsilon
    c.gravity[:] = [float(g) for g in cfg.gravity]
    c.stab_iterations = cfg.stab_iterations
    c.stab_threshold = cfg.stab_threshold
    c.particle_radius = cfg.particle_radius
    c.mode = int(cfg.mode)
    c.velocity_cap = cfg.velocity_cap
    c.inactive_lambda_zero = int(cfg.inactive_lambda_zero)
    c.deterministic = int(cfg.deterministic)
    c.record_residuals = int(cfg.record_residuals)
    return c


def ref_prims(scene: SdfScene):
    from paper_1608_04721_b200.api import Box, Cone, HalfSpace, Sphere
    arr = (ref_prim * max(1, len(scene.primitives)))()
    for k, p in enumerate(scene.primitives):
        c = arr[k]
        if isinstance(p, HalfSpace):
            c.kind, c.a = 0, p.offset
            c.p[:] = [float(v) for v in p.normal]
        elif isinstance(p, Sphere):
            c.kind, c.a, c.interior = 1, p.radius, int(p.interior)
            c.p[:] = [float(v) for v in p.center]
        elif isinstance(p, Box):
            c.kind, c.interior = 2, int(p.interior)
            c.p[:] = [float(v) for v in p.center]
            c.q[:] = [float(v) for v in p.half_extents]
        elif isinstance(p, Cone):
            c.kind, c.a, c.b = 3, p.base_radius, p.height
            c.p[:] = [float(v) for v in p.base_center]
    return arr, len(scene.primitives)


def ref_cam(cam: Camera) -> ref_camera:
    c = ref_camera()
    c.eye[:] = [float(v) for v in cam.eye]
    c.look_at[:] = [float(v) for v in cam.look_at]
    c.up[:] = [float(v) for v in cam.up]
    c.vertical_fov = cam.vertical_fov
    c.width, c.height = cam.width, cam.height
    c.near_clip = cam.near_clip
    return c


def ref_lodc(l: LodModelConfig) -> ref_lod:
    c = ref_lod()
    c.model = int(l.model)
    c.d_min, c.d_max = l.d_min, l.d_max
    c.n_min, c.n_max = l.range.n_min, l.range.n_max
    c.auto_range = int(l.auto_range)
    return c


class RefState:
    """A ParticleSet in float64 arrays for the reference driver."""

    def __init__(self, x, x_star, v, mass, inv_mass, lambda_, level):
        self.x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
        self.x_star = np.ascontiguousarray(x_star, np.float64).reshape(-1, 3)
        self.v = np.ascontiguousarray(v, np.float64).reshape(-1, 3)
        self.mass = np.ascontiguousarray(mass, np.float64)
        self.inv_mass = np.ascontiguousarray(inv_mass, np.float64)
        self.lambda_ = np.ascontiguousarray(lambda_, np.float64)
        self.level = np.ascontiguousarray(level, np.int32)

    @staticmethod
    def from_set(s: ParticleSet) -> "RefState":
        return RefState(s.x, s.x_star, s.v, s.mass, s.inv_mass, s.lambda_, s.level)

    def count(self):
        return self.x.shape[0]


class RefSolver:
    """The reference's own Solver<float> (prec=4) / Solver<double> (prec=8)."""

    def __init__(self, cfg: SolverConfig, scene: SdfScene | None = None, prec: int = 4):
        self.L = rlib()
        scene = scene if scene is not None else SdfScene()
        prims, n = ref_prims(scene)
        err = ref_error()
        self.h = self.L.ref_solver_create(prec, C.byref(ref_cfg(cfg)), prims, n,
                                          scene.gradient_step, C.byref(err))
        if not self.h:
            _rraise(err.code or 1, err)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_solver_destroy(self.h)
            self.h = None

    def _set(self, s: RefState):
        self.L.ref_set_state(self.h, s.count(), dp(s.x), dp(s.x_star), dp(s.v), dp(s.mass),
                             dp(s.inv_mass), dp(s.lambda_), ip(s.level))

    def _get(self, s: RefState):
        self.L.ref_get_state(self.h, dp(s.x), dp(s.x_star), dp(s.v), dp(s.mass), dp(s.inv_mass),
                             dp(s.lambda_), ip(s.level))

    @staticmethod
    def _stats(st: ref_stats) -> FrameStats:
        return FrameStats(st.frame, st.wall_ms, st.avg_density_pct, st.min_density_pct,
                          st.max_density_pct, st.total_iterations, st.contacts,
                          [st.residuals[k] for k in range(min(256, st.n_residuals))])

    def step_frame(self, state: RefState, cam: Camera, lod: LodModelConfig, frame: int) -> FrameStats:
        self._set(state)
        st, err = ref_stats(), ref_error()
        rc = self.L.ref_step_frame(self.h, C.byref(ref_cam(cam)), C.byref(ref_lodc(lod)), frame,
                                   C.byref(st), C.byref(err))
        self._get(state)
        _rraise(rc, err)
        return self._stats(st)

    def step_frame_with_levels(self, state: RefState, frame: int) -> FrameStats:
        self._set(state)
        st, err = ref_stats(), ref_error()
        rc = self.L.ref_step_frame_with_levels(self.h, frame, C.byref(st), C.byref(err))
        self._get(state)
        _rraise(rc, err)
        return self._stats(st)


def ref_build_scenario(name: str, scale: float, seed: int):
    """buildScenario + makeState of the reference: (positions f64 (n,3), info)."""
    L = rlib()
    info = ref_scenario()
    err = ref_error()
    rc = L.ref_build_scenario(name.encode(), scale, seed, C.byref(info), None, C.byref(err))
    _rraise(rc, err)
    pos = np.zeros((info.n_particles, 3), np.float64)
    rc = L.ref_build_scenario(name.encode(), scale, seed, C.byref(info), dp(pos), C.byref(err))
    _rraise(rc, err)
    return pos, info


def ref_grid_build(positions, h, padding, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    n = p.shape[0]
    perm = np.zeros(max(1, n), np.int32)
    origin = np.zeros(3)
    dims = np.zeros(3, np.int32)
    cells = C.c_int64()
    err = ref_error()
    rc = L.ref_grid_build(prec, n, dp(p), h, padding, ip(perm), dp(origin), ip(dims), None, 0,
                          C.byref(cells), C.byref(err))
    _rraise(rc, err)
    cs = np.zeros(cells.value + 1, np.int32)
    rc = L.ref_grid_build(prec, n, dp(p), h, padding, ip(perm), dp(origin), ip(dims), ip(cs),
                          cs.shape[0], C.byref(cells), C.byref(err))
    _rraise(rc, err)
    return perm[:n], origin, dims, cs


def ref_neighbor_lists(positions, h, padding, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    n = p.shape[0]
    off = np.zeros(n + 1, np.int32)
    tot = C.c_int64()
    err = ref_error()
    rc = L.ref_neighbor_lists(prec, n, dp(p), h, padding, ip(off), None, 0, C.byref(tot), C.byref(err))
    _rraise(rc, err)
    idx = np.zeros(max(1, tot.value), np.int32)
    rc = L.ref_neighbor_lists(prec, n, dp(p), h, padding, ip(off), ip(idx), idx.shape[0],
                              C.byref(tot), C.byref(err))
    _rraise(rc, err)
    return off, idx[:tot.value]


def ref_all_densities(positions, masses, h, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    m = np.ascontiguousarray(masses, np.float64)
    rho = np.zeros(max(1, p.shape[0]))
    err = ref_error()
    rc = L.ref_all_densities(prec, p.shape[0], dp(p), dp(m), h, dp(rho), C.byref(err))
    _rraise(rc, err)
    return rho[:p.shape[0]]


def ref_lod_levels(positions, cam: Camera, cfg: LodModelConfig, r: float = 0.0, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    out = np.zeros(max(1, p.shape[0]), np.int32)
    err = ref_error()
    rc = L.ref_lod_levels(prec, p.shape[0], dp(p), C.byref(ref_cam(cam)), C.byref(ref_lodc(cfg)), r,
                          ip(out), C.byref(err))
    _rraise(rc, err)
    return out[:p.shape[0]]


def ref_splat(positions, r, cam: Camera, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    out = np.zeros(cam.width * cam.height)
    err = ref_error()
    rc = L.ref_splat(prec, p.shape[0], dp(p), r, C.byref(ref_cam(cam)), dp(out), C.byref(err))
    _rraise(rc, err)
    return out.reshape(cam.height, cam.width)


def ref_render_level_image(positions, levels, r, cam: Camera, nmin, nmax, prec=4):
    """renderLevelImage<S> of the reference: (height, width, 3) uint8."""
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    lv = np.ascontiguousarray(levels, np.int32)
    out = np.zeros(cam.width * cam.height * 3, np.uint8)
    err = ref_error()
    rc = L.ref_render_level_image(prec, p.shape[0], dp(p), lv.ctypes.data_as(C.POINTER(C.c_int32)), r,
                                  C.byref(ref_cam(cam)), nmin, nmax,
                                  out.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(err))
    _rraise(rc, err)
    return out.reshape(cam.height, cam.width, 3)


def ref_write_particle_snapshot(path, positions, levels, prec=4):
    L = rlib()
    p = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    lv = np.ascontiguousarray(levels, np.int32)
    err = ref_error()
    rc = L.ref_write_particle_snapshot(prec, p.shape[0], dp(p), lv.ctypes.data_as(C.POINTER(C.c_int32)),
                                       str(path).encode(), C.byref(err))
    _rraise(rc, err)


def ref_run_scenario(name, scale, mode, out_dir, frames, seed=0, lod=-1, rng=None, deterministic=True,
                     images_every=0, particles_every=0):
    """The reference's own runScenario (Solver<double>), writing into out_dir."""
    L = rlib()
    err = ref_error()
    nmin, nmax = (rng.n_min, rng.n_max) if rng is not None else (0, 0)
    rc = L.ref_run_scenario(name.encode(), scale, mode, lod, nmin, nmax, frames, seed, int(deterministic),
                            str(out_dir).encode(), images_every, particles_every, C.byref(err))
    _rraise(rc, err)


def ref_format_bench_report(results):
    """formatBenchReport of [(token, median_ms, iterations, frames, particles)]."""
    L = rlib()
    k = len(results)
    toks = (C.c_char_p * k)(*[r[0].encode() for r in results])
    med = np.array([r[1] for r in results], np.float64)
    its = (C.c_int64 * k)(*[r[2] for r in results])
    fr = np.array([r[3] for r in results], np.int32)
    pa = np.array([r[4] for r in results], np.int32)
    buf = C.create_string_buffer(1 << 16)
    err = ref_error()
    rc = L.ref_format_bench_report(k, toks, dp(med), its, fr.ctypes.data_as(C.POINTER(C.c_int32)),
                                   pa.ctypes.data_as(C.POINTER(C.c_int32)), buf, len(buf), C.byref(err))
    _rraise(rc, err)
    return buf.value.decode()


def ref_parse_bench_mode(token):
    """(mode, iterations, lod) or ValueError(message) like parseBenchMode."""
    L = rlib()
    m, it, lod = C.c_int32(), C.c_int32(), C.c_int32()
    err = ref_error()
    rc = L.ref_parse_bench_mode(token.encode(), C.byref(m), C.byref(it), C.byref(lod), C.byref(err))
    _rraise(rc, err)
    return m.value, it.value, lod.value


def ref_scene_distance(scene: SdfScene, point, prec=4):
    L = rlib()
    prims, n = ref_prims(scene)
    q = np.asarray(point, np.float64)
    phi = np.zeros(1)
    g = np.zeros(3)
    err = ref_error()
    rc = L.ref_scene_distance(prec, prims, n, scene.gradient_step, dp(q), dp(phi), dp(g), C.byref(err))
    _rraise(rc, err)
    return float(phi[0]), g
