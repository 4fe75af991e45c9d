"""Host-side mirror of the reference's solver API (Python over the C-ABI).

Names, argument meaning and error behaviour follow the reference classes in
/root/reference/proj/include/apbf/ (SolverConfig solver.hpp:26-67, FrameStats
:69-78, Solver :208-392, ParticleSet particle_state.hpp:33-121, SdfScene
sdf.hpp:18-85, Camera depth_splat.hpp:19-43, LodModelConfig lod.hpp:16-29)
so that tests read like the reference's own tests.  Exceptions map as
std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError,
apbf::NumericalError -> NumericalError, std::out_of_range -> IndexError.

All particle arrays are float32, 3-vectors as (n, 3) rows (one row per
particle, the transpose view of the reference's column-major Mat3X).  Every
compute call goes to libapbf_gpu.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Sequence

import numpy as np

from . import capi

F32 = np.float32


# --------------------------------------------------------------- errors

class NumericalError(RuntimeError):
    """apbf::NumericalError (types.hpp:25-39)."""

    def __init__(self, pass_: str, particle: int, message: str):
        super().__init__(message)
        self.pass_ = pass_
        self.particle = particle

    def pass_name(self) -> str:
        return self.pass_


class CudaError(RuntimeError):
    pass


def raise_for(code: int, err: capi.apbf_error) -> None:
    if code == capi.APBF_OK:
        return
    msg = err.message.decode(errors="replace")
    if code == capi.APBF_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == capi.APBF_ERR_NUMERICAL:
        raise NumericalError(err.pass_.decode(), int(err.particle), msg)
    if code == capi.APBF_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if code == capi.APBF_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


# ----------------------------------------------------------- value types

class SolverMode(IntEnum):
    PBF = capi.MODE_PBF
    APBF = capi.MODE_APBF


class LodModel(IntEnum):
    DTC = capi.LOD_DTC
    DTVS = capi.LOD_DTVS


@dataclass
class IterationRange:
    """IterationRange (particle_state.hpp:16-29)."""
    n_min: int = 1
    n_max: int = 1

    def __post_init__(self):
        if self.n_min < 1 or self.n_max < self.n_min:
            raise ValueError("iteration range requires 1 <= n_min <= n_max")

    def contains(self, level: int) -> bool:
        return self.n_min <= level <= self.n_max


@dataclass
class SolverConfig:
    """SolverConfig<Scalar> (solver.hpp:26-67); derived values in float32."""
    dt_frame: float = 0.0016
    substeps: int = 2
    range: IterationRange = field(default_factory=lambda: IterationRange(3, 6))
    rest_density: float = 1000.0
    h: float = 0.05
    epsilon: float = 1e-5
    gravity: Sequence[float] = (0.0, -9.81, 0.0)
    stab_iterations: int = 2
    stab_threshold: int = 0
    particle_radius: float = 0.0
    mode: SolverMode = SolverMode.APBF
    velocity_cap: float = 0.0
    inactive_lambda_zero: bool = False
    deterministic: bool = False
    record_residuals: bool = False
    # opt-in PBF post-pass, absent from the reference (0 = off, bit-identical frames)
    xsph_viscosity: float = 0.0
    vorticity_epsilon: float = 0.0

    def dt_substep(self) -> float:
        return float(F32(self.dt_frame) / F32(self.substeps))

    def effective_stab_threshold(self) -> int:
        return self.stab_threshold if self.stab_threshold > 0 else self.range.n_max

    def effective_particle_radius(self) -> float:
        return float(self.particle_radius) if self.particle_radius > 0 else float(F32(self.h) / F32(4))

    def effective_velocity_cap(self) -> float:
        if self.velocity_cap > 0:
            return float(self.velocity_cap)
        return float(F32(self.h) / F32(self.dt_substep()))

    def validate(self) -> None:
        if not self.dt_frame > 0:
            raise ValueError("dt_frame must be positive")
        if self.substeps < 1:
            raise ValueError("substeps must be at least 1")
        if not self.rest_density > 0:
            raise ValueError("rest density must be positive")
        if not self.h > 0:
            raise ValueError("smoothing length must be positive")
        if self.epsilon < 0:
            raise ValueError("epsilon must be non-negative")
        if self.stab_iterations < 0:
            raise ValueError("stab iterations must be non-negative")
        if self.stab_threshold != 0 and not (1 <= self.stab_threshold <= self.range.n_max):
            raise ValueError("stab threshold must lie in [1, n_max]")
        if self.particle_radius < 0:
            raise ValueError("particle radius must be non-negative")
        if self.velocity_cap < 0:
            raise ValueError("velocity cap must be non-negative")
        if not all(math.isfinite(g) for g in self.gravity):
            raise ValueError("gravity must be finite")

    def to_c(self) -> capi.apbf_solver_config:
        c = capi.apbf_solver_config()
        c.dt_frame = self.dt_frame
        c.substeps = self.substeps
        c.n_min = self.range.n_min
        c.n_max = self.range.n_max
        c.rest_density = self.rest_density
        c.h = self.h
        c.epsilon = self.epsilon
        for a in range(3):
            c.gravity[a] = self.gravity[a]
        c.stab_iterations = self.stab_iterations
        c.stab_threshold = self.stab_threshold
        c.particle_radius = self.particle_radius
        c.mode = int(self.mode)
        c.velocity_cap = self.velocity_cap
        c.inactive_lambda_zero = int(self.inactive_lambda_zero)
        c.deterministic = int(self.deterministic)
        c.record_residuals = int(self.record_residuals)
        c.xsph_viscosity = self.xsph_viscosity
        c.vorticity_epsilon = self.vorticity_epsilon
        return c


@dataclass
class HalfSpace:
    """HalfSpace (sdf.hpp:18-30): phi = n.p - offset; n normalised in float."""
    normal: Sequence[float]
    offset: float


@dataclass
class Sphere:
    center: Sequence[float]
    radius: float
    interior: bool = False


@dataclass
class Box:
    center: Sequence[float]
    half_extents: Sequence[float]
    interior: bool = False


@dataclass
class Cone:
    """Solid cone along +y (sdf.hpp:60-74)."""
    base_center: Sequence[float]
    base_radius: float
    height: float


@dataclass
class SdfScene:
    primitives: list = field(default_factory=list)
    gradient_step: float = 1e-4

    def empty(self) -> bool:
        return not self.primitives

    def to_c(self):
        arr = (capi.apbf_sdf_primitive * max(1, len(self.primitives)))()
        for k, p in enumerate(self.primitives):
            c = arr[k]
            if isinstance(p, HalfSpace):
                c.kind = capi.SDF_HALF_SPACE
                c.p[:] = [float(v) for v in p.normal]
                c.a = p.offset
            elif isinstance(p, Sphere):
                c.kind = capi.SDF_SPHERE
                c.p[:] = [float(v) for v in p.center]
                c.a = p.radius
                c.interior = int(p.interior)
            elif isinstance(p, Box):
                c.kind = capi.SDF_BOX
                c.p[:] = [float(v) for v in p.center]
                c.q[:] = [float(v) for v in p.half_extents]
                c.interior = int(p.interior)
            elif isinstance(p, Cone):
                c.kind = capi.SDF_CONE
                c.p[:] = [float(v) for v in p.base_center]
                c.a = p.base_radius
                c.b = p.height
            else:
                raise ValueError(f"unknown primitive {p!r}")
        return arr, len(self.primitives)


@dataclass
class Camera:
    """Camera<Scalar> (depth_splat.hpp:19-43)."""
    eye: Sequence[float] = (0.0, 0.0, 0.0)
    look_at: Sequence[float] = (0.0, 0.0, -1.0)
    up: Sequence[float] = (0.0, 1.0, 0.0)
    vertical_fov: float = 1.0471975511965976
    width: int = 256
    height: int = 256
    near_clip: float = 1e-3

    def to_c(self) -> capi.apbf_camera:
        c = capi.apbf_camera()
        c.eye[:] = [float(v) for v in self.eye]
        c.look_at[:] = [float(v) for v in self.look_at]
        c.up[:] = [float(v) for v in self.up]
        c.vertical_fov = self.vertical_fov
        c.width = self.width
        c.height = self.height
        c.near_clip = self.near_clip
        return c


@dataclass
class LodModelConfig:
    """LodModelConfig<Scalar> (lod.hpp:16-29)."""
    model: LodModel = LodModel.DTVS
    d_min: float = 0.0
    d_max: float = 1.0
    range: IterationRange = field(default_factory=IterationRange)
    auto_range: bool = True

    def to_c(self) -> capi.apbf_lod_config:
        c = capi.apbf_lod_config()
        c.model = int(self.model)
        c.d_min = self.d_min
        c.d_max = self.d_max
        c.n_min = self.range.n_min
        c.n_max = self.range.n_max
        c.auto_range = int(self.auto_range)
        return c


@dataclass
class FrameStats:
    """FrameStats (solver.hpp:69-78)."""
    frame: int = 0
    wall_ms: float = 0.0
    avg_density_pct: float = 0.0
    min_density_pct: float = 0.0
    max_density_pct: float = 0.0
    total_iterations: int = 0
    contacts: int = 0
    residuals: list = field(default_factory=list)

    @staticmethod
    def from_c(s: capi.apbf_frame_stats, res) -> "FrameStats":
        n = min(int(s.n_residuals), len(res)) if res is not None else 0
        return FrameStats(int(s.frame), float(s.wall_ms), float(s.avg_density_pct),
                          float(s.min_density_pct), float(s.max_density_pct),
                          int(s.total_iterations), int(s.contacts),
                          [float(res[k]) for k in range(n)])


class ParticleSet:
    """ParticleSet<float> (particle_state.hpp:33-121) as numpy arrays."""

    def __init__(self, positions=None, particle_mass: float = 1.0, initial_level: int = 1):
        if positions is None:
            positions = np.zeros((0, 3), F32)
        if not particle_mass > 0:
            raise ValueError("particle mass must be positive")
        pos = np.ascontiguousarray(np.asarray(positions, dtype=F32).reshape(-1, 3))
        n = pos.shape[0]
        self.x = pos.copy()
        self.x_star = pos.copy()
        self.v = np.zeros((n, 3), F32)
        self.mass = np.full(n, particle_mass, F32)
        self.inv_mass = np.full(n, F32(1) / F32(particle_mass), F32)
        self.lambda_ = np.zeros(n, F32)
        self.level = np.full(n, initial_level, np.int32)

    def count(self) -> int:
        return int(self.x.shape[0])

    def set_masses(self, masses) -> None:
        m = np.asarray(masses, dtype=F32)
        if m.shape[0] != self.count():
            raise ValueError("mass array size mismatch")
        if (m <= 0).any():
            raise ValueError("particle masses must be positive")
        self.mass = m.copy()
        self.inv_mass = (F32(1) / m).astype(F32)

    def copy(self) -> "ParticleSet":
        o = ParticleSet.__new__(ParticleSet)
        for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
            setattr(o, k, getattr(self, k).copy())
        return o

    def apply_permutation(self, perm) -> None:
        """particle_state.hpp:74-98: entry k of the result is entry perm[k]."""
        perm = np.asarray(perm)
        if perm.shape[0] != self.count():
            raise ValueError("permutation size mismatch")
        for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
            setattr(self, k, getattr(self, k)[perm].copy())

    def _normalise(self) -> None:
        for k in ("x", "x_star", "v"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=F32).reshape(-1, 3))
        for k in ("mass", "inv_mass", "lambda_"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=F32).reshape(-1))
        self.level = np.ascontiguousarray(self.level, dtype=np.int32).reshape(-1)


def _fp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


# stepFrame reads x, v, mass and inv_mass and overwrites x*, lambda and level
# before reading them.  (Every field is an output: the frame reorders storage.)
FRAME_INPUTS = ("x", "v", "mass", "inv_mass")


def state_pointers(state, only=None):
    """(x, x_star, v, mass, inv_mass, lambda_, level) pointers; fields not in
    `only` (when given) are NULL."""
    keep = lambda k: only is None or k in only  # noqa: E731
    return (_fp(state.x if keep("x") else None), _fp(state.x_star if keep("x_star") else None),
            _fp(state.v if keep("v") else None), _fp(state.mass if keep("mass") else None),
            _fp(state.inv_mass if keep("inv_mass") else None),
            _fp(state.lambda_ if keep("lambda_") else None), _ip(state.level if keep("level") else None))


# ---------------------------------------------------------------- solver

class Solver:
    """apbf::Solver<float> on one B200 (solver.hpp:208-392).

    ``step_frame``/``step_frame_with_levels`` keep the reference semantics:
    the caller's ParticleSet is uploaded, stepped and written back (reordered
    into the last substep's cell order).  The ``*_resident`` variants keep the
    state on the device between frames (``upload``/``download``).
    """

    def __init__(self, cfg: SolverConfig, scene: Optional[SdfScene] = None, device: int = 0):
        self._lib = capi.lib()
        self._h = None
        self.cfg = cfg
        self.scene_ = scene if scene is not None else SdfScene()
        prims, n = self.scene_.to_c()
        err = capi.apbf_error()
        h = C.c_void_p()
        rc = self._lib.apbf_gpu_solver_create(C.byref(cfg.to_c()), prims, n,
                                              float(self.scene_.gradient_step), device,
                                              C.byref(h), C.byref(err))
        raise_for(rc, err)
        self._h = h
        self._observer = None
        self._observer_c = None
        self._observer_state = None
        self._res = (C.c_double * max(1, cfg.substeps * cfg.range.n_max))()

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.apbf_gpu_solver_destroy(self._h)
            self._h = None

    def config(self) -> SolverConfig:
        return self.cfg

    def scene(self) -> SdfScene:
        return self.scene_

    # iterationObserver (solver.hpp:222-224): fn(substep, iteration, state)
    @property
    def iteration_observer(self):
        return self._observer

    @iteration_observer.setter
    def iteration_observer(self, fn: Optional[Callable]):
        self._observer = fn
        if fn is None:
            self._observer_c = None
            self._lib.apbf_gpu_set_iteration_observer(self._h, capi.OBSERVER(), None)
            return

        def tramp(user, substep, it):
            st = self._observer_state
            self.download(st)
            fn(int(substep), int(it), st)

        self._observer_c = capi.OBSERVER(tramp)
        self._lib.apbf_gpu_set_iteration_observer(self._h, self._observer_c, None)

    # --- resident state ---
    def upload(self, state: ParticleSet, frame_inputs_only: bool = False) -> None:
        """apbf_gpu_set_state.  frame_inputs_only: upload just what stepFrame
        reads (FRAME_INPUTS); step_frame_with_levels then needs a full upload."""
        state._normalise()
        err = capi.apbf_error()
        ptrs = state_pointers(state, FRAME_INPUTS if frame_inputs_only else None)
        rc = self._lib.apbf_gpu_set_state(self._h, state.count(), *ptrs, C.byref(err))
        raise_for(rc, err)

    def download(self, state: ParticleSet) -> None:
        """apbf_gpu_get_state (every field)."""
        n = self._lib.apbf_gpu_particle_count(self._h)
        if state.count() != n:
            state.x = np.zeros((n, 3), F32)
            state.x_star = np.zeros((n, 3), F32)
            state.v = np.zeros((n, 3), F32)
            state.mass = np.zeros(n, F32)
            state.inv_mass = np.zeros(n, F32)
            state.lambda_ = np.zeros(n, F32)
            state.level = np.zeros(n, np.int32)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_get_state(self._h, *state_pointers(state), C.byref(err))
        raise_for(rc, err)

    def step_frame_multi_resident(self, cams, lods, frame_index: int) -> FrameStats:
        """Multi-camera frame: levels = blendLod of each camera's assignLevels,
        then stepFrameWithLevels (apbf_gpu_step_frame_multi)."""
        if len(cams) != len(lods):
            raise ValueError("one LOD config per camera")
        k = len(cams)
        cs = (capi.apbf_camera * max(k, 1))(*[c.to_c() for c in cams])
        ls = (capi.apbf_lod_config * max(k, 1))(*[l.to_c() for l in lods])
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_step_frame_multi(self._h, k, cs, ls, frame_index, C.byref(st), C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame_multi(self, state: ParticleSet, cams, lods, frame_index: int) -> FrameStats:
        """step_frame_multi_resident on the caller's state (uploaded, stepped,
        downloaded like step_frame)."""
        self.upload(state)
        st = self.step_frame_multi_resident(cams, lods, frame_index)
        self.download(state)
        return st

    def render_levels(self, cam: Camera, r: float, rng: IterationRange) -> np.ndarray:
        """renderLevelImage of the resident state (x, level) on the device."""
        out = np.zeros(max(1, cam.width * cam.height * 3), np.uint8)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_render_levels(self._h, C.byref(cam.to_c()), r, rng.n_min, rng.n_max,
                                              out.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(err))
        raise_for(rc, err)
        return out.reshape(cam.height, cam.width, 3)

    def step_frame_resident(self, cam: Camera, lod_cfg: LodModelConfig, frame_index: int) -> FrameStats:
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_step_frame(self._h, C.byref(cam.to_c()), C.byref(lod_cfg.to_c()),
                                           frame_index, C.byref(st), C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame_with_levels_resident(self, frame_index: int) -> FrameStats:
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_step_frame_with_levels(self._h, frame_index, C.byref(st),
                                                       C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    # --- reference semantics (state in, state out) ---
    def step_frame(self, state: ParticleSet, cam: Camera, lod_cfg: LodModelConfig,
                   frame_index: int) -> FrameStats:
        """stepFrame(ParticleSet&) (solver.hpp:228-233) on the caller's arrays:
        one apbf_gpu_step_frame_host call uploads what the frame reads, steps,
        and writes the reordered state back in place (pinned arrays copy at
        full PCIe rate)."""
        state._normalise()
        self._observer_state = state
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_step_frame_host(self._h, state.count(), *state_pointers(state),
                                                C.byref(cam.to_c()), C.byref(lod_cfg.to_c()), frame_index,
                                                C.byref(st), C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame_with_levels(self, state: ParticleSet, frame_index: int) -> FrameStats:
        state._normalise()
        bad = ~((state.level >= self.cfg.range.n_min) & (state.level <= self.cfg.range.n_max))
        if bad.any():
            raise ValueError("particle level outside configured iteration range")
        self.upload(state)
        self._observer_state = state
        try:
            stats = self.step_frame_with_levels_resident(frame_index)
        finally:
            self.download(state)
        return stats

    # --- profiling hooks ---
    def set_fast_math(self, enabled: bool) -> None:
        """apbf_gpu_set_fast_math: contracted lambda / delta-p pair arithmetic
        (outside the bitwise contract; tier-B tolerance)."""
        self._lib.apbf_gpu_set_fast_math(self._h, int(enabled))

    def set_frame_metrics(self, enabled: bool) -> None:
        self._lib.apbf_gpu_set_frame_metrics(self._h, int(enabled))

    def set_phase_timing(self, enabled: bool) -> None:
        self._lib.apbf_gpu_set_phase_timing(self._h, int(enabled))

    def last_phase_ms(self) -> list:
        out = (C.c_float * 5)()
        self._lib.apbf_gpu_last_phase_ms(self._h, out)
        return [float(v) for v in out]

    def stream_handle(self) -> int:
        """cudaStream_t of this solver (all its kernels launch there)."""
        return int(self._lib.apbf_gpu_stream(self._h) or 0)

    @staticmethod
    def launch_count() -> int:
        return int(capi.lib().apbf_gpu_launch_count())

    def set_kernel_timing(self, enabled: bool) -> None:
        err = capi.apbf_error()
        raise_for(self._lib.apbf_gpu_set_kernel_timing(self._h, int(enabled), C.byref(err)), err)

    def kernel_times(self) -> dict:
        a, b = C.c_double(), C.c_double()
        n, it = C.c_int64(), C.c_int64()
        self._lib.apbf_gpu_kernel_times(self._h, C.byref(a), C.byref(b), C.byref(n), C.byref(it))
        return {"lambda_ms": a.value, "deltap_ms": b.value, "launches": n.value,
                "particle_iterations": it.value}

    def last_neighbor_stats(self):
        a, b = C.c_int64(), C.c_int64()
        self._lib.apbf_gpu_last_neighbor_stats(self._h, C.byref(a), C.byref(b))
        return int(a.value), int(b.value)


# ------------------------------------------------------ free functions

def _pos(positions):
    return np.ascontiguousarray(np.asarray(positions, dtype=F32).reshape(-1, 3))


@dataclass
class GridBuild:
    perm: np.ndarray
    origin: np.ndarray
    dims: np.ndarray
    cell_start: np.ndarray


def grid_build(positions, h: float, padding: float) -> GridBuild:
    """UniformGrid<float>::build (uniform_grid.hpp:42-98)."""
    lib = capi.lib()
    p = _pos(positions)
    n = p.shape[0]
    perm = np.zeros(max(n, 1), np.int32)
    origin = np.zeros(3, F32)
    dims = np.zeros(3, np.int32)
    cells = C.c_int64()
    err = capi.apbf_error()
    rc = lib.apbf_gpu_grid_build(n, _fp(p), h, padding, _ip(perm), _fp(origin), _ip(dims), None, 0,
                                 C.byref(cells), C.byref(err))
    raise_for(rc, err)
    cs = np.zeros(cells.value + 1, np.int32)
    rc = lib.apbf_gpu_grid_build(n, _fp(p), h, padding, _ip(perm), _fp(origin), _ip(dims), _ip(cs),
                                 cs.shape[0], C.byref(cells), C.byref(err))
    raise_for(rc, err)
    return GridBuild(perm[:n], origin, dims, cs)


def neighbor_lists(positions, h: float, padding: float):
    """UniformGrid::build + buildNeighborLists (uniform_grid.hpp:179-213):
    (offsets, indices) over sorted slots."""
    lib = capi.lib()
    p = _pos(positions)
    n = p.shape[0]
    offsets = np.zeros(n + 1, np.int32)
    total = C.c_int64()
    err = capi.apbf_error()
    rc = lib.apbf_gpu_neighbor_lists(n, _fp(p), h, padding, _ip(offsets), None, 0, C.byref(total),
                                     C.byref(err))
    raise_for(rc, err)
    idx = np.zeros(max(1, total.value), np.int32)
    rc = lib.apbf_gpu_neighbor_lists(n, _fp(p), h, padding, _ip(offsets), _ip(idx), idx.shape[0],
                                     C.byref(total), C.byref(err))
    raise_for(rc, err)
    return offsets, idx[:total.value]


def all_densities(positions, masses, h: float) -> np.ndarray:
    """allDensities (solver.hpp:145-162), original index order."""
    lib = capi.lib()
    p = _pos(positions)
    m = np.ascontiguousarray(np.asarray(masses, dtype=F32))
    rho = np.zeros(max(1, p.shape[0]), F32)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_all_densities(p.shape[0], _fp(p), _fp(m), h, _fp(rho), C.byref(err))
    raise_for(rc, err)
    return rho[:p.shape[0]]


def vorticity(positions, velocities, h: float) -> np.ndarray:
    """The post-pass vorticity estimate (Macklin & Mueller 2013 eq. 15; not in
    the reference), (n, 3) in input order."""
    lib = capi.lib()
    p = _pos(positions)
    v = _pos(velocities)
    if v.shape != p.shape:
        raise ValueError("positions and velocities must have the same shape")
    out = np.zeros((max(1, p.shape[0]), 3), F32)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_vorticity(p.shape[0], _fp(p), _fp(v), h, _fp(out), C.byref(err))
    raise_for(rc, err)
    return out[:p.shape[0]]


def lod_dtc(positions, cam: Camera, cfg: LodModelConfig) -> np.ndarray:
    """lodDtc (lod.hpp:83-104)."""
    lib = capi.lib()
    p = _pos(positions)
    out = np.zeros(max(1, p.shape[0]), np.int32)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_lod_dtc(p.shape[0], _fp(p), C.byref(cam.to_c()), C.byref(cfg.to_c()),
                              _ip(out), C.byref(err))
    raise_for(rc, err)
    return out[:p.shape[0]]


def lod_dtvs(positions, cam: Camera, cfg: LodModelConfig, r: float) -> np.ndarray:
    """lodDtvs (lod.hpp:109-156)."""
    lib = capi.lib()
    p = _pos(positions)
    out = np.zeros(max(1, p.shape[0]), np.int32)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_lod_dtvs(p.shape[0], _fp(p), C.byref(cam.to_c()), C.byref(cfg.to_c()), r,
                               _ip(out), C.byref(err))
    raise_for(rc, err)
    return out[:p.shape[0]]


def splat(positions, r: float, cam: Camera) -> np.ndarray:
    """splat (depth_splat.hpp:201-228): (height, width) depths, +inf unwritten."""
    lib = capi.lib()
    p = _pos(positions)
    out = np.zeros(max(1, cam.width * cam.height), F32)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_splat(p.shape[0], _fp(p), r, C.byref(cam.to_c()), _fp(out), C.byref(err))
    raise_for(rc, err)
    return out.reshape(cam.height, cam.width)


def blend_lod(per_camera) -> np.ndarray:
    """blendLod (lod.hpp:160-172): elementwise max of level arrays."""
    arrs = [np.ascontiguousarray(a, np.int32) for a in per_camera]
    if not arrs:
        raise ValueError("blend requires at least one level array")
    n = arrs[0].shape[0]
    if any(a.shape[0] != n for a in arrs):
        raise ValueError("level array length mismatch")
    out = np.zeros(n, np.int32)
    ptrs = (C.POINTER(C.c_int32) * len(arrs))(*[_ip(a) for a in arrs])
    err = capi.apbf_error()
    rc = capi.lib().apbf_gpu_blend_lod(len(arrs), n, ptrs, _ip(out), C.byref(err))
    raise_for(rc, err)
    return out


def render_level_image(positions, levels, r: float, cam: Camera, rng: IterationRange) -> np.ndarray:
    """renderLevelImage (depth_splat.hpp:314-350) on the device: (height,
    width, 3) uint8, each pixel the levelColor of its nearest particle."""
    lib = capi.lib()
    p = _pos(positions)
    lv = np.ascontiguousarray(levels, np.int32)
    if lv.shape[0] != p.shape[0]:
        raise ValueError("level array size mismatch")
    out = np.zeros(max(1, cam.width * cam.height * 3), np.uint8)
    err = capi.apbf_error()
    rc = lib.apbf_gpu_render_level_image(p.shape[0], _fp(p), _ip(lv), r, C.byref(cam.to_c()), rng.n_min,
                                         rng.n_max, out.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(err))
    raise_for(rc, err)
    return out.reshape(cam.height, cam.width, 3)


def write_ppm(image: np.ndarray, path) -> None:
    """writePpm (depth_splat.hpp:251-262): binary P6."""
    h, w, _ = image.shape
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(np.ascontiguousarray(image, np.uint8).tobytes())


def read_ppm(path) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    parts = data.split(b"\n", 3)
    if parts[0] != b"P6" or parts[2] != b"255":
        raise ValueError(f"{path}: not a P6/255 image")
    w, h = (int(v) for v in parts[1].split())
    return np.frombuffer(parts[3], np.uint8, count=w * h * 3).reshape(h, w, 3)


def write_particle_snapshot(path, state: ParticleSet) -> None:
    """writeParticleSnapshot (particle_state.hpp:148-167): x,y,z,level per
    particle, coordinates as %.17g of their (float) values."""
    with open(path, "w") as f:
        f.write("x,y,z,level\n")
        x = state.x.astype(np.float64)
        f.writelines(f"{a:.17g},{b:.17g},{c:.17g},{int(lv)}\n" for (a, b, c), lv in zip(x, state.level))


def count_contacts(scene: SdfScene, positions, r: float) -> int:
    """findContacts(scene, positions, r).size() (sdf.hpp:226-250)."""
    lib = capi.lib()
    p = _pos(positions)
    prims, n = scene.to_c()
    out = C.c_int64()
    err = capi.apbf_error()
    rc = lib.apbf_gpu_count_contacts(p.shape[0], _fp(p), prims, n, scene.gradient_step, r,
                                     C.byref(out), C.byref(err))
    raise_for(rc, err)
    return int(out.value)
