"""Scenario library: host-side input generation, restated from the reference
harness (/root/reference/proj/src/scenario.{hpp,cpp}) so the GPU path and
the reference see identical inputs.  Pure numpy, float64 exactly as the
reference spawns (SplitMix64 jitter, scenario.hpp:39-56; spawnBlock
scenario.cpp:153-176).  Not on the hot path.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import (Box, Camera, Cone, HalfSpace, IterationRange, LodModel, LodModelConfig,
                  ParticleSet, SdfScene, SolverConfig, SolverMode, Sphere)

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """The first `count` outputs of SplitMix64(seed).next() (scenario.hpp:44-49)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def symmetric(raw: np.ndarray) -> np.ndarray:
    """SplitMix64::symmetric (scenario.hpp:52-55): uniform in [-1, 1)."""
    u = (raw >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return u * 2.0 - 1.0


@dataclass
class FluidBlock:
    origin: tuple = (0.0, 0.0, 0.0)
    counts: tuple = (1, 1, 1)
    spacing: float = 0.025


@dataclass
class ScenarioSpec:
    """ScenarioSpec (scenario.hpp:23-35), float64 values as the reference."""
    name: str = ""
    scale: float = 1.0
    blocks: List[FluidBlock] = field(default_factory=list)
    scene: SdfScene = field(default_factory=SdfScene)
    camera: Camera = field(default_factory=Camera)
    solver: SolverConfig = field(default_factory=SolverConfig)
    lod: LodModelConfig = field(default_factory=LodModelConfig)
    frames: int = 300
    jitter: float = 0.005

    def particle_count(self) -> int:
        return int(sum(b.counts[0] * b.counts[1] * b.counts[2] for b in self.blocks))


def _scaled_counts(base, scale: float):
    if not scale > 0.0:
        raise ValueError("scenario scale must be positive")
    f = math.cbrt(scale)
    out = []
    for b in base:
        v = b * f
        r = math.floor(abs(v) + 0.5) * (1 if v >= 0 else -1)  # llround: half away from zero
        out.append(max(1, int(r)))
    return tuple(out)


def _common(spec: ScenarioSpec) -> None:
    """applyCommonDefaults (scenario.cpp:39-57)."""
    s = spec.solver
    s.dt_frame = 0.0016
    s.substeps = 2
    s.rest_density = 1000.0
    s.h = 0.05
    s.epsilon = 1e-5
    s.gravity = (0.0, -9.81, 0.0)
    s.stab_iterations = 2
    s.particle_radius = 0.0125
    spec.scene.gradient_step = 1e-4 * s.h
    spec.lod.model = LodModel.DTVS
    spec.lod.auto_range = True
    spec.camera.vertical_fov = math.pi / 3.0
    spec.camera.width = 256
    spec.camera.height = 256
    spec.camera.near_clip = 1e-3
    spec.frames = 300
    spec.jitter = 0.005


def dam_break(scale: float) -> ScenarioSpec:
    """buildDamBreak (scenario.cpp:59-81)."""
    spec = ScenarioSpec(name="dam_break", scale=scale)
    _common(spec)
    spec.solver.range = IterationRange(3, 6)
    s = 0.025
    counts = _scaled_counts((60, 60, 60), scale)
    spec.blocks.append(FluidBlock((s / 2, s / 2, s / 2), counts, s))
    L = [counts[a] * s for a in range(3)]
    C = (4.0 * L[0], 2.5 * L[1], L[2])
    spec.scene.primitives.append(Box(tuple(c / 2 for c in C), tuple(c / 2 for c in C), True))
    spec.camera.eye = (1.1 * C[0], 1.2 * C[1], 2.6 * C[2])
    spec.camera.look_at = (0.25 * C[0], 0.2 * C[1], 0.5 * C[2])
    spec.lod.range = spec.solver.range
    return spec


def double_dam_break(scale: float) -> ScenarioSpec:
    """buildDoubleDamBreak (scenario.cpp:83-106)."""
    spec = ScenarioSpec(name="double_dam_break", scale=scale)
    _common(spec)
    spec.solver.range = IterationRange(5, 10)
    s = 0.025
    counts = _scaled_counts((58, 100, 58), scale)
    L = [counts[a] * s for a in range(3)]
    C = (3.0 * L[0], 1.6 * L[1], L[2])
    spec.blocks.append(FluidBlock((s / 2, s / 2, s / 2), counts, s))
    spec.blocks.append(FluidBlock((C[0] - L[0] + s / 2, s / 2, s / 2), counts, s))
    spec.scene.primitives.append(Box(tuple(c / 2 for c in C), tuple(c / 2 for c in C), True))
    spec.camera.eye = (0.5 * C[0], 1.3 * C[1], 3.2 * C[2])
    spec.camera.look_at = (0.5 * C[0], 0.25 * C[1], 0.5 * C[2])
    spec.lod.range = spec.solver.range
    return spec


def multi_dam_break(scale: float) -> ScenarioSpec:
    """buildMultiDamBreak (scenario.cpp:108-143)."""
    spec = ScenarioSpec(name="multi_dam_break", scale=scale)
    _common(spec)
    spec.solver.range = IterationRange(4, 8)
    s = 0.025
    counts = _scaled_counts((35, 46, 35), scale)
    L = [counts[a] * s for a in range(3)]
    side = 3.2 * L[0]
    height = 2.2 * L[1]
    lo = s / 2
    hiX = side - L[0] + s / 2
    hiZ = side - L[2] + s / 2
    for corner in ((lo, lo, lo), (hiX, lo, lo), (lo, lo, hiZ), (hiX, lo, hiZ)):
        spec.blocks.append(FluidBlock(corner, counts, s))
    C = (side, height, side)
    spec.scene.primitives.append(Box(tuple(c / 2 for c in C), tuple(c / 2 for c in C), True))
    spec.scene.primitives.append(Cone((side / 2, 0.0, side / 2), 0.5 * L[0], 1.2 * L[1]))
    spec.camera.eye = (1.15 * side, 1.5 * height, 1.15 * side)
    spec.camera.look_at = (0.5 * side, 0.2 * height, 0.5 * side)
    spec.lod.range = spec.solver.range
    return spec


BUILTINS = {"dam_break": dam_break, "double_dam_break": double_dam_break,
            "multi_dam_break": multi_dam_break}

SCENARIO_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "scenarios")


def build_scenario(name_or_path: str, scale: float = 1.0) -> ScenarioSpec:
    """buildScenario (scenario.cpp:201-209); also finds scenarios/<name>.cfg."""
    if name_or_path in BUILTINS:
        return BUILTINS[name_or_path](scale)
    path = name_or_path
    if not os.path.exists(path):
        cand = os.path.join(SCENARIO_DIR, name_or_path + ".cfg")
        if os.path.exists(cand):
            path = cand
    if os.path.exists(path):
        return load_scenario_file(path, scale)
    raise ValueError(f"unknown scenario '{name_or_path}'; valid names: dam_break, "
                     "double_dam_break, multi_dam_break, or a config file path")


def _vec3(v: str):
    t = v.split()
    if len(t) != 3:
        raise ValueError(f"expected three numbers, got '{v}'")
    return tuple(float(x) for x in t)


def _bool(v: str) -> bool:
    if v in ("true", "1", "yes", "on"):
        return True
    if v in ("false", "0", "no", "off"):
        return False
    raise ValueError(f"expected a boolean, got '{v}'")


def _int(v: str) -> int:
    d = float(v)
    if d != int(d):
        raise ValueError(f"expected an integer, got '{v}'")
    return int(d)


def _range(v: str) -> IterationRange:
    if ".." not in v:
        raise ValueError(f"expected a range like 3..6, got '{v}'")
    a, b = v.split("..", 1)
    return IterationRange(_int(a), _int(b))


def _primitive(v: str):
    t = v.split()
    interior = len(t) > 0 and t[-1] == "interior"
    if t[0] == "half_space":
        return HalfSpace(tuple(float(x) for x in t[1:4]), float(t[4]))
    if t[0] == "sphere":
        return Sphere(tuple(float(x) for x in t[1:4]), float(t[4]), interior)
    if t[0] == "box":
        return Box(tuple(float(x) for x in t[1:4]), tuple(float(x) for x in t[4:7]), interior)
    if t[0] == "cone":
        return Cone(tuple(float(x) for x in t[1:4]), float(t[4]), float(t[5]))
    raise ValueError(f"unknown primitive kind '{t[0]}'")


def load_scenario_file(path: str, scale: float = 1.0) -> ScenarioSpec:
    """loadScenarioFile (scenario.cpp:320-430), docs/scenario_format.md."""
    spec = ScenarioSpec(name=os.path.splitext(os.path.basename(path))[0], scale=scale)
    _common(spec)
    spec.solver.range = IterationRange(3, 6)
    section = ""
    grad_set = False
    raw_counts = []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            line = line.strip()
            if not line or line[0] in "#;":
                continue
            if line[0] == "[":
                if line[-1] != "]":
                    raise RuntimeError(f"{path}:{lineno}: unterminated section header")
                section = line[1:-1].strip()
                if section == "fluid":
                    spec.blocks.append(FluidBlock())
                    raw_counts.append((1, 1, 1))
                elif section not in ("solver", "lod", "camera", "scene"):
                    raise RuntimeError(f"{path}:{lineno}: unknown section [{section}]")
                continue
            if "=" not in line:
                raise RuntimeError(f"{path}:{lineno}: expected 'key = value'")
            key, value = (s.strip() for s in line.split("=", 1))
            s = spec.solver
            if section == "":
                if key == "name":
                    spec.name = value
                elif key == "frames":
                    spec.frames = _int(value)
                elif key == "jitter":
                    spec.jitter = float(value)
                else:
                    raise RuntimeError(f"{path}:{lineno}: unknown key '{key}'")
            elif section == "solver":
                m = {"dt_frame": ("dt_frame", float), "substeps": ("substeps", _int),
                     "iterations": ("range", _range), "rest_density": ("rest_density", float),
                     "smoothing_length": ("h", float), "epsilon": ("epsilon", float),
                     "gravity": ("gravity", _vec3), "stab_iterations": ("stab_iterations", _int),
                     "stab_threshold": ("stab_threshold", _int),
                     "particle_radius": ("particle_radius", float),
                     "velocity_cap": ("velocity_cap", float),
                     "inactive_lambda_zero": ("inactive_lambda_zero", _bool)}
                if key not in m:
                    raise RuntimeError(f"{path}:{lineno}: unknown solver key '{key}'")
                attr, conv = m[key]
                setattr(s, attr, conv(value))
            elif section == "lod":
                if key == "model":
                    if value not in ("dtc", "dtvs"):
                        raise RuntimeError(f"{path}:{lineno}: lod model must be dtc or dtvs")
                    spec.lod.model = LodModel.DTC if value == "dtc" else LodModel.DTVS
                elif key == "auto_range":
                    spec.lod.auto_range = _bool(value)
                elif key == "d_min":
                    spec.lod.d_min = float(value)
                elif key == "d_max":
                    spec.lod.d_max = float(value)
                else:
                    raise RuntimeError(f"{path}:{lineno}: unknown lod key '{key}'")
            elif section == "camera":
                c = spec.camera
                if key == "eye":
                    c.eye = _vec3(value)
                elif key == "look_at":
                    c.look_at = _vec3(value)
                elif key == "up":
                    c.up = _vec3(value)
                elif key == "fov_deg":
                    c.vertical_fov = float(value) * math.pi / 180.0
                elif key == "resolution":
                    t = value.split()
                    c.width, c.height = _int(t[0]), _int(t[1])
                elif key == "near":
                    c.near_clip = float(value)
                else:
                    raise RuntimeError(f"{path}:{lineno}: unknown camera key '{key}'")
            elif section == "scene":
                if key == "primitive":
                    spec.scene.primitives.append(_primitive(value))
                elif key == "gradient_step":
                    spec.scene.gradient_step = float(value)
                    grad_set = True
                else:
                    raise RuntimeError(f"{path}:{lineno}: unknown scene key '{key}'")
            elif section == "fluid":
                b = spec.blocks[-1]
                if key == "origin":
                    b.origin = _vec3(value)
                elif key == "counts":
                    raw_counts[-1] = tuple(_int(x) for x in value.split())
                elif key == "spacing":
                    b.spacing = float(value)
                else:
                    raise RuntimeError(f"{path}:{lineno}: unknown fluid key '{key}'")
    if not spec.blocks:
        raise RuntimeError(f"{path}: scenario file declares no [fluid] block")
    for b, rc in zip(spec.blocks, raw_counts):
        b.counts = _scaled_counts(rc, scale)
    if not grad_set:
        spec.scene.gradient_step = 1e-4 * spec.solver.h
    spec.lod.range = spec.solver.range
    spec.solver.validate()
    return spec


def spawn_block(origin, counts, spacing, jitter_amp, raw):
    """spawnBlock (scenario.cpp:153-176), x fastest; `raw` = SplitMix64 draws."""
    nx, ny, nz = counts
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    idx = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1).astype(np.float64)
    pos = np.asarray(origin, np.float64)[None, :] + spacing * idx
    if raw is not None and jitter_amp > 0.0:
        # Vec3(rng.symmetric(), rng.symmetric(), rng.symmetric()) at
        # scenario.cpp:168-169: GCC evaluates constructor arguments right to
        # left, so the first draw lands in z and the third in x.
        pos = pos + jitter_amp * symmetric(raw).reshape(-1, 3)[:, ::-1]
    return pos


def spawn_scenario(spec: ScenarioSpec, seed: int) -> np.ndarray:
    """spawnScenario (scenario.cpp:178-189): one jitter stream across blocks."""
    total = spec.particle_count()
    raw_all = splitmix64(seed, 3 * total)
    out = []
    at = 0
    for b in spec.blocks:
        n = b.counts[0] * b.counts[1] * b.counts[2]
        amp = spec.jitter * b.spacing
        raw = raw_all[3 * at: 3 * (at + n)]
        out.append(spawn_block(b.origin, b.counts, b.spacing, amp, raw))
        at += n
    return np.concatenate(out, axis=0) if out else np.zeros((0, 3))


def make_state(spec: ScenarioSpec, seed: int) -> ParticleSet:
    """makeState (scenario.cpp:191-199) as a float32 ParticleSet: positions
    cast from the float64 spawn, mass = (float)(rho0*s^3), invMass = 1/mass in
    float (the ParticleSet<float> constructor, particle_state.hpp:45-57)."""
    if not spec.blocks:
        raise ValueError("scenario has no fluid blocks")
    pos = spawn_scenario(spec, seed)
    s = spec.blocks[0].spacing
    mass = spec.solver.rest_density * s * s * s
    return ParticleSet(pos.astype(np.float32), float(np.float32(mass)), spec.solver.range.n_max)


def scenario_mass(spec: ScenarioSpec) -> float:
    s = spec.blocks[0].spacing
    return spec.solver.rest_density * s * s * s


def _num(v) -> str:
    return "%.17g;" % float(v)


def fnv1a64(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for c in data:
        h ^= c
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def scenario_hash(spec: ScenarioSpec, seed: int) -> int:
    """scenarioHash (scenario.cpp:441-499), physics-only fields."""
    s = spec.name + ";"
    s += _num(spec.scale) + _num(seed) + _num(spec.jitter)
    for b in spec.blocks:
        s += "".join(_num(v) for v in b.origin)
        s += "".join(_num(v) for v in b.counts) + _num(b.spacing)
    for p in spec.scene.primitives:
        if isinstance(p, HalfSpace):
            n = np.asarray(p.normal, np.float64)
            n = n / math.sqrt((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2])
            s += "half_space;" + "".join(_num(v) for v in n) + _num(p.offset)
        elif isinstance(p, Sphere):
            s += "sphere;" + "".join(_num(v) for v in p.center) + _num(p.radius) + _num(int(p.interior))
        elif isinstance(p, Box):
            s += ("box;" + "".join(_num(v) for v in p.center)
                  + "".join(_num(v) for v in p.half_extents) + _num(int(p.interior)))
        else:
            s += "cone;" + "".join(_num(v) for v in p.base_center) + _num(p.base_radius) + _num(p.height)
    s += _num(spec.scene.gradient_step)
    c = spec.camera
    s += "".join(_num(v) for v in c.eye) + "".join(_num(v) for v in c.look_at)
    s += "".join(_num(v) for v in c.up)
    s += _num(c.vertical_fov) + _num(c.width) + _num(c.height) + _num(c.near_clip)
    sv = spec.solver
    s += _num(sv.dt_frame) + _num(sv.substeps) + _num(sv.rest_density) + _num(sv.h)
    s += _num(sv.epsilon) + "".join(_num(v) for v in sv.gravity)
    radius = sv.particle_radius if sv.particle_radius > 0 else sv.h / 4
    cap = sv.velocity_cap if sv.velocity_cap > 0 else sv.h / (sv.dt_frame / sv.substeps)
    s += _num(radius) + _num(cap) + _num(int(sv.inactive_lambda_zero))
    return fnv1a64(s.encode())


def ocean_weak(nranks: int) -> ScenarioSpec:
    """Weak-scaling tank for the slab decomposition: the C3 ocean layer
    (scenarios/ocean_1m.cfg) repeated `nranks` times along z (the slab axis),
    i.e. counts 200 x 50 x (100 * nranks) in a box nranks x deeper; 1M
    particles per GPU and exactly ocean_1m at nranks = 1."""
    spec = build_scenario("ocean_1m")
    if nranks == 1:
        return spec
    b = spec.blocks[0]
    b.counts = (b.counts[0], b.counts[1], b.counts[2] * nranks)
    box = spec.scene.primitives[0]
    c, he = list(box.center), list(box.half_extents)
    c[2] *= nranks
    he[2] *= nranks
    spec.scene.primitives[0] = Box(tuple(c), tuple(he), box.interior)
    spec.name = f"ocean_weak_{nranks}"
    return spec
