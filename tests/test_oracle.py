"""The C oracle (oracle/apbf_oracle.c) against (a) the known-answer values of
the reference's own unit tests and (b) the golden fixtures generated from the
reference itself (tests/golden/make_golden.py).  CPU only."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import (Camera, IterationRange, LodModel, LodModelConfig, NumericalError,
                                   ParticleSet, SdfScene, SolverConfig, SolverMode, Box, HalfSpace,
                                   Sphere, Cone)
from paper_1608_04721_b200 import scenario as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
L = O.olib()


def W(r2, h):
    return L.orc_density_kernel_r2(r2, h)


def gradW(r, h):
    out = np.zeros(3, np.float32)
    L.orc_gradient_kernel(O.fp(np.asarray(r, np.float32)), h, O.fp(out))
    return out


# ---------------------------------------------- kernels (test_kernels.cpp)

def test_density_kernel_closed_form_at_origin():
    # test_kernels.cpp:29-32: W(0, h=1) = 315/(64 pi)
    assert W(0.0, 1.0) == pytest.approx(315.0 / (64.0 * math.pi), rel=1e-6)


def test_density_kernel_support_zeros():
    # test_kernels.cpp:34-41: zero at and beyond r = h
    assert W(1.0, 1.0) == 0.0
    assert W(1.5, 1.0) == 0.0
    assert W(0.999, 1.0) > 0.0


def test_gradient_kernel_closed_form():
    # test_kernels.cpp:76-81: grad W((0.5,0,0), 1) = (-45/pi * 0.25, 0, 0)
    g = gradW([0.5, 0, 0], 1.0)
    assert g[0] == pytest.approx(-45.0 / math.pi * 0.25, rel=1e-6)
    assert g[1] == 0.0 and g[2] == 0.0


def test_gradient_kernel_zero_at_origin_and_outside():
    assert not gradW([0, 0, 0], 1.0).any()
    assert not gradW([1.0, 0, 0], 1.0).any()


def test_gradient_kernel_exact_antisymmetry():
    # test_kernels.cpp:87-100
    rng = np.random.default_rng(3)
    for _ in range(200):
        r = rng.uniform(-0.1, 0.1, 3).astype(np.float32)
        assert np.array_equal(gradW(r, 0.12), -gradW(-r, 0.12))


# ----------------------------------------------- solver (test_solver.cpp)

def cfg_(**kw):
    c = SolverConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def pair_lists():
    return np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32)


def test_isolated_lambda_is_constraint_over_epsilon():
    # test_solver.cpp:111-126
    c = cfg_(h=0.1, rest_density=1000.0, epsilon=1e-5)
    off, idx = np.array([0, 1], np.int32), np.array([0], np.int32)
    x = np.zeros(3, np.float32)
    m = np.array([0.03], np.float32)
    w = (np.float32(1) / m).astype(np.float32)
    lam = L.orc_compute_lambda(0, O.ip(off), O.ip(idx), O.fp(x), O.fp(m), O.fp(w), c.to_c())
    cc = np.float32(0.03) * np.float32(W(0.0, 0.1)) * (np.float32(1) / np.float32(1000)) - np.float32(1)
    assert lam == np.float32(-cc) / np.float32(1e-5)


def test_two_body_lambda_closed_form():
    # test_solver.cpp:128-158 (tolerance relaxed from 1e-10 for float32)
    h, d, m, rho0 = 0.2, 0.1, 0.8, 3.0
    c = cfg_(h=h, rest_density=rho0, epsilon=1e-6)
    x = np.array([0, 0, 0, d, 0, 0], np.float32)
    mm = np.full(2, m, np.float32)
    w = (np.float32(1) / mm).astype(np.float32)
    off, idx = pair_lists()
    w0 = 315.0 / (64.0 * math.pi * h ** 3)
    wd = 315.0 / (64.0 * math.pi * h ** 9) * (h * h - d * d) ** 3
    gmag = 45.0 / (math.pi * h ** 6) * (h - d) ** 2
    cc = m * (w0 + wd) / rho0 - 1.0
    denom = (1 / m) * (gmag / rho0) ** 2 + (1.0 / rho0 ** 2) * (1 / m) * gmag * gmag + 1e-6
    for i in (0, 1):
        got = L.orc_compute_lambda(i, O.ip(off), O.ip(idx), O.fp(x), O.fp(mm), O.fp(w), c.to_c())
        assert got == pytest.approx(-cc / denom, rel=1e-5)


def test_symmetric_pair_corrections_cancel_exactly():
    # test_solver.cpp:160-181
    c = cfg_(h=0.2, rest_density=3.0)
    x = np.array([0.03, -0.01, 0.02, 0.11, 0.05, -0.04], np.float32)
    w = np.full(2, np.float32(1) / np.float32(0.8), np.float32)
    lam = np.full(2, -0.4, np.float32)
    lv = np.ones(2, np.int32)
    off, idx = pair_lists()
    d0, d1 = np.zeros(3, np.float32), np.zeros(3, np.float32)
    L.orc_compute_deltap(0, O.ip(off), O.ip(idx), O.fp(x), O.fp(w), O.fp(lam), O.ip(lv), c.to_c(), 0, O.fp(d0))
    L.orc_compute_deltap(1, O.ip(off), O.ip(idx), O.fp(x), O.fp(w), O.fp(lam), O.ip(lv), c.to_c(), 0, O.fp(d1))
    assert np.array_equal(d0, -d1)
    assert np.linalg.norm(d0) > 0


def test_free_fall_bitwise():
    # test_solver.cpp:214-245: one particle, substeps 1, no neighbours
    c = cfg_(h=0.1, substeps=1, dt_frame=0.004, range=IterationRange(1, 1), stab_iterations=0,
             mode=SolverMode.PBF, deterministic=True)
    s = ParticleSet(np.array([[0.3, 2.0, -0.1]], np.float32), 1.0, 1)
    sv = O.OracleSolver(c)
    mx = s.x[0].copy()
    mv = np.zeros(3, np.float32)
    dt = np.float32(0.004) / np.float32(1)
    g = np.array(c.gravity, np.float32)
    cap = np.float32(0.1) / dt
    for f in range(3):
        sv.step_frame_with_levels(s, f)
        mv = mv + dt * g
        xs = mx + dt * mv
        v = (xs - mx) / dt
        speed = np.sqrt(v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]))
        if speed > cap:
            v = v * (cap / speed)
        mx, mv = xs, v.astype(np.float32)
        assert np.array_equal(s.x[0], mx) and np.array_equal(s.v[0], mv)


def test_iteration_totals():
    # test_solver.cpp:285-307
    n = 8
    x = np.array([[0.4 * i, 0, 0] for i in range(n)], np.float32)
    c = cfg_(h=0.1, substeps=2, range=IterationRange(3, 6), deterministic=True, stab_iterations=0)
    s = ParticleSet(x, 0.001, 6)
    assert O.OracleSolver(c).step_frame_with_levels(s, 0).total_iterations == 6 * n * 2
    s2 = ParticleSet(x, 0.001, 6)
    s2.level = np.array([3, 4, 5, 6, 3, 4, 5, 6], np.int32)
    assert O.OracleSolver(c).step_frame_with_levels(s2, 0).total_iterations == 36 * 2


def test_nan_reported_with_pass_and_particle():
    # test_solver.cpp:532-550
    x = np.zeros((4, 3), np.float32)
    x[:, 0] = 0.5 * np.arange(4)
    x[2, 1] = np.nan
    s = ParticleSet(x, 1.0, 1)
    with pytest.raises(NumericalError) as e:
        O.OracleSolver(cfg_(h=0.1, range=IterationRange(1, 1), deterministic=True)).step_frame_with_levels(s, 0)
    assert e.value.pass_ == "predict" and e.value.particle == 2


def test_level_range_checked():
    # test_solver.cpp:676-690
    x = np.zeros((2, 3), np.float32)
    x[1, 0] = 1.0
    c = cfg_(range=IterationRange(3, 6))
    for bad in (7, 2):
        s = ParticleSet(x, 1.0, 6)
        s.level[1] = bad
        with pytest.raises(ValueError):
            O.OracleSolver(c).step_frame_with_levels(s, 0)


@pytest.mark.parametrize("field,value", [("dt_frame", 0.0), ("substeps", 0), ("rest_density", 0.0),
                                         ("h", -1.0), ("epsilon", -1e-9), ("stab_iterations", -1),
                                         ("stab_threshold", 7), ("particle_radius", -0.1),
                                         ("velocity_cap", -1.0), ("gravity", (0, float("nan"), 0))])
def test_config_validation(field, value):
    # test_solver.cpp:568-641
    c = cfg_()
    setattr(c, field, value)
    with pytest.raises(ValueError):
        c.validate()
    with pytest.raises(ValueError):
        O.OracleSolver(c)


# --------------------------------------------------------- LOD (test_lod.cpp)

def test_map_distance_to_level():
    # test_lod.cpp:37-55
    f = L.orc_map_distance_to_level
    assert f(5.5, 1.0, 10.0, 3, 6) == 5
    assert f(1.0, 1.0, 10.0, 3, 6) == 6
    assert f(10.0, 1.0, 10.0, 3, 6) == 3
    assert f(-5.0, 1.0, 10.0, 3, 6) == 6
    assert f(50.0, 1.0, 10.0, 3, 6) == 3
    assert f(2.0, 3.0, 3.0, 3, 6) == 6  # collapsed span -> full budget


def test_percentile_interpolates():
    # test_lod.cpp:231-238
    v = np.array([4, 1, 3, 2], np.float32)
    assert L.orc_percentile(O.fp(v), 4, 50.0) == 2.5
    assert L.orc_percentile(O.fp(v), 4, 0.0) == 1.0
    assert L.orc_percentile(O.fp(v), 4, 100.0) == 4.0


def test_dtvs_offscreen_and_behind_get_floor():
    # test_lod.cpp:129-140
    cam = Camera(eye=(0, 0, 5), look_at=(0, 0, 0))
    x = np.array([[0, 0, 0], [100, 0, 0], [0, 0, 10]], np.float32)
    lod = LodModelConfig(LodModel.DTVS, 0.0, 1.0, IterationRange(2, 7), True)
    lv = O.oracle_lod(x, cam, lod, 0.05)
    assert lv[1] == 2 and lv[2] == 2 and lv[0] == 7


# --------------------------------------------------------- SDF (test_collision_sdf.cpp)

def test_sdf_landmarks():
    # test_collision_sdf.cpp:35-55
    phi, g = O.oracle_scene_distance(SdfScene([HalfSpace((0, 2, 0), 1.0)]), [3, 4, 5])
    assert phi == 3.0 and np.array_equal(g, [0, 1, 0])
    phi, g = O.oracle_scene_distance(SdfScene([Sphere((0, 0, 0), 1.0)]), [0, 3, 0])
    assert phi == 2.0 and np.array_equal(g, [0, 1, 0])
    phi, g = O.oracle_scene_distance(SdfScene([Sphere((0, 0, 0), 1.0, True)]), [0, 0.25, 0])
    assert phi == 0.75 and np.array_equal(g, [0, -1, 0])  # interior: inward (sdf.hpp:157)
    phi, g = O.oracle_scene_distance(SdfScene([Box((0, 0, 0), (1, 1, 1))]), [3, 0, 0])
    assert phi == 2.0 and np.array_equal(g, [1, 0, 0])
    phi, _ = O.oracle_scene_distance(SdfScene([Cone((0, 0, 0), 1.0, 2.0)]), [0, 3, 0])
    assert phi == pytest.approx(1.0, rel=1e-6)  # apex distance (test_collision_sdf.cpp:83-99)


# ------------------------------------------------------- golden fixtures

def _g(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


@pytest.mark.parametrize("tag", ["dam_pbf_dtc", "dam_apbf_dtvs", "multi_apbf_dtc"])
def test_oracle_matches_reference_golden_solver(tag):
    g = _g(f"solver_{tag}.npz")
    name, scale, mode, model, n0, n1, frames = [str(v) for v in g["meta"]]
    spec = S.build_scenario(name, float(scale))
    spec.solver.mode = SolverMode[mode]
    spec.solver.range = IterationRange(int(n0), int(n1))
    spec.lod.model = LodModel[model]
    spec.lod.range = spec.solver.range
    st = ParticleSet()
    for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
        setattr(st, k, g[f"init_{k}"].copy())
    sv = O.OracleSolver(spec.solver, spec.scene)
    for f in range(int(frames)):
        s = sv.step_frame(st, spec.camera, spec.lod, f)
        assert s.total_iterations == g["stats"][f][0]
        assert s.contacts == g["stats"][f][1]
        assert s.min_density_pct == g["stats"][f][3]
        assert s.max_density_pct == g["stats"][f][4]
    for k in ("x", "x_star", "v", "lambda_", "level"):
        assert np.array_equal(getattr(st, k), g[k]), k


def test_oracle_matches_reference_golden_components():
    g = _g("components.npz")
    for tag in ("cloud", "dam"):
        p = g[tag]
        perm, origin, dims, cs = O.oracle_grid_build(p, 0.05, 0.05)
        assert np.array_equal(perm, g[f"{tag}_perm"])
        assert np.array_equal(origin, g[f"{tag}_origin"])
        assert np.array_equal(dims, g[f"{tag}_dims"])
        assert np.array_equal(cs, g[f"{tag}_cell_start"])
        off, idx = O.oracle_neighbor_lists(p, 0.05, 0.05)
        assert np.array_equal(off, g[f"{tag}_offsets"]) and np.array_equal(idx, g[f"{tag}_indices"])
        assert np.array_equal(O.oracle_all_densities(p, g[f"{tag}_mass"], 0.05), g[f"{tag}_rho"])
    spec = S.build_scenario("dam_break", 1728 / 216000)
    lod = LodModelConfig(LodModel.DTC, 0.0, 1.0, IterationRange(3, 6), True)
    assert np.array_equal(O.oracle_lod(g["dam"], spec.camera, lod), g["dam_dtc"])
    lod.model = LodModel.DTVS
    assert np.array_equal(O.oracle_lod(g["dam"], spec.camera, lod, 0.0125), g["dam_dtvs"])
    assert np.array_equal(O.oracle_splat(g["dam"], 0.0125, spec.camera), g["dam_depth"])
