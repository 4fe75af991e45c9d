"""Multi-camera LOD: blendLod on the device
(test_lod.cpp:240-259) and the multi-camera frame -- each camera's
assignLevels, blended, then stepFrameWithLevels -- against the float oracle
composing the same reference calls."""
import numpy as np
import pytest

from oracle.oracle import OracleSolver, oracle_lod
from paper_1608_04721_b200 import (Camera, IterationRange, LodModel, LodModelConfig, Solver, SolverMode,
                                   blend_lod)
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu
FIELDS = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")


def test_blend_keeps_the_highest_level_per_particle():
    a = np.array([3, 6, 4, 5], np.int32)
    b = np.array([5, 4, 4, 6], np.int32)
    out = blend_lod([a, b])
    assert out.tolist() == [5, 6, 4, 6]
    assert np.array_equal(blend_lod([a]), a)
    assert np.array_equal(blend_lod([out, a]), out)
    with pytest.raises(ValueError):
        blend_lod([a, np.array([1, 2, 3], np.int32)])
    with pytest.raises(ValueError):
        blend_lod([])
    rng = np.random.default_rng(3)
    many = [rng.integers(1, 20, 10000).astype(np.int32) for _ in range(5)]
    assert np.array_equal(blend_lod(many), np.maximum.reduce(many))


@pytest.mark.parametrize("models", [(LodModel.DTC, LodModel.DTC), (LodModel.DTVS, LodModel.DTC),
                                    (LodModel.DTVS, LodModel.DTVS)])
def test_multi_camera_frames_match_the_oracle(models):
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.solver.range = IterationRange(3, 8)
    cam2 = Camera(eye=(-1.0, 0.6, 0.4), look_at=(0.3, 0.1, 0.3), up=(0, 1, 0), width=160, height=120)
    cams = [spec.camera, cam2]
    lods = [LodModelConfig(m, 0.0, 1.0, IterationRange(1, 2), True) for m in models]  # range ignored:
    gpu = Solver(spec.solver, spec.scene)                                               # the solver's wins
    orc = OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 2)
    b = a.copy()
    r = spec.solver.effective_particle_radius()
    for f in range(4):
        sa = gpu.step_frame_multi(a, cams, lods, f)
        per = []
        for c, l in zip(cams, lods):
            lc = LodModelConfig(l.model, l.d_min, l.d_max, spec.solver.range, l.auto_range)
            per.append(oracle_lod(b.x, c, lc, r if l.model == LodModel.DTVS else None))
        b.level = np.maximum.reduce(per).astype(np.int32)
        sb = orc.step_frame_with_levels(b, f)
        assert (sa.total_iterations, sa.contacts) == (sb.total_iterations, sb.contacts)
        for k in FIELDS:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)


def test_multi_camera_with_one_camera_is_step_frame_and_pbf_is_uniform():
    spec = S.build_scenario("dam_break", 8000 / 216000)
    one, ref = Solver(spec.solver, spec.scene), Solver(spec.solver, spec.scene)
    a = S.make_state(spec, 4)
    b = a.copy()
    for f in range(3):
        one.step_frame_multi(a, [spec.camera], [spec.lod], f)
        ref.step_frame(b, spec.camera, spec.lod, f)
        for k in FIELDS:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)
    spec.solver.mode = SolverMode.PBF
    pbf = Solver(spec.solver, spec.scene)
    c = S.make_state(spec, 4)
    st = pbf.step_frame_multi(c, [spec.camera, spec.camera], [spec.lod, spec.lod], 0)
    assert (c.level == spec.solver.range.n_max).all()
    assert st.total_iterations == c.count() * spec.solver.range.n_max * spec.solver.substeps
    with pytest.raises(ValueError):
        pbf.step_frame_multi(c, [], [], 0)
