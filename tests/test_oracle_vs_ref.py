"""Pin the C restatement against the reference itself (oracle/_ref: the
unmodified /root/reference sources, Solver<float> through the Eigen shim).
Runs wherever oracle/_ref was built (this container); skipped elsewhere --
tests/golden carries the same evidence to machines without the reference."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import (Camera, IterationRange, LodModel, LodModelConfig, SolverMode)
from paper_1608_04721_b200 import scenario as S

pytestmark = [pytest.mark.ref,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

CASES = [
    ("dam_break", 1728 / 216000, dict(mode=SolverMode.PBF), LodModel.DTC, 1),
    ("dam_break", 3375 / 216000, dict(), LodModel.DTVS, 2),
    ("dam_break", 3375 / 216000, dict(inactive_lambda_zero=True), LodModel.DTC, 3),
    ("dam_break", 1728 / 216000, dict(stab_threshold=2, substeps=3), LodModel.DTVS, 4),
    ("dam_break", 1728 / 216000, dict(record_residuals=True, substeps=1), LodModel.DTC, 5),
    ("multi_dam_break", 0.05, dict(), LodModel.DTVS, 1),
    ("double_dam_break", 0.03, dict(range=IterationRange(2, 7)), LodModel.DTC, 1),
]


@pytest.mark.parametrize("name,scale,overrides,model,seed", CASES)
def test_restatement_bitwise_vs_reference_solver(name, scale, overrides, model, seed):
    spec = S.build_scenario(name, scale)
    for k, v in overrides.items():
        setattr(spec.solver, k, v)
    spec.lod.model = model
    spec.lod.range = spec.solver.range
    a = S.make_state(spec, seed)
    b = O.RefState.from_set(a)
    orc = O.OracleSolver(spec.solver, spec.scene)
    ref = O.RefSolver(spec.solver, spec.scene, prec=4)
    for f in range(4):
        sa = orc.step_frame(a, spec.camera, spec.lod, f)
        sb = ref.step_frame(b, spec.camera, spec.lod, f)
        for k in ("x", "x_star", "v", "lambda_", "mass", "inv_mass"):
            assert np.array_equal(getattr(a, k).astype(np.float64), getattr(b, k)), (f, k)
        assert np.array_equal(a.level, b.level)
        assert (sa.total_iterations, sa.contacts) == (sb.total_iterations, sb.contacts)
        assert sa.min_density_pct == sb.min_density_pct
        assert sa.max_density_pct == sb.max_density_pct
        assert sa.avg_density_pct == pytest.approx(sb.avg_density_pct, rel=1e-5)
        assert len(sa.residuals) == len(sb.residuals)
        assert sa.residuals == pytest.approx(sb.residuals, rel=1e-6)


def test_restatement_components_vs_reference():
    rng = np.random.default_rng(11)
    for p in (rng.uniform(0, 0.3, (257, 3)).astype(np.float32),
              rng.normal(0, 0.1, (500, 3)).astype(np.float32)):
        p64 = p.astype(np.float64)
        for h in (0.05, 0.07):
            g1 = O.oracle_grid_build(p, h, h)
            g2 = O.ref_grid_build(p64, h, h)
            assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[3], g2[3])
            assert np.array_equal(g1[1].astype(np.float64), g2[1]) and np.array_equal(g1[2], g2[2])
            o1, i1 = O.oracle_neighbor_lists(p, h, h)
            o2, i2 = O.ref_neighbor_lists(p64, h, h)
            assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
        m = rng.uniform(0.5, 2.0, p.shape[0]).astype(np.float32)
        assert np.array_equal(O.oracle_all_densities(p, m, 0.06).astype(np.float64),
                              O.ref_all_densities(p64, m.astype(np.float64), 0.06))
        cam = Camera(eye=(0.8, 0.6, 1.2), look_at=(0.1, 0.1, 0.1))
        for auto in (True, False):
            lod = LodModelConfig(LodModel.DTC, 0.2, 1.5, IterationRange(2, 9), auto)
            assert np.array_equal(O.oracle_lod(p, cam, lod), O.ref_lod_levels(p64, cam, lod))
            lod.model = LodModel.DTVS
            assert np.array_equal(O.oracle_lod(p, cam, lod, 0.02), O.ref_lod_levels(p64, cam, lod, 0.02))
        assert np.array_equal(O.oracle_splat(p, 0.02, cam).astype(np.float64), O.ref_splat(p64, 0.02, cam))
