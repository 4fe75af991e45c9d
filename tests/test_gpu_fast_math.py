"""The fast build of the solver passes (apbf_gpu_set_fast_math): FMA
contraction, |g|^2 = c^2 r^2 and 1/|r| from one rsqrt approximation in the
lambda / delta-p pair arithmetic, instead of the reference's correctly
rounded sqrt and division (kernels.hpp:52-65, solver.hpp:98-141).  Outside
the bitwise contract, so it is checked the way SURVEY.md 8c's tier B checks a
float run: against the shipped Solver<double>, positions within 2x the
reference's own float-vs-double divergence after K frames (particles matched
by nearest position); the LOD levels and iteration totals of the first frame
(computed before any solver arithmetic) stay exact."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import IterationRange, LodModel, Solver, SolverMode
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu


def c1(mode="dtvs"):
    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.range = spec.lod.range = IterationRange(5, 10)
    if mode == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
    return spec


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mode", ["dtvs", "pbf"])
def test_fast_build_within_tier_b_of_reference_double(mode):
    from scipy.spatial import cKDTree
    spec = c1(mode)
    K = 10
    a = S.make_state(spec, 1)
    d64 = O.RefState.from_set(a)  # the same float-rounded inputs
    d32 = O.RefState.from_set(a)
    g = Solver(spec.solver, spec.scene)
    g.set_fast_math(True)
    r64, r32 = O.RefSolver(spec.solver, spec.scene, prec=8), O.RefSolver(spec.solver, spec.scene, prec=4)
    for f in range(K):
        sg = g.step_frame(a, spec.camera, spec.lod, f)
        s64 = r64.step_frame(d64, spec.camera, spec.lod, f)
        s32 = r32.step_frame(d32, spec.camera, spec.lod, f)
        if f == 0:  # levels and totals come from the frame-start positions (float LOD)
            assert sg.total_iterations == s32.total_iterations
        assert abs(sg.avg_density_pct - s64.avg_density_pct) < 0.5
    tree = cKDTree(d64.x)
    e_fast = tree.query(a.x.astype(np.float64))[0].max()
    e_ref = tree.query(d32.x)[0].max()
    assert e_fast <= 2 * e_ref + 1e-7, (e_fast, e_ref)
    assert e_fast < 0.0125  # well below the lattice spacing 0.025
    assert np.isfinite(a.v).all()


def test_fast_build_first_frame_levels_exact_and_close_to_parity_build():
    """Full 1M ocean frame: identical levels and totalIterations, densities
    within a small band of the bitwise build."""
    spec = S.build_scenario("ocean_1m")
    a = S.make_state(spec, 1)
    b = a.copy()
    exact, fast = Solver(spec.solver, spec.scene), Solver(spec.solver, spec.scene)
    fast.set_fast_math(True)
    sa = exact.step_frame(a, spec.camera, spec.lod, 0)
    sb = fast.step_frame(b, spec.camera, spec.lod, 0)
    assert sa.total_iterations == sb.total_iterations
    assert np.array_equal(np.sort(a.level), np.sort(b.level))
    assert abs(sa.avg_density_pct - sb.avg_density_pct) < 1e-3
    assert abs(sa.max_density_pct - sb.max_density_pct) < 0.5
    assert np.isfinite(b.x).all() and np.isfinite(b.v).all()
    # off again: the bitwise build comes back (graph re-recorded)
    fast.set_fast_math(False)
    c = S.make_state(spec, 1)
    fast.step_frame(c, spec.camera, spec.lod, 0)
    for k in ("x", "v", "lambda_", "level"):
        assert np.array_equal(getattr(a, k), getattr(c, k)), k
