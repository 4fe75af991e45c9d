"""Eager launches (APBF_GRAPHS=0) must give the CUDA Graph replay's frames
bit for bit; the list-stride fallback (per-warp allocated slabs for very
long lists) must match the oracle."""
import numpy as np
import pytest

from paper_1608_04721_b200 import IterationRange, LodModel, ParticleSet, Solver
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu

FIELDS = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")
VARIANTS = [
    {"APBF_GRAPHS": "0"},
]


def frames(spec, n, seed=1):
    sv = Solver(spec.solver, spec.scene)
    st = S.make_state(spec, seed)
    stats = [sv.step_frame(st, spec.camera, spec.lod, f) for f in range(n)]
    return st, [(s.total_iterations, s.contacts, s.min_density_pct, s.max_density_pct) for s in stats]


def spec_apbf(zero_lambda):
    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.range = IterationRange(5, 10)
    spec.solver.inactive_lambda_zero = zero_lambda
    spec.lod.range = spec.solver.range
    spec.lod.model = LodModel.DTVS
    return spec


@pytest.mark.parametrize("zero_lambda", [False, True])
@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_matches_default(monkeypatch, env, zero_lambda):
    spec = spec_apbf(zero_lambda)
    ref, ref_stats = frames(spec, 5)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got, got_stats = frames(spec, 5)
    assert got_stats == ref_stats
    for k in FIELDS:
        assert np.array_equal(getattr(ref, k), getattr(got, k)), k


def test_dense_cluster_switches_to_allocated_list_slabs():
    """Spacing h/4 gives ~270 neighbours per particle, far past the initial
    64-row slab stride and the 128-row cap: the build flags the overflow, the
    host switches to per-warp slabs from the allocating builder and re-runs
    the frame, which must still match the oracle."""
    from oracle.oracle import OracleSolver
    h = 0.1
    side = 14
    g = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    x = (g * (h / 4) + 0.5).astype(np.float32)
    cfg = S.build_scenario("dam_break", 0.01).solver
    cfg.h = h
    cfg.range = IterationRange(2, 3)
    a = ParticleSet(x, 0.002, 3)
    b = a.copy()
    gpu = Solver(cfg)
    sa = gpu.step_frame_with_levels(a, 0)
    sb = OracleSolver(cfg).step_frame_with_levels(b, 0)
    assert sa.total_iterations == sb.total_iterations
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    entries, _ = gpu.last_neighbor_stats()
    assert entries / a.count() > 100


def test_host_xstar_equals_x_after_clean_frames():
    """stepFrame on host arrays writes back x* == x bitwise after finalize
    (x = x*, solver.hpp:347-356)."""
    spec = spec_apbf(False)
    sv = Solver(spec.solver, spec.scene)
    st = S.make_state(spec, 1)
    for f in range(3):
        sv.step_frame(st, spec.camera, spec.lod, f)
        assert np.array_equal(st.x, st.x_star)
