"""Every solver-pass variant selectable by environment (A/B switches read at
Solver creation) must give the default path's frames bit for bit: compact
16-bit lists with and without the coefficient cache, the coefficient cache
itself, shared-memory list staging, the cell-tile solver, gather batch sizes,
CTA size, eager launches instead of CUDA Graph replay, the iteration order
window-sorted by list length.  Also the compact
lists' range fallback and the list stride fallback."""
import numpy as np
import pytest

from paper_1608_04721_b200 import IterationRange, LodModel, ParticleSet, Solver
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu

FIELDS = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")
VARIANTS = [
    {"APBF_C16": "1"},
    {"APBF_C16": "1", "APBF_COEF_CACHE": "1"},
    {"APBF_COEF_CACHE": "1"},
    {"APBF_STAGE_LISTS": "1"},
    {"APBF_TILES": "1"},
    {"APBF_CHUNK": "1"},
    {"APBF_CHUNK": "2"},
    {"APBF_CHUNK": "8"},
    {"APBF_BLOCK": "256"},
    {"APBF_GRAPHS": "0"},
    {"APBF_WSORT": "1"},
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


def test_compact_lists_fall_back_when_offsets_overflow(monkeypatch):
    """A 3000-cell-long sheet puts > 2^14 slots between a particle's first
    and last candidate rows of one layer: the compact build flags it and the
    frame is re-run on 32-bit lists, with the same result as starting there."""
    h = 0.1
    nx, ny = 6000, 6  # 2 particles per cell along x and y
    xs, ys = np.meshgrid(np.arange(nx) * (h / 2), np.arange(ny) * (h / 2), indexing="ij")
    x = np.stack([xs.ravel(), ys.ravel(), np.full(xs.size, 0.5)], 1).astype(np.float32)
    cfg = S.build_scenario("dam_break", 0.01).solver
    cfg.h = h
    cfg.range = IterationRange(2, 3)
    cfg.gravity = (0.0, 0.0, 0.0)
    base = ParticleSet(x, 0.01, 3)
    a = base.copy()
    Solver(cfg).step_frame_with_levels(a, 0)
    monkeypatch.setenv("APBF_C16", "1")
    b = base.copy()
    Solver(cfg).step_frame_with_levels(b, 0)
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


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
