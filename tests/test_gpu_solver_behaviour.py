"""The reference's own solver tests (test_solver.cpp, acceptance_main.cpp)
re-run on the GPU product path, plus full-size and long-horizon parity."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import (Camera, HalfSpace, IterationRange, LodModel, LodModelConfig,
                                   NumericalError, ParticleSet, SdfScene, Solver, SolverConfig,
                                   SolverMode)
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu


def cfg_(**kw):
    c = SolverConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def lattice(side, spacing, origin=(0, 0, 0)):
    idx = np.stack(np.meshgrid(np.arange(side), np.arange(side), np.arange(side), indexing="ij"), -1)
    pts = idx.reshape(-1, 3)[:, ::-1].astype(np.float64) * spacing + np.asarray(origin)
    return pts.astype(np.float32)


def test_free_fall_bitwise():
    # test_solver.cpp:214-245
    c = cfg_(h=0.1, substeps=1, dt_frame=0.004, range=IterationRange(1, 1), stab_iterations=0,
             mode=SolverMode.PBF, deterministic=True)
    s = ParticleSet(np.array([[0.3, 2.0, -0.1]], np.float32), 1.0, 1)
    sv = Solver(c)
    mx, mv = s.x[0].copy(), np.zeros(3, np.float32)
    dt = np.float32(0.004)
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


def test_uniform_budgets_make_both_modes_bit_identical():
    # test_solver.cpp:247-283 / acceptance criterion 1
    x = lattice(6, 0.024, (0, 0.024, 0))
    mass = 1000.0 * 0.024 ** 3
    c = cfg_(h=0.03, rest_density=1000.0, range=IterationRange(4, 4), deterministic=True,
             mode=SolverMode.PBF)
    ca = cfg_(h=0.03, rest_density=1000.0, range=IterationRange(4, 4), deterministic=True,
              mode=SolverMode.APBF)
    scene = SdfScene([HalfSpace((0, 1, 0), 0.0)])
    sp, sa = ParticleSet(x, mass, 4), ParticleSet(x, mass, 4)
    cam = Camera(eye=(0.3, 0.3, 0.5), look_at=(0.06, 0.06, 0.06))
    lod = LodModelConfig(LodModel.DTC)
    pbf, apbf = Solver(c, scene), Solver(ca, scene)
    for f in range(10):
        pbf.step_frame(sp, cam, lod, f)
        apbf.step_frame(sa, cam, lod, f)
        assert np.array_equal(sp.x, sa.x) and np.array_equal(sp.v, sa.v)
        assert (sp.level == 4).all() and (sa.level == 4).all()


def test_iteration_totals():
    # test_solver.cpp:285-307
    n = 8
    x = np.array([[0.4 * i, 0, 0] for i in range(n)], np.float32)
    c = cfg_(h=0.1, substeps=2, range=IterationRange(3, 6), deterministic=True, stab_iterations=0)
    s = ParticleSet(x, 0.001, 6)
    assert Solver(c).step_frame_with_levels(s, 0).total_iterations == 6 * n * 2
    s2 = ParticleSet(x, 0.001, 6)
    s2.level = np.array([3, 4, 5, 6, 3, 4, 5, 6], np.int32)
    assert Solver(c).step_frame_with_levels(s2, 0).total_iterations == 36 * 2


def test_particles_past_their_budget_freeze_mid_frame():
    # test_solver.cpp:309-350 through the iteration observer
    x = np.array([[0, 0, 0], [0.08, 0, 0]], np.float32)
    c = cfg_(h=0.1, rest_density=1000.0, range=IterationRange(1, 2), substeps=1, stab_iterations=0,
             gravity=(0, 0, 0), deterministic=True)
    s = ParticleSet(x, 0.64, 1)
    s.level = np.array([2, 1], np.int32)
    snaps = {}
    sv = Solver(c)
    sv.iteration_observer = lambda sub, it, st: snaps.__setitem__(
        it, (st.x_star.copy(), st.lambda_.copy(), st.level.copy()))
    stats = sv.step_frame_with_levels(s, 0)
    assert stats.total_iterations == 3
    assert sorted(snaps) == [1, 2]
    frozen = int(np.where(snaps[1][2] == 1)[0][0])
    live = 1 - frozen
    assert np.array_equal(snaps[1][0][frozen], snaps[2][0][frozen])
    assert snaps[1][1][frozen] == snaps[2][1][frozen] != 0.0
    assert not np.array_equal(snaps[1][0][live], snaps[2][0][live])


def test_zeroing_finished_neighbours_changes_trajectory():
    # test_solver.cpp:352-376
    x = np.array([[0, 0, 0], [0.08, 0, 0]], np.float32)
    base = dict(h=0.1, rest_density=1000.0, range=IterationRange(1, 2), substeps=1,
                stab_iterations=0, gravity=(0, 0, 0), deterministic=True)
    a = ParticleSet(x, 0.64, 1)
    a.level = np.array([2, 1], np.int32)
    b = a.copy()
    Solver(cfg_(**base)).step_frame_with_levels(a, 0)
    Solver(cfg_(inactive_lambda_zero=True, **base)).step_frame_with_levels(b, 0)
    assert not np.array_equal(a.x, b.x)


def test_residuals_decrease():
    # test_solver.cpp:426-447
    x = lattice(8, 0.08)
    c = cfg_(h=0.1, rest_density=1000.0, substeps=1, range=IterationRange(10, 10), stab_iterations=0,
             gravity=(0, 0, 0), record_residuals=True, deterministic=True)
    s = ParticleSet(x, 1.2 * 1000.0 * 0.08 ** 3, 10)
    st = Solver(c).step_frame_with_levels(s, 0)
    assert len(st.residuals) == 10
    assert 0.0 <= st.residuals[9] <= st.residuals[2]


def test_velocity_cap():
    # test_solver.cpp:506-530
    x = np.zeros((1, 3), np.float32)
    x[0, 1] = 100.0
    c = cfg_(h=0.1, substeps=1, dt_frame=0.01, range=IterationRange(1, 1), stab_iterations=0,
             gravity=(0, -1e4, 0), deterministic=True)
    s = ParticleSet(x, 1.0, 1)
    Solver(c).step_frame_with_levels(s, 0)
    assert np.linalg.norm(s.v[0]) == pytest.approx(0.1 / 0.01, rel=1e-6)
    c.velocity_cap = 0.5
    s2 = ParticleSet(x, 1.0, 1)
    Solver(c).step_frame_with_levels(s2, 0)
    assert np.linalg.norm(s2.v[0]) == pytest.approx(0.5, rel=1e-6)


def test_nan_reported_with_pass_and_particle():
    # test_solver.cpp:532-550
    x = np.zeros((4, 3), np.float32)
    x[:, 0] = 0.5 * np.arange(4)
    x[2, 1] = np.nan
    with pytest.raises(NumericalError) as e:
        Solver(cfg_(h=0.1, range=IterationRange(1, 1))).step_frame_with_levels(ParticleSet(x, 1.0, 1), 0)
    assert e.value.pass_ == "predict" and e.value.particle == 2


def test_nan_velocity_reports_finalize_like_oracle():
    x = lattice(3, 0.04)
    s = ParticleSet(x, 0.064, 2)
    s.v[5, 0] = np.inf
    c = cfg_(h=0.1, range=IterationRange(2, 2), substeps=1)
    with pytest.raises(NumericalError) as eg:
        Solver(c).step_frame_with_levels(s.copy(), 0)
    with pytest.raises(NumericalError) as eo:
        O.OracleSolver(c).step_frame_with_levels(s.copy(), 0)
    assert (eg.value.pass_, eg.value.particle) == (eo.value.pass_, eo.value.particle)


def test_level_range_checked():
    # test_solver.cpp:676-690
    x = np.zeros((2, 3), np.float32)
    x[1, 0] = 1.0
    c = cfg_(range=IterationRange(3, 6))
    for bad in (7, 2):
        s = ParticleSet(x, 1.0, 6)
        s.level[1] = bad
        with pytest.raises(ValueError):
            Solver(c).step_frame_with_levels(s, 0)


def test_config_validation_on_create():
    with pytest.raises(ValueError):
        Solver(cfg_(h=0.0))


def test_empty_state_steps():
    s = ParticleSet(np.zeros((0, 3), np.float32), 1.0, 6)
    st = Solver(cfg_()).step_frame(s, Camera(), LodModelConfig(), 3)
    assert st.frame == 3 and st.total_iterations == 0 and s.count() == 0


def test_frame_stats_densities_match_brute_force():
    # test_solver.cpp:643-674 (float tolerance)
    x = lattice(4, 0.024, (0, 0.024, 0))
    mass = 1000.0 * 0.024 ** 3
    c = cfg_(h=0.03, rest_density=1000.0, mode=SolverMode.PBF, deterministic=True)
    s = ParticleSet(x, mass, 6)
    st = Solver(c, SdfScene([HalfSpace((0, 1, 0), 0.0)])).step_frame(s, Camera(), LodModelConfig(), 7)
    h = np.float64(0.03)
    d = s.x.astype(np.float64)
    r2 = ((d[:, None, :] - d[None, :, :]) ** 2).sum(-1)
    w = np.where(r2 < h * h, 315 / (64 * math.pi * h ** 9) * (h * h - r2) ** 3, 0.0)
    rho = (w * np.float64(np.float32(mass))).sum(1) / 10.0
    assert st.frame == 7
    assert st.avg_density_pct == pytest.approx(rho.mean(), rel=1e-5)
    assert st.min_density_pct == pytest.approx(rho.min(), rel=1e-5)
    assert st.max_density_pct == pytest.approx(rho.max(), rel=1e-5)


# ------------------------------------------------ long horizon / full size

@pytest.mark.slow
@pytest.mark.parametrize("mode,rng,model", [(SolverMode.PBF, (5, 5), LodModel.DTC),
                                            (SolverMode.APBF, (5, 10), LodModel.DTVS),
                                            (SolverMode.APBF, (5, 10), LodModel.DTC)])
def test_c1_100_frames_bitwise(mode, rng, model):
    """BASELINE config C1: dam break 15,625, 100 steps, GPU == oracle bitwise."""
    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.mode = mode
    spec.solver.range = IterationRange(*rng)
    spec.lod.model = model
    spec.lod.range = spec.solver.range
    gpu, orc = Solver(spec.solver, spec.scene), O.OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 1)
    b = a.copy()
    gpu.upload(a)
    for f in range(100):
        sa = gpu.step_frame_resident(spec.camera, spec.lod, f)
        sb = orc.step_frame(b, spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts) == (sb.total_iterations, sb.contacts), f
    gpu.download(a)
    for k in ("x", "x_star", "v", "lambda_", "level"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.slow
def test_full_size_1m_frame_bitwise():
    """BASELINE config C3 at full size: one 1M-particle APBF/DTC frame."""
    spec = S.build_scenario("ocean_1m")
    gpu, orc = Solver(spec.solver, spec.scene), O.OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 1)
    b = a.copy()
    sa = gpu.step_frame(a, spec.camera, spec.lod, 0)
    sb = orc.step_frame(b, spec.camera, spec.lod, 0)
    assert (sa.total_iterations, sa.contacts) == (sb.total_iterations, sb.contacts)
    for k in ("x", "x_star", "v", "lambda_", "level"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    # size-independent properties at full size
    assert sa.total_iterations == spec.solver.substeps * int(a.level.astype(np.int64).sum())
    assert ((a.level >= 5) & (a.level <= 10)).all()


def test_full_size_c2_three_frames_bitwise():
    """BASELINE config C2 at full size: the 254,016-particle double dam break
    (APBF {5..10}, DTVS), three frames, every field bit-identical to the
    oracle; then 20 more resident frames stay finite and in range."""
    spec = S.build_scenario("double_dam_break", 0.3716)
    assert spec.particle_count() == 254016
    gpu, orc = Solver(spec.solver, spec.scene), O.OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 1)
    b = a.copy()
    for f in range(3):
        sa = gpu.step_frame(a, spec.camera, spec.lod, f)
        sb = orc.step_frame(b, spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct, sa.max_density_pct) == \
            (sb.total_iterations, sb.contacts, sb.min_density_pct, sb.max_density_pct), f
        for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)
    gpu.upload(a)
    for f in range(3, 23):
        gpu.step_frame_resident(spec.camera, spec.lod, f)
    gpu.download(a)
    assert np.isfinite(a.x).all() and np.isfinite(a.v).all()
    assert ((a.level >= 5) & (a.level <= 10)).all()


@pytest.mark.slow
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_tier_b_float_gpu_vs_reference_double():
    """Tier B: vs the shipped Solver<double>, positions within
    2x the reference's own float-vs-double divergence after K frames;
    particles matched by nearest position (no particle IDs exist)."""
    from scipy.spatial import cKDTree
    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.range = IterationRange(5, 10)
    spec.lod.range = spec.solver.range
    K = 10
    a = S.make_state(spec, 1)
    pos = S.spawn_scenario(spec, 1)
    m = S.scenario_mass(spec)
    n = pos.shape[0]
    d64 = O.RefState(pos, pos, np.zeros_like(pos), np.full(n, m), np.full(n, 1 / m), np.zeros(n),
                     np.full(n, 10, np.int32))
    d32 = O.RefState.from_set(a)
    g = Solver(spec.solver, spec.scene)
    r64, r32 = O.RefSolver(spec.solver, spec.scene, prec=8), O.RefSolver(spec.solver, spec.scene, prec=4)
    for f in range(K):
        g.step_frame(a, spec.camera, spec.lod, f)
        r64.step_frame(d64, spec.camera, spec.lod, f)
        r32.step_frame(d32, spec.camera, spec.lod, f)
    tree = cKDTree(d64.x)
    e_gpu = tree.query(a.x.astype(np.float64))[0].max()
    e_ref = tree.query(d32.x)[0].max()
    assert e_gpu <= 2 * e_ref + 1e-7
    assert e_gpu < 0.0125  # well below the lattice spacing 0.025


def test_frame_inputs_only_upload_matches_full_upload():
    """x*, lambda and level are dead inputs of stepFrame: uploading only x, v,
    mass and inv_mass (the e2e bench path) gives the same frames bit for bit,
    and stepFrameWithLevels refuses a state uploaded without levels."""
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.lod.model = LodModel.DTVS
    a = S.make_state(spec, 3)
    rng = np.random.default_rng(0)
    a.x_star[:] = rng.normal(size=a.x_star.shape)  # garbage the frame must not read
    a.lambda_[:] = rng.normal(size=a.lambda_.shape)
    b = a.copy()
    full, part = Solver(spec.solver, spec.scene), Solver(spec.solver, spec.scene)
    for f in range(3):
        full.upload(a)
        part.upload(b, frame_inputs_only=True)
        sa = full.step_frame_resident(spec.camera, spec.lod, f)
        sb = part.step_frame_resident(spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.min_density_pct) == (sb.total_iterations, sb.min_density_pct)
        full.download(a)
        part.download(b)
        for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)
    part.upload(b, frame_inputs_only=True)
    with pytest.raises(ValueError):
        part.step_frame_with_levels_resident(0)


def test_host_step_frame_follows_inverse_mass_mode_changes():
    """The host stepFrame launches with the previous upload's inverse-mass
    mode and scans the new one while the GPU runs; when the mode changed
    (uniform -> mixed -> non-finite -> uniform again with another value) the
    frame runs again: every frame equals a fresh solver's, bit for bit."""
    spec = S.build_scenario("dam_break", 4096 / 216000)
    base = S.make_state(spec, 5)
    states = [base.copy() for _ in range(4)]
    states[1].inv_mass[::5] = np.float32(0.0)                      # mixed, finite
    states[2].inv_mass[17] = np.float32(np.inf)                    # non-finite
    states[3].inv_mass[:] = np.float32(2.0) * states[3].inv_mass  # uniform, new w0
    states[3].mass[:] = np.float32(0.5) * states[3].mass
    reused = Solver(spec.solver, spec.scene)
    for f, st in enumerate(states + [base.copy()]):
        a, b = st.copy(), st.copy()
        errs = []
        for sv, s in ((reused, a), (Solver(spec.solver, spec.scene), b)):
            try:
                sv.step_frame(s, spec.camera, spec.lod, f)
                errs.append(None)
            except NumericalError as e:
                errs.append((e.pass_, e.particle))
        assert errs[0] == errs[1], f
        if errs[0] is None:
            for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
                assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)


@pytest.mark.parametrize("substeps", [1, 2, 3])
def test_state_set_rotation_and_graph_cache_bitwise(substeps):
    """Frames rotate through three state sets (period 3) with one cached CUDA
    Graph per start set: 10 resident frames and 3 host stepFrames (which
    restart from set 0) with odd and even substep counts stay equal to the
    oracle, bit for bit, through the eager, capture and replay phases."""
    spec = S.build_scenario("dam_break", 4096 / 216000)
    spec.solver.substeps = substeps
    gpu, orc = Solver(spec.solver, spec.scene), O.OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 4)
    b = a.copy()
    gpu.upload(a)
    for f in range(10):
        sa = gpu.step_frame_resident(spec.camera, spec.lod, f)
        sb = orc.step_frame(b, spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct) == \
            (sb.total_iterations, sb.contacts, sb.min_density_pct), f
    gpu.download(a)
    for f in range(10, 13):
        gpu.step_frame(a, spec.camera, spec.lod, f)
        orc.step_frame(b, spec.camera, spec.lod, f)
    for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


FIELDS7 = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")


@pytest.mark.parametrize("fault", ["nan_velocity", "blow_up"])
def test_failed_frame_leaves_caller_arrays_untouched(fault):
    """A frame that fails (NumericalError in predict, or the grid's cell-count
    guard) must not hand the caller a half-written state: the host stepFrame
    downloads overlap the frame, so a failure restores exactly the arrays the
    caller passed in -- in the eager first frame and in a replayed graph --
    and the solver carries on from its start state afterwards."""
    spec = S.build_scenario("dam_break", 4096 / 216000)
    spec.solver.range = IterationRange(3, 6)
    sv = Solver(spec.solver, spec.scene)
    orc = O.OracleSolver(spec.solver, spec.scene)
    good = S.make_state(spec, 2)
    ref = good.copy()
    for f in range(4):  # eager, capture, replay ...
        bad = good.copy()
        bad.x_star[:] = np.float32(7.0)  # not read by stepFrame, but must come back as passed
        bad.lambda_[:] = np.float32(-3.0)
        bad.level[:] = 4
        if fault == "nan_velocity":
            bad.v[123, 1] = np.nan
            exc = NumericalError
        else:
            bad.v[77, 0] = np.float32(1.25e8)  # x* 1e5 m away: > 2^26 grid cells
            exc = RuntimeError
        before = bad.copy()
        with pytest.raises(exc):
            sv.step_frame(bad, spec.camera, spec.lod, f)
        for k in FIELDS7:
            assert np.array_equal(getattr(bad, k), getattr(before, k), equal_nan=True), (f, k)
        sv.step_frame(good, spec.camera, spec.lod, f)
        orc.step_frame(ref, spec.camera, spec.lod, f)
        for k in FIELDS7:
            assert np.array_equal(getattr(good, k), getattr(ref, k)), (f, k)


def test_failed_resident_frame_keeps_start_state():
    """Resident frames: after a failure the device state is the frame-start
    state (step_frame_with_levels downloads it unchanged)."""
    spec = S.build_scenario("dam_break", 4096 / 216000)
    spec.solver.range = IterationRange(3, 6)
    st = S.make_state(spec, 3)
    st.level[:] = 5
    st.v[11, 0] = np.inf
    before = st.copy()
    sv = Solver(spec.solver, spec.scene)
    with pytest.raises(NumericalError):
        sv.step_frame_with_levels(st, 0)
    for k in FIELDS7:
        assert np.array_equal(getattr(st, k), getattr(before, k), equal_nan=True), k


def test_large_iteration_range_runs_like_oracle():
    """n_max past 1365 needs more than the 48 KB default of shared memory for
    the level tables (9 * (n_max + 1) ints in the stable level scatter): the
    kernels opt into the larger limit, so every n_max the config accepts runs."""
    x = lattice(4, 0.04, (0.2, 0.2, 0.2))
    c = cfg_(h=0.1, substeps=1, range=IterationRange(1500, 2000), mode=SolverMode.PBF)
    a = ParticleSet(x, 0.064, 2000)
    b = a.copy()
    sa = Solver(c).step_frame_with_levels(a, 0)
    sb = O.OracleSolver(c).step_frame_with_levels(b, 0)
    assert sa.total_iterations == sb.total_iterations == 64 * 2000
    for k in FIELDS7:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
