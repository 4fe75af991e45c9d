"""The reference's acceptance criteria (tests/acceptance_main.cpp, SPEC.md
559-570) re-run on the B200 product path.  Where a criterion's bar is about the
CPU's wall clock at 27k particles it is checked where a GPU frame is not
launch-bound (1M particles, the BASELINE workload)."""
import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_1608_04721_b200 import (Camera, HalfSpace, IterationRange, LodModel, LodModelConfig, ParticleSet,
                                   SdfScene, Solver, SolverConfig, SolverMode, lod_dtvs)
from paper_1608_04721_b200 import harness as H
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu


def test_criterion_2_3_density_tracks_pbf_and_adaptivity_cuts_work():
    """C2: |avg density| of APBF DTVS/DTC within 4 pct pts of PBF6 over 300
    frames; C3 (work part): APBF iteration totals < 0.85 x PBF6 and > PBF3
    (acceptance_main.cpp:28-50, 115-160)."""
    spec = S.build_scenario("dam_break", 1.0 / 27.0)
    base = dict(frames=300, seed=1, deterministic=True)
    pbf6 = H.run_scenario(spec, H.RunOptions(mode=SolverMode.PBF, range=IterationRange(6, 6), **base))
    dtvs = H.run_scenario(spec, H.RunOptions(mode=SolverMode.APBF, lod_model=LodModel.DTVS, **base))
    dtc = H.run_scenario(spec, H.RunOptions(mode=SolverMode.APBF, lod_model=LodModel.DTC, **base))

    def rows(rep):
        return H.MetricsFile(rep.hash, [H.MetricsRow(frame=f.frame, avg_density_pct=f.avg_density_pct)
                                        for f in rep.frames])
    assert H.compare_runs(rows(pbf6), rows(dtvs), 4.0).passed
    assert H.compare_runs(rows(pbf6), rows(dtc), 4.0).passed
    it6 = pbf6.total_iterations()
    for rep in (dtvs, dtc):
        assert it6 / 2 < rep.total_iterations() < 0.85 * it6


def test_criterion_3_wall_clock_reduction_at_1m():
    """C3 (time part), with the reference's own bar and protocol
    (acceptance_main.cpp:145-153): runBench over 80 frames -- "the settled
    regime where constraint work dominates the fixed per-frame costs" -- and
    a median-frame reduction (t_pbf - t_apbf) / t_pbf >= 15% for DTVS or DTC.
    On the BASELINE 1M ocean, APBF {5..10} vs PBF 10 (a 27k frame is
    launch-bound on a B200).  Measured: DTC 15.8%, DTVS 13.2%
    (profiles/README.md); the remaining gap to the 24% iteration cut is the
    per-frame fixed cost (grid, lists, LOD)."""
    spec = S.build_scenario("ocean_1m")
    res = H.run_bench(spec, H.parse_bench_modes("pbf:10,apbf:dtvs,apbf:dtc"), 1, 80, 1)
    t_pbf = res[0].median_frame_ms
    red = [(t_pbf - r.median_frame_ms) / t_pbf for r in res[1:]]
    assert red[0] >= 0.15 or red[1] >= 0.15, (H.format_bench_report(res), red)
    assert min(red) > 0.08, red  # both modes cut the frame


def test_criterion_4_residual_decreases_over_iterations():
    """C4 (convergence part): mean |density error| after 10 iterations <= after
    3, on a uniform-mass 20^3 lattice at 0.8 h spacing (acceptance_main.cpp:166-180)."""
    h, spacing = 0.05, 0.8 * 0.05
    g = np.stack(np.meshgrid(*[np.arange(20)] * 3, indexing="ij"), -1).reshape(-1, 3)
    x = (g * spacing).astype(np.float32)
    cfg = SolverConfig(h=h, rest_density=1000.0, gravity=(0.0, 0.0, 0.0), substeps=1,
                       range=IterationRange(10, 10), record_residuals=True, deterministic=True)
    st = ParticleSet(x, float(np.float32(1000.0 * spacing ** 3)), 10)
    stats = Solver(cfg).step_frame_with_levels(st, 0)
    assert stats.residuals[9] <= stats.residuals[2]


def test_criterion_8_prestabilization_slows_the_first_frame():
    """C8 (first part): a particle pushed 1.5 radii into the floor leaves its
    first frame no faster with pre-stabilization than without
    (acceptance_main.cpp:416-441)."""
    scene = SdfScene([HalfSpace((0.0, 1.0, 0.0), 0.0)])
    base = SolverConfig(h=0.05, substeps=1, range=IterationRange(1, 2), stab_threshold=2, deterministic=True)
    r = base.effective_particle_radius()
    x = np.array([[0.0, -0.5 * r, 0.0]], np.float32)

    def speed(stab):
        cfg = SolverConfig(**{**base.__dict__, "stab_iterations": stab})
        st = ParticleSet(x, 0.015625, 1)
        Solver(cfg, scene).step_frame_with_levels(st, 0)
        return float(np.linalg.norm(st.v[0]))
    assert speed(2) <= speed(0)


def test_criterion_9_dtvs_prefers_the_visible_slab():
    """C9: with one slab occluding another, DTVS gives the visible slab the
    higher mean level, all levels within range (acceptance_main.cpp:456-496)."""
    side, per = 20, 400
    rng = S.splitmix64(1212, 2 * per * 3)
    sym = S.symmetric(rng).reshape(2 * per, 3)  # SplitMix64::symmetric, x/y/z draw order per particle
    x = np.empty((2 * per, 3))
    k = 0
    for z in (-3.0, -4.5):
        for iy in range(side):
            for ix in range(side):
                x[k] = (-0.95 + 0.1 * ix + 0.01 * sym[k, 0], -0.95 + 0.1 * iy + 0.01 * sym[k, 1],
                        z + 0.01 * sym[k, 2])
                k += 1
    cam = Camera(eye=(0, 0, 0), look_at=(0, 0, -1), width=256, height=256)
    lod = LodModelConfig(LodModel.DTVS, 0.0, 1.0, IterationRange(3, 6), True)
    lv = lod_dtvs(x.astype(np.float32), cam, lod, 0.06)
    assert lv[:per].mean() > lv[per:].mean()
    assert lv.min() >= 3 and lv.max() <= 6


def test_criterion_10_thousand_frame_soak_bitwise():
    """C10: 1000 frames of the 8640-particle multi dam break (cone scene,
    APBF {4..8} DTVS): everything finite, speeds within the cap, levels in
    range -- and the final state equal to the float oracle's, bit for bit."""
    spec = S.build_scenario("multi_dam_break", 1.0 / 27.0)
    gpu, orc = Solver(spec.solver, spec.scene), OracleSolver(spec.solver, spec.scene)
    a = S.make_state(spec, 1)
    b = a.copy()
    cap = spec.solver.effective_velocity_cap()
    gpu.upload(a)
    max_speed = 0.0
    for f in range(1000):
        gpu.step_frame_resident(spec.camera, spec.lod, f)
        if f % 100 == 99:
            gpu.download(a)
            assert np.isfinite(a.x).all() and np.isfinite(a.v).all() and np.isfinite(a.x_star).all()
            sp = np.linalg.norm(a.v.astype(np.float64), axis=1).max()
            max_speed = max(max_speed, sp)
            assert sp <= cap * (1 + 1e-6)
            assert a.level.min() >= spec.solver.range.n_min and a.level.max() <= spec.solver.range.n_max
    gpu.download(a)
    for f in range(1000):
        orc.step_frame(b, spec.camera, spec.lod, f)
    for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
