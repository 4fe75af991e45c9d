"""The harness GPU backend end to end: runScenario on
the B200 writes the reference's metrics.csv and frame dumps; its frames equal
the float oracle's; the reference's own compareRuns accepts it against the
reference's Solver<double> run; the level image rendered on the device and
the particle snapshot equal the reference's renderLevelImage<float> /
writeParticleSnapshot<float> of the same state, byte for byte."""
import os

import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_1608_04721_b200 import (Camera, IterationRange, LodModel, SolverMode, read_ppm,
                                   render_level_image)
from paper_1608_04721_b200 import harness as H
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "harness.npz"))


def test_run_scenario_writes_metrics_and_frame_dumps(tmp_path):
    """runScenario writes metrics and frame dumps (test_harness.cpp:515-561)."""
    spec = S.build_scenario("dam_break", 0.001)
    opt = H.RunOptions(mode=SolverMode.APBF, frames=2, seed=11, deterministic=True, out_dir=str(tmp_path),
                       dump_images_every=1, dump_particles_every=1)
    rep = H.run_scenario(spec, opt)
    assert len(rep.frames) == 2 and rep.zero_time
    assert rep.hash == S.scenario_hash(spec, 11)
    echo = dict(rep.echo)
    assert (echo["scenario"], echo["particles"], echo["frames"], echo["mode"], echo["deterministic"]) == \
        ("dam_break", "216", "2", "apbf", "1")
    for f in ("metrics.csv", "frame_000000.ppm", "frame_000001.ppm", "particles_000000.csv",
              "particles_000001.csv"):
        assert (tmp_path / f).exists(), f
    mf = H.read_metrics_csv(tmp_path / "metrics.csv")
    assert mf.hash == rep.hash
    assert [(r.frame, r.time_ms, r.total_iterations) for r in mf.rows] == \
        [(f, 0.0, rep.frames[f].total_iterations) for f in range(2)]
    # the dumps equal the reference's float renderer / snapshot of the same state
    assert np.array_equal(read_ppm(tmp_path / "frame_000001.ppm"), GOLD["image_dam_f1"])
    assert (tmp_path / "particles_000001.csv").read_text() == str(GOLD["snapshot_dam_f1"][0])


def test_run_scenario_honors_mode_and_range_overrides():
    spec = S.build_scenario("dam_break", 0.001)
    rep = H.run_scenario(spec, H.RunOptions(mode=SolverMode.PBF, range=IterationRange(2, 2), frames=1,
                                            deterministic=True))
    assert rep.frames[0].total_iterations == 2 * 216 * spec.solver.substeps
    echo = dict(rep.echo)
    assert echo["mode"] == "pbf" and echo["iterations"] == "2..2"


def test_bench_totals_are_exact_for_uniform_budgets_and_bounded_otherwise():
    spec = S.build_scenario("dam_break", 0.001)
    frames, n, sub = 2, 216, spec.solver.substeps
    res = H.run_bench(spec, H.parse_bench_modes("pbf:6,pbf:3,apbf:dtc"), 1, frames, 1)
    assert res[0].iterations == 6 * n * frames * sub
    assert res[1].iterations == 3 * n * frames * sub
    assert 3 * n * frames * sub <= res[2].iterations < 6 * n * frames * sub
    assert (res[0].particles, res[0].frames) == (216, frames) and res[0].median_frame_ms >= 0.0
    table = H.format_bench_report(res)
    for s in ("speedup (t_pbf-t_apbf)/t_apbf", "reduction (t_pbf-t_apbf)/t_pbf", "iteration ratio",
              "apbf:dtc"):
        assert s in table
    with pytest.raises(ValueError):
        H.run_bench(spec, H.parse_bench_modes("pbf:6"), 0, 1, 1)


@pytest.mark.parametrize("key,mode,rng,frames", [("metrics_dam_apbf", SolverMode.APBF, None, 10),
                                                  ("metrics_dam_pbf3", SolverMode.PBF, IterationRange(3, 3), 4)])
def test_gpu_run_passes_the_reference_compare_and_equals_the_float_oracle(tmp_path, key, mode, rng, frames):
    spec = S.build_scenario("dam_break", 8000 / 216000)
    opt = H.RunOptions(mode=mode, range=rng, frames=frames, seed=1, deterministic=True, out_dir=str(tmp_path))
    rep = H.run_scenario(spec, opt)
    (tmp_path / "ref.csv").write_text(str(GOLD[key][0]))
    ref = H.read_metrics_csv(tmp_path / "ref.csv")
    gpu = H.read_metrics_csv(tmp_path / "metrics.csv")
    # same header as the reference's file (echo + hash): the runs are comparable
    head = lambda p: [l for l in p.read_text().splitlines() if l.startswith("#")]  # noqa: E731
    assert head(tmp_path / "metrics.csv") == head(tmp_path / "ref.csv")
    cmp = H.compare_runs(ref, gpu, 4.0)  # the reference CLI's default tolerance
    assert cmp.passed and cmp.frames == frames, cmp
    if mode == SolverMode.PBF:  # uniform budgets: iteration totals are exact in any precision
        assert [r.total_iterations for r in gpu.rows] == [r.total_iterations for r in ref.rows]
    # the float frames themselves are the oracle's, bit for bit
    s = spec
    if rng is not None:
        s.solver.range = rng
        s.lod.range = rng
    s.solver.mode = mode
    orc = OracleSolver(s.solver, s.scene)
    st = S.make_state(s, 1)
    for f, got in enumerate(rep.frames):
        want = orc.step_frame(st, s.camera, s.lod, f)
        assert (got.total_iterations, got.contacts, got.min_density_pct, got.max_density_pct) == \
            (want.total_iterations, want.contacts, want.min_density_pct, want.max_density_pct), f
        assert got.avg_density_pct == pytest.approx(want.avg_density_pct, rel=1e-9)


def test_render_level_image_matches_the_reference_float_renderer():
    spec = S.build_scenario("dam_break", 8000 / 216000)
    img = render_level_image(GOLD["render_x"], GOLD["render_level"], 0.0125, spec.camera, IterationRange(3, 6))
    assert np.array_equal(img, GOLD["render_image"])
    # nothing visible: black; radius must be positive; levels must match positions
    cam = Camera(eye=(0, 0, -5), look_at=(0, 0, -10), up=(0, 1, 0), width=32, height=16)
    assert not render_level_image(GOLD["render_x"], GOLD["render_level"], 0.0125, cam,
                                  IterationRange(3, 6)).any()
    with pytest.raises(ValueError):
        render_level_image(GOLD["render_x"], GOLD["render_level"], 0.0, spec.camera, IterationRange(3, 6))
    with pytest.raises(ValueError):
        render_level_image(GOLD["render_x"], GOLD["render_level"][:5], 0.0125, spec.camera,
                           IterationRange(3, 6))
