"""Host logic of the harness GPU backend (paper_1608_04721_b200/harness.py)
against the reference's own harness: the test_harness.cpp cases for the
metrics file, comparison, medians, bench-mode parsing and report formatting,
plus golden outputs of the reference's runScenario / parseBenchMode /
formatBenchReport (tests/golden/harness.npz, made by make_golden.py)."""
import json
import os

import numpy as np
import pytest

from paper_1608_04721_b200 import FrameStats, SolverMode
from paper_1608_04721_b200 import harness as H
from paper_1608_04721_b200 import scenario as S

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "harness.npz"))


def sample_report():
    """sampleReport (test_harness.cpp:40-56)."""
    r = H.RunReport(hash=0xdeadbeef12345678, echo=[("scenario", "sample"), ("mode", "apbf")])
    for f in range(3):
        r.frames.append(FrameStats(frame=f, wall_ms=2.125 + f, avg_density_pct=98.5 + 0.25 * f,
                                   min_density_pct=96.0625, max_density_pct=101.25,
                                   total_iterations=96000 + f, contacts=12 * f))
    return r


def test_metrics_round_trip_preserves_rows_hash_and_echo(tmp_path):
    path = tmp_path / "metrics.csv"
    rep = sample_report()
    H.write_metrics_csv(path, rep)
    lines = path.read_text().splitlines()
    assert lines[:4] == ["# scenario = sample", "# mode = apbf", "# scenario_hash = deadbeef12345678",
                         H.METRICS_HEADER]
    parsed = H.read_metrics_csv(path)
    assert parsed.hash == rep.hash
    assert len(parsed.rows) == 3
    for row, st in zip(parsed.rows, rep.frames):
        assert (row.frame, row.time_ms, row.avg_density_pct, row.min_density_pct, row.max_density_pct,
                row.total_iterations, row.contacts) == (
            st.frame, st.wall_ms, st.avg_density_pct, st.min_density_pct, st.max_density_pct,
            st.total_iterations, st.contacts)


def test_deterministic_reports_zero_out_the_time_column(tmp_path):
    rep = sample_report()
    rep.zero_time = True
    H.write_metrics_csv(tmp_path / "m.csv", rep)
    assert all(r.time_ms == 0.0 for r in H.read_metrics_csv(tmp_path / "m.csv").rows)


def test_metrics_reader_rejects_broken_files(tmp_path):
    with pytest.raises(RuntimeError):
        H.read_metrics_csv(tmp_path / "missing.csv")
    (tmp_path / "noheader.csv").write_text("# only comments\n")
    with pytest.raises(RuntimeError):
        H.read_metrics_csv(tmp_path / "noheader.csv")
    (tmp_path / "badrow.csv").write_text(H.METRICS_HEADER + "\n0,aa,bb\n")
    with pytest.raises(RuntimeError, match=":2: malformed"):
        H.read_metrics_csv(tmp_path / "badrow.csv")
    (tmp_path / "badhead.csv").write_text("frame,time\n")
    with pytest.raises(RuntimeError, match=":1: unexpected metrics header"):
        H.read_metrics_csv(tmp_path / "badhead.csv")


def test_run_comparison_measures_the_density_delta():
    ref = H.MetricsFile(hash=0x1111, rows=[H.MetricsRow(frame=f, avg_density_pct=100.0 + 0.1 * f)
                                           for f in range(5)])
    same = H.MetricsFile(ref.hash, [H.MetricsRow(**vars(r)) for r in ref.rows])
    eq = H.compare_runs(ref, same, 4.0)
    assert (eq.max_delta, eq.frames, eq.passed) == (0.0, 5, True)
    shifted = H.MetricsFile(ref.hash, [H.MetricsRow(frame=r.frame, avg_density_pct=r.avg_density_pct + 5)
                                       for r in ref.rows])
    fail = H.compare_runs(ref, shifted, 4.0)
    assert fail.max_delta == pytest.approx(5.0, rel=1e-12) and not fail.passed
    assert H.compare_runs(ref, shifted, 6.0).passed
    with pytest.raises(RuntimeError, match="hash mismatch"):
        H.compare_runs(ref, H.MetricsFile(0x2222, ref.rows), 4.0)
    H.compare_runs(ref, H.MetricsFile(None, ref.rows), 4.0)
    with pytest.raises(RuntimeError, match="frame count mismatch"):
        H.compare_runs(ref, H.MetricsFile(ref.hash, ref.rows[:-1]), 4.0)


def test_median_of_and_report_aggregates():
    assert H.median_of([3.0, 1.0, 2.0]) == 2.0
    assert H.median_of([4.0, 1.0, 3.0, 2.0]) == 2.5
    assert H.median_of([5.0]) == 5.0
    with pytest.raises(ValueError):
        H.median_of([])
    rep = sample_report()
    assert rep.median_frame_ms() == 3.125
    assert rep.total_iterations() == 3 * 96000 + 3
    assert rep.total_contacts() == 36


def test_reads_the_reference_runscenario_metrics_file(tmp_path):
    """metrics.csv written by the reference's runScenario parses, and its
    header is exactly the echo + hash this harness writes for the same run."""
    text = str(GOLD["metrics_dam_apbf"][0])
    (tmp_path / "ref.csv").write_text(text)
    mf = H.read_metrics_csv(tmp_path / "ref.csv")
    assert len(mf.rows) == 10 and all(r.time_ms == 0.0 for r in mf.rows)
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.solver.mode = SolverMode.APBF
    spec.solver.deterministic = True
    opt = H.RunOptions(mode=SolverMode.APBF, frames=10, seed=1, deterministic=True)
    echo = H.build_echo(spec, opt, 10, spec.particle_count())
    mine = [f"# {k} = {v}" for k, v in echo] + ["# scenario_hash = %016x" % S.scenario_hash(spec, 1),
                                                H.METRICS_HEADER]
    assert [l for l in text.splitlines() if l.startswith("#") or l.startswith("frame,")] == mine
    assert mf.hash == S.scenario_hash(spec, 1)


def test_bench_mode_parsing_matches_the_reference():
    g = json.loads(str(GOLD["bench"][0]))
    for token, want in g["modes"].items():
        if isinstance(want, str):
            with pytest.raises(ValueError) as e:
                H.parse_bench_mode(token)
            assert str(e.value) == want, token
        else:
            m = H.parse_bench_mode(token)
            lod = -1 if m.lod_model is None else int(m.lod_model)
            assert [0 if m.mode == SolverMode.PBF else 1, m.pbf_iterations, lod] == want, token
            assert m.token == token
    modes = H.parse_bench_modes("pbf:6,apbf:dtc")
    assert [m.token for m in modes] == ["pbf:6", "apbf:dtc"]
    with pytest.raises(ValueError):
        H.parse_bench_modes("")


def test_bench_report_text_matches_the_reference():
    g = json.loads(str(GOLD["bench"][0]))
    for rep, text in zip(g["reports"], g["texts"]):
        rs = [H.BenchResult(t, m, i, f, p) for t, m, i, f, p in rep]
        assert H.format_bench_report(rs) == text


def test_particle_snapshot_text_matches_the_reference(tmp_path):
    from paper_1608_04721_b200 import ParticleSet, write_particle_snapshot
    st = ParticleSet(GOLD["state_dam_f1_x"], 1.0, 1)
    st.level = GOLD["state_dam_f1_level"].copy()
    write_particle_snapshot(tmp_path / "p.csv", st)
    assert (tmp_path / "p.csv").read_text() == str(GOLD["snapshot_dam_f1"][0])


def test_ppm_writer_round_trip(tmp_path):
    from paper_1608_04721_b200 import read_ppm, write_ppm
    img = GOLD["image_dam_f1"]
    write_ppm(img, tmp_path / "f.ppm")
    data = (tmp_path / "f.ppm").read_bytes()
    assert data.startswith(b"P6\n256 256\n255\n") and len(data) == 15 + 256 * 256 * 3
    assert np.array_equal(read_ppm(tmp_path / "f.ppm"), img)
