"""Harness GPU backend: runScenario / runBench and the
metrics.csv format, mirroring the reference's src/runner.{hpp,cpp},
src/metrics.{hpp,cpp} and src/bench.{hpp,cpp}, with the frames stepped by
the B200 solver (state resident on the device between frames; only the dumps
a run asks for are rendered or downloaded).

Same names, options, file formats and error behaviour as the reference, so a
GPU run's metrics.csv is read and compared by the reference's own
`apbf compare` (metrics.cpp:112-131), and the frame dumps are the files
runScenario writes (runner.cpp:85-93).  The C++ drop-in of the same harness
is include/apbf_gpu/runner.hpp.
"""
from __future__ import annotations

import copy
import os
import re
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

from .api import (FrameStats, IterationRange, LodModel, Solver, SolverMode, write_particle_snapshot,
                  write_ppm)
from . import scenario as S

# metrics.cpp:13-14
METRICS_HEADER = ("frame,time_ms,avg_density_pct,min_density_pct,max_density_pct,"
                  "total_iterations,contacts")


def _num(v: float) -> str:
    """numStr (runner.cpp:10-14): %.17g."""
    return "%.17g" % float(v)


def mode_name(mode: SolverMode) -> str:
    """modeName (runner.cpp:56)."""
    return "pbf" if mode == SolverMode.PBF else "apbf"


def lod_model_name(model: LodModel) -> str:
    """lodModelName (runner.cpp:58)."""
    return "dtc" if model == LodModel.DTC else "dtvs"


def median_of(values) -> float:
    """medianOf (metrics.cpp:22-31)."""
    v = sorted(float(x) for x in values)
    if not v:
        raise ValueError("median of empty sample")
    mid = len(v) // 2
    return v[mid] if len(v) % 2 == 1 else 0.5 * (v[mid - 1] + v[mid])


@dataclass
class RunOptions:
    """RunOptions (runner.hpp:14-24)."""
    mode: SolverMode = SolverMode.APBF
    lod_model: Optional[LodModel] = None       # overrides the scenario's model
    range: Optional[IterationRange] = None     # overrides the scenario's range
    frames: int = 0                            # 0: scenario default
    seed: int = 0
    deterministic: bool = False
    out_dir: Optional[str] = None              # None/empty: nothing written
    dump_images_every: int = 0
    dump_particles_every: int = 0


@dataclass
class RunReport:
    """RunReport (metrics.hpp:20-30)."""
    frames: List[FrameStats] = field(default_factory=list)
    echo: List[Tuple[str, str]] = field(default_factory=list)
    hash: int = 0
    zero_time: bool = False

    def median_frame_ms(self) -> float:
        return median_of(f.wall_ms for f in self.frames)

    def total_iterations(self) -> int:
        return int(sum(f.total_iterations for f in self.frames))

    def total_contacts(self) -> int:
        return int(sum(f.contacts for f in self.frames))


@dataclass
class MetricsRow:
    """MetricsRow (metrics.hpp:32-40)."""
    frame: int = 0
    time_ms: float = 0.0
    avg_density_pct: float = 0.0
    min_density_pct: float = 0.0
    max_density_pct: float = 0.0
    total_iterations: int = 0
    contacts: int = 0


@dataclass
class MetricsFile:
    """MetricsFile (metrics.hpp:42-45)."""
    hash: Optional[int] = None
    rows: List[MetricsRow] = field(default_factory=list)


@dataclass
class CompareResult:
    """CompareResult (metrics.hpp:52-56)."""
    max_delta: float = 0.0
    frames: int = 0
    passed: bool = False


def write_metrics_csv(path, report: RunReport) -> None:
    """writeMetricsCsv (metrics.cpp:51-72): echo lines, hash, header, rows."""
    try:
        f = open(path, "w")
    except OSError as e:
        raise RuntimeError(f"cannot open metrics file for writing: {path}") from e
    with f:
        for k, v in report.echo:
            f.write(f"# {k} = {v}\n")
        f.write("# scenario_hash = %016x\n" % report.hash)
        f.write(METRICS_HEADER + "\n")
        for s in report.frames:
            f.write("%d,%.3f,%.6f,%.6f,%.6f,%d,%d\n" % (
                s.frame, 0.0 if report.zero_time else s.wall_ms, s.avg_density_pct,
                s.min_density_pct, s.max_density_pct, s.total_iterations, s.contacts))


_ROW = re.compile(r"^\s*([+-]?\d+),([^,]+),([^,]+),([^,]+),([^,]+),\s*([+-]?\d+),\s*([+-]?\d+)")
_HASH = re.compile(r"^# scenario_hash = ([0-9a-fA-F]+)")


def read_metrics_csv(path) -> MetricsFile:
    """readMetricsCsv (metrics.cpp:74-110)."""
    try:
        f = open(path)
    except OSError as e:
        raise RuntimeError(f"cannot open metrics file: {path}") from e
    out, saw_header = MetricsFile(), False
    with f:
        for line_no, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line:
                continue
            if line[0] == "#":
                m = _HASH.match(line)
                if m:
                    out.hash = int(m.group(1), 16)
                continue
            if not saw_header:
                if line != METRICS_HEADER:
                    raise RuntimeError(f"{path}:{line_no}: unexpected metrics header")
                saw_header = True
                continue
            m = _ROW.match(line)
            try:
                if not m:
                    raise ValueError
                row = MetricsRow(int(m.group(1)), float(m.group(2)), float(m.group(3)),
                                 float(m.group(4)), float(m.group(5)), int(m.group(6)),
                                 int(m.group(7)))
            except ValueError:
                raise RuntimeError(f"{path}:{line_no}: malformed metrics row") from None
            out.rows.append(row)
    if not saw_header:
        raise RuntimeError(f"{path}: no metrics header found")
    return out


def compare_runs(ref: MetricsFile, test: MetricsFile, tolerance_pct: float) -> CompareResult:
    """compareRuns (metrics.cpp:112-131): max per-frame |avg density| delta."""
    if ref.hash is not None and test.hash is not None and ref.hash != test.hash:
        raise RuntimeError("scenario hash mismatch: runs are not comparable")
    if len(ref.rows) != len(test.rows):
        raise RuntimeError(f"frame count mismatch: {len(ref.rows)} vs {len(test.rows)}")
    res = CompareResult(frames=len(ref.rows))
    for a, b in zip(ref.rows, test.rows):
        res.max_delta = max(res.max_delta, abs(b.avg_density_pct - a.avg_density_pct))
    res.passed = res.max_delta < tolerance_pct
    return res


def build_echo(s: S.ScenarioSpec, opt: RunOptions, frames: int, particles: int) -> List[Tuple[str, str]]:
    """buildEcho (runner.cpp:20-45): the config header of metrics.csv, with the
    derived values evaluated in double like SolverConfig<double>."""
    c = s.solver
    radius = c.particle_radius if c.particle_radius > 0 else c.h / 4.0
    stab = c.stab_threshold if c.stab_threshold > 0 else c.range.n_max
    cap = c.velocity_cap if c.velocity_cap > 0 else c.h / (c.dt_frame / c.substeps)
    r = c.range
    return [("scenario", s.name), ("scale", _num(s.scale)), ("particles", str(particles)),
            ("frames", str(frames)), ("seed", str(opt.seed)), ("mode", mode_name(c.mode)),
            ("lod_model", lod_model_name(s.lod.model)), ("iterations", f"{r.n_min}..{r.n_max}"),
            ("deterministic", "1" if opt.deterministic else "0"), ("dt_frame", _num(c.dt_frame)),
            ("substeps", str(c.substeps)), ("rest_density", _num(c.rest_density)),
            ("smoothing_length", _num(c.h)), ("epsilon", _num(c.epsilon)),
            ("particle_radius", _num(radius)), ("stab_iterations", str(c.stab_iterations)),
            ("stab_threshold", str(stab)), ("velocity_cap", _num(cap)),
            ("inactive_lambda_zero", "1" if c.inactive_lambda_zero else "0"),
            ("jitter", _num(s.jitter))]


def _frame_path(d: str, stem: str, frame: int, ext: str) -> str:
    return os.path.join(d, "%s_%06d.%s" % (stem, frame, ext))


def run_scenario(spec: S.ScenarioSpec, opt: RunOptions, device: int = 0) -> RunReport:
    """runScenario (runner.cpp:60-98) on the B200: spawn, simulate, and (with
    out_dir) write metrics.csv plus the requested frame dumps.  Level images
    are rendered on the device (render_levels); particle snapshots download
    the state."""
    s = copy.deepcopy(spec)
    if opt.range is not None:
        s.solver.range = opt.range
        s.lod.range = opt.range
    if opt.lod_model is not None:
        s.lod.model = opt.lod_model
    s.solver.mode = opt.mode
    s.solver.deterministic = opt.deterministic
    frames = opt.frames if opt.frames > 0 else s.frames

    state = S.make_state(s, opt.seed)
    solver = Solver(s.solver, s.scene, device)
    report = RunReport(hash=S.scenario_hash(s, opt.seed), zero_time=opt.deterministic,
                       echo=build_echo(s, opt, frames, state.count()))
    persist = bool(opt.out_dir)
    if persist:
        os.makedirs(opt.out_dir, exist_ok=True)
    radius = s.solver.effective_particle_radius()  # float32, as the solver's own
    solver.upload(state)
    for f in range(frames):
        report.frames.append(solver.step_frame_resident(s.camera, s.lod, f))
        if persist and opt.dump_images_every > 0 and f % opt.dump_images_every == 0:
            img = solver.render_levels(s.camera, radius, s.solver.range)
            write_ppm(img, _frame_path(opt.out_dir, "frame", f, "ppm"))
        if persist and opt.dump_particles_every > 0 and f % opt.dump_particles_every == 0:
            solver.download(state)
            write_particle_snapshot(_frame_path(opt.out_dir, "particles", f, "csv"), state)
    if persist:
        write_metrics_csv(os.path.join(opt.out_dir, "metrics.csv"), report)
    return report


# ------------------------------------------------------------------ bench

@dataclass
class BenchMode:
    """BenchMode (bench.hpp:15-20): "pbf:N", "apbf", "apbf:dtc", "apbf:dtvs"."""
    token: str = ""
    mode: SolverMode = SolverMode.APBF
    pbf_iterations: int = 0
    lod_model: Optional[LodModel] = None


def parse_bench_mode(token: str) -> BenchMode:
    """parseBenchMode (bench.cpp:9-42), same messages."""
    m = BenchMode(token=token)
    head, _, tail = token.partition(":")
    if head == "pbf":
        m.mode = SolverMode.PBF
        if not tail:
            raise ValueError("pbf bench mode needs an iteration count, e.g. pbf:6")
        t = tail.lstrip()
        digits = re.match(r"[+-]?\d+", t)  # std::stoi: leading integer, rest ignored
        if not digits:
            raise ValueError(f"invalid pbf iteration count '{tail}'")
        v = int(digits.group(0))
        if v > 2**31 - 1 or v < -2**31:
            raise ValueError(f"invalid pbf iteration count '{tail}'")
        m.pbf_iterations = v
        if v < 1:
            raise ValueError("pbf iteration count must be at least 1")
        return m
    if head == "apbf":
        m.mode = SolverMode.APBF
        if tail == "dtc":
            m.lod_model = LodModel.DTC
        elif tail == "dtvs":
            m.lod_model = LodModel.DTVS
        elif tail:
            raise ValueError(f"apbf bench mode takes dtc or dtvs, got '{tail}'")
        return m
    raise ValueError(f"unknown bench mode '{token}'; expected pbf:N or apbf:dtc|dtvs")


def parse_bench_modes(comma_separated: str) -> List[BenchMode]:
    """parseBenchModes (bench.cpp:44-56)."""
    out = [parse_bench_mode(t) for t in comma_separated.split(",") if t]
    if not out:
        raise ValueError("no bench modes given")
    return out


@dataclass
class BenchResult:
    """BenchResult (bench.hpp:25-31)."""
    token: str = ""
    median_frame_ms: float = 0.0
    iterations: int = 0
    frames: int = 0
    particles: int = 0


def run_bench(spec: S.ScenarioSpec, modes: List[BenchMode], reps: int, frames: int, seed: int,
              device: int = 0) -> List[BenchResult]:
    """runBench (bench.cpp:58-91): reps interleaved across modes; per mode the
    median over reps of each run's median frame time (device time)."""
    if reps < 1:
        raise ValueError("bench repetitions must be at least 1")
    results = [BenchResult() for _ in modes]
    medians: List[List[float]] = [[] for _ in modes]
    for _ in range(reps):
        for k, m in enumerate(modes):
            opt = RunOptions(mode=m.mode, lod_model=m.lod_model, frames=frames, seed=seed)
            if m.mode == SolverMode.PBF:
                opt.range = IterationRange(m.pbf_iterations, m.pbf_iterations)
            rep = run_scenario(spec, opt, device)
            medians[k].append(rep.median_frame_ms())
            results[k].token = m.token
            results[k].iterations = rep.total_iterations()
            results[k].frames = len(rep.frames)
    for k in range(len(modes)):
        results[k].median_frame_ms = median_of(medians[k])
        results[k].particles = spec.particle_count()
    return results


def format_bench_report(results: List[BenchResult]) -> str:
    """formatBenchReport (bench.cpp:93-123): table plus, against the first pbf
    row, both improvement conventions for every apbf row."""
    out = "%-12s %14s %18s %10s %10s\n" % ("mode", "median_ms", "total_iterations", "frames",
                                           "particles")
    for r in results:
        out += "%-12s %14.3f %18d %10d %10d\n" % (r.token, r.median_frame_ms, r.iterations, r.frames,
                                                  r.particles)
    base = next((r for r in results if r.token.startswith("pbf")), None)
    if base is not None:
        for r in results:
            if r is base or not r.token.startswith("apbf"):
                continue
            tp, ta = base.median_frame_ms, r.median_frame_ms
            if not ta > 0.0 or not tp > 0.0:
                continue
            out += ("%s vs %s: speedup (t_pbf-t_apbf)/t_apbf = %.1f%%, "
                    "reduction (t_pbf-t_apbf)/t_pbf = %.1f%%, iteration ratio = %.3f\n" % (
                        r.token, base.token, 100.0 * (tp - ta) / ta, 100.0 * (tp - ta) / tp,
                        r.iterations / base.iterations))
    return out
