"""Generate tests/golden/*.npz from the REFERENCE (oracle/_ref: the unmodified
/root/reference sources compiled against the Eigen shim, Solver<float>).

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tests/golden/make_golden.py
The fixtures are small and committed; tests compare the C oracle and the GPU
against them on machines where the reference does not exist.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1608_04721_b200 import IterationRange, LodModel, LodModelConfig, SolverMode  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def solver_case(tag, name, scale, mode, model, rng, frames):
    spec = S.build_scenario(name, scale)
    spec.solver.mode = mode
    spec.solver.range = IterationRange(*rng)
    spec.lod.model = model
    spec.lod.range = spec.solver.range
    st = S.make_state(spec, 1)
    init = {k: getattr(st, k).copy() for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")}
    rs = O.RefState.from_set(st)
    sv = O.RefSolver(spec.solver, spec.scene, prec=4)
    stats = []
    for f in range(frames):
        s = sv.step_frame(rs, spec.camera, spec.lod, f)
        stats.append([s.total_iterations, s.contacts, s.avg_density_pct, s.min_density_pct,
                      s.max_density_pct])
    out = {f"init_{k}": v for k, v in init.items()}
    out.update({"x": rs.x.astype(np.float32), "x_star": rs.x_star.astype(np.float32),
                "v": rs.v.astype(np.float32), "lambda_": rs.lambda_.astype(np.float32),
                "level": rs.level, "stats": np.array(stats, np.float64),
                "meta": np.array([name, str(scale), mode.name, model.name, str(rng[0]), str(rng[1]),
                                  str(frames)])})
    np.savez_compressed(os.path.join(OUT, f"solver_{tag}.npz"), **out)


def component_case():
    rng = np.random.default_rng(2024)
    cloud = rng.uniform(0.0, 0.4, (400, 3)).astype(np.float32)
    spec = S.build_scenario("dam_break", 1728 / 216000)
    dam = S.spawn_scenario(spec, 1).astype(np.float32)
    out = {"cloud": cloud, "dam": dam}
    for tag, p in (("cloud", cloud), ("dam", dam)):
        perm, origin, dims, cs = O.ref_grid_build(p.astype(np.float64), 0.05, 0.05, prec=4)
        off, idx = O.ref_neighbor_lists(p.astype(np.float64), 0.05, 0.05, prec=4)
        m = (1.0 + 0.01 * np.arange(p.shape[0])).astype(np.float32)
        rho = O.ref_all_densities(p.astype(np.float64), m.astype(np.float64), 0.05, prec=4)
        out.update({f"{tag}_perm": perm, f"{tag}_origin": origin.astype(np.float32),
                    f"{tag}_dims": dims, f"{tag}_cell_start": cs, f"{tag}_offsets": off,
                    f"{tag}_indices": idx, f"{tag}_mass": m, f"{tag}_rho": rho.astype(np.float32)})
    lod = LodModelConfig(LodModel.DTC, 0.0, 1.0, IterationRange(3, 6), True)
    out["dam_dtc"] = O.ref_lod_levels(dam.astype(np.float64), spec.camera, lod, prec=4)
    lod.model = LodModel.DTVS
    out["dam_dtvs"] = O.ref_lod_levels(dam.astype(np.float64), spec.camera, lod, 0.0125, prec=4)
    out["dam_depth"] = O.ref_splat(dam.astype(np.float64), 0.0125, spec.camera, prec=4).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "components.npz"), **out)


def scenario_case():
    out = {}
    for name, scale in (("dam_break", 15625 / 216000), ("double_dam_break", 0.05),
                        ("multi_dam_break", 0.1), (os.path.join(ROOT, "scenarios", "ocean_1m.cfg"), 0.01)):
        pos, info = O.ref_build_scenario(name, scale, 1)
        key = os.path.splitext(os.path.basename(name))[0]
        import hashlib
        out[f"{key}_sha256"] = np.array([hashlib.sha256(pos.tobytes()).hexdigest()])
        out[f"{key}_head"] = pos[:64]
        out[f"{key}_n"] = np.array([pos.shape[0]])
        out[f"{key}_hash"] = np.array([info.hash], np.uint64)
        out[f"{key}_mass"] = np.array([info.mass])
    out["splitmix0"] = np.array([O.rlib().ref_splitmix64_first(0)], np.uint64)
    np.savez_compressed(os.path.join(OUT, "scenarios.npz"), **out)


def harness_case():
    """The reference's own harness outputs (runner/metrics/bench): metrics.csv
    of runScenario (Solver<double>), the frame dumps that renderLevelImage<float>
    and writeParticleSnapshot<float> make of the reference Solver<float> state,
    formatBenchReport / parseBenchMode answers."""
    import json
    import tempfile
    out = {}
    with tempfile.TemporaryDirectory() as d:
        # C1-like dam break, 10 deterministic frames, DTVS (the scenario default)
        O.ref_run_scenario("dam_break", 8000 / 216000, 1, d, 10, seed=1)
        out["metrics_dam_apbf"] = np.array([open(os.path.join(d, "metrics.csv")).read()])
    with tempfile.TemporaryDirectory() as d:
        O.ref_run_scenario("dam_break", 8000 / 216000, 0, d, 4, seed=1, rng=IterationRange(3, 3))
        out["metrics_dam_pbf3"] = np.array([open(os.path.join(d, "metrics.csv")).read()])
    # dumps of the float reference after 2 frames of dam_break(0.001), seed 11
    spec = S.build_scenario("dam_break", 0.001)
    st = S.make_state(spec, 11)
    rs = O.RefState.from_set(st)
    sv = O.RefSolver(spec.solver, spec.scene, prec=4)
    for f in range(2):
        sv.step_frame(rs, spec.camera, spec.lod, f)
    r = float(np.float32(spec.solver.h) / np.float32(4))
    img = O.ref_render_level_image(rs.x, rs.level, r, spec.camera, spec.solver.range.n_min,
                                   spec.solver.range.n_max, prec=4)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.csv")
        O.ref_write_particle_snapshot(path, rs.x, rs.level, prec=4)
        out["snapshot_dam_f1"] = np.array([open(path).read()])
    out["image_dam_f1"] = img
    out["state_dam_f1_x"] = rs.x.astype(np.float32)
    out["state_dam_f1_level"] = rs.level.astype(np.int32)
    # a wider render: the dam_break(8000) initial lattice with mixed levels
    spec8 = S.build_scenario("dam_break", 8000 / 216000)
    x8 = S.spawn_scenario(spec8, 1).astype(np.float32)
    lv8 = (3 + (np.arange(x8.shape[0]) * 7919) % 4).astype(np.int32)
    out["render_x"] = x8
    out["render_level"] = lv8
    out["render_image"] = O.ref_render_level_image(x8, lv8, 0.0125, spec8.camera, 3, 6, prec=4)
    reports = [
        [("pbf:6", 10.0, 1000, 2, 216), ("apbf:dtc", 7.5, 800, 2, 216), ("apbf:dtvs", 8.25, 900, 2, 216)],
        [("apbf", 3.0, 10, 1, 8)],
        [("pbf:3", 2.0, 30, 1, 5), ("pbf:6", 4.0, 60, 1, 5), ("apbf", 0.0, 40, 1, 5)],
    ]
    tokens = ["pbf", "pbf:0", "pbf:x", "pbf:6x", "pbf: 7", "pbf:-2", "apbf:bogus", "zzz", "apbf",
              "apbf:dtc", "apbf:dtvs", "pbf:99999999999", "", "apbf:"]
    modes = {}
    for t in tokens:
        try:
            modes[t] = list(O.ref_parse_bench_mode(t))
        except ValueError as e:
            modes[t] = str(e)
    out["bench"] = np.array([json.dumps({"reports": [[list(r) for r in rep] for rep in reports],
                                         "texts": [O.ref_format_bench_report(rep) for rep in reports],
                                         "modes": modes})])
    np.savez_compressed(os.path.join(OUT, "harness.npz"), **out)


if __name__ == "__main__":
    solver_case("dam_pbf_dtc", "dam_break", 1728 / 216000, SolverMode.PBF, LodModel.DTC, (5, 5), 4)
    solver_case("dam_apbf_dtvs", "dam_break", 1728 / 216000, SolverMode.APBF, LodModel.DTVS, (5, 10), 4)
    solver_case("multi_apbf_dtc", "multi_dam_break", 0.03, SolverMode.APBF, LodModel.DTC, (4, 8), 3)
    component_case()
    scenario_case()
    harness_case()
    print("golden fixtures written to", OUT)
