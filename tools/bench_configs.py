"""Measure every BASELINE.json config on one B200 (bench.py times only C3).

  C1  dam break 15,625: PBF N=5 and APBF {5..10} (DTVS, DTC), 100 frames
  C2  double dam break ~254k ("breaking wave"), APBF {5..10} DTVS
  C3  (bench.py) ocean 1M, APBF {5..10} DTC
  C4  1M ocean sweep: PBF N vs APBF {ceil(N/2)..N} (DTC, DTVS) for N = 5..20,
      with the paper's improvement (t_pbf - t_apbf) / t_apbf
  C5  8M tank (200 x 100 x 400), APBF {5..10}, on ONE GPU (the 2/4/8-GPU slab
      runs need more GPUs than this round had)

Times are the harness's per-frame device time (FrameStats.wallMs: LOD +
substeps, the reference's wallMs convention; metrics pass excluded), median
over frames, via paper_1608_04721_b200.harness.run_bench (the GPU backend of
the reference's runBench).  Writes one JSON document to stdout.
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_04721_b200 import IterationRange, LodModel  # noqa: E402
from paper_1608_04721_b200 import harness as H  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402


def rows(spec, modes, frames, reps=1):
    res = H.run_bench(spec, H.parse_bench_modes(modes), reps, frames, 1)
    out = []
    for r in res:
        pis = r.iterations / r.frames / (r.median_frame_ms / 1e3)
        out.append({"mode": r.token, "median_frame_ms": r.median_frame_ms, "steps_per_s": 1e3 / r.median_frame_ms,
                    "particle_iterations_per_s": pis, "total_iterations": r.iterations, "frames": r.frames,
                    "particles": r.particles})
    return out, H.format_bench_report(res)


def main():
    quick = "--quick" in sys.argv
    doc = {"gpu": "1x B200", "timing": "median FrameStats.wallMs (device: LOD + substeps) per run"}
    t0 = time.time()

    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.range = spec.lod.range = IterationRange(5, 10)
    doc["C1"], rep = rows(spec, "pbf:5,apbf:dtvs,apbf:dtc", 20 if quick else 100)
    print(rep, file=sys.stderr)

    spec = S.build_scenario("double_dam_break", 0.3716)
    doc["C2"], rep = rows(spec, "apbf:dtvs,pbf:10", 10 if quick else 30)
    print(rep, file=sys.stderr)

    sweep = []
    for n in range(5, 21):
        spec = S.build_scenario("ocean_1m")
        lo = math.ceil(n / 2)
        spec.solver.range = spec.lod.range = IterationRange(lo, n)
        r, rep = rows(spec, f"pbf:{n},apbf:dtc,apbf:dtvs", 6 if quick else 12)
        print(rep, file=sys.stderr)
        t_p = r[0]["median_frame_ms"]
        entry = {"n_max": n, "apbf_range": [lo, n], "pbf": r[0], "apbf_dtc": r[1], "apbf_dtvs": r[2]}
        for k in ("apbf_dtc", "apbf_dtvs"):
            t_a = entry[k]["median_frame_ms"]
            entry[k]["improvement_paper"] = (t_p - t_a) / t_a
            entry[k]["iteration_ratio"] = entry[k]["total_iterations"] / r[0]["total_iterations"]
        sweep.append(entry)
        if quick and n >= 8:
            break
    doc["C4"] = sweep

    if not quick:
        spec = S.build_scenario("tank_8m")
        doc["C5_single_gpu"], rep = rows(spec, "apbf:dtc", 6)
        print(rep, file=sys.stderr)
    doc["seconds"] = time.time() - t0
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
