"""Criterion 3 of the reference (acceptance_main.cpp:136-163) on the B200:
median device ms/frame (LOD + substeps, FrameStats.wallMs, metrics off) on
the 1M ocean for PBF 10 and APBF {5..10} DTC / DTVS over `frames` frames
(the reference measures 80, the settled regime), and the reduction
(t_pbf - t_apbf) / t_pbf.  Extra args are APBF_* environment settings to
A/B, e.g. `python tools/dyn_ab.py 80 APBF_GRAPHS=0`."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04721_b200 import LodModel, Solver, SolverMode  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for setting in sys.argv[2:] or ["default"]:
    if "=" in setting:
        k, v = setting.split("=", 1)
        os.environ[k] = v
    res = {}
    for mode in ("pbf", "dtc", "dtvs"):
        spec = S.build_scenario("ocean_1m")
        if mode == "pbf":
            spec.solver.mode = SolverMode.PBF
        else:
            spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
        sv = Solver(spec.solver, spec.scene)
        sv.set_frame_metrics(False)
        sv.upload(S.make_state(spec, 1))
        ms = [sv.step_frame_resident(spec.camera, spec.lod, f).wall_ms for f in range(frames)]
        res[mode] = statistics.median(ms[3:])
    red = {m: (res["pbf"] - res[m]) / res["pbf"] for m in ("dtc", "dtvs")}
    print(f"{setting} ({frames} frames): pbf10 {res['pbf']:.3f} dtc {res['dtc']:.3f} dtvs {res['dtvs']:.3f} ms; "
          f"reduction dtc {100 * red['dtc']:.1f}% dtvs {100 * red['dtvs']:.1f}%", flush=True)
