"""Median device ms/frame (FrameStats.wallMs, metrics off) of the small
BASELINE scenes: C1 dam break 15,625 (PBF 5, APBF {5..10} DTVS / DTC) and a
131k dam break (APBF {5..10} DTVS), where the solver passes are launch-bound."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04721_b200 import IterationRange, LodModel, Solver, SolverMode  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
out = []
for name, scale, mode in (("C1", 15625 / 216000, "pbf"), ("C1", 15625 / 216000, "dtvs"),
                          ("C1", 15625 / 216000, "dtc"), ("dam131k", 131072 / 216000, "dtvs"),
                          ("C2", 0.3716, "dtvs")):
    spec = S.build_scenario("double_dam_break" if name == "C2" else "dam_break", scale)
    spec.solver.range = spec.lod.range = IterationRange(5, 5) if mode == "pbf" else IterationRange(5, 10)
    if mode == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
    sv = Solver(spec.solver, spec.scene)
    sv.set_frame_metrics(False)
    st = S.make_state(spec, 1)
    sv.upload(st)
    ms = [sv.step_frame_resident(spec.camera, spec.lod, f).wall_ms for f in range(frames)]
    out.append(f"{name} {st.count()} {mode}: {statistics.median(ms[3:]):.3f} ms")
print("; ".join(out), flush=True)
