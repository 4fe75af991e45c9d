"""A fixed launch sequence for ncu: `warm` frames of the 1M ocean (C3), then
one more frame, all with the parity build or all with the fast build
(--fast).  k_lambda / k_deltap_apply launch 10 times per substep (20 per
frame), the first of each substep at full activity, so
  ncu --set full -k regex:k_lambda --launch-skip 20*warm --launch-count 1
captures one full-activity launch of the last frame (cold cache under ncu).

usage: python tools/prof_kernels.py [--fast] [--warm 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fast", action="store_true")
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--scenario", default="ocean_1m")
ap.add_argument("--lod", default=None, choices=[None, "dtc", "dtvs"])
a = ap.parse_args()
spec = S.build_scenario(a.scenario)
if a.lod:
    from paper_1608_04721_b200 import LodModel
    spec.lod.model = LodModel.DTC if a.lod == "dtc" else LodModel.DTVS
sv = Solver(spec.solver, spec.scene)
sv.set_fast_math(a.fast)
sv.upload(S.make_state(spec, 1))
for f in range(a.warm + 1):
    st = sv.step_frame_resident(spec.camera, spec.lod, f)
print(f"{'fast' if a.fast else 'parity'} build: {a.warm + 1} frames, last totalIterations {st.total_iterations}")
