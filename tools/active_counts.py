"""Active particles per solver iteration of the ocean_1m frame (levels after
LOD), to read the per-launch solver times of a launch list against."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

spec = S.build_scenario(sys.argv[1] if len(sys.argv) > 1 else "ocean_1m")
st = S.make_state(spec, 1)
sv = Solver(spec.solver, spec.scene)
for f in range(4):
    sv.step_frame(st, spec.camera, spec.lod, f)
lv = st.level
print(json.dumps({"n": int(lv.size), "active": [int((lv >= it).sum()) for it in range(1, spec.solver.range.n_max + 1)]}))
