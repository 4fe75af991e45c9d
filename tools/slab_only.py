"""Four frames of the 1-rank NCCL slab path on ocean_1m (for an ncu launch list:
`ncu --metrics gpu__time_duration.sum ... python tools/slab_only.py`)."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1608_04721_b200 import scenario as S
from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id
spec = S.build_scenario("ocean_1m")
st = S.make_state(spec, 1)
sv = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
sv.upload_slice(st, st.count())
for f in range(4):
    sv.step_frame_resident(spec.camera, spec.lod, f)
