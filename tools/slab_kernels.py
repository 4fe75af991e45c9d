"""Per-kernel device time of 2 frames of the plain solver vs the 1-rank NCCL
slab frame (metrics off), for an ncu launch list:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file out.csv python tools/slab_kernels.py {plain|slab1}

Only the two frames between cudaProfilerStart/Stop are captured."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402
from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id  # noqa: E402

kind = sys.argv[1]
spec = S.build_scenario(sys.argv[2] if len(sys.argv) > 2 else "ocean_1m")
st = S.make_state(spec, 1)
if kind == "slab1":
    sv = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
    sv.upload_slice(st, st.count())
else:
    sv = Solver(spec.solver, spec.scene)
    sv.upload(st)
sv.set_frame_metrics(False)
for f in range(3):
    sv.step_frame_resident(spec.camera, spec.lod, f)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for f in range(2):
    sv.step_frame_resident(spec.camera, spec.lod, 3 + f)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
