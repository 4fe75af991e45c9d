"""Per-kernel device time of 2 frames (metrics off) for an ncu launch list:
the plain solver (its scenario's mode), the 1-rank NCCL slab frame, or the
1M ocean forced to PBF 10 / APBF DTC / APBF DTVS:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file out.csv python tools/slab_kernels.py {plain|slab1|pbf|dtc|dtvs} [scenario] [warm]

Only the two frames between cudaProfilerStart/Stop (after `warm` frames,
default 3) are captured."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402
from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id  # noqa: E402

kind = sys.argv[1]
spec = S.build_scenario(sys.argv[2] if len(sys.argv) > 2 else "ocean_1m")
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if kind in ("pbf", "dtc", "dtvs"):
    from paper_1608_04721_b200 import LodModel, SolverMode
    if kind == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if kind == "dtc" else LodModel.DTVS
st = S.make_state(spec, 1)
if kind == "slab1":
    sv = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
    sv.upload_slice(st, st.count())
else:
    sv = Solver(spec.solver, spec.scene)
    sv.upload(st)
sv.set_frame_metrics(False)
for f in range(warm):
    sv.step_frame_resident(spec.camera, spec.lod, f)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for f in range(2):
    st = sv.step_frame_resident(spec.camera, spec.lod, warm + f)
    print(kind, "frame", warm + f, "totalIterations", st.total_iterations, "wall_ms", round(st.wall_ms, 3))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
