"""Where the 1-rank slab frame's extra time goes: plain solver (graph replay
and eager launches) vs the 1-rank NCCL slab frame, device time per frame and
host time per frame (the wall time of the step_frame calls)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402
from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ocean_1m"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = S.build_scenario(name)
for kind in ("graph", "eager", "slab1", "slab1_nometrics", "graph_nometrics"):
    os.environ["APBF_GRAPHS"] = "0" if kind == "eager" else "1"
    st = S.make_state(spec, 1)
    if kind.startswith("slab"):
        sv = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
        sv.upload_slice(st, st.count())
    else:
        sv = Solver(spec.solver, spec.scene)
        sv.upload(st)
    if kind.endswith("nometrics"):
        sv.set_frame_metrics(False)
    ext = torch.cuda.ExternalStream(sv.stream_handle())
    for f in range(3):
        sv.step_frame_resident(spec.camera, spec.lod, f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0.record(ext)
    for f in range(frames):
        sv.step_frame_resident(spec.camera, spec.lod, 3 + f)
    e1.record(ext)
    e1.synchronize()
    wall = (time.perf_counter() - t) * 1e3 / frames
    print(f"{kind}: device {e0.elapsed_time(e1) / frames:.3f} ms/frame, host wall {wall:.3f} ms/frame, "
          f"launches/frame {Solver.launch_count()}", flush=True)
    del sv
