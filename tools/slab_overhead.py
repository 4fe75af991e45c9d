"""Per-frame cost of the slab (multi-GPU) path on ONE GPU: a 1-rank NCCL
SlabSolver (every exchange, all-reduce and host step of the decomposition,
with trivial peers) against the plain Solver on the same workload."""
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
for kind in ("solver", "slab1"):
    st = S.make_state(spec, 1)
    if kind == "solver":
        sv = Solver(spec.solver, spec.scene)
        sv.upload(st)
    else:
        sv = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
        sv.upload_slice(st, st.count())
    ext = torch.cuda.ExternalStream(sv.stream_handle())
    for f in range(3):
        sv.step_frame_resident(spec.camera, spec.lod, f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0.record(ext)
    its = 0
    for f in range(frames):
        its += sv.step_frame_resident(spec.camera, spec.lod, 3 + f).total_iterations
    e1.record(ext)
    e1.synchronize()
    wall = (time.perf_counter() - t) * 1e3 / frames
    print(f"{kind}: device {e0.elapsed_time(e1) / frames:.3f} ms/frame, host wall {wall:.3f} ms/frame, "
          f"{its / frames / 1e6:.2f} M PI/frame", flush=True)
