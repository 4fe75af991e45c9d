"""Device-time A/B of library variants: CUDA events around `frames` resident
frames of a scenario after 3 warm-up frames, metrics on and off.
APBF_LIB=<lib> python tools/ab_device.py [frames] [scenario]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 20
spec = S.build_scenario(sys.argv[2] if len(sys.argv) > 2 else "ocean_1m")
out = []
for metrics in (True, False):
    sv = Solver(spec.solver, spec.scene)
    sv.set_frame_metrics(metrics)
    sv.upload(S.make_state(spec, 1))
    ext = torch.cuda.ExternalStream(sv.stream_handle())
    for f in range(3):
        sv.step_frame_resident(spec.camera, spec.lod, f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ext)
    for f in range(frames):
        sv.step_frame_resident(spec.camera, spec.lod, 3 + f)
    e1.record(ext)
    e1.synchronize()
    out.append(f"metrics={int(metrics)} {e0.elapsed_time(e1) / frames:.4f}")
print(os.environ.get("APBF_LIB", "libapbf_gpu.so"), " ".join(out), "ms/frame", flush=True)
