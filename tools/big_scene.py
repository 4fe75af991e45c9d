"""A big single-GPU scene (ocean_weak(n): n x 1M particles): frame time,
PI/s and peak device memory."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1608_04721_b200 import Solver
from paper_1608_04721_b200 import scenario as S
n_slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 32
spec = S.ocean_weak(n_slabs)  # n_slabs x the 1M ocean along z, one GPU
st = S.make_state(spec, 1)
print("particles", st.count(), flush=True)
sv = Solver(spec.solver, spec.scene)
sv.upload(st)
for f in range(3):
    sv.step_frame_resident(spec.camera, spec.lod, f)
ext = torch.cuda.ExternalStream(sv.stream_handle())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ext); its = 0
for f in range(3):
    its += sv.step_frame_resident(spec.camera, spec.lod, 3 + f).total_iterations
e1.record(ext); e1.synchronize()
ms = e0.elapsed_time(e1) / 3
sv.download(st)
print(f"{ms:.2f} ms/frame, {its/3/ms*1e3/1e9:.2f} G PI/s, finite={np.isfinite(st.x).all()}, mem GB={torch.cuda.max_memory_allocated()/1e9:.1f}")
