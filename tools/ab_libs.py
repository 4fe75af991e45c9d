"""A/B of library variants on the 1M ocean (graph replay, metrics on):
APBF_LIB=<lib> python tools/ab_libs.py [frames] -> median frame ms, parity and fast builds."""
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04721_b200 import Solver  # noqa: E402
from paper_1608_04721_b200 import scenario as S  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 30
spec = S.build_scenario(sys.argv[2] if len(sys.argv) > 2 else "ocean_1m")
for fast in (0, 1):
    sv = Solver(spec.solver, spec.scene)
    sv.set_fast_math(bool(fast))
    sv.upload(S.make_state(spec, 1))
    ms = [sv.step_frame_resident(spec.camera, spec.lod, f).wall_ms for f in range(frames)]
    print(f"{os.environ.get('APBF_LIB', 'libapbf_gpu.so')} fast={fast}: median {statistics.median(ms[5:]):.3f} ms",
          flush=True)
