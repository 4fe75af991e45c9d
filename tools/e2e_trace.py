"""End-to-end stepFrame(ParticleSet&) timeline on pinned host arrays: APBF_E2E_TRACE=1 python tools/e2e_trace.py [phase]"""
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_1608_04721_b200 import Solver
from paper_1608_04721_b200 import scenario as S
spec = S.build_scenario("ocean_1m")
sv = Solver(spec.solver, spec.scene)
host = S.make_state(spec, 1)
def pinned(shape, dtype):
    return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()
n = host.count()
st = S.ParticleSet.__new__(S.ParticleSet)
for k, dt, sh in [("x", torch.float32, (n, 3)), ("x_star", torch.float32, (n, 3)), ("v", torch.float32, (n, 3)),
                  ("mass", torch.float32, n), ("inv_mass", torch.float32, n), ("lambda_", torch.float32, n),
                  ("level", torch.int32, n)]:
    a = pinned(sh, dt); a[...] = getattr(host, k); setattr(st, k, a)
if len(sys.argv) > 1: sv.set_phase_timing(True)
for f in range(8):
    t = time.perf_counter()
    sv.step_frame(st, spec.camera, spec.lod, f)
    print(f"frame {f}: {1e3*(time.perf_counter()-t):.3f} ms", file=sys.stderr, flush=True)
