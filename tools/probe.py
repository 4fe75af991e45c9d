"""Per-frame timing probe of the resident path (phases, kernels)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04721_b200 import Solver
from paper_1608_04721_b200 import scenario as S
name = sys.argv[1] if len(sys.argv) > 1 else "ocean_1m"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 12
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
spec = S.build_scenario(name, scale)
sv = Solver(spec.solver, spec.scene)
st = S.make_state(spec, 1)
sv.upload(st)
sv.set_phase_timing(True)
for f in range(frames):
    if f == frames // 2:
        sv.set_kernel_timing(True)
    t = time.perf_counter()
    s = sv.step_frame_resident(spec.camera, spec.lod, f)
    dt = (time.perf_counter() - t) * 1e3
    ent, cap = sv.last_neighbor_stats()
    print(f"frame {f}: host {dt:.2f} ms wall(lod+substeps) {s.wall_ms:.2f} ms PI {s.total_iterations} "
          f"phases {['%.2f' % x for x in sv.last_phase_ms()]} nbar {ent/st.count():.2f} cap {cap/st.count():.2f}", flush=True)
print(json.dumps(sv.kernel_times()))
