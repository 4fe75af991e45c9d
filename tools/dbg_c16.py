import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1608_04721_b200 import IterationRange, ParticleSet, Solver
from paper_1608_04721_b200 import scenario as S
h = 0.1
nx, ny = int(sys.argv[1]), 6
xs, ys = np.meshgrid(np.arange(nx) * (h / 2), np.arange(ny) * (h / 2), indexing="ij")
x = np.stack([xs.ravel(), ys.ravel(), np.full(xs.size, 0.5)], 1).astype(np.float32)
cfg = S.build_scenario("dam_break", 0.01).solver
cfg.h = h
cfg.range = IterationRange(2, 3)
cfg.gravity = (0.0, 0.0, 0.0)
base = ParticleSet(x, 0.01, 3)
a = base.copy()
sa = Solver(cfg).step_frame_with_levels(a, 0)
os.environ["APBF_C16"] = "1"
b = base.copy()
sv = Solver(cfg)
sb = sv.step_frame_with_levels(b, 0)
print(sa.total_iterations, sb.total_iterations, sv.last_neighbor_stats())
print(np.abs(a.x - b.x).max(), np.abs(a.x - base.x).max(), np.abs(b.x - base.x).max())
