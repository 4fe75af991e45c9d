"""Localize the first GPU/oracle divergence of one frame via iteration observers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import OracleSolver
from paper_1608_04721_b200 import Solver
from paper_1608_04721_b200 import scenario as S

name = sys.argv[1] if len(sys.argv) > 1 else "double_dam_break"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
spec = S.build_scenario(name, scale)
snaps = {"g": {}, "o": {}}
def obs(tag):
    def f(s, it, st):
        snaps[tag][(s, it)] = {k: getattr(st, k).copy() for k in ("x", "x_star", "v", "lambda_", "level")}
    return f
g = Solver(spec.solver, spec.scene); g.iteration_observer = obs("g")
o = OracleSolver(spec.solver, spec.scene); o.iteration_observer = obs("o")
a = S.make_state(spec, 1); b = a.copy()
sa = g.step_frame(a, spec.camera, spec.lod, 0); sb = o.step_frame(b, spec.camera, spec.lod, 0)
print("iters", sa.total_iterations, sb.total_iterations, "contacts", sa.contacts, sb.contacts)
print("keys", sorted(snaps["g"]) == sorted(snaps["o"]), len(snaps["g"]), len(snaps["o"]))
for key in sorted(snaps["o"]):
    if key not in snaps["g"]:
        print("missing", key); break
    bad = [k for k in snaps["o"][key] if not np.array_equal(snaps["g"][key][k], snaps["o"][key][k])]
    if bad:
        print("first divergence at (substep, iter)", key, "fields", bad)
        for k in bad:
            d = np.argwhere(snaps["g"][key][k] != snaps["o"][key][k])
            print(" ", k, len(d), d[:5].tolist())
            i = d[0][0]
            print("   gpu", snaps["g"][key][k][i], "orc", snaps["o"][key][k][i], "level", snaps["o"][key]["level"][i])
        break
else:
    print("all iteration snapshots equal")
for k in ("x", "v", "level", "lambda_"):
    print("final", k, np.array_equal(getattr(a, k), getattr(b, k)))
