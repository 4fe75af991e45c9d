import sys; sys.path.insert(0,'.')
from paper_1608_04721_b200 import scenario as S, IterationRange
from paper_1608_04721_b200.slab import SlabGroup
spec = S.build_scenario("dam_break", 8000/216000)
g = SlabGroup(spec.solver, spec.scene, nranks=2, devices=[0,0])
a = S.make_state(spec, 1)
g.upload(a)
print(g.particle_counts())
try:
    print(g.step_frame_resident(spec.camera, spec.lod, 0))
except Exception as e: print("ERR", e)
