"""Parity on every BASELINE.json config, on the GPU
product path, bit for bit:

  C1  dam break 15,625, 100 frames, GPU vs the REFERENCE's own Solver<float>
      (oracle/_ref: the unmodified /root/reference sources) -- the GPU ->
      reference chain pinned inside the GPU run, not only via the oracle;
  C4  the PBF N vs APBF {ceil(N/2)..N} sweep for every N in 5..20 (PBF N,
      APBF DTC, APBF DTVS) on the ocean scene at reduced size, 10 frames vs
      the C oracle; and one full 1M frame at N = 20 (PBF, DTC, DTVS) vs the
      reference Solver<float>;
  C5  one full 8M tank frame vs the reference Solver<float>; the z-slab
      decomposition on the tank at 1/8 scale (1M) with G = 2/4/8 ranks,
      bitwise vs one rank.

The reference runs with OpenMP over all host cores (deterministic = false):
its results do not depend on the thread count.  Match:
solver.hpp:228-345, acceptance_main.cpp:88-120.
"""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import IterationRange, LodModel, Solver, SolverMode
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu
FIELDS = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (the compiled reference) not present")


def stats_key(s):
    return (s.total_iterations, s.contacts, s.min_density_pct, s.max_density_pct)


def assert_same_state(a, b, where):
    for k in FIELDS:
        x, y = getattr(a, k), getattr(b, k)
        if k == "level":
            assert np.array_equal(x, y), (where, k)
        else:
            assert np.array_equal(np.asarray(x, np.float32), np.asarray(y, np.float32)), (where, k)


def sweep_spec(n_max, mode):
    spec = S.build_scenario("ocean_1m", 1.0 / 128)  # 40 x 10 x 20 = 8,000 particles
    spec.solver.range = spec.lod.range = IterationRange(math.ceil(n_max / 2), n_max)
    if mode == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
    return spec


def run_oracle(spec, frames, seed=1):
    st = S.make_state(spec, seed)
    orc = O.OracleSolver(spec.solver, spec.scene)
    stats = [stats_key(orc.step_frame(st, spec.camera, spec.lod, f)) for f in range(frames)]
    return st, stats


@pytest.mark.parametrize("n_max", range(5, 21))
def test_c4_sweep_bitwise(n_max):
    """C4 at reduced size: PBF N and APBF {ceil(N/2)..N} with DTC and DTVS,
    10 frames each.  The three oracle runs go in threads (the C oracle drops
    the GIL) while the GPU runs the same frames."""
    modes = ("pbf", "dtc", "dtvs")
    with ThreadPoolExecutor(3) as pool:
        futs = {m: pool.submit(run_oracle, sweep_spec(n_max, m), 10) for m in modes}
        for m in modes:
            spec = sweep_spec(n_max, m)
            st = S.make_state(spec, 1)
            gpu = Solver(spec.solver, spec.scene)
            stats = [stats_key(gpu.step_frame(st, spec.camera, spec.lod, f)) for f in range(10)]
            ref_st, ref_stats = futs[m].result()
            assert stats == ref_stats, m
            assert_same_state(st, ref_st, m)
            if m == "pbf":
                assert stats[-1][0] == 2 * n_max * st.count()


def ref_frames(spec, state, frames, start=0, with_levels=False):
    """The reference's Solver<float> on all host cores."""
    cfg = spec.solver
    cfg_par = type(cfg)(**{**cfg.__dict__, "deterministic": False})
    ref = O.RefSolver(cfg_par, spec.scene, prec=4)
    rs = O.RefState.from_set(state)
    stats = [stats_key(ref.step_frame(rs, spec.camera, spec.lod, f)) for f in range(start, start + frames)]
    return rs, stats


@need_ref
@pytest.mark.parametrize("mode", ["pbf", "dtc", "dtvs"])
def test_c4_full_1m_frame_at_n20_vs_reference(mode):
    """One full 1M ocean frame at N_max = 20 (PBF 20, APBF {10..20} DTC/DTVS)
    against the reference's Solver<float>."""
    spec = S.build_scenario("ocean_1m")
    spec.solver.range = spec.lod.range = IterationRange(10, 20)
    if mode == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
    st = S.make_state(spec, 1)
    assert st.count() == 1_000_000
    with ThreadPoolExecutor(1) as pool:
        fut = pool.submit(ref_frames, spec, st.copy(), 1)
        gpu = Solver(spec.solver, spec.scene)
        s = stats_key(gpu.step_frame(st, spec.camera, spec.lod, 0))
        rs, rstats = fut.result()
    assert s == rstats[0]
    assert_same_state(st, rs, mode)


@need_ref
def test_c1_100_frames_vs_reference_solver_float():
    """C1 (dam break 15,625, APBF {5..10}, DTVS and DTC, PBF 5): 100 frames,
    GPU vs the reference's own Solver<float>, every frame's stats and the
    final state bit for bit."""
    for mode in ("dtvs", "dtc", "pbf"):
        spec = S.build_scenario("dam_break", 15625 / 216000)
        spec.solver.range = spec.lod.range = IterationRange(5, 10)
        if mode == "pbf":
            spec.solver.mode = SolverMode.PBF
            spec.solver.range = spec.lod.range = IterationRange(5, 5)
        else:
            spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
        st = S.make_state(spec, 1)
        assert st.count() == 15625
        with ThreadPoolExecutor(1) as pool:
            fut = pool.submit(ref_frames, spec, st.copy(), 100)
            gpu = Solver(spec.solver, spec.scene)
            stats = [stats_key(gpu.step_frame(st, spec.camera, spec.lod, f)) for f in range(100)]
            rs, rstats = fut.result()
        assert stats == rstats, mode
        assert_same_state(st, rs, mode)


@need_ref
def test_c5_full_8m_tank_frame_vs_reference():
    """C5 at full size on one GPU: the 8M tank (200 x 100 x 400), one APBF
    {5..10} DTC frame, against the reference's Solver<float>."""
    spec = S.build_scenario("tank_8m")
    st = S.make_state(spec, 1)
    assert st.count() == 8_000_000
    with ThreadPoolExecutor(1) as pool:
        fut = pool.submit(ref_frames, spec, st.copy(), 1)
        gpu = Solver(spec.solver, spec.scene)
        s = stats_key(gpu.step_frame(st, spec.camera, spec.lod, 0))
        rs, rstats = fut.result()
    assert s == rstats[0]
    assert_same_state(st, rs, "tank_8m")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_c5_slabs_on_tank_at_one_eighth_bitwise(G):
    """The z-slab decomposition of C5 at 1/8 scale (100 x 50 x 200 = 1M),
    G ranks as host threads on one device, bitwise vs one rank over 2 frames."""
    from paper_1608_04721_b200.slab import SlabGroup
    spec = S.build_scenario("tank_8m", 1.0 / 8)
    a = S.make_state(spec, 1)
    assert a.count() == 1_000_000
    b = a.copy()
    one = Solver(spec.solver, spec.scene)
    grp = SlabGroup(spec.solver, spec.scene, nranks=G, devices=[0] * G)
    one.upload(a)
    grp.upload(b)
    for f in range(2):
        sa = one.step_frame_resident(spec.camera, spec.lod, f)
        sb = grp.step_frame_resident(spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct, sa.max_density_pct) == \
               (sb.total_iterations, sb.contacts, sb.min_density_pct, sb.max_density_pct), f
    one.download(a)
    grp.download(b)
    assert_same_state(a, b, f"G={G}")
    counts = grp.particle_counts()
    assert (counts > 0).all() and counts.sum() == a.count()
