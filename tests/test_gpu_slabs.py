"""z-slab decomposition on one GPU: G virtual ranks (host threads, own
streams, device-to-device exchanges) must reproduce the single-GPU frame bit
for bit ("a G-GPU run is bitwise equal to the 1-GPU run")."""
import numpy as np
import pytest

from paper_1608_04721_b200 import IterationRange, LodModel, NumericalError, ParticleSet, Solver, SolverMode
from paper_1608_04721_b200 import scenario as S
from paper_1608_04721_b200.slab import SlabGroup

pytestmark = pytest.mark.gpu

FIELDS = ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level")


def compare(spec, G, frames, seed=1, vary_mass_from=None):
    one = Solver(spec.solver, spec.scene)
    grp = SlabGroup(spec.solver, spec.scene, nranks=G, devices=[0] * G)
    a = S.make_state(spec, seed)
    if vary_mass_from is not None:  # non-uniform inverse mass on the last slice only
        k = vary_mass_from
        a.mass[k:] = (a.mass[k:] * np.float32(1.5)).astype(np.float32)
        a.inv_mass[k:] = (np.float32(1) / a.mass[k:]).astype(np.float32)
    b = a.copy()
    one.upload(a)
    grp.upload(b)
    for f in range(frames):
        sa = one.step_frame_resident(spec.camera, spec.lod, f)
        sb = grp.step_frame_resident(spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts) == (sb.total_iterations, sb.contacts), f
        assert sa.min_density_pct == sb.min_density_pct
        assert sa.max_density_pct == sb.max_density_pct
        assert sa.avg_density_pct == pytest.approx(sb.avg_density_pct, rel=1e-12)
    one.download(a)
    grp.download(b)
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    return grp


@pytest.mark.parametrize("G", [2, 3, 4])
def test_slabs_bitwise_dam_break_apbf(G):
    spec = S.build_scenario("dam_break", 15625 / 216000)
    spec.solver.range = IterationRange(5, 10)
    spec.lod.range = spec.solver.range
    spec.lod.model = LodModel.DTVS
    compare(spec, G, 6)


def test_slabs_bitwise_with_one_rank_holding_other_masses():
    """Only the last rank's slice has a different mass: no rank may take the
    uniform-inverse-mass lambda (the ranks agree on it at the first frame)."""
    spec = S.build_scenario("dam_break", 8000 / 216000)
    compare(spec, 2, 4, vary_mass_from=6000)


def test_slabs_bitwise_pbf_dtc():
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.solver.mode = SolverMode.PBF
    spec.lod.model = LodModel.DTC
    compare(spec, 2, 6)


def test_slabs_bitwise_multi_dam_break_cone():
    spec = S.build_scenario("multi_dam_break", 0.1)
    spec.lod.model = LodModel.DTC
    compare(spec, 3, 4)


def test_slabs_bitwise_tank_along_z():
    """C5 geometry (z = long axis = slab axis) at reduced size."""
    spec = S.build_scenario("tank_8m", 1.0 / 512)  # 25 x 12 x 50
    grp = compare(spec, 4, 4)
    counts = grp.particle_counts()
    assert (counts > 0).all()
    assert counts.max() <= 2 * counts.mean()  # equal-count slabs stay balanced


def test_slabs_report_numerical_error_like_single_gpu():
    x = np.zeros((40, 3), np.float32)
    x[:, 2] = 0.02 * np.arange(40)
    x[23, 1] = np.nan
    cfg = S.build_scenario("dam_break", 0.01).solver
    cfg.range = IterationRange(2, 2)
    s = ParticleSet(x, 0.01, 2)
    with pytest.raises(NumericalError) as e1:
        Solver(cfg).step_frame_with_levels(s.copy(), 0)
    with pytest.raises(NumericalError) as e2:
        SlabGroup(cfg, nranks=2, devices=[0, 0]).step_frame_with_levels(s.copy(), 0)
    assert (e1.value.pass_, e1.value.particle) == (e2.value.pass_, e2.value.particle) == ("predict", 23)


@pytest.mark.parametrize("mode,seg_graphs,frames", [("dtc", "1", 40), ("dtvs", "1", 6), ("pbf", "1", 6),
                                                    ("dtc", "0", 6)])
def test_nccl_transport_single_rank_matches_plain_solver(monkeypatch, mode, seg_graphs, frames):
    """The NCCL transport (dlopen'ed libnccl, ncclCommInitRank, all-reduce)
    with a 1-rank communicator runs the slab frame and must equal Solver.
    With NCCL the slab frame records its segments into CUDA graphs and
    updates them every substep (APBF_SLAB_GRAPHS=0: eager)."""
    from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id
    monkeypatch.setenv("APBF_SLAB_GRAPHS", seg_graphs)
    spec = S.build_scenario("dam_break", 8000 / 216000)
    if mode == "pbf":
        spec.solver.mode = SolverMode.PBF
    else:
        spec.lod.model = LodModel.DTC if mode == "dtc" else LodModel.DTVS
    one = Solver(spec.solver, spec.scene)
    nc = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
    a = S.make_state(spec, 1)
    b = a.copy()
    one.upload(a)
    nc.upload_slice(b, b.count())
    for f in range(frames):  # (40 frames: 80 substeps of in-place segment updates)
        sa = one.step_frame_resident(spec.camera, spec.lod, f)
        sb = nc.step_frame_resident(spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct, sa.max_density_pct) == \
               (sb.total_iterations, sb.contacts, sb.min_density_pct, sb.max_density_pct), f
        assert sa.avg_density_pct == pytest.approx(sb.avg_density_pct, rel=1e-12)
    one.download(a)
    nc.download(b)
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_nccl_recorded_segments_survive_a_failed_frame():
    """A frame that aborts inside a recorded segment (NaN found in predict)
    raises, keeps the start state, and the next frames still run through the
    recorded segments and match the plain solver."""
    from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.lod.model = LodModel.DTC
    nc = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
    one = Solver(spec.solver, spec.scene)
    good = S.make_state(spec, 1)
    nc.upload_slice(good.copy(), good.count())
    nc.step_frame_resident(spec.camera, spec.lod, 0)  # segments recorded once
    bad = good.copy()
    bad.v[100, 1] = np.nan
    nc.upload_slice(bad, bad.count())
    with pytest.raises(NumericalError):
        nc.step_frame_resident(spec.camera, spec.lod, 1)
    out = bad.copy()
    for k in FIELDS:
        getattr(out, k)[...] = 0
    nc.download(out)
    for k in FIELDS:
        assert np.array_equal(getattr(out, k), getattr(bad, k), equal_nan=True), k
    a, b = good.copy(), good.copy()
    one.upload(a)
    nc.upload_slice(b, b.count())
    for f in range(3):
        sa = one.step_frame_resident(spec.camera, spec.lod, f)
        sb = nc.step_frame_resident(spec.camera, spec.lod, f)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct) == \
               (sb.total_iterations, sb.contacts, sb.min_density_pct), f
    one.download(a)
    nc.download(b)
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_nccl_slab_host_round_trip_matches_plain_host_frames():
    """The N > 1 e2e path of bench.py on one rank: every frame uploads only the
    frame's inputs (upload_slice(frame_inputs_only=True)), steps, and
    downloads the reordered slice; the result equals the plain solver's host
    stepFrame, bit for bit."""
    from paper_1608_04721_b200.slab import SlabSolver, nccl_unique_id
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.lod.model = LodModel.DTC
    one = Solver(spec.solver, spec.scene)
    nc = SlabSolver(spec.solver, spec.scene, 0, 1, nccl_unique_id())
    a = S.make_state(spec, 1)
    b = a.copy()
    nc.upload_slice(b, b.count())  # full state once (levels etc.)
    for f in range(4):
        sa = one.step_frame(a, spec.camera, spec.lod, f)
        nc.upload_slice(b, b.count(), frame_inputs_only=True)
        sb = nc.step_frame_resident(spec.camera, spec.lod, f)
        nc.download(b)
        assert (sa.total_iterations, sa.contacts, sa.min_density_pct) == \
               (sb.total_iterations, sb.contacts, sb.min_density_pct), f
        for k in FIELDS:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (f, k)


def test_failed_slab_frame_keeps_start_state():
    """All-or-nothing across ranks too: after a failing slab frame (NaN in one
    rank's slice, found in predict) every rank holds its frame-start state,
    so the group downloads the input unchanged."""
    spec = S.build_scenario("dam_break", 8000 / 216000)
    spec.solver.range = IterationRange(3, 5)
    st = S.make_state(spec, 2)
    st.level[:] = 4
    st.v[6000, 2] = np.nan
    before = st.copy()
    grp = SlabGroup(spec.solver, spec.scene, nranks=2, devices=[0, 0])
    with pytest.raises(NumericalError):
        grp.step_frame_with_levels(st, 0)
    for k in FIELDS:
        assert np.array_equal(getattr(st, k), getattr(before, k), equal_nan=True), k
