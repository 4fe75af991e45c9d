"""Host-side input generation (paper_1608_04721_b200/scenario.py) against the
reference's own spawner: golden fixtures from tests/golden/make_golden.py and,
when oracle/_ref is built, the live reference."""
import hashlib
import os

import numpy as np
import pytest

from paper_1608_04721_b200 import scenario as S

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scenarios.npz"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_splitmix64_reference_value():
    # test_harness.cpp:154-156: SplitMix64(0).next() == 0xe220a8397b1dcdaf
    assert int(S.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF == int(GOLD["splitmix0"][0])


@pytest.mark.parametrize("name,scale", [("dam_break", 15625 / 216000), ("double_dam_break", 0.05),
                                        ("multi_dam_break", 0.1), ("ocean_1m", 0.01)])
def test_spawn_matches_reference_bitwise(name, scale):
    spec = S.build_scenario(name, scale)
    pos = S.spawn_scenario(spec, 1)
    assert pos.shape[0] == int(GOLD[f"{name}_n"][0])
    assert np.array_equal(pos[:64], GOLD[f"{name}_head"])
    assert hashlib.sha256(pos.tobytes()).hexdigest() == str(GOLD[f"{name}_sha256"][0])
    assert S.scenario_hash(spec, 1) == int(GOLD[f"{name}_hash"][0])
    assert S.scenario_mass(spec) == float(GOLD[f"{name}_mass"][0])


def test_builtin_particle_counts():
    # test_harness.cpp:88-122
    assert S.build_scenario("dam_break", 1.0).particle_count() == 216000
    assert S.build_scenario("double_dam_break", 1.0).particle_count() == 672800
    assert S.build_scenario("multi_dam_break", 1.0).particle_count() == 225400
    assert S.build_scenario("dam_break", 1 / 27).particle_count() == 8000
    assert S.build_scenario("ocean_1m").particle_count() == 1_000_000
    assert S.build_scenario("tank_8m").particle_count() == 8_000_000


def test_mass_and_levels_of_make_state():
    # test_harness.cpp:124-137: mass = rho0 * s^3 = 0.015625
    spec = S.build_scenario("dam_break", 1 / 27)
    st = S.make_state(spec, 1)
    assert S.scenario_mass(spec) == 0.015625
    assert (st.mass == np.float32(0.015625)).all()
    assert (st.level == spec.solver.range.n_max).all()


def test_unknown_scenario_and_bad_file(tmp_path):
    with pytest.raises(ValueError):
        S.build_scenario("no_such_scenario")
    p = tmp_path / "bad.cfg"
    p.write_text("[fluid]\ncounts = 2 2 2\nwobble = 3\n")
    with pytest.raises(RuntimeError, match="bad.cfg:3"):
        S.load_scenario_file(str(p))


@pytest.mark.ref
def test_live_reference_spawner_when_available():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built here")
    for name in ("dam_break", "multi_dam_break"):
        spec = S.build_scenario(name, 0.05)
        pos, info = O.ref_build_scenario(name, 0.05, 3)
        assert np.array_equal(S.spawn_scenario(spec, 3), pos)
        assert S.scenario_hash(spec, 3) == info.hash
