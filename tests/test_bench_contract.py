"""bench.py's contract pieces that run without a GPU: the workload per N (C3
at N = 1, the fixed C5 tank as strong scaling at N > 1), the `config`
object both arms print (the driver compares them), and the rooflines'
arithmetic from per-launch event times."""
import argparse
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def args(**kw):
    a = argparse.Namespace(gpus=1, steps=20, warmup=5, impl="ours", scenario="ocean_1m", seed=1,
                           no_cpu_baseline=False, no_e2e=False, no_fast=False, cpu_frames=1, slab_check=False)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_workload_per_gpu_count(bench):
    assert bench.bench_scenario(args(), 1) == "ocean_1m"
    for n in (2, 4, 8):
        assert bench.bench_scenario(args(gpus=n), n) == "tank_8m"
    # --slab-check: the N > 1 path (tank, slab solver) with one rank
    assert bench.bench_scenario(args(slab_check=True), 1) == "tank_8m"
    assert bench.slab_mode(args(slab_check=True), 1) and not bench.slab_mode(args(), 1)


def test_both_arms_print_the_same_config(bench):
    from paper_1608_04721_b200 import scenario as S
    for world in (1, 2, 8):
        a = args(gpus=world)
        spec = S.build_scenario(bench.bench_scenario(a, world))
        c1 = bench.make_config(spec, world, a)
        c2 = bench.make_config(S.build_scenario(bench.bench_scenario(a, world)), world, a)
        assert c1 == c2
        assert c1["scenario_file"] == f"scenarios/{spec.name}.cfg"
        assert str(spec.particle_count()) in c1["workload"]
        assert ("strong scaling" in c1["parallelism"]) == (world > 1)
    assert "8000000 particles" in bench.make_config(S.build_scenario("tank_8m"), 8, args(gpus=8))["workload"]


def test_roofline_arithmetic(bench):
    kt = {"lambda_ms": 20.0, "deltap_ms": 30.0, "launches": 400, "particle_iterations": 400 * 750_000}
    roof, roof32 = bench.rooflines(kt, ms_kt=80.0, nbar=31.0, sm_mhz=1965.0, hbm_peak=6544.0,
                                   peak_kind="measured", steps=20, fma=False)
    assert roof["kernel"] == "k_deltap_apply"
    per_launch_s = 30.0 / 400 / 1e3
    assert roof["achieved"] == pytest.approx(32 * 750_000 / per_launch_s / 1e9)
    assert roof["frac"] == pytest.approx(roof["achieved"] / 6544.0)
    assert roof["share_of_step"] == pytest.approx(30.0 / 80.0)
    flops = 23 * 30.0 + 7
    assert roof32["achieved"] == pytest.approx(flops * 750_000 / per_launch_s / 1e12)
    assert roof32["peak"] == pytest.approx(148 * 128 * 1965e6 / 1e12)
    _, fast32 = bench.rooflines(kt, 80.0, 31.0, 1965.0, 6544.0, "measured", 20, fma=True)
    assert fast32["peak"] == pytest.approx(2 * roof32["peak"])
