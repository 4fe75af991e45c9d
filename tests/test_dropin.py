"""The C++ drop-in (include/apbf_gpu/solver.hpp) compiled against the
reference's own headers (oracle/_ref/dropin_demo, built by oracle/Makefile)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


@pytest.mark.ref
def test_dropin_compiles_against_reference_headers():
    if not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference sources not present")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    assert os.access(DEMO, os.X_OK)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/dropin_demo not built")
@pytest.mark.parametrize("scenario,scale", [("multi_dam_break", "0.05"), ("dam_break", "0.03")])
def test_dropin_matches_reference_solver_bitwise(scenario, scale):
    out = subprocess.run([DEMO, scenario, scale, "4"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "DROPIN OK" in out.stdout


RUNNER = os.path.join(ROOT, "oracle", "_ref", "runner_demo")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(RUNNER), reason="oracle/_ref/runner_demo not built")
def test_runner_dropin_against_reference_harness():
    """include/apbf_gpu/runner.hpp: the reference harness test expectations
    for the GPU runScenario/runBench, and the reference's compareRuns
    accepting the GPU metrics.csv against the reference's own double run."""
    out = subprocess.run([RUNNER, str(8000 / 216000), "10"], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "RUNNER OK" in out.stdout
