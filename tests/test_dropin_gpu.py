"""The reference's own `planc verify` flow with planc_b200 dropped in.

oracle/_ref/verify_b200 (oracle/verify_b200.cpp, built against the
unmodified reference objects and include/planc_b200.hpp) loads plan and
graph with the reference loaders, draws the reference's seeded inputs, runs
the reference's sequential oracle, executes the plan on the GPU through
planc_b200::run_plan and lets the reference's compare_outputs decide —
exit 0 / 3 / 4 exactly like tools/planc.cpp. fp32 golden plans, bit-exact.
"""
import os
import subprocess

import pytest

import golden_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "verify_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/verify_b200 not built")]

FP32_CASES = [n for n in golden_cases.names() if golden_cases.load(n)["meta"]["rel_tol"] == 0.0]


@pytest.mark.parametrize("name", FP32_CASES)
def test_planc_verify_with_b200_executor(name):
    g = golden_cases.load(name)
    d = os.path.join(golden_cases.GOLDEN, name)
    r = subprocess.run([BIN, "--plan", os.path.join(d, "plan.json"), "--graph", os.path.join(d, "graph.json"),
                        "--seed", str(g["meta"]["seed"]), "--magnitude", str(g["meta"].get("magnitude", 4)),
                        "--lanes-on-one-gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


def test_verify_reports_input_errors_like_the_cli(tmp_path):
    d = os.path.join(golden_cases.GOLDEN, "mlp_dp2")
    bad = tmp_path / "plan.json"
    bad.write_text("{not json")
    r = subprocess.run([BIN, "--plan", str(bad), "--graph", os.path.join(d, "graph.json")], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 4


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/acceptance_b200 not built")
def test_reference_acceptance_suite_with_b200_run_plan():
    """The reference's own acceptance suite (acceptance.cpp, unmodified) with
    every planc::run_plan call routed to the B200 (oracle/refexec_b200.cpp,
    linker --wrap): criterion 1 is the 220-plan randomized corpus
    (acceptance.cpp:36-71) — every plan bit-exact against the sequential
    reference through testutil::oracle_ok; criteria 7 and 9 run their plans
    on the GPU too. All nine criteria must pass."""
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "PASS criterion 1: 220/220" in out, out
    assert r.returncode == 0 and "FAIL" not in out, out
    for c in range(1, 10):
        assert f"PASS criterion {c}:" in out, out
