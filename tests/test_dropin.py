"""The compiled drop-in (INTEGRATION.md sections 1-2; oracle/Makefile target
`dropin`): the reference's own sources with src/fc_core.cpp replaced by
oracle/dropin/fc_core_fcsg.cpp (fcs::fc on the B200 through libfcsg.so) and
Engine::run's loop by oracle/dropin/run_fcsg.cpp, built against the
reference's headers in the build container and run here:

* the reference's own tests/test_fc_core.cpp (16 doctest cases: operator
  sizes and profiles, derivative / filter accuracy, UsageError /
  ConfigError) against the B200 operator;
* oracle/dropin/engine_check.cpp: wb::riemann4 built by the reference,
  Engine::init, then Engine::run on the host cores against run_fcsg on the
  B200, both classifier variants, <= 1e-10 relative L2 per field.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
WEIGHTS = os.path.join(ROOT, "paper_2506_19370_b200", "data", "fcnn_v1.bin")


def _bin(name):
    p = os.path.join(REF, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not built (make -C oracle dropin, needs /root/reference at build time)")
    return p


@pytest.mark.gpu
def test_reference_fc_core_tests_against_the_b200_operator():
    r = subprocess.run([_bin("test_fc_core_fcsg")], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 16, failed: 0" in r.stdout


@pytest.mark.gpu
def test_reference_engine_run_against_run_fcsg():
    r = subprocess.run([_bin("dropin_engine_check"), WEIGHTS, "5"], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(": ok") == 2
