"""The reference's OWN unit tests (P/tests/test_*.cpp, unmodified) compiled
against the B200 drop-in headers and library (oracle/Makefile `reftests`),
run on the GPU.

The reference's float build itself fails a known set of cases whose
tolerances (1e-12 … 1e-14) or finite-difference probes only make sense in
double precision (pyramid 2, attention 5, attention_grad 3,
oracle 2).  The B200 build computes in fp32, so exactly those cases are
expected to fail here too, for the same reason; everything else must pass.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RT = os.path.join(ROOT, "oracle", "_ref", "reftests")

# Cases whose tolerance is double-only (fail identically in the reference's
# own LLSA_SINGLE_PRECISION build).
FP32_TOLERANCE_CASES = {
    "pyramid": {"column sums are preserved at every level",
                "pool_backward is the adjoint of pooling"},
    "attention": {"a constant value matrix collapses the output to that constant",
                  "keeping every block reduces to dense attention",
                  "the streaming pass matches the dense two-pass reference",
                  "running-max rescaling does not change well-scaled outputs",
                  "the input checksum pins data, plan, and config"},
    "attention_grad": {"with every block kept the gradient equals dense attention's",
                       "the sparse backward agrees with the dense-mask reference",
                       "the key-major pass matches its mask-driven baseline"},
    "oracle": {"dense attention outputs are convex combinations of the values",
               "logit biasing has a closed form when all logits tie"},
}
# This set is exactly what the reference's own float build fails when the same
# suites are linked against it (oracle/Makefile `reftests32`, recorded in
# tests/golden/ref_f32_suite_failures.json).
CPU_SUITES = ("core", "tensorio")
GPU_SUITES = ("pyramid", "selection", "indexmap", "attention", "attention_grad", "oracle",
              "reorder2d")


def _run(suite):
    exe = os.path.join(RT, f"test_{suite}")
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    failed = set(re.findall(r"^\[FAIL\] (.*)$", r.stdout, flags=re.M))
    passed = set(re.findall(r"^\[ OK \] (.*)$", r.stdout, flags=re.M))
    return r, failed, passed


@pytest.mark.parametrize("suite", CPU_SUITES)
def test_reference_suite_host_only(suite):
    r, failed, passed = _run(suite)
    assert not failed, r.stdout
    assert passed


@pytest.mark.gpu
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_suite_on_gpu(suite):
    r, failed, passed = _run(suite)
    print(r.stdout[-3000:])
    unexpected = failed - FP32_TOLERANCE_CASES.get(suite, set())
    assert not unexpected, r.stdout[-6000:]
    assert passed


# ---------------------------------------------------------------------------
# The reference's acceptance gate and its oracle-equivalence harness
# (P/tests/acceptance.cpp A1-A9 and P/src/bench.cpp run_verify, both
# unmodified) built against the drop-in (oracle/Makefile `acceptance`).
# tests/golden/ref_f32_acceptance.txt is the same gate on the reference's own
# f32 library: it fails A1 and A2 (1e-10 limits) and aborts A3 (finite
# differences throw PrecisionError below double precision) — the allowlist.
# (A6 is a wall-clock criterion; the f32 reference itself missed its spread
# limit on the 8-vCPU build host, so it is not in the allowlist: the drop-in
# must pass it.)
FP32_ACCEPTANCE_ALLOWED = {"A1", "A2", "A3"}


def _golden(name):
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        return f.read()


def test_f32_reference_gate_allowlist_is_recorded():
    g = _golden("ref_f32_acceptance.txt")
    failed = set(re.findall(r"^\[FAIL\] (A\d)", g, flags=re.M))
    assert FP32_ACCEPTANCE_ALLOWED <= failed
    assert re.search(r"^\[FAIL\] A3 aborted: finite differences need the double", g, re.M)
    assert "0 failed" in _golden("ref_f32_run_verify.txt")


@pytest.mark.gpu
def test_run_verify_on_drop_in():
    exe = os.path.join(RT, "run_verify")
    if not os.path.exists(exe):
        pytest.skip("acceptance harness not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    names = re.findall(r"^\[PASS\] (\S+)", r.stdout, flags=re.M)
    assert r.returncode == 0, r.stdout
    assert set(names) >= {"forward-oracle-scalekv", "forward-oracle-logitbias",
                          "forward-dense-reduction", "transpose-mask-equivalence",
                          "transpose-roundtrip", "backward-mask-scalekv",
                          "backward-mask-logitbias", "negative-control"}


@pytest.mark.gpu
def test_acceptance_gate_on_drop_in():
    exe = os.path.join(RT, "acceptance")
    if not os.path.exists(exe):
        pytest.skip("acceptance harness not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    passed = set(re.findall(r"^\[PASS\] (A\d)", r.stdout, flags=re.M))
    failed = set(re.findall(r"^\[FAIL\] (A\d)", r.stdout, flags=re.M))
    assert failed <= FP32_ACCEPTANCE_ALLOWED, r.stdout
    assert passed >= {"A4", "A5", "A6", "A7", "A8", "A9"}, r.stdout
