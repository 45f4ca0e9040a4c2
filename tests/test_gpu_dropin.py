"""The reference's own test programs, compiled unchanged against the reference headers
and linked with the C++ drop-in (paper_1701_08361_b200/compat/rtnlinv_compat.cpp) in
place of the reference's nlinv.cpp and fft.cpp, run on the B200.

Every test case must pass except the documented exception below, which asks for bit
equality between two computations the device performs in different orders; the same
property is checked within the north-star tolerances elsewhere (named in the table).
The cross-A bit equality of test_decomp.cpp:309-326 and acceptance check 7 holds on
the device: A WorkerGroup lanes run as an A-member channel group. A documented exception that starts passing is fine; anything else failing
is a regression.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1701_08361_b200", "compat", "_build")

pytestmark = pytest.mark.gpu

# test case -> why it cannot hold bit for bit on the device, and where the property is
# checked within tolerance instead
EXCEPTIONS = {
    "test_nlinv": {
        "a consistent estimate is a fixed point of the update": (
            "the test manufactures data with the reference's toeplitz_apply (fft::forward, a "
            "host complex multiply by P, fft::inverse) and expects the device Newton step's fused "
            "row/column passes to reproduce it to the last bit (residual exactly 0); the fused "
            "passes round in a different order -> tests/test_gpu_ops.py "
            "test_fixed_point_needs_no_iterations (residual <= 1e-5 |z|, update <= 1e-5)"),
    },
}

PROGRAMS = ["test_fft", "test_nlinv", "test_decomp", "test_preproc", "test_pipeline"]


def _run(prog):
    path = os.path.join(BUILD, prog)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build() compiles the drop-in and the reference tests in this container")
    out = subprocess.run([path], capture_output=True, text=True, timeout=900)
    ok = re.findall(r"^\[ OK \] (.*)$", out.stdout, flags=re.M)
    failed = re.findall(r"^\[FAIL\] (.*)$", out.stderr, flags=re.M)
    return out, ok, failed


@pytest.mark.parametrize("prog", PROGRAMS)
def test_reference_test_program_passes_against_the_drop_in(prog):
    out, ok, failed = _run(prog)
    allowed = EXCEPTIONS.get(prog, {})
    unexpected = [f for f in failed if f not in allowed]
    assert ok, out.stdout[-2000:] + out.stderr[-2000:]
    assert not unexpected, (unexpected, out.stderr[-4000:])
    summary = out.stdout.strip().splitlines()[-1]
    print(f"{prog}: {summary}; documented exceptions hit: {[f for f in failed if f in allowed]}")


def test_reference_acceptance_checks_pass_against_the_drop_in():
    """the reference's acceptance_test (checks 1-10: phantom quality, chaining, transform
    accounting, A-bit-equality, ordering, pipeline, ...) linked with the drop-in"""
    path = os.path.join(BUILD, "acceptance_test")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing")
    out = subprocess.run([path], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "all 10 checks passed" in out.stdout
