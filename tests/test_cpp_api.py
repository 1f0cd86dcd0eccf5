"""Header-level drop-in check: tests/cpp/api_test.cpp compiled against the
reference headers + the reference build (CPU) and against include/ + the
B200 library.  Both must pass the SPEC examples, and the fixed-iteration
cp_run fingerprints (sums over the returned fields) must be identical."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "_build")


def _run(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=False)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    fp = [l for l in r.stdout.splitlines() if l.startswith("FINGERPRINT")]
    return fp[0].split()


def test_api_against_reference_build():
    _run("api_test_ref")


@pytest.mark.gpu
def test_api_against_b200_library():
    ours = _run("api_test_b200")
    ref_exe = os.path.join(BUILD, "api_test_ref")
    if os.path.exists(ref_exe):
        ref = _run("api_test_ref")
        assert ours[1:4] == ref[1:4], (ours, ref)  # field fingerprints: bit-identical
        assert abs(float(ours[5]) - float(ref[5])) <= 1e-12 * abs(float(ref[5]))
