"""GPU: the reference's own callers, compiled unchanged against this repo's
C++ headers (include/pqkv/*.hpp ahead of the reference's) and linked with
libpqkv.so (oracle/Makefile `dropin`, built where /root/reference exists):

* the acceptance gate (reference tests/acceptance.cpp): all ten criteria
  PASS, the hot-path ones (1 score decomposition, 3 saturated codebook,
  4 clustering determinism, 8 block cache, 9 selection quality, 10 e2e
  determinism) computing on the GPU;
* run_recall on criterion 9's grid and run_e2e on criterion 10's config
  (experiments.cpp:74-275): their CSVs equal the reference build's byte for
  byte."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROP = os.path.join(ROOT, "oracle", "_ref", "dropin")


def _need(name):
    path = os.path.join(DROP, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle dropin needs /root/reference)")
    return path


def test_acceptance_gate_through_libpqkv():
    exe = _need("acceptance_b200")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion ")]
    assert len(lines) == 10, r.stdout + r.stderr
    for ln in lines:
        assert ": PASS - " in ln, ln
    assert r.returncode == 0


@pytest.mark.parametrize("mode", ["recall9", "e2e10"])
def test_experiment_csvs_equal_reference(mode):
    ours = subprocess.run([_need("dropin_csv_b200"), mode], capture_output=True, text=True, timeout=900)
    ref = subprocess.run([_need("dropin_csv_ref"), mode], capture_output=True, text=True, timeout=900)
    assert ours.returncode == 0, ours.stderr
    assert ref.returncode == 0, ref.stderr
    assert ours.stdout.count("\n") > 5
    if ours.stdout != ref.stdout:
        diff = [(a, b) for a, b in zip(ours.stdout.splitlines(), ref.stdout.splitlines()) if a != b]
        pytest.fail(f"{mode}: {len(diff)} CSV lines differ, first: {diff[:3]}")
