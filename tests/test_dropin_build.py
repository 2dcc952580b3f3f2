"""CPU: the drop-in recipe (oracle/Makefile `dropin`) compiles the
reference's own callers -- tests/acceptance.cpp and the kept sources
experiments/workload/simulate/cost_model/timeline -- UNCHANGED against
include/pqkv/*.hpp and links them with libpqkv.so (every hot-path symbol
they use resolves in the product library).  Skipped where /root/reference
is absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources absent")
def test_reference_callers_compile_and_link_against_libpqkv():
    lib = os.path.join(ROOT, "paper_2407_12820_b200", "lib", "libpqkv.so")
    if not os.path.exists(lib):
        pytest.skip("libpqkv.so not built")
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j4", "dropin"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin", "acceptance_b200")
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libpqkv.so" in ldd
    # the hot path is not linked from the reference: no pq/kmeans/attention
    # definitions in the executable itself
    nm = subprocess.run(["nm", "-C", "--defined-only", exe], capture_output=True, text=True).stdout
    for sym in ("pqkv::pq_construct", "pqkv::kmeans_fit", "pqkv::selective_attention", "pqkv::KvStore::fetch_topk",
                "pqkv::approx_topk"):
        assert sym not in nm, f"{sym} defined in the executable, not taken from libpqkv.so"
