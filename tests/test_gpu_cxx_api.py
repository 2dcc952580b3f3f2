"""GPU: the C++ drop-in API (include/pqkv/pqkv.hpp over libpqkv.so) runs the
reference's own unit-test cases (test_pq/test_kmeans/test_attention/
test_model/test_kv_store) and matches the reference library call for call
(tests/cpp/test_api.cpp, linked against oracle/_ref/libpqkv_ref.so)."""
import os
import subprocess

import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not oracle.has_ref(), reason="oracle/_ref not built")
def test_cxx_api_suite(tmp_path):
    exe = str(tmp_path / "test_api")
    lib = os.path.join(ROOT, "paper_2407_12820_b200", "lib")
    ref = os.path.join(ROOT, "oracle", "_ref")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "test_api.cpp"),
           "-o", exe, f"-L{lib}", "-lpqkv", f"-L{ref}", "-lpqkv_ref", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{ref}"]
    b = subprocess.run(cmd, capture_output=True, text=True)
    assert b.returncode == 0, b.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
