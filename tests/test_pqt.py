"""CPU: .pqt tensor / index files (tensor.cpp:46-150, pq.cpp:184-222) written
and read by paper_2407_12820_b200.pqt are byte-identical to, and readable by,
the reference library's own save_index / load_index / save_tensor
(oracle/_ref); malformed files fail like the reference."""
import ctypes as C
import io
import os
import struct

import numpy as np
import pytest

import oracle
from paper_2407_12820_b200 import pqt

pytestmark = pytest.mark.skipif(not oracle.has_ref(), reason="oracle/_ref not built")


def _ref():
    lib = oracle.ref().lib
    sz, vp = C.c_size_t, C.c_void_p
    lib.ref_save_index.argtypes = [C.c_char_p, vp, sz, sz, sz, vp, sz]
    lib.ref_load_index.argtypes = [C.c_char_p, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), vp, vp,
                                   sz, sz]
    lib.ref_save_tensor.argtypes = [C.c_char_p, vp, vp, sz]
    return lib


def _index(seed, m=2, b=6, d_m=64, s=1000):
    rng = np.random.default_rng(seed)
    cen = rng.standard_normal((m, 1 << b, d_m)).astype(np.float32)
    codes = rng.integers(0, 1 << b, size=(s, m)).astype(np.uint16)
    return cen, codes


def test_index_files_match_the_reference(tmp_path):
    lib = _ref()
    cen, codes = _index(1)
    ours, theirs = str(tmp_path / "ours.pqt"), str(tmp_path / "ref.pqt")
    pqt.save_index(ours, cen, codes)
    assert lib.ref_save_index(theirs.encode(), cen.ctypes.data, 2, 64, 64, codes.ctypes.data, 1000) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    got_c, got_k = pqt.load_index(theirs)
    assert np.array_equal(got_c, cen) and np.array_equal(got_k, codes)
    m, c_, d_m, s = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    rc = np.zeros_like(cen)
    rk = np.zeros_like(codes)
    assert lib.ref_load_index(ours.encode(), C.byref(m), C.byref(c_), C.byref(d_m), C.byref(s), rc.ctypes.data,
                              rk.ctypes.data, rc.size, rk.size) == 0
    assert (m.value, c_.value, d_m.value, s.value) == (2, 64, 64, 1000)
    assert np.array_equal(rc, cen) and np.array_equal(rk, codes)


def test_tensor_files_match_the_reference(tmp_path):
    lib = _ref()
    t = np.random.default_rng(2).standard_normal((3, 5, 7)).astype(np.float32)
    ours, theirs = str(tmp_path / "t.pqt"), str(tmp_path / "tr.pqt")
    pqt.save_tensor(ours, t)
    dims = np.array(t.shape, np.uint64)
    assert lib.ref_save_tensor(theirs.encode(), t.ctypes.data, dims.ctypes.data, 3) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(pqt.load_tensor(theirs), t)


def test_malformed_files_fail():
    cen, codes = _index(3, s=10)
    buf = io.BytesIO()
    pqt.write_index(buf, cen, codes)
    raw = buf.getvalue()
    with pytest.raises(RuntimeError, match="bad magic"):
        pqt.read_index(io.BytesIO(b"XQKV" + raw[4:]))
    with pytest.raises(RuntimeError, match="version"):
        pqt.read_index(io.BytesIO(raw[:4] + struct.pack("<I", 2) + raw[8:]))
    with pytest.raises(RuntimeError, match="truncated"):
        pqt.read_index(io.BytesIO(raw[:-3]))
    # a u16 grid where the f32 centroid tensor is expected
    g = io.BytesIO()
    pqt._write(g, pqt.U16, codes)
    with pytest.raises(RuntimeError, match="dtype"):
        pqt.read_tensor(io.BytesIO(g.getvalue()))
    bad = codes.copy()
    bad[4, 1] = 64
    b2 = io.BytesIO()
    pqt.write_tensor(b2, cen)
    pqt._write(b2, pqt.U16, bad)
    with pytest.raises(RuntimeError, match="out of range"):
        pqt.read_index(io.BytesIO(b2.getvalue()))
    with pytest.raises(ValueError):
        pqt.write_tensor(io.BytesIO(), np.array([1.0, np.nan], np.float32))
