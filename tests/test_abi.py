"""CPU: the C-ABI library loads, exports every symbol include/pqkv_c.h
declares, and the host-only entry points keep the reference's rules.  No
compute calls (no GPU here)."""
import ctypes as C
import os
import re

import pytest

import paper_2407_12820_b200 as pq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pqkv_c.h")).read()
    return sorted(set(re.findall(r"PQKV_API\s+[\w\s\*]*?\b(pqkv_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = pq.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.pqkv_abi_version() == 2


def test_pq_config_rules():
    # PqConfig::create (pq.cpp:13-25) / test_pq.cpp:50-59
    assert pq.pq_config(2, 6, 128) == (64, 64)
    assert pq.pq_config(4, 8, 128) == (32, 256)
    for bad in [(3, 6, 128), (0, 6, 128), (2, 0, 128), (2, 17, 128)]:
        with pytest.raises(ValueError):
            pq.pq_config(*bad)
    # codes_memory_ratio (pq.cpp:179-182), acceptance criterion 2
    assert pq.codes_memory_ratio(2, 6, 128) == 12.0 / 2048.0
    assert pq.codes_memory_ratio(4, 8, 128) == 1.0 / 64.0


def test_decode_launch_accounting():
    L = pq.pqkv_layer(d_h=128, kv_head_stride=128 * 10, n_heads=1, total=10, n_init=1, n_local=1, m=2, b=6)
    # one head: the per-head cluster grid is too small to gather -> select + attention
    assert pq.lib().pqkv_decode_launches(C.byref(L), 1, 0) == 2
    L.n_heads = 400  # >= 2 CTAs per SM: key select fused into the gather
    assert pq.lib().pqkv_decode_launches(C.byref(L), 1, 0) == 1
    L.n_heads = 1
    assert pq.lib().pqkv_decode_launches(C.byref(L), 3, 1) == 5


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        pq.Context(0)


def test_cxx_api_symbols_exported():
    out = os.popen(f"nm -DC --defined-only {pq.LIB_PATH}").read()
    for fn in ["pqkv::pq_construct", "pqkv::pq_score_gqa", "pqkv::approx_topk", "pqkv::kmeans_fit",
               "pqkv::selective_attention", "pqkv::softmax_attention", "pqkv::KvStore::evict_local_append"]:
        assert fn in out, fn
