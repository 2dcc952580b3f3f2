"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``orc``: the C restatement in ``oracle/pqkv_oracle.c`` (``liborc.so``).
* ``ref``: the unmodified reference library compiled from /root/reference by
  ``oracle/Makefile`` into ``oracle/_ref/libpqkv_ref.so`` (present when it was
  built in the CPU container; the built .so travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package, and only as the checker.  Both bindings expose the same
numpy-level functions, so a test can run one case through either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libpqkv_ref.so")

EINVAL, ERANGE, ESTATE = 1, 2, 3
GAUSSIAN, POWERLAW = 0, 1
KINDS = {"gaussian": GAUSSIAN, "powerlaw": POWERLAW}


class OracleError(Exception):
    def __init__(self, code, what=""):
        super().__init__(f"oracle status {code}: {what}")
        self.code = code


def build(ref_dir: str | None = None, quiet: bool = True) -> None:
    """Compile liborc.so (and _ref/libpqkv_ref.so when the reference exists)."""
    cmd = ["make", "-C", HERE, "-j8"]
    if ref_dir:
        cmd.append(f"REF_DIR={ref_dir}")
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


_sz = C.c_size_t
_u64 = C.c_uint64
_vp = C.c_void_p
_dbl = C.c_double


class _Lib:
    """One CPU checker library (prefix 'orc_' or 'ref_')."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        sig = {
            "rng_stream": (_u64, [_u64, _vp, _sz, C.c_int]),
            "gen_workload": (C.c_int, [_sz, _sz, _sz, _sz, C.c_int, _sz, _dbl, _dbl, _u64, _vp, _vp, _vp]),
            "kmeans_fit": (C.c_int, [_vp, _sz, _sz, _sz, _sz, _u64, _vp, _vp, _vp, _vp]),
            "assign_nearest": (C.c_int, [_vp, _sz, _sz, _vp, _sz, _vp]),
            "pq_construct": (C.c_int, [_vp, _sz, _sz, _sz, _sz, _sz, _u64, _vp, _vp]),
            "pq_encode_one": (C.c_int, [_vp, _vp, _sz, _sz, _sz, _vp]),
            "pq_score_gqa": (C.c_int, [_vp, _sz, _sz, _vp, _sz, _sz, _vp, _sz, _vp]),
            "top_k_desc": (C.c_int, [_vp, _sz, _sz, _vp, _vp]),
            "exact_scores": (C.c_int, [_vp, _vp, _sz, _sz, _vp]),
            "softmax_rows": (C.c_int, [_vp, _vp, _vp, _sz, _vp, _sz, _vp]),
            "selective_attention": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _sz, _sz, _vp, _sz, _vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
        if prefix == "ref_":
            self.lib.ref_last_error.restype = C.c_char_p
            self.lib.ref_bench_decode.restype = _dbl
            self.lib.ref_bench_decode.argtypes = [_sz] * 9 + [_vp] * 6 + [C.c_int]
            self.lib.ref_bench_decode_steps.restype = _dbl
            self.lib.ref_bench_decode_steps.argtypes = [_sz] * 9 + [_vp] * 3 + [_sz] + [_vp] * 3 + [C.c_int, _vp]
            self.lib.ref_bench_build.restype = _dbl
            self.lib.ref_bench_build.argtypes = [_sz] * 6 + [_vp] * 4 + [C.c_int]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            what = self.lib.ref_last_error().decode() if self.prefix == "ref_" else ""
            raise OracleError(rc, what)

    # -- rng -----------------------------------------------------------------
    def rng_stream(self, seed: int, n: int, kind: int = 0) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._fn("rng_stream")(seed, _p(out), n, kind)
        return out if kind in (0, 3) else out.view(np.float64)

    # -- workload ------------------------------------------------------------
    def gen_workload(self, s, d_h, h_kv=1, g=1, kind=GAUSSIAN, n_components=8, spread=0.5,
                     zipf=1.0, seed=1):
        k = np.zeros((h_kv, s, d_h), np.float32)
        v = np.zeros((h_kv, s, d_h), np.float32)
        q = np.zeros((h_kv, g, d_h), np.float32)
        self._check(self._fn("gen_workload")(s, d_h, h_kv, g, kind, n_components, spread, zipf,
                                             seed, _p(k), _p(v), _p(q)))
        return k, v, q

    # -- k-means / PQ ----------------------------------------------------------
    def kmeans_fit(self, points, n_clusters, max_iter, seed):
        pts = np.ascontiguousarray(points, np.float32)
        n, dim = pts.shape
        cen = np.zeros((n_clusters, dim), np.float32)
        asg = np.zeros(n, np.uint64)
        trace = np.zeros(max(max_iter, 1), np.float64)
        iters = _sz(0)
        self._check(self._fn("kmeans_fit")(_p(pts), n, dim, n_clusters, max_iter, seed, _p(cen),
                                           _p(asg), _p(trace), C.byref(iters)))
        return cen, asg, trace[: iters.value].copy(), iters.value

    def assign_nearest(self, points, centroids):
        pts = np.ascontiguousarray(points, np.float32)
        cen = np.ascontiguousarray(centroids, np.float32)
        out = np.zeros(pts.shape[0], np.uint64)
        self._check(self._fn("assign_nearest")(_p(pts), pts.shape[0], pts.shape[1], _p(cen),
                                               cen.shape[0], _p(out)))
        return out

    def pq_construct(self, keys, m, b, max_iter, seed):
        keys = np.ascontiguousarray(keys, np.float32)
        s, d_h = keys.shape
        C_ = 1 << b
        cen = np.zeros((m, C_, d_h // m if m else 1), np.float32)
        codes = np.zeros((s, m), np.uint16)
        self._check(self._fn("pq_construct")(_p(keys), s, d_h, m, b, max_iter, seed, _p(cen),
                                             _p(codes)))
        return cen, codes

    def pq_encode_one(self, key, centroids):
        key = np.ascontiguousarray(key, np.float32)
        cen = np.ascontiguousarray(centroids, np.float32)
        m, C_, d_m = cen.shape
        out = np.zeros(m, np.uint16)
        self._check(self._fn("pq_encode_one")(_p(key), _p(cen), m, C_, d_m, _p(out)))
        return out

    def pq_score_gqa(self, queries, centroids, codes):
        q = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
        cen = np.ascontiguousarray(centroids, np.float32)
        codes = np.ascontiguousarray(codes, np.uint16)
        m, C_, d_m = cen.shape
        out = np.zeros(codes.shape[0], np.float32)
        self._check(self._fn("pq_score_gqa")(_p(q), q.shape[0], q.shape[1], _p(cen), m, C_,
                                             _p(codes), codes.shape[0], _p(out)))
        return out

    # -- selection / attention -------------------------------------------------
    def top_k_desc(self, scores, k, excluded=None):
        sc = np.ascontiguousarray(scores, np.float32)
        ex = None
        if excluded is not None and len(excluded):
            ex = np.zeros(sc.shape[0], np.uint8)
            ex[np.asarray(list(excluded), np.int64)] = 1
        out = np.zeros(max(k, 1), np.uint64)
        self._check(self._fn("top_k_desc")(_p(sc), sc.shape[0], k, _p(ex), _p(out)))
        return out[:k]

    def exact_scores(self, query, keys):
        q = np.ascontiguousarray(query, np.float32)
        k = np.ascontiguousarray(keys, np.float32)
        out = np.zeros(k.shape[0], np.float32)
        self._check(self._fn("exact_scores")(_p(q), _p(k), k.shape[0], k.shape[1], _p(out)))
        return out

    def softmax_attention(self, query, keys, values, rows=None):
        q = np.ascontiguousarray(query, np.float32)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        r = None if rows is None else np.ascontiguousarray(rows, np.uint64)
        t = k.shape[0] if r is None else r.shape[0]
        out = np.zeros(k.shape[1], np.float32)
        self._check(self._fn("softmax_rows")(_p(q), _p(k), _p(v), k.shape[1], _p(r), t, _p(out)))
        return out

    def selective_attention(self, query, keys, values, n_init, n_local, middle_ids):
        q = np.ascontiguousarray(query, np.float32)
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        ids = np.ascontiguousarray(middle_ids, np.uint64)
        out = np.zeros(k.shape[1], np.float32)
        self._check(self._fn("selective_attention")(_p(q), _p(k), _p(v), k.shape[1], k.shape[0],
                                                    n_init, n_local, _p(ids), ids.shape[0],
                                                    _p(out)))
        return out

    # -- multi-threaded reference baselines (ref only) -------------------------
    def bench_decode(self, keys, values, queries, centroids, codes, n_init, n_local, k,
                     n_threads=0):
        P, total, d_h = keys.shape
        g = queries.shape[1]
        m, C_ = centroids.shape[1], centroids.shape[2]
        out = np.zeros((P, g, d_h), np.float32)
        secs = self.lib.ref_bench_decode(P, total, d_h, g, n_init, n_local, m, C_, k,
                                         _p(np.ascontiguousarray(keys)),
                                         _p(np.ascontiguousarray(values)),
                                         _p(np.ascontiguousarray(queries)),
                                         _p(np.ascontiguousarray(centroids)),
                                         _p(np.ascontiguousarray(codes)), _p(out), n_threads)
        return secs, out

    def bench_decode_steps(self, keys, values, queries, centroids, codes, n_init, n_local, k,
                           n_threads=0):
        """queries [n_steps][P][g][d_h]; HeadStates built once; returns per-step seconds."""
        P, total, d_h = keys.shape
        n_steps, g = queries.shape[0], queries.shape[2]
        m, C_ = centroids.shape[1], centroids.shape[2]
        out = np.zeros((P, g, d_h), np.float32)
        secs = np.zeros(n_steps, np.float64)
        self.lib.ref_bench_decode_steps(P, total, d_h, g, n_init, n_local, m, C_, k,
                                        _p(np.ascontiguousarray(keys)),
                                        _p(np.ascontiguousarray(values)),
                                        _p(np.ascontiguousarray(queries)), n_steps,
                                        _p(np.ascontiguousarray(centroids)),
                                        _p(np.ascontiguousarray(codes)), _p(out), n_threads, _p(secs))
        return secs, out

    def bench_build(self, keys, m, b, max_iter, seeds, n_threads=0):
        P, s, d_h = keys.shape
        cen = np.zeros((P, m, 1 << b, d_h // m), np.float32)
        codes = np.zeros((P, s, m), np.uint16)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        secs = self.lib.ref_bench_build(P, s, d_h, m, b, max_iter, _p(np.ascontiguousarray(keys)),
                                        _p(seeds), _p(cen), _p(codes), n_threads)
        return secs, cen, codes


_cache: dict = {}


def orc() -> _Lib:
    """The C restatement (always available once built)."""
    if "orc" not in _cache:
        if not os.path.exists(ORC_SO):
            build()
        _cache["orc"] = _Lib(ORC_SO, "orc_")
    return _cache["orc"]


def has_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> _Lib:
    """The reference library itself (oracle/_ref), when it was built."""
    if "ref" not in _cache:
        _cache["ref"] = _Lib(REF_SO, "ref_")
    return _cache["ref"]
