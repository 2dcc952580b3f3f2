"""B200-native PQCache hot paths (arxiv 2407.12820): Python host binding.

Thin ctypes layer over the C ABI in ``include/pqkv_c.h`` (the product is the
CUDA library ``lib/libpqkv.so``; PyTorch is only used here for device memory
and streams).  Every function takes CUDA tensors, launches on the current
torch stream and raises the reference's exception type on error
(``ValueError`` for std::invalid_argument, ``IndexError`` for
std::out_of_range, ``RuntimeError`` otherwise).

There is no CPU fallback: importing works without a GPU, but every compute
call needs the CUDA library and a device and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libpqkv.so")

PQKV_OK, PQKV_EINVAL, PQKV_ERANGE, PQKV_ESTATE, PQKV_ERUNTIME, PQKV_ECUDA = range(6)
PREC_F32, PREC_F64 = 0, 1
ASSIGN_FILTERED, ASSIGN_EXACT = 0, 1
TUPLE_CHUNK = 4096  # PQKV_TUPLE_CHUNK

_sz, _vp, _i, _u64 = C.c_size_t, C.c_void_p, C.c_int, C.c_uint64
PROF_SLOTS = 24  # PQKV_PROF_SLOTS (pqkv_c.h)


class pqkv_layer(C.Structure):
    """Mirror of the C struct pqkv_layer (pqkv_c.h)."""

    _fields_ = [
        ("keys", _vp), ("values", _vp), ("kv_head_stride", _sz), ("n_heads", _sz),
        ("total", _sz), ("n_init", _sz), ("n_local", _sz), ("d_h", _sz), ("m", _sz),
        ("b", _sz), ("centroids", _vp), ("codes", _vp), ("codes_head_stride", _sz),
        ("tuple_hist", _vp), ("tuple_chunk_hist", _vp), ("tuple_chunks", _sz),
    ]


class pqkv_decode_plan_t(C.Structure):
    """Mirror of pqkv_decode_plan_t (pqkv_c.h)."""

    _fields_ = [
        ("mode", _i), ("launches", _i), ("chunk_tokens", _i), ("ctas_per_head", _i), ("cluster", _i),
        ("staged", _i), ("window", _i), ("ring_depth", _i), ("smem_bytes", _sz),
    ]


PLAN_MODES = {1: "pairs_fused", 2: "keys_fused", 3: "keys_split", 4: "pairs_split", 5: "bitmap", 6: "generic"}

_SIGS = {
    "pqkv_abi_version": (_i, []),
    "pqkv_last_error": (C.c_char_p, []),
    "pqkv_ctx_create": (_i, [_i, C.POINTER(_vp)]),
    "pqkv_ctx_destroy": (_i, [_vp]),
    "pqkv_ctx_set_assign_mode": (_i, [_vp, _i]),
    "pqkv_ctx_last_build_stats": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u64)]),
    "pqkv_ctx_last_build_profile": (_i, [_vp, C.POINTER(_u64)]),
    "pqkv_ctx_set_profiling": (_i, [_vp, _i]),
    "pqkv_ctx_set_selection_dump": (_i, [_vp, _vp]),
    "pqkv_ctx_last_decode_profile": (_i, [_vp, C.POINTER(C.c_double)]),
    "pqkv_ctx_decode_profile_raw": (_i, [_vp, _vp, _sz, C.POINTER(_sz)]),
    "pqkv_device_alloc": (_i, [_vp, _sz, C.POINTER(_vp)]),
    "pqkv_device_free": (_i, [_vp, _vp]),
    "pqkv_copy": (_i, [_vp, _vp, _vp, _sz, _i]),
    "pqkv_stream_sync": (_i, [_vp, _vp]),
    "pqkv_pq_config": (_i, [_sz, _sz, _sz, C.POINTER(_sz), C.POINTER(_sz)]),
    "pqkv_codes_memory_ratio": (_i, [_sz, _sz, _sz, C.POINTER(C.c_double)]),
    "pqkv_kmeans_fit": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pqkv_pq_build": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _sz, _vp]),
    "pqkv_pq_encode": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _sz, _sz, _vp]),
    "pqkv_assign_nearest": (_i, [_vp, _vp, _sz, _sz, _vp, _sz, _vp, _vp]),
    "pqkv_pq_score": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _sz, _sz, _vp, _sz, _vp]),
    "pqkv_topk": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp, _vp]),
    "pqkv_pq_tuple_tables": (_i, [_vp, _sz, _sz, _vp, _sz, _sz, _sz, _vp, _vp, _sz, _vp]),
    "pqkv_pq_search": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _sz, _sz, _sz, _vp, _vp, _vp, _vp, _sz,
                            _vp]),
    "pqkv_exact_scores": (_i, [_vp, _vp, _sz, _sz, _sz, _vp, _sz, _vp, _sz, _vp, _vp]),
    "pqkv_attend_rows": (_i, [_vp, _vp, _sz, _sz, _sz, _vp, _vp, _sz, _vp, _sz, _i, _vp, _vp]),
    "pqkv_decode": (_i, [_vp, C.POINTER(pqkv_layer), _vp, _sz, _sz, _vp, _vp, _vp]),
    "pqkv_decode_step": (_i, [_vp, C.POINTER(pqkv_layer), _sz, _vp, _vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "pqkv_gen_workload": (_i, [_vp, _i, _sz, _sz, _sz, _sz, _sz, C.c_double, C.c_double, _u64, _vp, _vp, _vp,
                              _vp]),
    "pqkv_block_rank": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "pqkv_decode_attend": (_i, [_vp, C.POINTER(pqkv_layer), _vp, _sz, _vp, _vp, _vp]),
    "pqkv_decode_host": (_i, [_vp, C.POINTER(pqkv_layer), _vp, _sz, _sz, _vp, _vp]),
    "pqkv_decode_launches": (_i, [C.POINTER(pqkv_layer), _sz, _i]),
    "pqkv_decode_plan": (_i, [_vp, C.POINTER(pqkv_layer), _sz, _sz, _i, C.POINTER(pqkv_decode_plan_t)]),
    "pqkv_exact_topk": (_i, [_vp, _vp, _sz, _sz, _sz, _vp, _sz, _sz, _sz, _vp, _vp]),
    "pqkv_attend_dense": (_i, [_vp, _vp, _sz, _sz, _sz, _vp, _vp, _sz, _sz, _i, _vp, _vp]),
    "pqkv_relative_error": (_i, [_vp, _vp, _vp, _sz, _sz, _vp, _vp]),
    "pqkv_overlap_fraction": (_i, [_vp, _vp, _sz, _vp, _sz, _sz, _sz, _vp, _vp]),
    "pqkv_recall_seeds": (_i, [_u64, _sz, C.POINTER(_sz), _sz, _sz, _vp, _vp]),
    "pqkv_comm_unique_id": (_i, [C.c_char_p]),
    "pqkv_comm_init": (_i, [_vp, C.c_char_p, _i, _i, C.POINTER(_vp)]),
    "pqkv_comm_destroy": (_i, [_vp]),
    "pqkv_decode_sharded": (_i, [_vp, _vp, C.POINTER(pqkv_layer), _sz, _sz, C.POINTER(_vp), _sz, _sz, _vp, _vp]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded product library; raises if it was not built."""
    global _lib
    if _lib is None:
        path = os.environ.get("PQKV_LIB", LIB_PATH)  # experiment builds (tools/) only
        if not os.path.exists(path):
            raise RuntimeError(f"pqkv CUDA library missing: {path} (run __graft_entry__.build())")
        L = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class PqkvError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == PQKV_OK:
        return
    msg = lib().pqkv_last_error().decode()
    if rc == PQKV_EINVAL:
        raise ValueError(msg)
    if rc == PQKV_ERANGE:
        raise IndexError(msg)
    raise PqkvError(f"pqkv status {rc}: {msg}")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("pqkv: expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("pqkv: expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _stream():
    """The caller's current CUDA stream (torch's raw accessor: ~0.2 us instead of
    ~3.5 us for torch.cuda.current_stream() on the per-decode path)."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return C.c_void_p(raw(torch.cuda.current_device()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Context:
    """Owns a pqkv_ctx (scratch arena) bound to one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = device
        h = _vp()
        _check(lib().pqkv_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().pqkv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_assign_mode(self, mode: int) -> None:
        _check(lib().pqkv_ctx_set_assign_mode(self.h, mode))

    def last_build_stats(self):
        a, b = _u64(0), _u64(0)
        _check(lib().pqkv_ctx_last_build_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_profiling(self, on: bool) -> None:
        _check(lib().pqkv_ctx_set_profiling(self.h, int(on)))

    def last_decode_profile(self):
        """Mean SM cycles per attention CTA of the last decode (profiling mode)."""
        arr = (C.c_double * 4)()
        _check(lib().pqkv_ctx_last_decode_profile(self.h, arr))
        return {"prologue": arr[0], "pair_select": arr[1], "gather": arr[2], "ctas": int(arr[3])}

    def decode_profile_raw(self):
        """Per-CTA timestamps of the last attention launch, numpy u64 [n_ctas][PROF_SLOTS]
        (see pqkv_ctx_decode_profile_raw)."""
        import numpy as np

        n = _sz(0)
        _check(lib().pqkv_ctx_decode_profile_raw(self.h, None, 0, C.byref(n)))
        arr = np.zeros((n.value, PROF_SLOTS), np.uint64)
        if n.value:
            _check(lib().pqkv_ctx_decode_profile_raw(self.h, arr.ctypes.data, arr.size, C.byref(n)))
        return arr

    def set_selection_dump(self, bitmap):
        """Test hook: fused decodes write their selection words into bitmap (or None)."""
        _check(lib().pqkv_ctx_set_selection_dump(self.h, _ptr(bitmap)))

    def last_build_profile(self):
        """SM cycles per phase of problem 0 of the last build."""
        arr = (_u64 * 8)()
        _check(lib().pqkv_ctx_last_build_profile(self.h, arr))
        names = ["seed_chain", "seed_dist", "assign", "update_scatter", "update", "other", "skipped_points",
                 "seed_skipped_points"]
        return {n: int(arr[i]) for i, n in enumerate(names)}

    # ---- (A) build ---------------------------------------------------------
    def kmeans_fit(self, points, k: int, max_iter: int, seeds, inertia: bool = False):
        """points [Q][n][dim] f32 -> (centroids [Q][k][dim], assign [Q][n] i32,
        iterations [Q] i32, inertia [Q][max_iter] f64 | None)."""
        import torch

        Q, n, dim = points.shape
        cen = torch.empty((Q, k, dim), dtype=torch.float32, device=points.device)
        asg = torch.empty((Q, n), dtype=torch.int32, device=points.device)
        its = torch.empty((Q,), dtype=torch.int32, device=points.device)
        inr = torch.zeros((Q, max_iter), dtype=torch.float64, device=points.device) if inertia else None
        sd = (C.c_uint64 * Q)(*[int(s) & (2**64 - 1) for s in seeds])
        _check(lib().pqkv_kmeans_fit(self.h, _ptr(points), Q, n * dim, dim, n, dim, k, max_iter, sd,
                                     _ptr(cen), _ptr(asg), _ptr(its), _ptr(inr), _stream()))
        return cen, asg, its, inr

    def pq_build(self, keys, m: int, b: int, max_iter: int, seeds):
        """keys [P][s][d_h] f32 -> (centroids [P][m][2^b][d_m] f32, codes [P][s][m] i16 (u16 bits))."""
        import torch

        P, s, d_h = keys.shape
        cen = torch.empty((P, m, 1 << b, d_h // m), dtype=torch.float32, device=keys.device)
        codes = torch.empty((P, s, m), dtype=torch.int16, device=keys.device)
        sd = (C.c_uint64 * P)(*[int(x) & (2**64 - 1) for x in seeds])
        _check(lib().pqkv_pq_build(self.h, _ptr(keys), P, s * d_h, s, d_h, m, b, max_iter, sd, _ptr(cen),
                                   _ptr(codes), s * m, _stream()))
        return cen, codes

    def pq_encode(self, keys, centroids, b: int, codes, row: int):
        """Encode keys [P][d_h] and write code row `row` of codes [P][cap][m]."""
        P, d_h = keys.shape
        m = centroids.shape[1]
        _check(lib().pqkv_pq_encode(self.h, _ptr(keys), P, d_h, d_h, m, b, _ptr(centroids), _ptr(codes),
                                    codes.shape[1] * m, row, _stream()))

    def assign_nearest(self, points, centroids):
        import torch

        n, dim = points.shape
        out = torch.empty((n,), dtype=torch.int32, device=points.device)
        _check(lib().pqkv_assign_nearest(self.h, _ptr(points), n, dim, _ptr(centroids), centroids.shape[0],
                                         _ptr(out), _stream()))
        return out

    # ---- (B) decode retrieval ------------------------------------------------
    def pq_score(self, queries, centroids, codes, b: int):
        """queries [P][g][d_h], codes [P][s][m] -> scores [P][s] f32 (pq_score_gqa)."""
        import torch

        P, g, d_h = queries.shape
        m = centroids.shape[1]
        s = codes.shape[1]
        out = torch.empty((P, s), dtype=torch.float32, device=queries.device)
        _check(lib().pqkv_pq_score(self.h, _ptr(queries), P, g, d_h, m, b, _ptr(centroids), _ptr(codes),
                                   s * m, s, _ptr(out), s, _stream()))
        return out

    def topk(self, scores, k: int, excluded=None):
        """scores [R][n] -> ids [R][k] int64 in (score desc, id asc) order."""
        import torch

        R, n = scores.shape
        ids = torch.empty((R, max(k, 1)), dtype=torch.int64, device=scores.device)
        _check(lib().pqkv_topk(self.h, _ptr(scores), R, n, n, k, _ptr(excluded), _ptr(ids), _stream()))
        return ids[:, :k]

    def tuple_tables(self, codes, b: int, s: int | None = None, tables=None, row_begin: int = 0):
        """Code-pair tables for the m == 2 selection path: (thist [P][C*C] i32,
        chist [P][chunks][C*C] i16).  Adds rows [row_begin, s) to `tables`."""
        import torch

        P, cap, m = codes.shape
        s = cap if s is None else s
        C2 = (1 << b) ** 2
        chunks = max(1, (cap + TUPLE_CHUNK - 1) // TUPLE_CHUNK)
        if tables is None:
            tables = (torch.zeros((P, C2), dtype=torch.int32, device=codes.device),
                      torch.zeros((P, chunks, C2), dtype=torch.int16, device=codes.device))
        th, ch = tables
        _check(lib().pqkv_pq_tuple_tables(self.h, P, b, _ptr(codes), cap * m, row_begin, s, _ptr(th), _ptr(ch),
                                          ch.shape[1], _stream()))
        return tables

    def pq_search(self, queries, centroids, codes, b: int, k: int, s: int | None = None,
                  bitmap: bool = True, ordered: bool = True, tables=None):
        """Fused ADC + select -> (bitmap [P][ceil(s/32)] i32 | None, ids [P][k] | None)."""
        import torch

        P, g, d_h = queries.shape
        m = centroids.shape[1]
        cap = codes.shape[1]
        s = cap if s is None else s
        words = (s + 31) // 32
        bm = torch.empty((P, max(words, 1)), dtype=torch.int32, device=queries.device) if bitmap else None
        ids = torch.empty((P, max(k, 1)), dtype=torch.int64, device=queries.device) if ordered else None
        th, ch = tables if tables is not None else (None, None)
        _check(lib().pqkv_pq_search(self.h, _ptr(queries), P, g, d_h, m, b, _ptr(centroids), _ptr(codes),
                                    cap * m, s, k, _ptr(bm), _ptr(ids), _ptr(th), _ptr(ch),
                                    ch.shape[1] if ch is not None else 0, _stream()))
        return bm, (ids[:, :k] if ids is not None else None)

    def exact_scores(self, queries, keys, rows):
        import torch

        P, g, d_h = queries.shape
        t = rows.shape[1]
        out = torch.empty((P, g, t), dtype=torch.float32, device=queries.device)
        _check(lib().pqkv_exact_scores(self.h, _ptr(queries), P, g, d_h, _ptr(keys), keys[0].numel(),
                                       _ptr(rows), t, _ptr(out), _stream()))
        return out

    def attend_rows(self, queries, keys, values, rows, precision: int = PREC_F32):
        """Softmax attention of queries [P][g][d_h] over rows [P][t] of keys/values [P][S][d_h]."""
        import torch

        P, g, d_h = queries.shape
        t = rows.shape[1]
        out = torch.empty((P, g, d_h), dtype=torch.float32, device=queries.device)
        _check(lib().pqkv_attend_rows(self.h, _ptr(queries), P, g, d_h, _ptr(keys), _ptr(values),
                                      keys[0].numel(), _ptr(rows), t, precision, _ptr(out), _stream()))
        return out

    def decode(self, layer: "DecodeLayer", queries, k: int, want_ids: bool = False, out=None):
        import torch

        P, g, d_h = queries.shape
        if out is None:
            out = torch.empty((P, g, d_h), dtype=torch.float32, device=queries.device)
        ids = torch.empty((P, max(k, 1)), dtype=torch.int64, device=queries.device) if want_ids else None
        _check(lib().pqkv_decode(self.h, layer.ref(), _ptr(queries), g, k, _ptr(out), _ptr(ids), _stream()))
        return (out, ids[:, :k]) if want_ids else out

    def decode_plan(self, layer: "DecodeLayer", g: int, k: int, want_ids: bool = False) -> dict:
        """The launch plan pqkv_decode picks for this layer / g / k (pqkv_decode_plan)."""
        out = pqkv_decode_plan_t()
        L = layer.struct()
        _check(lib().pqkv_decode_plan(self.h, C.byref(L), g, k, int(want_ids), C.byref(out)))
        d = {name: getattr(out, name) for name, _ in pqkv_decode_plan_t._fields_}
        d["mode"] = PLAN_MODES.get(d["mode"], d["mode"])
        return d

    # ---- experiment metrics (experiments.cpp:26-139) -------------------------
    def exact_topk(self, queries, keys, k: int, n: int | None = None):
        """Top-k of the f32 row sum of queries [P][g][d_h] against key rows
        [0, n) of keys [P][S][d_h] (exact_scores, topk tie rule) -> [P][k] i64."""
        import torch

        P, g, d_h = queries.shape
        n = keys.shape[1] if n is None else n
        ids = torch.empty((P, max(k, 1)), dtype=torch.int64, device=queries.device)
        _check(lib().pqkv_exact_topk(self.h, _ptr(queries), P, g, d_h, _ptr(keys), keys[0].numel(), n, k, _ptr(ids),
                                     _stream()))
        return ids[:, :k]

    def attend_dense(self, queries, keys, values, t: int | None = None, precision: int = PREC_F64):
        """Attention of queries [P][g][d_h] over rows [0, t) -> [P][g][d_h]."""
        import torch

        P, g, d_h = queries.shape
        t = keys.shape[1] if t is None else t
        out = torch.empty((P, g, d_h), dtype=torch.float32, device=queries.device)
        _check(lib().pqkv_attend_dense(self.h, _ptr(queries), P, g, d_h, _ptr(keys), _ptr(values), keys[0].numel(), t,
                                       precision, _ptr(out), _stream()))
        return out

    def relative_error(self, got, want):
        """Per-row relative_error of [rows][...] f32 tensors -> [rows] f64."""
        import torch

        rows = got.shape[0]
        n = got[0].numel()
        out = torch.empty((rows,), dtype=torch.float64, device=got.device)
        _check(lib().pqkv_relative_error(self.h, _ptr(got.contiguous()), _ptr(want.contiguous()), rows, n, _ptr(out),
                                         _stream()))
        return out

    def overlap_fraction(self, got_ids, want_ids, n_ids: int):
        """Per-row |got ∩ want| / |want| of id lists [rows][k] -> [rows] f64."""
        import torch

        rows = want_ids.shape[0]
        out = torch.empty((rows,), dtype=torch.float64, device=want_ids.device)
        _check(lib().pqkv_overlap_fraction(self.h, _ptr(got_ids.contiguous()), got_ids.shape[1],
                                           _ptr(want_ids.contiguous()), want_ids.shape[1], rows, n_ids, _ptr(out),
                                           _stream()))
        return out

    def comm_init(self, unique_id: bytes, n_ranks: int, rank: int) -> "Comm":
        """NCCL communicator for pqkv_decode_sharded (ncclCommInitRank protocol:
        rank 0's comm_unique_id() broadcast to every rank)."""
        h = _vp()
        _check(lib().pqkv_comm_init(self.h, C.c_char_p(bytes(unique_id)), n_ranks, rank, C.byref(h)))
        return Comm(h, n_ranks, rank)

    def decode_sharded(self, comm: "Comm", layers, queries, k: int, units_per_rank: int, out=None):
        """This rank's shard of every layer decoded + one all-gather of all
        ranks' outputs -> [n_ranks][n_layers][units_per_rank][g][d_h]."""
        import torch

        n = len(layers)
        g, d_h = queries[0].shape[1], queries[0].shape[2]
        if out is None:
            out = torch.empty((comm.n_ranks, n, units_per_rank, g, d_h), dtype=torch.float32,
                              device=queries[0].device)
        arr = (pqkv_layer * n)(*[l.struct() for l in layers])
        qp = (_vp * n)(*[q.data_ptr() for q in queries])
        for q in queries:
            _ptr(q)
        _check(lib().pqkv_decode_sharded(self.h, comm.h, arr, n, units_per_rank, qp, g, k, _ptr(out), _stream()))
        return out

    def decode_step(self, layer: "DecodeLayer", new_keys, new_values, queries, k: int, want_ids: bool = False):
        """One e2e step (evict_local_append + decode, pqkv_decode_step): new_keys /
        new_values [P][d_h] become token layer.total; layer.total grows by one."""
        import torch

        P, g, d_h = queries.shape
        out = torch.empty((P, g, d_h), dtype=torch.float32, device=queries.device)
        ids = torch.empty((P, max(k, 1)), dtype=torch.int64, device=queries.device) if want_ids else None
        L = layer.struct()
        try:
            _check(lib().pqkv_decode_step(self.h, C.byref(L), layer.codes.shape[1], _ptr(new_keys),
                                          _ptr(new_values), _ptr(queries), g, k, _ptr(out), _ptr(ids), _stream()))
        finally:
            layer.total = L.total  # the C side grows total only once the token is appended
        return (out, ids[:, :k]) if want_ids else out

    def gen_workload(self, s: int, d_h: int = 128, h_kv: int = 1, g: int = 1, kind: str = "gaussian",
                     n_components: int = 8, spread: float = 0.5, zipf: float = 1.0, seed: int = 7, out=None):
        """Device-generated synthetic workload (pqkv_gen_workload): (keys [h][s][d],
        values [h][s][d], queries [h][g][d]) f32 on this context's device; `out` may
        supply (keys, values, queries) tensors (e.g. views of a larger cache)."""
        import torch

        dev = torch.device("cuda", self.device)
        if out is None:
            out = (torch.empty((h_kv, s, d_h), dtype=torch.float32, device=dev),
                   torch.empty((h_kv, s, d_h), dtype=torch.float32, device=dev),
                   torch.empty((h_kv, g, d_h), dtype=torch.float32, device=dev))
        k, v, q = out
        kd = {"gaussian": 0, "powerlaw": 1}[kind]
        _check(lib().pqkv_gen_workload(self.h, kd, s, d_h, h_kv, g, n_components, spread, zipf, seed, _ptr(k),
                                       _ptr(v), _ptr(q), _stream()))
        return k, v, q

    def block_rank(self, ids, n_tokens: int, block_size: int, k_cache: int):
        """Block-cache accounting of a fetch (pqkv_block_rank): ids [P][n] int64 token
        ids -> (bitmap [P][words] i32, counts [P][blocks] i32, ranked [P][k_cache] i64,
        touched [P] i32)."""
        import torch

        P, n = ids.shape
        words = (n_tokens + 31) // 32
        nb = max(1, (n_tokens + block_size - 1) // block_size)
        dev = ids.device
        bm = torch.empty((P, max(words, 1)), dtype=torch.int32, device=dev)
        counts = torch.empty((P, nb), dtype=torch.int32, device=dev)
        ranked = torch.empty((P, max(k_cache, 1)), dtype=torch.int64, device=dev)
        touched = torch.empty((P,), dtype=torch.int32, device=dev)
        _check(lib().pqkv_block_rank(self.h, _ptr(ids), P, ids.stride(0), n, n_tokens, block_size, k_cache,
                                     _ptr(bm), _ptr(counts), _ptr(ranked), _ptr(touched), _stream()))
        return bm, counts, ranked[:, :k_cache], touched

    def decode_attend(self, layer: "DecodeLayer", queries, bitmap, out=None):
        """Attention half of decode for a selection bitmap from pq_search."""
        import torch

        P, g, d_h = queries.shape
        if out is None:
            out = torch.empty((P, g, d_h), dtype=torch.float32, device=queries.device)
        L = layer.struct()
        _check(lib().pqkv_decode_attend(self.h, C.byref(L), _ptr(queries), g, _ptr(bitmap), _ptr(out),
                                        _stream()))
        return out

    def decode_host(self, layer: "DecodeLayer", h_queries, h_out, k: int):
        """h_queries / h_out: pinned CPU tensors [P][g][d_h]; synchronous."""
        P, g, d_h = h_queries.shape
        _check(lib().pqkv_decode_host(self.h, layer.ref(), C.c_void_p(h_queries.data_ptr()), g, k,
                                      C.c_void_p(h_out.data_ptr()), _stream()))


def recall_seeds(seed: int, h_kv: int, ks, s: int):
    """run_recall's seeder draws (experiments.cpp:90-113): (fork seeds [h_kv]
    u64, random ids [h_kv][sum ks] i64 -- per k, k distinct ids of [0, s))."""
    import numpy as np

    ks = [int(k) for k in ks]
    fs = np.zeros(h_kv, np.uint64)
    ri = np.zeros((h_kv, max(1, sum(ks))), np.int64)
    karr = (_sz * len(ks))(*ks)
    _check(lib().pqkv_recall_seeds(int(seed) & (2**64 - 1), h_kv, karr, len(ks), s, fs.ctypes.data, ri.ctypes.data))
    return fs, ri


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through libpqkv (run on rank 0, then broadcast)."""
    buf = C.create_string_buffer(128)
    _check(lib().pqkv_comm_unique_id(buf))
    return buf.raw


class Comm:
    """A pqkv_comm (NCCL communicator + its collective stream)."""

    def __init__(self, h, n_ranks: int, rank: int):
        self.h, self.n_ranks, self.rank = h, n_ranks, rank

    def close(self):
        if self.h:
            lib().pqkv_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class DecodeLayer:
    """Device-resident KV cache + PQ index of one layer (pqkv_layer).

    keys/values [P][S][d_h] f32 (row = token id, S >= total), centroids
    [P][m][2^b][d_m] f32, codes [P][cap][m] int16 (middle row r = token n_init+r).
    """

    keys: object
    values: object
    centroids: object
    codes: object
    total: int
    n_init: int
    n_local: int
    b: int
    tables: tuple | None = None  # (thist, chist) from Context.tuple_tables

    def struct(self) -> pqkv_layer:
        P, S, d_h = self.keys.shape
        m = self.centroids.shape[1]
        return pqkv_layer(
            keys=self.keys.data_ptr(), values=self.values.data_ptr(), kv_head_stride=S * d_h,
            n_heads=P, total=self.total, n_init=self.n_init, n_local=self.n_local, d_h=d_h, m=m,
            b=self.b, centroids=self.centroids.data_ptr(), codes=self.codes.data_ptr(),
            codes_head_stride=self.codes.shape[1] * m,
            tuple_hist=self.tables[0].data_ptr() if self.tables is not None else None,
            tuple_chunk_hist=self.tables[1].data_ptr() if self.tables is not None else None,
            tuple_chunks=self.tables[1].shape[1] if self.tables is not None else 0,
        )

    def ref(self):
        """ctypes reference to a cached pqkv_layer (rebuilt when the fields change)."""
        key = (self.keys.data_ptr(), self.values.data_ptr(), self.centroids.data_ptr(), self.codes.data_ptr(),
               self.total, self.n_init, self.n_local, self.b,
               None if self.tables is None else (self.tables[0].data_ptr(), self.tables[1].data_ptr()))
        cache = self.__dict__.get("_ref_cache")
        if cache is None or cache[0] != key:
            L = self.struct()
            cache = (key, L, C.byref(L))
            self.__dict__["_ref_cache"] = cache
        return cache[2]

    def launches(self, g: int, with_ids: bool = False) -> int:
        L = self.struct()
        return lib().pqkv_decode_launches(C.byref(L), g, int(with_ids))


def pq_config(m: int, b: int, d_h: int):
    """PqConfig::create -> (d_m, n_clusters); ValueError on the reference's rejections."""
    d_m, c = _sz(0), _sz(0)
    _check(lib().pqkv_pq_config(m, b, d_h, C.byref(d_m), C.byref(c)))
    return d_m.value, c.value


def codes_memory_ratio(m: int, b: int, d_h: int) -> float:
    r = C.c_double(0)
    _check(lib().pqkv_codes_memory_ratio(m, b, d_h, C.byref(r)))
    return r.value
