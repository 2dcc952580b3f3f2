"""Device-resident run_recall (reference experiments.cpp:74-139).

For every (m, b, seed) of a grid: PQ indexes of all kv heads built at once on
the GPU (pq_construct seeds from the reference's seeder stream), ADC scores,
approx top-k, exact top-k of the summed group query, a seeded random
selection, full attention over all tokens and attention over each selection
-- all batched over heads on the device -- then recall (overlap_fraction)
and output error (relative_error), averaged over heads.  Same arithmetic as
the reference (the fp64 attention path, bit-exact selections), so the CSV
equals write_recall_csv's byte for byte (tests/test_gpu_recall.py).

The workload (keys/values/queries per seed) is an input: device tensors
[h_kv][s][d_h] / [h_kv][g][d_h] from any generator.
"""
from __future__ import annotations

from dataclasses import dataclass

import paper_2407_12820_b200 as pq


@dataclass
class RecallRow:
    m: int
    b: int
    k: int
    seed: int
    recall: float = 0.0
    random_recall: float = 0.0
    output_error: float = 0.0
    random_output_error: float = 0.0


def run_recall(ctx, workloads, ms, bs, ks, max_iter: int = 15):
    """workloads: {seed: (keys, values, queries)} device tensors.  Returns
    RecallRows sorted by (m, b, k, seed) like the reference."""
    import torch

    rows = []
    for m in ms:
        for b in bs:
            for seed, (keys, values, queries) in workloads.items():
                h_kv, s, d_h = keys.shape
                fork, rnd = pq.recall_seeds(seed ^ 0x7EC411, h_kv, ks, s)
                cen, codes = ctx.pq_build(keys.contiguous(), m, b, max_iter, [int(x) for x in fork])
                scores = ctx.pq_score(queries, cen, codes, b)
                full = ctx.attend_dense(queries, keys, values, precision=pq.PREC_F64)
                off = 0
                rnd_d = torch.from_numpy(rnd).to(keys.device)
                for k in ks:
                    exact = ctx.exact_topk(queries, keys, k)
                    approx = ctx.topk(scores, k)
                    random = rnd_d[:, off:off + k].contiguous()
                    off += k

                    def err_of(ids):
                        srt, _ = torch.sort(ids, dim=1)
                        sel = ctx.attend_rows(queries, keys, values, srt.contiguous(), precision=pq.PREC_F64)
                        return ctx.relative_error(sel, full)

                    r = RecallRow(m, b, k, seed)
                    r.recall = _mean(ctx.overlap_fraction(approx, exact, s))
                    r.random_recall = _mean(ctx.overlap_fraction(random, exact, s))
                    r.output_error = _mean(err_of(approx))
                    r.random_output_error = _mean(err_of(random))
                    rows.append(r)
    rows.sort(key=lambda r: (r.m, r.b, r.k, r.seed))
    return rows


def _mean(v) -> float:
    """The reference's head average: a running fp64 sum, then * (1 / h_kv)."""
    acc = 0.0
    vals = v.cpu().tolist()
    for x in vals:
        acc += x
    return acc * (1.0 / len(vals))


def recall_csv(rows) -> str:
    """write_recall_csv (experiments.cpp:141-147), %.9g floats."""
    out = ["m,b,k,seed,recall,random_recall,output_error,random_output_error"]
    for r in rows:
        out.append(f"{r.m},{r.b},{r.k},{r.seed},{r.recall:.9g},{r.random_recall:.9g},{r.output_error:.9g},"
                   f"{r.random_output_error:.9g}")
    return "\n".join(out) + "\n"
