"""Per-CTA work balance of a fused decode: selected rows per attention CTA
(from the selection dump) against its measured gather span (profiling
timestamps), to tell row-count imbalance from per-SM speed differences.
Usage: python tools/cta_balance.py [config=cfg3_layer] [kind=gaussian]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_layer"
kind = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
c = bench.CONFIGS[name]
ctx = pq.Context(0)
layer, q, _ = bench.make_layer(ctx, name, kind, seed=1)
G, k = c["g"], bench.cfg_k(c)
plan = ctx.decode_plan(layer, G, k)
s_mid = c["s"] - bench.N_INIT - bench.N_LOCAL
words = torch.zeros((c["units"], (s_mid + 31) // 32), dtype=torch.int32, device="cuda")
for _ in range(3):
    ctx.decode(layer, q, k)
ctx.set_selection_dump(words)
ctx.set_profiling(True)
ctx.decode(layer, q, k)
torch.cuda.synchronize()
ctx.set_profiling(False)
ctx.set_selection_dump(None)
raw = ctx.decode_profile_raw().astype(np.int64)
bits = np.unpackbits(words.cpu().numpy().view(np.uint8), axis=1, bitorder="little")[:, :s_mid]
chunk, nch = plan["chunk_tokens"], plan["ctas_per_head"]
rows = np.zeros((c["units"], nch), np.int64)
for j in range(nch):
    rows[:, j] = bits[:, j * chunk:(j + 1) * chunk].sum(axis=1)
span = (raw[:, 6] - raw[:, 5]).reshape(c["units"], nch) / 1e3
sm = raw[:, 16].reshape(c["units"], nch)
r, sp = rows.ravel(), span.ravel()
print(name, kind, plan)
print("rows/CTA p0/p10/p50/p90/p100:", np.percentile(r, [0, 10, 50, 90, 100]).astype(int))
print("gather span us p0/p10/p50/p90/p100:", np.round(np.percentile(sp, [0, 10, 50, 90, 100]), 1))
print("corr(rows, span) = %.3f" % np.corrcoef(r, sp)[0, 1])
print("span / row (ns) p10/p50/p90:", np.round(np.percentile(sp[r > 0] * 1e3 / r[r > 0], [10, 50, 90]), 1))
ctas_per_sm = np.bincount(sm.ravel())
per = ctas_per_sm[sm.ravel()]
for n in sorted(set(per.tolist())):
    m = per == n
    print(f"CTAs on SMs with {n} CTAs: {m.sum()}, median span {np.median(sp[m]):.1f} us, median rows {np.median(r[m]):.0f}")
# per-SM view: total rows and the latest gather end of the SM's CTAs, and the
# same by SM-id block of 16 (to spot GPC-level structure)
end = (raw[:, 6] - raw[:, 4].min()).reshape(c["units"], nch) / 1e3
sm_rows = np.bincount(sm.ravel(), weights=rows.ravel())
sm_end = np.zeros(sm_rows.shape[0])
np.maximum.at(sm_end, sm.ravel(), end.ravel())
used = sm_rows > 0
print("per-SM rows p0/p50/p100:", np.percentile(sm_rows[used], [0, 50, 100]).astype(int),
      " per-SM last gather end us p0/p50/p100:", np.round(np.percentile(sm_end[used], [0, 50, 100]), 1))
for b0 in range(0, sm_rows.shape[0], 16):
    sl = slice(b0, b0 + 16)
    u = used[sl]
    if u.any():
        print(f"  SMs {b0:3d}-{b0 + 15:3d}: CTAs {int(ctas_per_sm[sl].sum()):3d} rows/SM {sm_rows[sl][u].mean():6.0f} "
              f"end us mean {sm_end[sl][u].mean():5.1f} max {sm_end[sl][u].max():5.1f}")
