#!/usr/bin/env python3
"""Benchmark: decode PQ-retrieve+attend us/layer @128K ctx (+ PQ build tokens/s, HBM GB/s).

Workload (BASELINE.json north_star, N=1): one decoder layer with 32 heads x 128
dim (MHA, g=1), 131072-token context, PQ m=2 b=6 (64 centroids), top-k =
round(s/5) = 26214 middle tokens + 4 initial + 64 local, decode batch 1.  A
"step" is one fused decode of that layer (ADC table -> code scan -> radix
select -> K/V gather -> split-K softmax -> combine) for all 32 heads.
Four independent layers (4 x 4.3 GB of fp32 K/V, each with its own GPU-built
PQ index) rotate across steps, so the 0.86 GB of selected rows per step never
fits the 126 MB L2; queries drift per step as in run_e2e
(experiments.cpp:212-216).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun, one rank per GPU; every rank decodes its own
layers (weak scaling, no collective on the data path); the timed region is
bracketed by barrier + synchronize and the max over ranks is reported.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S, H, DH, G = 131072, 32, 128, 1
M, B, T_ITERS = 2, 6, 10
N_INIT, N_LOCAL = 4, 64
K_SEL = round(S / 5)  # 26214 (k = round(s * ratio))
S_MID = S - N_INIT - N_LOCAL
N_LAYERS = 8
METRIC = "decode PQ-retrieve+attend us/layer @128K ctx"
WORKLOAD = "northstar-1layer-32h-128d-128Kctx-m2b6-top1/5+4init+64local-bs1"
KINDS = ("gaussian", "powerlaw")  # the reference's two key distributions (workload.cpp)


def workload_config(world):
    """The workload both arms run (ours and --impl reference print the same
    dict): geometry, the two key distributions and which one `value` is."""
    return {"workload": WORKLOAD, "global_batch": 1, "seq_len": S, "heads": H, "head_dim": DH, "g": G,
            "m": M, "b": B, "k": K_SEL, "n_init": N_INIT, "n_local": N_LOCAL,
            "key_distributions": list(KINDS), "value_is": "the slower of the two distributions",
            "parallelism": f"dp{world} (independent layers per GPU)",
            "l2": "inputs larger than L2: 8 rotating layers x 4.3 GB K/V per distribution (+26 MB codes and "
                  "pair tables each: 206 MB > L2), 0.86 GB gathered per step"}

# BASELINE.json configs as decode units (one unit = one (request, layer,
# kv_head) K/V set shared by g query heads).  "northstar" is the headline;
# the others are reported beside it (device-timed, rotating layers) and are
# the geometries tests/test_gpu_plans.py pins token for token.
CONFIGS = {
    "northstar": dict(units=32, g=1, s=131072, m=2, b=6, ratio=5, tables=True, layers=N_LAYERS,
                      what="configs[1] geometry at 128K: 32 heads x 128 dim, m2b6, top 1/5 + 4 + 64, bs1"),
    "cfg1": dict(units=8, g=1, s=4096, m=2, b=6, ratio=5, tables=True, layers=16,
                 what="configs[0]: 8 heads x 4K, m2b6, top 1/5 (the CPU reference's own case)"),
    "cfg2": dict(units=32, g=1, s=32768, m=2, b=6, ratio=5, tables=True, layers=4,
                 what="configs[1]: 32 heads x 32K, m2b6, top 1/5 + 4 + 64, bs1"),
    "cfg3_layer": dict(units=8, g=4, s=131072, m=2, b=6, ratio=5, tables=True, layers=4,
                       what="configs[2] per layer: Llama-3-8B shape, 8 kv heads x g4 x 128K, m2b6, top 1/5"),
    "cfg5_per_gpu": dict(units=16, g=4, s=131072, m=4, b=8, ratio=10, tables=False, layers=4,
                         what="configs[4] per GPU at 8 GPUs: 16 (request, kv head) units x g4 x 128K, m4b8, "
                              "top 1/10"),
}


def cfg_k(c):
    return round(c["s"] / c["ratio"])


def cfg_bytes(c):
    """B = units * [s_mid m b/8 + C d_h 4 + T_att d_h 4 2 + 2 g d_h 4]."""
    s_mid = c["s"] - N_INIT - N_LOCAL
    t_att = N_INIT + cfg_k(c) + N_LOCAL
    return c["units"] * (s_mid * c["m"] * c["b"] / 8 + (1 << c["b"]) * DH * 4 + t_att * DH * 4 * 2
                         + 2 * c["g"] * DH * 4)


def make_layer(ctx, name, kind="gaussian", seed=0):
    """One layer of config `name`: device-generated K/V/queries (pqkv_gen_workload,
    the reference's gaussian-mixture / powerlaw distributions) and its PQ index
    built on the GPU (pq_construct semantics, T = 10) plus the code-pair tables.
    Returns (DecodeLayer, base queries [units][g][d_h], build seconds)."""
    import torch

    import paper_2407_12820_b200 as pq

    c = CONFIGS[name]
    s, s_mid = c["s"], c["s"] - N_INIT - N_LOCAL
    keys, vals, base_q = ctx.gen_workload(s, DH, h_kv=c["units"], g=c["g"], kind=kind, n_components=8,
                                          spread=0.5, seed=seed)
    mids = keys[:, N_INIT:N_INIT + s_mid].contiguous()
    seeds = [7 + 131 * seed + h for h in range(c["units"])]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cen, codes = ctx.pq_build(mids, c["m"], c["b"], T_ITERS, seeds)
    tables = ctx.tuple_tables(codes, c["b"]) if c["tables"] else None
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    del mids
    layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=s, n_init=N_INIT,
                           n_local=N_LOCAL, b=c["b"], tables=tables)
    return layer, base_q, secs


def algorithmic_bytes_per_layer():
    return cfg_bytes(CONFIGS["northstar"])


def attend_bytes_per_launch():
    """Bytes the attention kernel pair must move: K+V of the T_att selected rows,
    the selection bitmap, queries in, outputs out."""
    t_att = N_INIT + K_SEL + N_LOCAL
    words = (S_MID + 31) // 32
    return H * (t_att * DH * 4 * 2 + words * 4 + 2 * G * DH * 4)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled every 10 ms by a separate process
    (tools/clock_sampler.py, NVML) while the timed region runs; only samples
    inside [enter, exit] are kept."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.out = None

    def start(self):
        import subprocess
        import tempfile

        self.out = tempfile.NamedTemporaryFile("w+", suffix=".jsonl", delete=False)
        try:
            self.proc = subprocess.Popen([sys.executable, os.path.join(ROOT, "tools", "clock_sampler.py"),
                                          str(self.device), "0.01"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
            time.sleep(1.0)  # sampler up before the timed region
        except Exception:
            self.proc = None
        return self

    def __enter__(self):
        self.windows = getattr(self, "windows", [])
        self.windows.append([time.time(), None])
        return self

    def __exit__(self, *a):
        self.windows[-1][1] = time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows, max_mhz = [], None
        if self.out:
            self.out.flush()
            with open(self.out.name) as f:
                for line in f:
                    try:
                        v = json.loads(line)
                    except Exception:
                        continue
                    if isinstance(v, dict):
                        max_mhz = v.get("max_mhz", max_mhz)
                    elif any(t0 - 0.005 <= v[0] <= t1 + 0.005 for t0, t1 in getattr(self, "windows", [])):
                        rows.append(v)
            os.unlink(self.out.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": max_mhz, "reasons": ["unsampled"], "samples": 0}
        bits = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
        sm = sorted(r[1] for r in rows)
        reasons = sorted({name for r in rows for bit, name in bits.items() if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max_mhz, "reasons": reasons, "samples": len(rows)}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU decode (oracle/_ref) on all host
    cores, bounded sample of the same workload, extrapolated to us/layer."""
    import numpy as np

    import oracle

    if rank != 0:
        return
    line = {"impl": "reference", "metric": METRIC, "unit": "us/layer", "higher_is_better": False,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "scaling": "weak",
            "dtype": "f32 storage, f64 arithmetic", "data": "synthetic", "config": workload_config(args.gpus)}
    if not oracle.has_ref():
        line["unavailable"] = "oracle/_ref/libpqkv_ref.so was not built (needs /root/reference at build time)"
        print(json.dumps(line), flush=True)
        return
    ref = oracle.ref()
    cores = os.cpu_count() or 1
    P = min(H, max(1, cores))  # one head per host thread
    rng = np.random.default_rng(17)
    n_total = args.warmup + args.steps
    sigma = 0.25 / math.sqrt(DH)
    per_kind = {}
    for kind in KINDS:
        # the reference's own generator (workload.cpp: gaussian mixture /
        # powerlaw keys) and its own index (pq_construct on all host cores),
        # both untimed setup
        keys, vals, queries = ref.gen_workload(S, DH, h_kv=P, g=G, kind=oracle.KINDS[kind], n_components=8,
                                               spread=0.5, seed=17 + KINDS.index(kind))
        mids = np.ascontiguousarray(keys[:, N_INIT:N_INIT + S_MID])
        _, cen, codes = ref.bench_build(mids, M, B, T_ITERS, np.arange(P, dtype=np.uint64) + 11, 0)
        del mids
        qs = (queries[None] + sigma * rng.standard_normal((n_total, P, G, DH))).astype(np.float32)
        # HeadStates are built once (kv_store offload_prefill); every step is
        # one decode of the P sampled heads (pq_score_gqa + approx_topk +
        # selective_attention), one head per host thread
        secs, _ = ref.bench_decode_steps(keys, vals, qs, cen, codes, N_INIT, N_LOCAL, K_SEL, 0)
        per_kind[kind] = float(np.mean(secs[args.warmup:])) * 1e6 * (H / P)
        del keys, vals, qs, cen, codes
    worst = max(per_kind, key=per_kind.get)
    per_layer_us = per_kind[worst]
    line.update({"value": per_layer_us, "ms_per_step": per_layer_us / 1e3,
                 "distributions": {"us_per_layer": per_kind, "slower": worst},
                 "cpu_baseline": {"value": per_layer_us, "unit": "us/layer", "cores": min(cores, P),
                                  "kind": "reference",
                                  "sample": f"{P} of {H} heads per step (x{H / P:g} to a layer), "
                                            "pq_score_gqa+approx_topk+selective_attention, keys from the "
                                            "reference's generator, index built by the reference's pq_construct; "
                                            "the slower of the two distributions"},
                 "e2e": {"value": per_layer_us, "unit": "us/layer", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(layer, base_q, gpu_out, gpu_words):
    """The reference (oracle/_ref, the unmodified library) on this box's host
    cores for a bounded sample: P = min(32, cores) heads of headline layer 0
    (same GPU-built index -- bit-identical to the reference's), one head per
    host thread, 1 warm-up + 3 timed steps, median extrapolated x32/P to the
    layer.  Parity on the same inputs: the GPU's selection words equal the
    reference's approx_topk set, and the outputs are within 1e-3 relative.
    Plus a build sample: pq_construct over P heads x 32K tokens on P threads."""
    import numpy as np

    import oracle

    if not oracle.has_ref():
        return None, None
    ref = oracle.ref()
    cores = os.cpu_count() or 1
    P = min(H, max(1, cores))
    k = layer.keys[:P].cpu().numpy()
    v = layer.values[:P].cpu().numpy()
    q = base_q[:P].cpu().numpy()
    c = layer.centroids[:P].cpu().numpy()
    cd = layer.codes[:P].cpu().numpy().view(np.uint16)
    qs = np.repeat(q[None], 4, axis=0)
    secs, want = ref.bench_decode_steps(k, v, qs, c, cd, N_INIT, N_LOCAL, K_SEL, P)
    dec = {"value": float(np.median(secs[1:])) * 1e6 * (H / P), "unit": "us/layer", "cores": P,
           "kind": "reference",
           "sample": f"{P} of {H} heads of one 128K layer (gaussian), one head per thread, median of 3 warm "
                     f"steps, x{H / P:g} to a layer"}
    got = gpu_out[:P].cpu().numpy()
    rel = float(np.abs(got - want).max() / np.abs(want).max())
    words = gpu_words[:P].cpu().numpy().view(np.uint32)
    sel_ok = True
    for p in range(min(P, 4)):  # selection sets of 4 heads against the reference's approx_topk
        rows = ref.top_k_desc(ref.pq_score_gqa(q[p], c[p], cd[p]), K_SEL)
        got_rows = np.flatnonzero(np.unpackbits(words[p].view(np.uint8), bitorder="little")[:S_MID])
        sel_ok = sel_ok and np.array_equal(got_rows, np.sort(rows).astype(np.int64))
    dec["parity"] = {"heads": P, "max_rel_err": rel, "tolerance": 1e-3, "selection_heads": min(P, 4),
                     "selection_equal": bool(sel_ok), "ok": bool(rel < 1e-3 and sel_ok)}
    sb = 32768
    mids = np.ascontiguousarray(k[:, N_INIT:N_INIT + sb])
    bsecs, _, _ = ref.bench_build(mids, M, B, T_ITERS, np.arange(P, dtype=np.uint64) + 5, P)
    bld = {"value": P * sb / bsecs, "unit": "key vectors/s", "cores": P, "kind": "reference",
           "sample": f"pq_construct m2b6 T={T_ITERS} on {P} heads x {sb} tokens, one head per thread"}
    return dec, bld


def time_steps(ctx, layers, queries, k, n_warm, n_steps, dist=None, dev=None, clk=None):
    """Device time (ms) of n_steps decodes rotating over `layers` (CUDA events on
    the launching stream, barrier + synchronize on both sides, max over ranks)."""
    import torch

    stream = torch.cuda.current_stream()
    nl = len(layers)
    for i in range(n_warm):
        ctx.decode(layers[i % nl], queries[i % len(queries)], k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clk:
        clk.__enter__()
    ev0.record(stream)
    for i in range(n_warm, n_warm + n_steps):
        ctx.decode(layers[i % nl], queries[i % len(queries)], k)
    ev1.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def drift_queries(base, n, sigma, gen):
    """Per-step query drift of run_e2e (experiments.cpp:212-216)."""
    import torch

    return [base + sigma * torch.randn(base.shape, generator=gen, device=base.device) for _ in range(n)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="headline only (skip cfg1/2/3/5 lines)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch

    import paper_2407_12820_b200 as pq

    assert args.warmup >= 3, "timing rules: >= 3 warm-up steps"
    # PQKV_BENCH_DEVICE / PQKV_BENCH_BACKEND: exercise the multi-rank logic on
    # one GPU (tests only: several ranks on one device over gloo)
    local_dev = int(os.environ.get("PQKV_BENCH_DEVICE", local))
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("PQKV_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    ctx = pq.Context(local_dev)
    n_total = args.warmup + args.steps
    sigma = 0.25 / math.sqrt(DH)
    gq = torch.Generator(device=dev)
    gq.manual_seed(99 + rank)

    # ---- headline: both of the reference's key distributions, 8 rotating layers each ----
    heads = {}
    build_s = []
    rech_tot = [0, 0]
    for kind in ("gaussian", "powerlaw"):
        layers, qs = [], []
        for li in range(N_LAYERS):
            layer, base_q, secs = make_layer(ctx, "northstar", kind, seed=1000 * rank + 16 * li + (kind == "powerlaw"))
            if kind == "gaussian":
                build_s.append(secs)
                r, t = ctx.last_build_stats()
                rech_tot[0] += r
                rech_tot[1] += t
            layers.append(layer)
            qs.append(base_q)
        queries = [qs[i % N_LAYERS] + sigma * torch.randn(qs[0].shape, generator=gq, device=dev)
                   for i in range(max(n_total, N_LAYERS))]
        heads[kind] = (layers, qs, queries)

    clk = ClockSampler(local_dev).start()
    timed = {}
    # warm-up: W steps, and at least one pass over every rotating layer (first
    # touches of a layer's 4.3 GB are TLB-cold)
    n_warm = max(args.warmup, 2 * N_LAYERS)
    for kind in ("gaussian", "powerlaw"):
        layers, _, queries = heads[kind]
        timed[kind] = time_steps(ctx, layers, queries, K_SEL, n_warm, args.steps, dist, dev, clk)
    worst = max(timed, key=lambda kd: timed[kd])
    ms = timed[worst]
    ms_per_step = ms / args.steps
    us_per_layer = ms * 1e3 / (args.steps * world)
    layers, base_qs, queries = heads[worst]
    plan = ctx.decode_plan(layers[0], G, K_SEL)
    launches_per_step = layers[0].launches(G)

    peak, peak_kind = peaks()

    # ---- dominant kernel (attention gather + combine) timed alone ----
    stream = torch.cuda.current_stream()
    bms = []
    for i in range(N_LAYERS):
        bm, _ = ctx.pq_search(queries[i], layers[i].centroids, layers[i].codes, B, K_SEL, s=S_MID,
                              bitmap=True, ordered=False, tables=layers[i].tables)
        bms.append(bm)
    out = torch.empty((H, G, DH), dtype=torch.float32, device=dev)
    sel_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
    reps = max(args.steps, 8)
    for i in range(3):
        ctx.decode_attend(layers[i % N_LAYERS], queries[i], bms[i % N_LAYERS], out)
    torch.cuda.synchronize()
    sel_ev[0][0].record(stream)
    for i in range(reps):
        ctx.decode_attend(layers[i % N_LAYERS], queries[i % N_LAYERS], bms[i % N_LAYERS], out)
    sel_ev[0][1].record(stream)
    sel_ev[1][0].record(stream)
    for i in range(reps):
        li = i % N_LAYERS
        ctx.pq_search(queries[li], layers[li].centroids, layers[li].codes, B, K_SEL, s=S_MID, bitmap=True,
                      ordered=False, tables=layers[li].tables)
    sel_ev[1][1].record(stream)
    torch.cuda.synchronize()
    attend_ms = sel_ev[0][0].elapsed_time(sel_ev[0][1]) / reps
    select_ms = sel_ev[1][0].elapsed_time(sel_ev[1][1]) / reps

    # ---- end to end through the C ABI with HOST buffers (pinned in, pinned out) ----
    hq = [q.cpu().pin_memory() for q in queries[:N_LAYERS]]
    ho = torch.empty((H, G, DH), dtype=torch.float32).pin_memory()
    # every rotating layer's call is captured as a CUDA graph on its second
    # sighting: warm up twice per layer so no capture lands in the timed loop
    for i in range(max(args.warmup, 2 * N_LAYERS)):
        ctx.decode_host(layers[i % N_LAYERS], hq[i % N_LAYERS], ho, K_SEL)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        ctx.decode_host(layers[i % N_LAYERS], hq[i % N_LAYERS], ho, K_SEL)
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_us = e2e_s * 1e6 / (args.steps * world)

    # ---- cfg4: one layer's heads sharded over the ranks + NCCL all-gather ----
    # (BASELINE configs[3]; the path itself has no exchange, the gathered
    # outputs are what the next layer's projection needs).  Through the C ABI:
    # pqkv_decode_sharded = this rank's decodes + one NCCL all-gather on a
    # collective stream, per layer and batched over the 8 layers of a call.
    from paper_2407_12820_b200 import shard

    hr = shard.partition(H, world, rank)
    upr = len(shard.partition(H, world, 0))  # units per rank (rank 0 has the most)
    subs = []
    for l0 in layers:
        th, ch = l0.tables
        subs.append(pq.DecodeLayer(keys=l0.keys[hr.start:hr.stop], values=l0.values[hr.start:hr.stop],
                                   centroids=l0.centroids[hr.start:hr.stop], codes=l0.codes[hr.start:hr.stop],
                                   total=S, n_init=N_INIT, n_local=N_LOCAL, b=B,
                                   tables=(th[hr.start:hr.stop], ch[hr.start:hr.stop])))
    qsub = [queries[i][hr.start:hr.stop].contiguous() for i in range(N_LAYERS)]
    hs = {}
    try:
        comm = shard.nccl_comm(ctx)
    except Exception as e:  # e.g. NCCL refusing several ranks on one device (tests)
        comm = None
        hs = {1: None, N_LAYERS: None, "error": repr(e)[:200]}
    for batch in ((1, N_LAYERS) if comm is not None else ()):
        calls = max(4, min(args.steps, 200) // batch)
        def call(i):
            ls = [subs[(i * batch + j) % N_LAYERS] for j in range(batch)]
            qq = [qsub[(i * batch + j) % N_LAYERS] for j in range(batch)]
            return ctx.decode_sharded(comm, ls, qq, K_SEL, upr)
        for i in range(3):
            call(i)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        hs0, hs1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hs0.record(stream)
        for i in range(calls):
            full = call(i)
        hs1.record(stream)
        torch.cuda.synchronize()
        hs[batch] = shard.max_over_ranks(hs0.elapsed_time(hs1) * 1e3 / (calls * batch), dev)
    if comm is not None:
        assert shard.unshard(full, H).shape[1] == H
        comm.close()
    del subs, qsub

    # ---- the other BASELINE configs, device-timed (rotating layers) ----
    extra = {}
    if not args.no_extra:
        for name in ("cfg1", "cfg2", "cfg3_layer", "cfg5_per_gpu"):
            c = CONFIGS[name]
            made = [make_layer(ctx, name, "gaussian", seed=5000 + 1000 * rank + li) for li in range(c["layers"])]
            ls = [m_[0] for m_ in made]
            qx = [made[i % len(made)][1] + sigma * torch.randn(made[0][1].shape, generator=gq, device=dev)
                  for i in range(len(made) * 4)]
            kx = cfg_k(c)
            n_steps = max(20, min(args.steps, 200))
            ms_x = time_steps(ctx, ls, qx, kx, max(args.warmup, 2 * len(ls)), n_steps, dist, dev)
            us = ms_x * 1e3 / n_steps
            byts = cfg_bytes(c)
            extra[name] = {"what": c["what"], "us_per_layer": us, "algorithmic_bytes": byts,
                           "gbs": byts / (us * 1e-6) / 1e9, "frac": byts / (us * 1e-6) / 1e9 / peak,
                           "k": kx, "build_s_per_layer": float(np.median([m_[2] for m_ in made])),
                           "plan": ctx.decode_plan(ls[0], c["g"], kx), "steps": n_steps,
                           "layers_rotated": len(ls)}
            del made, ls, qx
            torch.cuda.empty_cache()

    # ---- configs[2] whole model: Llama-3-8B shape, 32 layers x 8 kv heads x g4
    # x 128K, prefill PQ build + decode of every layer per token on one B200
    # (32 GB of fp32 K/V).  The headline layers except gaussian layer 0 (the
    # CPU-baseline sample) are released first.
    model_info = None
    if not args.no_extra:
        for kind in ("gaussian", "powerlaw"):
            ls, qs_, _ = heads[kind]
            keep = 1 if kind == "gaussian" else 0
            heads[kind] = (ls[:keep], qs_[:keep], [])
        layers = bms = hq = None
        torch.cuda.empty_cache()
        c3 = CONFIGS["cfg3_layer"]
        n_model = 32
        u3, s3 = c3["units"], c3["s"]
        sm3 = s3 - N_INIT - N_LOCAL
        # prefill: every layer's K/V, then ONE batched PQ build over all
        # 32 x 8 (layer, kv_head) problems (a batch of 256 heads builds ~2x
        # faster per head than per-layer batches of 8: tools/prof_build.py)
        kvs, mq = [], []
        for li in range(n_model):
            kk, vv, bq = ctx.gen_workload(s3, DH, h_kv=u3, g=c3["g"], kind="gaussian", n_components=8, spread=0.5,
                                          seed=9000 + li)
            kvs.append((kk, vv))
            mq.append(bq)
        mids = torch.empty((n_model * u3, sm3, DH), dtype=torch.float32, device=dev)
        for li, (kk, _) in enumerate(kvs):
            mids[li * u3:(li + 1) * u3] = kk[:, N_INIT:N_INIT + sm3]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cen_all, codes_all = ctx.pq_build(mids, c3["m"], c3["b"], T_ITERS, [9000 + h for h in range(n_model * u3)])
        tabs_all = ctx.tuple_tables(codes_all, c3["b"])
        torch.cuda.synchronize()
        build_total = time.perf_counter() - t0
        del mids
        mlayers = []
        for li, (kk, vv) in enumerate(kvs):
            sl = slice(li * u3, (li + 1) * u3)
            mlayers.append(pq.DecodeLayer(keys=kk, values=vv, centroids=cen_all[sl], codes=codes_all[sl], total=s3,
                                          n_init=N_INIT, n_local=N_LOCAL, b=c3["b"],
                                          tables=(tabs_all[0][sl], tabs_all[1][sl])))
        del kvs
        k3 = cfg_k(c3)
        n_tok = max(4, min(args.steps // 8, 32))
        tq = [[mq[li] + sigma * torch.randn(mq[0].shape, generator=gq, device=dev) for li in range(n_model)]
              for _ in range(2)]
        for li in range(n_model):  # warm every layer
            ctx.decode(mlayers[li], tq[0][li], k3)
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for t in range(n_tok):
            for li in range(n_model):
                ctx.decode(mlayers[li], tq[t & 1][li], k3)
        m1.record(stream)
        torch.cuda.synchronize()
        ms_tok = m0.elapsed_time(m1) / n_tok
        us_l = ms_tok * 1e3 / n_model
        model_info = {"what": "configs[2]: 32 layers x 8 kv heads x g4 x 128K (Llama-3-8B shape), m2b6, top 1/5 "
                              "+ 4 + 64; every token decodes all 32 layers (one launch each)",
                      "prefill_build_s": build_total, "build_context_tokens_per_s": c3["s"] / build_total,
                      "build_note": "one batched pq_build over all 256 (layer, kv_head) problems + pair tables",
                      "build_key_vectors_per_s": n_model * u3 * sm3 / build_total,
                      "decode_ms_per_token": ms_tok, "us_per_layer": us_l,
                      "frac": cfg_bytes(c3) / (us_l * 1e-6) / 1e9 / peak, "tokens": n_tok,
                      "kv_gb": n_model * c3["units"] * c3["s"] * DH * 4 * 2 / 1e9}
        del mlayers, mq, tq
        torch.cuda.empty_cache()

    # ---- run_recall on the device (experiments.cpp:74-139) ----
    recall_info = None
    if not args.no_extra:
        from paper_2407_12820_b200 import recall as rc

        rs, rh = 32768, 8
        wl = {sd: ctx.gen_workload(rs, DH, h_kv=rh, g=1, kind="powerlaw", seed=7000 + sd) for sd in (1, 2)}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rrows = rc.run_recall(ctx, wl, [2], [6], [round(rs / 20), round(rs / 10), round(rs / 5)], max_iter=15)
        torch.cuda.synchronize()
        recall_info = {"what": f"run_recall on the GPU: {rh} heads x {rs} tokens powerlaw, m2b6, T=15, "
                               "k = s/20, s/10, s/5, 2 seeds (fp64 attention path, reference arithmetic)",
                       "seconds": time.perf_counter() - t0,
                       "rows": [[r.k, r.seed, round(r.recall, 4), round(r.random_recall, 4), round(r.output_error, 4)]
                                for r in rrows]}
        del wl

    # ---- numbers ----
    # The step is ONE launch of attend_kernel (pair select + classification +
    # gather + softmax + combine fused), so the dominant
    # kernel's average launch duration is the device-timed step itself.
    layer_bytes = algorithmic_bytes_per_layer()
    achieved = layer_bytes / (ms_per_step * 1e-3) / 1e9
    attend_bytes = attend_bytes_per_launch()
    attend_only_gbs = attend_bytes / (attend_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("attend_kernel_fused")
        except Exception:
            traffic = None
    build_layer_s = float(np.median(build_s))
    line = {
        "metric": METRIC, "value": us_per_layer, "unit": "us/layer", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (K/V, attention), f64 (ADC table), u16 codes", "data": "synthetic",
        "config": workload_config(world),
        "distributions": {"us_per_layer": {kd: timed[kd] * 1e3 / (args.steps * world) for kd in timed},
                          "slower": worst, "steps_each": args.steps, "layers_rotated": N_LAYERS,
                          "warmup": f"max(W, 2 x {N_LAYERS} rotating layers) untimed steps before each timed region"},
        "plan": plan,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "tuple_select_kernel + attend_kernel<1,0> (pair-select launch chained by programmatic "
                               "launch to the attention launch; timed as the whole step, 2 launches/layer)",
                     "kernel_ms": ms_per_step, "algorithmic_bytes": layer_bytes,
                     "bytes_basis": "SURVEY 8(d): h_kv*(s_mid*m*b/8 + C*d_h*4 + T_att*d_h*4*2 + 2*g*d_h*4)"},
        "attend_only": {"kernel": "attend_kernel bitmap mode (gather + softmax + combine, selection precomputed)",
                        "ms": attend_ms, "gbs": attend_only_gbs, "frac": attend_only_gbs / peak,
                        "bytes": attend_bytes, "select_ms": select_ms},
        "e2e": {"value": e2e_us, "unit": "us/layer", "h2d_bytes_per_step": H * G * DH * 4,
                "d2h_bytes_per_step": H * G * DH * 4, "api": "pqkv_decode_host (C ABI, pinned host buffers)"},
        "gpu_launches": launches_per_step * args.steps * 2,
        "configs": extra,
        "recall_gpu": recall_info,
        "model_cfg3": model_info,
        "head_sharded": {"config": "cfg4: each layer's 32 heads split over the ranks; pqkv_decode_sharded = the "
                                   "rank's decodes + one NCCL all-gather of the per-head outputs (C ABI, collective "
                                   "stream), 8 rotating layers",
                         "us_per_layer": hs[1], "us_per_layer_batched8": hs[N_LAYERS], "heads_per_rank": len(hr),
                         "error": hs.get("error"),
                         "note": "device-timed, max over ranks; batched8 = one all-gather per 8 layers"},
        "build": {"layer_s": build_layer_s, "key_vectors_per_s": H * S_MID / build_layer_s,
                  "context_tokens_per_s": S_MID / build_layer_s, "layers": N_LAYERS,
                  "fp64_rechecked_points": rech_tot[0], "points": rech_tot[1],
                  # W = (T+2) s C d_h 3 fp64 ops per head for the reference's
                  # exact algorithm; the certified fp32 filter skips most of them, so the
                  # reference-equivalent rate exceeds the FP64 pipe (18.11 T op/s measured,
                  # profiles/r01_fp64_probe.txt)
                  "ref_equiv_fp64_ops_per_s": (T_ITERS + 2) * S_MID * (1 << B) * DH * 3 * H / build_layer_s,
                  "fp64_peak_ops_per_s": 18.11e12,
                  "key_bytes_per_s": H * S_MID * DH * 4 / build_layer_s},
    }
    clk.stop()
    line["clocks"] = clk.summary()
    if rank == 0 and not args.no_extra:
        # the reference's run_e2e decode loop on the C++ drop-in API
        # (include/pqkv/*.hpp: evict_local_append, pq_score_gqa, approx_topk,
        # fetch_topk, selective_attention per head, value semantics, fp64
        # attention), timed per layer-step by tools/cxx_e2e.cpp
        import subprocess

        exe = os.path.join(ROOT, "paper_2407_12820_b200", "lib", "pqkv_cxx_e2e")
        try:
            r = subprocess.run([exe, "8", "32768", "1", "5", "3"], capture_output=True, text=True, timeout=300)
            line["e2e_cxx"] = json.loads(r.stdout.strip().splitlines()[-1])
            line["e2e_cxx"]["what"] = ("run_e2e's per-head decode calls through the C++ drop-in API (host value "
                                       "types, device mirrors), 8 heads x 32K, m2b6, k = s/5, us per layer-step")
        except Exception as e:  # reported, not fatal
            line["e2e_cxx"] = {"error": repr(e)[:200]}
        # the same decode loop built entirely from the reference's sources
        # (oracle/Makefile cxx_e2e_ref), timed on the host cores: the CPU arm
        ref_exe = os.path.join(ROOT, "oracle", "_ref", "dropin", "cxx_e2e_ref")
        if not args.no_cpu_baseline and "error" not in line["e2e_cxx"] and os.path.exists(ref_exe):
            try:
                r = subprocess.run([ref_exe, "4", "32768", "1", "5", "2"], capture_output=True, text=True,
                                   timeout=600)
                ref = json.loads(r.stdout.strip().splitlines()[-1])
                line["e2e_cxx"]["cpu_baseline"] = {
                    "kind": "reference", "cores": 1, "sample": "4 heads x 32K, 2 decode steps (per-head-step "
                    "comparable)", "us_per_head_step": ref["us_per_head_step"], "per_call_us": ref["per_call_us"]}
            except Exception as e:
                line["e2e_cxx"]["cpu_baseline"] = {"error": repr(e)[:200]}
    if rank == 0 and not args.no_cpu_baseline:
        gl, gqs, _ = heads["gaussian"]
        words = torch.zeros((H, (S_MID + 31) // 32), dtype=torch.int32, device=dev)
        ctx.set_selection_dump(words)
        try:
            gpu_out = ctx.decode(gl[0], gqs[0], K_SEL)  # layer 0, base queries
        finally:
            ctx.set_selection_dump(None)
        dec, bld = cpu_baseline_leg(gl[0], gqs[0], gpu_out, words)
        line["cpu_baseline"] = dec
        line["cpu_baseline_build"] = bld
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
