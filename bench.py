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


def algorithmic_bytes_per_layer():
    """B = h_kv [s_mid m b/8 + C d_h 4 + T_att d_h 4 2 + 2 g d_h 4]."""
    t_att = N_INIT + K_SEL + N_LOCAL
    return H * (S_MID * M * B / 8 + (1 << B) * DH * 4 + t_att * DH * 4 * 2 + 2 * G * DH * 4)


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
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()

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
                    elif self.t0 - 0.005 <= v[0] <= self.t1 + 0.005:
                        rows.append(v)
            os.unlink(self.out.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": max_mhz, "reasons": ["unsampled"], "samples": 0}
        bits = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
        sm = sorted(r[1] for r in rows)
        reasons = sorted({name for r in rows for bit, name in bits.items() if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max_mhz, "reasons": reasons, "samples": len(rows)}


def make_layer_inputs(ctx, seed):
    """Gaussian-mixture keys (workload.cpp:39-51 distribution: 8 shared means,
    spread 0.5), N(0,1) values and base queries, generated in HBM by the
    library's counter-based generator (pqkv_gen_workload)."""
    return ctx.gen_workload(S, DH, h_kv=H, g=G, kind="gaussian", n_components=8, spread=0.5, seed=seed)


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU decode (oracle/_ref) on all host
    cores, bounded sample of the same workload, extrapolated to us/layer."""
    import numpy as np

    import oracle

    if rank != 0:
        return
    line = {"impl": "reference", "metric": METRIC, "unit": "us/layer", "higher_is_better": False,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "scaling": "weak",
            "dtype": "f32 storage, f64 arithmetic", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": 1, "seq_len": S}}
    if not oracle.has_ref():
        line["unavailable"] = "oracle/_ref/libpqkv_ref.so was not built (needs /root/reference at build time)"
        print(json.dumps(line), flush=True)
        return
    ref = oracle.ref()
    cores = os.cpu_count() or 1
    P = min(H, max(1, cores))  # one head per host thread
    rng = np.random.default_rng(17)
    keys = np.empty((P, S, DH), np.float32)
    vals = rng.standard_normal((P, S, DH), dtype=np.float32)
    for p in range(P):
        means = rng.standard_normal((8, DH)).astype(np.float32)
        keys[p] = means[rng.integers(0, 8, S)] + 0.5 * rng.standard_normal((S, DH), dtype=np.float32)
    queries = rng.standard_normal((P, G, DH)).astype(np.float32)
    # the reference builds its own index (pq_construct on all host cores, untimed setup)
    mids = np.ascontiguousarray(keys[:, N_INIT:N_INIT + S_MID])
    _, cen, codes = ref.bench_build(mids, M, B, T_ITERS, np.arange(P, dtype=np.uint64) + 11, 0)
    del mids
    n_total = args.warmup + args.steps
    sigma = 0.25 / math.sqrt(DH)
    queries = (queries[None] + sigma * rng.standard_normal((n_total, P, G, DH))).astype(np.float32)
    # HeadStates are built once (kv_store offload_prefill); every step is one
    # decode of the P sampled heads (pq_score_gqa + approx_topk +
    # selective_attention), one head per host thread
    secs, _ = ref.bench_decode_steps(keys, vals, queries, cen, codes, N_INIT, N_LOCAL, K_SEL, 0)
    timed = secs[args.warmup:]
    per_layer_us = float(np.mean(timed)) * 1e6 * (H / P)
    line.update({"value": per_layer_us, "ms_per_step": per_layer_us / 1e3,
                 "cpu_baseline": {"value": per_layer_us, "unit": "us/layer", "cores": min(cores, P),
                                  "kind": "reference",
                                  "sample": f"{P} of {H} heads per step (x{H / P:g} to a layer), "
                                            "pq_score_gqa+approx_topk+selective_attention, index built by "
                                            "the reference's pq_construct"},
                 "e2e": {"value": per_layer_us, "unit": "us/layer", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(layer0, cen, codes, torch, gpu_out=None):
    """The reference (oracle/_ref) on this box's host cores for a bounded sample
    (8 heads of layer 0, same GPU-built index -- bit-identical to the
    reference's), extrapolated x4 to the 32-head layer; plus a 1-head 32K-token
    pq_construct sample for the build."""
    import numpy as np

    import oracle

    if not oracle.has_ref():
        return None, None
    ref = oracle.ref()
    P = min(H, max(1, os.cpu_count() or 1))  # one head per host thread
    keys, vals, base_q = layer0
    k = keys[:P].cpu().numpy()
    v = vals[:P].cpu().numpy()
    q = base_q[:P].cpu().numpy()
    c = cen[:P].cpu().numpy()
    cd = codes[:P].cpu().numpy().view(np.uint16)
    cores = min(os.cpu_count() or 1, P)
    runs = [ref.bench_decode(k, v, q, c, cd, N_INIT, N_LOCAL, K_SEL, cores) for _ in range(3)]
    ts = [r[0] for r in runs]
    dec = {"value": float(np.median(ts)) * 1e6 * (H / P), "unit": "us/layer", "cores": cores,
           "kind": "reference", "sample": f"{P} of {H} heads of one 128K layer, x{H / P:g} to a layer, median of 3"}
    # parity on the benchmark's own inputs: the fused GPU decode of these heads
    # (same base queries, same index) against the reference library's outputs
    if gpu_out is not None:
        want = runs[0][1]
        got = gpu_out[:P].cpu().numpy()
        rel = float(np.abs(got - want).max() / max(1.0, float(np.abs(want).max())))
        dec["parity"] = {"heads": P, "max_rel_err": rel, "tolerance": 1e-3, "ok": rel < 1e-3}
    sb = 32768
    secs, _, _ = ref.bench_build(np.ascontiguousarray(k[:1, N_INIT:N_INIT + sb]), M, B, T_ITERS,
                                 np.array([5], np.uint64), 1)
    bld = {"value": sb / secs, "unit": "key vectors/s", "cores": 1, "kind": "reference",
           "sample": f"pq_construct m2b6 T={T_ITERS} on 1 head x {sb} tokens"}
    return dec, bld


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    ctx = pq.Context(local)

    # ---- per-rank layers: inputs + GPU PQ build (timed separately) ----
    layers, build_s = [], []
    keep0 = None
    for li in range(N_LAYERS):
        keys, vals, base_q = make_layer_inputs(ctx, 1000 * rank + li)
        mids = keys[:, N_INIT:N_INIT + S_MID]  # middle rows, strided view of the cache
        mids = mids.contiguous()
        seeds = [7 + 100 * rank + 10 * li + h for h in range(H)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cen, codes = ctx.pq_build(mids, M, B, T_ITERS, seeds)
        tables = ctx.tuple_tables(codes, B)  # code-pair histograms (part of the build)
        torch.cuda.synchronize()
        build_s.append(time.perf_counter() - t0)
        rech, tot = ctx.last_build_stats()
        del mids
        layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S,
                               n_init=N_INIT, n_local=N_LOCAL, b=B, tables=tables)
        layers.append((layer, base_q))
        if li == 0:
            keep0 = ((keys, vals, base_q), cen, codes)
    # per-step query drift (experiments.cpp:212-216)
    gq = torch.Generator(device=dev)
    gq.manual_seed(99 + rank)
    n_total = args.warmup + args.steps
    sigma = 0.25 / math.sqrt(DH)
    queries = [layers[i % N_LAYERS][1] + sigma * torch.randn((H, G, DH), generator=gq, device=dev)
               for i in range(n_total)]
    out = torch.empty((H, G, DH), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step(i):
        layer = layers[i % N_LAYERS][0]
        return ctx.decode(layer, queries[i], K_SEL)

    # ---- device-resident timing ----
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local).start()
    with clk:
        ev0.record(stream)
        for i in range(args.warmup, n_total):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    layers_done = args.steps * world
    us_per_layer = ms * 1e3 / layers_done

    # ---- dominant kernel (attention gather + combine) timed alone ----
    bms = []
    for i in range(N_LAYERS):
        bm, _ = ctx.pq_search(queries[i], layers[i][0].centroids, layers[i][0].codes, B, K_SEL, s=S_MID,
                              bitmap=True, ordered=False, tables=layers[i][0].tables)
        bms.append(bm)
    sel_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
    reps = max(args.steps, 8)
    for i in range(3):
        ctx.decode_attend(layers[i % N_LAYERS][0], queries[i], bms[i % N_LAYERS], out)
    torch.cuda.synchronize()
    sel_ev[0][0].record(stream)
    for i in range(reps):
        ctx.decode_attend(layers[i % N_LAYERS][0], queries[i % N_LAYERS], bms[i % N_LAYERS], out)
    sel_ev[0][1].record(stream)
    sel_ev[1][0].record(stream)
    for i in range(reps):
        ctx.pq_search(queries[i % N_LAYERS], layers[i % N_LAYERS][0].centroids, layers[i % N_LAYERS][0].codes,
                      B, K_SEL, s=S_MID, bitmap=True, ordered=False, tables=layers[i % N_LAYERS][0].tables)
    sel_ev[1][1].record(stream)
    torch.cuda.synchronize()
    attend_ms = sel_ev[0][0].elapsed_time(sel_ev[0][1]) / reps
    select_ms = sel_ev[1][0].elapsed_time(sel_ev[1][1]) / reps

    # ---- end to end through the C ABI with HOST buffers ----
    hq = [q.cpu().pin_memory() for q in queries[:N_LAYERS]]
    ho = torch.empty((H, G, DH), dtype=torch.float32).pin_memory()
    for i in range(3):
        ctx.decode_host(layers[i % N_LAYERS][0], hq[i % N_LAYERS], ho, K_SEL)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        ctx.decode_host(layers[i % N_LAYERS][0], hq[i % N_LAYERS], ho, K_SEL)
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_us = e2e_s * 1e6 / (args.steps * world)

    # ---- cfg4: one layer's heads sharded over the ranks + NCCL all-gather ----
    # (BASELINE configs[3]; the path itself has no exchange, the gathered
    # outputs are what the next layer's projection needs)
    from paper_2407_12820_b200 import shard

    hr = shard.partition(H, world, rank)
    l0 = layers[0][0]
    th, ch = l0.tables
    sub = pq.DecodeLayer(keys=l0.keys[hr.start:hr.stop], values=l0.values[hr.start:hr.stop],
                         centroids=l0.centroids[hr.start:hr.stop], codes=l0.codes[hr.start:hr.stop], total=S,
                         n_init=N_INIT, n_local=N_LOCAL, b=B, tables=(th[hr.start:hr.stop], ch[hr.start:hr.stop]))
    qsub = [queries[i][hr.start:hr.stop].contiguous() for i in range(N_LAYERS)]
    for i in range(3):
        shard.gather_heads(ctx.decode(sub, qsub[i % N_LAYERS], K_SEL), H)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    hs0, hs1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hs_steps = max(20, min(args.steps, 200))
    hs0.record(stream)
    for i in range(hs_steps):
        full = shard.gather_heads(ctx.decode(sub, qsub[i % N_LAYERS], K_SEL), H)
    hs1.record(stream)
    torch.cuda.synchronize()
    hs_us = shard.max_over_ranks(hs0.elapsed_time(hs1) * 1e3 / hs_steps, dev)
    assert full.shape[0] == H

    # ---- numbers ----
    # The step is ONE launch of attend_kernel (pair select + classification +
    # gather + softmax + combine fused), so the dominant
    # kernel's average launch duration is the device-timed step itself.
    peak, peak_kind = peaks()
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
    launches_per_step = layers[0][0].launches(G)
    line = {
        "metric": METRIC, "value": us_per_layer, "unit": "us/layer", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (K/V, attention), f64 (ADC table), u16 codes", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": 1, "seq_len": S, "heads": H, "head_dim": DH,
                   "m": M, "b": B, "k": K_SEL, "n_init": N_INIT, "n_local": N_LOCAL,
                   "layers_rotated": N_LAYERS, "parallelism": f"dp{world} (independent layers per GPU)",
                   "l2": "inputs larger than L2: 8 rotating layers x 4.3 GB K/V (+26 MB codes and pair tables each: 206 MB > L2), 0.86 GB gathered per step"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "attend_kernel<1> pair mode (the whole fused decode step, 1 launch/layer)",
                     "kernel_ms": ms_per_step, "algorithmic_bytes": layer_bytes,
                     "bytes_basis": "SURVEY 8(d): h_kv*(s_mid*m*b/8 + C*d_h*4 + T_att*d_h*4*2 + 2*g*d_h*4)"},
        "attend_only": {"kernel": "attend_kernel bitmap mode (gather + softmax + combine, selection precomputed)",
                        "ms": attend_ms, "gbs": attend_only_gbs, "frac": attend_only_gbs / peak,
                        "bytes": attend_bytes, "select_ms": select_ms},
        "e2e": {"value": e2e_us, "unit": "us/layer", "h2d_bytes_per_step": H * G * DH * 4,
                "d2h_bytes_per_step": H * G * DH * 4},
        "gpu_launches": launches_per_step * args.steps,
        "head_sharded": {"config": "cfg4: one layer's 32 heads split over the ranks, per-head outputs "
                                   "all-gathered (NCCL all_gather_into_tensor) every step",
                         "us_per_layer": hs_us, "heads_per_rank": len(hr), "steps": hs_steps,
                         "note": "device-timed, max over ranks; the same K/V layer every step (L2-warm rows "
                                 "possible at high rank counts)"},
        "build": {"layer_s": build_layer_s, "key_vectors_per_s": H * S_MID / build_layer_s,
                  "context_tokens_per_s": S_MID / build_layer_s, "layers": N_LAYERS,
                  "fp64_rechecked_points": rech, "points": tot,
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
    if rank == 0 and not args.no_cpu_baseline:
        gpu_out = ctx.decode(layers[0][0], layers[0][1], K_SEL)  # layer 0, base queries
        dec, bld = cpu_baseline_leg(keep0[0], keep0[1], keep0[2], torch, gpu_out)
        line["cpu_baseline"] = dec
        line["cpu_baseline_build"] = bld
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
