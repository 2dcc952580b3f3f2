"""One-line summary of a bench.py JSON line: headline, distributions, the
config lines and the side metrics.  Usage: python tools/bench_summary.py FILE"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("headline %.1f us (frac %.3f) dists %s" % (d["value"], d["roofline"]["frac"],
                                                 {k: round(v, 1) for k, v in d["distributions"]["us_per_layer"].items()}))
for k, v in (d.get("configs") or {}).items():
    print("  %-14s %6.1f us  frac %.3f" % (k, v.get("us_per_layer", float("nan")), v.get("frac", float("nan"))))
for k in ("attend_only", "e2e", "head_sharded", "model_cfg3", "build", "e2e_cxx", "clocks"):
    if k in d and d[k]:
        v = d[k]
        if k == "attend_only":
            print("  attend_only %.1f us frac %.3f" % (v["ms"] * 1e3, v["frac"]))
        elif k == "e2e":
            print("  e2e %.1f us" % v["value"])
        elif k == "head_sharded":
            print("  head_sharded %s / batched8 %s" % (v.get("us_per_layer"), v.get("us_per_layer_batched8")))
        elif k == "model_cfg3":
            print("  model_cfg3 %.1f us/layer, build %.2f s" % (v["us_per_layer"], v["prefill_build_s"]))
        elif k == "build":
            print("  build %.1f ms/layer" % (v["layer_s"] * 1e3))
        elif k == "e2e_cxx":
            print("  e2e_cxx %s us/head-step, cpu ref %s" % (v.get("us_per_head_step"),
                                                            (v.get("cpu_baseline") or {}).get("us_per_head_step")))
        elif k == "clocks":
            print("  clocks", v)
