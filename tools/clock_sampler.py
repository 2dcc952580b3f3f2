"""Out-of-process GPU clock sampler for bench.py (no GIL contention with the
launch loop).  Prints one JSON line per sample: [t, sm_mhz, reasons_mask].
usage: python tools/clock_sampler.py DEVICE INTERVAL_S"""
import json
import sys
import time

import pynvml

dev = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(dev)
print(json.dumps({"max_mhz": pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)}), flush=True)
get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
while True:
    try:
        print(json.dumps([time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                          int(get_reasons(h))]), flush=True)
    except Exception as e:  # keep sampling
        print(json.dumps({"err": repr(e)}), flush=True)
    time.sleep(dt)
