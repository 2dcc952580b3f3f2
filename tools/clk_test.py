import threading, time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
t0=time.time(); n=0; err=None
while time.time()-t0 < 0.5:
    try:
        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h); n+=1
    except Exception as e:
        err=repr(e); break
print("samples in 0.5s:", n, "err:", err, "mhz", mhz)
