import time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fn in [("clock_sm", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                 ("event_reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)),
                 ("throttle_reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)),
                 ("pstate", lambda: pynvml.nvmlDeviceGetPerformanceState(h)),
                 ("power", lambda: pynvml.nvmlDeviceGetPowerUsage(h))]:
    ts = []
    for _ in range(20):
        t = time.perf_counter(); fn(); ts.append((time.perf_counter() - t) * 1e3)
    ts.sort()
    print(f"{name:18s} min {ts[0]:.3f} ms  median {ts[10]:.3f} ms  max {ts[-1]:.3f} ms")
