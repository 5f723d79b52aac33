"""Break the end-to-end step (public TimeStepper.step with host buffers) into
its parts: H2D of the state, the device step, the D2H of u_next."""

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    for _ in range(3):
        st.step_device(prob)
    torch.cuda.synchronize()
    u_pin = torch.from_numpy(st.u.copy()).pin_memory()
    tt = {"set": 0.0, "dev": 0.0, "get": 0.0, "dev_sync": 0.0}
    n = 5
    for _ in range(n):
        t0 = time.perf_counter()
        st.u = u_pin
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st.step_device(prob)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        u = st.u.copy()
        u_pin.copy_(torch.from_numpy(u))
        t4 = time.perf_counter()
        tt["set"] += t1 - t0
        tt["dev"] += t2 - t1
        tt["dev_sync"] += t3 - t2
        tt["get"] += t4 - t3
    print({k: round(v / n * 1e3, 2) for k, v in tt.items()}, "ms per step")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        st.step_device(prob)
    e1.record()
    torch.cuda.synchronize()
    print("device loop: events %.2f ms/step, wall %.2f ms/step" % (
        e0.elapsed_time(e1) / n, (time.perf_counter() - w0) / n * 1e3))


if __name__ == "__main__":
    main()
