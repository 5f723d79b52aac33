"""CUPTI trace of time steps (torch.profiler; no nsys in the image): per
kernel totals, GPU busy vs idle time, and the largest idle gaps with the
kernels around them.  `python profiles/step_trace.py [config] [steps]`."""
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    wl = configs.build(k)
    st = wl.stepper
    for _ in range(3):
        st.step_device()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            st.step_device()
        torch.cuda.synchronize()
    out = Path("gpurun_out")
    out.mkdir(exist_ok=True)
    fn = out / f"trace_c{k}.json"
    prof.export_chrome_trace(str(fn))
    ev = json.loads(fn.read_text())["traceEvents"]
    kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
                  key=lambda e: e["ts"])
    if not kern:
        print("no kernel events")
        return
    t0, t1 = kern[0]["ts"], max(e["ts"] + e["dur"] for e in kern)
    busy = 0.0
    tot = defaultdict(lambda: [0, 0.0])
    gaps = []
    end = t0
    for i, e in enumerate(kern):
        if e["ts"] > end:
            gaps.append((e["ts"] - end, kern[i - 1]["name"][:60] if i else "", e["name"][:60]))
        s, f = max(e["ts"], end), e["ts"] + e["dur"]
        if f > s:
            busy += f - s
        end = max(end, f)
        tot[e["name"][:70]][0] += 1
        tot[e["name"][:70]][1] += e["dur"]
    span = t1 - t0
    print(f"span {span / steps / 1e3:.2f} ms/step, busy {busy / steps / 1e3:.2f} ms/step, "
          f"idle {(span - busy) / steps / 1e3:.2f} ms/step, {len(kern) / steps:.0f} events/step")
    for name, (n, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{d / steps / 1e3:8.3f} ms/step  {n / steps:7.1f}/step  {d / n:8.2f} us  {name}")
    gaps.sort(key=lambda g: -g[0])
    big = sum(g[0] for g in gaps if g[0] > 5)
    print(f"gaps > 5 us: {sum(1 for g in gaps if g[0] > 5) / steps:.0f}/step, "
          f"{big / steps / 1e3:.2f} ms/step")
    hist = defaultdict(lambda: [0, 0.0])
    for g, a, b in gaps:
        if g > 5:
            hist[(a[:40], b[:40])][0] += 1
            hist[(a[:40], b[:40])][1] += g
    for (a, b), (n, d) in sorted(hist.items(), key=lambda x: -x[1][1])[:15]:
        print(f"{d / steps / 1e3:8.3f} ms/step {n / steps:6.1f}/step  {a} -> {b}")


if __name__ == "__main__":
    main()
