"""Find the largest idle gaps of the GPU during time steps and what the host
was doing meanwhile (torch.profiler / CUPTI timeline)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st = wl.stepper
    for _ in range(3):
        st.step_device()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(12):
            st.step_device()
        torch.cuda.synchronize()
    evs = prof.events()
    gpu = sorted([e for e in evs if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    cpu = [e for e in evs if e.device_type.name == "CPU"]
    gaps = []
    for a, b in zip(gpu, gpu[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 0:
            gaps.append((g, a.time_range.end, b.time_range.start, a.name[:40], b.name[:40]))
    gaps.sort(reverse=True)
    tot = sum(g[0] for g in gaps)
    span = gpu[-1].time_range.end - gpu[0].time_range.start
    print(f"GPU span {span / 1e3:.1f} ms, idle gaps total {tot / 1e3:.1f} ms")
    for g, t0, t1, an, bn in gaps[:8]:
        over = [e for e in cpu if e.time_range.start < t1 and e.time_range.end > t0
                and (e.time_range.end - e.time_range.start) > 0.5 * g]
        over.sort(key=lambda e: e.time_range.end - e.time_range.start)
        host = ", ".join(f"{e.name[:50]} ({(e.time_range.end - e.time_range.start) / 1e3:.1f} ms)"
                         for e in over[:4])
        print(f"gap {g / 1e3:8.2f} ms after {an} before {bn}; host: {host}")


if __name__ == "__main__":
    main()
