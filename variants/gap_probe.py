"""GPU idle gaps inside one C2 step (torch.profiler / CUPTI): which host code runs while
the GPU waits.  python variants/gap_probe.py > gpurun_out/gaps.txt"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import bench
from paper_1711_07227_b200 import device

cfg = bench.CONFIGS["c2"]
E, x1, x2 = bench.make_data(cfg)
Ed = device.to_device(E, torch.float32)
dx1 = device.DeviceCSR.upload(x1, "x1")
dx2 = device.DeviceCSR.upload(x2, "x2")


def step():
    prep = device.PreparedEmbeddings(Ed)
    return device.symmetric(dx1, dx2, prep, 10)


for _ in range(2):
    step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 200:  # us
        gaps.append((g, a.name[:50], b.name[:50], a.time_range.end))
tot = sum(e.time_range.elapsed_us() for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"kernels {len(ev)} busy {tot/1e3:.1f} ms span {span/1e3:.1f} ms")
for g, a, b, t in sorted(gaps, reverse=True)[:20]:
    # host ops overlapping the gap
    cpu = [c for c in prof.events() if c.device_type.name == "CPU" and c.time_range.start <= t + g and c.time_range.end >= t
           and c.time_range.elapsed_us() > 0.5 * g]
    names = sorted({c.name[:60] for c in cpu})[:8]
    print(f"gap {g/1e3:7.2f} ms after {a!r} before {b!r}; host: {names}")
    inside = [c for c in prof.events() if c.device_type.name == "CPU" and t <= c.time_range.start <= t + g]
    inside.sort(key=lambda c: -c.time_range.elapsed_us())
    for c in inside[:12]:
        print(f"    {c.time_range.elapsed_us()/1e3:6.2f} ms  {c.name[:70]}  {' <- '.join(str(x) for x in (c.stack or [])[:4])[:200]}")
