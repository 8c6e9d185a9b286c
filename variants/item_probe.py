import sys, time, traceback
sys.path.insert(0, '.')
import torch, numpy as np
import bench
from paper_1711_07227_b200 import device
cfg = bench.CONFIGS["c2"]
E, x1, x2 = bench.make_data(cfg)
Ed = device.to_device(E, torch.float32)
dx1 = device.DeviceCSR.upload(x1, "x1"); dx2 = device.DeviceCSR.upload(x2, "x2")
def step():
    prep = device.PreparedEmbeddings(Ed)
    return device.symmetric(dx1, dx2, prep, 10)
step(); torch.cuda.synchronize()
log = []
orig_item = torch.Tensor.item
def item(self):
    v = orig_item(self)
    log.append((time.perf_counter(), 'item', ''.join(traceback.format_stack(limit=4)[:-1])[-300:]))
    return v
orig_td = device.to_device
def td(a, dtype, non_blocking=True):
    log.append((time.perf_counter(), 'to_device', ''.join(traceback.format_stack(limit=4)[:-1])[-300:]))
    return orig_td(a, dtype, non_blocking)
torch.Tensor.item = item
device.to_device = td
step(); torch.cuda.synchronize()
t0 = log[0][0]
for i, (t, k, s) in enumerate(log):
    dt = (t - log[i-1][0]) * 1e3 if i else 0
    print(f"{(t-t0)*1e3:8.2f} (+{dt:6.2f}) {k}: {s.strip().splitlines()[-2].strip() if s.strip() else ''} | {s.strip().splitlines()[0].strip() if s.strip() else ''}")
