"""Diagnostic: event-timed phases of one symmetric top-k step (C2 shape)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import ctypes as C
import numpy as np, torch
from paper_1711_07227_b200 import _lib, device, synthetic as S
V = int(os.environ.get("V", 100000)); N1 = int(os.environ.get("N1", 1000000)); N2 = 1000
E = S.embeddings(V, 300, seed=0); x1 = S.histograms(N1, V, 50, seed=1); x2 = S.histograms(N2, V, 50, seed=2)
Ed = device.to_device(E, torch.float32); dx1 = device.DeviceCSR.upload(x1); dx2 = device.DeviceCSR.upload(x2)
def run(mark):
    mark("start")
    prep = device.PreparedEmbeddings(Ed); mark("prep")
    res1 = device.Restricted.build(dx1, prep); mark("restrict1")
    d1 = device.one_direction(res1, prep, dx2, layout="panels"); mark("forward")
    del res1
    out = device.symmetric(dx1, dx2, prep, 10, d1=d1); mark("reverse+merge")
    return out
for it in range(3):
    evs = []; walls = []
    def mark(name):
        e = torch.cuda.Event(enable_timing=True); e.record(); evs.append((name, e)); walls.append(time.perf_counter())
    torch.cuda.synchronize()
    run(mark)
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    print({evs[i][0]: round(evs[i-1][1].elapsed_time(evs[i][1]), 1) for i in range(1, len(evs))},
          "host", {evs[i][0]: round((walls[i]-walls[i-1])*1e3, 1) for i in range(1, len(evs))}, "total", round(evs[0][1].elapsed_time(evs[-1][1]), 1))
