"""Per-role cycle counters of the instrumented Phase-1 build (variants/build_stats.sh)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("LCRW_LIB", "variants/stats/liblcrwmd.so")
import numpy as np, torch
from paper_1711_07227_b200 import _lib, device, synthetic as S
lib = _lib.load()
V = 50000
E = S.embeddings(V, 300, seed=0)
x1 = S.histograms(100000, V, 50, seed=1)
x2 = S.histograms(256, V, 50, seed=2)
prep = device.PreparedEmbeddings(E)
dx1, dx2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
out = (C.c_ulonglong * 8)()
for it in range(3):
    torch.cuda.synchronize()
    lib.lcrw_p1_stats(out, 1)
    device.symmetric(dx1, dx2, prep, 10)
    torch.cuda.synchronize()
    lib.lcrw_p1_stats(out, 1)
v = list(out)
et = max(v[3], 1); mt = max(v[6], 1)
print(f"epilogue per tile-warp: wait {v[0]/et:.0f}  work {v[1]/et:.0f} cycles (tile-warps {v[3]})")
print(f"mma per tile: wait t_empty {v[4]/mt:.0f}  wait b_full {v[5]/mt:.0f} cycles (tiles {v[6]})")
