#!/usr/bin/env python
"""Probe: table_min / reverse_panels time per C2 step with N SMs taken by spinning CTAs
(tools/sm_hog.cu).  python tools/sm_share.py 0 12 24 36"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1711_07227_b200 import _lib, device, synthetic as S  # noqa: E402

hog = C.CDLL(str(Path(__file__).resolve().parent / "libsmhog.so"))
V = 100_000
E = S.embeddings(V, 300, seed=0)
x1 = S.histograms(1_000_000, V, 50, seed=1)
x2 = S.histograms(1000, V, 50, seed=2)
prep = device.PreparedEmbeddings(E)
d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
device.symmetric(d1, d2, prep, 10)
torch.cuda.synchronize()
side = torch.cuda.Stream()
for n in [int(a) for a in sys.argv[1:]] or [0, 24]:
    stop = torch.zeros(1, dtype=torch.int32, device="cuda")
    if n:
        hog.sm_hog_launch(n, C.c_void_p(stop.data_ptr()), C.c_void_p(side.cuda_stream))
    _lib.profile_reset(True)
    device.symmetric(d1, d2, prep, 10)
    torch.cuda.current_stream().synchronize()
    t = _lib.profile_read()
    stop.fill_(1)
    torch.cuda.synchronize()
    _lib.profile_reset(False)
    print(n, {k: round(v["ms"], 1) for k, v in t.items() if k in ("table_min", "reverse_panels", "spmm")}, flush=True)
