"""Time the reverse Phase-1 kernel alone (mid config) for the library in $LCRW_LIB."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_07227_b200 import _lib, device, synthetic as S
V = 50000
E = S.embeddings(V, 300, seed=0)
x1 = S.histograms(100000, V, 50, seed=1)
x2 = S.histograms(256, V, 50, seed=2)
prep = device.PreparedEmbeddings(E)
dx1, dx2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
for it in range(3):
    _lib.profile_reset(True)
    device.symmetric(dx1, dx2, prep, 10)
    torch.cuda.synchronize()
    r = _lib.profile_read()
v_e2 = np.unique(x2.column_ids).size
fl = 2.0 * v_e2 * x1.nnz * 300
print(os.environ.get("LCRW_LIB", "default"), {k: round(v["ms"], 2) for k, v in r.items()}, "TF", round(fl / (r["phase1_rev"]["ms"] * 1e-3) / 1e12, 1))
