#!/usr/bin/env python
"""Two symmetric top-10 passes of BASELINE configs[1] (C2: 1M docs x 1k queries, V = 100k,
m = 300; bench.py's synthetic data) -- the command the ncu captures of profiles/ run, e.g.
    ncu --set full -k regex:table_min_kernel --launch-skip 3 -c 1 python tools/c2_pass.py
(the 4th table_min launch is the second pass's first full doc batch, bench.py's launch)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1711_07227_b200 import device, synthetic as S  # noqa: E402

V = 100_000
E = S.embeddings(V, 300, seed=0)
x1 = S.histograms(1_000_000, V, 50, seed=1)
x2 = S.histograms(1000, V, 50, seed=2)
prep = device.PreparedEmbeddings(E)
d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
for _ in range(2):
    d, i = device.symmetric(d1, d2, prep, 10)
torch.cuda.synchronize()
print("ok", tuple(d.shape))
