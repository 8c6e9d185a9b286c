"""Where the WMD row's time goes: bounds, host driver, EMD launches (sizes and times)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_07227_b200 import _lib, device, emd, synthetic as S
V, m, n1, nq, h, k = 20_000, 300, 20_000, 64, 40, 10
E = S.embeddings(V, m, seed=0)
x1 = S.histograms(n1, V, h, seed=1)
x2 = S.histograms(nq, V, h, seed=2)
Et = torch.from_numpy(E).cuda()
emd.prefiltered_topk_wmd_batch(x1, x2, Et, k)
orig = emd.solve_batch_csr
log = []
def wrapped(*a, **kw):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = orig(*a, **kw)
    torch.cuda.synchronize(); log.append((len(a[1]), (time.perf_counter() - t) * 1e3))
    return r
emd.solve_batch_csr = wrapped
_lib.profile_reset(True)
torch.cuda.synchronize(); t0 = time.perf_counter()
res, solves = emd.prefiltered_topk_wmd_batch(x1, x2, Et, k)
torch.cuda.synchronize(); tot = (time.perf_counter() - t0) * 1e3
prof = _lib.profile_read()
print(os.environ.get("LCRW_LIB", "in-tree"), "total ms", round(tot, 1),
      "solves counted", int(solves.sum()), "ids", hash(tuple(int(i) for r in res for i in r.ids)))
print("solve_batch calls (problems, wall ms):", [(n, round(t, 1)) for n, t in log])
print("kernel profile:", {k_: (round(v["ms"], 1), v["launches"]) for k_, v in prof.items()})
