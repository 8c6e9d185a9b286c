"""EMD kernel probe: augmentations per problem (LCRW_EMD_ROUNDS build) and time per launch."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_07227_b200 import _lib, device, emd, synthetic as S
V, m, h = 20_000, 300, 40
E = S.embeddings(V, m, seed=0)
x1 = S.histograms(4096, V, h, seed=1)
x2 = S.histograms(1, V, h, seed=2)
Et = torch.from_numpy(E).cuda()
q = x2.row(0)
rows = [x1.row(i) for i in range(4096)]
def run(n):
    return emd.solve_batch([r.weights for r in rows[:n]], [q.weights] * n, embeddings=Et,
                           ids1=[r.word_ids for r in rows[:n]], ids2=[q.word_ids] * n)
run(64)
for n in (64, 1184, 4096):
    torch.cuda.synchronize(); t = time.perf_counter(); run(n); torch.cuda.synchronize()
    print(n, "problems", round((time.perf_counter() - t) * 1e3, 1), "ms")
# augmentation counts (status = -rounds in the experiment build)
orig = emd._check_status
emd._check_status = lambda st: None
dev = torch.device("cuda")
n = 256
h1 = [len(r.word_ids) for r in rows[:n]]
import ctypes as C
sup = torch.tensor(np.concatenate([r.weights.astype(np.float64) for r in rows[:n]]), device=dev)
dem = torch.tensor(np.concatenate([q.weights.astype(np.float64)] * n), device=dev)
so = torch.tensor(emd._offsets(h1), device=dev); do = torch.tensor(emd._offsets([len(q.word_ids)] * n), device=dev)
co = torch.tensor(emd._offsets([a * len(q.word_ids) for a in h1]), device=dev)
i1 = torch.tensor(np.concatenate([r.word_ids for r in rows[:n]]), device=dev)
i2 = torch.tensor(np.concatenate([q.word_ids] * n), device=dev)
obj = torch.empty(n, dtype=torch.float64, device=dev); st = torch.empty(n, dtype=torch.int32, device=dev)
_p = device._p
_lib.call("lcrw_emd_batch", _p(sup), _p(so), _p(dem), _p(do), None, _p(co), _p(Et), V, m, _p(i1), _p(i2), n,
          max(h1), len(q.word_ids), _p(obj), _p(st), None, None, device._stream())
r = -st.cpu().numpy()
print("rounds: mean", r.mean(), "max", r.max(), "n+n", np.mean(h1) + len(q.word_ids))
