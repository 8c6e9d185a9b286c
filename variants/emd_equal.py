"""Objectives of one EMD batch, to compare two library builds bitwise."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_07227_b200 import emd, synthetic as S
V = 20_000
E = S.embeddings(V, 300, seed=0)
x1 = S.histograms(3000, V, 40, seed=1)
x2 = S.histograms(5, V, 40, seed=2)
rng = np.random.default_rng(0)
docs, qs = rng.integers(0, 3000, 4000), rng.integers(0, 5, 4000)
obj = emd.solve_batch_csr(x1, docs, x2, qs, torch.from_numpy(E).cuda())
np.save(sys.argv[1], obj)
