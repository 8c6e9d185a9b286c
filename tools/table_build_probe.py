import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_1711_07227_b200 import device, synthetic as S
V = 100_000
E = S.embeddings(V, 300, seed=0)
x2 = S.histograms(1000, V, 50, seed=2)
prep = device.PreparedEmbeddings(E)
res2 = device.Restricted.build(device.DeviceCSR.upload(x2), prep, host_plan=True)
for _ in range(2):
    T = device.distance_table(res2, prep)
torch.cuda.synchronize()
print("ok", T.numel())
