import sys, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1302_5995_b200 import hbs as H
d = 1.0 + (np.arange(64) % 7)
c = H.compress(np.diag(d), 1e-12, 16)
x = np.linspace(-1.0, 2.0, 64)
for i in range(4):
    y = H.apply(c, x)
    bad = np.nonzero(np.abs(y - d * x) > 1e-12)[0]
    print("host", i, bad[:20], len(bad))
xt = torch.tensor(x, device="cuda")
for i in range(3):
    y = H.apply(c, xt).cpu().numpy()
    bad = np.nonzero(np.abs(y - d * x) > 1e-12)[0]
    print("dev", i, bad[:20], len(bad))
X = np.random.default_rng(0).standard_normal((64, 5))
for i in range(3):
    y = H.apply(c, X)
    print("5col", i, np.abs(y - d[:, None] * X).max())
c2 = H.compress(np.diag(d) + 0.01 * np.random.default_rng(1).standard_normal((64, 64)), 1e-12, 16)
print(c2.ranks)
A = H.reconstruct(c2)
for i in range(3):
    print("c2 vec", i, np.abs(H.apply(c2, x) - A @ x).max())
