"""Profiling driver (not product code): FP32 rsvd on a 250000 x 10000 matrix
(config 4's row length and l, fewer rows) -- two calls; under ncu skip the
first call's kernels.  python tools/prof_fp32.py [m]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_02148_b200 as rb

m = int(sys.argv[1]) if len(sys.argv) > 1 else 250000
n = 10000
g = torch.Generator(device="cuda").manual_seed(5)
U = torch.randn(m, 200, device="cuda", generator=g)
V = torch.randn(n, 200, device="cuda", generator=g)
A = (U * torch.exp(-torch.arange(200, device="cuda") / 50.0)) @ V.T / 100.0
A += 1e-4 * torch.randn(m, n, device="cuda", generator=g)
del U, V
for _ in range(2):
    r = rb.rsvd(A, 100, p=20, q=1, seed=3)
torch.cuda.synchronize()
print("d[:3]", r.d[:3].tolist())
