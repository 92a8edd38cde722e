"""Small calls of every entry point (run with CUDA_LAUNCH_BLOCKING=1 to localise a fault)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import paper_1608_02148_b200 as rb
import synthetic
g = torch.Generator().manual_seed(3)
A = (torch.randn(700, 300, generator=g, dtype=torch.float64) * torch.exp(-torch.arange(300, dtype=torch.float64) / 20)).cuda()
r = rb.rsvd(A, 20, p=10, q=2, seed=1)
r = rb.rsvd(A, 20, p=10, q=1, seed=1, power="direct")
r = rb.rsvd(A, 20, p=10, q=1, seed=1, power="lu")
r = rb.rsvd(A.float(), 20, p=10, q=2, seed=1)
Q, B = rb.rqb(A, 20, p=10, q=1)
pc = rb.rpca(A, 10, center=True, scale=True)
d = rb.rid(A, 15, p=10, q=1)
c = rb.rcur(A, 15, p=10, q=1)
L0 = synthetic.sparse_plus_lowrank(800, 120, rank=4, frac=0.05, seed=2)[0].cuda()
rr = rb.rrpca(L0, k=0, p=10, q=2, tol=1e-6, maxiter=30)
rr = rb.rrpca(L0, k=8, p=10, q=2, tol=1e-6, maxiter=10, rand=False)
Ad = (torch.randn(300, 40, generator=g, dtype=torch.float64) @ torch.randn(40, 200, generator=g, dtype=torch.float64)).cuda()
r = rb.rsvd(Ad, 60, p=10, q=1, seed=2)          # rank-deficient: robust TSQR path
torch.cuda.synchronize()
print("sanitize smoke done")
