"""Debug: sharded vs single-rank rpca outputs (center, scale, eigvals) for several world sizes."""
import torch
import paper_1608_02148_b200 as rb

g = torch.Generator().manual_seed(4)
A = (torch.randn(6000, 300, generator=g, dtype=torch.float64) *
     torch.exp(-torch.arange(300, dtype=torch.float64) / 40) + torch.linspace(0, 5, 300, dtype=torch.float64))
Ad = A.cuda()
one = rb.rpca(Ad, 20, center=True, scale=True, seed=3)
for world in (2, 3, 4, 5, 6):
    parts = rb.row_partition(6000, world)

    def fn(ctx, r):
        off, rows = parts[r]
        return rb.rpca(Ad[off:off + rows], 20, center=True, scale=True, seed=3, ctx=ctx, m_global=6000, row_offset=off)
    out = rb.run_ranks(fn, world)
    msg = []
    for key in ("center", "scale", "eigvals"):
        rel = ((out[0][key] - one[key]).abs() / one[key].abs()).max().item()
        msg.append("%s %.2e" % (key, rel))
    print("world", world, *msg, flush=True)
for world in (3,):
    parts = rb.row_partition(6000, world)
    def fn(ctx, r):
        off, rows = parts[r]
        return rb.rpca(Ad[off:off + rows].clone(), 20, center=True, scale=True, seed=3, ctx=ctx, m_global=6000,
                       row_offset=off)["eigvals"]
    out = rb.run_ranks(fn, world)
    print("world 3 with cloned (separately allocated) shards: eig rel %.2e" %
          ((out[0] - one["eigvals"]).abs() / one["eigvals"]).max().item())
import os
os.environ["RSVD_FP64_PATH"] = "dmma"
def fn(ctx, r):
    off, rows = rb.row_partition(6000, 3)[r]
    return rb.rpca(Ad[off:off + rows], 20, center=True, scale=True, seed=3, ctx=ctx, m_global=6000, row_offset=off)["eigvals"]
out = rb.run_ranks(fn, 3)
print("world 3 DMMA path: eig rel %.2e" % ((out[0] - one["eigvals"]).abs() / one["eigvals"]).max().item())
