"""Debug: repeated sharded rpca / rsvd runs; prints the relative error per run."""
import os
import sys
import torch
import paper_1608_02148_b200 as rb

g = torch.Generator().manual_seed(4)
A = (torch.randn(6000, 300, generator=g, dtype=torch.float64) *
     torch.exp(-torch.arange(300, dtype=torch.float64) / 40) + torch.linspace(0, 5, 300, dtype=torch.float64))
Ad = A.cuda()
one = rb.rpca(Ad, 20, center=True, scale=True, seed=3)
one_s = rb.rsvd(Ad, 20, seed=3)
for call in ("rpca", "rsvd"):
    for world in (2, 3):
        errs = []
        for rep in range(6):
            parts = rb.row_partition(6000, world)

            def fn(ctx, r):
                off, rows = parts[r]
                if call == "rpca":
                    return rb.rpca(Ad[off:off + rows], 20, center=True, scale=True, seed=3, ctx=ctx, m_global=6000,
                                   row_offset=off)["eigvals"]
                return rb.rsvd(Ad[off:off + rows], 20, seed=3, ctx=ctx, m_global=6000, row_offset=off).d
            out = rb.run_ranks(fn, world)
            ref = one["eigvals"] if call == "rpca" else one_s.d
            errs.append(((out[0] - ref).abs() / ref).max().item())
        print(os.environ.get("TAG", ""), call, "world", world, " ".join("%.1e" % e for e in errs), flush=True)
