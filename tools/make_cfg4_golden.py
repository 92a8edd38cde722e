"""Config-4 oracle reference at full size (BASELINE.json configs[3]: FP32
1,000,000 x 10,000, rank-500 signal s_i = exp(-i/50) + N(0, 1e-4), k=100,
p=20, q=3, Gaussian Omega), written to tests/golden/cfg4_oracle.npz.

Calls only synthetic/ (the seeded input generator, run on the GPU box's GPU:
the same device generator tests/test_gpu_parity.py uses, so both sides see the
same bits) and oracle/ (oracle_rsvd, on the host CPU in FP64 on the exactly
upcast FP32 A, reading R12).  Nothing here comes from the CUDA path.  Needs
~130 GB of host RAM (the FP32 A plus the oracle's FP64 copy).

    python tools/make_cfg4_golden.py [out.npz]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synthetic  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "cfg4_oracle.npz")
    t0 = time.time()
    A, meta = synthetic.make_config(4, device="cuda")
    A_host = A.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    print("generated + copied %.1f s" % (time.time() - t0), flush=True)
    k, p, q = meta["k"], meta["p"], meta["q"]
    t1 = time.time()
    o = oracle.oracle_rsvd(A_host, k, p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"])
    t_oracle = time.time() - t1
    print("oracle_rsvd %.1f s, d[:5] %s" % (t_oracle, o["d"][:5]), flush=True)
    # ||A - U diag(d) V^T||_F / ||A||_F in row chunks (FP64)
    U, d, V = o["u"], o["d"], o["v"]
    num = 0.0
    den = 0.0
    for r0 in range(0, A_host.shape[0], 50000):
        blk = A_host[r0:r0 + 50000].astype(np.float64)
        den += float(np.sum(blk * blk))
        blk -= (U[r0:r0 + 50000] * d[None, :]) @ V.T
        num += float(np.sum(blk * blk))
    err = np.sqrt(num / den)
    info = dict(config=meta["name"], k=k, p=p, q=q, sdist=meta["sdist"], seed_omega=meta["seed_omega"],
                oracle_seconds=round(t_oracle, 1), host_cores=os.cpu_count(), recon_err=err,
                script="tools/make_cfg4_golden.py (oracle/ + synthetic/ only)")
    np.savez_compressed(out, d=d, v=V, u_rows=U[:2000], recon_err=np.array(err), info=json.dumps(info))
    print(json.dumps(info), flush=True)


if __name__ == "__main__":
    main()
