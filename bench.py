#!/usr/bin/env python
"""Benchmark: randomized SVD (arXiv 1608.02148, Alg. 5 / Alg. 6 / Alg. 7) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one call of the library's public API on one batch of the workload
(BASELINE.json configs): config 3 (default, the largest single-GPU FP64
workload) = rpca of the FP64 200000 x 4000 image-like matrix, column-centred,
k=100, p=20, q=2, uniform Omega (Alg. 6: colsum, Omega, 2q+2 passes over A,
panel orthonormalisations, Jacobi SVD of B, scores); configs 1, 2, 4 = rsvd
(Alg. 5); config 5 = rrpca (Alg. 7, the whole IALM loop).  Inputs are
synthetic (synthetic/__init__.py) and resident in HBM when the timed region
starts.  metric = A-bytes streamed per second = the step's algorithmic passes
over A (2q+2 per rsvd, +1 column-mean pass for rpca, + the fused IALM update
for rrpca) x m x n x sizeof / time (whole job, all ranks).  N > 1: A is
row-sharded over the ranks (strong scaling), the library's NCCL communicator
sums the n x l partials.  Steps are enqueued back to back (the calls do not
synchronise with the host); the timed region is bracketed by a barrier and a
device synchronisation, and is timed with CUDA events (max over ranks).

--impl reference times the CPU oracle (oracle/, numpy FP64) on the host cores
on a bounded row sample of the same workload (rank 0 only).
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402

PEAKS_BOX = os.path.join(ROOT, "profiles", "peaks_box.json")
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "rsvd_A_bytes_per_s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(n):
    """--gpus N without a torchrun environment: start N ranks (one per GPU) on
    this node through torch.distributed.run and exit with its status."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def peaks():
    hbm, src_hbm = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(MEASURED):
        try:
            hbm = float(json.load(open(MEASURED))["hbm_gbs"])
            src_hbm = "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            pass
    box = {}
    if os.path.exists(PEAKS_BOX):
        try:
            box = json.load(open(PEAKS_BOX))
        except Exception:
            box = {}
    return hbm, src_hbm, box


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), float(f[2]), f[3:7]))
            except ValueError:
                continue
        if not rows:
            return None
        loaded = [r for r in rows if r[2] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(loaded)}


def step_bytes_for(meta, m, n, es, iters=None):
    """Algorithmic A-bytes of one step: 2q+2 passes per rsvd,
    +1 column-mean pass for rpca; rrpca: (iters + 1) rsvds (||A||_2 and one per
    IALM iteration) + the fused update per iteration (reads A, S, Z; writes S,
    Z, M: 6 m x n arrays)."""
    passes = 2 * meta["q"] + 2
    a_bytes = m * n * es
    if meta.get("rrpca"):
        it = iters or 1
        return (it + 1) * passes * a_bytes + it * 6 * a_bytes
    return passes * a_bytes + (a_bytes if meta["center"] else 0)


def oracle_step(meta, An):
    """One step of the workload by the oracle (the same call the product arm makes)."""
    import oracle
    k, p, q = meta["k"], meta["p"], meta["q"]
    if meta.get("rrpca"):
        o = oracle.oracle_rrpca(An, k=k, p=p, q=q, tol=meta["tol"], maxiter=100, sdist=meta["sdist"],
                                seed=meta["seed_omega"])
        return o["iters"]
    if meta["center"]:
        oracle.oracle_rpca(An, k, center=True, scale=False, p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"])
        return None
    oracle.oracle_rsvd(An, k, p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"])
    return None


def sample_rows(meta, A, budget_s):
    """A row sample of the workload sized for about `budget_s` seconds of oracle
    work: time a small sample, scale linearly in rows (the oracle is O(m n l))."""
    m = A.shape[0]
    l = meta["k"] + meta["p"]
    r0 = int(min(m, max(4 * l, 2000)))
    t0 = time.perf_counter()
    oracle_step(meta, np.ascontiguousarray(A[:r0]))
    t = max(time.perf_counter() - t0, 1e-3)
    rows = int(min(m, max(r0, r0 * budget_s / t)))
    return np.ascontiguousarray(A[:rows]) if rows < m else A


def cpu_baseline_run(meta, A_host, budget_s):
    """The oracle as it stands, on the host cores, on a bounded row sample."""
    An = sample_rows(meta, A_host, budget_s)
    t0 = time.perf_counter()
    iters = oracle_step(meta, An)
    t = time.perf_counter() - t0
    b = step_bytes_for(meta, An.shape[0], An.shape[1], An.itemsize, iters)
    sample = "one oracle %s call on the first %d of %d rows of %s (full n = %d), numpy FP64, %d host threads%s" % (
        "rrpca" if meta.get("rrpca") else ("rpca" if meta["center"] else "rsvd"), An.shape[0], A_host.shape[0],
        meta["name"], An.shape[1], os.cpu_count(), (", %d IALM iterations" % iters) if iters else "")
    return {"value": round(b / t / 1e9, 4), "unit": "GB/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": sample, "ms_per_call": round(t * 1e3, 1)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    A, meta = synthetic.make_config(args.config)
    An = A.numpy()
    total = max(args.steps + args.warmup, 1)
    Ans = sample_rows(meta, An, 60.0 / total)
    for _ in range(args.warmup):
        oracle_step(meta, Ans)
    t0 = time.perf_counter()
    iters = None
    for _ in range(args.steps):
        iters = oracle_step(meta, Ans)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    b = step_bytes_for(meta, Ans.shape[0], An.shape[1], An.itemsize, iters)
    val = b / dt / 1e9
    sample = "oracle %s on the first %d of %d rows of %s (full n = %d), k=%d p=%d q=%d" % (
        "rrpca" if meta.get("rrpca") else ("rpca" if meta["center"] else "rsvd"), Ans.shape[0], An.shape[0],
        meta["name"], An.shape[1], meta["k"], meta["p"], meta["q"])
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if An.itemsize == 8 else "f32",
            "data": "synthetic", "config": {"workload": meta["name"], "rows_sampled": int(Ans.shape[0])},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    import paper_1608_02148_b200 as rb
    if world > torch.cuda.device_count():
        raise SystemExit("bench.py: %d ranks but only %d CUDA devices" % (world, torch.cuda.device_count()))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    A_full, meta = synthetic.make_config(args.config, device=dev)
    m, n = A_full.shape
    offset, m_loc = rb.row_partition(m, world)[rank]
    A = A_full[offset:offset + m_loc].contiguous() if world > 1 else A_full
    del A_full
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    ctx = rb.Context(local, st)
    if world > 1:
        ctx.init_comm(rank, world)
    k, p, q = meta["k"], meta["p"], meta["q"]
    l = min(k + p, min(m, n))
    es = A.element_size()
    center = meta["center"]
    is_rrpca = bool(meta.get("rrpca"))
    kw = dict(p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx, m_global=m, row_offset=offset)
    d = torch.empty(k, dtype=A.dtype, device=dev)
    u = torch.empty(m_loc, k, dtype=A.dtype, device=dev)
    v = torch.empty(n, k, dtype=A.dtype, device=dev)
    rr_state = {}

    def step():
        """One call of the public API (enqueued; no host synchronisation except rrpca's loop)."""
        if is_rrpca:
            out = rb.rrpca(A, k=k, p=p, q=q, tol=meta["tol"], maxiter=100, sdist=meta["sdist"],
                           seed=meta["seed_omega"], ctx=ctx, m_global=m, row_offset=offset)
            rr_state["iters"], rr_state["residual"] = out["iters"], out["residual"]
        elif center:
            rb.rpca(A, k, center=True, scale=False, sync=False, **kw)
        else:
            rb.rsvd(A, k, out=(d, u, v), sync=False, **kw)

    for _ in range(args.warmup):
        step()
    ctx.sync()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    ctx.profile_reset()
    ctx.set_profiling(2)            # the pass kernels (dominant-kernel roofline) timed live, least overhead
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    barrier()
    ctx.set_profiling(False)
    ctx.sync()                      # numerical status of every timed call
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1) / max(args.steps, 1)
    launches = ctx.launch_count()
    prof = {kind: ctx.profile(kind) for kind in range(7)}
    # per-kind breakdown (every kernel class) from a short separate profiled run
    ctx.profile_reset()
    ctx.set_profiling(1)
    n_diag = min(args.steps, 5)
    for _ in range(n_diag):
        step()
    ctx.sync()
    ctx.set_profiling(False)
    prof_all = {kind: ctx.profile(kind) for kind in range(7)}
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    passes = 2 * q + 2
    a_bytes = m * n * es
    step_bytes = step_bytes_for(meta, m, n, es, rr_state.get("iters"))
    value = step_bytes / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel: the streaming pass (kinds 0 = A.X, 1 = A^T.X)
    hbm_peak, hbm_src, box = peaks()
    diag = ctx.stats()
    if es == 8 and diag.get("ozaki_passes", 0) > 0:
        path = "ozaki"
        kinds = {0: "pass_AX (ozaki_pass_kernel NN: int8 slices on tcgen05)",
                 1: "pass_AtX (ozaki_pass_kernel TN: int8 slices on tcgen05)"}
    elif es == 4 and diag.get("ozaki_passes", 0) > 0:
        path = "ozaki32"
        kinds = {0: "pass_AX (ozaki_pass_kernel NN: 3-digit int8 slices of FP32 A on tcgen05)",
                 1: "pass_AtX (ozaki_pass_kernel TN: 3-digit int8 slices of FP32 A on tcgen05)"}
    elif es == 4:
        path = "tf32"
        kinds = {0: "pass_AX (pass_tf32_tn_kernel as X^T A^T: 3xTF32 on tcgen05)",
                 1: "pass_AtX (pass_tf32_tn_kernel as Q^T A: 3xTF32 on tcgen05)"}
    else:
        path = "dmma"
        kinds = {0: "pass_AX (gemm_pass_kernel NN, FP64 DMMA)", 1: "pass_AtX (gemm_pass_kernel TN, FP64 DMMA)"}
    dom = max((0, 1), key=lambda kk: prof[kk][0])
    tot_ms, cnt, _ = prof[dom]
    avg_ms = tot_ms / max(cnt, 1)
    # algorithmic bytes of one pass: A once + the n x l and m_loc x l panels
    bytes_launch = (m_loc * n + n * l + m_loc * l) * es
    flops_launch = 2.0 * m_loc * n * l
    gbs = bytes_launch / (avg_ms * 1e-3) / 1e9
    tf = flops_launch / (avg_ms * 1e-3) / 1e12
    tot_all = max(sum(prof_all[kk][0] for kk in range(7)), 1e-12)
    share = {"A.X": prof_all[0][0] / tot_all, "At.X": prof_all[1][0] / tot_all}
    per_kind = {name: round(prof_all[kk][0] / max(n_diag, 1), 4) for kk, name in
                enumerate(["pass_AX", "pass_AtX", "panel_orth", "jacobi_svd", "omega", "ozaki_slice_A",
                           "ozaki_slice_X"])}
    if path == "dmma":
        fp64 = float(box.get("dmma_m8n8k4_tflops_w8", 37.1))
        roof = {"bound": "tensor", "kernel": kinds[dom], "achieved": round(tf, 3), "peak": fp64,
                "unit": "TFLOP/s", "frac": round(tf / fp64, 4), "traffic": None,
                "peak_source": "profiles/peaks_box.json dmma_m8n8k4_tflops_w8 (FP64 DMMA)"}
    else:
        roof = {"bound": "hbm", "kernel": kinds[dom], "achieved": round(gbs, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(gbs / hbm_peak, 4), "traffic": None, "peak_source": hbm_src}
        # the sustained int8 roof of a kernel timed inside a long step: the MMA loop on
        # random operand bytes runs into the software power cap (~1600 MHz); the
        # zero-data / burst figure is reported beside it
        i8_key = next((k for k in ("tcgen05_i8_tops_sustained_random", "tcgen05_i8_tops_sustained", "tcgen05_i8_tops")
                       if k in box), None)
        i8_peak = box.get(i8_key) if i8_key else None
        i8_burst = box.get("tcgen05_i8_tops_sustained", box.get("tcgen05_i8_tops"))
        if path in ("ozaki", "ozaki32") and i8_peak:
            # the other roof: 28 (FP64 A, 7 digits) or 6 (FP32 A, 3 digits) int8 slice
            # products per product on the tensor pipe.  The binding roof is
            # the one with the longer floor: bytes / HBM peak or int8 ops / tcgen05 int8
            # peak (config 3, l = 120: tensor)
            ops_launch = (28.0 if path == "ozaki" else 6.0) * flops_launch
            # what the kernel itself streams: the digit slices of A (7 or 3 bytes per element)
            digits = 7 if path == "ozaki" else 3
            kbytes = m_loc * (-(-n // 128) * 128) * digits
            roof["slice_bytes_per_launch"] = kbytes
            roof["slice_bytes_frac"] = round(kbytes / (avg_ms * 1e-3) / 1e9 / hbm_peak, 4)
            i8 = ops_launch / (avg_ms * 1e-3) / 1e12
            src = "profiles/peaks_box.json %s (tools/peaks_tc.cu)" % i8_key
            t_hbm = bytes_launch / (hbm_peak * 1e9)
            t_i8 = ops_launch / (i8_peak * 1e12)
            hbm_view = {"achieved_gbs": round(gbs, 1), "peak_gbs": hbm_peak, "frac": round(gbs / hbm_peak, 4),
                        "floor_ms": round(t_hbm * 1e3, 4), "peak_source": hbm_src}
            i8_view = {"achieved_tops": round(i8, 1), "peak_tops": i8_peak, "frac": round(i8 / i8_peak, 4),
                       "floor_ms": round(t_i8 * 1e3, 4), "ops_per_launch": ops_launch, "peak_source": src,
                       "peak_burst_zero_data": i8_burst, "frac_vs_burst": round(i8 / i8_burst, 4)}
            if t_i8 > t_hbm:
                roof = {"bound": "tensor", "kernel": kinds[dom], "achieved": round(i8, 1), "peak": i8_peak,
                        "unit": "TOPS (int8)", "frac": round(i8 / i8_peak, 4), "traffic": None,
                        "peak_source": src, "peak_burst_zero_data": i8_burst,
                        "frac_vs_burst": round(i8 / i8_burst, 4), "hbm": hbm_view}
            else:
                roof["tensor_i8"] = i8_view
        if path == "tf32" and box.get("tcgen05_tf32_tflops"):
            t3 = 3.0 * flops_launch / (avg_ms * 1e-3) / 1e12
            roof["tensor_tf32"] = {"achieved_tflops": round(t3, 1), "peak_tflops": box["tcgen05_tf32_tflops"],
                                   "frac": round(t3 / box["tcgen05_tf32_tflops"], 4),
                                   "peak_source": "profiles/peaks_box.json tcgen05_tf32_tflops (tools/peaks_tc.cu)"}
    roof.update({"path": path, "algorithmic_per_launch": {"bytes": bytes_launch, "flops": flops_launch,
                                                          "recipe": "sizeof * (m_loc n + n l + m_loc l)"},
                 "avg_launch_ms": round(avg_ms, 5), "launches_timed": int(cnt),
                 "step_share": {kk: round(vv, 4) for kk, vv in share.items()},
                 "per_kind_ms_per_step": per_kind})
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic_cfg%d_%s.json" % (args.config, path))
    if os.path.exists(traffic_file) and world == 1:
        try:
            tr = json.load(open(traffic_file))
            roof["traffic"] = tr.get("AX" if dom == 0 else "AtX")
            roof["traffic_source"] = os.path.relpath(traffic_file, ROOT)
        except Exception:
            pass

    line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if es == 8 else "f32",
            "data": "synthetic (seeded, synthetic/__init__.py)",
            "config": {"workload": meta["name"], "call": "rrpca" if is_rrpca else ("rpca" if center else "rsvd"),
                       "m": m, "n": n, "k": k, "p": p, "q": q, "l": l,
                       "sdist": meta["sdist"], "center": bool(center), "passes_per_rsvd": passes,
                       "A_bytes": a_bytes, "bytes_per_step": step_bytes,
                       "rrpca_iters": rr_state.get("iters"), "rrpca_residual": rr_state.get("residual"),
                       "l2_policy": ("A per rank (%d MB) > L2 (126 MB): no flush" % ((m_loc * n * es) >> 20))
                       if m_loc * n * es > 126e6 else "A L2-resident per rank (latency-bound config)",
                       "parallelism": "row-sharded dp%d" % world, "rows_per_rank": m_loc},
            "roofline": roof, "gpu_launches": int(launches), "clocks": clocks, "diagnostics": diag}

    # end to end through the host-buffer C-ABI calls (rsvd_run_host / rsvd_rpca_host /
    # rsvd_rrpca_host): A copied in from pinned host memory, results copied out, per step
    # (N > 1: each rank passes its own row block from its pinned host memory)
    if not args.no_e2e:
        A_host = A.cpu().pin_memory()
        e2e_steps = max(2, min(args.steps, 10 if not is_rrpca else 2))
        d2h = {}

        def e2e_step():
            if is_rrpca:
                out = rb.rrpca(A_host, k=k, p=p, q=q, tol=meta["tol"], maxiter=100, sdist=meta["sdist"],
                               seed=meta["seed_omega"], ctx=ctx, m_global=m, row_offset=offset)
                res = [out["L"], out["S"]]
            elif center:
                out = rb.rpca(A_host, k, center=True, scale=False, p=p, q=q, sdist=meta["sdist"],
                              seed=meta["seed_omega"], ctx=ctx, m_global=m, row_offset=offset)
                res = [out["rotation"], out["eigvals"], out["sdev"], out["x"], out["center"]]
            else:
                r = rb.rsvd_host(A_host, k, p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx,
                                 m_global=m, row_offset=offset)
                res = [r.d, r.u, r.v]
            d2h["bytes"] = int(sum(t.numel() * t.element_size() for t in res))

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        ems = (time.perf_counter() - t0) * 1e3 / e2e_steps
        if world > 1:
            import torch.distributed as dist
            te = torch.tensor([ems, float(m_loc * n * es), float(d2h["bytes"])], dtype=torch.float64, device=dev)
            tmax = te.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(te, op=dist.ReduceOp.SUM)
            ems, a_in, d_out = float(tmax[0].item()), int(te[1].item()), int(te[2].item())
        else:
            a_in, d_out = int(a_bytes), d2h["bytes"]
        line["e2e"] = {"value": round(step_bytes / (ems * 1e-3) / 1e9, 2), "unit": "GB/s",
                       "ms_per_step": round(ems, 3), "steps": e2e_steps,
                       "h2d_bytes_per_step": a_in, "d2h_bytes_per_step": d_out,
                       "call": "rsvd_rrpca_host" if is_rrpca else ("rsvd_rpca_host" if center else "rsvd_run_host"),
                       "timing": "host wall clock around blocking calls (each returns after its D2H copy)"
                                 + ("; max over ranks, bytes summed over ranks" if world > 1 else "")}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_run(meta, A.cpu().numpy(), args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
