#!/usr/bin/env python
"""Benchmark: randomized SVD (arXiv 1608.02148, Alg. 5) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one full rsvd (Alg. 4 + 2 + 5: Omega, 2q+2 passes over A, panel
orthonormalisations, Jacobi SVD of B, U = Q U~) on device-resident A.  The
default workload is BASELINE.json configs[1] (config 2): FP64 10000 x 5000,
s_i = exp(-i/20) + N(0, 1e-6), k=50, p=10, q=2, Rademacher Omega.
metric = A-bytes streamed per second = (2q+2) * m * n * 8 / t_rsvd (whole job,
all ranks); ms_per_step = the rsvd wall time.  N > 1: A row-sharded over the
ranks (strong scaling), NCCL allreduce of the n x l partials inside the library.

--impl reference times the CPU oracle (oracle/, numpy FP64) on the host cores
on a bounded row sample of the same workload (rank 0 only).
"""
import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    hbm, src_hbm = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(MEASURED):
        try:
            hbm = float(json.load(open(MEASURED))["hbm_gbs"])
            src_hbm = "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            pass
    fp64, src64 = 37.1, "profiles/peaks_box.json (tools/peaks.cu DMMA)"
    if os.path.exists(PEAKS_BOX):
        try:
            fp64 = float(json.load(open(PEAKS_BOX))["dmma_m8n8k4_tflops_w8"])
        except Exception:
            pass
    return hbm, src_hbm, fp64, src64


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


def make_input(cfg, device, rank, world):
    A, meta = synthetic.make_config(cfg, device=device)
    m = A.shape[0]
    if world > 1:
        rows = [(m * r) // world for r in range(world + 1)]
        A = A[rows[rank]:rows[rank + 1]].contiguous()
        meta["row_offset"] = rows[rank]
    else:
        meta["row_offset"] = 0
    meta["m_global"] = m
    return A, meta


def cpu_baseline_run(A_host, meta, budget_s=12.0, max_reps=5, rows=None):
    """The oracle as it stands, on the host cores, on a bounded sample."""
    import oracle
    An = A_host if rows is None else A_host[:rows]
    q = meta["q"]
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_reps:
        t0 = time.perf_counter()
        oracle.oracle_rsvd(An, meta["k"], p=meta["p"], q=q, sdist=meta["sdist"], seed=meta["seed_omega"],
                           center=meta["center"])
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    t = float(np.median(times))
    bytes_ = (2 * q + 2) * An.shape[0] * An.shape[1] * An.itemsize
    return t, bytes_, len(times), An.shape


def run_reference(args, rank, world):
    if rank != 0:
        return
    meta = dict(synthetic.CONFIGS[args.config])
    A, meta = synthetic.make_config(args.config)
    An = A.numpy()
    l = meta["k"] + meta["p"]
    total = args.steps + args.warmup
    rows = int(min(An.shape[0], max(2 * l, An.shape[0] * 10 // max(total, 1))))
    Ans = np.ascontiguousarray(An[:rows])
    import oracle
    for _ in range(args.warmup):
        oracle.oracle_rsvd(Ans, meta["k"], p=meta["p"], q=meta["q"], sdist=meta["sdist"],
                           seed=meta["seed_omega"], center=meta["center"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.oracle_rsvd(Ans, meta["k"], p=meta["p"], q=meta["q"], sdist=meta["sdist"],
                           seed=meta["seed_omega"], center=meta["center"])
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    bytes_ = (2 * meta["q"] + 2) * rows * An.shape[1] * 8
    val = bytes_ / dt / 1e9
    cores = os.cpu_count()
    sample = "oracle rsvd on the first %d of %d rows of %s (full n=%d), k=%d p=%d q=%d" % (
        rows, An.shape[0], meta["name"], An.shape[1], meta["k"], meta["p"], meta["q"])
    line = {"impl": "reference", "metric": "rsvd_A_bytes_per_s", "value": round(val, 4), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": meta["name"], "rows_sampled": rows},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import paper_1608_02148_b200 as rb
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    A, meta = make_input(args.config, dev, rank, world)
    torch.cuda.synchronize()
    ctx = rb.Context(local)
    if world > 1:
        ctx.init_comm(rank, world)
    m, n = meta["m_global"], meta["n"]
    k, p, q = meta["k"], meta["p"], meta["q"]
    l = min(k + p, min(m, n))
    es = A.element_size()
    m_loc = A.shape[0]
    kw = dict(p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx, m_global=m,
              row_offset=meta["row_offset"])
    d = torch.empty(k, dtype=A.dtype, device=dev)
    u = torch.empty(m_loc, k, dtype=A.dtype, device=dev)
    v = torch.empty(n, k, dtype=A.dtype, device=dev)
    center = meta["center"]
    is_rrpca = bool(meta.get("rrpca"))
    rr_state = {}

    def step(Ain=A):
        """One call of the public API on Ain; returns the result tensors (device)."""
        if is_rrpca:
            out = rb.rrpca(Ain, k=k, p=p, q=q, tol=meta["tol"], maxiter=100, sdist=meta["sdist"],
                           seed=meta["seed_omega"], ctx=ctx, m_global=m, row_offset=meta["row_offset"])
            rr_state["iters"] = out["iters"]
            rr_state["residual"] = out["residual"]
            return [out["L"], out["S"]]
        elif center:
            out = rb.rpca(Ain, k, center=True, p=p, q=q, sdist=meta["sdist"], seed=meta["seed_omega"], ctx=ctx,
                          m_global=m, row_offset=meta["row_offset"])
            return [out["rotation"], out["eigvals"], out["x"]]
        else:
            rb.rsvd(Ain, k, out=(d, u, v), **kw)
            return [d, u, v]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

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
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    barrier()
    ctx.set_profiling(False)
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1) / max(args.steps, 1)
    launches = ctx.launch_count()
    prof = {kind: ctx.profile(kind) for kind in range(7)}
    # per-kind breakdown (every kernel class) from a short separate profiled run
    ctx.profile_reset()
    ctx.set_profiling(1)
    n_diag = min(args.steps, 10)
    for _ in range(n_diag):
        step()
    torch.cuda.synchronize(dev)
    ctx.set_profiling(False)
    prof_all = {kind: ctx.profile(kind) for kind in range(7)}
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    passes = 2 * q + 2
    a_bytes = m * n * es
    if is_rrpca:
        # per IALM iteration: one rsvd (2q+2 passes over M) + the fused update
        # (reads A, S, Z; writes S, Z, M = 6 m x n arrays); plus the ||A||_2 rsvd
        it = rr_state.get("iters", 1)
        step_bytes = (it + 1) * passes * a_bytes + it * 6 * a_bytes
    else:
        step_bytes = passes * a_bytes + (a_bytes if center else 0)     # + the column-mean pass
    value = step_bytes / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (the streaming passes; kinds 0 = A.X, 1 = A^T.X)
    hbm_peak, hbm_src, fp64_peak, fp64_src = peaks()
    diag = ctx.stats()
    if es == 8 and diag.get("ozaki_passes", 0) > 0:
        path = "ozaki"
        kinds = {0: "pass_AX (ozaki_pass_kernel NN: int8 slices on tcgen05)",
                 1: "pass_AtX (ozaki_pass_kernel TN: int8 slices on tcgen05)"}
    elif es == 4:
        path = "tf32"
        kinds = {0: "pass_AX (pass_tf32_kernel NN: 3xTF32 on tcgen05)", 1: "pass_AtX (pass_tf32_kernel TN: 3xTF32 on tcgen05)"}
    else:
        path = "dmma"
        kinds = {0: "pass_AX (gemm_pass_kernel NN, FP64 DMMA)", 1: "pass_AtX (gemm_pass_kernel TN, FP64 DMMA)"}
    dom = max((0, 1), key=lambda kk: prof[kk][0])
    tot_ms, cnt, by = prof[dom]
    avg_ms = tot_ms / max(cnt, 1)
    flops_launch = 2.0 * m_loc * n * l
    bytes_launch = m_loc * n * es          # algorithmic: A read once per pass (FP64 / FP32 bytes)
    tf = flops_launch / (avg_ms * 1e-3) / 1e12
    gbs = bytes_launch / (avg_ms * 1e-3) / 1e9
    tot_all = max(sum(prof_all[kk][0] for kk in range(7)), 1e-12)
    share = {"A.X": prof_all[0][0] / tot_all, "At.X": prof_all[1][0] / tot_all}
    per_kind = {name: round(prof_all[kk][0] / max(n_diag, 1), 4) for kk, name in
                enumerate(["pass_AX", "pass_AtX", "panel_orth", "jacobi_svd", "omega", "ozaki_slice_A",
                           "ozaki_slice_X"])}
    if path == "dmma":
        roof = {"bound": "tensor", "kernel": kinds[dom], "achieved": round(tf, 3), "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": round(tf / fp64_peak, 4), "traffic": None,
                "peak_source": fp64_src + " (FP64 DMMA; tcgen05 has no f64 kind)",
                "hbm": {"achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(gbs / hbm_peak, 4), "peak_source": hbm_src}}
    else:
        # tensor-core passes: the target roof is HBM (A read once per pass); the
        # FP64-equivalent flop rate is reported alongside
        roof = {"bound": "hbm", "kernel": kinds[dom], "achieved": round(gbs, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(gbs / hbm_peak, 4), "traffic": None, "peak_source": hbm_src,
                "fp64_equivalent": {"achieved_tflops": round(tf, 3), "dmma_peak_tflops": fp64_peak,
                                    "frac_of_dmma_peak": round(tf / fp64_peak, 4)}}
    roof.update({"path": path, "algorithmic_per_launch": {"flops": flops_launch, "bytes": bytes_launch},
                 "avg_launch_ms": round(avg_ms, 5), "step_share": {kk: round(vv, 4) for kk, vv in share.items()},
                 "per_kind_ms_per_step": per_kind})
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic_cfg%d_%s.json" % (args.config, path))
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file))
            roof["traffic"] = tr.get("AX" if dom == 0 else "AtX")
            roof["traffic_source"] = os.path.relpath(traffic_file, ROOT)
        except Exception:
            pass

    line = {"metric": "rsvd_A_bytes_per_s", "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if es == 8 else "f32",
            "data": "synthetic",
            "config": {"workload": meta["name"], "m": m, "n": n, "k": k, "p": p, "q": q, "l": l,
                       "sdist": meta["sdist"], "center": bool(center), "passes_per_step": passes,
                       "A_bytes": a_bytes, "bytes_per_step": step_bytes,
                       "rrpca_iters": rr_state.get("iters"), "rrpca_residual": rr_state.get("residual"),
                       "l2_policy": "A (%d MB) > L2 (126 MB): no flush" % (a_bytes >> 20)
                       if a_bytes > 126e6 else "A L2-resident (latency-bound config)",
                       "parallelism": "row-sharded dp%d" % world},
            "roofline": roof, "gpu_launches": int(launches), "clocks": clocks,
            "diagnostics": diag}

    # end-to-end: host A (pinned) -> device, rsvd, d/u/v -> host, through the same API
    # (rsvd: d, u, v; rpca: rotation, eigenvalues, scores; rrpca: L and S)
    if not args.no_e2e and world == 1:
        A_host = A.cpu().pin_memory()
        stage = torch.empty_like(A)
        res_h = []
        e2e_steps = max(3, min(args.steps, 20))

        def e2e_step():
            stage.copy_(A_host, non_blocking=True)
            res = step(stage)
            if not res_h:
                res_h.extend(torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res)
            for h, r in zip(res_h, res):
                h.copy_(r, non_blocking=True)
            return res

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(st)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / e2e_steps
        line["e2e"] = {"value": round(step_bytes / (ems * 1e-3) / 1e9, 2), "unit": "GB/s",
                       "ms_per_step": round(ems, 3), "steps": e2e_steps,
                       "h2d_bytes_per_step": int(a_bytes),
                       "d2h_bytes_per_step": int(sum(h.numel() * h.element_size() for h in res_h)),
                       "results": "rrpca L, S" if is_rrpca else ("rpca rotation, eigvals, x" if center
                                                                else "rsvd d, u, v")}

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not is_rrpca and m * n <= 2e8:
        t_cpu, b_cpu, reps, shape = cpu_baseline_run(A.cpu().numpy(), meta)
        line["cpu_baseline"] = {"value": round(b_cpu / t_cpu / 1e9, 4), "unit": "GB/s",
                                "cores": os.cpu_count(), "kind": "oracle",
                                "sample": "median of %d full oracle rsvd calls on %s (%dx%d), numpy FP64, "
                                          "%d host threads" % (reps, meta["name"], shape[0], shape[1],
                                                               os.cpu_count()),
                                "ms_per_rsvd": round(t_cpu * 1e3, 1)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
