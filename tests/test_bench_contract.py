"""The bench.py JSON line the driver consumes: keys, types and units.

CPU: the reference arm (`--impl reference`, the oracle on host cores) on the
small config.  GPU: the product arm on the bench default (config 3, rpca) with
a short run -- roofline, e2e through the host-buffer C-ABI call, launch count,
clocks and the cpu_baseline present and consistent.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"], timeout=600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference"
    assert d["metric"] == "rsvd_A_bytes_per_s" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg1")


@pytest.mark.gpu
def test_product_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--cpu-budget", "3"], timeout=900)
    assert BASE_KEYS <= set(d)
    assert d["metric"] == "rsvd_A_bytes_per_s" and d["dtype"] == "f64" and d["n_gpus"] == 1
    # value = bytes of A streamed per step / time
    assert abs(d["value"] - d["config"]["bytes_per_step"] / (d["ms_per_step"] * 1e-3) / 1e9) <= 1e-3 * d["value"] + 0.01
    r = d["roofline"]
    # the binding roof is the longer floor: config 3 (l = 120) is int8-tensor bound,
    # with the HBM view kept beside it
    assert r["path"] == "ozaki" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3 and 0 < r["frac"] <= 1.0
    if r["bound"] == "tensor":
        assert r["unit"] == "TOPS (int8)" and r["hbm"]["floor_ms"] > 0
        assert 0 < r["hbm"]["frac"] <= 1.0
    else:
        assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["tensor_i8"]["floor_ms"] <= r["avg_launch_ms"]
    e = d["e2e"]
    assert e["unit"] == "GB/s" and 0 < e["value"] < d["value"]
    assert e["h2d_bytes_per_step"] == d["config"]["A_bytes"] and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"] is not None and d["clocks"]["sm_mhz"] > 0
    assert d["config"]["workload"].startswith("cfg3") and d["config"]["call"] == "rpca"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    # the roofline counts the algorithmic bytes of one pass: A + the two panels
    c = d["config"]
    assert r["algorithmic_per_launch"]["bytes"] == 8 * (c["m"] * c["n"] + c["n"] * c["l"] + c["m"] * c["l"])


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """--gpus N without a torchrun environment re-executes bench.py under
    torch.distributed.run with N processes (the command is checked, not run)."""
    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit):
        bench.relaunch_under_torchrun(4)
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4" and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
