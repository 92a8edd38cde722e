"""Summarise an ncu report (raw page) into the metrics we track.
usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT]"""
import csv
import json
import subprocess
import sys

WANT = {
    "kernel": "Kernel Name", "grid": "Grid Size", "block": "Block Size",
    "time_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dmma_inst_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "tensor_pct_elapsed": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l2_bytes": "lts__t_bytes.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, col in WANT.items():
            if col in h:
                i = h.index(col)
                v = r[i]
                try:
                    v = float(v.replace(",", ""))
                    u = units[i]
                    if u == "Kbyte": v *= 1e3
                    elif u == "Mbyte": v *= 1e6
                    elif u == "Gbyte": v *= 1e9
                    elif u == "usecond": v *= 1e3
                    elif u == "msecond": v *= 1e6
                except ValueError:
                    pass
                d[k] = v
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
