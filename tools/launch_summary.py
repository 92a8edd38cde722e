"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_summary.py launches.csv [--only-ours]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    if "--only-ours" in sys.argv and "rsvd::" not in r[ki] and not name.startswith(("gemm_", "chol", "jacobi", "hqr", "omega", "tsqr", "colsum", "sign", "scale", "copy", "fill", "zero", "small", "pca", "check", "ialm", "lowrank", "reduce", "form")):
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] += 1
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("%10.1f us %5.1f%% n=%4d avg=%9.2f us  %s" % (v, 100 * v / allt, cnt[k], v / cnt[k], k[:90]))
print("total %.1f us" % allt)
