"""Top SASS lines of an ncu source page (csv) by stall samples / excessive smem wavefronts.
usage: ncu -i REP --page source --csv [--launch-skip N --launch-count 1] > src.csv; python tools/ncu_source.py src.csv"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(rows[1]) - 2 and not r[0].startswith("Kernel")]
col = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
tot = collections.Counter()
for r in data:
    for s in stalls:
        try:
            tot[s] += int(r[col[s]] or 0)
        except (ValueError, IndexError):
            pass
print("stall totals:", tot.most_common(8))
print("\nTop lines by samples:")
def num(r, c):
    try:
        return float(r[col[c]] or 0)
    except (ValueError, KeyError):
        return 0.0
for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:25]:
    top = sorted(((num(r, s), s) for s in stalls), reverse=True)[:2]
    print("%6d  %-60s exc_wf=%6d  %s" % (num(r, "Warp Stall Sampling (All Samples)"), r[1].strip()[:60],
                                        num(r, "L1 Wavefronts Shared Excessive"), top))
print("\nTop lines by excessive smem wavefronts:")
for r in sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:8]:
    print("%10d  %s  (n-way %s)" % (num(r, "L1 Wavefronts Shared Excessive"), r[1].strip()[:70], r[col["L1 Conflicts Shared N-Way"]]))
mix = collections.Counter()
for r in data:
    op = r[1].strip().split()[0] if r[1].strip() else ""
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    mix[op.split(".")[0]] += num(r, "Instructions Executed")
print("\nInstruction mix:", mix.most_common(14))
