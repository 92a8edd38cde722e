"""Per-kernel totals of the last complete rsvd in an ncu launch list
(--metrics gpu__time_duration.sum --csv): a step starts at omega_kernel.
    python tools/launch_step.py gpurun_out/launches_cfg3.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
ks = [(r[ki], float(r[vi].replace(',', ''))) for r in rows]
starts = [i for i, (k, _) in enumerate(ks) if 'omega_kernel' in k]
a, b = (starts[-2], starts[-1]) if len(starts) > 1 else (starts[-1], len(ks))
step = ks[a:b]
print('launches in step', len(step), 'sum of durations %.1f us' % (sum(v for _, v in step) / 1000))
agg = collections.OrderedDict()
for k, v in step:
    x = agg.setdefault(k.split('(')[0][:70], [0, 0.0])
    x[0] += 1
    x[1] += v
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print('%-70s %3d %10.1f us' % (k, c, v / 1000))
