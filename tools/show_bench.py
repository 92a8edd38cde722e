"""Print the key numbers of bench.py JSON lines in log files."""
import json
import sys

for fn in sys.argv[1:]:
    for line in open(fn):
        if not line.startswith('{'):
            continue
        d = json.loads(line)
        r = d.get('roofline', {})
        print("%-28s ms %8.4f val %8.1f frac %s launch %s kinds %s clk %s" % (
            fn.split('/')[-1], d.get('ms_per_step', 0), d.get('value', 0), r.get('frac'), r.get('avg_launch_ms'),
            r.get('per_kind_ms_per_step'), (d.get('clocks') or {}).get('sm_mhz')))
