"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name the
launch count, total time and share of the total.
    python tools/launch_summary.py gpurun_out/launches.csv > profiles/launches_summary.csv"""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if not l.startswith('==')]
rows = list(csv.DictReader(lines))
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    v = float(r['Metric Value'].replace(',', '')) * scale[r['Metric Unit']]
    a = agg[r['Kernel Name']]
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values()) or 1.0
w = csv.writer(sys.stdout)
w.writerow(['kernel', 'launches', 'total_us', 'share'])
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([k[:120], n, f'{t:.1f}', f'{t / tot:.4f}'])
