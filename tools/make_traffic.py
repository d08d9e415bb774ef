"""Write profiles/traffic.json from an ncu report holding one fused-matvec launch (k_fused / k_ws) per sweep degree.
    python tools/make_traffic.py gpurun_out/sweep.ncu-rep "<source description>"
Per degree: DRAM bytes (read + write) and the ncu (serialised, cold-cache) duration."""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv', '--metrics',
                      'gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}
per = {}
for r in rows[2:]:
    m = (re.search(r'k_fused<(\d+), (\d+), (\d+), (?:0|false)>', r[col['Kernel Name']]) or
         re.search(r'k_ws<(\d+), (\d+), (?:0|false)>', r[col['Kernel Name']]))
    if not m:
        continue
    v = lambda k: float(r[col[k]].replace(',', '')) * scale[units[col[k]]]
    per.setdefault(m.group(1), {"dram_bytes": v('dram__bytes_read.sum') + v('dram__bytes_write.sum'),
                                "ncu_time_us": v('gpu__time_duration.sum')})
json.dump({"source": src, "per_degree": per,
           # one sweep step = one launch per degree; comparable with the bench's aggregated algorithmic bytes
           "bytes_per_launch": sum(v["dram_bytes"] for v in per.values())}, open(os.path.join(os.path.dirname(__file__), '..', 'profiles', 'traffic.json'), 'w'), indent=1)
print(json.dumps(per, indent=1))
