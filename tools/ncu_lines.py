"""Attribute ncu SASS-level samples/instructions to CUDA source lines.
    python tools/ncu_lines.py report.ncu-rep object.o kernel_substring
Uses nvdisasm line info of the kernel (compiled with -lineinfo)."""
import csv
import io
import re
import subprocess
import sys
import tempfile
import os

rep, obj, ksub = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
src = list(csv.reader(io.StringIO(subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'],
                                                 capture_output=True, text=True).stdout)))
hdr = src[1]
rows = [dict(zip(hdr, x)) for x in src[2:]]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(['cuobjdump', '-xelf', 'all', obj], cwd=d, capture_output=True)
    dis = ''
    for f in sorted(os.listdir(d)):  # the cubin that holds the kernel
        if f.endswith('.cubin'):
            t = subprocess.run(['nvdisasm', '-g', '-c', os.path.join(d, f)], capture_output=True, text=True).stdout
            if ksub in t:
                dis = t
                break
# split per function
funcs = re.split(r'\n\s*\.text\.(\S+):', dis)
body = None
for i in range(1, len(funcs), 2):
    if ksub in funcs[i]:
        body = funcs[i + 1]
        break
line = None
lines = []
for ln in body.split('\n'):
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln):
        lines.append(line)
print('sass in ncu', len(rows), 'sass in nvdisasm', len(lines))
agg = {}
tot_i = sum(int(x['Instructions Executed'] or 0) for x in rows) or 1
tot_s = sum(int(x['Warp Stall Sampling (All Samples)'] or 0) for x in rows) or 1
for x, l in zip(rows, lines):
    a = agg.setdefault(l, [0, 0])
    a[0] += int(x['Instructions Executed'] or 0)
    a[1] += int(x['Warp Stall Sampling (All Samples)'] or 0)
srcfile = None
key = 0 if "--inst" in sys.argv else 1
for l, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:40]:
    print(f'line {l}: inst {100*i/tot_i:5.1f}%  samples {100*s/tot_s:5.1f}%')
