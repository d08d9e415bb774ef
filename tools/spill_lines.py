"""List the source lines of local-memory spill traffic (STL/LDL) in one kernel of a cubin.
    python tools/spill_lines.py build/sass/f2_p4.cubin k_fusedILi4ELi3ELi2E"""
import re
import subprocess
import sys
from collections import Counter

cub, ks = sys.argv[1], sys.argv[2]
dis = subprocess.run(['nvdisasm', '-g', '-c', cub], capture_output=True, text=True).stdout
funcs = re.split(r'\n\s*\.text\.(\S+):', dis)
body = next(funcs[i + 1] for i in range(1, len(funcs), 2) if ks in funcs[i])
line, c = None, Counter()
for ln in body.split('\n'):
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m:
        line = int(m.group(1))
        continue
    m = re.search(r'\b(STL|LDL)(\.\S+)?\s', ln)
    if m:
        c[(line, m.group(1))] += 1
for (l, op), n in sorted(c.items()):
    print(f'line {l} {op} x{n}')
