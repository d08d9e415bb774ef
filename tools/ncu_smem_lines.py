"""Shared-memory wavefronts per source line of one kernel in an ncu report.
    python tools/ncu_smem_lines.py report.ncu-rep lib.so kernel_substring [top]"""
import csv, io, os, re, subprocess, sys, tempfile
rep, obj, ks = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
src = list(csv.reader(io.StringIO(subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout)))
off = 1 if src and src[0] and src[0][0] == 'Kernel Name' else 0
end = next((i for i in range(off + 1, len(src)) if src[i] and src[i][0] == 'Kernel Name'), len(src))
hdr = src[off]; rows = [dict(zip(hdr, x)) for x in src[off + 1:end]]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(['cuobjdump', '-xelf', 'all', obj], cwd=d, capture_output=True)
    dis = ''
    for f in sorted(os.listdir(d)):
        if f.endswith('.cubin'):
            t = subprocess.run(['nvdisasm', '-g', '-c', os.path.join(d, f)], capture_output=True, text=True).stdout
            if ks in t:
                dis = t
                break
funcs = re.split(r'\n\s*\.text\.(\S+):', dis)
body = next(funcs[i + 1] for i in range(1, len(funcs), 2) if ks in funcs[i])
line, lines = None, []
for ln in body.split('\n'):
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m: line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln): lines.append(line)
f = lambda x, k: float(x.get(k) or 0)
agg = {}
for x, l in zip(rows, lines):
    a = agg.setdefault(l, [0, 0, 0, 0])
    a[0] += f(x, 'L1 Wavefronts Shared'); a[1] += f(x, 'L1 Wavefronts Shared Ideal')
    a[2] += f(x, 'Instructions Executed'); a[3] += f(x, 'Warp Stall Sampling (All Samples)')
tw = sum(a[0] for a in agg.values()) or 1
ti = sum(a[2] for a in agg.values()) or 1
ts = sum(a[3] for a in agg.values()) or 1
print(f"total shared wavefronts {tw:.3e}, instructions {ti:.3e}")
for l, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{str(l):34s} wf {a[0]/tw*100:5.1f}%  ideal {a[1]/tw*100:5.1f}%  inst {a[2]/ti*100:5.1f}%  samples {a[3]/ts*100:5.1f}%")
