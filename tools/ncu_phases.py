"""Aggregate ncu SASS samples/instructions by source-line ranges (phases).
    python tools/ncu_phases.py report obj kernel_substring name:lo-hi [name:lo-hi ...]"""
import subprocess, sys, os, re, csv, io, tempfile
rep, obj, ks = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    n, r = a.split(':'); lo, hi = r.split('-'); ranges.append((n, int(lo), int(hi)))
src = list(csv.reader(io.StringIO(subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'] + (['--launch-skip', os.environ['NCU_SKIP'], '--launch-count', '1'] if os.environ.get('NCU_SKIP') else []), capture_output=True, text=True).stdout)))
off = 1 if src and src[0] and src[0][0] == 'Kernel Name' else 0
end = next((i for i in range(off + 1, len(src)) if src[i] and src[i][0] == 'Kernel Name'), len(src))
hdr = src[off]; rows = [dict(zip(hdr, x)) for x in src[off + 1:end]]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(['cuobjdump', '-xelf', 'all', obj], cwd=d, capture_output=True)
    dis = ''
    for f in sorted(os.listdir(d)):  # the cubin that holds the kernel
        if f.endswith('.cubin'):
            t = subprocess.run(['nvdisasm', '-g', '-c', os.path.join(d, f)], capture_output=True, text=True).stdout
            if ks in t:
                dis = t
                break
funcs = re.split(r'\n\s*\.text\.(\S+):', dis)
body = next(funcs[i + 1] for i in range(1, len(funcs), 2) if ks in funcs[i])
line, lines = None, []
for ln in body.split('\n'):
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m: line = int(m.group(1)); continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln): lines.append(line)
agg = {}
ti = sum(int(x['Instructions Executed'] or 0) for x in rows) or 1
ts = sum(int(x['Warp Stall Sampling (All Samples)'] or 0) for x in rows) or 1
stall_keys = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
st = {}
for x, l in zip(rows, lines):
    name = 'other'
    for n, lo, hi in ranges:
        if l is not None and lo <= l <= hi: name = n; break
    a = agg.setdefault(name, [0, 0]); a[0] += int(x['Instructions Executed'] or 0); a[1] += int(x['Warp Stall Sampling (All Samples)'] or 0)
    d = st.setdefault(name, {})
    for k in stall_keys:
        d[k] = d.get(k, 0) + int(float(x.get(k) or 0))
for n, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    top = sorted(st[n].items(), key=lambda kv: -kv[1])[:4]
    tops = ' '.join(f'{k[6:]}={100*v/ts:.1f}' for k, v in top if v)
    print(f'{n:12s} inst {100*i/ti:5.1f}%  ({i/1e6:7.1f} M)   samples {100*s/ts:5.1f}%   [{tops}]')
