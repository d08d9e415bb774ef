"""Summarise an ncu report: key metrics + stall reasons + hottest SASS regions.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--blocks]
"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'launch__shared_mem_per_block_dynamic', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem']


def run(args):
    return subprocess.run(['ncu', '-i'] + args, capture_output=True, text=True).stdout


def main(path, blocks=False):
    raw = list(csv.reader(io.StringIO(run([path, '--page', 'raw', '--csv']))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        print('kernel:', d.get('Kernel Name', '')[:100])
        for k in KEYS:
            if k in d:
                print(f'  {k} = {d[k]} {units[hdr.index(k)]}')
        st = sorted(((float(d[h]), h) for h in hdr if 'average_warps_issue_stalled' in h and 'ratio' in h
                     and d[h] not in ('', 'n/a')), reverse=True)[:8]
        print('  stalls:', ', '.join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st))
    if blocks:
        src = list(csv.reader(io.StringIO(run([path, '--page', 'source', '--csv']))))
        h2 = src[1]
        rows = [dict(zip(h2, x)) for x in src[2:]]
        tot = sum(int(x['Instructions Executed'] or 0) for x in rows) or 1
        smp = sum(int(x['Warp Stall Sampling (All Samples)'] or 0) for x in rows) or 1
        B = 32
        blk = {}
        for i, x in enumerate(rows):
            e = blk.setdefault(i // B, [0, 0, x['Source'].strip()[:70]])
            e[0] += int(x['Instructions Executed'] or 0)
            e[1] += int(x['Warp Stall Sampling (All Samples)'] or 0)
        for b, (ins, s, txt) in sorted(blk.items(), key=lambda kv: -kv[1][1])[:12]:
            print(f'  sass[{b*B:5d}] inst {100*ins/tot:5.1f}%  samples {100*s/smp:5.1f}%  {txt}')


if __name__ == '__main__':
    main(sys.argv[1], '--blocks' in sys.argv)
