"""Summarise an ncu report: key raw metrics + SASS opcode histogram.
usage: python profiles/ncu_summarize.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum',
        'smsp__average_warp_latency_per_inst_issued.ratio', 'sm__inst_executed.sum']


def main(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')][:90]
        print('kernel:', name)
        for i, h in enumerate(hdr):
            if h in KEYS:
                print(f'  {h:60s} {r[i]} {units[i]}')
    src = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    c, cs = Counter(), Counter()
    i_src = i_s = i_ie = None
    for r in rows:
        if r and r[0] == 'Address':  # header of a kernel section
            i_src, i_s, i_ie = r.index('Source'), r.index('Warp Stall Sampling (All Samples)'), r.index('Instructions Executed')
            continue
        if i_src is None or len(r) <= max(i_src, i_s, i_ie) or not r[0].startswith('0x'):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith('@') else toks[0]
        op = op.split('.')[0]
        c[op] += int(r[i_ie] or 0)
        cs[op] += int(r[i_s] or 0)
    tot = sum(c.values())
    print(f'  warp instructions executed: {tot}  stall samples: {sum(cs.values())}')
    for op, v in c.most_common(12):
        print(f'    {op:10s} {v:12d} ({100 * v / max(1, tot):4.1f}%) samples={cs[op]}')


if __name__ == '__main__':
    main(sys.argv[1])
