"""Attribute executed warp instructions and stall samples of an ncu report
to CUDA source lines. usage: python profiles/ncu_lines.py <report> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file = cur_line = None
    ie = None
    stats = defaultdict(lambda: [0, 0])

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            cur_file = r[1].split('/')[-1]
            continue
        if r[0] == 'Line No':
            ie = r.index('Instructions Executed')
            continue
        if r[0] == 'Function Name':
            continue
        if r[0] != '':
            cur_line = (cur_file, int(r[0]), r[1][:80])
            continue
        if ie is not None and len(r) > ie:
            stats[cur_line][0] += num(r[ie])
            stats[cur_line][1] += num(r[4])
    tot = sum(v[0] for v in stats.values())
    print('total warp instructions', tot)
    for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f'{100 * v[0] / tot:5.1f}% samples={v[1]:5d} {k[0]}:{k[1]} {k[2]}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
