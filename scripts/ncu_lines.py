"""Per-source-line hot spots of an ncu capture (needs -lineinfo):
python scripts/ncu_lines.py <rep> [top]  -> lines by warp-stall samples and instructions executed."""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, top=30):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname = '?'
    agg = defaultdict(lambda: [0, 0, '', defaultdict(int)])
    hdr = None
    tot_s = tot_i = 0
    for r in rows:
        if r and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if not hdr or len(r) < 8 or not r[0].isdigit():
            continue
        try:
            s = int(r[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
            i = int(r[hdr.index('Instructions Executed')] or 0)
        except ValueError:
            continue
        a = agg[(fname, int(r[0]))]
        a[0] += s
        a[1] += i
        a[2] = r[1].strip()[:80]
        for k, name in enumerate(hdr):
            if name.startswith('stall_') and '(Not Issued)' not in name and r[k].isdigit():
                a[3][name[6:]] += int(r[k])
        tot_s += s
        tot_i += i
    print(f'# {rep}: {tot_s} samples, {tot_i:.3e} warp instructions')
    allst = defaultdict(int)
    for v in agg.values():
        for k, c in v[3].items():
            allst[k] += c
    tot = max(1, sum(allst.values()))
    print('# stall mix: ' + ', '.join(f'{k}={100 * c / tot:.1f}%' for k, c in sorted(allst.items(), key=lambda x: -x[1])[:8]))
    for (f, ln), (s, i, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        tops = ','.join(f'{k}={v}' for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f'{100 * s / max(1, tot_s):5.1f}% {100 * i / max(1, tot_i):5.1f}%i {f}:{ln:<5} {src:<60} {tops}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
