"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
python scripts/launch_summary.py gpurun_out/launches_<tag>.csv  -> per-kernel totals and shares."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[start]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    tot_ns, cnt, tot = defaultdict(float), defaultdict(int), 0.0
    scale = {'nsecond': 1.0, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
        name = r[ki].split('(')[0]
        tot_ns[name] += v
        cnt[name] += 1
        tot += v
    print(f"# {path}: {sum(cnt.values())} launches, {tot / 1e6:.3f} ms total (cold-cache, serialised)")
    print(f"{'ms':>10} {'n':>4} {'share':>6}  kernel")
    for k, v in sorted(tot_ns.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:10.3f} {cnt[k]:4d} {100 * v / tot:5.1f}%  {k}")


if __name__ == '__main__':
    for p in sys.argv[1:]:
        main(p)
