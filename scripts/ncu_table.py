"""Markdown table of per-kernel ncu counters (duration, DRAM traffic and rate,
L2 / L1 hit rate, warp execution efficiency, issue activity, occupancy):
python scripts/ncu_table.py <rep>...  (first capture of each kernel name wins)."""
import csv
import subprocess
import sys

W = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
     'l1tex__t_sector_hit_rate.pct', 'smsp__thread_inst_executed_per_inst_executed.ratio',
     'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active']
TSCALE = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
BSCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9, 'B': 1}


def main(reps):
    seen, out = set(), []
    for rep in reps:
        rows = list(csv.reader(subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                                              text=True).stdout.splitlines()))
        h, u = rows[0], rows[1]
        for v in rows[2:]:
            name = v[h.index('Kernel Name')].split('(')[0].replace('gl::<unnamed>::', '').replace('void ', '')
            if name in seen:
                continue
            seen.add(name)
            val = {w: float(v[h.index(w)].replace(',', '')) for w in W}
            ms = val[W[0]] * TSCALE[u[h.index(W[0])]]
            gb = (val[W[1]] + val[W[2]]) * BSCALE[u[h.index(W[1])]] / 1e9
            out.append((name, ms, gb, gb / (ms * 1e-3), val[W[3]], val[W[4]], val[W[5]] / 32 * 100, val[W[6]], val[W[7]]))
    print('| kernel | ms | DRAM GB | DRAM GB/s | L2 hit % | L1 hit % | warp exec eff % | issue active % | warps active % |')
    print('|---|---|---|---|---|---|---|---|---|')
    for r in out:
        print(f'| `{r[0]}` | {r[1]:.2f} | {r[2]:.2f} | {r[3]:.0f} | {r[4]:.1f} | {r[5]:.1f} | {r[6]:.1f} | {r[7]:.1f} | {r[8]:.1f} |')


if __name__ == '__main__':
    main(sys.argv[1:])
