"""Summarise ncu captures: python scripts/ncu_summary.py <rep>... (run where ncu exists)."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'sm__maximum_warps_per_active_cycle_pct',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_sectors_op_red.sum', 'lts__t_sectors_op_atom.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__grid_size', 'launch__block_size']
STALLS = 'smsp__average_warp_latency_issue_stalled_'


def summarize(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for w in WANT:
            if w in h:
                i = h.index(w)
                d[w] = (v[i], u[i])
        st = []
        for i, name in enumerate(h):
            if name.startswith('smsp__average_warp_latency_issue_stalled_') and name.endswith('.ratio'):
                try:
                    st.append((float(v[i]), name[len(STALLS):-6]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        d['top_stalls'] = st[:6]
        d['kernel'] = v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        res.append(d)
    return res


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        for d in summarize(rep):
            print('==', rep, d.pop('kernel')[:60])
            for k, (val, unit) in [(k, v) for k, v in d.items() if k != 'top_stalls']:
                print(f'  {k} = {val} {unit}')
            print('  top stalls (cycles/instr):', ', '.join(f'{n}={x:.1f}' for x, n in d['top_stalls']))
