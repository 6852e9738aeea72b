"""Summarise an ncu report: key metrics per kernel (reads `ncu -i --page raw --csv`)."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.per_cycle_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__registers_per_thread',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'smsp__inst_executed_op_global_red.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'lts__t_requests_srcunit_tex_op_red.sum']
STALL = 'smsp__average_warps_issue_stalled_'


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[h.index('Kernel Name')].split('(')[0]
        print('===', name)
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f'  {w:62s} {row[i]:>16s} {units[i]}')
        st = []
        for i, w in enumerate(h):
            if w.startswith(STALL) and w.endswith('_per_issue_active.ratio'):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.1:
                    st.append((v, w[len(STALL):-len('_per_issue_active.ratio')]))
        print('  stalls/issue:', ', '.join(f'{n}={v:.2f}' for v, n in sorted(st, reverse=True)))


if __name__ == '__main__':
    main(sys.argv[1])
