"""Summarise an .ncu-rep: key throughput metrics + warp stall reasons."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__inst_executed.avg.per_cycle_active', 'sm__inst_executed.sum', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum',
        'sm__cycles_elapsed.avg.per_second', 'launch__grid_size', 'launch__block_size',
        'launch__occupancy_limit_registers', 'launch__shared_mem_per_block_dynamic']


def main(path, kfilter=None):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')]
        if kfilter and kfilter not in name:
            continue
        print('==', name[:110])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f'  {k:62s} {vals[i]:>18s} {units[i]}')
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
                try:
                    st.append((float(vals[i]), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print('  stalls:', ', '.join(f'{n} {v / tot:.0%}' for v, n in sorted(st, reverse=True)[:8]))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
