"""Summarise an ncu report (raw page CSV) for the kernels in it: key throughput metrics and the
top warp-stall reasons.  Usage: python tools_ncu_summary.py report.ncu-rep"""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__grid_size', 'launch__block_size', 'launch__cluster_dim_x' ,
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        print('-----', d[hdr.index('Kernel Name')][:70])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f'  {w:60s} {d[i]} {units[i]}')
        st = [(hdr[i], d[i]) for i in range(len(hdr))
              if hdr[i].startswith('smsp__average_warps_issue_stalled_') and hdr[i].endswith('_per_issue_active.ratio')]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:7]
        print('  stalls/issue:', ', '.join(f"{a.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(b):.2f}" for a, b in st))


if __name__ == '__main__':
    main(sys.argv[1])
