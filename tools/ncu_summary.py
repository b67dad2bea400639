"""Summarise an ncu --set full report (raw page) for the kernels in it."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts.avg', 'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sectors.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']


def main(rep):
    if rep.endswith('.csv'):                 # raw page exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                             text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    i0 = next(i for i, row in enumerate(r) if row and row[0] == 'ID')
    h, units, rows = r[i0], r[i0 + 1], r[i0 + 2:]
    ki = h.index('Kernel Name')
    for row in rows:
        print('==', row[ki][:90])
        for k in KEYS:
            idx = [j for j, n in enumerate(h) if n == k or n.endswith('.' + k)]
            if idx:
                i = idx[0]
                print(f"   {k:72s} {row[i]:>20s} {units[i]}")
        stalls = [(float(row[i] or 0), n) for i, n in enumerate(h)
                  if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued')]
        tot = sum(v for v, _ in stalls) or 1
        top = sorted(stalls, reverse=True)[:6]
        print('   stalls:', ', '.join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                      f"{100 * v / tot:.0f}%" for v, n in top))


if __name__ == '__main__':
    main(sys.argv[1])
