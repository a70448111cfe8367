"""Key counters of every kernel in an ncu --set full report.
Usage: python tools/ncu_kernel.py report.ncu-rep"""
import csv, io, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed.avg.per_cycle_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
for r in rows[2:]:
    print(r[h.index('Kernel Name')].split('(')[0])
    for k in KEYS:
        if k in h:
            print(f"  {k} = {r[h.index(k)]} {u[h.index(k)]}")
    st = [(float(r[i] or 0), c.replace('smsp__pcsamp_warps_issue_stalled_', '')) for i, c in enumerate(h)
          if c.startswith('smsp__pcsamp_warps_issue_stalled') and not c.endswith('not_issued')]
    print('  stalls:', ', '.join(f"{c}={v:.0f}" for v, c in sorted(st, reverse=True)[:6]))
