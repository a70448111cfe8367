"""Summarise an ncu report (details page) into a few key metrics."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Compute (SM) Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'DRAM Throughput', 'Issue Slots Busy', 'Warp Cycles Per Issued Instruction',
        'Executed Ipc Active', 'Dynamic Shared Memory Per Block', 'Static Shared Memory Per Block']


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    mi, vi, ui, ki = (h.index(k) for k in ('Metric Name', 'Metric Value', 'Metric Unit',
                                            'Kernel Name'))
    lines = [rows[1][ki][:100]]
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and r[mi] + r[ui] not in seen:
            seen.add(r[mi] + r[ui])
            lines.append(f"  {r[mi]}: {r[vi]} {r[ui]}")
    return "\n".join(lines)


def raw(path, pattern):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    import re
    return "\n".join(f"  {a} = {c} {b}" for a, b, c in zip(h, u, v) if re.search(pattern, a))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
        print(raw(p, r'dram__bytes_(read|write)\.sum$|sm__inst_executed_pipe_fp64|sm__pipe_fp64_cycles_active|smsp__average_warp|stall'))
