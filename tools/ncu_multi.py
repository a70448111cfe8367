"""Per-launch summary of a multi-kernel ncu report (raw page): duration, DRAM
bytes, occupancy, issue activity, pipe use and the top stall reasons.

    python tools/ncu_multi.py report.ncu-rep > summary.txt
    python tools/ncu_multi.py report_raw.csv > summary.txt   (ncu -i ... --page raw --csv)
"""
import csv
import io
import re
import subprocess
import sys

COLS = [
    ("dur_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("occ_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("l2_hit", "lts__t_sector_hit_rate.pct", 1),
    ("fp64_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
]
UNIT = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
        "GB": 1e9}


def main(path):
    if path.endswith(".csv"):          # an exported raw page
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    idx = {k: i for i, k in enumerate(h)}
    name_i = idx.get("Kernel Name")
    stall = [(k, i) for k, i in idx.items()
             if re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active\.ratio$", k)]
    print("kernel".ljust(44) + " ".join(c[0].rjust(10) for c in COLS) + "  top stalls (per issue)")
    for r in data:
        cells = []
        for label, key, scale in COLS:
            i = idx.get(key)
            if i is None or not r[i]:
                cells.append("-".rjust(10))
                continue
            v = float(r[i].replace(",", ""))
            v *= UNIT.get(units[i], 1)
            cells.append(f"{v * scale:10.2f}" if label not in ("regs", "grid", "block")
                         else f"{int(v):10d}")
        st = []
        for k, i in stall:
            try:
                st.append((float(r[i]), re.sub(r"smsp__average_warps_issue_stalled_|_per_issue_active\.ratio", "", k)))
            except ValueError:
                pass
        st.sort(reverse=True)
        top = ", ".join(f"{n} {v:.2f}" for v, n in st[:4] if n not in ("selected",))
        nm = re.sub(r"\(.*", "", r[name_i]).replace("void ", "").replace("(anonymous namespace)::", "")
        print(nm[:43].ljust(44) + " ".join(cells) + "  " + top)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
