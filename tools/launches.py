"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``).

Usage: python tools/launches.py launches.csv [first_kernel_regex]

Takes the LAST complete evaluation in the capture (from the last launch of
``k_bbox``, the first kernel of an evaluation) and prints per-kernel totals
and shares.  ncu serialises launches and runs them cold, so compare shares,
not absolute times.
"""
import collections
import csv
import io
import re
import sys


def load(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    return [(r["Kernel Name"], float(r["Metric Value"])) for r in rows
            if r["Metric Name"] == "gpu__time_duration.sum"]


def short(name):
    m = re.search(r"(k_\w+|cub::\w+)", name)
    base = m.group(1) if m else name[:40]
    t = re.search(r"<(\d+)>", name)
    return base + (f"<{t.group(1)}>" if t and base.startswith("k_") else "")


def main():
    path = sys.argv[1]
    first = sys.argv[2] if len(sys.argv) > 2 else "k_bbox"
    launches = load(path)
    starts = [i for i, (n, _) in enumerate(launches) if re.search(first, n)]
    seg = launches[starts[-2]:starts[-1]] if len(starts) > 1 else launches[starts[-1]:]
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for n, v in seg:
        k = short(n)
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] += 1
    total = sum(tot.values())
    print(f"{len(seg)} launches, {total / 1e3:.1f} us total (serialised, cold)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {k:40s} x{cnt[k]:3d} {v / 1e3:9.1f} us  {100 * v / total:5.1f}%")


if __name__ == "__main__":
    main()
