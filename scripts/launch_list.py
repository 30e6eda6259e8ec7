"""Per-launch device times from `ncu --metrics gpu__time_duration.sum --csv --log-file X`:
the sequence, and totals per kernel name (cold-cache, serialised: compare shares)."""
import csv
import sys
from collections import defaultdict


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    return [(r[ki], float(r[vi].replace(",", "")) / 1000.0, r[gi]) for r in rows[1:]]


if __name__ == "__main__":
    seq = load(sys.argv[1])
    if "--seq" in sys.argv:
        for i, (k, us, g) in enumerate(seq):
            print(f"{i:4d} {us:9.1f} us  grid {g:14s} {k[:100]}")
    tot = defaultdict(lambda: [0, 0.0])
    for k, us, g in seq:
        name = k.split("(")[0]
        tot[name][0] += 1
        tot[name][1] += us
    all_us = sum(v[1] for v in tot.values())
    print(f"total {all_us:.1f} us over {len(seq)} launches")
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{us:9.1f} us {100 * us / all_us:5.1f}%  {n:4d}x  {k[:90]}")
