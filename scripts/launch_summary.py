"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel totals per step."""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    n = r[ki]
    n = n.split("(")[0][:60] if not n.startswith("void") else n[5:].split("(")[0][:60]
    agg[n][0] += 1
    agg[n][1] += v
    seq.append((n, v))
if "--period" in sys.argv:
    # exactly one step: the launches between two consecutive occurrences of an anchor kernel that
    # runs once per step (a step is periodic, so any such window is one whole step)
    anchor = sys.argv[sys.argv.index("--period") + 1]
    idx = [i for i, (n, _) in enumerate(seq) if anchor in n]
    seq = seq[idx[0]:idx[1]]
    steps = 1.0
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in seq:
        agg[n][0] += 1
        agg[n][1] += v
tot = sum(v for _, v in agg.values())
print(f"total {tot / 1e3 / steps:.1f} us/step over {len(seq)} launches ({steps} steps)")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c / steps:6.1f} x {v / 1e3 / steps:9.1f} us/step {100 * v / tot:5.1f}%  {n}")
if "--seq" in sys.argv:
    for n, v in seq:
        print(f"{v / 1e3:9.1f}  {n}")
