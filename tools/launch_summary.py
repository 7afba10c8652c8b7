"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (last N launches)."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
data = []
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("ns", "nsecond") else v * 1e3 if r[ui] in ("ms", "msecond") else v
    data.append((r[ki].split("(")[0][:70], v))
print(f"{len(data)} launches")
sel = data[-last:] if last else data
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in sel:
    agg[n][0] += 1
    agg[n][1] += v
tot = 0.0
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    tot += t
    print(f"{t / div:10.2f} us  x{c:<4d} {n}")
print(f"{tot / div:10.2f} us total")
