"""Instruction mix and top stall lines of the first kernel section in an ncu
`--page source --csv --print-source sass` export."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
sec = []
for r in rows[1:]:
    if r and r[0] == "Kernel Name":
        break
    sec.append(r)
hdr, data = sec[0], [r for r in sec[1:] if len(r) == len(sec[0])]
si, src, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
ops = collections.Counter()
for r in data:
    op = r[src].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    ops[o.split(".")[0]] += float(r[ie] or 0)
tot = sum(ops.values())
print(f"warp instructions executed: {tot:.0f}")
for o, c in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"  {o:10s} {c / tot * 100:5.1f}%")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("top stall instructions:")
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:12]:
    d = sorted(((h, float(r[hdr.index(h)] or 0)) for h in stalls), key=lambda x: -x[1])[:2]
    print(f"  {float(r[si] or 0):6.0f} {r[src][:56]:56s} {d}")
