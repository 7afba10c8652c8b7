"""Static SASS opcode histogram of the hot kernels in libnncp_b200.so (cuobjdump -sass):
the evidence that the partial MTTKRPs run on tcgen05 (UTCIMMA / UTCHMMA = tcgen05.mma,
LDTM = tcgen05.ld, UTMALDG / UTMASTG = TMA) or DMMA, per kernel.

    python tools/sass_static.py [lib] > profiles/r02_sass_histogram.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1909_01149_b200", "libnncp_b200.so")
HOT = ("sliced_gemm_kernel", "mttkrp_left_tma", "mttkrp_right_tma", "bslice_digits", "bseg_digits", "slice_planes",
       "ttv_trailing", "ttv_leading", "update_rows_kernel", "bpp_kernel", "normalize_gram_kernel")
KEY = ("UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "DMMA", "DFMA",
       "HMMA", "IMMA", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "BAR")

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
func, counts = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        counts[func] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and func:
        counts[func][m.group(2)] += 1
print(f"# static SASS opcode counts, {os.path.basename(LIB)} (cuobjdump -sass); one line per hot kernel instance")
print("# kernel | " + " ".join(KEY))
for f, c in sorted(counts.items()):
    if not any(h in f for h in HOT):
        continue
    name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()[:110]
    print(f"{name}\n    " + " ".join(f"{k}={c.get(k, 0)}" for k in KEY if c.get(k, 0)) + f"  (total {sum(c.values())})")
