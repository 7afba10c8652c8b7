"""Is the 2048^3 sliced partial power-bound?  Times the left partial back to back, with a
host sync between calls, and with short idle gaps, sampling SM clock and board power
(NVML, 20 ms) in each phase.

    python tools/power_probe.py [2048x2048x2048] [32]
"""
import os
import sys
import threading
import time

import numpy as np
import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.dimtree import SlicedTensor  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402
from paper_1909_01149_b200.tensor_ops import Workspace  # noqa: E402

dims = tuple(int(d) for d in (sys.argv[1] if len(sys.argv) > 1 else "2048x2048x2048").split("x"))
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
fs = truth_factors(dims, R, 1, "uniform")
x = synthetic_block(dims, fs, 0.01, 1)
plan = P.DimTreePlan.create(dims, R)
sl = SlicedTensor(x, dims, plan.split, 6)
ws = Workspace(plan.sliced_workspace_bytes(6))
hs = [torch.from_numpy(f).cuda() for f in fs]
out = torch.empty(int(np.prod(dims[:plan.split])) * R, dtype=torch.float64, device="cuda")

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, on = [], [False]


def sampler():
    while on[0]:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
        time.sleep(0.02)


def call():
    P.partial_mttkrp(x, hs, "left", plan, out=out, workspace=ws, sliced=sl)


def phase(name, n, gap_s=None, sync=False):
    samples.clear()
    on[0] = True
    t = threading.Thread(target=sampler, daemon=True)
    t.start()
    evs = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        evs.append((a, b))
        if sync or gap_s is not None:
            torch.cuda.synchronize()
        if gap_s:
            time.sleep(gap_s)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    on[0] = False
    t.join()
    ks = [a.elapsed_time(b) for a, b in evs]
    sm = [s[0] for s in samples]
    mem = [s[1] for s in samples]
    pw = [s[2] for s in samples]
    print(f"{name:22s} kernel median {np.median(ks):.3f} ms (min {min(ks):.3f} max {max(ks):.3f}) "
          f"wall/call {1e3 * wall / n:.3f} ms | SM MHz median {np.median(sm):.0f} (min {min(sm)}) "
          f"mem MHz {np.median(mem):.0f} | power median {np.median(pw):.0f} W max {max(pw):.0f}", flush=True)


call()
torch.cuda.synchronize()
for rep in range(2):
    phase("back-to-back", 60)
    phase("sync between", 60, sync=True)
    phase("gap 0.2 ms", 60, gap_s=0.0002)
    phase("gap 1 ms", 60, gap_s=0.001)
