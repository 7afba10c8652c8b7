#!/usr/bin/env python
"""Benchmark of the dense NNCP ALS hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

A *step* is one ALS outer iteration (all modes: dimension-tree MTTKRP, MU/HALS/
BPP update, normalisation, Grams, error) over the resident synthetic tensor.
Default workload: BASELINE.json configs[4], the north-star 3-way 2048^3
rank-32 HALS tensor (68.7 GB, larger than the 126 MB L2, so no flush is
needed between steps).  For N > 1 (torchrun) the tensor is split over the
reference's N-d grid (2x1x1 / 2x2x1 / 2x2x2), one block per GPU, NCCL
collectives; the total work is fixed (strong scaling).

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy port in oracle/, the reference being pure Python + numpy) on this host's
cores over a bounded slab of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(dims=(64, 64, 64), rank=10, algo="mu", eta=0.01, kind="uniform"),
    "c2": dict(dims=(512, 512, 512), rank=16, algo="hals", eta=0.01, kind="uniform"),
    "c3": dict(dims=(256, 256, 256, 256), rank=32, algo="bpp", eta=0.01, kind="uniform"),
    "c4": dict(dims=(4096, 2048, 256), rank=20, algo="hals", eta=0.05, kind="walk"),
    "c5": dict(dims=(2048, 2048, 2048), rank=32, algo="hals", eta=0.01, kind="uniform"),
    "c5r64": dict(dims=(2048, 2048, 2048), rank=64, algo="hals", eta=0.01, kind="uniform"),
    "c5mu": dict(dims=(2048, 2048, 2048), rank=32, algo="mu", eta=0.01, kind="uniform"),
    # the per-GPU block of c5 on the 2x2x2 grid: 1-GPU proxy for the 8-GPU strong-scaling step
    "c5blk8": dict(dims=(1024, 1024, 1024), rank=32, algo="hals", eta=0.01, kind="uniform"),
    # per-GPU blocks of c4 (2x2x2) and c3 (2x2x2x1): 1-GPU proxies for their 8-GPU steps
    "c4blk8": dict(dims=(2048, 1024, 128), rank=20, algo="hals", eta=0.05, kind="walk"),
    "c3blk8": dict(dims=(128, 128, 128, 256), rank=32, algo="bpp", eta=0.01, kind="uniform"),
}
GRIDS = {3: {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)},
         4: {1: (1, 1, 1, 1), 2: (2, 1, 1, 1), 4: (2, 2, 1, 1), 8: (2, 2, 2, 1)}}
DATA_SEED = 1
INIT_SEED = 0
METRIC = "sec per ALS outer iter + MTTKRP TFLOP/s (%roofline)"
# FP64 DMMA peak measured on this pool's B200 (profiles/r01_peaks_probe.log);
# MEASURED_PEAKS.json carries no FP64 figure.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SRC = "measured DMMA.8x8x4 microbenchmark, profiles/r01_peaks_probe.log"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback B200_PROFILING.md"


# ------------------------------------------------------------ clocks --------
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.first = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def mark(self):
        """Start of the timed region: samples from here on count.  (nvidia-smi is started
        before the warm-up: its NVML start-up inside the timed region cost up to ~2 ms per
        2048^3 step, measured.)"""
        t_end = time.perf_counter() + 3.0
        while self.proc is not None and not self.lines and time.perf_counter() < t_end:
            time.sleep(0.01)   # first sample = NVML initialised
        self.first = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines[self.first:]:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------ CPU side ------
def cpu_slab(dims, target_elems=1 << 28):
    """Leading modes kept, last mode cut so the slab holds ~2^28 elements (2 GiB)."""
    lead = math.prod(dims[:-1])
    last = max(1, min(dims[-1], target_elems // lead))
    return tuple(dims[:-1]) + (last,)


def cpu_reference_time(conf, steps, warmup):
    """Time the oracle port (numpy/OpenBLAS, all host threads) on a slab; s/iter scaled to the full tensor."""
    from oracle import nncp_oracle as O

    dims, rank = conf["dims"], conf["rank"]
    slab = cpu_slab(dims)
    rng = np.random.default_rng(DATA_SEED)
    hs = [rng.random((d, rank)) for d in slab]
    # sum of rank-one terms built slice by slice (no 2^28 x R Khatri-Rao temporary)
    lead = math.prod(slab[:-1])
    krp_lead = O.khatri_rao(hs[:-1])                     # (prod of leading dims, R)
    data = np.empty(math.prod(slab))
    for k in range(slab[-1]):
        data[k * lead:(k + 1) * lead] = krp_lead @ hs[-1][k]
    rms = float(np.sqrt(np.mean(data * data)))
    data += conf["eta"] * rms * np.abs(rng.standard_normal(data.size))
    timings = []
    O.run_sequential(data, slab, rank, conf["algo"], max_iters=warmup + steps, tol=0.0, seed=INIT_SEED,
                     timings=timings, init_error="tree")
    per_iter = timings[1 + warmup:]
    scale = math.prod(dims) / math.prod(slab)
    t = statistics.mean(per_iter) * scale
    cores = os.cpu_count()
    sample = (f"{len(per_iter)} outer iterations of the oracle port on a {'x'.join(map(str, slab))} slab "
              f"(same leading modes), s/iter scaled by I/I_slab = {scale:.1f}; init row excluded")
    return t, cores, sample


# ------------------------------------------------------------ GPU side ------
def gpu_run(args, conf):
    import torch
    import torch.distributed as dist

    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200 import _lib
    from paper_1909_01149_b200.driver import _Engine
    from paper_1909_01149_b200.grid import DistCollectives, Grid, IdentityCollectives, RankLayout
    from paper_1909_01149_b200.synth import synthetic_block, truth_factors

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # NNCP_DIST_BACKEND=gloo runs the multi-rank flow on fewer GPUs than ranks (ranks share
    # devices, host-staged collectives; for checking the path only -- timings are meaningless)
    backend = os.environ.get("NNCP_DIST_BACKEND", "nccl")
    dev = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    dims, R = conf["dims"], conf["rank"]
    grid = GRIDS[len(dims)][world]
    layout = RankLayout(Grid(grid), rank, dims)
    fs = truth_factors(dims, R, DATA_SEED, conf["kind"])
    offs = tuple(s.start for s in layout.slice_rows)
    x_local = synthetic_block(dims, fs, conf["eta"], DATA_SEED, offsets=offs, local_dims=layout.local_dims)
    coll = DistCollectives(layout) if world > 1 else IdentityCollectives()
    cfg = P.RunConfig(rank=R, algorithm=conf["algo"], max_iters=args.warmup + args.steps + 1, tol=0.0,
                      seed=INIT_SEED, cuda_graph=False if args.eager else None)
    eng = _Engine(x_local, layout.local_dims, dims, cfg, coll, layout if world > 1 else None, timing=False)
    clocks = ClockSampler(dev)
    clocks.start()
    eng.initialise()
    eng.iterate(args.warmup)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    eng.ctx.kernel_events = []
    launches0 = _lib.load().nncp_launch_count()
    replays0 = eng.graph_replays
    barrier()
    clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    eng.iterate(args.steps)
    e1.record()
    barrier()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    launches = _lib.load().nncp_launch_count() - launches0
    launches += (eng.graph_replays - replays0) * eng.graph_kernels   # kernel nodes replayed by the sweep graph
    dev_s = e0.elapsed_time(e1) / 1e3
    kev = eng.ctx.kernel_events
    if not kev:
        # graph replay records no per-kernel events: time the same kernels in 2 eager sweeps
        eng.graph, graph = None, eng.graph
        eng.cfg.cuda_graph = False
        eng.cfg.max_iters += 2
        eng.iterate(2)
        torch.cuda.synchronize()
        kev = eng.ctx.kernel_events
    eng.ctx.kernel_events = None
    k_left = [a.elapsed_time(b) / 1e3 for side, a, b in kev if side == "left"]
    k_right = [a.elapsed_time(b) / 1e3 for side, a, b in kev if side == "right"]
    t = torch.tensor([dev_s, sum(k_left), sum(k_right)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, kl_sum, kr_sum = t.tolist()
    errors = list(eng.report.errors)
    out = dict(dev_s=dev_s, wall=wall, k_left=kl_sum / max(1, len(k_left)), k_right=kr_sum / max(1, len(k_right)),
               n_left=len(k_left), n_right=len(k_right), clocks=clk, launches=int(launches), errors=errors,
               local_dims=layout.local_dims, grid=grid, world=world, rank=rank, split=eng.plan.split,
               levels=eng.sliced.levels if eng.sliced is not None else None)
    # ------------------------------------------------------- e2e leg ----------
    del eng
    try:
        host = torch.empty(x_local.numel(), dtype=torch.float64, pin_memory=True)
        out["e2e_host"] = "pinned"
    except RuntimeError:  # host cannot page-lock that much: pageable copy (slower H2D, reported)
        host = torch.empty(x_local.numel(), dtype=torch.float64)
        out["e2e_host"] = "pageable"
    host.copy_(x_local)
    del x_local
    torch.cuda.empty_cache()
    barrier()
    launches0 = _lib.load().nncp_launch_count()
    t0 = time.perf_counter()
    cfg_e2e = P.RunConfig(rank=R, algorithm=conf["algo"], max_iters=args.steps, tol=0.0, seed=INIT_SEED,
                          cuda_graph=False if args.eager else None)
    if world == 1:
        # the user's call: nncp_sequential on a host (pinned) tensor -> H2D, init, K sweeps, model D2H
        rep2 = P.nncp_sequential(P.DenseTensor(dims, host), cfg_e2e)
        model, lam = rep2.model.factors, rep2.model.lam
    else:
        xs = host.to("cuda", non_blocking=False)
        eng2, rep2 = P.run_local(xs, layout.local_dims, dims, cfg_e2e, DistCollectives(layout), layout,
                                 timing=False)
        model, lam = eng2.model_host()
        del eng2, xs
    barrier()
    e2e_wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_wall, op=dist.ReduceOp.MAX)
    out["e2e_s"] = float(e2e_wall.item())
    out["e2e_launches"] = int(_lib.load().nncp_launch_count() - launches0)
    out["h2d_bytes"] = int(host.numel() * 8)
    out["d2h_bytes"] = int(sum(m.size for m in model) * 8 + lam.size * 8 + 16 * args.steps)
    out["e2e_errors"] = list(rep2.errors)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--eager", action="store_true",
                    help="launch every kernel from the host each sweep (default: replay the sweep as a CUDA graph)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    conf = CONFIGS[args.config]
    dims, R = conf["dims"], conf["rank"]
    hbm_gbs, hbm_src = load_peaks()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    config = {"workload": f"{args.config}: {'x'.join(map(str, dims))} float64, rank {R}, {conf['algo'].upper()}, "
                          f"{conf['kind']} factors + {int(conf['eta'] * 100)}% |Gaussian| noise (BASELINE.json configs)",
              "dims": list(dims), "rank": R, "algorithm": conf["algo"],
              "grid": list(GRIDS[len(dims)][max(1, args.gpus)]) if args.gpus in GRIDS[len(dims)] else None,
              "l2": "inputs larger than L2 (tensor >> 126 MB), no flush needed",
              "data_seed": DATA_SEED, "init_seed": INIT_SEED}

    if args.impl == "reference":
        if rank != 0:
            return
        t, cores, sample = cpu_reference_time(conf, max(1, min(args.steps, 3)), 1)
        line = {"metric": METRIC, "impl": "reference", "value": t, "unit": "s/iter", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config,
                "cpu_baseline": {"value": t, "unit": "s/iter", "cores": cores, "kind": "port", "sample": sample},
                "e2e": {"value": t, "unit": "s/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    res = gpu_run(args, conf)
    if res["rank"] != 0:
        return
    s_iter = res["dev_s"] / args.steps
    size = math.prod(dims)
    dom = "left" if res["k_left"] >= res["k_right"] else "right"   # dominant (slower) partial MTTKRP
    k_dom = res["k_" + dom]
    mttkrp_s = res["k_left"] + res["k_right"]             # both partials of one sweep
    local = res["local_dims"]
    local_size = math.prod(local)
    # FP64-path roofline of the two partials: max(8 I / BW, 2 I R / P64) each
    t_fp64_roof = 2 * max(8.0 * local_size / (hbm_gbs * 1e9), 2.0 * local_size * R / (FP64_PEAK_TFLOPS * 1e12))
    L = res["levels"]
    if L is not None:
        # sliced engine: HBM-bound on the int8 digit planes
        s_ = res["split"]
        M, J = math.prod(local[:s_]), math.prod(local[s_:])
        Mp, Jp, RP = -(-M // 128) * 128, -(-J // 128) * 128, -(-R // 16) * 16
        planes = L * Mp * Jp
        kp = Jp if dom == "left" else Mp
        rows = M if dom == "left" else J
        alg = planes + L * RP * kp + rows * R * 8     # digit planes + factor digits + fp64 output
        achieved = alg / k_dom / 1e9
        t_sliced_roof = 2 * planes / (hbm_gbs * 1e9)
        roofline = {"kernel": f"sliced_gemm_kernel<{dom}> + factor-digit prep (tcgen05.mma kind::i8 over {L} int8 "
                              "digit planes of the once-sliced tensor, TMA 16 KB tiles, TMEM int32 accumulators)",
                    "bound": "hbm", "algorithmic": f"{alg:.4g} B per launch ({L} digit planes {planes:.4g} B + "
                                                   f"factor digits + fp64 output)",
                    "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs,
                    "peak_source": hbm_src + " (of measured)",
                    "peak_note": ("the peak is a device-to-device copy (half reads, half writes); this kernel's "
                                  "traffic is ~98% reads, which stream faster (read-only probe 6.87 TB/s, "
                                  "profiles/r01_peaks_probe.log; ncu shows 7.0-7.2 TB/s for the GEMMs), hence "
                                  "frac > 1")}
    else:
        t_sliced_roof = None
        bound = "tensor" if 2.0 * R / FP64_PEAK_TFLOPS / 1e12 >= 8.0 / hbm_gbs / 1e9 else "hbm"
        if bound == "tensor":
            achieved, peak, unit, psrc = 2.0 * local_size * R / k_dom / 1e12, FP64_PEAK_TFLOPS, "TFLOP/s", FP64_PEAK_SRC
        else:
            achieved, peak, unit, psrc = 8.0 * local_size / k_dom / 1e9, hbm_gbs, "GB/s", hbm_src
        roofline = {"kernel": f"mttkrp_{dom}_tma (FP64 DMMA GEMM fed by TMA, KRP on the fly)", "bound": bound,
                    "algorithmic": (f"{2 * local_size * R:.4g} flop" if bound == "tensor"
                                    else f"{8 * local_size:.4g} B") + " per launch",
                    "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak, "peak_source": psrc}
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    traffic = None
    if os.path.exists(prof):
        with open(prof) as fh:
            tr = json.load(fh)
        key = ("sliced_" if L is not None else "") + dom
        traffic = tr.get(key, {}).get("dram_bytes_per_launch")
    roofline["traffic"] = traffic
    mttkrp_tflops = 4.0 * local_size * R / mttkrp_s / 1e12 if mttkrp_s > 0 else None
    cpu = None
    if res["world"] == 1 and not args.no_cpu_baseline:
        try:
            t, cores, sample = cpu_reference_time(conf, 2, 1)
            cpu = {"value": t, "unit": "s/iter", "cores": cores, "kind": "port", "sample": sample}
        except MemoryError:
            cpu = None
    line = {
        "metric": METRIC, "value": s_iter, "unit": "s/iter", "n_gpus": res["world"], "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": s_iter * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, generated in HBM)", "config": config,
        "mttkrp_engine": f"sliced int8 tensor cores, {L} digit levels" if L is not None else "fp64 DMMA",
        "mttkrp_tflops": mttkrp_tflops,
        "mttkrp_tflops_note": "FP64-equivalent: 4 I R flop of the two partial MTTKRPs / their time",
        "mttkrp_vs_fp64_roofline": t_fp64_roof / mttkrp_s if mttkrp_s > 0 else None,
        "mttkrp_roofline_frac": (t_sliced_roof / mttkrp_s if t_sliced_roof else t_fp64_roof / mttkrp_s)
        if mttkrp_s > 0 else None,
        "partial_ms": {"left": res["k_left"] * 1e3, "right": res["k_right"] * 1e3},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": res["e2e_s"] / args.steps, "unit": "s/iter",
                "h2d_bytes_per_step": res["h2d_bytes"] // args.steps,
                "d2h_bytes_per_step": res["d2h_bytes"] // args.steps,
                "note": f"nncp_sequential(DenseTensor({res['e2e_host']} host tensor)) (N>1: per-rank block "
                        "through the engine): tensor H2D once per call of "
                        f"{args.steps} iterations + init + D2H of the model, divided by the steps"},
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "final_error": res["errors"][-1],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
