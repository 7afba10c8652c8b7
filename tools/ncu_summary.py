"""Per-launch summary of an ncu report (JSON): duration, DRAM bytes, achieved TB/s,
tensor-pipe activity, registers, grid.  python tools/ncu_summary.py rep.ncu-rep [key ...]"""
import csv
import io
import json
import subprocess
import sys


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = dict(zip(hdr, r))

        def num(name, scale=1.0):
            v = d.get(name, "")
            try:
                return float(v.replace(",", "")) * scale
            except ValueError:
                return None

        unit = dict(zip(hdr, units))
        dur = num("gpu__time_duration.sum")
        if dur is not None and unit.get("gpu__time_duration.sum") in ("nsecond", "ns"):
            dur /= 1e6
        elif dur is not None and unit.get("gpu__time_duration.sum") in ("usecond", "us"):
            dur /= 1e3
        rd = num("dram__bytes_read.sum")
        wr = num("dram__bytes_write.sum")
        for nm, val in (("dram__bytes_read.sum", rd), ("dram__bytes_write.sum", wr)):
            u = unit.get(nm, "byte")
            if val is not None and u != "byte":
                scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1.0)
                if nm.endswith("read.sum"):
                    rd = val * scale
                else:
                    wr = val * scale
        tensor = None
        for k in hdr:
            if k.startswith("sm__pipe_tensor") and k.endswith("pct_of_peak_sustained_active"):
                tensor = num(k)
                break
        res.append({"kernel": d.get("Kernel Name", "")[:120], "duration_ms": dur, "dram_read_bytes": rd,
                    "dram_write_bytes": wr,
                    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
                    "dram_TBps": ((rd or 0) + (wr or 0)) / (dur * 1e-3) / 1e12 if dur else None,
                    "tensor_pipe_active_pct": tensor,
                    "registers": num("launch__registers_per_thread"), "grid": num("launch__grid_size"),
                    "block": num("launch__block_size")})
    return res


if __name__ == "__main__":
    res = metrics(sys.argv[1])
    keys = sys.argv[2:]
    out = {(keys[i] if i < len(keys) else f"launch{i}"): r for i, r in enumerate(res)}
    print(json.dumps(out, indent=1))
