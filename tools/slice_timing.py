"""Device time of the one-off slicing passes at a BASELINE size: nncp_norm_rowmax (init
facts + row maxima), nncp_slice_tensor_planes, nncp_norm_squared_min alone.
    python tools/slice_timing.py 2048x2048x2048 [split]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1909_01149_b200 import _lib  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
split = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib = _lib.load()
x = synthetic_block(dims, truth_factors(dims, 32, 1, "uniform"), 0.01, 1)
nb = _lib.ctypes.c_size_t(0)
_lib.check(lib.nncp_sliced_tensor_bytes(len(dims), _lib.i64(dims), split, 6, _lib.ctypes.byref(nb)))
buf = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
sc = torch.zeros(4, dtype=torch.float64, device="cuda")
st = _lib.stream_handle()
calls = {
    "norm_rowmax": lambda: lib.nncp_norm_rowmax(_lib.ptr(x), len(dims), _lib.i64(dims), split, 6, _lib.ptr(buf),
                                                nb.value, _lib.ptr(sc), _lib.vp(sc.data_ptr() + 8),
                                                _lib.vp(ws.data_ptr()), ws.numel(), st),
    "slice_planes": lambda: lib.nncp_slice_tensor_planes(_lib.ptr(x), len(dims), _lib.i64(dims), split, 6,
                                                         _lib.ptr(buf), nb.value, st),
    "norm_squared_min": lambda: lib.nncp_norm_squared_min(_lib.ptr(x), x.numel(), _lib.ptr(sc),
                                                          _lib.vp(sc.data_ptr() + 8), _lib.vp(ws.data_ptr()),
                                                          ws.numel(), st),
}
for name, fn in calls.items():
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(fn())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:18s} ms: {[round(t, 2) for t in ts]}  ({8 * x.numel() / min(ts) / 1e6:.0f} GB/s of fp64 reads)")
