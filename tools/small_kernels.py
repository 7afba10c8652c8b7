"""Warm, graph-replayed time per launch of the per-mode small kernels at a given
(rows, rank): status reset, HALS/MU/BPP update, normalise+Gram, temp->rows, gamma.

    python tools/small_kernels.py 2048 32
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1909_01149_b200 import _lib  # noqa: E402
from paper_1909_01149_b200.tensor_ops import Workspace  # noqa: E402

rows, R = int(sys.argv[1]), int(sys.argv[2])
N = 3
lib = _lib.load()
dev = torch.device("cuda", 0)
f64 = dict(dtype=torch.float64, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
h = [torch.rand((rows, R), generator=g, **f64) for _ in range(N)]
grams = torch.stack([x.T @ x for x in h]).contiguous()
mrows = torch.rand((rows, R), generator=g, **f64) * rows
lam = torch.ones(R, **f64)
hhat = torch.empty((rows, R), **f64)
nsq = torch.empty(R, **f64)
scal = torch.zeros(5, **f64)
status = torch.zeros((N, _lib.STATUS_WORDS), dtype=torch.int32, device=dev)
ws = Workspace(64 << 20)
owned = h[0].clone()
out_g = torch.empty((R, R), **f64)


def st():
    return _lib.stream_handle()


def k_status():
    _lib.check(lib.nncp_status_reset(_lib.ptr(status[0]), st()))


def k_update(algo):
    code = _lib.ALGO_CODES[algo]

    def f():
        _lib.check(lib.nncp_update(code, _lib.ptr(grams), N, 0, R, _lib.ptr(mrows), _lib.ptr(owned), _lib.ptr(lam),
                                   rows, _lib.ptr(hhat), _lib.ptr(nsq), _lib.ptr(scal), _lib.ptr(status[0]), ws.ptr,
                                   ws.nbytes, st()))
    return f


def k_normgram():
    _lib.check(lib.nncp_normalize_gram(_lib.ptr(hhat), _lib.ptr(nsq), rows, R, _lib.ptr(owned), _lib.ptr(lam),
                                       _lib.ptr(out_g), ws.ptr, ws.nbytes, st()))


def k_rows():
    _lib.check(lib.nncp_temp_to_rows(_lib.ptr(mrows), rows, R, _lib.ptr(hhat), st()))


def k_gamma():
    _lib.check(lib.nncp_gamma(_lib.ptr(grams), N, R, _lib.ptr(lam), _lib.vp(scal.data_ptr() + 8), st()))


def timed(name, fn, reps=50):
    # prime (and normalise once so the update sees sane data)
    k_update("hals")()
    k_normgram()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) * 1e3 / (5 * reps):8.2f} us/launch", flush=True)


timed("status_reset", k_status)
timed("update hals", k_update("hals"))
timed("update mu", k_update("mu"))
timed("update bpp", k_update("bpp"))
timed("normalize_gram", k_normgram)
timed("temp_to_rows", k_rows)
timed("gamma", k_gamma)
timed("update hals + normalize_gram", lambda: (k_update("hals")(), k_normgram()))
