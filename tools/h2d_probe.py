import time, torch, numpy as np
n = 1 << 30  # 8 GiB of float64
a = np.empty(n); a[:] = 1.0
t = torch.from_numpy(a)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); d = t.to('cuda'); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"pageable .to(cuda): {8*n/(t1-t0)/1e9:.1f} GB/s"); del d
def staged(t, chunk_bytes):
    out = torch.empty(t.numel(), dtype=t.dtype, device='cuda')
    chunk = chunk_bytes // 8
    bufs = [torch.empty(chunk, dtype=t.dtype).pin_memory() for _ in range(2)]
    evs = [None, None]; s = torch.cuda.current_stream()
    for i, st in enumerate(range(0, t.numel(), chunk)):
        b = i % 2
        if evs[b] is not None: evs[b].synchronize()
        m = min(chunk, t.numel() - st)
        bufs[b][:m].copy_(t[st:st + m])
        out[st:st + m].copy_(bufs[b][:m], non_blocking=True)
        evs[b] = torch.cuda.Event(); evs[b].record(s)
    s.synchronize()
    return out
for cb in (64 << 20, 256 << 20):
    for rep in range(2):
        t0 = time.perf_counter(); d = staged(t, cb); t1 = time.perf_counter()
        print(f"staged {cb>>20} MiB: {8*n/(t1-t0)/1e9:.1f} GB/s"); del d
p = torch.empty(n).pin_memory(); p.copy_(t)
for rep in range(2):
    t0 = time.perf_counter(); d = p.to('cuda', non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"pinned .to(cuda): {8*n/(t1-t0)/1e9:.1f} GB/s"); del d
print("torch threads", torch.get_num_threads())
