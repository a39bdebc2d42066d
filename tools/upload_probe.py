"""Host -> device upload of a pageable 1M x 64 fp64 table (tuning aid):
pageable .to() vs chunked staging through pinned buffers (torch's CPU copy_
is multi-threaded) with the DMA of one chunk overlapping the next chunk's
host copy."""
import time

import numpy as np
import torch

X = np.random.default_rng(0).random((1_000_000, 64))
dev = torch.device("cuda")
torch.zeros(1, device=dev)


def pageable():
    return torch.from_numpy(X).to(dev)


def staged(chunk_mb=32, nbuf=3):
    flat = torch.from_numpy(X).view(-1)
    out = torch.empty(flat.numel(), dtype=torch.float64, device=dev)
    ce = chunk_mb * (1 << 20) // 8
    bufs = [torch.empty(ce, dtype=torch.float64, pin_memory=True) for _ in range(nbuf)]
    evs = [None] * nbuf
    st = torch.cuda.Stream()
    for i, o in enumerate(range(0, flat.numel(), ce)):
        k = i % nbuf
        if evs[k] is not None:
            evs[k].synchronize()
        c = min(ce, flat.numel() - o)
        bufs[k][:c].copy_(flat[o:o + c])
        with torch.cuda.stream(st):
            out[o:o + c].copy_(bufs[k][:c], non_blocking=True)
            evs[k] = torch.cuda.Event()
            evs[k].record(st)
    st.synchronize()
    return out.view(X.shape)


for name, f in (("pageable", pageable), ("staged32x3", staged),
                ("staged8x4", lambda: staged(8, 4)), ("staged64x2", lambda: staged(64, 2))):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        y = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    assert torch.equal(y.cpu(), torch.from_numpy(X))
    print(f"{name:12s} {min(ts) * 1e3:7.1f} ms  {X.nbytes / min(ts) / 1e9:6.1f} GB/s  threads {torch.get_num_threads()}")
