"""Where does the chunked host sweep spend its time?  Times each chunk's device
sweep alone, the copies alone, and the pipelined run.  Tuning aid."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_workload, make_ensembles  # noqa: E402
from paper_2305_01886_b200 import runtime as rt  # noqa: E402


class A:
    workload, kernels, trees, depth = "c2", 0, 500, 16


W = build_workload(A, 0)
dc = rt.DeviceCorpus.upload(W["corpus"])
dg = rt.DeviceGrid.build(dc, W["profiles"], W["configs"])
ens = [rt.DeviceEnsemble.upload(f) for f in make_ensembles(W, dc, dg, rt, 500, 16)]


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n, (time.perf_counter() - t0) / n * 1e3


full = rt.Sweep(dc, dg, ens, W["sel"])
print("full sweep (device, ms gpu / host):", timed(full.run))
for nc in (1, 4, 8):
    hs = rt.HostSweep(W["corpus"], W["profiles"], W["configs"], ens, W["sel"], n_chunks=nc)
    per = [timed(c["sweep"].run) for c in hs.chunks]
    print(f"{nc} chunks: sum of chunk sweeps {sum(p[0] for p in per):.3f} ms (host {sum(p[1] for p in per):.3f}),"
          f" each {[round(p[0], 3) for p in per]}")
    print(f"   pipelined run: {timed(hs.run)}")
