"""Run-to-run spread of the 500-tree config #3 fit (tuning aid): bench.py's
sequence (warm 128-tree fit, then timed fits, each model freed before the
next), with per-fit wall times and the caching allocator's cudaMalloc count.

    python tools/rf_fit_var.py [fits]"""
import gc
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.forest import RandomForestRegressor as M  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
X, y = config3_table(1_000_000)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
torch.cuda.empty_cache()
m = M(128, max_depth=16, random_state=0).fit(X, y)
del m
torch.cuda.synchronize()
for i in range(n):
    gc.collect()
    s0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    m = M(500, max_depth=16, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s1 = torch.cuda.memory_stats()
    print(f"fit {i}: {dt:.3f} s  cudaMalloc {s1['num_alloc_retries'] - s0['num_alloc_retries']} retries, "
          f"segments +{s1['segment.all.allocated'] - s0['segment.all.allocated']}, "
          f"reserved {s1['reserved_bytes.all.current'] / 2**30:.1f} GiB", flush=True)
    del m
