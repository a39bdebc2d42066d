"""One profiled 32-tree K5 batch for ncu (tuning aid, run on a GPU box).

    ncu --profile-from-start off ... python tools/k5_ncu.py [rows] [trees]

A warm fit first (not profiled), then cudaProfilerStart, one batch of `trees`
trees on one stream (config #3's table), cudaProfilerStop.  Launch order per
level: split kernels (small, medium, big), partition, next-level bookkeeping;
small tasks appear from level 11 on, medium from level 5 on (1M rows)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200 import forest  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
X, y = config3_table(rows)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
forest.RandomForestRegressor(2, max_depth=16, random_state=0).fit(X[:50000], y[:50000])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
forest.RandomForestRegressor(k, max_depth=16, random_state=0, trees_per_batch=k,
                             concurrent=False).fit(X, y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
