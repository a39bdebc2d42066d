"""Host-side profile (cProfile) of a 100-stage boosting fit at 1M x 64 (tuning aid)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.boosting import GradientBoostingRegressor as G  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

X, y = config3_table(1_000_000)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
G(5, max_depth=3, random_state=0).fit(X, y)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    G(100, max_depth=3, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    print(f"fit {time.perf_counter() - t0:.3f} s")
pr = cProfile.Profile()
pr.enable()
G(100, max_depth=3, random_state=0).fit(X, y)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
