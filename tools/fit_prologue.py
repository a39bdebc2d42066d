"""Time a forest fit's fixed costs (upload, checks, binning, fixed point):
fit(1 tree, depth 1) on config #3's 1M x 64 table, repeated.  Tuning aid."""
import sys
import time
from pathlib import Path

ROOT = Path(sys.argv[1] if len(sys.argv) > 1 else Path(__file__).resolve().parents[1])
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.forest import RandomForestRegressor  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

X, y = config3_table(1_000_000)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
ts = []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    RandomForestRegressor(1, max_depth=1, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(ROOT.name, "fit(1 tree, depth 1) s:", [round(t, 3) for t in ts])
