"""Where does a forest fit's wall time go (host bookkeeping vs device waits)?
cProfile of a serial fit (one batch stream).  Tuning aid.

    python tools/rf_host_probe.py [rows] [trees]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from bench import rf_table  # noqa: E402
from paper_2305_01886_b200.forest import RandomForestRegressor as M  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
X, y = rf_table(rows)
M(4, max_depth=16, random_state=0).fit(X, y)
for conc in (True, False):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M(k, max_depth=16, random_state=0, concurrent=conc).fit(X, y)
    torch.cuda.synchronize()
    print(f"concurrent={conc}: {time.perf_counter() - t0:.3f} s for {k} trees")
pr = cProfile.Profile()
pr.enable()
M(k, max_depth=16, random_state=0, concurrent=False).fit(X, y)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
