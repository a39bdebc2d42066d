"""Host-side profile (cProfile) of the reference-shaped train() at config #3
(tuning aid): a warm train first, then a profiled one.

    python tools/train_cprofile.py [rows] [trees]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import sklearn.metrics  # noqa: E402,F401
import sklearn.model_selection  # noqa: E402,F401
import sklearn.preprocessing  # noqa: E402,F401
import torch  # noqa: E402

from paper_2305_01886_b200 import trainer as T  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
trees = int(sys.argv[2]) if len(sys.argv) > 2 else 500
X, y = config3_table(rows)
names = tuple(f"f{i:02d}" for i in range(64))
t0 = time.perf_counter()
T.train((X, y, names), "random_forest", n_estimators=trees, max_depth=16, seed=0)
torch.cuda.synchronize()
print(f"warm train {time.perf_counter() - t0:.2f} s")
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
T.train((X, y, names), "random_forest", n_estimators=trees, max_depth=16, seed=0)
torch.cuda.synchronize()
pr.disable()
print(f"profiled train {time.perf_counter() - t0:.2f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_callers("method 'to' of")
st.print_callers("method 'cpu' of")
