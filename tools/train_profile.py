"""Where the reference-shaped train() spends its time at config #3 (tuning aid):
canonical rows, per-fold scaler / fit / predict, the final fit.

    python tools/train_profile.py [rows] [trees]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402
import sklearn.metrics  # noqa: E402,F401  (the reference imports these at module import)
import sklearn.model_selection  # noqa: E402,F401
import sklearn.preprocessing  # noqa: E402,F401
import torch  # noqa: E402

from paper_2305_01886_b200 import trainer as T  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
trees = int(sys.argv[2]) if len(sys.argv) > 2 else 500
X, y = config3_table(rows)
names = tuple(f"f{i:02d}" for i in range(64))
marks = []
orig_fit = T._make_model


def timed_model(*a, **k):
    m = orig_fit(*a, **k)
    f, p = m.fit, m.predict

    def fit(*aa, **kk):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*aa, **kk)
        torch.cuda.synchronize()
        marks.append(("fit", time.perf_counter() - t0))
        return r

    def predict(*aa, **kk):
        t0 = time.perf_counter()
        r = p(*aa, **kk)
        marks.append(("predict", time.perf_counter() - t0))
        return r

    m.fit, m.predict = fit, predict
    return m


T._make_model = timed_model
t0 = time.perf_counter()
Xc, yc = T.canonical_rows(X, y, names)
t_can = time.perf_counter() - t0
t0 = time.perf_counter()
res = T.train((X, y, names), "random_forest", n_estimators=trees, max_depth=16, seed=0)
torch.cuda.synchronize()
tt = time.perf_counter() - t0
fit = sum(v for k, v in marks if k == "fit")
pred = sum(v for k, v in marks if k == "predict")
print(f"train {tt:.2f} s: canonical rows {t_can:.2f} s, {sum(k == 'fit' for k, _ in marks)} fits "
      f"{fit:.2f} s ({[round(v, 2) for k, v in marks if k == 'fit']}), predicts {pred:.2f} s, "
      f"other {tt - fit - pred - t_can:.2f} s; cv r2 {res.mean_metrics.r2:.5f}")
