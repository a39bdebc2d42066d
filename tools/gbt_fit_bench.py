"""Gradient-boosting fit timing (config #3's 1M x 64 table): GPU stages vs
scikit-learn's GradientBoostingRegressor on a bounded sample.  Not the bench."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import rf_table  # noqa: E402
from paper_2305_01886_b200.boosting import GradientBoostingRegressor  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
stages = int(sys.argv[2]) if len(sys.argv) > 2 else 50
X, y = rf_table(rows)
GradientBoostingRegressor(3, random_state=0).fit(X[:5000], y[:5000])
torch.cuda.synchronize()
t0 = time.perf_counter()
m = GradientBoostingRegressor(stages, learning_rate=0.1, random_state=0).fit(X, y)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
r2 = 1 - np.mean((m.predict(X[:100000]) - y[:100000]) ** 2) / np.var(y[:100000])
print(f"gpu: {rows} rows, {stages} stages: {dt:.3f} s ({dt / stages * 1e3:.2f} ms/stage), train R2 {r2:.4f}")
from sklearn.ensemble import GradientBoostingRegressor as Sk  # noqa: E402

ns, ss = 100_000, 5
t0 = time.perf_counter()
Sk(n_estimators=ss, learning_rate=0.1, random_state=0).fit(X[:ns].astype(np.float32), y[:ns])
cs = time.perf_counter() - t0
print(f"sklearn: {ns} rows, {ss} stages: {cs:.3f} s ({cs / ss * 1e3:.1f} ms/stage, 1 core)")
