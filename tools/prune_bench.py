"""Correlation pruning timing: GPU Pearson / Kendall matrices on an n x K
table vs pandas DataFrame.corr on a bounded sample.  Not the bench."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402
import pandas as pd  # noqa: E402
import torch  # noqa: E402

from bench import rf_table  # noqa: E402
from paper_2305_01886_b200.pruning import kendall_matrix, pearson_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
X, _ = rf_table(n)
X = X[:, :K]
kendall_matrix(X[:5000])
torch.cuda.synchronize()
t0 = time.perf_counter()
P = pearson_matrix(X)
t1 = time.perf_counter()
T = kendall_matrix(X)
t2 = time.perf_counter()
print(f"gpu {n} x {K}: pearson {t1 - t0:.3f} s, kendall {t2 - t1:.3f} s ({K * (K - 1) // 2} pairs)")
ns, ks = 100_000, 6
df = pd.DataFrame(X[:ns, :ks])
t0 = time.perf_counter()
ref = df.corr("kendall").to_numpy()
t1 = time.perf_counter()
pairs = ks * (ks - 1) // 2
print(f"pandas kendall {ns} x {ks}: {t1 - t0:.3f} s ({(t1 - t0) / pairs:.3f} s/pair; "
      f"{n} rows x {K * (K - 1) // 2} pairs extrapolates to "
      f"{(t1 - t0) / pairs * (n / ns) * np.log2(n) / np.log2(ns) * K * (K - 1) / 2:.0f} s)")
got = kendall_matrix(X[:ns, :ks])
print("bit-identical on the sample:", np.array_equal(got.view(np.uint64), ref.view(np.uint64)))
