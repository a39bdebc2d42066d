"""Per-level, per-class device time of the K5 split search (tuning aid).

    python tools/k5_levels.py [rows] [trees]

One batch of `trees` trees (serial, one stream) on config #3's table; for
each level: task counts per class (small <= 64 rows, medium <= 32k, big),
the largest medium / big task, and the device ms of the small / medium / big
split kernels and of partition + next-level bookkeeping."""
import sys
import time
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
forest._LEVEL_LOG = []
t0 = time.perf_counter()
forest.RandomForestRegressor(k, max_depth=16, random_state=0, trees_per_batch=k,
                             concurrent=False).fit(X, y)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tot = {"small_ms": 0.0, "med_ms": 0.0, "big_ms": 0.0, "part_next_ms": 0.0}
print(f"{'d':>2} {'small':>7} {'med':>6} {'big':>4} {'maxmed':>7} {'maxbig':>7} "
      f"{'s_ms':>7} {'m_ms':>7} {'b_ms':>7} {'pn_ms':>7}")
for r in forest._LEVEL_LOG:
    print(f"{r['depth']:2d} {r['n_small']:7d} {r['n_med']:6d} {r['n_big']:4d} {r['max_med']:7d} "
          f"{r['max_big']:7d} {r['small_ms']:7.2f} {r['med_ms']:7.2f} {r['big_ms']:7.2f} "
          f"{r['part_next_ms']:7.2f}")
    for key in tot:
        tot[key] += r[key]
print("total", {k_: round(v, 2) for k_, v in tot.items()}, f"wall {wall * 1e3:.0f} ms ({k} trees)")
