"""Time the GPU random-forest fit on BASELINE config #3's table shape.

    python tools/rf_fit_bench.py [--rows 1000000] [--trees 32] [--depth 16] [--batch 32]

X [rows x 64] ~ U[0,1) with 8 integer columns, y = 30 + 40 x0 + 20 x1^2 +
12 [x2 > 0.5] + 60 x3 + N(0,1)."""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402


def table(rows, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.random((rows, 64))
    X[:, 56:] = np.floor(X[:, 56:] * 20)
    y = (30 + 40 * X[:, 0] + 20 * X[:, 1] ** 2 + 12 * (X[:, 2] > 0.5) + 0.003 * 20000 * X[:, 3]
         + rng.normal(0, 1, rows))
    return X, y


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--trees", type=int, default=32)
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    import torch

    from paper_2305_01886_b200.forest import RandomForestRegressor

    X, y = table(a.rows)
    Xs = (X - X.min(0)) / (X.max(0) - X.min(0))
    RandomForestRegressor(2, max_depth=4, random_state=0).fit(Xs[:5000], y[:5000])  # warm-up
    torch.cuda.synchronize()
    prof = None
    if a.profile:
        import cProfile

        prof = cProfile.Profile()
        prof.enable()
    for _ in range(a.repeat):
        t0 = time.perf_counter()
        m = RandomForestRegressor(a.trees, max_depth=a.depth, random_state=0,
                                  trees_per_batch=a.batch, streams=a.streams).fit(Xs, y)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if a.repeat > 1:
            print(f"fit {dt:.3f} s ({a.trees} trees, batch {a.batch}, streams {a.streams})")
    if prof is not None:
        import pstats

        prof.disable()
        pstats.Stats(prof).sort_stats("tottime").print_stats(18)
    nodes = np.mean([e.tree_.node_count for e in m.estimators_])
    p = m.predict(Xs[:100000])
    r2 = 1 - np.mean((p - y[:100000]) ** 2) / np.var(y[:100000])
    print(json.dumps({"rows": a.rows, "trees": a.trees, "depth": a.depth, "fit_s": dt,
                      "s_per_tree": dt / a.trees, "nodes_per_tree": nodes, "train_r2": r2}))


if __name__ == "__main__":
    main()
