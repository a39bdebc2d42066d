"""A/B a K5 build knob for identical trees: `save PATH` fits a forest (and a
boosted model) and stores every tree array; `check PATH` fits again with the
current build and asserts the arrays are identical.  Tuning aid.

    GK_NVCC_EXTRA=-DGK_SMALL_RANK=0 python -c '...build(force=True)'; python tools/k5_ab.py save /tmp/a.npz
    python -c '...build(force=True)'; python tools/k5_ab.py check /tmp/a.npz"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402

from bench import rf_table  # noqa: E402
from paper_2305_01886_b200.boosting import GradientBoostingRegressor  # noqa: E402
from paper_2305_01886_b200.forest import RandomForestRegressor  # noqa: E402

FIELDS = ("children_left", "children_right", "feature", "threshold", "value", "impurity",
          "n_node_samples", "weighted_n_node_samples")


def arrays():
    X, y = rf_table(300_000)
    out = {}
    rf = RandomForestRegressor(12, max_depth=None, random_state=5).fit(X, y)
    gb = GradientBoostingRegressor(8, learning_rate=0.1, max_depth=5, random_state=0).fit(X, y)
    trees = [e.tree_ for e in rf.estimators_] + [e[0].tree_ for e in gb.estimators_]
    for k, t in enumerate(trees):
        for f in FIELDS:
            out[f"{k}_{f}"] = getattr(t, f)
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    got = arrays()
    if mode == "save":
        np.savez(path, **got)
        print(f"saved {len(got)} arrays")
    else:
        want = np.load(path)
        bad = [k for k in want.files if not np.array_equal(want[k], got[k])]
        print(f"checked {len(want.files)} arrays, {len(bad)} differ {bad[:5]}")
        sys.exit(1 if bad else 0)
