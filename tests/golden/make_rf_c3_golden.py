"""Golden: the REFERENCE trainer's random forest at config #3's shape.

Runs ``gpukalc_trainer.train(ds, "random_forest", n_estimators=32,
max_depth=16, seed=0)`` (training.py:94-160, scikit-learn's
RandomForestRegressor behind ``_make_model``, training.py:73-76) on a
200,000 x 64 table drawn from config #3's distribution
(``workloads.config3_table``: 56 continuous columns with ~200k distinct values
each + 8 integer columns) and records each fold's R^2 / RMSE / MAE plus the
fold's MAPE, computed from the very predictions the reference made (the
estimator is wrapped only to keep a copy of ``predict``'s output; the forest,
the folds and the scaling are the reference's).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_rf_c3_golden.py      # ~10 min on 8 cores

Output: tests/golden/trainer_rf_c3.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path[:0] = [str(REF / "src"), str(REF / "trainer" / "src"), str(ROOT)]

ROWS, TREES, DEPTH, SEED, FRAME_SEED = 200_000, 32, 16, 0, 3


def main():
    import joblib
    import pandas as pd
    import sklearn
    from gpukalc_trainer import training
    from gpukalc_trainer.dataset import Dataset
    from sklearn.ensemble import RandomForestRegressor

    from paper_2305_01886_b200.workloads import config3_table

    X, y = config3_table(ROWS, FRAME_SEED)
    names = [f"f{i:02d}" for i in range(X.shape[1])]
    ds = Dataset(X=pd.DataFrame(X, columns=names), y=pd.Series(y, name="power_w"),
                 provenance=pd.DataFrame({"kernel": [f"r{i}" for i in range(ROWS)]}))

    preds = []

    class Recording(RandomForestRegressor):
        def predict(self, X):
            p = super().predict(X)
            preds.append(p)
            return p

    orig = training._make_model

    def make(family, n_estimators, learning_rate, max_depth, seed):
        m = orig(family, n_estimators, learning_rate, max_depth, seed)
        return Recording(**m.get_params())

    training._make_model = make
    t0 = time.time()
    # n_jobs only spreads trees over processes; the forest is identical (seeded per tree)
    with joblib.parallel_config(n_jobs=-1):
        res = training.train(ds, "random_forest", n_estimators=TREES, max_depth=DEPTH, seed=SEED)
    dt = time.time() - t0
    training._make_model = orig

    from sklearn.model_selection import KFold

    mapes = []
    for (tr, te), p in zip(KFold(5, shuffle=True, random_state=SEED).split(res.X), preds):
        yt = res.y[te]
        mapes.append(float(np.mean(np.abs((yt - p) / yt)) * 100))
    out = {
        "n_rows": ROWS, "frame_seed": FRAME_SEED, "n_estimators": TREES, "max_depth": DEPTH,
        "seed": SEED, "generator": "paper_2305_01886_b200.workloads.config3_table",
        "folds": [m.as_dict() for m in res.fold_metrics], "mean": res.mean_metrics.as_dict(),
        "fold_mape_pct": mapes, "mean_mape_pct": float(np.mean(mapes)),
        "final_nodes_per_tree": float(np.mean([e.tree_.node_count for e in res.model.estimators_])),
        "sklearn_version": sklearn.__version__, "reference_train_s": dt,
    }
    (HERE / "trainer_rf_c3.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out["mean"]), out["mean_mape_pct"], f"{dt:.0f} s")


if __name__ == "__main__":
    main()
