"""trainer.canonical_rows == the reference's canonical row order
(training.py:82-91: pandas sort_values by every feature then the target,
kind="mergesort") on tie-heavy frames, -0.0 / 0.0 mixes and duplicate rows."""

import numpy as np
import pandas as pd

from paper_2305_01886_b200.trainer import canonical_rows


def _reference(X, y, manifest):
    frame = pd.DataFrame(np.asarray(X, dtype=float), columns=list(manifest))
    frame["__target__"] = np.asarray(y, dtype=float)
    frame = frame.sort_values(by=list(manifest) + ["__target__"], kind="mergesort")
    return frame[list(manifest)].to_numpy(dtype=float), frame["__target__"].to_numpy(dtype=float)


def test_canonical_rows_match_pandas_stable_lexsort():
    rng = np.random.default_rng(0)
    for trial in range(400):
        n, F = int(rng.integers(1, 300)), int(rng.integers(1, 7))
        X = rng.integers(0, int(rng.integers(1, 5)), (n, F)).astype(float)
        if trial % 3 == 0:
            X[rng.random((n, F)) < 0.3] = -0.0
        if trial % 5 == 0:
            X[:, 0] = rng.random(n)
        if trial % 7 == 0:
            X[:, -1] = rng.normal(size=n)
        y = rng.integers(0, 3, n).astype(float) + (rng.random(n) < 0.5) * 0.5
        y[rng.random(n) < 0.2] = -0.0
        man = [f"c{i}" for i in range(F)]
        a, b = _reference(X, y, man), canonical_rows(X, y, man)
        assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64)), trial
        assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64)), trial
